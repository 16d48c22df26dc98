"""Paged KV pool shared by every prefill module and the shared decode module.

Physical layout (one tensor per GPU, include/sun_b200.h SunKvPool):
    pool[page, layer, kv(0=K post-RoPE, 1=V), kv_head, slot(16), head_dim]  bf16
A page holds 16 consecutive tokens of ONE sequence for all layers, so a
sequence's cache is a list of page ids (its block-table row) and a hand-off
moves whole pages. The pool is decoder-compatible by construction: every task
prefill module writes the same geometry the frozen decoder reads
(Eq. 4 C_<=t = C_X || C_y<=t).

``PageAllocator`` is the memory side of the reference's admission control:
the reference reserves a member's final footprint (isl + osl - 1) * kvb at
admission (engine.py:135-145, 405-419); here that reservation is a page count.
"""
from __future__ import annotations

import torch

from .errors import OverCapacity
from .spec import DecoderSpec

PAGE_TOKENS = 16


def pages_for(tokens: int) -> int:
    return (tokens + PAGE_TOKENS - 1) // PAGE_TOKENS


class KvPool:
    def __init__(self, spec: DecoderSpec, num_pages: int, device: torch.device | str):
        self.spec = spec
        self.num_pages = int(num_pages)
        self.tensor = torch.empty(self.num_pages, spec.n_layers, 2, spec.n_kv_heads, PAGE_TOKENS, spec.head_dim,
                                  dtype=torch.bfloat16, device=device)
        self.page_bytes = spec.n_layers * 2 * spec.n_kv_heads * PAGE_TOKENS * spec.head_dim * 2

    def struct(self):
        """The C ``SunKvPool`` (include/sun_b200.h): base, size and the KV geometry every
        decoder over this pool must match (SUN_ERR_MIXED_DECODER otherwise)."""
        from . import _lib

        dev = self.tensor.device
        return _lib.SunKvPool(self.tensor.data_ptr(), self.num_pages, self.spec.n_layers, self.spec.n_kv_heads,
                              self.spec.head_dim, PAGE_TOKENS, float(self.spec.rope_theta),
                              dev.index if dev.type == "cuda" and dev.index is not None else 0)

    @classmethod
    def for_bytes(cls, spec: DecoderSpec, nbytes: int, device) -> "KvPool":
        page_bytes = spec.n_layers * 2 * spec.n_kv_heads * PAGE_TOKENS * spec.head_dim * 2
        return cls(spec, max(1, nbytes // page_bytes), device)

    def fill_random_(self, seed: int, std: float = 1.0) -> None:
        """Seeded on-device KV fill (bench staging; cost excluded from timing)."""
        g = torch.Generator(device=self.tensor.device).manual_seed(seed)
        flat = self.tensor.view(self.num_pages, -1)
        for i in range(0, self.num_pages, 256):
            blk = flat[i:i + 256]
            blk.copy_((torch.randn(blk.shape, generator=g, device=blk.device) * std).to(torch.bfloat16))


class PageAllocator:
    """LIFO free list of page ids with all-or-nothing allocation."""

    def __init__(self, num_pages: int):
        self.num_pages = num_pages
        self._free = list(range(num_pages - 1, -1, -1))

    @property
    def free_pages(self) -> int:
        return len(self._free)

    def alloc(self, n: int) -> list[int]:
        if n > len(self._free):
            raise OverCapacity(f"need {n} KV pages, {len(self._free)} free")
        out = [self._free.pop() for _ in range(n)]
        return out

    def alloc_contiguous(self, n: int) -> list[int]:
        """n consecutive page ids if such a run is free (so a hand-off payload can
        land in place), otherwise any n pages."""
        if n > len(self._free):
            raise OverCapacity(f"need {n} KV pages, {len(self._free)} free")
        free = sorted(self._free)
        run_start, run_len = free[0], 1
        for prev, p in zip(free, free[1:]):
            if run_len >= n:
                break
            if p == prev + 1:
                run_len += 1
            else:
                run_start, run_len = p, 1
        if run_len >= n:
            pages = list(range(run_start, run_start + n))
            taken = set(pages)
            self._free = [p for p in self._free if p not in taken]
            return pages
        return self.alloc(n)

    def free(self, pages: list[int]) -> None:
        self._free.extend(reversed(pages))
