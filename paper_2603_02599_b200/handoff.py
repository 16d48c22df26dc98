"""Prefill -> decode KV hand-off between workers (one process per GPU).

The reference models the hand-off as ``latency + tokens * kvb / bandwidth``
(costmodel.py:148-155) of the ``KvHandle`` created at prefill completion
(engine.py:330-350). Here the handle's pages move for real: the sender ships
a small header (request id, resident tokens, bytes/token, page count, task id)
then the page payload; the receiver reserves pages in its own pool (a
contiguous run when possible, so the payload lands in place) and returns a
``KvHandle`` whose ``pages`` index its pool. Transport is torch.distributed
point-to-point — NCCL over NVLink 5 / NVSwitch on B200 boxes, gloo on CPU
(tests/test_handoff.py). No collective is involved in the decode step itself.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .kvpool import KvPool, PageAllocator
from .sun_types import IN_TRANSIT, KvHandle

HEADER_LEN = 5


def page_runs(pages: list[int]) -> list[tuple[int, int]]:
    """Maximal runs of consecutive page ids: [(start, length), ...]."""
    runs: list[tuple[int, int]] = []
    for p in pages:
        if runs and runs[-1][0] + runs[-1][1] == p:
            runs[-1] = (runs[-1][0], runs[-1][1] + 1)
        else:
            runs.append((p, 1))
    return runs


def _payload(pool: KvPool, pages: list[int]) -> torch.Tensor:
    runs = page_runs(pages)
    if len(runs) == 1:
        a, n = runs[0]
        return pool.tensor[a:a + n]
    idx = torch.tensor(pages, dtype=torch.long, device=pool.tensor.device)
    return pool.tensor.index_select(0, idx)


def send_kv(handle: KvHandle, pool: KvPool, dst: int, group=None) -> None:
    """Ship one request's KV pages to rank ``dst`` (blocking)."""
    dev = pool.tensor.device
    hdr = torch.tensor([handle.request_id, handle.resident_tokens, handle.bytes_per_token, len(handle.pages),
                        handle.model_id], dtype=torch.int64, device=dev)
    dist.send(hdr, dst, group=group)
    if handle.pages:
        dist.send(_payload(pool, handle.pages).contiguous(), dst, group=group)


def recv_kv(pool: KvPool, alloc: PageAllocator, src: int, group=None) -> KvHandle:
    """Receive one request's KV from rank ``src`` into freshly reserved pages."""
    dev = pool.tensor.device
    hdr = torch.empty(HEADER_LEN, dtype=torch.int64, device=dev)
    dist.recv(hdr, src, group=group)
    rid, tokens, bpt, n_pages, model_id = (int(x) for x in hdr.tolist())
    pages = alloc.alloc_contiguous(n_pages) if n_pages else []
    if n_pages:
        runs = page_runs(pages)
        if len(runs) == 1:
            a, n = runs[0]
            dist.recv(pool.tensor[a:a + n], src, group=group)
        else:
            buf = torch.empty((n_pages,) + tuple(pool.tensor.shape[1:]), dtype=pool.tensor.dtype, device=dev)
            dist.recv(buf, src, group=group)
            pool.tensor.index_copy_(0, torch.tensor(pages, dtype=torch.long, device=dev), buf)
    return KvHandle(request_id=rid, resident_tokens=tokens, bytes_per_token=bpt, location=IN_TRANSIT, pages=pages,
                    model_id=model_id)


def handoff_bytes(handle: KvHandle, pool: KvPool) -> int:
    return len(handle.pages) * pool.page_bytes
