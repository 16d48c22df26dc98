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


class PendingSend:
    """In-flight asynchronous send (keeps the payload alive until ``wait``)."""

    def __init__(self, works: list, payload: torch.Tensor | None):
        self.works, self.payload = works, payload

    def wait(self) -> None:
        for w in self.works:
            w.wait()
        self.payload = None


def send_kv_async(handle: KvHandle, pool: KvPool, dst: int, group=None) -> PendingSend:
    """Non-blocking ``send_kv``: the transfer proceeds (NCCL: on its own stream)
    while the caller keeps stepping; ``wait()`` before the pages are freed."""
    dev = pool.tensor.device
    hdr = torch.tensor([handle.request_id, handle.resident_tokens, handle.bytes_per_token, len(handle.pages),
                        handle.model_id], dtype=torch.int64, device=dev)
    works = [dist.isend(hdr, dst, group=group)]
    payload = None
    if handle.pages:
        payload = _payload(pool, handle.pages).contiguous()
        works.append(dist.isend(payload, dst, group=group))
    return PendingSend(works, payload if payload is not None else hdr)


class PendingKv:
    """A hand-off whose header has arrived and whose page payload is landing in
    reserved pages of the receiver's pool; ``wait()`` returns the KvHandle. The
    decode worker keeps stepping meanwhile (the request is only admitted — its
    pages only read — after ``wait``), which is the reference's transfer window
    (engine.py:350-392) overlapped with decode for real."""

    def __init__(self, pool: KvPool, hdr: list[int], pages: list[int], work, buf: torch.Tensor | None):
        self.pool, self.hdr, self.pages, self.work, self.buf = pool, hdr, pages, work, buf

    def wait(self) -> KvHandle:
        if self.work is not None:
            self.work.wait()
            self.work = None
        if self.buf is not None:
            idx = torch.tensor(self.pages, dtype=torch.long, device=self.pool.tensor.device)
            self.pool.tensor.index_copy_(0, idx, self.buf)
            self.buf = None
        rid, tokens, bpt, _, model_id = self.hdr
        return KvHandle(request_id=rid, resident_tokens=tokens, bytes_per_token=bpt, location=IN_TRANSIT,
                        pages=list(self.pages), model_id=model_id)


def recv_kv_async(pool: KvPool, alloc: PageAllocator, src: int, group=None) -> PendingKv:
    """Receive the (small) header, reserve pages (a contiguous run when possible),
    post the payload receive straight into them and return without waiting."""
    dev = pool.tensor.device
    hdr_t = torch.empty(HEADER_LEN, dtype=torch.int64, device=dev)
    dist.recv(hdr_t, src, group=group)
    hdr = [int(x) for x in hdr_t.tolist()]
    n_pages = hdr[3]
    pages = alloc.alloc_contiguous(n_pages) if n_pages else []
    work, buf = None, None
    if n_pages:
        runs = page_runs(pages)
        if len(runs) == 1:
            a, n = runs[0]
            work = dist.irecv(pool.tensor[a:a + n], src, group=group)
        else:
            buf = torch.empty((n_pages,) + tuple(pool.tensor.shape[1:]), dtype=pool.tensor.dtype, device=dev)
            work = dist.irecv(buf, src, group=group)
    return PendingKv(pool, hdr, pages, work, buf)


def handoff_bytes(handle: KvHandle, pool: KvPool) -> int:
    return len(handle.pages) * pool.page_bytes
