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


# --------------------------------------------------------------------------- peer copy (K8 over the copy engines)
# The decode worker exports its pool once (CUDA IPC, sun_kv_pool_export); each
# prefill worker maps it (sun_kv_pool_import) and, per request, copies the
# request's pages straight into the pages the decode worker reserved
# (sun_kv_handoff_copy: cudaMemcpyAsync per consecutive run — NVLink 5 between
# GPUs, HBM within one). Only small control messages cross torch.distributed
# (gloo is enough: no NCCL kernel takes SMs from the decode step, whose persistent
# layer chain needs every SM co-resident).
PEER_HDR = 5  # request id, resident tokens, bytes/token, page count, task id


def export_pool(pool: KvPool) -> torch.Tensor:
    """uint8 bytes of the pool's SunKvPoolHandle (send them to the prefill workers)."""
    import ctypes

    from . import _lib

    h = _lib.SunKvPoolHandle()
    st = pool.struct()
    _lib.check(_lib.load().sun_kv_pool_export(ctypes.byref(st), ctypes.byref(h)), "sun_kv_pool_export")
    return torch.frombuffer(bytearray(bytes(h)), dtype=torch.uint8).clone()


class RemotePool:
    """A decode worker's pool mapped into this (prefill) process."""

    def __init__(self, handle_bytes: torch.Tensor):
        import ctypes

        from . import _lib

        self._lib = _lib
        h = _lib.SunKvPoolHandle.from_buffer_copy(bytes(handle_bytes.cpu().numpy().tobytes()))
        self.struct = _lib.SunKvPool()
        _lib.check(_lib.load().sun_kv_pool_import(ctypes.byref(h), ctypes.byref(self.struct)), "sun_kv_pool_import")
        self.num_pages = self.struct.num_pages

    def close(self) -> None:
        import ctypes

        if self.struct.base:
            self._lib.check(self._lib.load().sun_kv_pool_close(ctypes.byref(self.struct)), "sun_kv_pool_close")


def copy_pages(src: KvPool, src_pages: list[int], dst_struct, dst_pages: list[int], stream=None) -> None:
    """Enqueue the copy of src_pages (local pool) into dst_pages of a pool (local or
    imported) on ``stream`` (default: the current stream); geometry-checked by the
    library (MixedDecoderError for pools of different KV geometry)."""
    import ctypes

    from . import _lib

    n = len(src_pages)
    if n != len(dst_pages):
        raise ValueError("source and destination page lists differ in length")
    sp = (ctypes.c_int32 * max(n, 1))(*src_pages)
    dp = (ctypes.c_int32 * max(n, 1))(*dst_pages)
    st = (stream or torch.cuda.current_stream()).cuda_stream
    s = src.struct()
    _lib.check(_lib.load().sun_kv_handoff_copy(ctypes.byref(s), sp, ctypes.byref(dst_struct), dp, n, st),
               "sun_kv_handoff_copy")


def peer_send_kv(handle: KvHandle, pool: KvPool, remote, dst: int, group=None, copier=None, stream=None,
                 timing: list | None = None) -> list[int]:
    """Prefill side of one hand-off: header -> the decode rank reserves pages and
    answers their ids -> copy the pages into them -> "landed". Returns the
    destination page ids. ``copier(src_pool, src_pages, remote, dst_pages)`` replaces
    the copy-engine copy (tests without a GPU); ``timing`` collects the device ms
    of each copy (CUDA events around it on the copy stream)."""
    hdr = torch.tensor([handle.request_id, handle.resident_tokens, handle.bytes_per_token, len(handle.pages),
                        handle.model_id], dtype=torch.int64)
    dist.send(hdr, dst, group=group)
    pages_t = torch.empty(len(handle.pages), dtype=torch.int64)
    if handle.pages:
        dist.recv(pages_t, dst, group=group)
    dst_pages = [int(p) for p in pages_t.tolist()]
    if handle.pages:
        if copier is not None:
            copier(pool, handle.pages, remote, dst_pages)
        else:
            s = stream or torch.cuda.current_stream()
            if timing is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
            copy_pages(pool, handle.pages, remote.struct, dst_pages, s)
            if timing is not None:
                e1.record(s)
            s.synchronize()  # the pages are in the decode worker's HBM before "landed"
            if timing is not None:
                timing.append(e0.elapsed_time(e1))
    dist.send(torch.tensor([handle.request_id], dtype=torch.int64), dst, group=group)
    return dst_pages


class PendingPeerKv:
    """Decode side of a peer-copy hand-off in flight: pages reserved, the prefill
    worker is copying into them; ``wait()`` returns the KvHandle once it reports
    the copy landed (the decode worker keeps stepping meanwhile)."""

    def __init__(self, hdr: list[int], pages: list[int], src: int, group):
        self.hdr, self.pages, self.src, self.group = hdr, pages, src, group
        self._done = torch.empty(1, dtype=torch.int64)
        self._work = dist.irecv(self._done, src, group=group)

    def ready(self) -> bool:
        return self._work.is_completed()

    def wait(self) -> KvHandle:
        self._work.wait()
        rid, tokens, bpt, _, model_id = self.hdr
        if int(self._done.item()) != rid:
            raise RuntimeError(f"hand-off of request {rid} completed as {int(self._done.item())}")
        return KvHandle(request_id=rid, resident_tokens=tokens, bytes_per_token=bpt, location=IN_TRANSIT,
                        pages=list(self.pages), model_id=model_id)


def peer_recv_kv(alloc: PageAllocator, src: int, group=None) -> PendingPeerKv:
    """Decode side: take the header, reserve the final pages (a contiguous run when
    possible: one copy), answer their ids and return while the copy proceeds."""
    hdr_t = torch.empty(PEER_HDR, dtype=torch.int64)
    dist.recv(hdr_t, src, group=group)
    hdr = [int(x) for x in hdr_t.tolist()]
    pages = alloc.alloc_contiguous(hdr[3]) if hdr[3] else []
    if pages:
        dist.send(torch.tensor(pages, dtype=torch.int64), src, group=group)
    return PendingPeerKv(hdr, pages, src, group)
