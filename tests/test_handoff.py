"""KV hand-off protocol between two processes (gloo, world_size 2, CPU): the
decode side receives exactly the prefill side's pages, into its own page ids,
with the KvHandle fields preserved (domain.py:96-113)."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_02599_b200.handoff import page_runs, recv_kv, recv_kv_async, send_kv, send_kv_async
from paper_2603_02599_b200.kvpool import KvPool, PageAllocator
from paper_2603_02599_b200.spec import TINY
from paper_2603_02599_b200.sun_types import KvHandle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        pool = KvPool(TINY, 24, "cpu")
        g = torch.Generator().manual_seed(100 + rank)
        pool.tensor.copy_(torch.randn(pool.tensor.shape, generator=g).to(torch.bfloat16))
        alloc = PageAllocator(pool.num_pages)
        if rank == 0:  # prefill side: two requests, scattered and contiguous pages
            out = []
            for rid, pages in ((7, [5, 2, 9]), (8, [11, 12, 13, 14])):
                h = KvHandle(request_id=rid, resident_tokens=len(pages) * 16 - 3, bytes_per_token=TINY.kv_bytes_per_token,
                             pages=pages, model_id=rid % 2)
                send_kv(h, pool, 1)
                out.append(pool.tensor[pages].float().numpy().copy())  # numpy: no fd sharing across exit
            q.put(("sent", out))
        else:  # decode side
            alloc.alloc(3)  # pool partly in use already
            got = []
            for _ in range(2):
                h = recv_kv(pool, alloc, 0)
                got.append((h.request_id, h.resident_tokens, h.bytes_per_token, h.model_id, list(h.pages),
                            pool.tensor[h.pages].float().numpy().copy()))
            q.put(("recv", got, alloc.free_pages))
    finally:
        dist.destroy_process_group()


def test_kv_handoff_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((m[0], m[1:]) for m in (q.get(timeout=120), q.get(timeout=120)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sent = res["sent"][0]
    got, free_after = res["recv"]
    assert [g[0] for g in got] == [7, 8]
    assert got[0][1] == 3 * 16 - 3 and got[0][2] == TINY.kv_bytes_per_token and got[0][3] == 1
    for (payload, g) in zip(sent, got):
        assert (payload == g[5]).all()
        assert len(page_runs(g[4])) == 1  # landed in a contiguous run of the receiver's pool
    assert free_after == 24 - 3 - 3 - 4


def test_page_runs():
    assert page_runs([3, 4, 5, 9, 10, 2]) == [(3, 3), (9, 2), (2, 1)]
    assert page_runs([]) == []


def _async_worker(rank, port, q):
    """Async hand-off overlapped with decode work: the receiver posts the payload
    receives for two requests, keeps 'stepping' (CPU work standing in for decode
    steps on other pages), and only then waits and admits."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        pool = KvPool(TINY, 24, "cpu")
        g = torch.Generator().manual_seed(200 + rank)
        pool.tensor.copy_(torch.randn(pool.tensor.shape, generator=g).to(torch.bfloat16))
        alloc = PageAllocator(pool.num_pages)
        if rank == 0:
            sends, out = [], []
            for rid, pages in ((3, [1, 7]), (4, [8, 9, 10])):
                h = KvHandle(request_id=rid, resident_tokens=len(pages) * 16, bytes_per_token=TINY.kv_bytes_per_token,
                             pages=pages, model_id=rid)
                sends.append(send_kv_async(h, pool, 1))
                out.append(pool.tensor[pages].float().numpy().copy())  # numpy: no fd sharing across exit
            for s in sends:
                s.wait()
            q.put(("sent", out))
        else:
            alloc.alloc(5)
            pending = [recv_kv_async(pool, alloc, 0) for _ in range(2)]
            busy = pool.tensor[:5].float().sum().item()  # decode work on resident pages meanwhile
            got = []
            for p_ in pending:
                h = p_.wait()
                got.append((h.request_id, list(h.pages), pool.tensor[h.pages].float().numpy().copy()))
            q.put(("recv", got, busy))
    finally:
        dist.destroy_process_group()


def test_kv_handoff_async_overlap_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_async_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((m[0], m[1:]) for m in (q.get(timeout=120), q.get(timeout=120)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sent = res["sent"][0]
    got = res["recv"][0]
    assert [g[0] for g in got] == [3, 4]
    for payload, g in zip(sent, got):
        assert (payload == g[2]).all()
        assert len(page_runs(g[1])) == 1 and min(g[1]) >= 5  # fresh pages, one contiguous run each


def _peer_worker(rank, port, q, shared):
    """Peer-copy hand-off protocol (handoff.peer_send_kv / peer_recv_kv): the decode
    rank reserves pages and answers their ids, the prefill rank writes its pages
    straight into them (here a shared-memory CPU tensor stands in for the decode
    GPU's IPC-mapped pool and the copy engine), then reports them landed."""
    from paper_2603_02599_b200.handoff import peer_recv_kv, peer_send_kv

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        if rank == 0:  # prefill side
            pool = KvPool(TINY, 16, "cpu")
            g = torch.Generator().manual_seed(300)
            pool.tensor.copy_(torch.randn(pool.tensor.shape, generator=g).to(torch.bfloat16))

            def copier(src, src_pages, remote, dst_pages):
                remote[dst_pages] = src.tensor[src_pages]

            out = []
            for rid, pages in ((21, [3, 4, 5]), (22, [9, 1])):
                h = KvHandle(request_id=rid, resident_tokens=len(pages) * 16 - 1,
                             bytes_per_token=TINY.kv_bytes_per_token, pages=pages, model_id=rid % 3)
                dst = peer_send_kv(h, pool, shared, 1, copier=copier)
                out.append((dst, pool.tensor[pages].float().numpy().copy()))
            q.put(("sent", out))
        else:  # decode side: owns `shared`
            alloc = PageAllocator(shared.shape[0])
            alloc.alloc(2)
            got = []
            for _ in range(2):
                p_ = peer_recv_kv(alloc, 0)
                h = p_.wait()
                got.append((h.request_id, h.resident_tokens, h.model_id, list(h.pages),
                            shared[h.pages].float().numpy().copy()))
            q.put(("recv", got))
    finally:
        dist.destroy_process_group()


def test_kv_handoff_peer_copy_protocol_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    shared = torch.zeros((20,) + tuple(KvPool(TINY, 1, "cpu").tensor.shape[1:]), dtype=torch.bfloat16).share_memory_()
    procs = [ctx.Process(target=_peer_worker, args=(r, port, q, shared)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((m[0], m[1:]) for m in (q.get(timeout=120), q.get(timeout=120)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sent, got = res["sent"][0], res["recv"][0]
    assert [g[0] for g in got] == [21, 22] and got[0][1] == 47 and got[1][2] == 1
    for (dst, payload), g in zip(sent, got):
        assert dst == g[3] and min(dst) >= 2 and len(page_runs(dst)) == 1
        assert (payload == g[4]).all()
