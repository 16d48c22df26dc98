"""B200Executor driven by the reference's own member objects (CPU, stub modules):
poolsim's ``_Member`` (engine.py:135-145) and ``KvHandle`` (domain.py:96-113, no
``pages`` field) work unchanged — the INTEGRATION.md §2 binding. The executor's real
GPU run is tests/test_serving_gpu.py."""
import torch

from paper_2603_02599_b200.executor import B200Executor
from paper_2603_02599_b200.kvpool import PageAllocator, pages_for


class _Req:  # poolsim.domain.Request's fields the executor reads
    def __init__(self, rid, model_id, isl, osl):
        self.id, self.model_id, self.isl, self.target_osl = rid, model_id, isl, osl


class _KvHandle:  # poolsim KvHandle: no pages field
    __slots__ = ("request_id", "resident_tokens", "bytes_per_token", "location")

    def __init__(self, rid):
        self.request_id, self.resident_tokens, self.bytes_per_token, self.location = rid, 0, 131072, 0


class _Member:  # poolsim engine._Member
    __slots__ = ("request", "kv", "reserved_bytes", "retire_at", "steps_done")

    def __init__(self, request, kv):
        self.request, self.kv = request, kv
        self.reserved_bytes = (request.isl + request.target_osl - 1) * kv.bytes_per_token
        self.retire_at, self.steps_done = -1, 0


class _Spec:
    vocab = 1000


class _Dec:  # records what the shared decode module is asked to do
    spec, max_batch, max_context = _Spec(), 16, 4096

    def __init__(self):
        self.calls = []

    def decode(self, tokens, positions, bt, graph=True):
        self.calls.append((tokens.tolist(), positions.tolist(), bt.tolist()))
        return (tokens + 1) % self.spec.vocab


class _Pre:
    def __init__(self, tag):
        self.tag, self.calls = tag, []

    def prefill(self, prompts, pages):
        self.calls.append((len(prompts[0]), list(pages[0])))
        return [self.tag * 100 + len(prompts[0])], [torch.zeros(4)]


def test_executor_with_reference_member_objects():
    dec, pres = _Dec(), {0: _Pre(1), 1: _Pre(2)}
    ex = B200Executor(dec, pres, PageAllocator(64), graph=False)
    ms = [_Member(_Req(7, 0, 40, 5), _KvHandle(7)), _Member(_Req(9, 1, 17, 3), _KvHandle(9))]
    for m in ms:
        assert ex.fits(m, 0) == "ok"
        ex.admit(m)
    assert [len(c[1]) for c in pres[0].calls + pres[1].calls] == [pages_for(44), pages_for(19)]
    out = ex.step(ms)
    tok, pos, bt = dec.calls[-1]
    assert tok == [140, 217] and pos == [40, 17] and out == [141, 218]
    assert bt[0][:pages_for(44)] == ex.pages[7] and bt[1][:pages_for(19)] == ex.pages[9]
    for m in ms:
        m.steps_done += 1
    ex.step(ms)
    assert dec.calls[-1][0] == [141, 218] and dec.calls[-1][1] == [41, 18]
    free0 = ex.alloc.free_pages
    ex.retire(ms[0])
    assert ex.alloc.free_pages == free0 + pages_for(44) and 7 not in ex.pages
