"""Real execution of scheduled shared-decode steps on one B200.

``B200Executor`` plugs into ``scheduler.ServingLoop`` as a decode worker's
``StepExecutor``: at admission it reserves the member's final KV footprint in
pages (the physical form of the reference's ``(isl + osl - 1) * kvb``
reservation, engine.py:135-145) and has the request's *task* prefill module
fill the prompt KV into those pages (Eq. 2); every scheduled step runs
the frozen shared decode module over the batch's block tables (Eq. 3); at
retirement the pages go back to the allocator (the reference's ``_free_kv``,
engine.py:360-365).

Members only need the reference's ``_Member`` fields (engine.py:135-145): ``request``
(``id``, ``model_id``, ``isl``, ``target_osl``) and ``steps_done``. The physical pages of a
request are kept here, keyed by request id, and mirrored onto ``member.kv.pages`` when the
handle has that field (this package's ``KvHandle``) — so poolsim's own ``_Member`` /
``KvHandle`` objects drive it unchanged (tests/test_executor.py).
"""
from __future__ import annotations

import random
from typing import Callable

import torch

from .kvpool import PageAllocator, pages_for
from .modules import PrefillModule, SharedDecodeModule
from .scheduler import Member


def synthetic_prompt(request_id: int, isl: int, vocab: int, seed: int = 1234) -> list[int]:
    """Deterministic prompt tokens for a request id (synthetic workload)."""
    r = random.Random(seed * 1_000_003 + request_id)
    return [r.randrange(vocab) for _ in range(isl)]


class B200Executor:
    def __init__(self, decoder: SharedDecodeModule, prefills: dict[int, PrefillModule], allocator: PageAllocator,
                 prompt_of: Callable[[int, int], list[int]] | None = None, graph: bool = True,
                 keep_logits: bool = False):
        self.dec = decoder
        self.prefills = prefills
        self.alloc = allocator
        self.prompt_of = prompt_of or (lambda rid, isl: synthetic_prompt(rid, isl, decoder.spec.vocab))
        self.graph = graph
        self.last_token: dict[int, int] = {}
        self.first_token: dict[int, int] = {}
        self.pages: dict[int, list[int]] = {}  # request id -> its pages in the shared pool
        self.steps_run = 0
        self.keep_logits = keep_logits
        self.logits: dict[int, list] = {}  # request id -> [first-token logits, step logits...] (testing)

    def fits(self, m: Member, batch: int) -> str:
        """Physical admission (scheduler.StepExecutor.fits): the final-footprint pages
        and the decoder's context / batch limits of this GPU."""
        r = m.request
        need = pages_for(r.isl + r.target_osl - 1)
        if need > self.alloc.num_pages or r.isl + r.target_osl - 1 > self.dec.max_context:
            return "never"
        if batch >= self.dec.max_batch or need > self.alloc.free_pages:
            return "never" if batch == 0 else "wait"
        return "ok"

    def admit(self, m: Member) -> None:
        r = m.request
        pages = self.alloc.alloc(pages_for(r.isl + r.target_osl - 1))
        self.pages[r.id] = pages
        if hasattr(m.kv, "pages"):
            m.kv.pages = pages
        pre = self.prefills[r.model_id]
        first, lg = pre.prefill([self.prompt_of(r.id, r.isl)], [pages])
        if self.keep_logits:
            self.logits[r.id] = [lg[0].cpu()]
        self.first_token[r.id] = first[0]
        self.last_token[r.id] = first[0]

    def step(self, members: list[Member]) -> list[int]:
        b = len(members)
        tokens = torch.tensor([self.last_token[m.request.id] for m in members], dtype=torch.int32)
        positions = torch.tensor([m.request.isl + m.steps_done for m in members], dtype=torch.int32)
        rows = [self.pages[m.request.id] for m in members]
        width = max(len(p) for p in rows)
        bt = torch.zeros(b, width, dtype=torch.int32)
        for i, p in enumerate(rows):
            bt[i, :len(p)] = torch.tensor(p, dtype=torch.int32)
        if torch.cuda.is_available():
            tokens, positions, bt = tokens.pin_memory(), positions.pin_memory(), bt.pin_memory()
        nxt = self.dec.decode(tokens, positions, bt, graph=self.graph).cpu()
        out = [int(x) for x in nxt]
        lg = self.dec.logits[:b].cpu() if self.keep_logits else None
        for i, (m, t) in enumerate(zip(members, out)):
            self.last_token[m.request.id] = t
            if lg is not None:
                self.logits[m.request.id].append(lg[i].clone())
        self.steps_run += 1
        return out

    def retire(self, m: Member) -> None:
        self.alloc.free(self.pages.pop(m.request.id))
        if hasattr(m.kv, "pages"):
            m.kv.pages = []
