"""Prefill-module / decode-module split of SUN on the B200 (Eqs. 2-4).

``SharedDecodeModule`` is the frozen decode module D_θd: one ``sun_decode_step``
per step over a mixed-model batch (members prefilled by different task
modules), optionally replayed from a CUDA graph per (batch, split) bucket.
``PrefillModule`` is a task-specific P_θp^τ: it writes the prompt's KV into the
shared paged pool with the same kernels — token-parallel, up to ``max_batch``
prompt positions per step — and returns the first generated
token, as Eq. 2 specifies.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from .kvpool import PAGE_TOKENS, KvPool, pages_for
from .spec import DecoderSpec
from .weights import DeviceWeights


W4_CHAIN_MAX_BATCH = 128  # sun_capi.cu kW4ChainMaxBn: QSUN chain up to bn = 128
W4_GEMV_MAX_BATCH = 8  # sun_capi.cu kGemvMaxBatch: QSUN steps of <= 8 rows run the W4 GEMV


def uses_w4_gemv(weight_bits: int, batch: int, env: str | None = None) -> bool:
    """Whether a QSUN step runs the small-batch W4 GEMV launches (mirrors sun_capi.cu
    use_gemv; SUN_W4_GEMV=0 keeps the tcgen05 path)."""
    if env is None:
        env = os.environ.get("SUN_W4_GEMV")
    try:
        on = int(env) != 0 if env is not None else True
    except ValueError:  # atoi semantics
        on = False
    return weight_bits == 4 and on and batch <= W4_GEMV_MAX_BATCH


def uses_gemm_chain(weight_bits: int, distinct_rows: bool, env: str | None, batch: int = 1) -> bool:
    """Whether sun_decode_step runs the persistent layer GEMM chain (mirrors
    sun_capi.cu use_chain): decode batches by default (QSUN: 9..128 rows; at <= 8 rows the
    W4 GEMV's separate launches unless SUN_W4_GEMV_CHAIN=1), SUN_GEMM_CHAIN=0/1 forces."""
    if weight_bits == 4 and (batch + 15) // 16 * 16 > W4_CHAIN_MAX_BATCH:
        return False
    if uses_w4_gemv(weight_bits, batch) and os.environ.get("SUN_W4_GEMV_CHAIN", "0") in ("", "0"):
        return False  # the W4 GEMV's separate launches (its chain is opt-in)
    if env is not None:
        try:
            return int(env) == 1
        except ValueError:  # atoi semantics: not a number -> 0
            return False
    return distinct_rows


class _StepRunner:
    """Owns one C decoder (TMA descriptors + workspace) over a weight set."""

    # rows of a step are different sequences (SUN_STEP_DISTINCT_ROWS): true for the
    # decode batch, not for token-parallel prefill rows of one prompt
    distinct_rows = False

    def __init__(self, spec: DecoderSpec, weights: DeviceWeights, kv: KvPool, max_batch: int, max_context: int,
                 use_pdl: bool = True):
        self.spec, self.weights, self.kv = spec, weights, kv
        self.max_batch, self.max_context = int(max_batch), int(max_context)
        self.max_pages = pages_for(self.max_context)
        lib = _lib.load()
        self.dims = _lib.SunDecoderDims(
            vocab=spec.vocab, hidden=spec.hidden, n_layers=spec.n_layers, n_q_heads=spec.n_q_heads,
            n_kv_heads=spec.n_kv_heads, head_dim=spec.head_dim, ffn=spec.ffn, page_size=PAGE_TOKENS,
            max_context=self.max_context, weight_bits=spec.weight_bits, group_size=spec.group_size,
            qkv_bias=int(spec.qkv_bias), rms_eps=spec.rms_eps, rope_theta=spec.rope_theta)
        nb = ctypes.c_size_t()
        _lib.check(lib.sun_decoder_workspace_bytes(ctypes.byref(self.dims), self.max_batch, ctypes.byref(nb)),
                   "workspace sizing")
        dev = weights.device
        self.workspace = torch.zeros(nb.value, dtype=torch.uint8, device=dev)
        self._pool = kv.struct()
        h = ctypes.c_void_p()
        _lib.check(lib.sun_decoder_create(ctypes.byref(self.dims), ctypes.byref(weights.struct),
                                          ctypes.byref(self._pool), self.workspace.data_ptr(), self.workspace.numel(),
                                          self.max_batch, int(use_pdl), ctypes.byref(h)), "sun_decoder_create")
        self._h = h
        self._lib = lib
        import os as _os
        self.fused_combine = _os.environ.get("SUN_ATTN_FUSED_COMBINE", "0") == "1"
        flags = _lib.SUN_STEP_DISTINCT_ROWS if self.distinct_rows else 0
        chain = ctypes.c_int32()
        _lib.check(lib.sun_decoder_uses_chain(h, flags, ctypes.byref(chain)), "sun_decoder_uses_chain")
        self.gemm_chain = bool(chain.value)  # (the library also checks the grid fits this device)

    def status(self, clear: bool = True) -> int:
        """The decoder's device error word (SUN_STEP_ERR_* bits raised by the steps
        since the last clear; synchronises the current stream)."""
        v = ctypes.c_uint32()
        _lib.check(self._lib.sun_decoder_status(self._h, ctypes.byref(v), int(clear),
                                                torch.cuda.current_stream().cuda_stream), "sun_decoder_status")
        return v.value

    def check(self) -> None:
        """Raise ValueError if a step since the last check saw invalid inputs."""
        bits = self.status(clear=True)
        if bits:
            names = [n for b, n in ((_lib.SUN_STEP_ERR_TOKEN, "token outside the vocabulary"),
                                    (_lib.SUN_STEP_ERR_POSITION, "position outside [0, max_context)"),
                                    (_lib.SUN_STEP_ERR_PAGE, "block-table page outside the KV pool"),
                                    (_lib.SUN_STEP_ERR_NAN, "logits without a finite maximum")) if bits & b]
            raise ValueError("decode step inputs invalid: " + "; ".join(names))

    def validate_host(self, tokens: torch.Tensor, positions: torch.Tensor, block_tables: torch.Tensor) -> None:
        """Host-side bounds of a batch given in host memory (the device re-checks)."""
        if tokens.device.type != "cpu":
            return
        if tokens.numel() and (int(tokens.min()) < 0 or int(tokens.max()) >= self.spec.vocab):
            raise ValueError("token outside the vocabulary")
        if positions.numel() and (int(positions.min()) < 0 or int(positions.max()) >= self.max_context):
            raise ValueError(f"position outside [0, {self.max_context})")
        npg = (positions.to(torch.int64) // PAGE_TOKENS + 1).clamp(max=block_tables.shape[1])
        used = torch.arange(block_tables.shape[1])[None, :] < npg[:, None]
        pages = block_tables[used]
        if pages.numel() and (int(pages.min()) < 0 or int(pages.max()) >= self.kv.num_pages):
            raise ValueError("block-table page outside the KV pool")
        if int((positions.to(torch.int64) // PAGE_TOKENS).max()) >= block_tables.shape[1]:
            raise ValueError("block table shorter than a position needs")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.sun_decoder_destroy(h)
            self._h = None

    def launch(self, tokens: torch.Tensor, positions: torch.Tensor, block_tables: torch.Tensor, batch: int,
               next_tokens: torch.Tensor, logits: torch.Tensor | None = None, pages_per_split: int = 0,
               feedback: bool = False, groups: tuple[torch.Tensor, torch.Tensor] | None = None) -> None:
        """Enqueue one decode step on the current stream (all tensors on device).

        feedback=True also writes the sampled tokens back into ``tokens`` and
        advances ``positions`` on the device (autoregressive loop without host)."""
        if batch < 1:
            raise ValueError("decode batch must be non-empty")
        if block_tables.shape[1] < 1 or block_tables.dtype != torch.int32:
            raise ValueError("block_tables must be int32 [B, max_pages]")
        st = torch.cuda.current_stream().cuda_stream
        if groups is not None:  # rows grouped by prompt for the attention (token-parallel prefill)
            gs, gl = groups
            _lib.check(self._lib.sun_decode_step_grouped(
                self._h, tokens.data_ptr(), positions.data_ptr(), block_tables.data_ptr(), block_tables.stride(0),
                batch, pages_per_split, None if logits is None else logits.data_ptr(), next_tokens.data_ptr(),
                _lib.SUN_STEP_FEEDBACK if feedback else 0, st, gs.data_ptr(), gl.data_ptr(), gs.numel()),
                "sun_decode_step_grouped")
            return
        flags = (_lib.SUN_STEP_FEEDBACK if feedback else 0) | (_lib.SUN_STEP_DISTINCT_ROWS if self.distinct_rows else 0)
        _lib.check(self._lib.sun_decode_step(
            self._h, tokens.data_ptr(), positions.data_ptr(), block_tables.data_ptr(), block_tables.stride(0), batch,
            pages_per_split, None if logits is None else logits.data_ptr(), next_tokens.data_ptr(), flags, st),
            "sun_decode_step")

    def profile(self, tokens, positions, block_tables, batch, next_tokens, logits=None, pages_per_split=0):
        """Serialised step with a CUDA event after every kernel -> per-launch device ms."""
        cap = 16 + 16 * self.spec.n_layers
        buf = (ctypes.c_float * cap)()
        n = ctypes.c_int32()
        st = torch.cuda.current_stream().cuda_stream
        _lib.check(self._lib.sun_decode_step_profile(
            self._h, tokens.data_ptr(), positions.data_ptr(), block_tables.data_ptr(), block_tables.stride(0), batch,
            pages_per_split, None if logits is None else logits.data_ptr(), next_tokens.data_ptr(), st, buf, cap,
            ctypes.byref(n)), "sun_decode_step_profile")
        return [buf[i] for i in range(min(n.value, cap))]

    def kernel_names(self, combine: bool | None = None, batch: int | None = None) -> list[str]:
        """Launch order of one step of `batch` rows (default max_batch; matches
        sun_decode_step). The split combine is launched unless fused or the attention
        ran unsplit (combine=False)."""
        combine = (not self.fused_combine) if combine is None else combine
        batch = self.max_batch if batch is None else batch
        # (the decoder's flag, then this batch width's W4 rules)
        chain = self.gemm_chain and uses_gemm_chain(self.spec.weight_bits, True, "1", batch)
        names = ["embed_norm"]
        if chain:  # O -> gate_up -> down -> next QKV as one launch per layer
            names.append("gemm_qkv_rope_kv")
            for _ in range(self.spec.n_layers):
                names += ["attention"] + (["attn_combine"] if combine else []) + ["gemm_chain"]
            return names + ["gemm_lm_head_argmax", "argmax"]
        for _ in range(self.spec.n_layers):
            names += ["gemm_qkv_rope_kv", "attention"] + (["attn_combine"] if combine else []) + [
                "gemm_o_resid_norm", "gemm_gate_up_swiglu", "gemm_down_resid_norm"]
        return names + ["gemm_lm_head_argmax", "argmax"]


def launch_count() -> int:
    """Kernels launched by libsun_b200.so on this thread so far."""
    n = ctypes.c_int64()
    _lib.check(_lib.load().sun_launch_count(ctypes.byref(n)), "sun_launch_count")
    return n.value


class SharedDecodeModule(_StepRunner):
    """D_θd — the frozen shared decode module serving every task's requests.

    Static device buffers (tokens / positions / block tables / next tokens /
    logits) back an optional CUDA graph per (batch, pages_per_split) bucket, so
    a step is one graph launch (32 layers x 8 kernels otherwise). Every row is a
    different request (the scheduler's batch), which lets the attention stage KV
    pages ahead of the step's KV append (``distinct_rows``).
    """

    distinct_rows = True

    def __init__(self, spec, weights, kv, max_batch, max_context, use_pdl: bool = True, keep_logits: bool = True):
        super().__init__(spec, weights, kv, max_batch, max_context, use_pdl)
        dev = weights.device
        self.tokens = torch.zeros(self.max_batch, dtype=torch.int32, device=dev)
        self.positions = torch.zeros(self.max_batch, dtype=torch.int32, device=dev)
        self.block_tables = torch.zeros(self.max_batch, self.max_pages, dtype=torch.int32, device=dev)
        self.next_tokens = torch.zeros(self.max_batch, dtype=torch.int32, device=dev)
        self.logits = torch.zeros(self.max_batch, spec.vocab, dtype=torch.float32, device=dev) if keep_logits else None
        self._graphs: dict[tuple, torch.cuda.CUDAGraph] = {}

    def step_static(self, batch: int, pages_per_split: int = 0, graph: bool = True, feedback: bool = False) -> None:
        """One step over the static buffers' first ``batch`` rows (device-resident inputs)."""
        if not graph:
            self.launch(self.tokens, self.positions, self.block_tables, batch, self.next_tokens, self.logits,
                        pages_per_split, feedback)
            return
        key = (batch, pages_per_split, feedback)
        g = self._graphs.get(key)
        if g is None:
            # warm (TMA descriptor cache for this batch bucket) then capture; the
            # inputs are saved before the side stream is ordered after the current one,
            # so the warm launch (whose feedback advances them) runs after the clones
            saved = (self.tokens.clone(), self.positions.clone())
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self.launch(self.tokens, self.positions, self.block_tables, batch, self.next_tokens, self.logits,
                            pages_per_split, feedback)
            torch.cuda.current_stream().wait_stream(s)
            self.tokens.copy_(saved[0])
            self.positions.copy_(saved[1])
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.launch(self.tokens, self.positions, self.block_tables, batch, self.next_tokens, self.logits,
                            pages_per_split, feedback)
            self._graphs[key] = g
        g.replay()

    def decode_host(self, tokens: torch.Tensor, positions: torch.Tensor, block_tables: torch.Tensor,
                    out: torch.Tensor, pages_per_split: int = 0, sync: bool = True) -> torch.Tensor:
        """Eq. 3 from pinned host buffers as ONE graph launch: the inputs' host->device
        copies, the step and the next tokens' device->host copy into pinned ``out``;
        returns ``out`` once the stream has synchronised. The host buffers are baked
        into the captured graph (keyed by their addresses): reuse the same buffers
        from step to step, as a serving loop does.

        ``sync=False`` returns right after the launch (the caller orders its host reads
        and rewrites of the buffers with events): a serving loop can then pass the same
        pinned buffer as ``out`` and as the next step's ``tokens`` — the device-to-host
        copy of step i and the host-to-device copy of step i + 1 are stream-ordered — and
        keep the GPU one step ahead of its host bookkeeping."""
        b = int(tokens.shape[0])
        if b < 1:
            raise ValueError("decode batch must be non-empty")
        if b > self.max_batch:
            raise ValueError(f"batch {b} > max_batch {self.max_batch}")
        for t in (tokens, positions, block_tables, out):
            if t.device.type != "cpu" or not t.is_pinned() or t.dtype != torch.int32:
                raise ValueError("decode_host takes pinned int32 host tensors")
        npg = int(block_tables.shape[1])
        if npg > self.max_pages:
            raise ValueError(f"block table width {npg} > {self.max_pages} pages")
        key = ("host", b, npg, pages_per_split, tokens.data_ptr(), positions.data_ptr(), block_tables.data_ptr(),
               out.data_ptr())
        g = self._graphs.get(key)
        if g is None:  # first call: run the step on the ordinary path, then capture for the next ones
            self.decode(tokens, positions, block_tables, pages_per_split)
            out.copy_(self.next_tokens[:b])
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.tokens[:b].copy_(tokens, non_blocking=True)
                self.positions[:b].copy_(positions, non_blocking=True)
                self.block_tables[:b, :npg].copy_(block_tables, non_blocking=True)
                self.launch(self.tokens, self.positions, self.block_tables, b, self.next_tokens, self.logits,
                            pages_per_split)
                out.copy_(self.next_tokens[:b], non_blocking=True)
            self._graphs[key] = g
            return out
        g.replay()
        if sync:
            torch.cuda.current_stream().synchronize()
        return out

    def decode(self, tokens: torch.Tensor, positions: torch.Tensor, block_tables: torch.Tensor,
               pages_per_split: int = 0, graph: bool = True, validate: bool = True) -> torch.Tensor:
        """Eq. 3 over a batch: copy inputs (host or device) into the static
        buffers, run the step, return next tokens (device int32 view [B])."""
        b = int(tokens.shape[0])
        if b < 1:
            raise ValueError("decode batch must be non-empty")
        if b > self.max_batch:
            raise ValueError(f"batch {b} > max_batch {self.max_batch}")
        if block_tables.shape[1] > self.max_pages:
            raise ValueError(f"block table width {block_tables.shape[1]} > {self.max_pages} pages")
        if validate:
            self.validate_host(tokens, positions, block_tables)
        self.tokens[:b].copy_(tokens, non_blocking=True)
        self.positions[:b].copy_(positions, non_blocking=True)
        self.block_tables[:b, :block_tables.shape[1]].copy_(block_tables, non_blocking=True)
        self.step_static(b, pages_per_split, graph)
        return self.next_tokens[:b]


class PrefillModule(_StepRunner):
    """P_θp^τ — a task-specific prefill module writing into the shared pool."""

    def __init__(self, spec, weights, kv, max_batch, max_context, task_id: int, use_pdl: bool = True,
                 grouped: bool = True):
        super().__init__(spec, weights, kv, max_batch, max_context, use_pdl)
        self.task_id = task_id
        self.grouped = grouped  # one attention CTA per (prompt, consecutive positions) group
        dev = weights.device
        self._next = torch.zeros(self.max_batch, dtype=torch.int32, device=dev)
        self._logits = torch.zeros(self.max_batch, spec.vocab, dtype=torch.float32, device=dev)

    def prefill(self, prompts: list[list[int]], block_tables: list[list[int]]) -> tuple[list[int], torch.Tensor]:
        """Fill each prompt's pages and return (first tokens, first-token logits [B, V]).

        Token-parallel chunked prefill: every (prompt, position) pair is one row of
        a ``sun_decode_step`` batch (its own position, its prompt's block table), up
        to ``max_batch`` rows per step. Inside a step each layer's QKV epilogue
        appends the KV of all rows before that layer's attention runs, so a row at
        position t attends over positions 0..t whether they came from an earlier
        step or from the same one; a prompt's rows are issued in position order.
        Same math per token as decoding the prompt one position at a time."""
        dev = self.weights.device
        B = len(prompts)
        lens = [len(p) for p in prompts]
        if B < 1 or min(lens) < 1:
            raise ValueError("isl must be >= 1")
        for i, row in enumerate(block_tables):
            if len(row) * PAGE_TOKENS < lens[i]:
                raise ValueError(f"prompt {i}: {len(row)} pages cannot hold {lens[i]} tokens")
        bt = torch.zeros(B, self.max_pages, dtype=torch.int32)
        for i, row in enumerate(block_tables):
            bt[i, :len(row)] = torch.tensor(row, dtype=torch.int32)
        rows = [(i, t) for i in range(B) for t in range(lens[i])]  # prompt-major, positions ascending
        first = [0] * B
        last_logits = torch.zeros(B, self.spec.vocab, dtype=torch.float32, device=dev)
        C = self.max_batch
        R = max(1, 16 // (self.spec.n_q_heads // self.spec.n_kv_heads))  # rows per attention group
        for c0 in range(0, len(rows), C):
            chunk = rows[c0:c0 + C]
            toks = torch.tensor([prompts[i][t] for i, t in chunk], dtype=torch.int32).to(dev)
            pos = torch.tensor([t for _, t in chunk], dtype=torch.int32).to(dev)
            bts = bt[[i for i, _ in chunk]].to(dev)
            gstart, glen = [], []
            for j, (i, t) in enumerate(chunk):  # runs of one prompt's consecutive positions, <= R rows
                if glen and glen[-1] < R and chunk[j - 1][0] == i and chunk[j - 1][1] == t - 1:
                    glen[-1] += 1
                else:
                    gstart.append(j)
                    glen.append(1)
            groups = (torch.tensor(gstart, dtype=torch.int32).to(dev), torch.tensor(glen, dtype=torch.int32).to(dev))
            self.launch(toks, pos, bts, len(chunk), self._next, self._logits, groups=groups if self.grouped else None)
            done = [(j, i) for j, (i, t) in enumerate(chunk) if t == lens[i] - 1]
            if done:
                nt = self._next[:len(chunk)].cpu()
                for j, i in done:
                    first[i] = int(nt[j])
                    last_logits[i] = self._logits[j]
        return first, last_logits
