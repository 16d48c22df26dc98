"""Kernel-level entry points over torch device tensors (unit parity surface).

Each function calls exactly one C-ABI symbol of libsun_b200.so on the current
torch stream. Tensors must already live on the GPU; nothing here falls back to
PyTorch math.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import UnsupportedShape


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("SUN kernels take CUDA tensors only (no CPU fallback)")


def gemm_workspace(n_out: int, k: int, batch: int, device) -> torch.Tensor:
    lib = _lib.load()
    nb = ctypes.c_size_t()
    _lib.check(lib.sun_gemm_workspace_bytes(n_out, k, batch, ctypes.byref(nb)), "sun_gemm_workspace_bytes")
    return torch.zeros(nb.value, dtype=torch.uint8, device=device)


def block_weights(w: torch.Tensor) -> torch.Tensor:
    """bf16 [rows, k] -> SUN-BLK (16 KB pre-swizzled 128x64 blocks), on the GPU."""
    _need_cuda(w)
    rows, k = w.shape
    lib = _lib.load()
    nb = ctypes.c_size_t()
    _lib.check(lib.sun_blocked_bytes(rows, k, ctypes.byref(nb)), "sun_blocked_bytes")
    out = torch.empty(nb.value, dtype=torch.uint8, device=w.device)
    _lib.check(lib.sun_block_weights_bf16(w.contiguous().data_ptr(), rows, k, out.data_ptr(), _stream()),
               "sun_block_weights_bf16")
    return out


def gemm_bf16(w: torch.Tensor, x: torch.Tensor, batch: int, out: torch.Tensor | None = None,
              accumulate: bool = False, workspace: torch.Tensor | None = None,
              shape: tuple[int, int] | None = None) -> torch.Tensor:
    """out[b, n] (=|+=) sum_k w[n, k] x[b, k] with the tcgen05 swap-AB GEMM.

    ``w`` is bf16 [n, k] (blocked here) or already SUN-BLK uint8 with ``shape``.
    ``x`` must have at least round_up(batch, 16) rows (rows >= batch are ignored).
    """
    _need_cuda(w, x)
    assert x.dtype == torch.bfloat16
    if w.dtype == torch.bfloat16:
        n_out, k = w.shape
        w = block_weights(w)
    else:
        n_out, k = shape
    if out is None:
        out = torch.zeros(batch, n_out, dtype=torch.float32, device=w.device)
    if workspace is None:
        workspace = gemm_workspace(n_out, k, batch, w.device)
    lib = _lib.load()
    _lib.check(lib.sun_gemm_bf16(w.data_ptr(), n_out, k, x.data_ptr(), x.stride(0), x.shape[0], batch,
                                 out.data_ptr(), out.stride(0), int(accumulate), workspace.data_ptr(),
                                 workspace.numel(), _stream()), "sun_gemm_bf16")
    return out


def gemm_w4(packed: torch.Tensor, scales: torch.Tensor, n_out: int, k: int, x: torch.Tensor, batch: int,
            out: torch.Tensor | None = None, accumulate: bool = False,
            workspace: torch.Tensor | None = None, gemv: bool = False) -> torch.Tensor:
    """QSUN W4A16 GEMM: out[b, n] (=|+=) sum_k deq(w)[n, k] x[b, k]. gemv=True runs the
    small-batch GEMV kernel (batch <= 16) that QSUN decode steps of <= 16 rows use."""
    _need_cuda(packed, scales, x)
    if out is None:
        out = torch.zeros(batch, n_out, dtype=torch.float32, device=x.device)
    ws = gemm_workspace(n_out, k, batch, x.device) if workspace is None else workspace
    lib = _lib.load()
    fn = lib.sun_gemv_w4 if gemv else lib.sun_gemm_w4
    _lib.check(fn(packed.data_ptr(), scales.data_ptr(), n_out, k, x.data_ptr(), x.stride(0), x.shape[0],
                  batch, out.data_ptr(), out.stride(0), int(accumulate), ws.data_ptr(), ws.numel(),
                  _stream()), "sun_gemv_w4" if gemv else "sun_gemm_w4")
    return out


def attention_decode(dims: _lib.SunDecoderDims, kv_pool: torch.Tensor, layer: int, q: torch.Tensor,
                     positions: torch.Tensor, block_tables: torch.Tensor, pages_per_split: int = 0,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """Paged split-K decode attention for one layer; q bf16 [B, nq, d] post-RoPE."""
    _need_cuda(kv_pool, q, positions, block_tables)
    batch = q.shape[0]
    if out is None:
        out = torch.empty(batch, dims.n_q_heads * dims.head_dim, dtype=torch.bfloat16, device=q.device)
    max_pages = (dims.max_context + 15) // 16
    ws = torch.zeros(batch * dims.n_q_heads * max_pages * (dims.head_dim + 2) * 4 + batch * dims.n_kv_heads * 4 + 8192,
                     dtype=torch.uint8, device=q.device)  # zeroed: split counters must start at 0
    pool = _lib.SunKvPool(kv_pool.data_ptr(), kv_pool.shape[0], dims.n_layers, dims.n_kv_heads, dims.head_dim,
                          dims.page_size, dims.rope_theta, q.device.index or 0)
    lib = _lib.load()
    _lib.check(lib.sun_attention_decode(ctypes.byref(dims), ctypes.byref(pool), layer, q.data_ptr(),
                                        positions.data_ptr(), block_tables.data_ptr(), block_tables.stride(0),
                                        batch, pages_per_split, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                        _stream()), "sun_attention_decode")
    return out


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    _need_cuda(x, w)
    b, h = x.shape
    y = torch.empty(b, h, dtype=torch.bfloat16, device=x.device)
    lib = _lib.load()
    _lib.check(lib.sun_rmsnorm(x.data_ptr(), w.data_ptr(), y.data_ptr(), b, h, eps, _stream()), "sun_rmsnorm")
    return y


def quantize_w4(w: torch.Tensor, group: int = 128) -> tuple[torch.Tensor, torch.Tensor]:
    """QSUN SUN-W4 quantisation on the GPU -> (packed uint8, scales bf16 [rows_pad/128, K/g, 128])."""
    _need_cuda(w)
    rows, k = w.shape
    rows_pad = (rows + 127) // 128 * 128
    packed = torch.zeros(rows_pad * k // 2, dtype=torch.uint8, device=w.device)
    scales = torch.zeros(rows_pad // 128, k // group, 128, dtype=torch.bfloat16, device=w.device)
    lib = _lib.load()
    _lib.check(lib.sun_quantize_w4(w.contiguous().data_ptr(), rows, k, group, packed.data_ptr(), scales.data_ptr(),
                                   _stream()), "sun_quantize_w4")
    return packed, scales


def import_w4_ct(ct_packed: torch.Tensor, ct_scales: torch.Tensor, group: int = 128
                 ) -> tuple[torch.Tensor, torch.Tensor]:
    """compressed-tensors pack-quantized W4 (int32 [rows, K/8], bf16 [rows, K/group]) -> SUN-W4
    (packed uint8, scales bf16 [rows_pad/128, K/g, 128]) on the GPU, bit-preserving."""
    _need_cuda(ct_packed, ct_scales)
    if ct_packed.dtype != torch.int32 or ct_scales.dtype != torch.bfloat16:
        raise UnsupportedShape("compressed-tensors import needs int32 weight_packed and bf16 weight_scale")
    rows, k8 = ct_packed.shape
    k = k8 * 8
    if tuple(ct_scales.shape) != (rows, k // group):
        raise UnsupportedShape(f"weight_scale {tuple(ct_scales.shape)} does not match {rows} x {k}/{group}")
    rows_pad = (rows + 127) // 128 * 128
    packed = torch.zeros(rows_pad * k // 2, dtype=torch.uint8, device=ct_packed.device)
    scales = torch.zeros(rows_pad // 128, k // group, 128, dtype=torch.bfloat16, device=ct_packed.device)
    lib = _lib.load()
    _lib.check(lib.sun_import_w4_ct(ct_packed.contiguous().data_ptr(), ct_scales.contiguous().data_ptr(), rows, k,
                                    group, packed.data_ptr(), scales.data_ptr(), _stream()), "sun_import_w4_ct")
    return packed, scales
