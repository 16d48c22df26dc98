"""ORACLE — test infrastructure only. CPU restatement of QSUN's SUN-W4 format.

QSUN: weight-only post-training quantisation of the shared
decoder, every linear layer to 4 bits, symmetric, group size 128, lm_head kept
in full precision. The paper used AWQ via LLM Compressor; that
dependency is not vendored and not pinned (no lockfile; pkg/pyproject.toml:10-13
lists only numpy, tomli), so the activation-aware scale search is out of scope
and the *storage + dequantisation arithmetic* is restated here as a
builder-defined format, checked bit-for-bit against the GPU quantiser and the
in-kernel dequantiser (parity unpinned w.r.t. AWQ's scales).

SUN-W4 (matches paper_2603_02599_b200/csrc/gemm_w4.cuh):
  s   = bf16(absmax(group) / 7.5)            per (row, 128-wide K group)
  q   = clamp(rint(w / s), -8, 7)  (q = 0 if s == 0), rint = half-to-even
  deq = bf16(q * s)                          (the tcgen05 operand)
  scales stored [K/128][round_up(rows,128)] bf16
  packed: block (row//128, k//128) is 128 rows x 64 B contiguous (8 KB); in each
  32-bit little-endian word the 8 consecutive k elements e0..e7 sit in nibbles
  [e0,e2,e4,e6,e1,e3,e5,e7] (nibble 0 = bits 0..3) as offset-binary q + 8.
"""
from __future__ import annotations

import numpy as np
import torch

NIBBLE_OF_ELEM = [0, 4, 1, 5, 2, 6, 3, 7]  # element e -> nibble position


def quantize(w: torch.Tensor, group: int = 128) -> tuple[torch.Tensor, torch.Tensor]:
    """w bf16 [rows, K] -> (q int8 [rows, K], s bf16 [rows, K/group])."""
    rows, k = w.shape
    wf = w.float().view(rows, k // group, group)
    amax = wf.abs().amax(-1)
    s = (amax / 7.5).to(torch.bfloat16)
    sf = s.float()[..., None]
    safe = torch.where(sf > 0, sf, torch.ones_like(sf))
    q = torch.round(wf / safe).clamp(-8, 7)
    q = torch.where(sf > 0, q, torch.zeros_like(q))
    return q.view(rows, k).to(torch.int8), s


def dequantize(q: torch.Tensor, s: torch.Tensor, group: int = 128) -> torch.Tensor:
    rows, k = q.shape
    v = q.float().view(rows, k // group, group) * s.float()[..., None]
    return v.view(rows, k).to(torch.bfloat16)


def pack(q: torch.Tensor, s: torch.Tensor) -> tuple[np.ndarray, np.ndarray]:
    """(q [rows,K], s [rows,K/128]) -> (packed uint8 flat, scales bf16-bits uint16 [K/128, rows_pad])."""
    rows, k = q.shape
    rows_pad = (rows + 127) // 128 * 128
    u = np.zeros((rows_pad, k), dtype=np.uint32)
    u[:rows] = (q.numpy().astype(np.int32) + 8).astype(np.uint32)
    u[rows:] = 8  # zero weights in padding rows
    words = np.zeros((rows_pad, k // 8), dtype=np.uint32)
    for e in range(8):
        words |= u[:, e::8] << np.uint32(4 * NIBBLE_OF_ELEM[e])
    # tile-contiguous: [row_tile][k_block][128 rows][16 words]
    kb = k // 128
    t = words.reshape(rows_pad // 128, 128, kb, 16).transpose(0, 2, 1, 3)
    packed = np.ascontiguousarray(t).view(np.uint8).reshape(-1)
    sc = np.zeros((kb, rows_pad), dtype=np.uint16)
    sc[:, :rows] = s.view(torch.int16).numpy().astype(np.uint16).T
    return packed, sc


def unpack(packed: np.ndarray, rows: int, k: int) -> torch.Tensor:
    rows_pad = (rows + 127) // 128 * 128
    kb = k // 128
    words = packed.view(np.uint32).reshape(rows_pad // 128, kb, 128, 16).transpose(0, 2, 1, 3).reshape(rows_pad, k // 8)
    u = np.zeros((rows_pad, k), dtype=np.int32)
    for e in range(8):
        u[:, e::8] = (words >> np.uint32(4 * NIBBLE_OF_ELEM[e])) & np.uint32(0xF)
    return torch.from_numpy(u[:rows] - 8).to(torch.int8)
