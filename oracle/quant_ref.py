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
  scales stored tile-major [round_up(rows,128)/128][K/128][128] bf16 (a weight stage's
  scales for consecutive K blocks are one contiguous run), the 128 scales of a block
  row-interleaved: row r of the tile at position (r & 7) * 16 + (r >> 3)
  packed: block (row//128, k//128) is 8 KB contiguous, laid out [chunk 4][row 128][16 B]:
  chunk c of row r holds k = 32c .. 32c+31 of that row as 4 words; in each
  32-bit little-endian word the 8 consecutive k elements e0..e7 sit in nibbles
  [e0,e2,e4,e6,e1,e3,e5,e7] (nibble 0 = bits 0..3) as offset-binary q + 8.
"""
from __future__ import annotations

import numpy as np
import torch

NIBBLE_OF_ELEM = [0, 4, 1, 5, 2, 6, 3, 7]  # element e -> nibble position
SCALE_POS = np.array([(r & 7) * 16 + (r >> 3) for r in range(128)])  # row -> position in a block's scale run


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
    """(q [rows,K], s [rows,K/128]) -> (packed uint8 flat, scales bf16-bits uint16 [rows_pad/128, K/128, 128])."""
    rows, k = q.shape
    rows_pad = (rows + 127) // 128 * 128
    u = np.zeros((rows_pad, k), dtype=np.uint32)
    u[:rows] = (q.numpy().astype(np.int32) + 8).astype(np.uint32)
    u[rows:] = 8  # zero weights in padding rows
    words = np.zeros((rows_pad, k // 8), dtype=np.uint32)
    for e in range(8):
        words |= u[:, e::8] << np.uint32(4 * NIBBLE_OF_ELEM[e])
    # tile-contiguous: [row_tile][k_block][chunk 4][128 rows][4 words]
    kb = k // 128
    t = words.reshape(rows_pad // 128, 128, kb, 4, 4).transpose(0, 2, 3, 1, 4)
    packed = np.ascontiguousarray(t).view(np.uint8).reshape(-1)
    sc = np.zeros((rows_pad, kb), dtype=np.uint16)
    sc[:rows] = s.view(torch.int16).numpy().astype(np.uint16)
    sc = np.ascontiguousarray(sc.reshape(rows_pad // 128, 128, kb).transpose(0, 2, 1))
    out = np.empty_like(sc)
    out[..., SCALE_POS] = sc  # row r of a block at (r & 7) * 16 + (r >> 3)
    return packed, out


def unpack(packed: np.ndarray, rows: int, k: int) -> torch.Tensor:
    rows_pad = (rows + 127) // 128 * 128
    kb = k // 128
    words = (packed.view(np.uint32).reshape(rows_pad // 128, kb, 4, 128, 4).transpose(0, 3, 1, 2, 4)
             .reshape(rows_pad, k // 8))
    u = np.zeros((rows_pad, k), dtype=np.int32)
    for e in range(8):
        u[:, e::8] = (words >> np.uint32(4 * NIBBLE_OF_ELEM[e])) & np.uint32(0xF)
    return torch.from_numpy(u[:rows] - 8).to(torch.int8)
