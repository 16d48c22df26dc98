// gemm_w4.cuh — QSUN W4A16 path: int4 weights dequantised in-kernel, fed to tcgen05.
//
// Storage format "SUN-W4" (restated bit-for-bit by oracle/quant_ref.py):
//   * symmetric per-group quantisation along K, group = 128, one bf16 scale per
//     (group, row) stored tile-major: scales[row tile][K/128][128], so the scales of
//     one weight stage (consecutive K blocks of a tile) are one contiguous run;
//   * q = clamp(rint(w / s), -8, 7), s = bf16(absmax / 7.5) (s = 0 -> q = 0);
//   * packed bytes are tile-contiguous: block (row/128, k/128) is 8 KB (one bulk copy
//     per stage) laid out [chunk 4][row 128][16 B], chunk c = k 32c..32c+31 of the row
//     (a converter warp's loads are then 512 B contiguous); every 32-bit word holds 8 consecutive k elements
//     as offset-binary nibbles (q + 8) in nibble order [0,2,4,6,1,3,5,7], so one
//     shift + LOP3 yields a bf16x2 pair (128 + u_even, 128 + u_odd).
// Dequantised operand = bf16(q * s) exactly (HSUB2 is exact, HMUL2 rounds once).
//
// Pipeline per 128-wide K block: bulk copies {packed 8 KB, scales 256 B, X 2 x bn x 128 B}
// -> 8 converter warps (warps 6..13; TMEM lane group = warp % 4, one K half each)
// dequantise in registers and tcgen05.st the bf16 A tile into tensor memory
// (a ring of up to 6 tiles at the top of the 512 columns, above the accumulators;
// no shared-memory round trip, which capped the
// first version at ~1 TB/s of weights on smem bandwidth) -> warp 1 issues 8
// tcgen05.mma (K=16 each) with A from TMEM and X from smem -> warps 2..5 epilogue.
// The kernel is gemm_kernel<EPI, true> in gemm_tc.cuh (same schedules as bf16);
// the lm_head stays bf16.
#pragma once
#include "gemm_tc.cuh"
