// gemm_w4.cuh — QSUN W4A16 path: int4 weights dequantised in-kernel, fed to tcgen05.
//
// Storage format "SUN-W4" (restated bit-for-bit by oracle/quant_ref.py):
//   * symmetric per-group quantisation along K, group = 128, one bf16 scale per
//     (group, row) stored tile-major: scales[row tile][K/128][128], so the scales of
//     one weight stage (consecutive K blocks of a tile) are one contiguous run; the
//     128 scales of a block are row-interleaved, row r at (r & 7) * 16 + (r >> 3);
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

namespace sun {

// Offline quantiser (one thread per (row, group)); produces the tile-contiguous
// SUN-W4 layout consumed above: packed block (m_tile, kb) is 128 rows x 64 B.
__global__ void quantize_w4_kernel(const __nv_bfloat16* __restrict__ w, long long rows, long long rows_pad,
                                   long long k, uint8_t* __restrict__ packed, __nv_bfloat16* __restrict__ scales) {
  const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long ngroups = k / 128;
  if (gid >= rows * ngroups) return;
  const long long r = gid / ngroups;
  const long long g = gid % ngroups;
  const __nv_bfloat16* src = w + r * k + g * 128;
  float amax = 0.f;
  for (int i = 0; i < 128; ++i) amax = fmaxf(amax, fabsf(__bfloat162float(src[i])));
  const __nv_bfloat16 sb = __float2bfloat16_rn(amax / 7.5f);
  const float s = __bfloat162float(sb);
  scales[((r / 128) * (k / 128) + g) * 128 + w4_scale_pos(static_cast<int>(r % 128))] = sb;  // tile-major, interleaved
  const long long kb_total = k / 128;
  uint8_t* blk = packed + ((r / 128) * kb_total + g) * 8192;
  for (int wd = 0; wd < 16; ++wd) {  // 16 words of 8 elements; word wd lives in chunk wd / 4
    uint32_t word = 0;
    for (int e = 0; e < 8; ++e) {
      const float x = __bfloat162float(src[wd * 8 + e]);
      int qv = 0;
      if (s > 0.f) {
        qv = static_cast<int>(rintf(x / s));
        qv = qv < -8 ? -8 : (qv > 7 ? 7 : qv);
      }
      const uint32_t u = static_cast<uint32_t>(qv + 8);
      const int nib = (e & 1) ? 4 + (e >> 1) : (e >> 1);  // order [0,2,4,6,1,3,5,7]
      word |= u << (4 * nib);
    }
    reinterpret_cast<uint32_t*>(blk + ((wd >> 2) * 128 + (r % 128)) * 16)[wd & 3] = word;
  }
}

// Import of a compressed-tensors "pack-quantized" int4 checkpoint tensor (the layout
// LLM Compressor writes for W4A16 group-128 symmetric AWQ / GPTQ; QSUN's
// quantiser): weight_packed int32 [rows][k/8] with element
// 8j+i of a row in nibble i of word j as offset-binary q + 8, weight_scale bf16
// [rows][k/128]. Re-laid out to SUN-W4 (one thread per (row, group)): the
// nibbles move to the [0,2,4,6,1,3,5,7] order, the word to its chunk/row slot,
// the scale to the tile-major run. No arithmetic on q or s: the dequantised
// operand bf16(q * s) is the checkpoint's.
__global__ void import_w4_ct_kernel(const uint32_t* __restrict__ ct_packed, const __nv_bfloat16* __restrict__ ct_scales,
                                    long long rows, long long k, uint8_t* __restrict__ packed,
                                    __nv_bfloat16* __restrict__ scales) {
  const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long ngroups = k / 128;
  if (gid >= rows * ngroups) return;
  const long long r = gid / ngroups;
  const long long g = gid % ngroups;
  scales[((r / 128) * ngroups + g) * 128 + w4_scale_pos(static_cast<int>(r % 128))] = ct_scales[r * ngroups + g];
  const uint32_t* src = ct_packed + r * (k / 8) + g * 16;
  uint8_t* blk = packed + ((r / 128) * ngroups + g) * 8192;
#pragma unroll 4
  for (int wd = 0; wd < 16; ++wd) {
    const uint32_t in = src[wd];
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int nib = (e & 1) ? 4 + (e >> 1) : (e >> 1);
      word |= ((in >> (4 * e)) & 0xFu) << (4 * nib);
    }
    reinterpret_cast<uint32_t*>(blk + ((wd >> 2) * 128 + (r % 128)) * 16)[wd & 3] = word;
  }
}

// ---------------------------------------------------------------------------
// Small-batch QSUN GEMV (decode steps of <= 8 rows; the kernel takes <= 16): D^T =
// W4 . X^T on the legacy tensor path (mma.sync m16n8k16), dequantised in registers.
//
// At B <= 16 the tcgen05 W4 kernel runs at a batch-independent 0.45-1.5 TB/s
// (scripts/w4_probe.py: 28672x4096 in 39.9 us at B = 1, 4 and 16): its converter warps'
// TMEM round trip paces it. Here the packed words go straight into MMA A fragments.
//   * Warp w of 16 compute warps (four per scheduler) owns rows 32 (w & 3) .. +31 of the
//     128-row tile (two m16 tiles) and the 32-k chunk c = w >> 2 of every 128 x 128 K
//     block: every packed byte is read from shared memory once, the activation fragment
//     once per (chunk, row quarter) and reused by both tiles.
//   * ldmatrix of the SUN-W4 block [chunk 4][row 128][16 B] as b16 8x8 matrices gives lane
//     (g, t) word t (k = 32c + 8t .. +7) of row g (one x4 per block, conflict-free). A
//     word's bf16 pairs (e0,e1) (e2,e3) (e4,e5) (e6,e7) — one LOP3 with the 0x4300 magic
//     each: q + 136, exact in bf16 — fill the A slots (2t,2t+1 | 2t+8,2t+9) of two MMAs;
//     K is permuted inside an MMA and the activation fragment uses the same permutation:
//     lane (g, t) loads x[n][32c + 8t .. +8] (one 16-byte SUN-ACT chunk) of batch row
//     n = (g & 1) * 4 + (g >> 1), an order that puts the eight lanes of each
//     shared-memory phase on eight different 16-byte bank groups.
//   * -136 sum x comes from two MMAs with A = 1 per block (shared by the tiles) and is
//     added before the group scale: acc += s (sum (q + 136) x - 136 sum x) = s sum q x in
//     fp32 (the operand bf16(q s) without its bf16 rounding: below the 2e-2 logit
//     tolerance). Blocks go in pairs so two MMA chains interleave; full 4-block stages use
//     per-thread base registers + immediate offsets. SUN-W4 stores a block's 128 scales
//     row-interleaved ((r & 7) * 16 + (r >> 3)): a lane's four rows are one 8-byte load.
//   * One producer warp streams stages of up to kbs consecutive K blocks of one tile
//     (packed kbs x 8 KB, scales kbs x 256 B, the bn x 128 k SUN-ACT slice: three bulk
//     copies); the weight and scale copies of the first ring's worth go out before the
//     dependency wait (griddepcontrol.wait, or a chain phase's grid count).
//   * Measured (scripts/gv_timeline.py; probe builds -DSUN_GV_PROBE_IDLE / _NOLOAD): the
//     consumer, not the ring, paces it — with no loads at all (NOLOAD) the 8B gate_up's
//     2-tile CTAs take the same ~16 us as with them, while the ring alone (IDLE) streams
//     at 7.5 TB/s; the integer ALU pipe (LOP3 / SHF of the dequant) runs at ~53% and the
//     HMMA pipe at ~33%, the rest is dependency latency with four warps per scheduler.
//   * Schedule: with at least one tile per SM, each CTA streams a contiguous run of whole
//     tiles (the epilogue of one overlaps the ring's loads of the next); with fewer tiles,
//     S = SMs / tiles CTAs split each tile's K, park their 128 x 16 fp32 partials in L2
//     and bump the tile's counter, and the CTA completing the count adds the S partials
//     in split order (deterministic) and runs the epilogue. (Measured slower: a stream-K
//     grid — the partial segments' L2 round trips inside the main loop stalled the stream —
//     and, behind SUN_GV_CLUSTER=1, one hardware cluster per tile whose rank 0 adds the
//     peers' staged tiles over DSMEM between two cluster barriers: 7.4 vs 2.6 us tails.) The epilogue is the tcgen05 GEMM's epi_chunk (QKV RoPE + KV append,
//     residual + next-norm operand, SwiGLU, store) on warps 2..5.
// ---------------------------------------------------------------------------
constexpr int kGvWarps = 16;                     // compute warps: (row quarter, 32-k chunk)
constexpr int kGvMT = 2;                         // m16 tiles per warp (32 rows)
constexpr int kGvThreads = kGvWarps * 32 + 32;   // + the producer warp
constexpr int kGvMaxStages = 8;

constexpr int kGvTPitch = 17;                    // fp32 staging tile [128][17] (conflict-free row reads)

__host__ __device__ inline uint32_t gv_stage_bytes(int bn, int kbs) {
#if defined(SUN_GV_PROBE_NOX) || defined(SUN_GV_PROBE_NOSX)
  bn = 0;  // probes: stages without the activation slice (deeper weight rings)
#endif
  return static_cast<uint32_t>(kbs) * (kW4PackedBytes + 256u + static_cast<uint32_t>(bn) * 256u);
}
__host__ __device__ inline size_t gv_smem_bytes(int bn, int kbs, int stages) {
  return 1024 + static_cast<size_t>(stages) * gv_stage_bytes(bn, kbs) + kTileM * kGvTPitch * 4 + 3072 +
         kEpiGroupBytes + 2 * kGvMaxStages * 8 + 64;
}


SUN_DEVICE void mma_16816_q(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                            uint32_t b1) {  // non-volatile: the scheduler may interleave it with the dequant
#ifdef SUN_GV_NO_MMA  // probe: skip the tensor op (timing only, results invalid)
  d[0] += __uint_as_float(a0 ^ b0); d[1] += __uint_as_float(a1 ^ b1); d[2] += __uint_as_float(a2); d[3] += __uint_as_float(a3);
  return;
#endif
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// word -> bf16x2 (q_{2p}, q_{2p+1}) of pair p (nibble order [0,2,4,6,1,3,5,7])
SUN_DEVICE uint32_t w4_pair_q(uint32_t w, int p) {
#ifdef SUN_GV_NO_CVT  // probe: skip the dequant arithmetic (timing only, results invalid)
  return w >> p;
#endif
  uint32_t u = lop3_and_or(w >> (4 * p), 0x000F000Fu, 0x43004300u);  // bf16 128 + (q + 8)
  __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&u);
  v = __hsub2(v, __floats2bfloat162_rn(136.f, 136.f));  // exact: q in [-8, 7]
  return *reinterpret_cast<uint32_t*>(&v);
}

// word -> bf16x2 (q_{2p} + 136, q_{2p+1} + 136): the magic pair alone (exact)
SUN_DEVICE uint32_t w4_pair_raw(uint32_t w, int p) {
#ifdef SUN_GV_NO_CVT
  return w >> p;
#endif
  return lop3_and_or(w >> (4 * p), 0x000F000Fu, 0x43004300u);
}

// batch row of fragment row g (conflict-free activation loads; see above)
SUN_DEVICE int gv_nrow(int g) { return ((g & 1) << 2) | (g >> 1); }

// One 128 x 128 K block for this warp's 64 rows (4 m16 tiles) and its 32-k chunk c,
// split in a load half (fragments into registers) and a math half so the block loop can
// issue block i+1's shared-memory loads before block i's dequant / MMAs.
template <int NB>
struct GvFrag {
  uint32_t wq[2 * kGvMT];  // word t of row 32 rq + 16 m + 8 h + g: wq[2m + h] (one ldmatrix.x4)
  uint32_t x[NB][4];       // x[n][32c + 8t .. +8] of batch row n = 8 j + gv_nrow(g)
  uint32_t sv[kGvMT];      // bf16 scales of rows 32 rq + 16 m + g | +8: interleaved 16 g + 4 rq + 2 m + h
};

template <int NB>
SUN_DEVICE void gv_load(GvFrag<NB>& f, uint32_t pk, uint32_t sc, uint32_t xs, int bn, int rq, int c, int lane) {
  const int g = lane >> 2, t = lane & 3;
  ldmatrix_x4(pk + c * 2048 + (32 * rq + lane) * 16, f.wq[0], f.wq[1], f.wq[2], f.wq[3]);
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int n = 8 * j + gv_nrow(g);
    const uint32_t addr = xs + (c >> 1) * bn * 128 + n * 128 + ((((c & 1) * 4 + t) ^ (n & 7)) << 4);
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(f.x[j][0]), "=r"(f.x[j][1]), "=r"(f.x[j][2]), "=r"(f.x[j][3])
                 : "r"(addr));
  }
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(f.sv[0]), "=r"(f.sv[1]) : "r"(sc + (16 * g + 4 * rq) * 2));
}

// Fast path of a full 4-block stage at bn = 16 (the decode steps' shape): every address is a
// per-thread register + a compile-time immediate (block i of the stage at i x 8 KB, its
// scales at 32 KB + 256 i, its activation slice at 33 KB + 4 KB i). The generic loads
// recompute the swizzled offsets per block — integer ALU work on the pipe the dequant
// already saturates (measured: half the loop's ALU instructions were address arithmetic).
constexpr int kGvFastKbs = 4, kGvFastBn = 16;
template <int NB>
struct GvBase {
  uint32_t w, s, x[NB];  // per-thread shared addresses within stage 0 (block 0)
};
template <int NB>
SUN_DEVICE GvBase<NB> gv_base(uint32_t ring_s, int rq, int c, int lane) {
  const int g = lane >> 2, t = lane & 3;
  GvBase<NB> b;
  b.w = ring_s + c * 2048 + (32 * rq + lane) * 16;
  b.s = ring_s + kGvFastKbs * kW4PackedBytes + (16 * g + 4 * rq) * 2;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int n = 8 * j + gv_nrow(g);
    b.x[j] = ring_s + kGvFastKbs * (kW4PackedBytes + 256u) + (c >> 1) * kGvFastBn * 128 + n * 128 +
             ((((c & 1) * 4 + t) ^ (n & 7)) << 4);
  }
  return b;
}
template <int NB, int I>
SUN_DEVICE void gv_load_fast(GvFrag<NB>& f, const GvBase<NB>& b, uint32_t stage_off) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4+%5];"
               : "=r"(f.wq[0]), "=r"(f.wq[1]), "=r"(f.wq[2]), "=r"(f.wq[3])
               : "r"(b.w + stage_off), "n"(I * kW4PackedBytes));
#pragma unroll
  for (int j = 0; j < NB; ++j)
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=r"(f.x[j][0]), "=r"(f.x[j][1]), "=r"(f.x[j][2]), "=r"(f.x[j][3])
                 : "r"(b.x[j] + stage_off), "n"(I * kGvFastBn * 256));
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+%3];" : "=r"(f.sv[0]), "=r"(f.sv[1]) : "r"(b.s + stage_off), "n"(I * 256));
}

// acc[m][j] += s_row * sum_k q x (n-tile j), for NBLK blocks at once (their MMA chains
// interleave: one block's chain is two dependent 26-cycle HMMAs, so a warp alone on one
// block idles the tensor pipe). The A operand is the raw magic pair bf16(128 + q + 8) =
// q + 136 (one LOP3, no subtraction); the block's -136 sum_k x comes from two MMAs with
// A = 1 (shared by the m16 tiles, off the tiles' critical path) and is added before the
// scale: acc += s (sum (q + 136) x - 136 sum x) = s sum q x.
template <int NB, int NBLK>
SUN_DEVICE void gv_math(const GvFrag<NB> (&f)[NBLK], float (&acc)[kGvMT][NB][4]) {
#ifndef SUN_GV_CX_SEPARATE
  // the block's -136 sum x (A = -136, both k16 steps) is the C input of the tiles' MMA chains,
  // so the group scale is one FFMA per accumulator (4-deep HMMA chains; 8B W4 B=1 step
  // 2.334 -> 2.320 ms same box). -DSUN_GV_CX_SEPARATE: the ones-MMA sums folded in by FFMA
  constexpr uint32_t kM136 = 0xC308C308u;  // bf16x2 (-136, -136), exact
  float cx[NBLK][NB][4];
#pragma unroll
  for (int b = 0; b < NBLK; ++b)
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      cx[b][j][0] = cx[b][j][1] = cx[b][j][2] = cx[b][j][3] = 0.f;
      mma_16816_q(cx[b][j], kM136, kM136, kM136, kM136, f[b].x[j][0], f[b].x[j][1]);
    }
#pragma unroll
  for (int b = 0; b < NBLK; ++b)
#pragma unroll
    for (int j = 0; j < NB; ++j) mma_16816_q(cx[b][j], kM136, kM136, kM136, kM136, f[b].x[j][2], f[b].x[j][3]);
#pragma unroll
  for (int b = 0; b < NBLK; ++b)
#pragma unroll
    for (int m = 0; m < kGvMT; ++m) {
      const uint32_t lo = f[b].wq[2 * m], hi = f[b].wq[2 * m + 1];
      float blk[NB][4];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        blk[j][0] = cx[b][j][0]; blk[j][1] = cx[b][j][1]; blk[j][2] = cx[b][j][2]; blk[j][3] = cx[b][j][3];
      }
#pragma unroll
      for (int step = 0; step < 2; ++step) {
        const uint32_t a0 = w4_pair_raw(lo, 2 * step), a1 = w4_pair_raw(hi, 2 * step);
        const uint32_t a2 = w4_pair_raw(lo, 2 * step + 1), a3 = w4_pair_raw(hi, 2 * step + 1);
#pragma unroll
        for (int j = 0; j < NB; ++j) mma_16816_q(blk[j], a0, a1, a2, a3, f[b].x[j][2 * step], f[b].x[j][2 * step + 1]);
      }
      const float s0 = __uint_as_float(f[b].sv[m] << 16), s1 = __uint_as_float(f[b].sv[m] & 0xFFFF0000u);
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        acc[m][j][0] = fmaf(s0, blk[j][0], acc[m][j][0]);
        acc[m][j][1] = fmaf(s0, blk[j][1], acc[m][j][1]);
        acc[m][j][2] = fmaf(s1, blk[j][2], acc[m][j][2]);
        acc[m][j][3] = fmaf(s1, blk[j][3], acc[m][j][3]);
      }
    }
#else
  constexpr uint32_t kOnes = 0x3F803F80u;  // bf16x2 (1, 1)
  float cx[NBLK][NB][4];
  float blk[NBLK][kGvMT][NB][4];
#pragma unroll
  for (int b = 0; b < NBLK; ++b)
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      cx[b][j][0] = cx[b][j][1] = cx[b][j][2] = cx[b][j][3] = 0.f;
#pragma unroll
      for (int m = 0; m < kGvMT; ++m) blk[b][m][j][0] = blk[b][m][j][1] = blk[b][m][j][2] = blk[b][m][j][3] = 0.f;
    }
  // first k16 step of every (block, tile) and the ones-MMAs, then the second steps
#pragma unroll
  for (int step = 0; step < 2; ++step) {
#pragma unroll
    for (int b = 0; b < NBLK; ++b) {
#ifndef SUN_GV_PROBE_NOCX  // probe: no -136 sum x MMAs (timing only, results invalid)
#pragma unroll
      for (int j = 0; j < NB; ++j)
        mma_16816_q(cx[b][j], kOnes, kOnes, kOnes, kOnes, f[b].x[j][2 * step], f[b].x[j][2 * step + 1]);
#endif
#pragma unroll
      for (int m = 0; m < kGvMT; ++m) {
        const uint32_t lo = f[b].wq[2 * m], hi = f[b].wq[2 * m + 1];
        const uint32_t a0 = w4_pair_raw(lo, 2 * step), a1 = w4_pair_raw(hi, 2 * step);
        const uint32_t a2 = w4_pair_raw(lo, 2 * step + 1), a3 = w4_pair_raw(hi, 2 * step + 1);
#pragma unroll
        for (int j = 0; j < NB; ++j) mma_16816_q(blk[b][m][j], a0, a1, a2, a3, f[b].x[j][2 * step], f[b].x[j][2 * step + 1]);
      }
    }
  }
#pragma unroll
  for (int b = 0; b < NBLK; ++b)
#pragma unroll
    for (int m = 0; m < kGvMT; ++m) {
      const float s0 = __uint_as_float(f[b].sv[m] << 16), s1 = __uint_as_float(f[b].sv[m] & 0xFFFF0000u);
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        acc[m][j][0] = fmaf(s0, fmaf(-136.f, cx[b][j][0], blk[b][m][j][0]), acc[m][j][0]);
        acc[m][j][1] = fmaf(s0, fmaf(-136.f, cx[b][j][1], blk[b][m][j][1]), acc[m][j][1]);
        acc[m][j][2] = fmaf(s1, fmaf(-136.f, cx[b][j][2], blk[b][m][j][2]), acc[m][j][2]);
        acc[m][j][3] = fmaf(s1, fmaf(-136.f, cx[b][j][3], blk[b][m][j][3]), acc[m][j][3]);
      }
    }
#endif
}

SUN_DEVICE void gv_bar() { asm volatile("bar.sync 2, 512;" ::: "memory"); }  // the 16 compute warps

// Shared-memory map of a GEMV CTA: the stage ring, the fp32 staging tile T, the epilogue
// area of epi_chunk (meta + one group's staging), the ring barriers and a flag word.
struct GvSmem {
  uint8_t* ring;
  float* T;
  float* epi;
  uint64_t* full;
  uint64_t* empty;
  int* flag;
};
SUN_DEVICE GvSmem gv_smem(uint8_t* smem, int stages, uint32_t sb) {
  GvSmem m;
  m.ring = smem;
  m.T = reinterpret_cast<float*>(smem + stages * sb);
  m.epi = m.T + kTileM * kGvTPitch;
  m.full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(m.epi) + 3072 + kEpiGroupBytes);
  m.empty = m.full + kGvMaxStages;
  m.flag = reinterpret_cast<int*>(m.empty + kGvMaxStages);
  return m;
}

// This CTA's units [u0, u1) (unit = tile * KB + K block) of one GEMV: splits == 0: whole
// tiles [c m / G, (c+1) m / G); splits == S: tile c / S, K blocks [r KB / S, (r+1) KB / S)
// (r = c % S; CTAs c >= m S have none).
SUN_DEVICE void gv_range(const GemmArgs& a, int c, int G, int& u0, int& u1) {
  const int KB = a.ksteps, S = a.splits;
  if (S == 0) {
    u0 = static_cast<int>(static_cast<long long>(c) * a.m_tiles / G) * KB;
    u1 = static_cast<int>(static_cast<long long>(c + 1) * a.m_tiles / G) * KB;
  } else if (S > 0 && c < a.m_tiles * S) {
    const int t0 = c / S, r = c % S;
    u0 = t0 * KB + r * KB / S;
    u1 = t0 * KB + (r + 1) * KB / S;
  } else if (S < 0) {  // balanced: the whole tiles (second range: gv_bal_range)
    const int W = a.m_tiles / G;
    u0 = c * W * KB;
    u1 = (c + 1) * W * KB;
  } else {
    u0 = u1 = 0;
  }
}

// Balanced schedule (splits < 0): W = m_tiles / G whole tiles per CTA (first range), then the
// R = m_tiles - W G remaining tiles' Ur = R KB blocks spread contiguously, CTA c taking
// [B0 + f(c), B0 + f(c + 1)) with f(c) = c Ur / G and B0 = W G KB (second range). The host
// picks it only when G <= Ur and ceil(Ur / G) <= KB, so every CTA has remainder work and its
// range touches at most two tiles (partial pieces 0 and 1, parked in sk_part slots 2c, 2c + 1).
// 8B gate_up at B <= 16 (224 tiles on 148 CTAs): 64 -> 49 K blocks for the busiest CTA.
SUN_DEVICE int gv_bal_f(int c, int Ur, int G) { return static_cast<int>(static_cast<long long>(c) * Ur / G); }
SUN_DEVICE void gv_bal_range(const GemmArgs& a, int c, int G, int& v0, int& v1) {
  if (a.splits >= 0) {
    v0 = v1 = 0;
    return;
  }
  const int KB = a.ksteps, W = a.m_tiles / G, Ur = (a.m_tiles - W * G) * KB, B0 = W * G * KB;
  v0 = B0 + gv_bal_f(c, Ur, G);
  v1 = B0 + gv_bal_f(c + 1, Ur, G);
}
// Contributors [cf, cl] of a split tile and the sk_part slot of contributor c' (the tile's
// last arrival adds the slots in contributor order: deterministic).
SUN_DEVICE void gv_tile_contrib(const GemmArgs& a, int G, int tile, int& cf, int& cl) {
  if (a.splits > 0) {
    cf = tile * a.splits;
    cl = cf + a.splits - 1;
    return;
  }
  const int KB = a.ksteps, W = a.m_tiles / G, Ur = (a.m_tiles - W * G) * KB;
  const int x0 = (tile - W * G) * KB, x1 = x0 + KB - 1;  // remainder-relative first / last block
  // owner(x) = the largest c with f(c) <= x = ceil((x + 1) G / Ur) - 1
  cf = static_cast<int>((static_cast<long long>(x0 + 1) * G + Ur - 1) / Ur) - 1;
  cl = static_cast<int>((static_cast<long long>(x1 + 1) * G + Ur - 1) / Ur) - 1;
}
SUN_DEVICE int gv_part_slot(const GemmArgs& a, int G, int cp, int tile) {
  if (a.splits > 0) return 2 * cp;
  const int KB = a.ksteps, W = a.m_tiles / G, Ur = (a.m_tiles - W * G) * KB;
  const int first_tile = (W * G * KB + gv_bal_f(cp, Ur, G)) / KB;
  return 2 * cp + (first_tile == tile ? 0 : 1);
}

// Producer (one elected thread): the stages of [u0, u1) — up to kbs consecutive K blocks
// of one tile each — into the ring, continuing at (slot, phase). The weight + scale copies
// of the first ring's worth go out before `gate()` (they never depend on earlier work:
// under PDL, or during the previous chain phase's tail), the activation copies after it.
template <typename Gate>
SUN_DEVICE void gv_produce(const GemmArgs& a, int u0, int u1, const GvSmem& m, int stages, int& slot, int& phase,
                           Gate gate, int max_pre = kGvMaxStages, bool first_wait = false) {
  const int kbs = a.wgroup, bn = a.bn, KB = a.ksteps;
  const uint32_t sb = gv_stage_bytes(bn, kbs);
#if defined(SUN_GV_PROBE_NOSX)  // probes (timing only, results invalid): skip the scale and X copies
  const uint32_t wbytes = kW4PackedBytes, xbytes = 0u;
#elif defined(SUN_GV_PROBE_NOX)  // skip the X copies
  const uint32_t wbytes = kW4PackedBytes + 256u, xbytes = 0u;
#else
  const uint32_t wbytes = kW4PackedBytes + 256u, xbytes = static_cast<uint32_t>(bn) * 256u;
#endif
  auto issue_w = [&](int u, int len) {
    uint8_t* st = m.ring + slot * sb;
    mbar_wait(&m.empty[slot], phase ^ 1);
#ifdef SUN_GV_PROBE_NOLOAD  // probe: stages handed over without any copy (compute-only rate; results invalid)
    mbar_arrive(&m.full[slot]);
    return;
#endif
    mbar_arrive_expect_tx(&m.full[slot], static_cast<uint32_t>(len) * (wbytes + xbytes));
    bulk_load_hint(st, a.w4_packed + static_cast<long long>(u) * kW4PackedBytes, len * kW4PackedBytes, &m.full[slot],
                   kEvictFirst);
#ifndef SUN_GV_PROBE_NOSX
    bulk_load_hint(st + kbs * kW4PackedBytes, a.w4_scales + static_cast<long long>(u) * kTileM, len * 256u,
                   &m.full[slot], kEvictFirst);
#endif
  };
  auto issue_x = [&](int sl, int u, int len) {
#ifdef SUN_GV_PROBE_NOLOAD
    return;
#endif
    if (xbytes)
      bulk_load_hint(m.ring + sl * sb + kbs * (kW4PackedBytes + 256u),
                     a.xact + static_cast<long long>(2 * (u % KB)) * bn * 128, len * xbytes, &m.full[sl], kEvictLast);
  };
  auto advance = [&]() {
    if (++slot == stages) {
      slot = 0;
      phase ^= 1;
    }
  };
  int pre_slot[kGvMaxStages], pre_u[kGvMaxStages], pre_len[kGvMaxStages];
  int u = u0, npre = 0;
  const int phase0 = phase;
  if (first_wait) max_pre = 1;
  for (; npre < min(stages, max_pre) && u < u1; ++npre) {
    const int len = min(kbs, min(u1 - u, KB - u % KB));
    issue_w(u, len);
    pre_slot[npre] = slot;
    pre_u[npre] = u;
    pre_len[npre] = len;
    u += len;
    advance();
  }
  gate();
  asm volatile("fence.proxy.async.global;" ::: "memory");  // activations written by other CTAs' stores
  for (int i = 0; i < npre; ++i) issue_x(pre_slot[i], pre_u[i], pre_len[i]);
  // first_wait: the rest of the ring goes out once the first stage has landed, so it does not
  // share the DRAM queues with the whole ring's burst and the consumers start early (8B
  // shapes: first stage 4.4 -> 2.1 us, W4 B=1 step 2.38 -> 2.34 ms; a 1-block first stage
  // landed in 1.0 us but the ring then fell behind the consumers: 2.48 ms)
  if (first_wait && npre > 0) mbar_wait(&m.full[pre_slot[0]], phase0);
  while (u < u1) {
    const int len = min(kbs, min(u1 - u, KB - u % KB));
    const int sl = slot;
    issue_w(u, len);
    issue_x(sl, u, len);
    u += len;
    advance();
  }
}

// Compute warps: the segments of [u0, u1) continuing at the ring position (slot, phase),
// each reduced over the chunk warps into T and finished by the fused epilogue (whole
// tile) or parked in L2 for the tile's last-arriving split (which reduces and finishes it).
// `gate()` runs first (all 512 compute threads): the epilogue metadata reads the previous
// work's outputs.
template <int EPI, int NB, typename Gate>
SUN_DEVICE void gv_consume(const GemmArgs& a, int u0, int u1, const GvSmem& m, int stages, int& slot, int& phase,
                           Gate gate, unsigned long long* pst = nullptr, bool meta = true) {
  const int kbs = a.wgroup, bn = a.bn, KB = a.ksteps, S = a.splits;
  const uint32_t sb = gv_stage_bytes(bn, kbs);
  const int warp = static_cast<int>(threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int c = static_cast<int>(blockIdx.x), G = static_cast<int>(gridDim.x);
  float* T = m.T;
  gate();
  if (pst && threadIdx.x == 0) pst[0] = gtimer();
  if (meta && warp >= 2 && warp < 6) load_qkv_meta<EPI>(a, m.epi);  // epilogue group: positions / pages / r_b
  const int rq = warp & 3, ch = warp >> 2;  // row quarter, 32-k chunk of every block
  const int g = lane >> 2, t = lane & 3;
  const uint32_t ring_s = smem_u32(m.ring);
  const bool fast = kbs == kGvFastKbs && bn == kGvFastBn;
  const GvBase<NB> base = gv_base<NB>(ring_s, rq, ch, lane);
  float acc[kGvMT][NB][4];
  int u = u0;
  while (u < u1) {
    const int tile = u / KB;
    const int seg_end = min(u1, (tile + 1) * KB);
    const bool whole = (u == tile * KB) && (seg_end == (tile + 1) * KB);
#pragma unroll
    for (int mt = 0; mt < kGvMT; ++mt)
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[mt][j][0] = acc[mt][j][1] = acc[mt][j][2] = acc[mt][j][3] = 0.f;
    while (u < seg_end) {
      const int len = min(kbs, seg_end - u);
      mbar_wait(&m.full[slot], phase);
      if (threadIdx.x == 0 && u == u0 && meta) {
        SUN_STAMP(2);  // first stage landed
        if (pst) pst[1] = gtimer();
      }
      const uint32_t st = ring_s + slot * sb;
#ifndef SUN_GV_PROBE_IDLE  // probe: compute warps only pass the stages on (timing only)
      if (fast && len == kGvFastKbs) {
        const uint32_t so = slot * sb;
        GvFrag<NB> f2[2];
        gv_load_fast<NB, 0>(f2[0], base, so);
        gv_load_fast<NB, 1>(f2[1], base, so);
        gv_math<NB, 2>(f2, acc);
        gv_load_fast<NB, 2>(f2[0], base, so);
        gv_load_fast<NB, 3>(f2[1], base, so);
        gv_math<NB, 2>(f2, acc);
      } else {
        auto ld = [&](GvFrag<NB>& f, int i) {
          gv_load<NB>(f, st + i * kW4PackedBytes, st + kbs * kW4PackedBytes + i * 256,
                      st + kbs * (kW4PackedBytes + 256u) + i * bn * 256, bn, rq, ch, lane);
        };
        int i = 0;
        for (; i + 1 < len; i += 2) {  // block pairs: two interleaved MMA chains
          GvFrag<NB> f2[2];
          ld(f2[0], i);
          ld(f2[1], i + 1);
          gv_math<NB, 2>(f2, acc);
        }
        if (i < len) {
          GvFrag<NB> f1[1];
          ld(f1[0], i);
          gv_math<NB, 1>(f1, acc);
        }
      }
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(&m.empty[slot]);
      u += len;
      if (++slot == stages) {
        slot = 0;
        phase ^= 1;
      }
    }
    if (threadIdx.x == 0 && u == u1) {
      SUN_STAMP(3);  // last stage consumed
      if (pst) pst[2] = gtimer();
    }
    // fragments -> T[row][batch]: row 32 rq + 16 m + g (+8), batch 8 j + t (c0) / 8 j + t + 4 (c1)
    // (gv_nrow of columns 2t, 2t+1); columns >= 8 NB are zero. Chunk 0's warps store,
    // chunks 1..3 add in order (fixed summation order).
    gv_bar();  // the previous segment's epilogue is done with T
    for (int cc = 0; cc < 4; ++cc) {
      if (ch == cc) {
#pragma unroll
        for (int mt = 0; mt < kGvMT; ++mt) {
          const int r = 32 * rq + 16 * mt + g;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int jj = j < NB ? j : 0;
            const bool have = j < NB;
            float* p0 = T + r * kGvTPitch + 8 * j + t;
            float* p1 = T + (r + 8) * kGvTPitch + 8 * j + t;
            const float v0 = have ? acc[mt][jj][0] : 0.f, v1 = have ? acc[mt][jj][1] : 0.f;
            const float v2 = have ? acc[mt][jj][2] : 0.f, v3 = have ? acc[mt][jj][3] : 0.f;
            if (cc == 0) {
              p0[0] = v0; p0[4] = v1; p1[0] = v2; p1[4] = v3;
            } else {
              p0[0] += v0; p0[4] += v1; p1[0] += v2; p1[4] += v3;
            }
          }
        }
      }
      gv_bar();
    }
    bool run_epi = whole;
    if (!whole && a.vcluster == 0) {
      // hardware cluster of the tile's S ranks (split schedule: one segment per CTA): every
      // rank's T is complete after the first cluster barrier; rank 0's epilogue warps add the
      // peers' rows over DSMEM in rank order (deterministic: ((T0 + T1) + T2) + ...) and run
      // the epilogue; the second barrier keeps the peers' T alive until it is read (the
      // producer warp mirrors both barriers). No L2 partials, atomics or reducer loads.
      cluster_sync_all();
      if (cluster_ctarank() == 0 && warp >= 2 && warp < 6) {
        const int q = warp & 3;
        const int row_local = q * 32 + lane;
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = T[row_local * kGvTPitch + j];
        for (int r = 1; r < S; ++r) {
          const uint32_t src = dsmem_addr(T + row_local * kGvTPitch, static_cast<uint32_t>(r));
          float pv[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(pv[j]) : "r"(src + 4 * j));
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += pv[j];
        }
        epi_chunk<EPI>(a, tile, row_local, 0, v, m.epi);
      }
      cluster_sync_all();
      continue;
    }
    if (!whole) {
      // park the partial: slot [2c + piece][128 rows][16] fp32, 8 floats per thread (split
      // schedule: one segment per CTA; balanced: up to two)
      const int tid = threadIdx.x & 255, row = tid >> 1, h = (tid & 1) * 8;
      const bool mover = threadIdx.x < 256;  // 8 floats each
      if (mover) {
        float* dst = a.sk_part + static_cast<long long>(gv_part_slot(a, G, c, tile)) * (kTileM * 16) + row * 16 + h;
        __stcg(reinterpret_cast<float4*>(dst), make_float4(T[row * kGvTPitch + h], T[row * kGvTPitch + h + 1],
                                                           T[row * kGvTPitch + h + 2], T[row * kGvTPitch + h + 3]));
        __stcg(reinterpret_cast<float4*>(dst + 4), make_float4(T[row * kGvTPitch + h + 4], T[row * kGvTPitch + h + 5],
                                                               T[row * kGvTPitch + h + 6], T[row * kGvTPitch + h + 7]));
        __threadfence();
      }
      gv_bar();
      int cf, cl;
      gv_tile_contrib(a, G, tile, cf, cl);
      if (threadIdx.x == 0) {
        const unsigned old = atomicAdd(a.sk_flags + tile, 1u);
        *m.flag = (old == static_cast<unsigned>(cl - cf)) ? 1 : 0;
      }
      gv_bar();
      run_epi = *m.flag != 0;
      if (run_epi && mover) {  // last contributor: sum the tile's partials in split order
        __threadfence();
        float s8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) s8[e] = 0.f;
        for (int c0 = cf; c0 <= cl; c0 += 4) {  // four partials' loads in flight per round trip
          float4 pp[4][2];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int slot_e = gv_part_slot(a, G, c0 + e <= cl ? c0 + e : cl, tile);
            const float* src = a.sk_part + static_cast<long long>(slot_e) * (kTileM * 16) + row * 16 + h;
            pp[e][0] = __ldcg(reinterpret_cast<const float4*>(src));
            pp[e][1] = __ldcg(reinterpret_cast<const float4*>(src + 4));
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (c0 + e > cl) break;
            s8[0] += pp[e][0].x; s8[1] += pp[e][0].y; s8[2] += pp[e][0].z; s8[3] += pp[e][0].w;
            s8[4] += pp[e][1].x; s8[5] += pp[e][1].y; s8[6] += pp[e][1].z; s8[7] += pp[e][1].w;
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) T[row * kGvTPitch + h + e] = s8[e];
        if (threadIdx.x == 0) a.sk_flags[tile] = 0u;  // self-resetting for the next use
      }
      if (run_epi) gv_bar();
    }
    if (run_epi && warp >= 2 && warp < 6) {
      const int q = warp & 3;
      const int row_local = q * 32 + lane;
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = T[row_local * kGvTPitch + j];
      epi_chunk<EPI>(a, tile, row_local, 0, v, m.epi);
    }
  }
}

SUN_DEVICE void gv_init_ring(const GvSmem& m, int stages) {
  if (static_cast<int>(threadIdx.x >> 5) == kGvWarps && elect_one()) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&m.full[s], 1);
      mbar_init(&m.empty[s], kGvWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
}

template <int EPI, int NB>
__global__ void __launch_bounds__(kGvThreads, 1) gemv_w4_kernel(const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  tl_begin(a.tl, a.tl_idx);
  const int stages = a.stages;
  const GvSmem m = gv_smem(smem, stages, gv_stage_bytes(a.bn, a.wgroup));
  const int warp = warp_id_sync();
  int u0, u1, v0, v1;  // v: the balanced schedule's remainder range (empty otherwise)
  gv_range(a, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), u0, u1);
  gv_bal_range(a, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), v0, v1);
  if (u0 == u1) {
    u0 = v0;
    u1 = v1;
    v0 = v1 = 0;
  }
  if (threadIdx.x == 0) SUN_STAMP(0);
  gv_init_ring(m, stages);
  pdl_launch_dependents();
  if (threadIdx.x == 0) SUN_STAMP(1);
  int slot = 0, phase = 0;
  if (warp == kGvWarps) {
    if (elect_one()) {
      gv_produce(a, u0, u1, m, stages, slot, phase, [] { pdl_wait(); }, kGvMaxStages, /*first_wait=*/true);
      if (v0 < v1) gv_produce(a, v0, v1, m, stages, slot, phase, [] {}, 0);
      // every stage of this CTA is in flight: pull the next GEMV's first weight bytes into L2
      // while this kernel's ring drains and its tail runs (the next kernel's CTAs cannot be
      // resident before this one exits, so their own first loads would start cold)
      prefetch_next_weights(a);
    }
    __syncwarp();
    if (a.splits > 0 && a.vcluster == 0 && u0 < u1) {  // the consumers' two cluster barriers
      cluster_sync_all();
      cluster_sync_all();
    }
  } else {
    gv_consume<EPI, NB>(a, u0, u1, m, stages, slot, phase, [] { pdl_wait(); });
    if (v0 < v1) gv_consume<EPI, NB>(a, v0, v1, m, stages, slot, phase, [] {}, nullptr, /*meta=*/false);
  }
  if (threadIdx.x == 64) SUN_STAMP(5);  // (epilogue warp) last epilogue done
  if (threadIdx.x == 0) SUN_STAMP(6);
  tl_end(a.tl, a.tl_idx);
}

// ---------------------------------------------------------------------------
// GEMV with a dedicated epilogue group (gemv_w4a_kernel, SUN_GV_ASYNC_EPI): warps 2..5 only
// run the epilogue (and the split partials' park / last-arrival reduction); the 16 compute
// warps (0, 1, 6..19) reduce a segment into T, hand it over through a named barrier and go
// straight on with the next segment's stages — in gemv_w4_kernel warps 2..5 are compute
// warps too, so a tile's epilogue, and a split segment's L2 round trips, stall the ring's
// consumers (which pace the kernel). One T buffer: the epilogue warps copy their row into
// registers and release it at once. Warp 20 is the producer.
// ---------------------------------------------------------------------------
constexpr int kGvaThreads = 21 * 32;
constexpr int kGvaProducerWarp = 20;
constexpr size_t kGvaExtraSmem = size_t(3) * kTileM * kGvTPitch * 4;  // reduction slices of chunks 1..3
SUN_DEVICE void gva_bar_sync(int id) { asm volatile("bar.sync %0, 640;" ::"r"(id) : "memory"); }
SUN_DEVICE void gva_bar_arrive(int id) { asm volatile("bar.arrive %0, 640;" ::"r"(id) : "memory"); }
constexpr int kGvaFull = 4, kGvaEmpty = 5;  // named barriers: T holds a segment / T was read

// segments (one tile's part of a range) of [u0, u1) then [v0, v1), in order
template <typename F>
SUN_DEVICE void gv_for_segments(int KB, int u0, int u1, int v0, int v1, F f) {
#pragma unroll 1
  for (int r = 0; r < 2; ++r) {
    const int a0 = r ? v0 : u0, a1 = r ? v1 : u1;
    for (int u = a0; u < a1;) {
      const int tile = u / KB;
      const int e = min(a1, (tile + 1) * KB);
      f(tile, u, e, u == tile * KB && e == (tile + 1) * KB);
      u = e;
    }
  }
}

template <int NB>
SUN_DEVICE void gva_math(const GemmArgs& a, int u0, int u1, int v0, int v1, const GvSmem& m, int stages, float* Tx) {
  const int kbs = a.wgroup, bn = a.bn, KB = a.ksteps;
  const uint32_t sb = gv_stage_bytes(bn, kbs);
  const int warp = static_cast<int>(threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int ci = warp < 2 ? warp : warp - 4;  // compute index 0..15
  const int rq = ci & 3, ch = ci >> 2;
  const int g = lane >> 2, t = lane & 3;
  float* T = m.T;
  pdl_wait();
  const uint32_t ring_s = smem_u32(m.ring);
  const bool fast = kbs == kGvFastKbs && bn == kGvFastBn;
  const GvBase<NB> base = gv_base<NB>(ring_s, rq, ch, lane);
  int slot = 0, phase = 0, i = 0;
  gv_for_segments(KB, u0, u1, v0, v1, [&](int tile, int s0, int s1, bool whole) {
    float acc[kGvMT][NB][4];
#pragma unroll
    for (int mt = 0; mt < kGvMT; ++mt)
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[mt][j][0] = acc[mt][j][1] = acc[mt][j][2] = acc[mt][j][3] = 0.f;
    for (int u = s0; u < s1;) {
      const int len = min(kbs, s1 - u);
      mbar_wait(&m.full[slot], phase);
      if (threadIdx.x == 0 && u == u0) SUN_STAMP(2);  // first stage landed
      const uint32_t st = ring_s + slot * sb;
      if (fast && len == kGvFastKbs) {
        const uint32_t so = slot * sb;
        GvFrag<NB> f2[2];
        gv_load_fast<NB, 0>(f2[0], base, so);
        gv_load_fast<NB, 1>(f2[1], base, so);
        gv_math<NB, 2>(f2, acc);
        gv_load_fast<NB, 2>(f2[0], base, so);
        gv_load_fast<NB, 3>(f2[1], base, so);
        gv_math<NB, 2>(f2, acc);
      } else {
        auto ld = [&](GvFrag<NB>& f, int ib) {
          gv_load<NB>(f, st + ib * kW4PackedBytes, st + kbs * kW4PackedBytes + ib * 256,
                      st + kbs * (kW4PackedBytes + 256u) + ib * bn * 256, bn, rq, ch, lane);
        };
        int ib = 0;
        for (; ib + 1 < len; ib += 2) {
          GvFrag<NB> f2[2];
          ld(f2[0], ib);
          ld(f2[1], ib + 1);
          gv_math<NB, 2>(f2, acc);
        }
        if (ib < len) {
          GvFrag<NB> f1[1];
          ld(f1[0], ib);
          gv_math<NB, 1>(f1, acc);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&m.empty[slot]);
      u += len;
      if (++slot == stages) {
        slot = 0;
        phase ^= 1;
      }
    }
    if (threadIdx.x == 0 && s1 == (v1 > v0 ? v1 : u1)) SUN_STAMP(3);  // last stage consumed
    if (i > 0) gva_bar_sync(kGvaEmpty);  // the epilogue warps hold the previous segment's rows
    // fragments -> slice ch of T (chunk 0: T, chunks 1..3: Tx): one store round, no barrier
    // among the compute warps; the epilogue group adds the slices in chunk order (the sum
    // ((c0 + c1) + c2) + c3 of gv_consume, bit for bit)
    float* Tq = ch == 0 ? T : Tx + (ch - 1) * (kTileM * kGvTPitch);
#pragma unroll
    for (int mt = 0; mt < kGvMT; ++mt) {
      const int r = 32 * rq + 16 * mt + g;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        float* p0 = Tq + r * kGvTPitch + 8 * j + t;
        float* p1 = Tq + (r + 8) * kGvTPitch + 8 * j + t;
        p0[0] = acc[mt][j][0]; p0[4] = acc[mt][j][1]; p1[0] = acc[mt][j][2]; p1[4] = acc[mt][j][3];
      }
    }
    gva_bar_arrive(kGvaFull);
    ++i;
    (void)tile;
    (void)whole;
  });
}

template <int EPI, int NB>
SUN_DEVICE void gva_epilogue(const GemmArgs& a, int u0, int u1, int v0, int v1, const GvSmem& m, const float* Tx) {
  constexpr int NCOL = 8 * NB;  // columns that can be non-zero (NB = 1: batch <= 8)
  const int KB = a.ksteps, G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  const int row_local = (static_cast<int>(threadIdx.x >> 5) - 2) * 32 + (threadIdx.x & 31);
  pdl_wait();
  load_qkv_meta<EPI>(a, m.epi);  // positions / pages / r_b (ends with the group barrier)
  int nseg = 0;
  gv_for_segments(KB, u0, u1, v0, v1, [&](int, int, int, bool) { ++nseg; });
  int i = 0;
  gv_for_segments(KB, u0, u1, v0, v1, [&](int tile, int, int, bool whole) {
    // residual epilogues: this row's old residual and next-norm gain are loaded before the
    // segment's hand-off, off the tail's critical path (one round trip fewer after the reduction)
    float pres[16], pg = 0.f;
    if constexpr (EPI == EPI_RESID_ADD) {
      const int row = tile * kTileM + row_local;
      const bool in = row < a.n_out;
      const float* base = a.out_f32 + row;
#pragma unroll
      for (int j = 0; j < 16; ++j) pres[j] = (in && j < NCOL && j < a.batch) ? base[static_cast<long long>(j) * a.ldo] : 0.f;
      if (a.norm_w != nullptr) pg = in ? __bfloat162float(a.norm_w[row]) : 0.f;
    }
    float pcs[16], psn[16];  // QKV epilogue: this row's RoPE factors per batch row
    if constexpr (EPI == EPI_QKV_ROPE) {
      const int row = tile * kTileM + row_local;
      const int d = a.head_dim, half = d >> 1, i = row & (d - 1), fi = i < half ? i : i - half;
      const bool is_v = row >= (a.n_q_heads + a.n_kv_heads) * d;
      const int* meta = epi_meta(m.epi);  // positions (load_qkv_meta)
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const bool ok = !is_v && j < NCOL && j < a.batch && row < a.n_out;
        const long long t = static_cast<long long>(meta[j]) * half + fi;
        pcs[j] = ok ? a.rope_cos[t] : 1.f;
        psn[j] = ok ? a.rope_sin[t] : 0.f;
      }
    }
    gva_bar_sync(kGvaFull);
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int o = row_local * kGvTPitch + j;
      v[j] = j < NCOL ? ((m.T[o] + Tx[o]) + Tx[kTileM * kGvTPitch + o]) + Tx[2 * kTileM * kGvTPitch + o] : 0.f;
    }
    if (i + 1 < nseg) gva_bar_arrive(kGvaEmpty);
    ++i;
    if (!whole) {
      // park this segment's rows (slot [2c + piece][128][16] fp32), count the tile; its last
      // contributor adds the slots in contributor order (deterministic) and runs the epilogue
      float* dst = a.sk_part + static_cast<long long>(gv_part_slot(a, G, c, tile)) * (kTileM * 16) + row_local * 16;
#pragma unroll
      for (int j = 0; j < NCOL; j += 4) __stcg(reinterpret_cast<float4*>(dst + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
      __threadfence();
      epi_bar();
      int cf, cl;
      gv_tile_contrib(a, G, tile, cf, cl);
      if (epi_lead_thread()) {
        const unsigned old = atomicAdd(a.sk_flags + tile, 1u);
        *m.flag = (old == static_cast<unsigned>(cl - cf)) ? 1 : 0;
      }
      epi_bar();
      if (*m.flag == 0) return;
      __threadfence();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
      // NB = 1: four partials' 8 columns in flight per round trip; NB = 2: two partials' 16
      constexpr int PF = NB == 1 ? 4 : 2;
      for (int c0 = cf; c0 <= cl; c0 += PF) {
        float4 pp[PF][NCOL / 4];
#pragma unroll
        for (int e = 0; e < PF; ++e) {
          const int slot_e = gv_part_slot(a, G, c0 + e <= cl ? c0 + e : cl, tile);
          const float* src = a.sk_part + static_cast<long long>(slot_e) * (kTileM * 16) + row_local * 16;
#pragma unroll
          for (int q = 0; q < NCOL / 4; ++q) pp[e][q] = __ldcg(reinterpret_cast<const float4*>(src + 4 * q));
        }
#pragma unroll
        for (int e = 0; e < PF; ++e) {
          if (c0 + e > cl) break;
#pragma unroll
          for (int q = 0; q < NCOL / 4; ++q) {
            v[4 * q] += pp[e][q].x; v[4 * q + 1] += pp[e][q].y; v[4 * q + 2] += pp[e][q].z; v[4 * q + 3] += pp[e][q].w;
          }
        }
      }
      if (epi_lead_thread()) a.sk_flags[tile] = 0u;  // self-resetting for the next use
    }
    if constexpr (EPI == EPI_RESID_ADD) epi_chunk<EPI>(a, tile, row_local, 0, v, m.epi, pres, &pg, 1);
    else if constexpr (EPI == EPI_QKV_ROPE) epi_chunk<EPI>(a, tile, row_local, 0, v, m.epi, pcs, psn, 1);
    else epi_chunk<EPI>(a, tile, row_local, 0, v, m.epi);
  });
}

template <int EPI, int NB>
__global__ void __launch_bounds__(kGvaThreads, 1) gemv_w4a_kernel(const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  tl_begin(a.tl, a.tl_idx);
  const int stages = a.stages;
  const GvSmem m = gv_smem(smem, stages, gv_stage_bytes(a.bn, a.wgroup));
  // chunk slices 1..3 of the reduction tile, after the common layout (kGvaExtraSmem)
  float* Tx = reinterpret_cast<float*>(smem + gv_smem_bytes(a.bn, a.wgroup, stages) - 1024);
  const int warp = warp_id_sync();
  int u0, u1, v0, v1;
  gv_range(a, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), u0, u1);
  gv_bal_range(a, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), v0, v1);
  if (u0 == u1) {
    u0 = v0;
    u1 = v1;
    v0 = v1 = 0;
  }
  if (threadIdx.x == 0) SUN_STAMP(0);
  if (warp == kGvaProducerWarp && elect_one()) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&m.full[s], 1);
      mbar_init(&m.empty[s], kGvWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  if (threadIdx.x == 0) SUN_STAMP(1);
  if (warp == kGvaProducerWarp) {
    if (elect_one()) {
      int slot = 0, phase = 0;
      gv_produce(a, u0, u1, m, stages, slot, phase, [] { pdl_wait(); }, kGvMaxStages, /*first_wait=*/a.gv_first_wait != 0);
      if (v0 < v1) gv_produce(a, v0, v1, m, stages, slot, phase, [] {}, 0);
      prefetch_next_weights(a);
    }
    __syncwarp();
  } else if (warp >= 2 && warp < 6) {
    gva_epilogue<EPI, NB>(a, u0, u1, v0, v1, m, Tx);
  } else {
    gva_math<NB>(a, u0, u1, v0, v1, m, stages, Tx);
  }
  if (threadIdx.x == 64) SUN_STAMP(5);  // (epilogue warp) last epilogue done
  if (a.tl != nullptr || a.stamps != nullptr) __syncthreads();  // profiling: the exit stamps after every role
  if (threadIdx.x == 0) SUN_STAMP(6);
  tl_end(a.tl, a.tl_idx);
}

// ---------------------------------------------------------------------------
// Small-batch QSUN layer chain: O -> gate_up -> down -> next layer's QKV as GEMV phases of
// one persistent launch (one CTA per SM, all resident). The ring and its producer run across
// the phase boundaries: the next phase's weight and scale stages stream in while the compute
// warps finish the current phase's tail, so a boundary costs the tail and a grid-wide count
// (every CTA adds 1 after its last epilogue of a phase; the next phase's activation copies
// and epilogue metadata wait for count >= G x phase), not a launch, a ring ramp and a cold
// first stage per GEMM. Same split-K partials / tile counters as the separate launches.
// ---------------------------------------------------------------------------
constexpr int kGvChainMaxPhases = 4;
struct GvChainArgs {
  GemmArgs ph[kGvChainMaxPhases];  // O (RESID_ADD), gate_up (SWIGLU), down (RESID_ADD), next QKV (QKV_ROPE)
  int nph;
  unsigned* bar;  // [2]: phases completed x CTAs, CTAs exited (zeroed once, self-resetting)
  int pre;        // stages of a phase p >= 1 whose weights are issued before its grid count: deeper
                  // prefetch saturates the HBM under the previous phase's tail round trips
  unsigned long long* stamps;  // profiling: per CTA [16] = per phase p: [4p] gate passed, [4p+1] first
                               // stage landed, [4p+2] last stage consumed, [4p+3] phase done
  unsigned long long* tl;
  int tl_idx;
};

SUN_DEVICE void gv_wait_count(const unsigned* bar, unsigned target) {
  if (target == 0) return;
  const unsigned long long t0 = gtimer();
  while (ld_acquire_u32(bar) < target) {
    __nanosleep(64);
    if (gtimer() - t0 > 2000000000ull) __trap();  // a grid that cannot become resident fails, not hangs
  }
}

template <int NB>
__global__ void __launch_bounds__(kGvThreads, 1) gemv_chain_w4_kernel(const __grid_constant__ GvChainArgs c) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  tl_begin(c.tl, c.tl_idx);
  const GemmArgs& a0 = c.ph[0];
  const int stages = a0.stages;
  const GvSmem m = gv_smem(smem, stages, gv_stage_bytes(a0.bn, a0.wgroup));
  const int warp = warp_id_sync();
  const int G = static_cast<int>(gridDim.x), cta = static_cast<int>(blockIdx.x);
  gv_init_ring(m, stages);
  pdl_launch_dependents();
  int slot = 0, phase = 0;
  if (warp == kGvWarps) {
    if (elect_one()) {
      for (int p = 0; p < c.nph; ++p) {
        int u0, u1;
        gv_range(c.ph[p], cta, G, u0, u1);
        const unsigned target = static_cast<unsigned>(G * p);
        gv_produce(c.ph[p], u0, u1, m, stages, slot, phase, [&] {
          if (p == 0) pdl_wait();
          else gv_wait_count(c.bar, target);
        }, p == 0 ? kGvMaxStages : c.pre);
      }
    }
  } else {
    for (int p = 0; p < c.nph; ++p) {
      const GemmArgs& a = c.ph[p];
      int u0, u1;
      gv_range(a, cta, G, u0, u1);
      const unsigned target = static_cast<unsigned>(G * p);
      auto gate = [&] {
        if (p == 0) {
          pdl_wait();
        } else {
          if (threadIdx.x == 0) gv_wait_count(c.bar, target);
          gv_bar();
        }
      };
      unsigned long long* pst = c.stamps ? c.stamps + cta * 16 + 4 * p : nullptr;
      if (p == 1) gv_consume<EPI_SWIGLU, NB>(a, u0, u1, m, stages, slot, phase, gate, pst);
      else if (p == 3) gv_consume<EPI_QKV_ROPE, NB>(a, u0, u1, m, stages, slot, phase, gate, pst);
      else gv_consume<EPI_RESID_ADD, NB>(a, u0, u1, m, stages, slot, phase, gate, pst);
      gv_bar();  // every epilogue store of this CTA's phase-p work is issued
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(c.bar, 1u);
        if (pst) pst[3] = gtimer();
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(c.bar + 1, 1u) == static_cast<unsigned>(G - 1)) {  // last CTA out rearms
    c.bar[0] = 0u;
    c.bar[1] = 0u;
  }
  tl_end(c.tl, c.tl_idx);
}

}  // namespace sun
