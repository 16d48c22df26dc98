// gemm_tc.cuh — tcgen05/TMEM swap-AB GEMM for the decode module's linear layers.
//
//   D^T[n_out, B] = W[n_out, K] . X[B, K]^T
//
// Weight rows are the MMA M dimension (128 per tile), the cross-model decode
// batch is the MMA N dimension (bn = round_up(B, 16) <= 256). K advances 128 per
// pipeline stage (two 64-wide SWIZZLE_128B atoms). Both operands are stored in
// the exact shared-memory image the UMMA descriptors expect, so every stage is
// one linear cp.async.bulk copy:
//   * SUN-BLK weights: [m_tiles][k/64][128 rows][64 cols] with 16-byte chunk c of
//     row r at position c ^ (r & 7) — a tile's whole K is one sequential stream;
//   * SUN-ACT activations: [k/64][bn rows][64 cols], same swizzle, written in
//     that form by the kernels that produce them (GEMM epilogues, attention).
// Per-request cost dominates small bulk copies on B200 (a 4 KB stream reaches
// ~2.3 TB/s, 16 KB 6.3, 64 KB 7.2; scripts/probe/stream_probe.cu), hence the
// large linear requests. Weights and activations have separate rings, each fed by
// its own producer warp, so the weight ring runs ahead by its whole depth.
// QSUN W4 (gemm_w4.cuh): packed int4 + scales stages, converter warps dequantise
// in registers and store the A tile into tensor memory.
//
// Schedules: with <= 148 tiles the S CTAs of a thread-block cluster split K for
// one tile and reduce through DSMEM in fixed rank order (deterministic, one
// wave, no global partials) — or through L2 ("virtual clusters") where S-CTA
// hardware clusters do not pack the GPCs; with more tiles one persistent CTA per
// SM walks a contiguous range of whole tiles with a double-buffered TMEM
// accumulator so a tile's epilogue overlaps the next tile's stream (stream-K is
// available behind SUN_GEMM_SCHED).
// Warp roles, bf16 (352 threads): 0 = weight producer, 1 = TMEM owner + single-
// thread MMA issuer, 2..5 = epilogue group A, 6 = activation producer, 7..10 =
// epilogue group B (groups take alternate 16-column chunks). W4 (480 threads):
// 0 = weight producer, 1 = MMA, 2..5 = epilogue, 6..13 = converters (TMEM lane
// group = warp % 4), 14 = activation producer. Weights are issued before
// griddepcontrol.wait (they never depend on the previous kernel).
//
// Replaces the weight term `decoder_weight_bytes / (mbu * hbm_bandwidth)` of
// the reference's step price (poolsim costmodel.py:101-113) with real work.
#pragma once
#include <type_traits>

#include "sun_common.cuh"

namespace sun {

enum EpiKind : int {
  EPI_STORE_F32 = 0,  // out_f32[b*ldo + row] = acc
  EPI_RESID_ADD = 1,  // out_f32[b*ldo + row] += acc           (O-proj, down-proj)
  EPI_QKV_ROPE = 2,   // +bias, RoPE(q,k), q -> bf16, k/v -> paged KV cache
  EPI_SWIGLU = 3,     // rows pair-interleaved (2i gate, 2i+1 up): act = silu(gate) * up
  EPI_LOGITS = 4,     // logits fp32 + per-tile (max, argmax) per batch column
};

struct GemmArgs {
  const uint8_t* wblk;     // bf16 weights, SUN-BLK
  const uint8_t* w4_packed;  // QSUN: SUN-W4 packed int4 (tile-contiguous 128x64 B blocks)
  const __nv_bfloat16* w4_scales;  // QSUN: tile-major [m_tiles][k/128][128 row-interleaved, w4_scale_pos]
  const uint8_t* xact;     // activations, SUN-ACT with bn rows per atom
  int n_out;         // rows of W (incl. zero padding rows for SWIGLU)
  int k;             // reduction length
  int batch;         // valid batch columns
  int bn;            // padded N: multiple of 16, <= 256
  int kb64;          // ceil(k / 64): 64-wide k blocks per tile
  int ksteps;        // ceil(kb64 / 2): 128-wide pipeline stages per tile
  int m_tiles;       // ceil(n_out / 128)
  int splits;        // split-K factor S (> 1: S CTAs per tile)
  int vcluster;      // 1: the S CTAs of a tile are not a hardware cluster: partials and the
                     // rank-sliced reduction go through L2 (sk_part) with a per-tile counter
  int stages;        // smem pipeline depth (W4: weight stages of wgroup K blocks)
  int gv_first_wait; // W4 GEMV (epilogue-group kernel): the rest of the ring after the first stage landed
  int xstages;       // W4: activation stages of xk K blocks
  int wgroup;        // W4: K blocks per weight stage (packed [wgroup][8 KB] | scales [wgroup][256 B])
  int xk;            // W4: K blocks per activation stage
  int push_bytes;    // hardware cluster split-K, push mode (> 0): every rank bulk-copies the
                     // chunks other ranks own into their receive areas (this many bytes of
                     // smem after the barriers, [S-1 senders][ceil(bn/16/S) chunks][8 KB]);
                     // 0: owners pull the peers' parked partials over DSMEM
  // STORE / RESID / LOGITS
  float* out_f32;
  long long ldo;
  // SWIGLU (act, written SUN-ACT with bn rows) / QKV (q, row-major with ldb)
  __nv_bfloat16* out_bf16;
  long long ldb;
  int n_valid_out;   // SWIGLU: ffn width f (outputs j < f are written)
  // QKV
  const __nv_bfloat16* bias;  // [n_out] or null
  const float* rope_cos;      // [max_pos][head_dim/2]
  const float* rope_sin;
  const int* positions;       // [B] position of the token being decoded
  const int* block_tables;    // [B][bt_stride]
  int bt_stride;
  __nv_bfloat16* kv_base;     // paged pool, page = [L][2][n_kv][P][d]
  long long page_stride;      // elements per page
  int layer;
  int n_q_heads;
  int n_kv_heads;
  int head_dim;
  int page_size;
  int max_pos;                // positions are clamped to [0, max_pos) for the RoPE tables
  long long kv_pages;         // pool size: an append page outside [0, kv_pages) is not written
  // LOGITS
  float* amax_val;  // [m_tiles][bn]
  int* amax_idx;    // [m_tiles][bn]
  // Fused RMSNorm, factored (see epi_chunk): producers (RESID_ADD) write
  // xg = bf16(x * g_next) in SUN-ACT plus per-tile sums of squares; consumers
  // (QKV / SWIGLU / LOGITS) scale their accumulators by r_b = rsqrt(mean + eps).
  const __nv_bfloat16* norm_w;  // producer: gain of the next RMSNorm [n_out] (null: off)
  __nv_bfloat16* xg_out;        // producer: SUN-ACT output, bn rows
  float* ss_out;                // producer: [m_tiles][bn] partial sums of squares
  const float* ss_in;           // consumer: [ss_tiles][bn] (null: no scaling)
  int ss_tiles;
  int norm_h;                   // hidden size (mean denominator)
  float norm_eps;
  // Stream-K schedule (sk_units > 0): the m_tiles x ksteps work units are split
  // evenly over the grid; a CTA whose range starts inside a tile parks its fp32
  // partial in sk_part[blockIdx.x] and raises sk_flags[blockIdx.x]; the tile's
  // owner (the CTA holding k-step 0) adds the partials in CTA order, runs the
  // epilogue and clears the flags (zeroed once, self-resetting).
  int sk_units;
  float* sk_part;      // [grid][bn/16][128][16] fp32
  unsigned* sk_flags;  // [grid]
  // L2 prefetch of the next GEMM's first weight stages, issued by this kernel's
  // producer once its own loads are out (fills HBM during the epilogue/launch gap)
  const uint8_t* pf_w;  // next weights (SUN-BLK or SUN-W4 packed); null = off
  int pf_w4, pf_m_tiles, pf_ksteps, pf_kb64, pf_splits, pf_grid, pf_sk_units, pf_bytes;
  // optional per-CTA %globaltimer stamps [gridDim.x][8] (profiling only)
  unsigned long long* stamps;
  unsigned long long* tl;  // step timeline slot array (profiling only) and this launch's index
  int tl_idx;
};

SUN_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SUN_STAMP(i) \
  do { if (a.stamps) a.stamps[blockIdx.x * 16 + (i)] = gtimer(); } while (0)

constexpr int kGemmThreads = 352;  // producer(W), MMA, epilogue group A (4), producer(X), epilogue group B (4)
#ifndef SUN_W4_CONV_WARPS
#define SUN_W4_CONV_WARPS 8
#endif
// converter warps: 4 per SM sub-partition (lane group) hide ALU / TMEM-store latency;
// each takes 128 / (warps / 4) K elements of its 32 rows per 128-wide K block
constexpr int kW4ConvThreads = SUN_W4_CONV_WARPS * 32;
constexpr int kW4KParts = SUN_W4_CONV_WARPS / 4;
constexpr int kW4Chunks = 4 / kW4KParts;  // 16-byte packed chunks (32 k) per converter thread
constexpr int kW4Threads = 192 + kW4ConvThreads + 32;  // + the activation-producer warp
constexpr int kTileM = 128;
constexpr int kTileK = 64;
constexpr uint32_t kTileWBytes = kTileM * kTileK * 2;  // 16 KB: one SUN-BLK block
constexpr uint32_t kW4PackedBytes = kTileM * 128 / 2;  // 8 KB: one SUN-W4 block (128 x 128)
__host__ __device__ inline uint32_t w4_wstage_bytes(int wgroup) { return static_cast<uint32_t>(wgroup) * (kW4PackedBytes + 256u); }
constexpr int kMaxWStages = 16, kMaxXStages = 8;
constexpr int kW4MaxABufs = 6;
// SUN-W4 stores a K block's 128 row scales row-interleaved: row r at (r & 7) * 16 + (r >> 3)
// (the small-batch GEMV's lane g reads rows g, g + 8, ... as one 16-byte load)
__host__ __device__ inline int w4_scale_pos(int r) { return ((r & 7) << 4) | (r >> 3); }  // W4: dequantised 128x128 A tiles (64 TMEM columns each) at the top of TMEM

// column meta: pos[256], page[256], r_b[256] | per epilogue group: partner staging [16][128] f32 + 512 B scratch
constexpr uint32_t kEpiGroupBytes = 16 * kTileM * 4 + 512;
constexpr uint32_t kEpiSmemBytes = 3072 + 2 * kEpiGroupBytes;

// byte offset of activation element (row b, column k) in SUN-ACT with `rows` rows per atom
__host__ __device__ inline long long act_offset(int b, long long k, int rows) {
  return (k >> 6) * (static_cast<long long>(rows) * 128) + static_cast<long long>(b) * 128 +
         (((((k & 63) >> 3) ^ (b & 7))) << 4) + (k & 7) * 2;
}

// bf16: a weight stage is one 128-wide K step (two 16 KB SUN-BLK blocks), an
// activation stage the matching bn x 128 SUN-ACT slice; separate rings.
__host__ __device__ inline uint32_t gemm_stage_bytes(int bn, bool w4) { return 2u * kTileWBytes; }
__host__ __device__ inline uint32_t gemm_xstage_bytes(int bn) { return static_cast<uint32_t>(bn) * 256u; }
__host__ __device__ inline size_t gemm_smem_bytes(int bn, int stages, int xstages) {
  return 1024 + static_cast<size_t>(stages) * 2u * kTileWBytes + static_cast<size_t>(xstages) * gemm_xstage_bytes(bn) +
         kEpiSmemBytes + 1024;
}
__host__ __device__ inline uint32_t w4_xstage_bytes(int bn, int xk) { return static_cast<uint32_t>(xk * bn) * 256u; }
__host__ __device__ inline size_t gemm_smem_bytes_w4(int bn, int wgroup, int wstages, int xk, int xstages) {
  return 1024 + (static_cast<size_t>(wstages) * w4_wstage_bytes(wgroup) + 1023) / 1024 * 1024 +
         static_cast<size_t>(xstages) * w4_xstage_bytes(bn, xk) + kEpiSmemBytes + 1024;
}

__host__ __device__ inline uint32_t tmem_cols_for(int bn) {
  uint32_t c = 32;
  while (c < static_cast<uint32_t>(2 * bn)) c <<= 1;
  return c;
}
// accumulator buffers: 2 (epilogue of tile i overlaps tile i+1) unless W4's A tiles leave no room
__host__ __device__ inline int acc_buffers(int bn, bool w4) { return (w4 && 2 * bn > 512 - 2 * 64) ? 1 : 2; }
// W4 A-tile ring depth: what the 512 TMEM columns leave after the accumulators
__host__ __device__ inline int w4_abufs(int bn) {
  const int n = (512 - acc_buffers(bn, true) * bn) / 64;
  return n < kW4MaxABufs ? n : kW4MaxABufs;
}

// Epilogue warps form groups of four (one per TMEM lane quarter): group A =
// warps 2..5, group B = warps 7..10 (bf16 kernel only); a group takes every other
// 16-column chunk, with its own named barrier and staging smem.
SUN_DEVICE int epi_grp() { return threadIdx.x >= 224 ? 1 : 0; }
SUN_DEVICE bool epi_lead_warp() { return static_cast<int>(threadIdx.x >> 5) == (epi_grp() ? 7 : 2); }
SUN_DEVICE bool epi_lead_thread() { return threadIdx.x == (epi_grp() ? 224u : 64u); }
SUN_DEVICE void epi_bar() {  // immediate ids keep the kernel's named-barrier count small
  if (epi_grp()) asm volatile("bar.sync 3, 128;" ::: "memory");
  else asm volatile("bar.sync 1, 128;" ::: "memory");
}
SUN_DEVICE int* epi_meta(float* epi) { return reinterpret_cast<int*>(epi); }
SUN_DEVICE float* epi_stage(float* epi) {
  return reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(epi) + 3072 + epi_grp() * kEpiGroupBytes);
}

template <int EPI, int NC = 16>  // NC: columns in this chunk (16, or 8 for a half chunk)
SUN_DEVICE void epi_chunk(const GemmArgs& a, int m_tile, int row_local, int c0, float (&v)[NC], float* epi,
                          const float* pre0 = nullptr, const float* pre1 = nullptr, int pstride = 1) {
  const int row = m_tile * kTileM + row_local;
  const int B = a.batch;
  float* stage_f32 = epi_stage(epi);
  float* red_val = stage_f32 + 16 * kTileM;
  int* red_idx = reinterpret_cast<int*>(red_val + 64);
  if (a.ss_in != nullptr) {  // consumer of a factored RMSNorm: W.(x*g) * r_b
    const float* rb = reinterpret_cast<const float*>(epi_meta(epi) + 512);
#pragma unroll
    for (int j = 0; j < NC; ++j) v[j] *= rb[c0 + j];
  }
  if constexpr (EPI == EPI_STORE_F32 || EPI == EPI_RESID_ADD) {
    if constexpr (EPI == EPI_RESID_ADD) {
      if (a.norm_w != nullptr) {  // producer of the next RMSNorm's operand + sums of squares
        float nw[NC];
        const bool in = row < a.n_out;
        float* base = a.out_f32 + static_cast<long long>(c0) * a.ldo + row;
        float old[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) old[j] = pre0 ? pre0[j * pstride] : ((in && c0 + j < B) ? base[j * a.ldo] : 0.f);
        const float g = pre1 ? pre1[0] : (in ? __bfloat162float(a.norm_w[row]) : 0.f);
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          nw[j] = old[j] + v[j];
          if (in && c0 + j < B) {
            base[j * a.ldo] = nw[j];
            *reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(a.xg_out) + act_offset(c0 + j, row, a.bn)) =
                __float2bfloat16_rn(nw[j] * g);
          }
          nw[j] = in ? nw[j] * nw[j] : 0.f;
        }
        // sum of squares over the tile's 128 rows, fixed order: warp tree, then 4 warps
        const int lane = threadIdx.x & 31;
        const int q = (threadIdx.x / 32) & 3;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) nw[j] += __shfl_xor_sync(0xffffffffu, nw[j], off);
        }
        if (lane == 0) {
#pragma unroll
          for (int j = 0; j < NC; ++j) red_val[q * NC + j] = nw[j];
        }
        epi_bar();
        if (epi_lead_warp() && lane < NC) {
          const float t = ((red_val[lane] + red_val[NC + lane]) + red_val[2 * NC + lane]) + red_val[3 * NC + lane];
          a.ss_out[static_cast<long long>(m_tile) * a.bn + c0 + lane] = t;
        }
        epi_bar();
        return;
      }
    }
    if (row < a.n_out) {
      float* base = a.out_f32 + static_cast<long long>(c0) * a.ldo + row;
      if constexpr (EPI == EPI_RESID_ADD) {
        // issue all 16 residual loads before any store (one memory round trip)
        float old[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) old[j] = pre0 ? pre0[j * pstride] : ((c0 + j < B) ? base[j * a.ldo] : 0.f);
#pragma unroll
        for (int j = 0; j < NC; ++j)
          if (c0 + j < B) base[j * a.ldo] = old[j] + v[j];
      } else {
#pragma unroll
        for (int j = 0; j < NC; ++j)
          if (c0 + j < B) base[j * a.ldo] = v[j];
      }
    }
  } else if constexpr (EPI == EPI_LOGITS) {
    const int lane = threadIdx.x & 31;
    const int q = (threadIdx.x / 32) & 3;
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int b = c0 + j;
      float val = v[j];
      int idx = row;
      if (row >= a.n_out) {
        val = -INFINITY;
        idx = 0x7fffffff;
      } else if (b < B) {
        a.out_f32[static_cast<long long>(b) * a.ldo + row] = val;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, val, off);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
        if (ov > val || (ov == val && oi < idx)) {
          val = ov;
          idx = oi;
        }
      }
      if (lane == 0) {
        red_val[q * NC + j] = val;
        red_idx[q * NC + j] = idx;
      }
    }
    epi_bar();
    if (epi_lead_warp() && lane < NC) {
      float val = red_val[lane];
      int idx = red_idx[lane];
#pragma unroll
      for (int w = 1; w < 4; ++w) {
        const float ov = red_val[w * NC + lane];
        const int oi = red_idx[w * NC + lane];
        if (ov > val || (ov == val && oi < idx)) {
          val = ov;
          idx = oi;
        }
      }
      a.amax_val[static_cast<long long>(m_tile) * a.bn + c0 + lane] = val;
      a.amax_idx[static_cast<long long>(m_tile) * a.bn + c0 + lane] = idx;
    }
    epi_bar();
  } else if constexpr (EPI == EPI_SWIGLU) {
    // tile rows 2i / 2i+1 are gate / up of output m_tile*64 + i: the partner is the
    // neighbouring lane (no staging, no barrier). The gate lane writes the chunk's first
    // H = NC/2 columns, the up lane the rest (the sigmoid's division was the epilogue's
    // critical path when one thread did all NC), one shuffle per column pair: the gate
    // lane sends v[jj + H], the up lane v[jj]; indices stay compile-time (no local memory).
    constexpr int H = NC / 2;
    const bool is_gate = (row_local & 1) == 0;
    const int jo = m_tile * 64 + (row_local >> 1);
    const int cb = c0 + (is_gate ? 0 : H);
#pragma unroll
    for (int jj = 0; jj < H; ++jj) {
      const float recv = __shfl_xor_sync(0xffffffffu, is_gate ? v[jj + H] : v[jj], 1);
      const float g = is_gate ? v[jj] : recv;
      const float u = is_gate ? recv : v[jj + H];
      const int b = cb + jj;
      if (jo < a.n_valid_out && b < B) {
        // fast exp / divide (~2 ulp in fp32, below the bf16 rounding of the output):
        // the IEEE versions were a third of the gate_up epilogue tail
        const float s = __fdividef(g, 1.f + __expf(-g));
        *reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(a.out_bf16) + act_offset(b, jo, a.bn)) =
            __float2bfloat16_rn(s * u);
      }
    }
  } else {
    // QKV_ROPE needs a partner row half a head away: stage through smem.
    epi_bar();  // previous chunk's partner reads are done
    {
      const float bias = (a.bias != nullptr && row < a.n_out) ? __bfloat162float(a.bias[row]) : 0.f;
#pragma unroll
      for (int j = 0; j < NC; ++j) v[j] += bias;
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) stage_f32[j * kTileM + row_local] = v[j];
    epi_bar();
    {
      if (row < a.n_out) {
        const int d = a.head_dim;
        const int half = d >> 1;
        const int qd = a.n_q_heads * d;
        const int kd = a.n_kv_heads * d;
        const int i = row & (d - 1);  // head_dim is 64 or 128 (sun_decoder_create)
        const int fi = i < half ? i : i - half;
        const int partner = i < half ? row_local + half : row_local - half;
        const bool is_v = row >= qd + kd;
        const int* meta = epi_meta(epi);  // [0,256) pos, [256,512) page
        // hoisted, independent loads: one round trip for the 32 table values
        float cs[NC], sn[NC], pv[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const int pos = meta[(c0 + j) & 255];
          const bool ok = !is_v && (c0 + j < B);
          cs[j] = pre0 ? pre0[j] : (ok ? a.rope_cos[static_cast<long long>(pos) * half + fi] : 1.f);
          sn[j] = pre1 ? pre1[j] : (ok ? a.rope_sin[static_cast<long long>(pos) * half + fi] : 0.f);
          pv[j] = stage_f32[j * kTileM + partner];
        }
        const bool lo_half = i < half;
        if (row < qd) {
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            if (c0 + j < B) {
              const float o = lo_half ? (v[j] * cs[j] - pv[j] * sn[j]) : (v[j] * cs[j] + pv[j] * sn[j]);
              a.out_bf16[static_cast<long long>(c0 + j) * a.ldb + row] = __float2bfloat16_rn(o);
            }
          }
        } else {
          const int kvsel = is_v ? 1 : 0;
          const int g = (row - qd - kvsel * kd) >> (d == 128 ? 7 : 6);
          const long long inner = ((static_cast<long long>(a.layer * 2 + kvsel) * a.n_kv_heads + g) * a.page_size) * d + i;
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            if (c0 + j < B) {
              const float o = is_v ? v[j] : (lo_half ? (v[j] * cs[j] - pv[j] * sn[j]) : (v[j] * cs[j] + pv[j] * sn[j]));
              const int pos = meta[(c0 + j) & 255];
              const int page = meta[256 + ((c0 + j) & 255)];
              if (page < 0) continue;  // invalid append page (flagged at step start): no write
              a.kv_base[static_cast<long long>(page) * a.page_stride + inner + static_cast<long long>(pos & 15) * d] =
                  __float2bfloat16_rn(o);
            }
          }
        }
      }
    }
  }
}


// SUN-BLK: W[rows][k] bf16 -> [m_tiles][k/64][128 rows][64 cols] with the
// 16-byte chunk c of row r stored at chunk position c ^ (r & 7) (SWIZZLE_128B
// image), zero padded to whole tiles / k-blocks. One-time, at weight load.
__global__ void block_weights_kernel(const __nv_bfloat16* __restrict__ w, long long rows, long long k, int kb64,
                                     uint8_t* __restrict__ out) {
  const long long blk = blockIdx.x;  // tile * kb64 + kb
  const long long tile = blk / kb64;
  const int kb = static_cast<int>(blk % kb64);
  uint8_t* dst = out + blk * kTileWBytes;
  for (int i = threadIdx.x; i < kTileM * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    const long long row = tile * kTileM + r;
    const long long col = static_cast<long long>(kb) * kTileK + c * 8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (row < rows && col < k) v = *reinterpret_cast<const uint4*>(w + row * k + col);  // k % 8 == 0
    *reinterpret_cast<uint4*>(dst + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
}

// Row-major bf16 X[rows][k] (stride ld) -> SUN-ACT with `act_rows` rows per atom.
__global__ void block_activations_kernel(const __nv_bfloat16* __restrict__ x, int rows, long long k, long long ld,
                                         int act_rows, uint8_t* __restrict__ out) {
  const long long n = static_cast<long long>(act_rows) * ((k + 63) / 64) * 8;  // 16-byte chunks
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i & 7);
    const int b = static_cast<int>((i >> 3) % act_rows);
    const long long kb = (i >> 3) / act_rows;
    const long long col = kb * 64 + c * 8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (b < rows && col < k) v = *reinterpret_cast<const uint4*>(x + b * ld + col);
    *reinterpret_cast<uint4*>(out + act_offset(b, col, act_rows)) = v;
  }
}

// Unsplit tile: TMEM accumulator -> fused epilogue directly.
template <int EPI>
SUN_DEVICE void direct_epilogue(const GemmArgs& a, int tile, uint32_t taddr, float* epi, int ngroups) {
  const int q = (threadIdx.x / 32) & 3;
  const int row_local = q * 32 + (threadIdx.x & 31);
  float v[16];
  for (int c0 = 16 * epi_grp(); c0 < a.bn; c0 += 16 * ngroups) {
    tmem_ld16(taddr + c0, v);
    epi_chunk<EPI>(a, tile, row_local, c0, v, epi);
  }
}

// Split-K epilogue inputs that do not depend on this GEMM's result (previous
// residual + next-norm gain; RoPE cos/sin of the columns), loaded by the epilogue
// warps while the main loop still runs: under a saturated HBM a global round
// trip costs ~2 us, which otherwise sat between the reduction and the stores.
struct EpiPreNone {};
struct EpiPre {
  float p0[16], p1[16];
  int c0 = -1;
};
template <int EPI>
SUN_DEVICE void epi_preload(const GemmArgs& a, int m_tile, int row_local, int c0, int nc, float* epi, EpiPre& pr) {
  const int row = m_tile * kTileM + row_local;
  const int B = a.batch;
  pr.c0 = c0;
  if constexpr (EPI == EPI_RESID_ADD) {
    const bool in = row < a.n_out;
    const float* base = a.out_f32 + static_cast<long long>(c0) * a.ldo + row;
#pragma unroll
    for (int j = 0; j < 16; ++j) pr.p0[j] = (j < nc && in && c0 + j < B) ? base[j * a.ldo] : 0.f;
    pr.p1[0] = (a.norm_w != nullptr && in) ? __bfloat162float(a.norm_w[row]) : 0.f;
  } else if constexpr (EPI == EPI_QKV_ROPE) {
    const int d = a.head_dim, half = d >> 1, qd = a.n_q_heads * d, kd = a.n_kv_heads * d;
    const int i = row & (d - 1);
    const int fi = i < half ? i : i - half;
    const bool is_v = row >= qd + kd;
    const int* meta = epi_meta(epi);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int pos = meta[(c0 + j) & 255];
      const bool ok = j < nc && row < a.n_out && !is_v && (c0 + j < B);
      pr.p0[j] = ok ? a.rope_cos[static_cast<long long>(pos) * half + fi] : 1.f;
      pr.p1[j] = ok ? a.rope_sin[static_cast<long long>(pos) * half + fi] : 0.f;
    }
  }
}

// Per-column epilogue metadata, once per CTA: QKV positions / KV pages, and the
// factored RMSNorm scale r_b = rsqrt(sum_t ss[t][b] / h + eps) (tile order fixed).
template <int EPI>
SUN_DEVICE void load_qkv_meta(const GemmArgs& a, float* epi) {  // epilogue group A
  int* meta = epi_meta(epi);
  if constexpr (EPI == EPI_QKV_ROPE) {
    for (int b = threadIdx.x - 64; b < a.bn; b += 128) {
      int pos = b < a.batch ? a.positions[b] : 0;
      const bool pos_ok = pos >= 0 && pos < a.max_pos;  // (flagged by embed_norm_kernel)
      pos = pos_ok ? pos : 0;
      int page = (b < a.batch && pos_ok) ? a.block_tables[static_cast<long long>(b) * a.bt_stride + (pos >> 4)] : -1;
      if (page < 0 || static_cast<long long>(page) >= a.kv_pages) page = -1;  // 16-token pages; -1: no append
      meta[b] = pos;
      meta[256 + b] = page;
    }
  }
  if (a.ss_in != nullptr) {
    float* rb = reinterpret_cast<float*>(meta + 512);
    for (int b = threadIdx.x - 64; b < a.bn; b += 128) {
      // issue 16 independent loads per round trip, then add in tile order (the
      // sum is unchanged; a load-add-load chain cost one L2 round trip per tile,
      // ~10 us for 32 tiles — longer than the whole QKV main loop)
      float t = 0.f;
      for (int i0 = 0; i0 < a.ss_tiles; i0 += 16) {
        float x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          x[i] = (i0 + i < a.ss_tiles) ? a.ss_in[static_cast<long long>(i0 + i) * a.bn + b] : 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i0 + i < a.ss_tiles) t += x[i];
      }
      rb[b] = rsqrtf(t / static_cast<float>(a.norm_h) + a.norm_eps);
    }
  }
  epi_bar();
}

// Prefetch into L2 the first pf_bytes of the weight stream of every next-GEMM
// CTA c == blockIdx.x (mod gridDim.x), using the next launch's schedule.
SUN_DEVICE void prefetch_next_weights(const GemmArgs& a) {
  if (a.pf_w == nullptr) return;
  const int KS = a.pf_ksteps;
  for (int c = blockIdx.x; c < a.pf_grid; c += gridDim.x) {
    long long u0, u1;
    if (a.pf_splits > 1) {
      const int S = a.pf_splits, t = c / S, r = c % S;
      u0 = static_cast<long long>(t) * KS + r * KS / S;
      u1 = static_cast<long long>(t) * KS + (r + 1) * KS / S;
    } else if (a.pf_sk_units > 0) {
      u0 = static_cast<long long>(c) * a.pf_sk_units / a.pf_grid;
      u1 = static_cast<long long>(c + 1) * a.pf_sk_units / a.pf_grid;
    } else {
      u0 = static_cast<long long>(c) * a.pf_m_tiles / a.pf_grid * KS;
      u1 = static_cast<long long>(c + 1) * a.pf_m_tiles / a.pf_grid * KS;
    }
    long long off, len;
    if (a.pf_w4) {  // 8 KB packed per K block, contiguous along the range
      off = u0 * kW4PackedBytes;
      len = (u1 - u0) * kW4PackedBytes;
    } else {  // SUN-BLK: 16 KB blocks, unit = two blocks (one for an odd tail)
      const long long t0 = u0 / KS, t1 = (u1 - 1) / KS;
      const long long b0 = t0 * a.pf_kb64 + 2 * (u0 % KS);
      const long long b1 = t1 * a.pf_kb64 + min(2 * ((u1 - 1) % KS) + 2, static_cast<long long>(a.pf_kb64));
      off = b0 * kTileWBytes;
      len = (b1 - b0) * kTileWBytes;
    }
    const uint32_t bytes = static_cast<uint32_t>(min(len, static_cast<long long>(a.pf_bytes))) & ~15u;
    if (bytes > 0)
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a.pf_w + off), "r"(bytes),
                   "l"(kEvictLast)
                   : "memory");
  }
}

SUN_DEVICE unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SUN_DEVICE void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// fp32 split-K partial tile layout [bn/16][4][128 rows][4]: float4 j (columns
// c0+4j..c0+4j+3) of row r; a warp's float4 accesses are 512 B contiguous, so
// shared-memory / DSMEM reads are conflict-free and global ones fully coalesced.
SUN_DEVICE int part_index(int c0, int j, int row) { return (c0 >> 4) * (kTileM * 16) + (j * kTileM + row) * 4; }

// Stream-K contributor: TMEM accumulator -> sk_part[blockIdx.x] (chunk-major
// [bn/16][128][16], a warp's chunk is 2 KB contiguous), then raise the flag.
SUN_DEVICE void sk_store_partial(const GemmArgs& a, uint32_t taddr, int row_local) {
  float* base = a.sk_part + static_cast<long long>(blockIdx.x) * a.bn * kTileM;
  float v[16];
  for (int c0 = 0; c0 < a.bn; c0 += 16) {
    tmem_ld16(taddr + c0, v);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      __stcg(reinterpret_cast<float4*>(base + part_index(c0, j, row_local)),
             make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
  }
  __threadfence();
  epi_bar();
  if (threadIdx.x == 64) {
    st_release_u32(a.sk_flags + blockIdx.x, 1u);
    SUN_STAMP(13);
  }
}

// Stream-K owner of `tile` (its range holds k-step 0 but not the last): wait for
// the contributors (the following CTAs whose ranges start inside the tile), pull
// their partials into the idle stage ring with bulk copies (one round trip), add
// them in CTA order to the TMEM accumulator and run the fused epilogue.
template <int EPI>
SUN_DEVICE void sk_owner_epilogue(const GemmArgs& a, int tile, uint32_t taddr, int row_local, float* epi,
                                  uint8_t* ring, uint64_t* bar) {
  const int G = static_cast<int>(gridDim.x);
  const int c = static_cast<int>(blockIdx.x);
  const long long tile_end = static_cast<long long>(tile + 1) * a.ksteps;
  int c_hi = c + 1;
  while (c_hi < G && static_cast<long long>(c_hi) * a.sk_units / G < tile_end) ++c_hi;
  const uint32_t pbytes = static_cast<uint32_t>(a.bn) * kTileM * 4;
  if (threadIdx.x == 64) {
    for (int cc = c + 1; cc < c_hi; ++cc)
      while (ld_acquire_u32(a.sk_flags + cc) == 0u) {
      }
    SUN_STAMP(12);
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_arrive_expect_tx(bar, pbytes * static_cast<uint32_t>(c_hi - c - 1));
    for (int cc = c + 1; cc < c_hi; ++cc)
      bulk_load(ring + static_cast<size_t>(cc - c - 1) * pbytes, a.sk_part + static_cast<long long>(cc) * a.bn * kTileM,
                pbytes, bar);
  }
  mbar_wait(bar, 0);
  const float* parts = reinterpret_cast<const float*>(ring);
  float v[16];
  for (int c0 = 0; c0 < a.bn; c0 += 16) {
    tmem_ld16(taddr + c0, v);
    for (int cc = 0; cc < c_hi - c - 1; ++cc) {
      const float* src = parts + static_cast<size_t>(cc) * a.bn * kTileM;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 x = *reinterpret_cast<const float4*>(src + part_index(c0, j, row_local));
        v[4 * j] += x.x;
        v[4 * j + 1] += x.y;
        v[4 * j + 2] += x.z;
        v[4 * j + 3] += x.w;
      }
    }
    epi_chunk<EPI>(a, tile, row_local, c0, v, epi);
  }
  epi_bar();
  if (threadIdx.x == 64)
    for (int cc = c + 1; cc < c_hi; ++cc) a.sk_flags[cc] = 0u;
}


SUN_DEVICE uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t magic) {  // (a & mask) | magic
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(mask), "r"(magic));
  return d;
}

// QSUN dequantisation for one converter thread and one 128x128 K block: its TMEM
// lane `row`, K part `part` (kW4Chunks packed 16-byte chunks of the SUN-W4 block
// [4 chunks][128 rows][16 B], so a warp's 16-byte loads are 512 B contiguous).
// Per packed word (8 k): 3 shifts, 4 LOP3 (mask | magic -> bf16 128 + u), 4 HSUB2
// (exact), 4 HMUL2 (one rounding) -> bf16(q * s); output column c of the A tile
// holds k = (2c, 2c + 1), written with one tcgen05.st of 32 columns.
SUN_DEVICE void w4_dequant_row(uint32_t pk, uint32_t sc, int row, int part, uint32_t (&o)[16 * kW4Chunks]) {
  const uint32_t magic = 0x43004300u;
  const __nv_bfloat162 off = __floats2bfloat162_rn(136.f, 136.f);
  uint32_t words[4 * kW4Chunks];
#pragma unroll
  for (int c = 0; c < kW4Chunks; ++c)
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(words[4 * c]), "=r"(words[4 * c + 1]), "=r"(words[4 * c + 2]), "=r"(words[4 * c + 3])
                 : "r"(pk + ((kW4Chunks * part + c) * kTileM + row) * 16));
  unsigned short sraw;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(sraw) : "r"(sc + w4_scale_pos(row) * 2));
  __nv_bfloat16 sb;
  *reinterpret_cast<unsigned short*>(&sb) = sraw;
  const __nv_bfloat162 s2 = __bfloat162bfloat162(sb);
#ifdef SUN_W4_NO_CVT  // probe: skip the arithmetic (timing only, results invalid)
#pragma unroll
  for (int q = 0; q < 16 * kW4Chunks; ++q) o[q] = words[q & (4 * kW4Chunks - 1)] ^ sraw;
  return;
#endif
#pragma unroll
  for (int q = 0; q < 4 * kW4Chunks; ++q) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t u = lop3_and_or(words[q] >> (4 * e), 0x000F000Fu, magic);
      __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&u);
      v = __hmul2(__hsub2(v, off), s2);
      o[q * 4 + e] = *reinterpret_cast<uint32_t*>(&v);
    }
  }
}


template <int EPI, bool W4>
__global__ void __launch_bounds__(W4 ? kW4Threads : kGemmThreads, 1) gemm_kernel(const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  tl_begin(a.tl, a.tl_idx);
  const int stages = a.stages;
  const uint32_t sb = W4 ? w4_wstage_bytes(a.wgroup) : gemm_stage_bytes(a.bn, W4);
  const int xstages = a.xstages;
  const uint32_t xsb = W4 ? w4_xstage_bytes(a.bn, a.xk) : gemm_xstage_bytes(a.bn);
  const int wg = a.wgroup;
  uint8_t* stg = smem;
  uint8_t* xstg = stg + ((stages * sb + 1023u) & ~1023u);  // W4 activation ring (SW128 atoms: 1 KB aligned)
  float* epi = reinterpret_cast<float*>(xstg + xstages * xsb);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(epi) + kEpiSmemBytes);
  uint64_t* empty = full + kMaxWStages;
  uint64_t* xfull = empty + kMaxWStages;       // [kMaxXStages] W4
  uint64_t* xempty = xfull + kMaxXStages;      // [kMaxXStages] W4
  uint64_t* tfull = xempty + kMaxXStages;      // [2]
  uint64_t* tempty = tfull + 2;                // [2]
  uint64_t* dfull = tempty + 2;                // [kW4MaxABufs] W4: A tile dequantised
  uint64_t* dempty = dfull + kW4MaxABufs;      // [kW4MaxABufs] W4: A tile consumed by the MMA
  uint64_t* skbar = dempty + kW4MaxABufs;      // stream-K owner: contributor partials landed
  uint64_t* rbar = skbar + 1;                   // push mode: the peers' chunks landed in recv
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 1);
  float* recv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 1024);

  const int warp = warp_id_sync();
  constexpr bool kPre = !W4 && (EPI == EPI_RESID_ADD || EPI == EPI_QKV_ROPE);
  std::conditional_t<kPre, EpiPre, EpiPreNone> pre;  // this epilogue group's first split-K chunk
  const uint32_t S = a.splits > 1 ? static_cast<uint32_t>(a.splits) : 1u;
  const bool clustered = S > 1;  // split-K over S CTAs (hardware cluster or virtual)
  const bool vcl = clustered && a.vcluster;
  const uint32_t rank = clustered ? (vcl ? blockIdx.x % S : cluster_ctarank()) : 0u;
  const bool push = clustered && !vcl && a.push_bytes > 0;
  const int nch = a.bn / 16;                                       // 16-column chunks; chunk c is
  const int nmax = (nch + static_cast<int>(S) - 1) / static_cast<int>(S);  // reduced by rank c % S
  // this CTA's work: the contiguous range [u0, u1) of work units u = tile * ksteps + ks
  const int KS = a.ksteps;
  int u0, u1;
  if (clustered) {  // one tile, k-steps split over the cluster
    const int t = static_cast<int>(blockIdx.x / S);
    u0 = t * KS + static_cast<int>(rank * KS / S);
    u1 = t * KS + static_cast<int>((rank + 1) * KS / S);
  } else if (a.sk_units > 0) {  // stream-K
    u0 = static_cast<int>(static_cast<long long>(blockIdx.x) * a.sk_units / gridDim.x);
    u1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * a.sk_units / gridDim.x);
  } else {  // whole tiles
    u0 = static_cast<int>(static_cast<long long>(blockIdx.x) * a.m_tiles / gridDim.x) * KS;
    u1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * a.m_tiles / gridDim.x) * KS;
  }
  const int n = u1 - u0;
  const int t_first = u0 / KS;
  const int nseg = n > 0 ? (u1 - 1) / KS - t_first + 1 : 0;
  const uint32_t ncols = W4 ? 512u : tmem_cols_for(a.bn);
  const int nbuf = acc_buffers(a.bn, W4);
  // W4: converter warps 7..10 (TMEM lane groups 3, 0, 1, 2) become epilogue group B for
  // this CTA's last segment once their conversions are done (not under stream-K)
  const bool w4join = W4 && a.sk_units == 0;
  auto last_full_tile = [&]() {
    if (nseg == 0) return false;
    const int t = t_first + nseg - 1;
    return max(u0, t * KS) - t * KS == 0 && min(u1, (t + 1) * KS) - t * KS == KS;
  };
  // W4: each converter / MMA iteration covers kp K blocks (2 when bn <= 128: halves the
  // per-block hand-off overhead that bounded the pipeline); A slot i = 64 kp TMEM
  // columns ending at column 512 - 64 kp i
  const int kp = (W4 && a.bn <= 128 && a.xk % 2 == 0 && a.wgroup % 2 == 0) ? 2 : 1;
  const int na = W4 ? min(kW4MaxABufs, (512 - acc_buffers(a.bn, true) * a.bn) / (64 * kp)) : 1;
  const long long rows_pad = static_cast<long long>(a.m_tiles) * kTileM;
  if (threadIdx.x == 0) SUN_STAMP(0);

  if (warp == 0 && elect_one()) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W4 ? kW4ConvThreads / 32 : 1);  // W4: every converter warp; bf16: MMA commit
    }
    for (int s = 0; s < xstages; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int j = 0; j < 2; ++j) {
      mbar_init(&tfull[j], 1);
      mbar_init(&tempty[j], W4 ? 1 : 2);  // one arrival per epilogue group
    }
    for (int j = 0; j < kW4MaxABufs; ++j) {
      mbar_init(&dfull[j], kW4ConvThreads / 32);
      mbar_init(&dempty[j], 1);
    }
    mbar_init(skbar, 1);
    mbar_init(rbar, 1);
    fence_barrier_init();
    if (push) {  // (S - 1) peers x this rank's chunks x 8 KB will complete_tx on rbar
      const int mine = static_cast<int>(rank) < nch ? (nch - static_cast<int>(rank) + static_cast<int>(S) - 1) / static_cast<int>(S) : 0;
      mbar_arrive_expect_tx(rbar, static_cast<uint32_t>(mine) * (S - 1) * 8192u);
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // push mode: this arrival publishes rbar's init cluster-wide; the matching wait sits
  // just before the first remote copy, long after every peer has arrived
  if (push) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  if (threadIdx.x == 0) SUN_STAMP(1);
  // Early trigger: the next kernel may launch now and run its prologue (and, for
  // a GEMM, its weight prefetch) as SMs free up; its griddepcontrol.wait still
  // orders every dependent memory access after this grid completes.
  pdl_launch_dependents();

  auto nblk_of = [&](int ks) { return min(2, a.kb64 - 2 * ks); };

  if (W4 && (warp == 0 || warp == 6 + kW4ConvThreads / 32)) {
    // ---------------- W4 producers (blocking, one per ring): warp 0 streams the
    // weight stages (wgroup K blocks: packed + scales, two bulk requests), the
    // last warp the activation stages (xk K blocks, one request), so the weight
    // ring runs ahead of the MMA by its whole depth whatever the activation ring's.
    if (elect_one()) {
      const bool wprod = warp == 0;
      const int grp = wprod ? wg : a.xk;
      const int depth = wprod ? stages : xstages;
      uint64_t* fb = wprod ? full : xfull;
      uint64_t* eb = wprod ? empty : xempty;
      if (!wprod) pdl_wait();  // activations are the previous kernel's output
      int ks = u0 % KS, seg_left = min(KS - ks, n), slot = 0, phase = 0;
      for (int j = 0; j < n;) {
        const int len = min(grp, seg_left);
        if (j >= depth) mbar_wait(&eb[slot], phase ^ 1);
        if (wprod) {
          const long long blk = static_cast<long long>(u0 + j);  // = tile * KS + ks
          uint8_t* st = stg + slot * sb;
          mbar_arrive_expect_tx(&fb[slot], static_cast<uint32_t>(len) * (kW4PackedBytes + 256u));
          bulk_load_hint(st, a.w4_packed + blk * kW4PackedBytes, len * kW4PackedBytes, &fb[slot], kEvictFirst);
          bulk_load_hint(st + wg * kW4PackedBytes, a.w4_scales + blk * kTileM, len * 256u, &fb[slot], kEvictFirst);
        } else {
          mbar_arrive_expect_tx(&fb[slot], static_cast<uint32_t>(len) * a.bn * 256u);
          bulk_load_hint(xstg + slot * xsb, a.xact + static_cast<long long>(2 * ks) * a.bn * 128, len * a.bn * 256u,
                         &fb[slot], kEvictLast);
        }
        j += len;
        ks += len;
        seg_left -= len;
        if (seg_left == 0) {
          ks = 0;
          seg_left = min(KS, n - j);
        }
        if (++slot == depth) {
          slot = 0;
          phase ^= 1;
        }
      }
      if (wprod) prefetch_next_weights(a);
    }
  } else if (W4 && warp == 1) {
    // ---------------- W4 MMA issuer: A (dequantised weights) from TMEM, X from smem
    const uint32_t idesc = make_idesc_bf16(kTileM, a.bn);
    int ks = u0 % KS, seg_left = min(KS - ks, n);
    int xslot = 0, xphase = 0, xpos = 0, aslot = 0, aphase = 0, buf = 0, tphase = 0;
#ifdef SUN_W4_ROLE_CLOCKS  // probe: MMA warp waits on X / A -> stamps [9], [10], issue [11]
    long long mk_x = 0, mk_a = 0, mk_i = 0, mk0 = clock64();
#endif
    for (int j = 0; j < n;) {
      const int nbk = min(kp, seg_left);  // K blocks this iteration (never straddles a segment / stage)
      const bool first = j == 0 || ks == 0, last = seg_left == nbk;
      const bool xlast = xpos + nbk == a.xk || last;
      if (first) {
        mbar_wait(&tempty[buf], tphase ^ 1);
        tc_fence_after();
      }
      if (xpos == 0) mbar_wait(&xfull[xslot], xphase);
#ifdef SUN_W4_ROLE_CLOCKS
      { const long long t_ = clock64(); mk_x += t_ - mk0; mk0 = t_; }
#endif
      mbar_wait(&dfull[aslot], aphase);
      tc_fence_after();
#ifdef SUN_W4_ROLE_CLOCKS
      { const long long t_ = clock64(); mk_a += t_ - mk0; mk0 = t_; }
#endif
      if (j == 0 && threadIdx.x == 32) SUN_STAMP(2);
      if (elect_one()) {
        const uint32_t xa = smem_u32(xstg + xslot * xsb) + static_cast<uint32_t>(xpos) * 2u * a.bn * 128u;
        const uint32_t tacc = tmem_base + static_cast<uint32_t>(buf * a.bn);
        const uint32_t ta = tmem_base + static_cast<uint32_t>(512 - 64 * kp * (aslot + 1));
#ifndef SUN_W4_NO_MMA  // probe: skip the MMAs (timing only, results invalid)
        for (int b = 0; b < nbk; ++b)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ta(tacc, ta + b * 64 + kk * 8,
                         make_sw128_desc(xa + (2 * b + (kk >> 2)) * (a.bn * 128u) + (kk & 3) * 32), idesc,
                         (first && b == 0 && kk == 0) ? 0u : 1u);
#endif
        umma_commit(&dempty[aslot]);
        if (xlast) umma_commit(&xempty[xslot]);
        if (last) umma_commit(&tfull[buf]);
      }
      __syncwarp();
#ifdef SUN_W4_ROLE_CLOCKS
      { const long long t_ = clock64(); mk_i += t_ - mk0; mk0 = t_; }
#endif
      if (++aslot == na) {
        aslot = 0;
        aphase ^= 1;
      }
      if (xlast) {
        xpos = 0;
        if (++xslot == xstages) {
          xslot = 0;
          xphase ^= 1;
        }
      } else {
        xpos += nbk;
      }
      ks += nbk;
      j += nbk;
      seg_left -= nbk;
      if (seg_left == 0) {
        ks = 0;
        seg_left = min(KS, n - j);
        if (++buf == nbuf) {
          buf = 0;
          tphase ^= 1;
        }
      }
    }
    if (threadIdx.x == 32) SUN_STAMP(3);
#ifdef SUN_W4_ROLE_CLOCKS
    if (threadIdx.x == 32 && a.stamps) {
      a.stamps[blockIdx.x * 16 + 9] = mk_x;
      a.stamps[blockIdx.x * 16 + 10] = mk_a;
      a.stamps[blockIdx.x * 16 + 11] = mk_i;
    }
#endif
  } else if (!W4 && (warp == 0 || warp == 6)) {
    // ---------------- bf16 producers (blocking, one per ring): warp 0 streams the
    // weight stages (32 KB: one 128-wide K step of SUN-BLK), warp 6 the activation
    // stages (bn x 128 SUN-ACT), so the weight ring runs ahead by its whole depth.
    if (elect_one()) {
      const bool wprod = warp == 0;
      const int depth = wprod ? stages : xstages;
      uint64_t* fb = wprod ? full : xfull;
      uint64_t* eb = wprod ? empty : xempty;
      if (!wprod) pdl_wait();  // activations are the previous kernel's output
      int ks = u0 % KS, tile = u0 / KS, slot = 0, phase = 0;
      for (int j = 0; j < n; ++j) {
        const int nb = nblk_of(ks);
        if (j >= depth) mbar_wait(&eb[slot], phase ^ 1);
        if (wprod) {
          mbar_arrive_expect_tx(&fb[slot], nb * kTileWBytes);
          bulk_load_hint(stg + slot * sb, a.wblk + (static_cast<long long>(tile) * a.kb64 + 2 * ks) * kTileWBytes,
                         nb * kTileWBytes, &fb[slot], kEvictFirst);
        } else {
          mbar_arrive_expect_tx(&fb[slot], nb * a.bn * 128u);
          bulk_load_hint(xstg + slot * xsb, a.xact + static_cast<long long>(2 * ks) * a.bn * 128, nb * a.bn * 128u,
                         &fb[slot], kEvictLast);
        }
        if (++ks == KS) {
          ks = 0;
          ++tile;
        }
        if (++slot == depth) {
          slot = 0;
          phase ^= 1;
        }
      }
      if (wprod) prefetch_next_weights(a);
    }
  } else if (warp == 1 && !W4) {
    const uint32_t idesc = make_idesc_bf16(kTileM, a.bn);
    int ks = u0 % KS, wslot = 0, wphase = 0, xslot = 0, xphase = 0, buf = 0, tphase = 0;
    for (int j = 0; j < n; ++j) {
      const bool first = j == 0 || ks == 0, last = j == n - 1 || ks == KS - 1;
      const int nb = nblk_of(ks);
      if (first) {
        mbar_wait(&tempty[buf], tphase ^ 1);
        tc_fence_after();
      }
      mbar_wait(&full[wslot], wphase);
      mbar_wait(&xfull[xslot], xphase);
      tc_fence_after();
      if (j == 0 && threadIdx.x == 32) SUN_STAMP(2);
      if (elect_one()) {
        const uint32_t xa = smem_u32(xstg + xslot * xsb);
        const uint32_t tacc = tmem_base + static_cast<uint32_t>(buf * a.bn);
        const uint32_t wa = smem_u32(stg + wslot * sb);
        for (int kk = 0; kk < nb * 4; ++kk) {
          const uint32_t atom = kk >> 2;
          const uint32_t koff = (kk & 3) * 32;
          umma_bf16(tacc, make_sw128_desc(wa + atom * kTileWBytes + koff),
                    make_sw128_desc(xa + atom * (a.bn * 128u) + koff), idesc, (first && kk == 0) ? 0u : 1u);
        }
        umma_commit(&empty[wslot]);
        umma_commit(&xempty[xslot]);
        if (last) umma_commit(&tfull[buf]);
      }
      __syncwarp();
      if (++wslot == stages) {
        wslot = 0;
        wphase ^= 1;
      }
      if (++xslot == xstages) {
        xslot = 0;
        xphase ^= 1;
      }
      if (++ks == KS) ks = 0;
      if (last && ++buf == nbuf) {
        buf = 0;
        tphase ^= 1;
      }
    }
    if (threadIdx.x == 32) SUN_STAMP(3);
  } else if (warp < 6 || (!W4 && warp >= 7)) {
    // ---------------- epilogue: group A = warps 2..5 (+ group B = warps 7..10, bf16) ----------------
    pdl_wait();
    if (warp < 6) load_qkv_meta<EPI>(a, epi);
    if constexpr (!W4) asm volatile("bar.sync 4, 256;" ::: "memory");  // group B waits for the meta
    if constexpr (kPre) {
      if (clustered) {  // the first chunk this group will handle after the reduction
        const int rl = (warp & 3) * 32 + (threadIdx.x & 31);
        const int nmine = (a.bn / 16 - static_cast<int>(rank) + static_cast<int>(S) - 1) / static_cast<int>(S);
        if (nmine == 1) epi_preload<EPI>(a, t_first, rl, static_cast<int>(rank) * 16 + 8 * epi_grp(), 8, epi, pre);
        else if (static_cast<int>(rank + S * epi_grp()) * 16 < a.bn)
          epi_preload<EPI>(a, t_first, rl, static_cast<int>(rank + S * epi_grp()) * 16, 16, epi, pre);
      }
    }
    const int q = warp & 3;
    const int row_local = q * 32 + (threadIdx.x & 31);
    for (int seg = 0; seg < nseg; ++seg) {
      const int buf = seg % nbuf;
      const int tile = t_first + seg;
      const int kb = max(u0, tile * KS) - tile * KS;
      const int ke = min(u1, (tile + 1) * KS) - tile * KS;
      mbar_wait(&tfull[buf], (seg / nbuf) & 1);
      tc_fence_after();
      if (threadIdx.x == 64 && seg == 0) SUN_STAMP(4);
      const uint32_t taddr = tmem_base + static_cast<uint32_t>(buf * a.bn) + (static_cast<uint32_t>(q * 32) << 16);
      if (!clustered) {
        const bool join = w4join && seg == nseg - 1 && kb == 0 && ke == KS;
        if (join) asm volatile("bar.sync 4, 256;" ::: "memory");  // group B (converters) joins
        if (kb == 0 && ke == KS) direct_epilogue<EPI>(a, tile, taddr, epi, (W4 && !join) ? 1 : 2);
        else if (epi_grp() == 0 && kb > 0) sk_store_partial(a, taddr, row_local);  // stream-K: group A only
        else if (epi_grp() == 0) sk_owner_epilogue<EPI>(a, tile, taddr, row_local, epi, stg, skbar);
        tc_fence_before();
        epi_bar();
        if (epi_lead_thread()) mbar_arrive(&tempty[buf]);
      } else if (epi_grp() == 0) {
        // park the partial (part_index layout) in the now idle shared memory
        // (hardware cluster: peers read it over DSMEM) or in L2 (virtual cluster)
        float* part = vcl ? a.sk_part + static_cast<long long>(blockIdx.x) * a.bn * kTileM
                          : reinterpret_cast<float*>(smem);
        float v[16];
        for (int c0 = 0; c0 < a.bn; c0 += 16) {
          tmem_ld16(taddr + c0, v);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 f = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            if (vcl) __stcg(reinterpret_cast<float4*>(part + part_index(c0, j, row_local)), f);
            else *reinterpret_cast<float4*>(part + part_index(c0, j, row_local)) = f;
          }
        }
        if (vcl) __threadfence();
        if (push) fence_proxy_async_smem();  // the parked chunks are the bulk copies' source
      }
    }
  } else if (W4 && warp < 6 + kW4ConvThreads / 32) {
    // ---------------- converters: lane group warp % 4, K part (warp - 6) / 4 ----------------
    const int lg = warp & 3;  // TMEM lanes this warp may access
    const int row = lg * 32 + (threadIdx.x & 31);
    const int part = (warp - 6) >> 2;  // columns [16 * kW4Chunks * part, +16 * kW4Chunks) of each A tile
    const uint32_t lane_off = static_cast<uint32_t>(lg * 32) << 16;
    int ks = u0 % KS, seg_left = min(KS - ks, n);
    int wslot = 0, wphase = 0, wpos = 0, aslot = 0, aphase = 0, it = 0;
#ifdef SUN_W4_ROLE_CLOCKS  // probe: per-role cycle split of converter warp 6 -> stamps [12..15]
    long long ck_w = 0, ck_c = 0, ck_a = 0, ck_s = 0, ck0 = clock64();
#define SUN_CK(acc) do { const long long t_ = clock64(); acc += t_ - ck0; ck0 = t_; } while (0)
#else
#define SUN_CK(acc) do {} while (0)
#endif
    for (int j = 0; j < n;) {
      const int nbk = min(kp, seg_left);
      if (wpos == 0) mbar_wait(&full[wslot], wphase);
      SUN_CK(ck_w);
      const bool wlast = wpos + nbk == wg || seg_left == nbk;
      const uint32_t st = smem_u32(stg + wslot * sb);
      uint32_t o0[16 * kW4Chunks], o1[16 * kW4Chunks];
#ifndef SUN_W4_PROBE_STREAM  // probe: converters only pass the stages through (timing only)
      w4_dequant_row(st + wpos * kW4PackedBytes, st + wg * kW4PackedBytes + wpos * 256u, row, part, o0);
      if (nbk == 2)
        w4_dequant_row(st + (wpos + 1) * kW4PackedBytes, st + wg * kW4PackedBytes + (wpos + 1) * 256u, row, part, o1);
#endif
      SUN_CK(ck_c);
      if (wlast) {  // this warp is done reading the weight stage
        __syncwarp();
        if (elect_one()) mbar_arrive(&empty[wslot]);
        wpos = 0;
        if (++wslot == stages) {
          wslot = 0;
          wphase ^= 1;
        }
      } else {
        wpos += nbk;
      }
      if (it >= na) mbar_wait(&dempty[aslot], aphase ^ 1);  // MMA it-na done with this A slot
      tc_fence_after();
      SUN_CK(ck_a);
      const uint32_t ta = tmem_base + lane_off + static_cast<uint32_t>(512 - 64 * kp * (aslot + 1) + 16 * kW4Chunks * part);
#if !defined(SUN_W4_PROBE_STREAM) && !defined(SUN_W4_PROBE_NOTST)  // probes: no TMEM stores (timing only)
      tmem_st(ta, o0);
      if (nbk == 2) tmem_st(ta + 64, o1);
#else
      if (o0[0] == 0x12345u && o1[0] == 0x12345u) asm volatile("trap;");  // keep the dequant live
#endif
      tc_fence_before();
      __syncwarp();
      if (elect_one()) mbar_arrive(&dfull[aslot]);
      SUN_CK(ck_s);
      if (++aslot == na) {
        aslot = 0;
        aphase ^= 1;
      }
      ++it;
      j += nbk;
      seg_left -= nbk;
      if (seg_left == 0) seg_left = min(KS, n - j);
    }
#ifdef SUN_W4_ROLE_CLOCKS
    if (warp == 6 && (threadIdx.x & 31) == 0 && a.stamps) {
      a.stamps[blockIdx.x * 16 + 12] = ck_w;
      a.stamps[blockIdx.x * 16 + 13] = ck_c;
      a.stamps[blockIdx.x * 16 + 14] = ck_a;
      a.stamps[blockIdx.x * 16 + 15] = ck_s;
    }
#endif
#undef SUN_CK
    if (w4join && !clustered && warp >= 7 && warp < 11 && last_full_tile()) {
      // epilogue group B for the last tile: chunks alternate with group A
      asm volatile("bar.sync 4, 256;" ::: "memory");
      const int seg = nseg - 1, buf = seg % nbuf;
      mbar_wait(&tfull[buf], (seg / nbuf) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + static_cast<uint32_t>(buf * a.bn) + (static_cast<uint32_t>((warp & 3) * 32) << 16);
      direct_epilogue<EPI>(a, t_first + seg, taddr, epi, 2);
      tc_fence_before();
    }
  }

  if (clustered) {
    if (threadIdx.x == 64) SUN_STAMP(8);
    unsigned* tile_cnt = vcl ? a.sk_flags + blockIdx.x / S : nullptr;
    if (vcl) {  // every rank's partial is in L2: count arrivals of the tile's S CTAs
      __syncthreads();
      if (threadIdx.x == 64) {
        atomicAdd(tile_cnt, 1u);
        while (ld_acquire_u32(tile_cnt) < S) {
        }
      }
      __syncthreads();
    } else if (push) {
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // peers' rbar initialised
      __syncthreads();                                                     // our partial is parked
      if (threadIdx.x == 64) {
        // send every chunk another rank reduces to that rank's receive area (slot = our
        // rank among its S - 1 senders); completion is counted on the owner's rbar
        const float* part = reinterpret_cast<const float*>(smem);
        for (int c = 0; c < nch; ++c) {
          const uint32_t o = static_cast<uint32_t>(c) % S;
          if (o == rank) continue;
          const uint32_t slot = rank < o ? rank : rank - 1;
          const uint32_t dst = dsmem_addr(recv + (slot * nmax + static_cast<uint32_t>(c) / S) * 2048u, o);
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];" ::"r"(dst),
              "r"(smem_u32(part + c * 2048)), "r"(dsmem_addr(rbar, o))
              : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      cluster_sync_all();  // every rank's partial is visible cluster-wide
    }
    if (threadIdx.x == 64) SUN_STAMP(9);
    if ((warp >= 2 && warp < 6) || ((!W4 || w4join) && warp >= 7 && warp < 11)) {
      const int q = warp & 3;
      const int row_local = q * 32 + (threadIdx.x & 31);
      float* part = reinterpret_cast<float*>(smem);
      const float* gpart = vcl ? a.sk_part + static_cast<long long>(blockIdx.x - rank) * a.bn * kTileM : nullptr;
      if (push) mbar_wait(rbar, 0);  // every peer's copy of our chunks has landed
      // reduce columns [c0, c0 + NC) over the S ranks (float4 slots q0.. of the chunk), in rank order
      auto reduce_cols = [&](int c0, int q0, auto& v) {
        constexpr int NQ = sizeof(v) / sizeof(float) / 4;
        float4 x[4][NQ];
#pragma unroll
        for (int j = 0; j < 4 * NQ; ++j) v[j] = 0.f;
        const int cbase = c0 & ~15;
        for (uint32_t r0 = 0; r0 < S; r0 += 4) {  // 4 ranks' loads in flight
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < NQ; ++j)
              x[u][j] = (r0 + u >= S) ? make_float4(0.f, 0.f, 0.f, 0.f)
                        : vcl ? __ldcg(reinterpret_cast<const float4*>(gpart + static_cast<long long>(r0 + u) * a.bn * kTileM +
                                                                      part_index(cbase, q0 + j, row_local)))
                        : push ? *reinterpret_cast<const float4*>(
                                     (r0 + u == rank ? part + part_index(cbase, 0, 0)
                                                     : recv + ((r0 + u < rank ? r0 + u : r0 + u - 1) * nmax +
                                                               static_cast<uint32_t>(cbase >> 4) / S) * 2048u) +
                                     part_index(0, q0 + j, row_local))
                              : ld_dsmem_f4(dsmem_addr(part + part_index(cbase, q0 + j, row_local), r0 + u));
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
              v[4 * j] += x[u][j].x;
              v[4 * j + 1] += x[u][j].y;
              v[4 * j + 2] += x[u][j].z;
              v[4 * j + 3] += x[u][j].w;
            }
        }
      };
      const int nmine = (a.bn / 16 - static_cast<int>(rank) + static_cast<int>(S) - 1) / static_cast<int>(S);
      if ((!W4 || w4join) && nmine == 1) {
        // one 16-column chunk for this rank: each epilogue group takes 8 columns
        const int c0 = static_cast<int>(rank) * 16 + 8 * epi_grp();
        float v[8];
        reduce_cols(c0, 2 * epi_grp(), v);
        if (threadIdx.x == 64) SUN_STAMP(10);
        if constexpr (kPre) epi_chunk<EPI, 8>(a, t_first, row_local, c0, v, epi, pre.p0, pre.p1);
        else epi_chunk<EPI, 8>(a, t_first, row_local, c0, v, epi);
        if (threadIdx.x == 64) SUN_STAMP(11);
      } else {
        const int ng = (W4 && !w4join) ? 1 : 2;  // the rank's chunks alternate between the epilogue groups
        for (int c0 = static_cast<int>(rank + S * epi_grp()) * 16; c0 < a.bn; c0 += static_cast<int>(S * ng) * 16) {
          float v[16];
          reduce_cols(c0, 0, v);
          if (threadIdx.x == 64) SUN_STAMP(10);
          if constexpr (kPre) {
            if (c0 == pre.c0) epi_chunk<EPI>(a, t_first, row_local, c0, v, epi, pre.p0, pre.p1);
            else epi_chunk<EPI>(a, t_first, row_local, c0, v, epi);
          } else {
            epi_chunk<EPI>(a, t_first, row_local, c0, v, epi);
          }
          if (threadIdx.x == 64) SUN_STAMP(11);
        }
      }
    }
    if (vcl) {  // the last of the tile's 2S arrivals rearms the counter for the next launch
      __syncthreads();
      if (threadIdx.x == 64 && atomicAdd(tile_cnt, 1u) == 2 * S - 1) *tile_cnt = 0u;
    } else if (push) {
      if (threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // sources read
    } else {
      cluster_sync_all();  // nobody exits while a peer may still read its partial
    }
  }
  if (threadIdx.x == 64) SUN_STAMP(5);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, ncols);
  }
  if (threadIdx.x == 0) SUN_STAMP(6);
  tl_end(a.tl, a.tl_idx);
}

}  // namespace sun
