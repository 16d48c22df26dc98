// attention.cuh — paged split-K flash-decoding attention over the shared KV pool.
//
// One CTA = one (split, kv_head, sequence) work unit. The GQA group of query
// heads sharing that kv head (4 for Llama-3 shapes, 5 for Qwen2.5-14B) forms
// the rows of an m16n8k16 tile, so K/V bytes are read exactly once per group.
// K/V pages are staged by TMA (3-D tensor map over the page pool, SWIZZLE_128B,
// 16-token x 128 B boxes) into per-warp mbarrier rings; each warp consumes every
// NWARPS-th page with ldmatrix + mma.sync, online softmax in fp32 with
// quad-shuffle reductions, then the warps merge through shared memory. A
// single-split sequence writes its output directly; otherwise each split
// publishes (m, l, O) and the last-arriving split merges them (fused combine).
//
// Replaces the KV term `sum(resident_tokens * kv_bytes_per_token)` of the
// reference step price (poolsim costmodel.py:112, 139; engine.py:427-428).
#pragma once
#include "gemm_tc.cuh"  // act_offset (SUN-ACT layout)

namespace sun {

constexpr int kPageTokens = 16;  // tokens per KV page (one m16n8k16 k-step of P.V)

struct AttnArgs {
  const __nv_bfloat16* q;  // [B][n_q_heads][D]
  const int* positions;    // [B] position of the decoded token; ctx = pos + 1
  const int* block_tables; // [B][bt_stride]
  int bt_stride;
  int layer;
  int n_q_heads;
  int n_kv_heads;
  int pages_per_split;
  int max_splits;
  float scale_log2;        // log2(e) / sqrt(D)
  float* part_o;           // [B][n_q_heads][max_splits][D]
  float* part_ml;          // [B][n_q_heads][max_splits][2]
  __nv_bfloat16* out;      // [B][n_q_heads * D]   (combine output)
  long long ld_out;
  int act_rows;            // > 0: write `out` in SUN-ACT (the O-projection operand)
  unsigned* counters;      // [B][n_kv_heads] split arrival counters (zeroed once, self-resetting)
  int fused_combine;       // 1: last split merges in-kernel; 0: attn_combine_kernel does it
  unsigned long long* tl;  // step timeline (profiling only)
  int tl_idx;
  // grouped rows (token-parallel prefill): grid z = groups; group z is rows
  // [group_start[z], group_start[z] + group_len[z]) of one sequence at ascending
  // positions, all read against the same KV pages (<= 16 / GQA-group rows each)
  const int* group_start;
  const int* group_len;
  // 1: every row is a different sequence (the decode batch), so the step's QKV
  // kernel writes only each row's last page: the other pages are staged before
  // griddepcontrol.wait, i.e. while the QKV grid is still finishing (PDL)
  int prestage;
  // non-null (decode, layer >= 1, prestage): per-tile writer counts of this layer's QKV output,
  // published by the previous layer chain's epilogues; the kernel waits for its Q / K / V tiles
  // (>= ready_writers each) instead of the chain grid, and runs griddepcontrol.wait before it
  // exits so that completion still orders the chain before the next kernel
  const unsigned* qkv_ready;
  unsigned ready_writers;
  int max_ctx;             // tokens a block-table row can address (decoder max_context): positions
                           // outside [0, max_ctx) are clamped, so a bad position cannot read past
                           // its block-table row (sun_decode_step flags it in the error word)
};

// context length of row b (clamped; see AttnArgs::max_ctx)
SUN_DEVICE int row_ctx(const AttnArgs& a, int b) {
  const int p = a.positions[b];
  return (p < 0 ? 0 : (p >= a.max_ctx ? a.max_ctx - 1 : p)) + 1;
}

template <int D>
SUN_DEVICE void store_attn_out(const AttnArgs& a, int b, int head, int dim, float v) {
  const __nv_bfloat16 o = __float2bfloat16_rn(v);
  if (a.act_rows > 0)
    *reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(a.out) + act_offset(b, head * D + dim, a.act_rows)) = o;
  else
    a.out[static_cast<long long>(b) * a.ld_out + head * D + dim] = o;
}

#ifndef SUN_ATTN_D64_STAGES
#define SUN_ATTN_D64_STAGES 3  // (C2 same-box: 2 stages 1.538 ms, 3: 1.506, 4: 1.678 — 3 keeps 4 CTAs per SM)
#endif
#ifndef SUN_ATTN_D128_STAGES
#define SUN_ATTN_D128_STAGES 3
#endif
template <int D>
struct AttnCfg {
  static constexpr int kWarps = 4;
  static constexpr int kStages = (D == 128) ? SUN_ATTN_D128_STAGES : SUN_ATTN_D64_STAGES;
  static constexpr int kBoxes = D / 64;                          // 128 B boxes per row
  static constexpr uint32_t kTileBytes = kPageTokens * D * 2;    // K (or V) of one page
  static constexpr uint32_t kStageBytes = 2 * kTileBytes;
  static constexpr size_t kSmem = 1024 + size_t(kWarps) * kStages * kStageBytes + 1024;
};

// byte offset of (token, dim) inside one staged [16][D] tile (boxes of 64 cols, SW128)
SUN_DEVICE uint32_t kv_swz(int tok, int dim) {
  const int box = dim >> 6;
  const int chunk = (dim & 63) >> 3;
  return static_cast<uint32_t>(box * 2048 + tok * 128 + ((chunk ^ (tok & 7)) << 4));
}

template <int D>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(const __grid_constant__ CUtensorMap tm_kv, const AttnArgs a) {
  using C = AttnCfg<D>;
  const int split = blockIdx.x;
  const int kvh = blockIdx.y;
  const int b = blockIdx.z;
  tl_begin(a.tl, a.tl_idx);
  // positions / block tables are inputs of the whole step (never written inside it)
  const bool pre = a.prestage != 0;
  if (!pre) {
    pdl_wait();
    pdl_launch_dependents();  // early: the next kernel may start its prologue / weight prefetch
  }
  const int ctx = row_ctx(a, b);
  const int n_pages = (ctx + kPageTokens - 1) / kPageTokens;
  const int p0 = split * a.pages_per_split;
  if (p0 >= n_pages) {
    tl_end(a.tl, a.tl_idx);
    return;
  }
  const int p1 = min(n_pages, p0 + a.pages_per_split);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kWarps * C::kStages * C::kStageBytes);
  float* merge_ml = reinterpret_cast<float*>(bars + C::kWarps * C::kStages);  // [warps][8][2]

  const int warp = warp_id_sync();
  const int lane = threadIdx.x & 31;
  const int G = a.n_q_heads / a.n_kv_heads;  // <= 8
  const int g = lane >> 2;                   // query row owned by this quad
  const int t = lane & 3;
  uint8_t* my_stages = smem + warp * C::kStages * C::kStageBytes;
  uint64_t* my_bars = bars + warp * C::kStages;

  const int n_my = (p1 - p0 - warp + C::kWarps - 1) / C::kWarps > 0 ? (p1 - p0 - warp + C::kWarps - 1) / C::kWarps : 0;
  const int* bt = a.block_tables + static_cast<long long>(b) * a.bt_stride;
  const int row_k = ((a.layer * 2 + 0) * a.n_kv_heads + kvh) * kPageTokens;
  const int row_v = ((a.layer * 2 + 1) * a.n_kv_heads + kvh) * kPageTokens;

  auto issue = [&](int i) {  // lane 0 only: stage the i-th page of this warp
    const int s = i % C::kStages;
    const int page = bt[p0 + warp + i * C::kWarps];
    uint8_t* dst = my_stages + s * C::kStageBytes;
    mbar_arrive_expect_tx(&my_bars[s], C::kStageBytes);
#pragma unroll
    for (int bx = 0; bx < C::kBoxes; ++bx) {
      tma_load_3d(dst + bx * 2048, &tm_kv, &my_bars[s], bx * 64, row_k, page, kEvictFirst);
      tma_load_3d(dst + C::kTileBytes + bx * 2048, &tm_kv, &my_bars[s], bx * 64, row_v, page, kEvictFirst);
    }
  };

  const int npre = min(n_my, C::kStages);
  int ipre = 0;
  if (lane == 0) {
    for (int s = 0; s < C::kStages; ++s) mbar_init(&my_bars[s], 1);
    fence_barrier_init();
    if (pre)  // pages before the row's last one: untouched by this step's KV append
      for (; ipre < npre && p0 + warp + ipre * C::kWarps < n_pages - 1; ++ipre) issue(ipre);
  }
  const bool tile_ready = pre && a.qkv_ready != nullptr;
  if (tile_ready) {
    // q and the appended K/V of this (kv head, group) are written once their QKV tiles are
    // published (tile = 128 rows of [Q heads | K heads | V heads] x head_dim)
    if (threadIdx.x < 3) {
      const int qd = a.n_q_heads * D, kd = a.n_kv_heads * D;
      int lo, hi;
      if (threadIdx.x == 0) {
        lo = (kvh * G * D) / 128;
        hi = ((kvh + 1) * G * D - 1) / 128;
      } else {
        lo = hi = (qd + (threadIdx.x == 2 ? kd : 0) + kvh * D) / 128;
      }
      const unsigned long long t0 = global_timer_ns();
      for (int t = lo; t <= hi; ++t) {
        while (ld_acquire_u32(a.qkv_ready + t) < a.ready_writers) {
          __nanosleep(32);
          if (global_timer_ns() - t0 > 2000000000ull) __trap();  // (never: the chain is resident)
        }
      }
    }
    __syncthreads();
    asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy stores -> TMA page loads
    pdl_launch_dependents();
  } else if (pre) {
    pdl_wait();  // q and the appended K/V are the QKV kernel's outputs
    pdl_launch_dependents();
  }
  if (lane == 0)
    for (; ipre < npre; ++ipre) issue(ipre);
  __syncwarp();

  // Q fragments (A operand, rows = query heads of the group, zero-padded to 16).
  uint32_t qa[D / 16][2];
  {
    const __nv_bfloat16* qrow = a.q + (static_cast<long long>(b) * a.n_q_heads + kvh * G + g) * D;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      if (g < G) {
        qa[kk][0] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t);
        qa[kk][1] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * t);
      } else {
        qa[kk][0] = 0u;
        qa[kk][1] = 0u;
      }
    }
  }

  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_run = -INFINITY;
  float l_run = 0.f;

  const int mi = lane >> 3;  // ldmatrix matrix index supplied by this lane
  const int mr = lane & 7;   // row within that matrix

  for (int i = 0; i < n_my; ++i) {
    const int s = i % C::kStages;
    mbar_wait(&my_bars[s], (i / C::kStages) & 1);
    const uint32_t kbase = smem_u32(my_stages + s * C::kStageBytes);
    const uint32_t vbase = kbase + C::kTileBytes;
    const int tok0 = (p0 + warp + i * C::kWarps) * kPageTokens;

    // S = Q . K^T  (two n-tiles of 8 tokens)
    float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t r0, r1, r2, r3;
      const int tok = ((mi >> 1) << 3) + mr;
      const int dim = kk * 16 + ((mi & 1) << 3);
      ldmatrix_x4(kbase + kv_swz(tok, dim), r0, r1, r2, r3);
      mma_16816(sacc[0], qa[kk][0], 0u, qa[kk][1], 0u, r0, r1);
      mma_16816(sacc[1], qa[kk][0], 0u, qa[kk][1], 0u, r2, r3);
    }
    // scale, mask, online softmax (row g; c2/c3 are padding rows)
    float sv[4];
    float mx = -INFINITY;
#pragma unroll
    for (int n = 0; n < 2; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = tok0 + n * 8 + 2 * t + e;
        const float x = tok < ctx ? sacc[n][e] * a.scale_log2 : -INFINITY;
        sv[n * 2 + e] = x;
        mx = fmaxf(mx, x);
      }
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    const float corr = exp2f(m_run - m_new);  // m_run = -inf -> 0
    m_run = m_new;
    float p[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = exp2f(sv[e] - m_new);
    l_run = l_run * corr + (p[0] + p[1] + p[2] + p[3]);
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      o[n][0] *= corr;
      o[n][1] *= corr;
    }
    // P is split into bf16 hi + lo parts (p = hi + lo to ~16 mantissa bits) so the
    // bf16 tensor-core P.V keeps fp32-grade probabilities: with near-uniform
    // attention a plain bf16 P perturbs the output by ~0.1% (1/3 of the bf16
    // output roundings flip), which the hi/lo pair removes for 2x P.V mma.
    const uint32_t pa0 = pack_bf16x2(p[0], p[1]);
    const uint32_t pa2 = pack_bf16x2(p[2], p[3]);
    const uint32_t pl0 = pack_bf16x2(p[0] - bf16_round(p[0]), p[1] - bf16_round(p[1]));
    const uint32_t pl2 = pack_bf16x2(p[2] - bf16_round(p[2]), p[3] - bf16_round(p[3]));
    // O += P . V
#pragma unroll
    for (int nn = 0; nn < D / 16; ++nn) {
      uint32_t r0, r1, r2, r3;
      const int tok = ((mi & 1) << 3) + mr;
      const int dim = nn * 16 + ((mi >> 1) << 3);
      ldmatrix_x4_trans(vbase + kv_swz(tok, dim), r0, r1, r2, r3);
      mma_16816(o[2 * nn], pa0, 0u, pa2, 0u, r0, r1);
      mma_16816(o[2 * nn + 1], pa0, 0u, pa2, 0u, r2, r3);
      mma_16816(o[2 * nn], pl0, 0u, pl2, 0u, r0, r1);
      mma_16816(o[2 * nn + 1], pl0, 0u, pl2, 0u, r2, r3);
    }
    __syncwarp();
    if (lane == 0 && i + C::kStages < n_my) {
      fence_proxy_async_smem();
      issue(i + C::kStages);
    }
  }
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);

  // ---- merge the warps of this CTA through shared memory ----
  __syncthreads();  // every warp is done with its stage ring
  float* merge_o = reinterpret_cast<float*>(smem);  // [warps][8][D]
  if (g < G) {
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      merge_o[(warp * 8 + g) * D + n * 8 + 2 * t] = o[n][0];
      merge_o[(warp * 8 + g) * D + n * 8 + 2 * t + 1] = o[n][1];
    }
    if (t == 0) {
      merge_ml[(warp * 8 + g) * 2 + 0] = m_run;
      merge_ml[(warp * 8 + g) * 2 + 1] = l_run;
    }
  }
  __syncthreads();
  const int n_splits = (n_pages + a.pages_per_split - 1) / a.pages_per_split;
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int gg = idx / D;
    const int dim = idx % D;
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < C::kWarps; ++w) mm = fmaxf(mm, merge_ml[(w * 8 + gg) * 2]);
    float acc = 0.f, ll = 0.f;
#pragma unroll
    for (int w = 0; w < C::kWarps; ++w) {
      const float mw = merge_ml[(w * 8 + gg) * 2];
      const float sc = (mw == -INFINITY) ? 0.f : exp2f(mw - mm);
      acc += merge_o[(w * 8 + gg) * D + dim] * sc;
      ll += merge_ml[(w * 8 + gg) * 2 + 1] * sc;
    }
    const int head = kvh * G + gg;
    if (n_splits == 1) {  // whole context in this CTA: emit the output directly
      store_attn_out<D>(a, b, head, dim, acc / ll);
      continue;
    }
    const long long u = (static_cast<long long>(b) * a.n_q_heads + head) * a.max_splits + split;
    a.part_o[u * D + dim] = acc;
    if (dim == 0) {
      a.part_ml[u * 2 + 0] = mm;
      a.part_ml[u * 2 + 1] = ll;
    }
  }
  if (a.fused_combine && n_splits > 1) {
    // split-K combine fused in: the last-arriving split of (b, kv head) merges
    // all splits in split order (deterministic) and writes the GQA group's output
    __shared__ int is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned* cnt = a.counters + static_cast<long long>(b) * a.n_kv_heads + kvh;
      const unsigned prev = atomicAdd(cnt, 1u);
      is_last = prev == static_cast<unsigned>(n_splits - 1);
      if (is_last) *cnt = 0u;
    }
    __syncthreads();
    if (is_last) {
      __threadfence();
      for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
        const int gg = idx / D;
        const int dim = idx % D;
        const int head = kvh * G + gg;
        const long long u0 = (static_cast<long long>(b) * a.n_q_heads + head) * a.max_splits;
        float mm = -INFINITY;
        for (int s2 = 0; s2 < n_splits; ++s2) mm = fmaxf(mm, __ldcg(&a.part_ml[(u0 + s2) * 2]));
        float acc = 0.f, ll = 0.f;
        for (int s2 = 0; s2 < n_splits; ++s2) {
          const float sc = exp2f(__ldcg(&a.part_ml[(u0 + s2) * 2]) - mm);
          acc += __ldcg(&a.part_o[(u0 + s2) * D + dim]) * sc;
          ll += __ldcg(&a.part_ml[(u0 + s2) * 2 + 1]) * sc;
        }
        store_attn_out<D>(a, b, head, dim, acc / ll);
      }
    }
  }
  if (tile_ready) pdl_wait();  // completion of this grid still implies the chain's (PDL ordering)
  tl_end(a.tl, a.tl_idx);
}

// Grouped-rows variant for token-parallel prefill: the rows of one prompt at
// consecutive positions share the KV pages, so one CTA stages each page once for
// up to 16 query rows (rows x GQA heads fill the m16n8k16 A tile whose upper
// half the decode kernel leaves at zero); each row keeps its own causal limit
// and online-softmax state. Same arithmetic per row as attn_decode_kernel.
template <int D>
__global__ void __launch_bounds__(128)
    attn_group_kernel(const __grid_constant__ CUtensorMap tm_kv, const AttnArgs a) {
  using C = AttnCfg<D>;
  const int split = blockIdx.x;
  const int kvh = blockIdx.y;
  const int b0 = a.group_start[blockIdx.z];
  const int nr = a.group_len[blockIdx.z];
  pdl_wait();
  pdl_launch_dependents();
  const int ctx = row_ctx(a, b0 + nr - 1);  // the group's longest context
  const int n_pages = (ctx + kPageTokens - 1) / kPageTokens;
  const int p0 = split * a.pages_per_split;
  if (p0 >= n_pages) return;
  const int p1 = min(n_pages, p0 + a.pages_per_split);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kWarps * C::kStages * C::kStageBytes);
  float* merge_ml = reinterpret_cast<float*>(bars + C::kWarps * C::kStages);  // [warps][16][2]

  const int warp = warp_id_sync();
  const int lane = threadIdx.x & 31;
  const int G = a.n_q_heads / a.n_kv_heads;
  const int g = lane >> 2;
  const int t = lane & 3;
  uint8_t* my_stages = smem + warp * C::kStages * C::kStageBytes;
  uint64_t* my_bars = bars + warp * C::kStages;
  // query rows g (lower half) and g + 8 (upper half) -> (row of the group, head)
  const int r_lo = g / G, r_hi = (g + 8) / G;
  const bool v_lo = r_lo < nr, v_hi = r_hi < nr;
  const bool has_hi = nr * G > 8;  // warp-uniform
  const int ctx_lo = v_lo ? row_ctx(a, b0 + r_lo) : ctx;
  const int ctx_hi = v_hi ? row_ctx(a, b0 + r_hi) : ctx;

  const int n_my = (p1 - p0 - warp + C::kWarps - 1) / C::kWarps > 0 ? (p1 - p0 - warp + C::kWarps - 1) / C::kWarps : 0;
  const int* bt = a.block_tables + static_cast<long long>(b0) * a.bt_stride;
  const int row_k = ((a.layer * 2 + 0) * a.n_kv_heads + kvh) * kPageTokens;
  const int row_v = ((a.layer * 2 + 1) * a.n_kv_heads + kvh) * kPageTokens;
  auto issue = [&](int i) {
    const int s = i % C::kStages;
    const int page = bt[p0 + warp + i * C::kWarps];
    uint8_t* dst = my_stages + s * C::kStageBytes;
    mbar_arrive_expect_tx(&my_bars[s], C::kStageBytes);
#pragma unroll
    for (int bx = 0; bx < C::kBoxes; ++bx) {
      tma_load_3d(dst + bx * 2048, &tm_kv, &my_bars[s], bx * 64, row_k, page, kEvictFirst);
      tma_load_3d(dst + C::kTileBytes + bx * 2048, &tm_kv, &my_bars[s], bx * 64, row_v, page, kEvictFirst);
    }
  };
  if (lane == 0) {
    for (int s = 0; s < C::kStages; ++s) mbar_init(&my_bars[s], 1);
    fence_barrier_init();
    const int pre = min(n_my, C::kStages);
    for (int i = 0; i < pre; ++i) issue(i);
  }
  __syncwarp();

  uint32_t qa[D / 16][2], qb[D / 16][2];
  {
    const __nv_bfloat16* ql = a.q + (static_cast<long long>(b0 + r_lo) * a.n_q_heads + kvh * G + g % G) * D;
    const __nv_bfloat16* qh = a.q + (static_cast<long long>(b0 + r_hi) * a.n_q_heads + kvh * G + (g + 8) % G) * D;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      qa[kk][0] = v_lo ? *reinterpret_cast<const uint32_t*>(ql + kk * 16 + 2 * t) : 0u;
      qa[kk][1] = v_lo ? *reinterpret_cast<const uint32_t*>(ql + kk * 16 + 8 + 2 * t) : 0u;
      qb[kk][0] = v_hi ? *reinterpret_cast<const uint32_t*>(qh + kk * 16 + 2 * t) : 0u;
      qb[kk][1] = v_hi ? *reinterpret_cast<const uint32_t*>(qh + kk * 16 + 8 + 2 * t) : 0u;
    }
  }
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_lo = -INFINITY, l_lo = 0.f, m_hi = -INFINITY, l_hi = 0.f;
  const int mi = lane >> 3;
  const int mr = lane & 7;

  // online softmax of one half (e0: accumulator element offset 0 = row g, 2 = row g + 8)
  auto soft = [&](const float (&sacc)[2][4], int e0, int row_ctx, int tok0, float& m_run, float& l_run, float (&p)[4]) {
    float sv[4];
    float mx = -INFINITY;
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = tok0 + n * 8 + 2 * t + e;
        const float x = tok < row_ctx ? sacc[n][e0 + e] * a.scale_log2 : -INFINITY;
        sv[n * 2 + e] = x;
        mx = fmaxf(mx, x);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    // a page wholly past this row's causal limit leaves the state untouched
    const float corr = (m_new == -INFINITY) ? 1.f : exp2f(m_run - m_new);
    m_run = m_new;
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = (m_new == -INFINITY) ? 0.f : exp2f(sv[e] - m_new);
    l_run = l_run * corr + (p[0] + p[1] + p[2] + p[3]);
    return corr;
  };

  for (int i = 0; i < n_my; ++i) {
    const int s = i % C::kStages;
    mbar_wait(&my_bars[s], (i / C::kStages) & 1);
    const uint32_t kbase = smem_u32(my_stages + s * C::kStageBytes);
    const uint32_t vbase = kbase + C::kTileBytes;
    const int tok0 = (p0 + warp + i * C::kWarps) * kPageTokens;
    float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t r0, r1, r2, r3;
      const int tok = ((mi >> 1) << 3) + mr;
      const int dim = kk * 16 + ((mi & 1) << 3);
      ldmatrix_x4(kbase + kv_swz(tok, dim), r0, r1, r2, r3);
      mma_16816(sacc[0], qa[kk][0], qb[kk][0], qa[kk][1], qb[kk][1], r0, r1);
      mma_16816(sacc[1], qa[kk][0], qb[kk][0], qa[kk][1], qb[kk][1], r2, r3);
    }
    float pl[4], ph[4] = {0.f, 0.f, 0.f, 0.f};
    const float c_lo = soft(sacc, 0, ctx_lo, tok0, m_lo, l_lo, pl);
    float c_hi = 1.f;
    if (has_hi) c_hi = soft(sacc, 2, ctx_hi, tok0, m_hi, l_hi, ph);
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      o[n][0] *= c_lo;
      o[n][1] *= c_lo;
      o[n][2] *= c_hi;
      o[n][3] *= c_hi;
    }
    const uint32_t a0 = pack_bf16x2(pl[0], pl[1]), a2 = pack_bf16x2(pl[2], pl[3]);
    const uint32_t a1 = pack_bf16x2(ph[0], ph[1]), a3 = pack_bf16x2(ph[2], ph[3]);
    const uint32_t b0l = pack_bf16x2(pl[0] - bf16_round(pl[0]), pl[1] - bf16_round(pl[1]));
    const uint32_t b2l = pack_bf16x2(pl[2] - bf16_round(pl[2]), pl[3] - bf16_round(pl[3]));
    const uint32_t b1l = pack_bf16x2(ph[0] - bf16_round(ph[0]), ph[1] - bf16_round(ph[1]));
    const uint32_t b3l = pack_bf16x2(ph[2] - bf16_round(ph[2]), ph[3] - bf16_round(ph[3]));
#pragma unroll
    for (int nn = 0; nn < D / 16; ++nn) {
      uint32_t r0, r1, r2, r3;
      const int tok = ((mi & 1) << 3) + mr;
      const int dim = nn * 16 + ((mi >> 1) << 3);
      ldmatrix_x4_trans(vbase + kv_swz(tok, dim), r0, r1, r2, r3);
      mma_16816(o[2 * nn], a0, a1, a2, a3, r0, r1);
      mma_16816(o[2 * nn + 1], a0, a1, a2, a3, r2, r3);
      mma_16816(o[2 * nn], b0l, b1l, b2l, b3l, r0, r1);
      mma_16816(o[2 * nn + 1], b0l, b1l, b2l, b3l, r2, r3);
    }
    __syncwarp();
    if (lane == 0 && i + C::kStages < n_my) {
      fence_proxy_async_smem();
      issue(i + C::kStages);
    }
  }
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);

  __syncthreads();
  float* merge_o = reinterpret_cast<float*>(smem);  // [warps][16][D]
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    merge_o[(warp * 16 + g) * D + n * 8 + 2 * t] = o[n][0];
    merge_o[(warp * 16 + g) * D + n * 8 + 2 * t + 1] = o[n][1];
    merge_o[(warp * 16 + g + 8) * D + n * 8 + 2 * t] = o[n][2];
    merge_o[(warp * 16 + g + 8) * D + n * 8 + 2 * t + 1] = o[n][3];
  }
  if (t == 0) {
    merge_ml[(warp * 16 + g) * 2 + 0] = m_lo;
    merge_ml[(warp * 16 + g) * 2 + 1] = l_lo;
    merge_ml[(warp * 16 + g + 8) * 2 + 0] = m_hi;
    merge_ml[(warp * 16 + g + 8) * 2 + 1] = l_hi;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nr * G * D; idx += blockDim.x) {
    const int qr = idx / D;
    const int dim = idx % D;
    const int b = b0 + qr / G;
    const int head = kvh * G + qr % G;
    // this row's own split count (the combine kernel uses the same rule)
    const int npr = (row_ctx(a, b) + kPageTokens - 1) / kPageTokens;
    const int nsr = (npr + a.pages_per_split - 1) / a.pages_per_split;
    if (split >= nsr) continue;  // wholly past this row's causal limit
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < C::kWarps; ++w) mm = fmaxf(mm, merge_ml[(w * 16 + qr) * 2]);
    float acc = 0.f, ll = 0.f;
#pragma unroll
    for (int w = 0; w < C::kWarps; ++w) {
      const float mw = merge_ml[(w * 16 + qr) * 2];
      const float sc = (mw == -INFINITY) ? 0.f : exp2f(mw - mm);
      acc += merge_o[(w * 16 + qr) * D + dim] * sc;
      ll += merge_ml[(w * 16 + qr) * 2 + 1] * sc;
    }
    if (nsr == 1) {
      store_attn_out<D>(a, b, head, dim, acc / ll);
      continue;
    }
    const long long u = (static_cast<long long>(b) * a.n_q_heads + head) * a.max_splits + split;
    a.part_o[u * D + dim] = acc;
    if (dim == 0) {
      a.part_ml[u * 2 + 0] = mm;
      a.part_ml[u * 2 + 1] = ll;
    }
  }
}

// Merge the split partials of one (sequence, query head) and emit the bf16
// output (used when fused_combine == 0: all (b, head) merged in parallel).
template <int D>
__global__ void __launch_bounds__(128) attn_combine_kernel(const AttnArgs a) {
  pdl_wait();
  pdl_launch_dependents();
  const int head = blockIdx.x;
  const int b = blockIdx.y;
  const int ctx = row_ctx(a, b);
  const int n_pages = (ctx + kPageTokens - 1) / kPageTokens;
  const int n_splits = (n_pages + a.pages_per_split - 1) / a.pages_per_split;
  if (n_splits == 1) return;  // the attention kernel emitted this sequence's output directly
  const long long u0 = (static_cast<long long>(b) * a.n_q_heads + head) * a.max_splits;
  float mm = -INFINITY;
  for (int s = 0; s < n_splits; ++s) mm = fmaxf(mm, a.part_ml[(u0 + s) * 2]);
  for (int dim = threadIdx.x; dim < D; dim += blockDim.x) {
    float acc = 0.f, ll = 0.f;
    for (int s = 0; s < n_splits; ++s) {
      const float sc = exp2f(a.part_ml[(u0 + s) * 2] - mm);
      acc += a.part_o[(u0 + s) * D + dim] * sc;
      ll += a.part_ml[(u0 + s) * 2 + 1] * sc;
    }
    store_attn_out<D>(a, b, head, dim, acc / ll);
  }
}

}  // namespace sun
