// gemm_tc.cuh — tcgen05/TMEM swap-AB GEMM for the decode module's linear layers.
//
//   D^T[n_out, B] = W[n_out, K] . X[B, K]^T
//
// Weight rows are the MMA M dimension (128 per tile), the cross-model decode
// batch is the MMA N dimension (bn = round_up(B, 16) <= 256), K is streamed in
// 64-element (128 B, SWIZZLE_128B) blocks by TMA through an mbarrier ring.
// Warp roles: warp 0 = TMA producer, warp 1 = TMEM allocator + single-thread
// MMA issuer, warps 2..5 = epilogue (TMEM -> registers -> fused epilogue).
// Split-K across CTAs is reduced deterministically by the last-arriving CTA of
// each tile (fixed split order), so results are run-to-run bit-identical.
//
// Replaces the weight term `decoder_weight_bytes / (mbu * hbm_bandwidth)` of
// the reference's step price (poolsim costmodel.py:101-113) with real work.
#pragma once
#include "sun_common.cuh"

namespace sun {

enum EpiKind : int {
  EPI_STORE_F32 = 0,  // out_f32[b*ldo + row] = acc
  EPI_RESID_ADD = 1,  // out_f32[b*ldo + row] += acc           (O-proj, down-proj)
  EPI_QKV_ROPE = 2,   // +bias, RoPE(q,k), q -> bf16, k/v -> paged KV cache
  EPI_SWIGLU = 3,     // rows interleaved in 64-row blocks: act = silu(gate) * up
  EPI_LOGITS = 4,     // logits fp32 + per-tile (max, argmax) per batch column
};

struct GemmArgs {
  int n_out;         // rows of W (incl. zero padding rows for SWIGLU)
  int k;             // reduction length
  int batch;         // valid batch columns
  int bn;            // padded N: multiple of 16, <= 256
  int kb_total;      // ceil(k / 64)
  int kb_per_split;  // k-blocks handled by one CTA
  int splits;        // gridDim.y
  int stages;        // smem pipeline depth
  int weight_bits;   // 16 (bf16) — 4 handled by the W4 kernel
  float* partial;    // [m_tiles][splits][bn][128] fp32 (splits > 1)
  unsigned* counters;  // [m_tiles], zero-initialised, self-resetting
  // STORE / RESID / LOGITS
  float* out_f32;
  long long ldo;
  // SWIGLU (act) / QKV (q)
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
  // LOGITS
  float* amax_val;  // [m_tiles][bn]
  int* amax_idx;    // [m_tiles][bn]
};

constexpr int kGemmThreads = 192;
constexpr int kTileM = 128;
constexpr int kTileK = 64;
constexpr uint32_t kTileWBytes = kTileM * kTileK * 2;  // 16 KB
constexpr uint32_t kTmemCols = 256;

__host__ __device__ inline size_t gemm_smem_bytes(int bn, int stages) {
  return 1024 + static_cast<size_t>(stages) * (kTileWBytes + bn * 128) + 256;
}

SUN_DEVICE void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

template <int EPI>
SUN_DEVICE void epi_chunk(const GemmArgs& a, int m_tile, int row_local, int c0, float (&v)[16],
                          float* stage_f32, float* red_val, int* red_idx) {
  const int row = m_tile * kTileM + row_local;
  const int B = a.batch;
  if constexpr (EPI == EPI_STORE_F32 || EPI == EPI_RESID_ADD) {
    if (row < a.n_out) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int b = c0 + j;
        if (b < B) {
          float* p = a.out_f32 + static_cast<long long>(b) * a.ldo + row;
          if constexpr (EPI == EPI_RESID_ADD) *p += v[j];
          else *p = v[j];
        }
      }
    }
  } else if constexpr (EPI == EPI_LOGITS) {
    const int lane = threadIdx.x & 31;
    const int q = (threadIdx.x / 32) & 3;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
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
        red_val[q * 16 + j] = val;
        red_idx[q * 16 + j] = idx;
      }
    }
    epi_bar();
    if (threadIdx.x / 32 == 2 && lane < 16) {
      float val = red_val[lane];
      int idx = red_idx[lane];
#pragma unroll
      for (int w = 1; w < 4; ++w) {
        const float ov = red_val[w * 16 + lane];
        const int oi = red_idx[w * 16 + lane];
        if (ov > val || (ov == val && oi < idx)) {
          val = ov;
          idx = oi;
        }
      }
      a.amax_val[static_cast<long long>(m_tile) * a.bn + c0 + lane] = val;
      a.amax_idx[static_cast<long long>(m_tile) * a.bn + c0 + lane] = idx;
    }
    epi_bar();
  } else {
    // QKV_ROPE / SWIGLU need a partner row of the same tile: stage through smem.
    epi_bar();  // previous chunk's partner reads are done
    if constexpr (EPI == EPI_QKV_ROPE) {
      const float bias = (a.bias != nullptr && row < a.n_out) ? __bfloat162float(a.bias[row]) : 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] += bias;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) stage_f32[j * kTileM + row_local] = v[j];
    epi_bar();
    if constexpr (EPI == EPI_SWIGLU) {
      if (row_local < 64) {
        const int jo = m_tile * 64 + row_local;
        if (jo < a.n_valid_out) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int b = c0 + j;
            if (b < B) {
              const float g = v[j];
              const float u = stage_f32[j * kTileM + row_local + 64];
              const float s = g / (1.f + expf(-g));
              a.out_bf16[static_cast<long long>(b) * a.ldb + jo] = __float2bfloat16_rn(s * u);
            }
          }
        }
      }
    } else {  // EPI_QKV_ROPE
      if (row < a.n_out) {
        const int d = a.head_dim;
        const int half = d >> 1;
        const int qd = a.n_q_heads * d;
        const int kd = a.n_kv_heads * d;
        const int i = row % d;
        const int fi = i < half ? i : i - half;
        const int partner = i < half ? row_local + half : row_local - half;
        const bool is_v = row >= qd + kd;
#pragma unroll 4
        for (int j = 0; j < 16; ++j) {
          const int b = c0 + j;
          if (b >= B) break;
          const int pos = a.positions[b];
          float o = v[j];
          if (!is_v) {
            const float pv = stage_f32[j * kTileM + partner];
            const float cs = a.rope_cos[static_cast<long long>(pos) * half + fi];
            const float sn = a.rope_sin[static_cast<long long>(pos) * half + fi];
            o = i < half ? (v[j] * cs - pv * sn) : (v[j] * cs + pv * sn);
          }
          const __nv_bfloat16 ob = __float2bfloat16_rn(o);
          if (row < qd) {
            a.out_bf16[static_cast<long long>(b) * a.ldb + row] = ob;
          } else {
            const int kvsel = is_v ? 1 : 0;
            const int g = (row - qd - kvsel * kd) / d;
            const int page = a.block_tables[static_cast<long long>(b) * a.bt_stride + pos / a.page_size];
            const int slot = pos % a.page_size;
            const long long off =
                static_cast<long long>(page) * a.page_stride +
                ((static_cast<long long>(a.layer * 2 + kvsel) * a.n_kv_heads + g) * a.page_size + slot) * d + i;
            a.kv_base[off] = ob;
          }
        }
      }
    }
  }
}

template <int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                     const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stages = a.stages;
  const uint32_t x_bytes = static_cast<uint32_t>(a.bn) * 128u;
  const uint32_t stage_bytes = kTileWBytes + x_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tmem_full = empty + stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = warp_id_sync();
  const int lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x;
  const int split = blockIdx.y;
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(a.kb_total, kb0 + a.kb_per_split);
  const int nkb = kb1 - kb0;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // Weights do not depend on the previous kernel: start streaming them
      // before the grid dependency resolves, then the activations.
      const int pre = min(nkb, stages);
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], stage_bytes);
        tma_load_2d(smem + i * stage_bytes, &tm_w, &full[i], (kb0 + i) * kTileK, m_tile * kTileM, kEvictFirst);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i)
        tma_load_2d(smem + i * stage_bytes + kTileWBytes, &tm_x, &full[i], (kb0 + i) * kTileK, 0, kEvictLast);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % stages;
        const uint32_t ph = (i / stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        tma_load_2d(smem + s * stage_bytes, &tm_w, &full[s], (kb0 + i) * kTileK, m_tile * kTileM, kEvictFirst);
        tma_load_2d(smem + s * stage_bytes + kTileWBytes, &tm_x, &full[s], (kb0 + i) * kTileK, 0, kEvictLast);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc_bf16(kTileM, a.bn);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t wa = smem_u32(smem + s * stage_bytes);
        const uint32_t xa = wa + kTileWBytes;
#pragma unroll
        for (int kk = 0; kk < kTileK / 16; ++kk) {
          umma_bf16(tmem_base, make_sw128_desc(wa + kk * 32), make_sw128_desc(xa + kk * 32), idesc,
                    (i | kk) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);
        if (i == nkb - 1) umma_commit(tmem_full);
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: warps 2..5 ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_local = q * 32 + lane;
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    float* stage_f32 = reinterpret_cast<float*>(smem);  // pipeline buffers are idle now
    float* red_val = stage_f32 + 16 * kTileM;
    int* red_idx = reinterpret_cast<int*>(red_val + 64);
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    float v[16];
    if (a.splits == 1) {
      for (int c0 = 0; c0 < a.bn; c0 += 16) {
        tmem_ld16(taddr + c0, v);
        epi_chunk<EPI>(a, m_tile, row_local, c0, v, stage_f32, red_val, red_idx);
      }
    } else {
      float* part = a.partial + (static_cast<long long>(m_tile) * a.splits + split) * a.bn * kTileM;
      for (int c0 = 0; c0 < a.bn; c0 += 16) {
        tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) part[(c0 + j) * kTileM + row_local] = v[j];
      }
      __threadfence();
      epi_bar();
      if (threadIdx.x == 64) {
        const unsigned prev = atomicAdd(&a.counters[m_tile], 1u);
        const int last = (prev == static_cast<unsigned>(a.splits - 1));
        if (last) a.counters[m_tile] = 0u;
        *last_flag = last;
      }
      epi_bar();
      if (*last_flag) {
        __threadfence();
        const float* base = a.partial + static_cast<long long>(m_tile) * a.splits * a.bn * kTileM;
        for (int c0 = 0; c0 < a.bn; c0 += 16) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __ldcg(base + (c0 + j) * kTileM + row_local);
          for (int s = 1; s < a.splits; ++s) {
            const float* ps = base + static_cast<long long>(s) * a.bn * kTileM;
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += __ldcg(ps + (c0 + j) * kTileM + row_local);
          }
          epi_chunk<EPI>(a, m_tile, row_local, c0, v, stage_f32, red_val, red_idx);
        }
      }
    }
  }
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

}  // namespace sun
