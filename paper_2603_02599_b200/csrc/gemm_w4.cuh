// gemm_w4.cuh — QSUN W4A16 path: int4 weights dequantised in-kernel, fed to tcgen05.
//
// Storage format "SUN-W4" (restated bit-for-bit by oracle/quant_ref.py):
//   * symmetric per-group quantisation along K, group = 128, one bf16 scale per
//     (group, row) stored group-major: scales[K/128][round_up(rows,128)];
//   * q = clamp(rint(w / s), -8, 7), s = bf16(absmax / 7.5) (s = 0 -> q = 0);
//   * packed bytes are tile-contiguous: block (row/128, k/128) is 128 rows x 64 B
//     (8 KB, one bulk copy per stage); every 32-bit word holds 8 consecutive k elements
//     as offset-binary nibbles (q + 8) in nibble order [0,2,4,6,1,3,5,7], so one
//     shift + LOP3 yields a bf16x2 pair (128 + u_even, 128 + u_odd).
// Dequantised operand = bf16(q * s) exactly (HSUB2 is exact, HMUL2 rounds once).
//
// Pipeline per 128-wide K block: TMA {packed 8 KB, scales 256 B, X 2 x bn x 128 B}
// -> warps 2..5 dequantise into a SW128 bf16 tile (2 atoms x 128 rows x 128 B)
// -> warp 1 issues 8 tcgen05.mma (K=16 each) -> same warps run the epilogue.
// The lm_head stays bf16 and uses gemm_bf16_kernel.
#pragma once
#include "gemm_tc.cuh"

namespace sun {

struct W4Weights {
  const void* packed;  // uint8, tile-contiguous 128x64 B blocks
  const void* scales;  // bf16 [K/128][round_up(rows,128)]
};

constexpr int kW4Threads = 192;
constexpr int kW4K = 128;                            // K per stage (= quant group)
constexpr uint32_t kW4PackedBytes = kTileM * kW4K / 2;  // 8 KB
constexpr uint32_t kW4ScaleBytes = kTileM * 2;          // 256 B
constexpr uint32_t kW4DeqBytes = kTileM * kW4K * 2;     // 32 KB (2 SW128 atoms)
constexpr int kW4DeqBufs = 2;

__host__ __device__ inline uint32_t w4_stage_bytes(int bn) {
  return kW4PackedBytes + 1024 + static_cast<uint32_t>(bn) * 256;  // scales padded to 1 KB
}
__host__ __device__ inline size_t w4_smem_bytes(int bn, int stages) {
  return 1024 + size_t(kW4DeqBufs) * kW4DeqBytes + size_t(stages) * w4_stage_bytes(bn) + 512;
}

template <int EPI>
__global__ void __launch_bounds__(kW4Threads, 1)
    gemm_w4_kernel(const W4Weights ww, const __grid_constant__ CUtensorMap tm_x, const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stages = a.stages;
  const uint32_t sb = w4_stage_bytes(a.bn);
  uint8_t* deq = smem;                                   // [2][32 KB]
  uint8_t* stg = smem + kW4DeqBufs * kW4DeqBytes;        // [stages][packed | scales | X]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + stages * sb);
  uint64_t* empty = full + stages;          // count 2: converter done + MMA done with X
  uint64_t* dfull = empty + stages;         // count 1: converters published the bf16 tile
  uint64_t* dempty = dfull + kW4DeqBufs;    // count 1: MMA done with the bf16 tile
  uint64_t* tmem_full = dempty + kW4DeqBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = warp_id_sync();
  const int lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x;
  const int split = blockIdx.y;
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(a.kb_total, kb0 + a.kb_per_split);
  const int nkb = kb1 - kb0;
  const long long rows_pad = static_cast<long long>(a.kb_total > 0 ? (a.n_out + kTileM - 1) / kTileM : 0) * kTileM;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_x);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);
    }
    for (int j = 0; j < kW4DeqBufs; ++j) {
      mbar_init(&dfull[j], 1);
      mbar_init(&dempty[j], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const uint8_t* gpk = static_cast<const uint8_t*>(ww.packed);
  const __nv_bfloat16* gsc = static_cast<const __nv_bfloat16*>(ww.scales);

  if (warp == 0) {
    if (elect_one()) {
      bool waited = false;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % stages;
        const uint32_t ph = (i / stages) & 1;
        if (i >= stages) mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = stg + s * sb;
        const int kb = kb0 + i;
        mbar_arrive_expect_tx(&full[s], kW4PackedBytes + kW4ScaleBytes + a.bn * 256);
        // packed rows of this tile are 64 B apart in smem: 128 row copies of 64 B
        // would be slow; the packed matrix is tile-contiguous (see quantizer), so
        // one bulk copy moves the whole 8 KB block.
        const uint8_t* src = gpk + (static_cast<long long>(m_tile) * a.kb_total + kb) * kW4PackedBytes;
        bulk_load(st, src, kW4PackedBytes, &full[s]);
        bulk_load(st + kW4PackedBytes, gsc + static_cast<long long>(kb) * rows_pad + static_cast<long long>(m_tile) * kTileM,
                  kW4ScaleBytes, &full[s]);
        if (!waited) {
          pdl_wait();
          waited = true;
        }
        tma_load_2d(st + kW4PackedBytes + 1024, &tm_x, &full[s], kb * kW4K, 0, kEvictLast);
        tma_load_2d(st + kW4PackedBytes + 1024 + a.bn * 128, &tm_x, &full[s], kb * kW4K + 64, 0, kEvictLast);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc_bf16(kTileM, a.bn);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % stages;
      const int j = i % kW4DeqBufs;
      mbar_wait(&full[s], (i / stages) & 1);
      mbar_wait(&dfull[j], (i / kW4DeqBufs) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t wa = smem_u32(deq + j * kW4DeqBytes);
        const uint32_t xa = smem_u32(stg + s * sb + kW4PackedBytes + 1024);
#pragma unroll
        for (int kk = 0; kk < kW4K / 16; ++kk) {
          const uint32_t atom = kk >> 2;
          const uint32_t koff = (kk & 3) * 32;
          umma_bf16(tmem_base, make_sw128_desc(wa + atom * (kTileM * 128) + koff),
                    make_sw128_desc(xa + atom * (a.bn * 128) + koff), idesc, (i | kk) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);
        umma_commit(&dempty[j]);
        if (i == nkb - 1) umma_commit(tmem_full);
      }
      __syncwarp();
    }
  } else {
    // ---------------- converters (mainloop), then epilogue ----------------
    const int ct = threadIdx.x - 64;  // 0..127
    for (int i = 0; i < nkb; ++i) {
      const int s = i % stages;
      const int j = i % kW4DeqBufs;
      mbar_wait(&full[s], (i / stages) & 1);
      if (i >= kW4DeqBufs) mbar_wait(&dempty[j], ((i / kW4DeqBufs) & 1) ^ 1);
      const uint8_t* pk = stg + s * sb;
      const __nv_bfloat16* sc = reinterpret_cast<const __nv_bfloat16*>(pk + kW4PackedBytes);
      uint8_t* dq = deq + j * kW4DeqBytes;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int r = p * 32 + (ct >> 2);
        const int c4 = ct & 3;  // 16-byte packed chunk = 32 k elements
        const uint4 w = *reinterpret_cast<const uint4*>(pk + r * 64 + c4 * 16);
        const __nv_bfloat162 s2 = __bfloat162bfloat162(sc[r]);
        const __nv_bfloat162 off = __floats2bfloat162_rn(136.f, 136.f);
        const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t u = ((words[q] >> (4 * e)) & 0x000F000Fu) | 0x43004300u;
            __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&u);
            v = __hmul2(__hsub2(v, off), s2);
            o[e] = *reinterpret_cast<uint32_t*>(&v);
          }
          // chunk index within the 128-wide k block: (c4*32 + q*8) / 8
          const int c = c4 * 4 + q;
          const int atom = c >> 3;
          const int phys = (c & 7) ^ (r & 7);
          *reinterpret_cast<uint4*>(dq + atom * (kTileM * 128) + r * 128 + phys * 16) = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      fence_proxy_async_smem();
      epi_bar();
      if (ct == 0) {
        mbar_arrive(&dfull[j]);
        mbar_arrive(&empty[s]);
      }
    }
    // ---------------- epilogue ----------------
    pdl_wait();
    const int q = warp & 3;
    const int row_local = q * 32 + lane;
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    float* stage_f32 = reinterpret_cast<float*>(deq);  // deq buffers idle once tmem_full fires
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
        for (int jj = 0; jj < 16; ++jj) part[(c0 + jj) * kTileM + row_local] = v[jj];
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
          for (int jj = 0; jj < 16; ++jj) v[jj] = __ldcg(base + (c0 + jj) * kTileM + row_local);
          for (int s = 1; s < a.splits; ++s) {
            const float* ps = base + static_cast<long long>(s) * a.bn * kTileM;
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) v[jj] += __ldcg(ps + (c0 + jj) * kTileM + row_local);
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
  scales[g * rows_pad + r] = sb;
  const long long kb_total = k / 128;
  uint8_t* dst = packed + ((r / 128) * kb_total + g) * 8192 + (r % 128) * 64;
  for (int wd = 0; wd < 16; ++wd) {  // 16 words of 8 elements
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
    reinterpret_cast<uint32_t*>(dst)[wd] = word;
  }
}

}  // namespace sun
