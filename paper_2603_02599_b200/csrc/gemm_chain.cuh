// gemm_chain.cuh — a layer's GEMM chain (O-proj -> gate_up -> down -> next QKV) as
// one persistent launch of 148 CTAs (one per SM).
//
// Why: between two separate GEMM launches the next GEMM's CTAs only become resident
// when the previous GEMM's CTAs exit (each holds ~200 KB of shared memory), so its
// weight stream starts after the previous tail (split-K reduction + fused epilogue,
// several µs) and its ramp is exposed. Here the weight producer of every CTA runs
// ahead across phase boundaries — the next GEMM's weights stream into the ring
// while the epilogue warps finish the current phase — and only the activation
// producer waits for the grid-wide "phase p done" count before loading phase p's
// input. Whole-tile phases use the TMEM double buffer across phase boundaries. Split
// phases reduce either through DSMEM (launched as 4-CTA clusters, c.hw: S = 4 or 2
// ranks of a tile inside one cluster st.async the chunks their peers own into the
// peers' receive areas) or through L2 (148 plain CTAs: virtual clusters, gemm_tc.cuh).
//
// Deadlock freedom: the host sizes the grid so that every CTA (every cluster) is
// co-resident once the previous kernel drains (PDL: the dependent launch needs every
// CTA of this grid to have started); the only cross-CTA waits are phase counts,
// per-tile split counters and DSMEM receive barriers, all fed by epilogue warps that
// never wait on anything but their own CTA's MMA and the previous phase.
#pragma once
#include "gemm_tc.cuh"

namespace sun {

constexpr int kChainMaxPhases = 4;

struct ChainArgs {
  GemmArgs ph[kChainMaxPhases];
  int epi[kChainMaxPhases];  // EpiKind per phase
  int nph;
  int hw;  // 1: launched as 4-CTA clusters; split phases with vcluster == 0 (S = 4) reduce
           // through DSMEM: ranks st.async the chunks their peers own into the peers'
           // receive areas (smem after the barriers), completion on per-phase mbarriers
  unsigned long long* stamps;  // profiling: per CTA [16] = per phase p: [4p] activations ready,
                               // [4p+1] first MMA, [4p+2] last MMA issued, [4p+3] epilogue done
  unsigned* bar;  // [2]: phases completed x CTAs, CTAs exited (zeroed once, self-resetting)
  unsigned* ready;  // bf16 chain, non-null: [kChainMaxPhases][kChainReadyTiles] per-tile counts of the
                    // CTAs that finished writing a phase's output tile; the next phase's activation
                    // stages wait only for the tiles they read (zeroed by the last CTA out)
  unsigned* qkv_ready;  // non-null: the last (QKV) phase publishes its tiles here (per-tile writer
                        // counts) for the next layer's attention (SUN_ATTN_TILE_READY)
  unsigned* qkv_reset;  // non-null: this layer's counters, read by the attention that precedes this
                        // chain: zeroed once that attention has completed (after griddepcontrol.wait)
  int qkv_reset_n;
  unsigned long long* tl;
  int tl_idx;
};

struct PhaseSched {
  int u0, u1, n, t_first, nseg, S, rank;
};

SUN_DEVICE PhaseSched phase_sched(const GemmArgs& a) {
  PhaseSched p;
  const int KS = a.ksteps, G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  p.S = a.splits > 1 ? a.splits : 1;
  p.rank = 0;
  if (p.S > 1) {
    if (c < a.m_tiles * p.S) {
      const int t = c / p.S;
      p.rank = c % p.S;
      p.u0 = t * KS + p.rank * KS / p.S;
      p.u1 = t * KS + (p.rank + 1) * KS / p.S;
    } else {
      p.u0 = p.u1 = 0;  // idle in this phase
    }
  } else {
    p.u0 = static_cast<int>(static_cast<long long>(c) * a.m_tiles / G) * KS;
    p.u1 = static_cast<int>(static_cast<long long>(c + 1) * a.m_tiles / G) * KS;
  }
  p.n = p.u1 - p.u0;
  p.t_first = p.n > 0 ? p.u0 / KS : 0;
  p.nseg = p.n > 0 ? (p.u1 - 1) / KS - p.t_first + 1 : 0;
  return p;
}

#define SUN_CSTAMP(i) \
  do { if (c.stamps) c.stamps[blockIdx.x * 16 + (i)] = gtimer(); } while (0)

// Cross-CTA waits carry a watchdog: a grid that cannot become resident as a whole
// (e.g. another persistent kernel holding SMs) traps after 2 s — the launch fails with
// an error instead of hanging the GPU.
constexpr unsigned long long kChainWatchdogNs = 2000000000ull;
constexpr int kChainReadyTiles = 1024;
constexpr int kQkvReadyStride = 256;  // per-layer QKV tile counters of the attention hand-off

// Per-tile readiness (bf16 chain): the activation producer of phase p waits for the
// producer tiles of phase p - 1 that its K steps read, instead of the whole phase. `rp`
// is the ready prefix of the producer's tiles (tiles < rp all complete); a poll round
// reads 16 counters at once (relaxed loads, then an acquire fence: one round trip) and
// the grid count (every tile of the phase done).
SUN_DEVICE void chain_wait_tiles(const unsigned* rd, unsigned writers, int need_hi, int tiles, int& rp,
                                 const unsigned* bar, unsigned phase_target) {
  if (need_hi < rp) return;
  const unsigned long long t0 = gtimer();
  for (;;) {
    unsigned v[16];
    const int base = rp;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      v[i] = base + i < tiles ? *reinterpret_cast<const volatile unsigned*>(rd + base + i) : writers;
    const unsigned b = *reinterpret_cast<const volatile unsigned*>(bar);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (b >= phase_target) {
      rp = tiles;
      return;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (rp == base + i && v[i] >= writers) ++rp;
    }
    if (need_hi < rp) return;
    __nanosleep(32);
    if (gtimer() - t0 > kChainWatchdogNs) __trap();
  }
}

SUN_DEVICE void chain_wait_phase(const unsigned* bar, unsigned target) {
  if (target == 0) return;
  const unsigned long long t0 = gtimer();
  while (ld_acquire_u32(bar) < target) {
    __nanosleep(64);
    if (gtimer() - t0 > kChainWatchdogNs) __trap();
  }
}

SUN_DEVICE void chain_wait_mbar(uint64_t* bar, uint32_t parity) {
  const unsigned long long t0 = gtimer();
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (gtimer() - t0 > kChainWatchdogNs) __trap();
  }
}

SUN_DEVICE void epi_pair_bar() { asm volatile("bar.sync 4, 256;" ::: "memory"); }  // both epilogue groups

// One phase of the epilogue warps (both groups). Returns after every segment of
// this CTA's range is written out and the TMEM buffers are released.
SUN_DEVICE void st_async_f4(uint32_t addr, const float* v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "r"(mbar)
               : "memory");
}

template <int EPI>
SUN_DEVICE void chain_epilogue_phase(const GemmArgs& a, const PhaseSched& ps, float* epi, uint32_t tmem_base,
                                     uint64_t* tfull, uint64_t* tempty, int& buf, int& tphase, float* recv,
                                     uint64_t* rbar, unsigned* ready_p) {
  // this CTA's share of `tile` is written: publish it to the next phase's activation loads
  auto publish = [&](int tile, bool need_bar) {
    if (ready_p == nullptr) return;
    if (need_bar) epi_pair_bar();
    if (threadIdx.x == 64) {
      __threadfence();
      atomicAdd(ready_p + tile, 1u);
    }
  };
  const int warp = static_cast<int>(threadIdx.x >> 5);
  const int q = warp & 3;
  const int row_local = q * 32 + (threadIdx.x & 31);
  const int KS = a.ksteps;
  if (warp < 6) load_qkv_meta<EPI>(a, epi);
  epi_pair_bar();
  // Residual-phase inputs that do not depend on this phase's result — the previous
  // residual of the columns this group will finish and the next norm's gain — are copied
  // into the group's staging area with cp.async now, while the phase's MMAs run (no
  // registers held: the register preload measured slower through spills); the tail then
  // reads shared memory instead of paying a global round trip under a saturated HBM.
  // Hardware-cluster split phases with one 8-column chunk per group (O / down at bn <= 64).
  const float* pre_res = nullptr;
  float pre_gain = 0.f;
  if constexpr (EPI == EPI_RESID_ADD) {
#ifndef SUN_NO_RESPRE  // (A/B build switch)
    if (ps.nseg == 1 && ps.S > 1 && !a.vcluster && a.norm_w != nullptr &&
        (a.bn / 16 - ps.rank + ps.S - 1) / ps.S == 1) {
      float* dst = epi_stage(epi);  // [8 columns][128 rows]; the ss scratch sits above 8 KB
      const int row = ps.t_first * kTileM + row_local;
      const int c0 = ps.rank * 16 + 8 * epi_grp();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (row < a.n_out && c0 + j < a.batch)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst + j * kTileM + row_local)),
                       "l"(a.out_f32 + static_cast<long long>(c0 + j) * a.ldo + row)
                       : "memory");
        else
          dst[j * kTileM + row_local] = 0.f;
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      pre_gain = row < a.n_out ? __bfloat162float(a.norm_w[row]) : 0.f;
      pre_res = dst + row_local;
    }
#endif
  }
  for (int seg = 0; seg < ps.nseg; ++seg) {
    const int tile = ps.t_first + seg;
    mbar_wait(&tfull[buf], tphase);
    tc_fence_after();
    const uint32_t taddr = tmem_base + static_cast<uint32_t>(buf * a.bn) + (static_cast<uint32_t>(q * 32) << 16);
    if (ps.S == 1) {
      direct_epilogue<EPI>(a, tile, taddr, epi, 2);
      tc_fence_before();
      epi_bar();
      if (epi_lead_thread()) mbar_arrive(&tempty[buf]);
      publish(tile, true);
    } else if (!a.vcluster) {
      // hardware cluster (S = 2 or 4 ranks of one tile, 4 / S tiles per 4-CTA cluster):
      // send every chunk another rank owns (chunk c -> rank c % S, slot = our rank among
      // its S - 1 senders) straight from TMEM into its receive area; the two groups take
      // alternate chunks
      const int S = ps.S, rank = ps.rank, nch = a.bn / 16, nmax = (nch + S - 1) / S;
      const int cta0 = static_cast<int>(blockIdx.x & 3u) - rank;  // cluster rank of the tile's rank 0
      int idx = 0;
      for (int c = 0; c < nch; ++c) {
        const int o = c % S;
        if (o == rank) continue;
        if ((idx++ & 1) != epi_grp()) continue;
        const int slot = rank < o ? rank : rank - 1;
        float v[16];
        tmem_ld16(taddr + c * 16, v);
        const float* dst = recv + (slot * nmax + c / S) * 2048;
        const uint32_t mb = dsmem_addr(rbar, static_cast<uint32_t>(cta0 + o));
#pragma unroll
        for (int j = 0; j < 4; ++j)
          st_async_f4(dsmem_addr(dst + part_index(0, j, row_local), static_cast<uint32_t>(cta0 + o)), v + 4 * j, mb);
      }
      // reduce our chunks: rank order, our own partial read from TMEM (same sums as
      // the L2 path: ((0 + p0) + p1) + ...)
      chain_wait_mbar(rbar, 0);
      auto reduce_own = [&](int c, int q0, auto& v) {
        constexpr int NQ = sizeof(v) / sizeof(float) / 4;
        float own[4 * NQ];
        if constexpr (NQ == 4) tmem_ld16(taddr + c * 16, own);
        else tmem_ld8(taddr + c * 16 + 4 * q0, own);
#pragma unroll
        for (int j = 0; j < 4 * NQ; ++j) v[j] = 0.f;
        for (int r = 0; r < S; ++r) {
          if (r == rank) {
#pragma unroll
            for (int j = 0; j < 4 * NQ; ++j) v[j] += own[j];
          } else {
            const float* src = recv + ((r < rank ? r : r - 1) * nmax + c / S) * 2048;
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
              const float4 x = *reinterpret_cast<const float4*>(src + part_index(0, q0 + j, row_local));
              v[4 * j] += x.x;
              v[4 * j + 1] += x.y;
              v[4 * j + 2] += x.z;
              v[4 * j + 3] += x.w;
            }
          }
        }
      };
      const int nmine = (nch - rank + S - 1) / S;
      if (nmine == 1) {
        float v[8];
        reduce_own(rank, 2 * epi_grp(), v);
        tc_fence_before();
        epi_pair_bar();
        if (epi_lead_thread()) mbar_arrive(&tempty[buf]);  // accumulator read: the MMA may reuse it
        if (pre_res != nullptr) {
          asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's own prefetched values
          epi_chunk<EPI, 8>(a, tile, row_local, rank * 16 + 8 * epi_grp(), v, epi, pre_res, &pre_gain, kTileM);
        } else {
          epi_chunk<EPI, 8>(a, tile, row_local, rank * 16 + 8 * epi_grp(), v, epi);
        }
        publish(tile, true);
      } else {
        for (int c = rank + S * epi_grp(); c < nch; c += 2 * S) {
          float v[16];
          reduce_own(c, 0, v);
          epi_chunk<EPI>(a, tile, row_local, c * 16, v, epi);
        }
        tc_fence_before();
        epi_pair_bar();
        if (epi_lead_thread()) mbar_arrive(&tempty[buf]);
        publish(tile, false);
      }
    } else {
      // split phase: park this rank's partial in L2, meet the tile's S CTAs, reduce
      // this rank's columns (chunks rank, rank + S, ... alternate between the groups)
      const int S = ps.S, rank = ps.rank;
      if (epi_grp() == 0) {
        float* part = a.sk_part + static_cast<long long>(blockIdx.x) * a.bn * kTileM;
        float v[16];
        for (int c0 = 0; c0 < a.bn; c0 += 16) {
          tmem_ld16(taddr + c0, v);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            __stcg(reinterpret_cast<float4*>(part + part_index(c0, j, row_local)),
                   make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
        }
        __threadfence();
      }
      tc_fence_before();
      epi_pair_bar();
      if (epi_lead_thread()) mbar_arrive(&tempty[buf]);  // accumulator parked: the MMA may reuse it
      unsigned* tile_cnt = a.sk_flags + tile;
      if (threadIdx.x == 64) {
        atomicAdd(tile_cnt, 1u);
        const unsigned long long t0 = gtimer();
        while (ld_acquire_u32(tile_cnt) < static_cast<unsigned>(S))
          if (gtimer() - t0 > kChainWatchdogNs) __trap();
      }
      epi_pair_bar();
      const float* gpart = a.sk_part + static_cast<long long>(blockIdx.x - rank) * a.bn * kTileM;
      auto reduce_cols = [&](int c0, int q0, auto& v) {
        constexpr int NQ = sizeof(v) / sizeof(float) / 4;
        float4 x[4][NQ];
#pragma unroll
        for (int j = 0; j < 4 * NQ; ++j) v[j] = 0.f;
        const int cbase = c0 & ~15;
        for (int r0 = 0; r0 < S; r0 += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < NQ; ++j)
              x[u][j] = (r0 + u >= S) ? make_float4(0.f, 0.f, 0.f, 0.f)
                                      : __ldcg(reinterpret_cast<const float4*>(
                                            gpart + static_cast<long long>(r0 + u) * a.bn * kTileM +
                                            part_index(cbase, q0 + j, row_local)));
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
      const int cfirst = rank * 16, cstride = S * 16;
      const int nmine = (a.bn - cfirst + cstride - 1) / cstride;
      if (nmine == 1) {
        const int c0 = cfirst + 8 * epi_grp();
        float v[8];
        reduce_cols(c0, 2 * epi_grp(), v);
        epi_chunk<EPI, 8>(a, tile, row_local, c0, v, epi);
      } else {
        for (int c0 = cfirst + epi_grp() * cstride; c0 < a.bn; c0 += 2 * cstride) {
          float v[16];
          reduce_cols(c0, 0, v);
          epi_chunk<EPI>(a, tile, row_local, c0, v, epi);
        }
      }
      epi_pair_bar();  // the last of the tile's 2S arrivals rearms its counter
      if (threadIdx.x == 64 && atomicAdd(tile_cnt, 1u) == 2u * S - 1u) *tile_cnt = 0u;
      publish(tile, false);
    }
    if (++buf == 2) {
      buf = 0;
      tphase ^= 1;
    }
  }
}

__global__ void __launch_bounds__(kGemmThreads, 1) gemm_chain_kernel(const __grid_constant__ ChainArgs c) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  tl_begin(c.tl, c.tl_idx);
  const GemmArgs& a0 = c.ph[0];
  const int stages = a0.stages, xstages = a0.xstages, bn = a0.bn;
  const uint32_t sb = gemm_stage_bytes(bn, false);
  const uint32_t xsb = gemm_xstage_bytes(bn);
  uint8_t* stg = smem;
  uint8_t* xstg = stg + ((stages * sb + 1023u) & ~1023u);
  float* epi = reinterpret_cast<float*>(xstg + xstages * xsb);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(epi) + kEpiSmemBytes);
  uint64_t* empty = full + kMaxWStages;
  uint64_t* xfull = empty + kMaxWStages;
  uint64_t* xempty = xfull + kMaxXStages;
  uint64_t* tfull = xempty + kMaxXStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;  // [kChainMaxPhases] hardware split phases: peers' chunks landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + kChainMaxPhases);
  float* recv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 1024);
  const int warp = warp_id_sync();
  const unsigned G = gridDim.x;
  const uint32_t ncols = tmem_cols_for(bn);

  if (warp == 0 && elect_one()) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < xstages; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int j = 0; j < 2; ++j) {
      mbar_init(&tfull[j], 1);
      mbar_init(&tempty[j], 2);
    }
    for (int p = 0; p < kChainMaxPhases; ++p) mbar_init(&rbar[p], 1);
    fence_barrier_init();
    if (c.hw) {  // each hardware split phase: (S - 1) senders x our chunks x 8 KB
      for (int p = 0; p < c.nph; ++p) {
        const GemmArgs& a = c.ph[p];
        if (a.splits > 1 && !a.vcluster) {
          const int S = a.splits, r = static_cast<int>(blockIdx.x) % S, nch = a.bn / 16;
          const int mine = r < nch ? (nch - r + S - 1) / S : 0;
          mbar_arrive_expect_tx(&rbar[p], static_cast<uint32_t>(mine * (S - 1)) * 8192u);
        }
      }
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // hardware clusters: publish the receive barriers' init cluster-wide; the epilogue
  // warps wait before their first st.async, the other warps before they exit
  if (c.hw) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  pdl_launch_dependents();

  if (warp == 0 || warp == 6) {
    // producers: warp 0 streams every phase's weights back to back (no waits but
    // ring slots); warp 6 loads a phase's activations once all CTAs finished the
    // previous phase (phase 0: once the previous kernel completed)
    if (elect_one()) {
      const bool wprod = warp == 0;
      const int depth = wprod ? stages : xstages;
      uint64_t* fb = wprod ? full : xfull;
      uint64_t* eb = wprod ? empty : xempty;
      int slot = 0, phase = 0, issued = 0;
      for (int p = 0; p < c.nph; ++p) {
        const GemmArgs& a = c.ph[p];
        const PhaseSched ps = phase_sched(a);
        // per-tile readiness of the producing phase (bf16 chain, p >= 1): K step ks reads
        // rows 128 ks .. 128 ks + 127 of its output = tiles of `rows_per` rows
        const bool tiles_wait = !wprod && p > 0 && c.ready != nullptr;
        const int rows_per = (p > 0 && c.epi[p - 1] == EPI_SWIGLU) ? 64 : kTileM;
        const unsigned writers = p > 0 && c.ph[p - 1].splits > 1 ? static_cast<unsigned>(c.ph[p - 1].splits) : 1u;
        const int ptiles = p > 0 ? c.ph[p - 1].m_tiles : 0;
        int rp = 0;
        if (!wprod) {
          if (p == 0) {
            pdl_wait();
            if (c.qkv_reset != nullptr)  // the previous attention has completed: its counters are free
              for (int t = static_cast<int>(blockIdx.x); t < c.qkv_reset_n; t += G) c.qkv_reset[t] = 0u;
          }
          else if (!tiles_wait) chain_wait_phase(c.bar, G * p);
          SUN_CSTAMP(4 * p);
        }
        const int KS = a.ksteps;
        int ks = ps.n > 0 ? ps.u0 % KS : 0, tile = ps.n > 0 ? ps.u0 / KS : 0;
        for (int j = 0; j < ps.n; ++j) {
          const int nb = min(2, a.kb64 - 2 * ks);
          if (issued >= depth) mbar_wait(&eb[slot], phase ^ 1);
          if (tiles_wait) {
            chain_wait_tiles(c.ready + (p - 1) * kChainReadyTiles, writers,
                             min(ptiles - 1, (kTileM * ks + kTileM - 1) / rows_per), ptiles, rp, c.bar, G * p);
            asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy stores -> bulk copy
          }
          if (wprod) {
            mbar_arrive_expect_tx(&fb[slot], nb * kTileWBytes);
            bulk_load_hint(stg + slot * sb, a.wblk + (static_cast<long long>(tile) * a.kb64 + 2 * ks) * kTileWBytes,
                           nb * kTileWBytes, &fb[slot], kEvictFirst);
          } else {
            mbar_arrive_expect_tx(&fb[slot], nb * a.bn * 128u);
            bulk_load_hint(xstg + slot * xsb, a.xact + static_cast<long long>(2 * ks) * a.bn * 128, nb * a.bn * 128u,
                           &fb[slot], kEvictLast);
          }
          ++issued;
          if (++ks == KS) {
            ks = 0;
            ++tile;
          }
          if (++slot == depth) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: one TMEM double buffer and one pair of rings across all phases
    const uint32_t idesc = make_idesc_bf16(kTileM, bn);
    int wslot = 0, wphase = 0, xslot = 0, xphase = 0, buf = 0, tphase = 0;
    for (int p = 0; p < c.nph; ++p) {
      const GemmArgs& a = c.ph[p];
      const PhaseSched ps = phase_sched(a);
      const int KS = a.ksteps;
      int ks = ps.n > 0 ? ps.u0 % KS : 0;
      for (int j = 0; j < ps.n; ++j) {
        const bool first = j == 0 || ks == 0, last = j == ps.n - 1 || ks == KS - 1;
        const int nb = min(2, a.kb64 - 2 * ks);
        if (first) {
          mbar_wait(&tempty[buf], tphase ^ 1);
          tc_fence_after();
        }
        mbar_wait(&full[wslot], wphase);
        mbar_wait(&xfull[xslot], xphase);
        tc_fence_after();
        if (j == 0 && threadIdx.x == 32) SUN_CSTAMP(4 * p + 1);
        if (j == ps.n - 1 && threadIdx.x == 32) SUN_CSTAMP(4 * p + 2);
        if (elect_one()) {
          const uint32_t xa = smem_u32(xstg + xslot * xsb);
          const uint32_t wa = smem_u32(stg + wslot * sb);
          const uint32_t tacc = tmem_base + static_cast<uint32_t>(buf * bn);
          for (int kk = 0; kk < nb * 4; ++kk) {
            const uint32_t atom = kk >> 2;
            const uint32_t koff = (kk & 3) * 32;
            umma_bf16(tacc, make_sw128_desc(wa + atom * kTileWBytes + koff),
                      make_sw128_desc(xa + atom * (bn * 128u) + koff), idesc, (first && kk == 0) ? 0u : 1u);
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
        if (last && ++buf == 2) {
          buf = 0;
          tphase ^= 1;
        }
      }
    }
  } else if (warp < 6 || warp >= 7) {
    // epilogue groups A (warps 2..5) and B (7..10)
    if (c.hw) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    int buf = 0, tphase = 0;
    for (int p = 0; p < c.nph; ++p) {
      const GemmArgs& a = c.ph[p];
      const PhaseSched ps = phase_sched(a);
      if (p == 0) {
        pdl_wait();
      } else {  // this phase's input, norm statistics and positions are final: one thread polls
        if (threadIdx.x == 64) chain_wait_phase(c.bar, G * p);
        epi_pair_bar();
      }
      unsigned* ready_p = (c.ready != nullptr && p + 1 < c.nph) ? c.ready + p * kChainReadyTiles
                          : (p + 1 == c.nph && c.qkv_ready != nullptr && c.epi[p] == EPI_QKV_ROPE) ? c.qkv_ready
                                                                                                  : nullptr;
      switch (c.epi[p]) {
        case EPI_RESID_ADD: chain_epilogue_phase<EPI_RESID_ADD>(a, ps, epi, tmem_base, tfull, tempty, buf, tphase, recv, &rbar[p], ready_p); break;
        case EPI_SWIGLU: chain_epilogue_phase<EPI_SWIGLU>(a, ps, epi, tmem_base, tfull, tempty, buf, tphase, recv, &rbar[p], ready_p); break;
        case EPI_QKV_ROPE: chain_epilogue_phase<EPI_QKV_ROPE>(a, ps, epi, tmem_base, tfull, tempty, buf, tphase, recv, &rbar[p], ready_p); break;
        default: __trap();  // the layer chain's phases are O / gate_up / down / QKV
      }
      epi_pair_bar();
      if (threadIdx.x == 64) {  // this CTA's outputs of phase p are written
        SUN_CSTAMP(4 * p + 3);
        count_arrive_release(c.bar);
      }
    }
  }
  if (c.hw && !(warp >= 2 && warp < 6) && warp < 7) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, ncols);
  }
  if (c.ready == nullptr) {
    if (threadIdx.x == 0 && atomicAdd(c.bar + 1, 1u) == G - 1) {  // last CTA out rearms the counters
      c.bar[0] = 0u;
      c.bar[1] = 0u;
    }
  } else {
    __shared__ int last_out;
    if (threadIdx.x == 0) last_out = atomicAdd(c.bar + 1, 1u) == G - 1;
    __syncthreads();
    if (last_out) {  // every CTA is past its last read of the tile counters: rearm them too
      for (int p = 0; p + 1 < c.nph; ++p)
        for (int t = threadIdx.x; t < c.ph[p].m_tiles; t += blockDim.x) c.ready[p * kChainReadyTiles + t] = 0u;
      if (threadIdx.x == 0) {
        c.bar[0] = 0u;
        c.bar[1] = 0u;
      }
    }
  }
  tl_end(c.tl, c.tl_idx);
}

// Arrive on the mbarrier at cluster-shared address `remote` (another CTA of the
// cluster), releasing this CTA's prior shared-memory writes at cluster scope.
SUN_DEVICE void mbar_arrive_cluster(uint32_t remote) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
SUN_DEVICE void chain_wait_mbar_cluster(uint64_t* bar, uint32_t parity) {  // acquire at cluster scope
  const unsigned long long t0 = gtimer();
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (gtimer() - t0 > kChainWatchdogNs) __trap();
  }
}

#ifdef SUN_W4_SEG_STAMPS  // probe: O-phase segment epilogue split -> chain stamps [12..15] (overwrites QKV's)
#define SUN_SEGSTAMP(i) \
  do { if (seg_stamps && threadIdx.x == 64) seg_stamps[blockIdx.x * 16 + (i)] = gtimer(); } while (0)
#else
#define SUN_SEGSTAMP(i) do {} while (0)
#endif
template <int EPI>
SUN_DEVICE void w4_chain_segment(const GemmArgs& a, const PhaseSched& ps, int tile, uint32_t taddr, float* epi,
                                 uint64_t* tempty_buf, float* park, uint64_t* pbar,
                                 unsigned long long* seg_stamps = nullptr, const float* pre_res = nullptr,
                                 const float* pre_gain = nullptr) {
  SUN_SEGSTAMP(12);
  const int q = static_cast<int>(threadIdx.x >> 5) & 3;
  const int row_local = q * 32 + (threadIdx.x & 31);
  auto bar = [&]() { epi_bar(); };
  if (ps.S == 1) {
    direct_epilogue<EPI>(a, tile, taddr, epi, 1);
    tc_fence_before();
    bar();
    if (threadIdx.x == 64) mbar_arrive(tempty_buf);
    return;
  }
  const int S = ps.S, rank = ps.rank;
  if (!a.vcluster) {
    // hardware cluster (S = 2 or 4 ranks of the tile in one 4-CTA cluster), pull mode:
    // park the partial in this CTA's idle activation ring (its last MMA of the phase is
    // done; the next phase's activations wait for every CTA's epilogue), tell the S - 1
    // peers, then reduce our chunks reading the peers' partials over DSMEM in rank order
    // (the L2 path's sums). The peers' rings stay untouched until the phase count.
    const int cta0 = static_cast<int>(blockIdx.x & 3u) - rank;  // cluster rank of the tile's rank 0
    {
      float v[16];
      for (int c0 = 0; c0 < a.bn; c0 += 16) {
        tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<float4*>(park + part_index(c0, j, row_local)) =
              make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
    tc_fence_before();
    bar();
    SUN_SEGSTAMP(13);
    if (threadIdx.x == 64) {
      mbar_arrive(tempty_buf);  // accumulator read: the MMA may reuse it
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      for (int r = 0; r < S; ++r)
        if (r != rank) mbar_arrive_cluster(dsmem_addr(pbar, static_cast<uint32_t>(cta0 + r)));
    }
    chain_wait_mbar_cluster(pbar, 0);  // every peer's partial is parked
    SUN_SEGSTAMP(14);
    auto reduce_cols = [&](int c0, int q0, auto& v) {
      constexpr int NQ = sizeof(v) / sizeof(float) / 4;
      float4 x[4][NQ];
      const int cbase = c0 & ~15;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < NQ; ++j)
          x[u][j] = u >= S ? make_float4(0.f, 0.f, 0.f, 0.f)
                           : ld_dsmem_f4(dsmem_addr(park + part_index(cbase, q0 + j, row_local), static_cast<uint32_t>(cta0 + u)));
#pragma unroll
      for (int j = 0; j < 4 * NQ; ++j) v[j] = 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          v[4 * j] += x[u][j].x;
          v[4 * j + 1] += x[u][j].y;
          v[4 * j + 2] += x[u][j].z;
          v[4 * j + 3] += x[u][j].w;
        }
    };
    int k = 0;
    for (int c0 = rank * 16; c0 < a.bn; c0 += S * 16, ++k) {
      float v[16];
      reduce_cols(c0, 0, v);
      if (pre_res != nullptr) {
        asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's own prefetched values
        // chunk k's residual columns: group A's staging area (k = 0) or group B's (k = 1)
        epi_chunk<EPI>(a, tile, row_local, c0, v, epi, pre_res + k * (kEpiGroupBytes / 4), pre_gain, kTileM);
      } else {
        epi_chunk<EPI>(a, tile, row_local, c0, v, epi);
      }
    }
    bar();
    SUN_SEGSTAMP(15);
    return;
  }
  float* part = a.sk_part + static_cast<long long>(blockIdx.x) * a.bn * kTileM;
  {
    float v[16];
    for (int c0 = 0; c0 < a.bn; c0 += 16) {
      tmem_ld16(taddr + c0, v);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        __stcg(reinterpret_cast<float4*>(part + part_index(c0, j, row_local)),
               make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
    }
  }
  __threadfence();
  tc_fence_before();
  bar();
  if (threadIdx.x == 64) mbar_arrive(tempty_buf);  // accumulator parked: the MMA may reuse it
  unsigned* tile_cnt = a.sk_flags + tile;
  if (threadIdx.x == 64) {
    atomicAdd(tile_cnt, 1u);
    const unsigned long long t0 = gtimer();
    while (ld_acquire_u32(tile_cnt) < static_cast<unsigned>(S))
      if (gtimer() - t0 > kChainWatchdogNs) __trap();
  }
  bar();
  const float* gpart = a.sk_part + static_cast<long long>(blockIdx.x - rank) * a.bn * kTileM;
  auto reduce_cols = [&](int c0, int q0, auto& v) {
    constexpr int NQ = sizeof(v) / sizeof(float) / 4;
    float4 x[4][NQ];
#pragma unroll
    for (int j = 0; j < 4 * NQ; ++j) v[j] = 0.f;
    const int cbase = c0 & ~15;
    for (int r0 = 0; r0 < S; r0 += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < NQ; ++j)
          x[u][j] = (r0 + u >= S) ? make_float4(0.f, 0.f, 0.f, 0.f)
                                  : __ldcg(reinterpret_cast<const float4*>(gpart + static_cast<long long>(r0 + u) * a.bn * kTileM +
                                                                           part_index(cbase, q0 + j, row_local)));
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
  for (int c0 = rank * 16; c0 < a.bn; c0 += S * 16) {
    float v[16];
    reduce_cols(c0, 0, v);
    epi_chunk<EPI>(a, tile, row_local, c0, v, epi);
  }
  bar();  // the last of the tile's 2S arrivals rearms its counter
  if (threadIdx.x == 64 && atomicAdd(tile_cnt, 1u) == 2u * S - 1u) *tile_cnt = 0u;
}

SUN_DEVICE void w4_segment(int epi_kind, const GemmArgs& a, const PhaseSched& ps, int tile, uint32_t taddr, float* epi,
                           uint64_t* tempty_buf, float* park, uint64_t* pbar, unsigned long long* seg_stamps,
                           const float* pre_res = nullptr, const float* pre_gain = nullptr) {
  switch (epi_kind) {
    case EPI_RESID_ADD:
      w4_chain_segment<EPI_RESID_ADD>(a, ps, tile, taddr, epi, tempty_buf, park, pbar, seg_stamps, pre_res, pre_gain);
      break;
    case EPI_SWIGLU: w4_chain_segment<EPI_SWIGLU>(a, ps, tile, taddr, epi, tempty_buf, park, pbar); break;
    case EPI_QKV_ROPE: w4_chain_segment<EPI_QKV_ROPE>(a, ps, tile, taddr, epi, tempty_buf, park, pbar); break;
    default: __trap();
  }
}

// QSUN layer chain: the same phases (O -> gate_up -> down -> next QKV) over SUN-W4
// weights, one persistent launch of plain CTAs (one per SM; split phases reduce
// through L2). Warp roles as gemm_kernel<EPI, true>: 0 = weight producer (packed +
// scales stages of wgroup K blocks), 1 = MMA issuer (A from TMEM), 2..5 = epilogue,
// 6..13 = converters (dequantise into the TMEM A ring), 14 = activation producer.
// Every ring (weights, activations, TMEM A tiles, TMEM accumulators) runs across
// the phase boundaries: the converters dequantise the next phase's first weight
// blocks while the epilogue finishes the current phase, so a phase boundary costs
// the grid-wide count and the first activation load, not a launch, a TMEM
// allocation, a ring ramp and the separate kernels' tails.
__global__ void __launch_bounds__(kW4Threads, 1) gemm_chain_w4_kernel(const __grid_constant__ ChainArgs c) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  tl_begin(c.tl, c.tl_idx);
  const GemmArgs& a0 = c.ph[0];
  const int stages = a0.stages, xstages = a0.xstages, bn = a0.bn, wg = a0.wgroup, xk = a0.xk;
  const uint32_t sb = w4_wstage_bytes(wg);
  const uint32_t xsb = w4_xstage_bytes(bn, xk);
  uint8_t* stg = smem;
  uint8_t* xstg = stg + ((stages * sb + 1023u) & ~1023u);
  float* epi = reinterpret_cast<float*>(xstg + xstages * xsb);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(epi) + kEpiSmemBytes);
  uint64_t* empty = full + kMaxWStages;
  uint64_t* xfull = empty + kMaxWStages;
  uint64_t* xempty = xfull + kMaxXStages;
  uint64_t* tfull = xempty + kMaxXStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* dfull = tempty + 2;
  uint64_t* dempty = dfull + kW4MaxABufs;
  uint64_t* pbar = dempty + kW4MaxABufs;  // [kChainMaxPhases] hardware split phases: the peers' partials are parked
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pbar + kChainMaxPhases);
  float* park = reinterpret_cast<float*>(xstg);  // split-K partial, in the activation ring (idle at a phase tail)
  const int warp = warp_id_sync();
  const unsigned G = gridDim.x;
  constexpr int kXProd = 6 + kW4ConvThreads / 32;
  // K blocks per converter / MMA iteration and the TMEM A ring (as gemm_kernel<EPI, true>)
  const int kp = (bn <= 128 && xk % 2 == 0 && wg % 2 == 0) ? 2 : 1;
  const int na = min(kW4MaxABufs, (512 - 2 * bn) / (64 * kp));

  if (warp == 0 && elect_one()) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kW4ConvThreads / 32);
    }
    for (int s = 0; s < xstages; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int j = 0; j < 2; ++j) {
      mbar_init(&tfull[j], 1);
      mbar_init(&tempty[j], 1);
    }
    for (int j = 0; j < kW4MaxABufs; ++j) {
      mbar_init(&dfull[j], kW4ConvThreads / 32);
      mbar_init(&dempty[j], 1);
    }
    for (int p = 0; p < kChainMaxPhases; ++p)  // S - 1 peer arrivals per hardware split phase
      mbar_init(&pbar[p], (p < c.nph && c.ph[p].splits > 1 && !c.ph[p].vcluster) ? c.ph[p].splits - 1 : 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // hardware clusters: publish the parked-partial barriers' init cluster-wide; the
  // epilogue warps wait before their first remote arrive, every other warp before exit
  if (c.hw) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  pdl_launch_dependents();

  if (warp == 0 || warp == kXProd) {
    // producers: warp 0 streams every phase's weight stages back to back (no waits but
    // ring slots); the last warp loads a phase's activations once all CTAs finished the
    // previous phase (phase 0: once the previous kernel completed)
    if (elect_one()) {
      const bool wprod = warp == 0;
      const int grp = wprod ? wg : xk;
      const int depth = wprod ? stages : xstages;
      uint64_t* fb = wprod ? full : xfull;
      uint64_t* eb = wprod ? empty : xempty;
      int slot = 0, phase = 0, issued = 0;
      for (int p = 0; p < c.nph; ++p) {
        const GemmArgs& a = c.ph[p];
        const PhaseSched ps = phase_sched(a);
        if (!wprod) {
          if (p == 0) pdl_wait();
          else chain_wait_phase(c.bar, G * p);
#ifdef SUN_W4_SEG_STAMPS
          if (p < 3)
#endif
          SUN_CSTAMP(4 * p);
        }
        const int KS = a.ksteps;
        int ks = ps.n > 0 ? ps.u0 % KS : 0, seg_left = min(KS - ks, ps.n);
        for (int j = 0; j < ps.n;) {
          const int len = min(grp, seg_left);
          if (issued >= depth) mbar_wait(&eb[slot], phase ^ 1);
          if (wprod) {
            const long long blk = static_cast<long long>(ps.u0 + j);  // = tile * KS + ks
            uint8_t* st = stg + slot * sb;
            mbar_arrive_expect_tx(&fb[slot], static_cast<uint32_t>(len) * (kW4PackedBytes + 256u));
            bulk_load_hint(st, a.w4_packed + blk * kW4PackedBytes, len * kW4PackedBytes, &fb[slot], kEvictFirst);
            bulk_load_hint(st + wg * kW4PackedBytes, a.w4_scales + blk * kTileM, len * 256u, &fb[slot], kEvictFirst);
          } else {
            mbar_arrive_expect_tx(&fb[slot], static_cast<uint32_t>(len) * a.bn * 256u);
            bulk_load_hint(xstg + slot * xsb, a.xact + static_cast<long long>(2 * ks) * a.bn * 128, len * a.bn * 256u,
                           &fb[slot], kEvictLast);
          }
          ++issued;
          j += len;
          ks += len;
          seg_left -= len;
          if (seg_left == 0) {
            ks = 0;
            seg_left = min(KS, ps.n - j);
          }
          if (++slot == depth) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: A (dequantised weights) from the TMEM ring, X from smem; one TMEM
    // accumulator double buffer across all phases
    const uint32_t idesc = make_idesc_bf16(kTileM, bn);
    int xslot = 0, xphase = 0, xpos = 0, aslot = 0, aphase = 0, buf = 0, tphase = 0;
    for (int p = 0; p < c.nph; ++p) {
      const GemmArgs& a = c.ph[p];
      const PhaseSched ps = phase_sched(a);
      const int KS = a.ksteps;
      int ks = ps.n > 0 ? ps.u0 % KS : 0, seg_left = min(KS - ks, ps.n);
      for (int j = 0; j < ps.n;) {
        const int nbk = min(kp, seg_left);
        const bool first = j == 0 || ks == 0, last = seg_left == nbk;
        const bool xlast = xpos + nbk == xk || last;
        if (first) {
          mbar_wait(&tempty[buf], tphase ^ 1);
          tc_fence_after();
        }
        if (xpos == 0) mbar_wait(&xfull[xslot], xphase);
        mbar_wait(&dfull[aslot], aphase);
        tc_fence_after();
#ifdef SUN_W4_SEG_STAMPS
        if (p < 3)
#endif
        if (j == 0 && threadIdx.x == 32) SUN_CSTAMP(4 * p + 1);
        if (elect_one()) {
          const uint32_t xa = smem_u32(xstg + xslot * xsb) + static_cast<uint32_t>(xpos) * 2u * bn * 128u;
          const uint32_t tacc = tmem_base + static_cast<uint32_t>(buf * bn);
          const uint32_t ta = tmem_base + static_cast<uint32_t>(512 - 64 * kp * (aslot + 1));
          for (int b = 0; b < nbk; ++b)
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              umma_bf16_ta(tacc, ta + b * 64 + kk * 8,
                           make_sw128_desc(xa + (2 * b + (kk >> 2)) * (bn * 128u) + (kk & 3) * 32), idesc,
                           (first && b == 0 && kk == 0) ? 0u : 1u);
          umma_commit(&dempty[aslot]);
          if (xlast) umma_commit(&xempty[xslot]);
          if (last) umma_commit(&tfull[buf]);
        }
        __syncwarp();
#ifdef SUN_W4_SEG_STAMPS
        if (p < 3)
#endif
        if (j + nbk == ps.n && threadIdx.x == 32) SUN_CSTAMP(4 * p + 2);
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
          seg_left = min(KS, ps.n - j);
          if (++buf == 2) {
            buf = 0;
            tphase ^= 1;
          }
        }
      }
    }
  } else if (warp < 6) {
    // epilogue (warps 2..5; a second group taken from the converter warps for each
    // phase's last segment measured slower: it delays the next phase's first conversions)
    if (c.hw) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    int buf = 0, tphase = 0;
    for (int p = 0; p < c.nph; ++p) {
      const GemmArgs& a = c.ph[p];
      const PhaseSched ps = phase_sched(a);
      if (p == 0) {
        pdl_wait();
      } else {  // this phase's input, norm statistics and positions are final: one thread polls
        if (threadIdx.x == 64) chain_wait_phase(c.bar, G * p);
        epi_bar();
      }
      switch (c.epi[p]) {
        case EPI_RESID_ADD: load_qkv_meta<EPI_RESID_ADD>(a, epi); break;
        case EPI_SWIGLU: load_qkv_meta<EPI_SWIGLU>(a, epi); break;
        case EPI_QKV_ROPE: load_qkv_meta<EPI_QKV_ROPE>(a, epi); break;
        default: __trap();
      }
      // Residual-phase inputs that do not depend on this phase's result (the previous
      // residual of this rank's columns, the next norm's gain) into both epilogue staging
      // areas with cp.async while the phase's MMAs run (hardware-cluster split phases with
      // up to two 16-column chunks per rank, one segment): the tail reads shared memory
      // instead of paying a global round trip under a saturated HBM.
      const float* pre_res = nullptr;
      float pre_gain = 0.f;
#ifndef SUN_NO_RESPRE  // (A/B build switch)
      if (c.epi[p] == EPI_RESID_ADD && ps.nseg == 1 && ps.S > 1 && !a.vcluster && a.norm_w != nullptr &&
          (a.bn / 16 - ps.rank + ps.S - 1) / ps.S <= 2) {
        const int row_local = (warp & 3) * 32 + (threadIdx.x & 31);
        const int row = ps.t_first * kTileM + row_local;
        float* base = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(epi) + 3072);  // group A | group B staging
        int k = 0;
        for (int c0 = ps.rank * 16; c0 < a.bn; c0 += ps.S * 16, ++k) {
          float* dst = base + k * (kEpiGroupBytes / 4);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (row < a.n_out && c0 + j < a.batch)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst + j * kTileM + row_local)),
                           "l"(a.out_f32 + static_cast<long long>(c0 + j) * a.ldo + row)
                           : "memory");
            else
              dst[j * kTileM + row_local] = 0.f;
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        pre_gain = row < a.n_out ? __bfloat162float(a.norm_w[row]) : 0.f;
        pre_res = base + row_local;
      }
#endif
      for (int seg = 0; seg < ps.nseg; ++seg) {
        mbar_wait(&tfull[buf], tphase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + static_cast<uint32_t>(buf * bn) + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        w4_segment(c.epi[p], a, ps, ps.t_first + seg, taddr, epi, &tempty[buf], park, &pbar[p],
                   p == 0 ? c.stamps : nullptr, pre_res, &pre_gain);
        if (++buf == 2) {
          buf = 0;
          tphase ^= 1;
        }
      }
      epi_bar();
      if (threadIdx.x == 64) {  // this CTA's outputs of phase p are written
#ifdef SUN_W4_SEG_STAMPS
        if (p < 3)
#endif
        SUN_CSTAMP(4 * p + 3);
        count_arrive_release(c.bar);
      }
    }
  } else if (warp < kXProd) {
    // converters: TMEM lane group warp % 4, K part (warp - 6) / 4
    const int lg = warp & 3;
    const int row = lg * 32 + (threadIdx.x & 31);
    const int part = (warp - 6) >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(lg * 32) << 16;
    int wslot = 0, wphase = 0, wpos = 0, aslot = 0, aphase = 0, it = 0;
    for (int p = 0; p < c.nph; ++p) {
      const GemmArgs& a = c.ph[p];
      const PhaseSched ps = phase_sched(a);
      const int KS = a.ksteps;
      int seg_left = min(KS - (ps.n > 0 ? ps.u0 % KS : 0), ps.n);
      for (int j = 0; j < ps.n;) {
        const int nbk = min(kp, seg_left);
        if (wpos == 0) mbar_wait(&full[wslot], wphase);
        const bool wlast = wpos + nbk == wg || seg_left == nbk;
        const uint32_t st = smem_u32(stg + wslot * sb);
        uint32_t o0[16 * kW4Chunks], o1[16 * kW4Chunks];
        w4_dequant_row(st + wpos * kW4PackedBytes, st + wg * kW4PackedBytes + wpos * 256u, row, part, o0);
        if (nbk == 2)
          w4_dequant_row(st + (wpos + 1) * kW4PackedBytes, st + wg * kW4PackedBytes + (wpos + 1) * 256u, row, part, o1);
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
        const uint32_t ta =
            tmem_base + lane_off + static_cast<uint32_t>(512 - 64 * kp * (aslot + 1) + 16 * kW4Chunks * part);
        tmem_st(ta, o0);
        if (nbk == 2) tmem_st(ta + 64, o1);
        tc_fence_before();
        __syncwarp();
        if (elect_one()) mbar_arrive(&dfull[aslot]);
        if (++aslot == na) {
          aslot = 0;
          aphase ^= 1;
        }
        ++it;
        j += nbk;
        seg_left -= nbk;
        if (seg_left == 0) seg_left = min(KS, ps.n - j);
      }
    }
  }
  if (c.hw) {  // nobody exits while a peer may still read its parked partial
    if (!(warp >= 2 && warp < 6)) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
  if (threadIdx.x == 0 && atomicAdd(c.bar + 1, 1u) == G - 1) {  // last CTA out rearms the counters
    c.bar[0] = 0u;
    c.bar[1] = 0u;
  }
  tl_end(c.tl, c.tl_idx);
}

}  // namespace sun
