// sun_capi.cu — C ABI + native step orchestration of the SUN shared decode path.
//
// One translation unit: the kernels (gemm_tc.cuh, gemm_w4.cuh, attention.cuh,
// elementwise.cuh) plus the host runtime that encodes TMA descriptors, carves
// the caller-owned workspace, plans split-K / attention splits and launches the
// per-layer kernel chain of a decode step (optionally with programmatic
// dependent launch so each kernel's prologue and weight prefetch overlap the
// previous kernel's tail). Declared in include/sun_b200.h.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sun_b200.h"
#include "attention.cuh"
#include "elementwise.cuh"
#include "gemm_tc.cuh"
#include "gemm_w4.cuh"
#include "gemm_chain.cuh"

using namespace sun;

namespace {

thread_local std::string g_last_error;

SunStatus fail(SunStatus st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define SUN_CUDA(expr)                                                                 \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail(SUN_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                 \
  } while (0)

// ---------------------------------------------------------------------------
// TMA descriptor encoding through the driver entry point (no -lcuda needed)
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}

typedef CUresult (*PFN_getAddressRange_t)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_getAddressRange_t address_range_fn() {  // allocation containing a device pointer (IPC export / close)
  static PFN_getAddressRange_t fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
               ? reinterpret_cast<PFN_getAddressRange_t>(p)
               : nullptr;
  }();
  return fn;
}

// 2-D bf16 [rows][cols] (row stride ld elements), box {64 cols, box_rows}, SW128.
SunStatus make_map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                      uint32_t box_rows, CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  auto fn = encode_fn();
  if (!fn) return fail(SUN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((ld * 2) % 16 != 0) return fail(SUN_ERR_UNSUPPORTED, "row stride %llu not 16B aligned", (unsigned long long)ld);
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SUN_ERR_CUDA, "cuTensorMapEncodeTiled(2d) -> %d", (int)r);
  return SUN_OK;
}

// 3-D view of the KV pool: {head_dim, rows_per_page, num_pages}, box {64, 16, 1}.
SunStatus make_map_kv(CUtensorMap* m, const SunDecoderDims& d, const SunKvPool& kv) {
  auto fn = encode_fn();
  if (!fn) return fail(SUN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const uint64_t rows_per_page = uint64_t(d.n_layers) * 2 * d.n_kv_heads * d.page_size;
  cuuint64_t dims[3] = {uint64_t(d.head_dim), rows_per_page, uint64_t(kv.num_pages)};
  cuuint64_t strides[2] = {uint64_t(d.head_dim) * 2, rows_per_page * d.head_dim * 2};
  cuuint32_t box[3] = {64, uint32_t(kPageTokens), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, kv.base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SUN_ERR_CUDA, "cuTensorMapEncodeTiled(kv) -> %d", (int)r);
  return SUN_OK;
}

// ---------------------------------------------------------------------------
// planning
// ---------------------------------------------------------------------------
constexpr int kNumSms = 148;

struct GemmPlan {
  int m_tiles, kb64, ksteps;
};

GemmPlan plan_gemm(int64_t n_out, int64_t k) {
  GemmPlan p;
  p.m_tiles = int((n_out + kTileM - 1) / kTileM);
  p.kb64 = int((k + kTileK - 1) / kTileK);
  p.ksteps = (p.kb64 + 1) / 2;
  return p;
}

constexpr int kSmemPerSm = 226 * 1024;  // usable dynamic smem per SM (227 KB minus reserve)

// CTAs per SM for a GEMM. 1 (deep pipeline, ~200 KB smem) measured faster than
// 2 x ~108 KB on B200 for C3 (5.62 vs 5.83 ms/step); SUN_GEMM_CTAS_PER_SM=2
// selects the two-CTA variant (needs two double-buffered TMEM accumulators).
int gemm_ctas_per_sm(int bn, bool w4) {
  static int forced = [] {
    const char* e = getenv("SUN_GEMM_CTAS_PER_SM");
    return e ? atoi(e) : 1;
  }();
  if (forced == 2 && !w4 && 2 * tmem_cols_for(bn) <= 512) return 2;
  return 1;
}

// Optional grid cap (SUN_GEMM_MAX_GRID): with 2-per-SM smem budgets and a
// 148-CTA grid, the next kernel's CTAs can be co-resident (PDL prefetch).
int gemm_max_grid() {
  static int v = [] {
    const char* e = getenv("SUN_GEMM_MAX_GRID");
    return e ? atoi(e) : 1 << 30;
  }();
  return v;
}

// bf16 ring depths: 3 activation stages (2 at bn > 128), weight stages (32 KB)
// fill the rest of the SM's shared memory (C3, bn = 64: 5 weight stages).
int gemm_xstages(int bn) {
  static const int env = [] { const char* e = getenv("SUN_GEMM_XSTAGES"); return e ? atoi(e) : 0; }();
  return env > 0 ? env : (bn > 128 ? 2 : 3);
}
int gemm_stages(int bn, bool w4, int per_sm) {
  const int budget = kSmemPerSm / per_sm - 2048 - 2048 - int(kEpiSmemBytes) - 1024 -
                     gemm_xstages(bn) * int(gemm_xstage_bytes(bn));
  const int st = budget / int(gemm_stage_bytes(bn, w4));
  return std::max(2, std::min(8, st));
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int round16(int b) { return (b + 15) / 16 * 16; }

template <typename K>
void set_max_smem(K kern) {
  cudaFuncAttributes fa;
  size_t static_bytes = 0;
  if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) static_bytes = fa.sharedSizeBytes;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(227 * 1024 - static_bytes)) !=
      cudaSuccess) {
    fprintf(stderr, "sun_b200: cudaFuncSetAttribute(max dynamic smem) failed\n");
    cudaGetLastError();
  }
}

std::once_flag g_attr_once;
void init_kernel_attrs() {
  std::call_once(g_attr_once, [] {
    set_max_smem(gemm_kernel<EPI_STORE_F32, false>);
    set_max_smem(gemm_kernel<EPI_RESID_ADD, false>);
    set_max_smem(gemm_kernel<EPI_QKV_ROPE, false>);
    set_max_smem(gemm_kernel<EPI_SWIGLU, false>);
    set_max_smem(gemm_kernel<EPI_LOGITS, false>);
    set_max_smem(gemm_kernel<EPI_STORE_F32, true>);
    set_max_smem(gemm_kernel<EPI_RESID_ADD, true>);
    set_max_smem(gemm_kernel<EPI_QKV_ROPE, true>);
    set_max_smem(gemm_kernel<EPI_SWIGLU, true>);
    set_max_smem(gemv_w4_kernel<EPI_STORE_F32, 1>);
    set_max_smem(gemv_w4_kernel<EPI_STORE_F32, 2>);
    set_max_smem(gemv_w4_kernel<EPI_RESID_ADD, 1>);
    set_max_smem(gemv_w4_kernel<EPI_RESID_ADD, 2>);
    set_max_smem(gemv_w4_kernel<EPI_QKV_ROPE, 1>);
    set_max_smem(gemv_w4_kernel<EPI_QKV_ROPE, 2>);
    set_max_smem(gemv_w4_kernel<EPI_SWIGLU, 1>);
    set_max_smem(gemv_w4_kernel<EPI_SWIGLU, 2>);
    set_max_smem(gemv_w4a_kernel<EPI_STORE_F32, 1>);
    set_max_smem(gemv_w4a_kernel<EPI_STORE_F32, 2>);
    set_max_smem(gemv_w4a_kernel<EPI_RESID_ADD, 1>);
    set_max_smem(gemv_w4a_kernel<EPI_RESID_ADD, 2>);
    set_max_smem(gemv_w4a_kernel<EPI_QKV_ROPE, 1>);
    set_max_smem(gemv_w4a_kernel<EPI_QKV_ROPE, 2>);
    set_max_smem(gemv_w4a_kernel<EPI_SWIGLU, 1>);
    set_max_smem(gemv_w4a_kernel<EPI_SWIGLU, 2>);
    set_max_smem(gemv_chain_w4_kernel<1>);
    set_max_smem(gemv_chain_w4_kernel<2>);
    set_max_smem(gemm_chain_kernel);
    set_max_smem(gemm_chain_w4_kernel);
    set_max_smem(attn_group_kernel<64>);
    set_max_smem(attn_group_kernel<128>);
    set_max_smem(attn_decode_kernel<64>);
    set_max_smem(attn_decode_kernel<128>);
    (void)0;
  });
}

thread_local unsigned g_cluster = 1;  // cluster size for the next launch_raw (1 = none)

template <typename... KArgs, typename... Args>
cudaError_t launch_raw(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (g_cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = g_cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  g_cluster = 1;
  return e;
}

// How many clusters of `size` CTAs (each `smem` bytes, 1 per SM) can be co-resident.
int max_active_clusters(unsigned size, size_t smem, bool w4) {
  static std::map<std::pair<unsigned, size_t>, int> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(size * 2 + (w4 ? 1u : 0u), smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(size * 16);
  cfg.blockDim = dim3(w4 ? kW4Threads : kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = size;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  const cudaError_t e = w4 ? cudaOccupancyMaxActiveClusters(&n, gemm_kernel<EPI_STORE_F32, true>, &cfg)
                           : cudaOccupancyMaxActiveClusters(&n, gemm_kernel<EPI_STORE_F32, false>, &cfg);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = size == 1 ? kNumSms : 0;
  }
  cache[key] = n;
  return n;
}

// Per-thread launch accounting + optional per-kernel event timing (profile mode).
struct LaunchTrace {
  long long launches = 0;
  std::vector<cudaEvent_t>* events = nullptr;  // record one event after each launch
};
thread_local LaunchTrace g_trace;

// Step timeline (sun_decode_step_timeline): device slot array + next launch index.
struct TimelineState {
  unsigned long long* tl = nullptr;
  int next = 0, capacity = 0;
  unsigned long long* stamps = nullptr;  // per-CTA phase stamps for launch `stamp_idx` (GEMMs)
  int stamp_idx = -1;
};
thread_local TimelineState g_tl;
template <typename A>
void tl_assign(A& a) {
  if (g_tl.tl != nullptr && g_tl.next < g_tl.capacity) {
    a.tl = g_tl.tl;
    a.tl_idx = g_tl.next++;
  }
}
void tl_stamps(GemmArgs& a) {
  if (g_tl.stamps != nullptr && a.tl != nullptr && a.tl_idx == g_tl.stamp_idx) a.stamps = g_tl.stamps;
}

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                   Args&&... args) {
  cudaError_t e = launch_raw(kern, grid, block, smem, st, pdl, std::forward<Args>(args)...);
  if (e == cudaSuccess) {
    ++g_trace.launches;
    if (g_trace.events) {
      cudaEvent_t ev;
      e = cudaEventCreate(&ev);
      if (e == cudaSuccess) {
        g_trace.events->push_back(ev);
        e = cudaEventRecord(ev, st);
      }
    }
  }
  return e;
}

// Stream-K GEMM scratch: one fp32 [bn][128] partial and one flag per CTA slot.
constexpr int kMaxGemmCtas = 2 * kNumSms;
size_t sk_part_bytes(int bn) { return size_t(kMaxGemmCtas) * size_t(bn) * kTileM * 4; }
// Small-batch W4 GEMV scratch: two 128 x 16 fp32 partial slots per CTA, one counter per tile.
constexpr int kGvMaxTiles = 4096;
size_t gv_part_bytes() { return size_t(kMaxGemmCtas) * 2 * kTileM * 16 * 4; }
constexpr int kGemvKernelMaxBatch = 16;  // gemv_w4_kernel: one or two 8-column MMA tiles
constexpr int kGemvMaxBatch = 8;  // decode steps use it up to 8 rows: at 9..16 the W4 chain measured faster (B=16 2.65 vs 2.82 ms)

// GEMM schedule. 0 (default): cluster split-K for <= 148 tiles, whole tiles
// otherwise. 1: stream-K for GEMMs with more tiles than SMs (even split of
// tiles x k-steps; measured 37.4 vs 40.4 us for the 8B gate_up alone, but the
// step got slower — with whole tiles the CTAs holding one tile finish early and
// the next kernel's CTAs start prefetching under PDL). 2: stream-K everywhere
// it fits (tests).
int gemm_sched() {
  static int v = [] {
    const char* e = getenv("SUN_GEMM_SCHED");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// Workspace layout shared by sizing and creation.
struct WsLayout {
  size_t resid, xn, q, attn, act, part_o, part_ml, attn_cnt, ss, amax_val, amax_idx, logits, sk_part, sk_flags,
      chain_bar, err, gv_part, gv_cnt, qkv_ready, total;
  int max_splits;
};

int d_cnt_heads(const SunDecoderDims& d) { return d.n_kv_heads; }
int gu_rows(const SunDecoderDims& d) { return (d.ffn + 63) / 64 * 128; }
int qkv_rows(const SunDecoderDims& d) { return (d.n_q_heads + 2 * d.n_kv_heads) * d.head_dim; }

WsLayout layout_ws(const SunDecoderDims& d, int max_batch) {
  WsLayout w{};
  const int bmp = round16(max_batch);
  const int qd = d.n_q_heads * d.head_dim;
  const int max_pages = (d.max_context + kPageTokens - 1) / kPageTokens;
  w.max_splits = max_pages;  // pages_per_split >= 1
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 1024);
    return o;
  };
  auto act_bytes = [&](int k) { return size_t(bmp) * size_t((k + 63) / 64) * 128; };  // SUN-ACT, padded K
  w.resid = take(size_t(max_batch) * d.hidden * 4);
  w.xn = take(act_bytes(d.hidden));
  w.q = take(size_t(max_batch) * qd * 2);
  w.attn = take(act_bytes(qd));
  w.act = take(act_bytes(d.ffn));
  w.part_o = take(size_t(max_batch) * d.n_q_heads * w.max_splits * d.head_dim * 4);
  w.part_ml = take(size_t(max_batch) * d.n_q_heads * w.max_splits * 2 * 4);
  w.attn_cnt = take(size_t(max_batch) * d.n_kv_heads * 4);
  w.ss = take(size_t((d.hidden + kTileM - 1) / kTileM) * bmp * 4);
  const int lm_tiles = (d.vocab + kTileM - 1) / kTileM;
  w.amax_val = take(size_t(lm_tiles) * bmp * 4);
  w.amax_idx = take(size_t(lm_tiles) * bmp * 4);
  w.logits = take(size_t(max_batch) * d.vocab * 4);
  w.sk_part = take(sk_part_bytes(bmp));
  w.sk_flags = take(kMaxGemmCtas * 4);
  w.chain_bar = take(64 + size_t(kChainMaxPhases) * kChainReadyTiles * 4);  // phase counts | per-tile readiness
  w.err = take(64);
  w.gv_part = take(gv_part_bytes());
  w.gv_cnt = take(kGvMaxTiles * 4);
  w.qkv_ready = take(size_t(d.n_layers) * kQkvReadyStride * 4);
  w.total = off;
  return w;
}

SunStatus check_dims(const SunDecoderDims* d) {
  if (!d) return fail(SUN_ERR_VALUE, "null dims");
  if (d->vocab < 1 || d->hidden < 1 || d->n_layers < 1 || d->n_q_heads < 1 || d->n_kv_heads < 1 || d->ffn < 1)
    return fail(SUN_ERR_VALUE, "non-positive decoder dimension");
  if (d->head_dim != 64 && d->head_dim != 128) return fail(SUN_ERR_UNSUPPORTED, "head_dim %d not in {64,128}", d->head_dim);
  if (d->page_size != kPageTokens) return fail(SUN_ERR_UNSUPPORTED, "page_size must be %d", kPageTokens);
  if (d->n_q_heads % d->n_kv_heads != 0 || d->n_q_heads / d->n_kv_heads > 8)
    return fail(SUN_ERR_UNSUPPORTED, "GQA group must divide and be <= 8");
  if (d->hidden % 64 != 0) return fail(SUN_ERR_UNSUPPORTED, "hidden must be a multiple of 64");
  if (d->ffn % 8 != 0) return fail(SUN_ERR_UNSUPPORTED, "ffn must be a multiple of 8");
  if (d->weight_bits != 16 && d->weight_bits != 4) return fail(SUN_ERR_VALUE, "weight_bits must be 16 or 4");
  if (d->weight_bits == 4) {
    if (d->group_size != 128) return fail(SUN_ERR_UNSUPPORTED, "W4 group_size must be 128");
    if (d->hidden % 128 || (d->n_q_heads * d->head_dim) % 128 || d->ffn % 128)
      return fail(SUN_ERR_UNSUPPORTED, "W4 needs K dims multiple of 128");
  }
  if (d->max_context < 1) return fail(SUN_ERR_VALUE, "max_context must be >= 1");
  return SUN_OK;
}

// The shared-decoder invariant at the device boundary: a decoder (shared decode
// module or task prefill module) only reads / writes a pool laid out for its KV
// geometry (domain.py:266-279 shared models agree on the decoder; costmodel.py:132-138).
SunStatus check_kv_geometry(const SunDecoderDims& d, const SunKvPool& kv) {
  if (kv.n_layers != d.n_layers || kv.n_kv_heads != d.n_kv_heads || kv.head_dim != d.head_dim ||
      kv.page_size != d.page_size || kv.rope_theta != d.rope_theta)
    return fail(SUN_ERR_MIXED_DECODER,
                "KV pool geometry (layers %d, kv heads %d, head_dim %d, page %d, rope theta %g) does not match the "
                "decoder's (%d, %d, %d, %d, %g)",
                kv.n_layers, kv.n_kv_heads, kv.head_dim, kv.page_size, (double)kv.rope_theta, d.n_layers,
                d.n_kv_heads, d.head_dim, d.page_size, (double)d.rope_theta);
  if (kv.num_pages < 1 || kv.base == nullptr) return fail(SUN_ERR_VALUE, "empty KV pool");
  return SUN_OK;
}

size_t kv_page_bytes(const SunKvPool& kv) {
  return size_t(kv.n_layers) * 2 * kv.n_kv_heads * kv.page_size * kv.head_dim * 2;
}

int device_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return kNumSms;
  }
  return n;
}

}  // namespace

struct SunDecoder {
  SunDecoderDims d;
  int max_batch = 0, bmp = 0;
  bool pdl = false;
  std::vector<SunLayerWeights> layers;
  SunWeights w;
  SunKvPool kv;
  long long page_stride = 0;
  CUtensorMap tm_kv;
  WsLayout L;
  uint8_t* ws = nullptr;
  float* resid;
  __nv_bfloat16 *xn, *q, *attn, *act;  // xn / attn / act in SUN-ACT (GEMM operands)
  float *part_o, *part_ml, *amax_val, *logits;
  unsigned* attn_cnt;
  float* ss;  // [h/128][bn] per-tile sums of squares of the residual (factored RMSNorm)
  int* amax_idx;
  float* sk_part;
  unsigned* sk_flags;
  unsigned* chain_bar;
  unsigned* qkv_ready;  // [layer][kQkvReadyStride] QKV tiles written by the previous layer's chain
  unsigned* err;  // SUN_STEP_ERR_* bits (sun_decoder_status)
  float* gv_part;     // small-batch W4 GEMV partials / per-tile counters
  unsigned* gv_cnt;
  int num_sms = kNumSms;
  bool chain_ok = false;     // the layer chain's grid fits this device co-resident (chain_fits)
  bool chain_w4_ok = false;  // same for the QSUN chain (chain_w4_fits)
  GemmPlan p_qkv, p_o, p_gu, p_down, p_lm;
};

namespace {

GemmArgs base_args(const GemmPlan& p, int64_t n_out, int64_t k, int batch, int bn, const void* xact,
                   float* sk_part = nullptr, unsigned* sk_flags = nullptr) {
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.sk_part = sk_part;
  a.sk_flags = sk_flags;
  a.n_out = int(n_out);
  a.k = int(k);
  a.batch = batch;
  a.bn = bn;
  a.kb64 = p.kb64;
  a.ksteps = p.ksteps;
  a.m_tiles = p.m_tiles;
  a.xact = static_cast<const uint8_t*>(xact);
  return a;
}

// Cluster split factor for a GEMM with <= 148 tiles: the largest S <= 8 (and
// <= k-steps) whose m_tiles clusters of S CTAs are co-resident in one wave.
int cluster_splits(const GemmPlan& p, size_t smem, bool w4, int slots) {
  if (p.m_tiles > slots) return 1;
  int s = std::min(std::min(8, slots / std::max(1, p.m_tiles)), p.ksteps);
  while (s > 1 && max_active_clusters(unsigned(s), smem, w4) < p.m_tiles) --s;
  return std::max(1, s);
}

// Launch one GEMM: bf16 SUN-BLK weights (wblk) or QSUN SUN-W4 (packed, scales).
// Launch configuration of one GEMM (also used to aim the previous GEMM's L2
// prefetch at the CTAs that will start streaming first).
struct LaunchCfg {
  int grid, splits, vcluster, sk_units, stages, xstages, wgroup, xk, push;
  size_t smem;
};

// Push-mode split-K reduction (SUN_GEMM_PUSH=1, default off): hardware-cluster ranks
// bulk-copy the chunks their peers reduce into the peers' receive areas (DSMEM,
// completion on the owner's mbarrier) instead of the owners pulling them after a
// cluster barrier; no cluster barrier at the end either. Used when the receive
// area fits next to the ring. Measured neutral on C3 (5.055 vs 5.061 ms/step) and
// C4 (14.76 vs 14.73): the tail is the slowest rank and the epilogue's stores,
// not the barrier.
int gemm_push() {
  static int v = [] {
    const char* e = getenv("SUN_GEMM_PUSH");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// Virtual clusters (SUN_GEMM_VCLUSTER, default on): when the hardware cannot
// co-schedule enough S-CTA clusters (QKV: 48 tiles want S = 3 -> 144 CTAs, but
// 3-CTA clusters do not pack the GPCs), split K over S plain CTAs that reduce
// through L2 instead of DSMEM.
int gemm_vcluster() {
  static int v = [] {
    const char* e = getenv("SUN_GEMM_VCLUSTER");
    return e ? atoi(e) : 1;
  }();
  return v;
}

LaunchCfg launch_cfg(const GemmPlan& p, int bn, bool w4, bool have_sk) {
  LaunchCfg c{};
  const int per_sm = gemm_ctas_per_sm(bn, w4);
  const int slots = std::min(kNumSms * per_sm, gemm_max_grid());
  size_t ring;
  if (w4) {
    // weight stages of wgroup K blocks (one packed + one scales request each),
    // activation stages of xk K blocks; 3 activation stages, weights fill the rest
    static const int env_wg = [] { const char* e = getenv("SUN_W4_WGROUP"); return e ? atoi(e) : 0; }();
    static const int env_xk = [] { const char* e = getenv("SUN_W4_XK"); return e ? atoi(e) : 0; }();
    static const int env_xs = [] { const char* e = getenv("SUN_W4_XSTAGES"); return e ? atoi(e) : 0; }();
    c.wgroup = env_wg > 0 ? env_wg : 4;
    // K-block pairs per converter / MMA iteration need activation stages of an even
    // number of blocks when bn <= 128 (gemm_tc.cuh `kp`)
    c.xk = env_xk > 0 ? env_xk : (bn <= 32 ? 4 : (bn <= 128 ? 2 : 1));
    c.xstages = env_xs > 0 ? env_xs : (bn > 64 ? 2 : 3);
    const int budget = kSmemPerSm - 2048 - 2048 - int(kEpiSmemBytes) - 1024 - c.xstages * int(w4_xstage_bytes(bn, c.xk));
    c.stages = std::max(2, std::min(16, budget / int(w4_wstage_bytes(c.wgroup))));
    c.smem = gemm_smem_bytes_w4(bn, c.wgroup, c.stages, c.xk, c.xstages);
    ring = size_t(c.stages) * w4_wstage_bytes(c.wgroup) + size_t(c.xstages) * w4_xstage_bytes(bn, c.xk);
  } else {
    c.stages = gemm_stages(bn, w4, per_sm);
    c.xstages = gemm_xstages(bn);
    c.smem = gemm_smem_bytes(bn, c.stages, c.xstages);
    ring = size_t(c.stages) * gemm_stage_bytes(bn, w4) + size_t(c.xstages) * gemm_xstage_bytes(bn);
  }
  // Stream-K where whole tiles cannot balance over the SMs (more tiles than CTA
  // slots, e.g. gate_up 224 tiles / 148 SMs = 1.51) and every owner's
  // contributor partials fit in its stage ring; cluster split-K (<= slots
  // tiles) or whole tiles otherwise.
  const int units = p.m_tiles * p.ksteps;
  const int sk_grid = std::min(units, std::min(slots, kMaxGemmCtas));
  const int max_contrib = (p.ksteps + (units / sk_grid) - 1) / std::max(1, units / sk_grid) + 1;
  // (SUN_GEMM_SCHED=2 forces stream-K on every GEMM whose partials fit: tests)
  const bool sk = gemm_sched() != 0 && have_sk &&
                  (gemm_sched() == 2 || (p.m_tiles > slots && p.m_tiles % sk_grid != 0)) &&
                  size_t(max_contrib) * bn * kTileM * 4 <= ring;
  if (sk) {
    c.splits = 1;
    c.sk_units = units;
    c.grid = sk_grid;
  } else {
    c.splits = cluster_splits(p, c.smem, w4, slots);
    c.sk_units = 0;
    c.vcluster = 0;
    const int want = p.m_tiles <= slots ? std::min(std::min(8, slots / std::max(1, p.m_tiles)), p.ksteps) : 1;
    // (SUN_GEMM_VCLUSTER=2 uses virtual clusters wherever a split pays: tests)
    if (gemm_vcluster() && have_sk && (want > c.splits || (gemm_vcluster() == 2 && want > 1)) &&
        p.m_tiles * want <= kMaxGemmCtas) {
      c.splits = want;
      c.vcluster = 1;
    }
    c.grid = c.splits > 1 ? p.m_tiles * c.splits : std::min(p.m_tiles, slots);
    if (c.splits > 1 && !c.vcluster && gemm_push()) {
      const int nch = bn / 16, nmax = (nch + c.splits - 1) / c.splits;
      const size_t recv = size_t(c.splits - 1) * nmax * 8192;
      if (c.smem + recv <= size_t(kSmemPerSm) / per_sm) {
        c.push = int(recv);
        c.smem += recv;
      }
    }
  }
  return c;
}

// L2 prefetch budget per next-GEMM CTA (SUN_GEMM_PREFETCH_KB). Default off:
// measured on C3 (8B bf16, B=64) 5.375 ms/step without, 5.347 at 64 KB, 5.47 at
// 128 KB, 5.75 at 512 KB; C4 unchanged — the HBM is not idle enough between
// GEMMs for a prefetch to pay, and larger ones compete with the live stream.
int gemm_prefetch_bytes() {
  static int v = [] {
    const char* e = getenv("SUN_GEMM_PREFETCH_KB");
    return (e ? atoi(e) : 0) * 1024;
  }();
  return v;
}

// Aim this GEMM's tail-time L2 prefetch at the first weight stages of `next`.
void set_prefetch(GemmArgs& a, const void* next_w, const GemmPlan& np, int bn, bool w4) {
  const int bytes = gemm_prefetch_bytes();
  if (!next_w || bytes <= 0) return;
  const LaunchCfg c = launch_cfg(np, bn, w4, a.sk_part != nullptr && a.sk_flags != nullptr);
  a.pf_w = static_cast<const uint8_t*>(next_w);
  a.pf_w4 = w4 ? 1 : 0;
  a.pf_m_tiles = np.m_tiles;
  a.pf_ksteps = np.ksteps;
  a.pf_kb64 = np.kb64;
  a.pf_splits = c.splits;
  a.pf_grid = c.grid;
  a.pf_sk_units = c.sk_units;
  a.pf_bytes = bytes;
}

template <int EPI>
SunStatus run_gemm(const void* wblk, const void* packed, const void* scales, GemmArgs a, const GemmPlan& p,
                   cudaStream_t st, bool pdl) {
  const bool w4 = packed != nullptr;
  a.wblk = static_cast<const uint8_t*>(wblk);
  a.w4_packed = static_cast<const uint8_t*>(packed);
  a.w4_scales = static_cast<const __nv_bfloat16*>(scales);
  const LaunchCfg c = launch_cfg(p, a.bn, w4, a.sk_part != nullptr && a.sk_flags != nullptr);
  a.stages = c.stages;
  a.xstages = c.xstages;
  a.wgroup = c.wgroup;
  a.xk = c.xk;
  tl_assign(a);
  tl_stamps(a);
  a.splits = c.splits;
  a.vcluster = c.vcluster;
  a.sk_units = c.sk_units;
  a.push_bytes = c.push;
  g_cluster = c.vcluster ? 1u : unsigned(c.splits);
  if (w4) {
    if constexpr (EPI == EPI_LOGITS) return fail(SUN_ERR_UNSUPPORTED, "lm_head is bf16");
    else SUN_CUDA(launch(gemm_kernel<EPI, true>, dim3(c.grid), dim3(kW4Threads), c.smem, st, pdl, a));
  } else {
    SUN_CUDA(launch(gemm_kernel<EPI, false>, dim3(c.grid), dim3(kGemmThreads), c.smem, st, pdl, a));
  }
  return SUN_OK;
}

// Small-batch QSUN GEMV (gemv_w4_kernel, gemm_w4.cuh) for decode batches of <= 8
// rows (kernel: <= 16): one CTA per SM (SUN_GV_CTAS_PER_SM), whole tiles or split-K per tile, a ring of
// SUN_GV_STAGES stages of SUN_GV_KBS K blocks. SUN_W4_GEMV=0 keeps the tcgen05 path.
struct GvCfg {
  int kbs, stages, per_sm;
  size_t smem;
};
int gv_async_epi() {  // SUN_GV_ASYNC_EPI (default 1): the kernel with a dedicated epilogue group
  static const int v = [] { const char* e = getenv("SUN_GV_ASYNC_EPI"); return e ? atoi(e) : 1; }();
  return v;
}
GvCfg gv_cfg(int bn, bool async = false) {
  static const int env_kbs = [] { const char* e = getenv("SUN_GV_KBS"); return e ? atoi(e) : 0; }();
  static const int env_st = [] { const char* e = getenv("SUN_GV_STAGES"); return e ? atoi(e) : 0; }();
  static const int env_ps = [] { const char* e = getenv("SUN_GV_CTAS_PER_SM"); return e ? atoi(e) : 0; }();
  GvCfg c{};
  c.kbs = env_kbs > 0 ? env_kbs : 4;
  c.per_sm = env_ps > 0 ? env_ps : 1;
  const int budget = kSmemPerSm / c.per_sm - int(gv_smem_bytes(bn, c.kbs, 0)) - 1024;
  c.stages = std::max(2, std::min(kGvMaxStages, budget / int(gv_stage_bytes(bn, c.kbs))));
  // gemv_w4a_kernel: a 3-stage ring (12 K blocks in flight; 2 / 3 / 4 stages 2.33 / 2.34 /
  // 2.39 ms before the tail changes, 3 vs 2 after them: B=1 2.130 vs 2.133, B=8 2.232 vs
  // 2.246 ms same box — profiles/r02/gv_async_stages.txt)
  if (async) c.stages = std::min(c.stages, 3);
  if (env_st > 0) c.stages = std::min(env_st, kGvMaxStages);
  c.smem = gv_smem_bytes(bn, c.kbs, c.stages);
  return c;
}
int max_active_clusters_gv(unsigned size, size_t smem) {
  static std::map<std::pair<unsigned, size_t>, int> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(size, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(size * 16);
  cfg.blockDim = dim3(kGvThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = size;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemv_w4_kernel<EPI_STORE_F32, 1>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[key] = n;
  return n;
}

bool use_gemv(bool w4, int batch) {
  static const int v = [] { const char* e = getenv("SUN_W4_GEMV"); return e ? atoi(e) : 1; }();
  static const int mb = [] {  // SUN_GV_MAX_BATCH: largest decode batch on the GEMV (kernel: <= 16)
    const char* e = getenv("SUN_GV_MAX_BATCH");
    return e ? std::max(1, std::min(atoi(e), kGemvKernelMaxBatch)) : kGemvMaxBatch;
  }();
  return w4 && v != 0 && batch <= mb;
}

// L2 prefetch budget per next-GEMV CTA (SUN_GV_PREFETCH_KB, default 0: 32-128 KB measured
// neutral on the 8B W4 B=1 / B=8 steps) and its target: the next W4 GEMV of the step (its
// schedule as run_gemv_w4 will launch it).
int gv_prefetch_bytes() {
  static const int v = [] { const char* e = getenv("SUN_GV_PREFETCH_KB"); return (e ? atoi(e) : 0) * 1024; }();
  return v;
}
void gv_set_prefetch(GemmArgs& a, const void* next_packed, const GemmPlan& np, int num_sms) {
  const int bytes = gv_prefetch_bytes();
  if (!next_packed || bytes <= 0) return;
  const GvCfg c = gv_cfg(a.bn);
  const int slots = std::min(num_sms * c.per_sm, kMaxGemmCtas);
  a.pf_w = static_cast<const uint8_t*>(next_packed);
  a.pf_w4 = 1;
  a.pf_m_tiles = np.m_tiles;
  a.pf_ksteps = np.ksteps;
  a.pf_kb64 = np.kb64;
  a.pf_sk_units = 0;
  if (np.m_tiles >= slots) {
    a.pf_splits = 0;
    a.pf_grid = slots;
  } else {
    a.pf_splits = std::max(1, std::min(np.ksteps, slots / np.m_tiles));
    a.pf_grid = np.m_tiles * a.pf_splits;
  }
  a.pf_bytes = bytes;
}

template <int EPI>
SunStatus run_gemv_w4(const void* packed, const void* scales, GemmArgs a, const GemmPlan& p, float* part,
                      unsigned* cnt, cudaStream_t st, bool pdl, int num_sms) {
  if (a.bn != 16 || a.batch > kGemvKernelMaxBatch) return fail(SUN_ERR_VALUE, "W4 GEMV takes batches of <= 16 rows");
  if (p.m_tiles > kGvMaxTiles) return fail(SUN_ERR_UNSUPPORTED, "W4 GEMV: %d tiles > %d", p.m_tiles, kGvMaxTiles);
  static const int cl_env = [] { const char* e = getenv("SUN_GV_CLUSTER"); return e ? atoi(e) : 0; }();
  const bool async = gv_async_epi() && !cl_env;  // (the DSMEM cluster reduction is gemv_w4_kernel's)
  const GvCfg c = gv_cfg(a.bn, async);
  a.w4_packed = static_cast<const uint8_t*>(packed);
  a.w4_scales = static_cast<const __nv_bfloat16*>(scales);
  a.wgroup = c.kbs;
  a.stages = c.stages;
  // SUN_GV_FIRST_WAIT (default 0): the epilogue-group GEMV issues its whole 2-stage ring at
  // once; 1 holds the second stage until the first has landed (helped the 4-stage ring of
  // gemv_w4_kernel; here B=1 2.333 vs 2.347 ms same box, profiles/r02/gv_first_wait_ab.txt)
  static const int fw_env = [] { const char* e = getenv("SUN_GV_FIRST_WAIT"); return e ? atoi(e) : 0; }();
  a.gv_first_wait = fw_env;
  a.sk_units = 0;
  a.sk_part = part;
  a.sk_flags = cnt;
  tl_assign(a);
  tl_stamps(a);
  // whole tiles when every SM gets one (splits = 0), else S-way split-K per tile with the
  // partials reduced through L2 by the tile's last arrival — or (SUN_GV_CLUSTER=1, off: measured
  // slower, the 8B O / down GEMV tails 2.6 -> 7.4 us, W4 B=1 step 2.35 -> 2.52 ms) one hardware
  // cluster of S CTAs per tile reducing over DSMEM between two cluster barriers
  const int slots = std::min(num_sms * c.per_sm, kMaxGemmCtas);
  int grid;
  a.vcluster = 1;
  g_cluster = 1;
  // SUN_GV_BALANCE (default 0: off): 1 the balanced schedule (gv_bal_range) when whole tiles
  // leave a remainder (8B gate_up: 224 tiles on 148 CTAs), 2 also in place of the per-tile
  // split. Measured slower (profiles/r02/gv_balance_ab.txt, same box): gate_up 24.1 -> 28.7 us
  // at B=1, W4 B=1 step 2.44 -> 2.62 ms (2: 3.13) — every CTA now streams, and the mid-stream
  // partial park / reduction round trips stall the compute warps that also run the epilogue
  static const int bal_env = [] { const char* e = getenv("SUN_GV_BALANCE"); return e ? atoi(e) : 0; }();
  const int W = p.m_tiles / slots, Ur = (p.m_tiles - W * slots) * p.ksteps;
  const bool bal_ok = Ur >= slots && (Ur + slots - 1) / slots <= p.ksteps;
  if (bal_ok && ((W >= 1 && bal_env >= 1) || (W == 0 && bal_env >= 2))) {
    a.splits = -1;
    grid = slots;
  } else if (p.m_tiles >= slots) {
    a.splits = 0;
    grid = slots;
  } else {
    // SUN_GV_SPLIT_CAP: largest split-K factor per tile (default: as many as the SMs allow)
    static const int cap_env = [] { const char* e = getenv("SUN_GV_SPLIT_CAP"); return e ? atoi(e) : 0; }();
    a.splits = std::max(1, std::min(p.ksteps, slots / p.m_tiles));
    if (cap_env > 0) a.splits = std::min(a.splits, cap_env);
    grid = p.m_tiles * a.splits;
    if (cl_env && a.splits > 1 && a.splits <= 8 && max_active_clusters_gv(unsigned(a.splits), c.smem) >= p.m_tiles) {
      a.vcluster = 0;
      g_cluster = unsigned(a.splits);
    }
  }
  if (async && a.vcluster) {
    const size_t sm = c.smem + kGvaExtraSmem;
    if (a.batch <= 8) SUN_CUDA(launch(gemv_w4a_kernel<EPI, 1>, dim3(grid), dim3(kGvaThreads), sm, st, pdl, a));
    else SUN_CUDA(launch(gemv_w4a_kernel<EPI, 2>, dim3(grid), dim3(kGvaThreads), sm, st, pdl, a));
    return SUN_OK;
  }
  if (a.batch <= 8) SUN_CUDA(launch(gemv_w4_kernel<EPI, 1>, dim3(grid), dim3(kGvThreads), c.smem, st, pdl, a));
  else SUN_CUDA(launch(gemv_w4_kernel<EPI, 2>, dim3(grid), dim3(kGvThreads), c.smem, st, pdl, a));
  return SUN_OK;
}

// Small-batch QSUN layer chain (gemv_chain_w4_kernel): the W4 GEMV phases O -> gate_up ->
// down -> next QKV in one persistent launch of one CTA per SM (all resident: 1 x ~222 KB).
SunStatus run_gemv_chain_w4(GemmArgs* ph, const GemmPlan* plans, const void* const* packed,
                            const void* const* scales, int nph, float* part, unsigned* cnt, unsigned* bar,
                            cudaStream_t st, bool pdl, int num_sms) {
  GvChainArgs c;
  memset(&c, 0, sizeof(c));
  const int bn = ph[0].bn;
  if (bn != 16 || ph[0].batch > kGemvKernelMaxBatch) return fail(SUN_ERR_VALUE, "W4 GEMV chain takes <= 16 rows");
  const GvCfg g = gv_cfg(bn);
  const int G = std::min(num_sms, kMaxGemmCtas);
  for (int i = 0; i < nph; ++i) {
    GemmArgs a = ph[i];
    if (plans[i].m_tiles > kGvMaxTiles) return fail(SUN_ERR_UNSUPPORTED, "W4 GEMV chain: too many tiles");
    a.w4_packed = static_cast<const uint8_t*>(packed[i]);
    a.w4_scales = static_cast<const __nv_bfloat16*>(scales[i]);
    a.wgroup = g.kbs;
    a.stages = g.stages;
    a.sk_units = 0;
    a.sk_part = part;
    a.sk_flags = cnt;
    a.splits = plans[i].m_tiles >= G ? 0 : std::max(1, std::min(plans[i].ksteps, G / plans[i].m_tiles));
    a.vcluster = 1;  // (split tiles reduce through L2: the chain is not a cluster launch)
    c.ph[i] = a;
  }
  c.nph = nph;
  c.bar = bar;
  static const int pre_env = [] { const char* e = getenv("SUN_GVC_PRE"); return e ? atoi(e) : 2; }();
  c.pre = pre_env;
  tl_assign(c);
  if (g_tl.stamps != nullptr && c.tl != nullptr && c.tl_idx == g_tl.stamp_idx) c.stamps = g_tl.stamps;
  g_cluster = 1;
  if (ph[0].batch <= 8) SUN_CUDA(launch(gemv_chain_w4_kernel<1>, dim3(G), dim3(kGvThreads), g.smem, st, pdl, c));
  else SUN_CUDA(launch(gemv_chain_w4_kernel<2>, dim3(G), dim3(kGvThreads), g.smem, st, pdl, c));
  return SUN_OK;
}

// Layer GEMM chain (bf16): the phases' GemmArgs are filled as for run_gemm; every
// split phase reduces through L2 over 148 persistent CTAs. Used by default for
// decode batches (SUN_STEP_DISTINCT_ROWS; measured C2 1.65 -> 1.59 ms, C3 5.03 ->
// 4.95, C5 22.6 -> 22.3 once the attention prestages its pages);
// SUN_GEMM_CHAIN=0 / 1 forces it off / on. Its grid-count phase barriers need all
// 148 CTAs resident together: one step in flight per GPU (the workspace is not
// re-entrant anyway), no second persistent decoder on another stream.
// QSUN (W4) decode batches run the W4 layer chain (gemm_chain_w4_kernel) up to bn = 128:
// its TMEM holds two accumulators next to the dequantised A ring only up to there.
constexpr int kW4ChainMaxBn = 128;

bool use_chain(int flags, bool w4, int bn = 16) {
  static int v = [] {
    const char* e = getenv("SUN_GEMM_CHAIN");
    return e ? atoi(e) : -1;
  }();
  if (w4 && bn > kW4ChainMaxBn) return false;
  return v == 1 || (v < 0 && (flags & SUN_STEP_DISTINCT_ROWS));
}

// QSUN chain ring geometry for a batch width (as launch_cfg's W4 defaults): weight
// stages of 4 K blocks, activation stages of xk blocks, weights fill the rest.
struct W4ChainCfg {
  int wgroup, xk, xstages, stages;
  size_t smem;
};
W4ChainCfg w4_chain_cfg(int bn) {
  // (SUN_W4_WGROUP / SUN_W4_XK / SUN_W4_XSTAGES override, as for the separate W4 GEMMs)
  static const int env_wg = [] { const char* e = getenv("SUN_W4_WGROUP"); return e ? atoi(e) : 0; }();
  static const int env_xk = [] { const char* e = getenv("SUN_W4_XK"); return e ? atoi(e) : 0; }();
  static const int env_xs = [] { const char* e = getenv("SUN_W4_XSTAGES"); return e ? atoi(e) : 0; }();
  W4ChainCfg c{};
  c.wgroup = env_wg > 0 ? env_wg : 4;
  c.xk = env_xk > 0 ? env_xk : (bn <= 32 ? 4 : 2);
  c.xstages = env_xs > 0 ? env_xs : (bn > 64 ? 2 : 3);
  const int budget = kSmemPerSm - 2048 - 2048 - int(kEpiSmemBytes) - 1024 - c.xstages * int(w4_xstage_bytes(bn, c.xk));
  c.stages = std::max(2, std::min(kMaxWStages, budget / int(w4_wstage_bytes(c.wgroup))));
  c.smem = gemm_smem_bytes_w4(bn, c.wgroup, c.stages, c.xk, c.xstages);
  return c;
}

// Can every CTA of the chain's grid be resident at once on this device (one per SM,
// at the chain's shared-memory size)? Checked once per decoder; without it the
// chain's phase barriers could not make progress, so the step uses separate launches.
bool chain_fits(int num_sms) {
  int per_sm = 0;
  const size_t smem = gemm_smem_bytes(16, gemm_stages(16, false, 1), gemm_xstages(16));
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_chain_kernel, kGemmThreads, smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return per_sm >= 1 && num_sms >= 16;
}

// Co-resident 4-CTA clusters of the QSUN chain at this shared-memory size (cached).
int max_active_clusters_w4chain(size_t smem) {
  static std::map<size_t, int> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(smem);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(4 * kNumSms / 4);
  cfg.blockDim = dim3(kW4Threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 4;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_chain_w4_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[smem] = n;
  return n;
}

bool chain_w4_fits(int num_sms) {
  int per_sm = 0;
  const W4ChainCfg w = w4_chain_cfg(kW4ChainMaxBn);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_chain_w4_kernel, kW4Threads, w.smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return per_sm >= 1 && num_sms >= 16;
}

// QSUN layer chain: one CTA per SM, split phases (<= G tiles) as virtual clusters
// reduced through L2, whole tiles otherwise; packed[i] / scales[i] per phase.
SunStatus run_chain_w4(GemmArgs* ph, const int* epi, const GemmPlan* plans, const void* const* packed,
                       const void* const* scales, int nph, unsigned* bar, cudaStream_t st, bool pdl, int num_sms) {
  ChainArgs c;
  memset(&c, 0, sizeof(c));
  const int bn = ph[0].bn;
  const W4ChainCfg w = w4_chain_cfg(bn);
  // 4-CTA clusters (SUN_CHAIN_CLUSTER, default on) when every cluster of the grid can be
  // resident at once: split phases with S = 4 or 2 reduce over DSMEM (partials parked in
  // the idle activation ring), the rest through L2; else 148 plain CTAs, L2 only
  static const int cl_env = [] { const char* e = getenv("SUN_CHAIN_CLUSTER"); return e ? atoi(e) : 1; }();
  int G = num_sms;
  if (cl_env) {
    const int ncl = std::min(num_sms / 4, max_active_clusters_w4chain(w.smem));
    bool any = false;
    for (int i = 0; i < nph; ++i)
      any = any || (plans[i].m_tiles <= ncl && plans[i].ksteps >= 4 && 4 * ncl / plans[i].m_tiles >= 4);
    if (ncl >= 16 && (any || cl_env == 2)) {
      c.hw = 1;
      G = 4 * ncl;
    }
  }
  for (int i = 0; i < nph; ++i) {
    GemmArgs a = ph[i];
    const GemmPlan& p = plans[i];
    a.wblk = nullptr;
    a.w4_packed = static_cast<const uint8_t*>(packed[i]);
    a.w4_scales = static_cast<const __nv_bfloat16*>(scales[i]);
    a.stages = w.stages;
    a.xstages = w.xstages;
    a.wgroup = w.wgroup;
    a.xk = w.xk;
    const int want = p.m_tiles <= G ? std::min(std::min(8, G / std::max(1, p.m_tiles)), p.ksteps) : 1;
    if (c.hw && want >= 2 && p.ksteps >= 4) {  // 4 / S tiles per cluster, DSMEM
      a.splits = want >= 4 ? 4 : 2;
      a.vcluster = 0;
    } else {
      a.splits = want;
      a.vcluster = want > 1 ? 1 : 0;
    }
    a.sk_units = 0;
    c.ph[i] = a;
    c.epi[i] = epi[i];
  }
  c.nph = nph;
  c.bar = bar;
  tl_assign(c);
  if (g_tl.stamps != nullptr && c.tl != nullptr && c.tl_idx == g_tl.stamp_idx) c.stamps = g_tl.stamps;
  g_cluster = c.hw ? 4u : 1u;
  SUN_CUDA(launch(gemm_chain_w4_kernel, dim3(G), dim3(kW4Threads), w.smem, st, pdl, c));
  return SUN_OK;
}

SunStatus run_chain(GemmArgs* ph, const int* epi, const GemmPlan* plans, const void* const* wblk, int nph,
                    unsigned* bar, cudaStream_t st, bool pdl, int num_sms, unsigned* qkv_ready = nullptr,
                    unsigned* qkv_reset = nullptr, int* qkv_writers = nullptr) {
  ChainArgs c;
  memset(&c, 0, sizeof(c));
  const int bn = ph[0].bn;
  const int stages = gemm_stages(bn, false, 1), xstages = gemm_xstages(bn);
  size_t smem = gemm_smem_bytes(bn, stages, xstages);
  // 4-CTA clusters (SUN_CHAIN_CLUSTER, default on) when the DSMEM receive area
  // ([3 senders][ceil(bn/64) chunks][8 KB]) fits and every cluster of the grid can be
  // resident at once (the phase barriers need the whole grid): grid = 4 x clusters
  static const int cl_env = [] { const char* e = getenv("SUN_CHAIN_CLUSTER"); return e ? atoi(e) : 1; }();
  const size_t recv = size_t(3) * ((bn / 16 + 3) / 4) * 8192;
  int G = num_sms;  // L2 chain: one CTA per SM of this device (all co-resident)
  if (cl_env && smem + recv <= size_t(kSmemPerSm)) {
    const int ncl = std::min(num_sms / 4, max_active_clusters(4, smem + recv, false));
    bool any = false;  // some phase must get one tile per cluster (else the smaller grid only costs)
    for (int i = 0; i < nph; ++i)
      any = any || (plans[i].m_tiles <= ncl && plans[i].ksteps >= 4 && 4 * ncl / plans[i].m_tiles >= 4);
    if (ncl >= 32 && (any || cl_env == 2)) {  // (2: clusters even without an S = 4 phase)
      c.hw = 1;
      G = 4 * ncl;
      smem += recv;
    }
  }
  for (int i = 0; i < nph; ++i) {
    GemmArgs a = ph[i];
    const GemmPlan& p = plans[i];
    a.wblk = static_cast<const uint8_t*>(wblk[i]);
    a.stages = stages;
    a.xstages = xstages;
    const int want = p.m_tiles <= G ? std::min(std::min(8, G / std::max(1, p.m_tiles)), p.ksteps) : 1;
    static const int hw2 = [] { const char* e = getenv("SUN_CHAIN_HW2"); return e ? atoi(e) : 1; }();
    if (c.hw && (want >= 4 || (want >= 2 && hw2)) && p.ksteps >= 4) {  // 4 / S tiles per cluster, DSMEM
      a.splits = want >= 4 ? 4 : 2;
      a.vcluster = 0;
    } else {
      a.splits = want;
      a.vcluster = want > 1 ? 1 : 0;
    }
    a.sk_units = 0;
    c.ph[i] = a;
    c.epi[i] = epi[i];
  }
  c.nph = nph;
  c.bar = bar;
  // per-tile readiness between the phases (SUN_CHAIN_TILE_READY=1, default off: measured
  // slower, C2 1.540 -> 1.606 ms, C3 4.762 -> 4.882 — the early starters' streams lengthen
  // the stragglers' epilogue tails, and the phase's epilogues still wait for the whole
  // previous phase's norm statistics); the counters sit after the two phase counts
  static const int tr_env = [] { const char* e = getenv("SUN_CHAIN_TILE_READY"); return e ? atoi(e) : 0; }();
  bool tr = tr_env != 0;
  for (int i = 0; i < nph; ++i) tr = tr && plans[i].m_tiles <= kChainReadyTiles;
  if (tr) c.ready = bar + 16;
  // per-tile hand-off of the last (QKV) phase to the next layer's attention (SUN_ATTN_TILE_READY)
  if (qkv_ready && epi[nph - 1] == EPI_QKV_ROPE && plans[nph - 1].m_tiles <= kQkvReadyStride) {
    c.qkv_ready = qkv_ready;
    if (qkv_writers) *qkv_writers = c.ph[nph - 1].splits > 1 ? c.ph[nph - 1].splits : 1;
  }
  c.qkv_reset = qkv_reset;
  c.qkv_reset_n = kQkvReadyStride;
  tl_assign(c);
  if (g_tl.stamps != nullptr && c.tl != nullptr && c.tl_idx == g_tl.stamp_idx) c.stamps = g_tl.stamps;
  g_cluster = c.hw ? 4u : 1u;
  SUN_CUDA(launch(gemm_chain_kernel, dim3(G), dim3(kGemmThreads), smem, st, pdl, c));
  return SUN_OK;
}

// Split combine inside the attention kernel (last split merges) or as a separate
// grid (default: measured faster on B200 for C3, the parallel merge has no
// serial tail). Env SUN_ATTN_FUSED_COMBINE=1 selects the fused variant.
int attn_fused_combine() {
  static int v = [] {
    const char* e = getenv("SUN_ATTN_FUSED_COMBINE");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// The decode attention of layer l >= 1 starts on the QKV tiles it reads as soon as the previous
// layer chain's epilogues publish them (per-tile counters) instead of waiting for that chain
// grid to complete (SUN_ATTN_TILE_READY, bf16 layer chain only).
int attn_tile_ready() {
  static const int v = [] { const char* e = getenv("SUN_ATTN_TILE_READY"); return e ? atoi(e) : 0; }();
  return v;
}

int auto_pages_per_split(const SunDecoderDims& d, int batch) {
  // With >= 3 (sequence, kv head) units per SM the attention is balanced without
  // splitting: one split per sequence, no partials, no combine launch (C3: 5.347 vs
  // 5.379 ms/step). Otherwise enough (split, kv_head, seq) units for ~4 resident
  // waves of 2 CTAs/SM at the longest context the decoder admits; at least 8
  // pages (128 tokens) so a unit amortises its TMA ramp.
  const int max_pages = (d.max_context + kPageTokens - 1) / kPageTokens;
  const long long pairs = (long long)batch * d.n_kv_heads;
  // (d = 64 was split-faster before the attention prestaged its pages: C2 0.99 vs 0.96 ms;
  // now unsplit wins there too, 1.541 vs 1.566 ms)
  if (pairs >= 3LL * kNumSms) return max_pages;
  const long long want_units = 8LL * kNumSms;
  long long splits = (want_units + pairs - 1) / pairs;
  if (splits < 1) splits = 1;
  long long pps = (max_pages + splits - 1) / splits;
  if (pps < 8) pps = 8;
  if (pps > max_pages) pps = max_pages;
  return int(pps);
}

// Row groups for the attention of the next sun_decode_step (sun_decode_step_grouped).
struct RowGroups {
  const int* start = nullptr;
  const int* len = nullptr;
  int n = 0;
};
thread_local RowGroups g_groups;

SunStatus run_attention(const SunDecoderDims& d, const CUtensorMap& tm_kv, AttnArgs aa, int batch,
                        cudaStream_t st, bool pdl) {
  tl_assign(aa);
  if (g_groups.start != nullptr) {  // token-parallel prefill: rows of a prompt share KV page loads
    aa.group_start = g_groups.start;
    aa.group_len = g_groups.len;
    aa.fused_combine = 0;
    aa.qkv_ready = nullptr;
    dim3 ggrid(aa.max_splits, d.n_kv_heads, g_groups.n);
    if (d.head_dim == 128) SUN_CUDA(launch(attn_group_kernel<128>, ggrid, dim3(128), AttnCfg<128>::kSmem, st, pdl, tm_kv, aa));
    else SUN_CUDA(launch(attn_group_kernel<64>, ggrid, dim3(128), AttnCfg<64>::kSmem, st, pdl, tm_kv, aa));
    if (aa.max_splits > 1) {
      if (d.head_dim == 128)
        SUN_CUDA(launch(attn_combine_kernel<128>, dim3(d.n_q_heads, batch), dim3(128), 0, st, pdl, aa));
      else
        SUN_CUDA(launch(attn_combine_kernel<64>, dim3(d.n_q_heads, batch), dim3(128), 0, st, pdl, aa));
    }
    return SUN_OK;
  }
  dim3 grid(aa.max_splits, d.n_kv_heads, batch);
  if (d.head_dim == 128) {
    SUN_CUDA(launch(attn_decode_kernel<128>, grid, dim3(128), AttnCfg<128>::kSmem, st, pdl, tm_kv, aa));
    if (!aa.fused_combine && aa.max_splits > 1)
      SUN_CUDA(launch(attn_combine_kernel<128>, dim3(d.n_q_heads, batch), dim3(128), 0, st, pdl, aa));
  } else {
    SUN_CUDA(launch(attn_decode_kernel<64>, grid, dim3(128), AttnCfg<64>::kSmem, st, pdl, tm_kv, aa));
    if (!aa.fused_combine && aa.max_splits > 1)
      SUN_CUDA(launch(attn_combine_kernel<64>, dim3(d.n_q_heads, batch), dim3(128), 0, st, pdl, aa));
  }
  return SUN_OK;
}

}  // namespace

extern "C" {

int32_t sun_abi_version(void) { return SUN_ABI_VERSION; }
const char* sun_last_error(void) { return g_last_error.c_str(); }

SunStatus sun_decoder_workspace_bytes(const SunDecoderDims* dims, int32_t max_batch, size_t* bytes) {
  SunStatus st = check_dims(dims);
  if (st != SUN_OK) return st;
  if (max_batch < 1 || max_batch > 256) return fail(SUN_ERR_VALUE, "max_batch must be in [1,256]");
  *bytes = layout_ws(*dims, max_batch).total;
  return SUN_OK;
}

SunStatus sun_decoder_create(const SunDecoderDims* dims, const SunWeights* weights, const SunKvPool* kv,
                             void* workspace, size_t workspace_bytes, int32_t max_batch, int32_t use_pdl,
                             SunDecoder** out) {
  SunStatus st = check_dims(dims);
  if (st != SUN_OK) return st;
  if (!weights || !kv || !out || !weights->layers) return fail(SUN_ERR_VALUE, "null argument");
  if (max_batch < 1 || max_batch > 256) return fail(SUN_ERR_VALUE, "max_batch must be in [1,256]");
  if ((st = check_kv_geometry(*dims, *kv)) != SUN_OK) return st;
  init_kernel_attrs();
  SunDecoder* dec = new SunDecoder();
  dec->num_sms = device_sms();
  dec->chain_ok = chain_fits(dec->num_sms);
  dec->chain_w4_ok = chain_w4_fits(dec->num_sms);
  dec->d = *dims;
  dec->max_batch = max_batch;
  dec->bmp = round16(max_batch);
  dec->pdl = use_pdl != 0;
  dec->layers.assign(weights->layers, weights->layers + dims->n_layers);
  dec->w = *weights;
  dec->w.layers = dec->layers.data();
  dec->kv = *kv;
  dec->page_stride = (long long)dims->n_layers * 2 * dims->n_kv_heads * dims->page_size * dims->head_dim;
  dec->L = layout_ws(*dims, max_batch);
  if (workspace_bytes < dec->L.total) {
    delete dec;
    return fail(SUN_ERR_CAPACITY, "workspace %zu < required %zu bytes", workspace_bytes, dec->L.total);
  }
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  dec->ws = ws;
  dec->resid = reinterpret_cast<float*>(ws + dec->L.resid);
  dec->xn = reinterpret_cast<__nv_bfloat16*>(ws + dec->L.xn);
  dec->q = reinterpret_cast<__nv_bfloat16*>(ws + dec->L.q);
  dec->attn = reinterpret_cast<__nv_bfloat16*>(ws + dec->L.attn);
  dec->act = reinterpret_cast<__nv_bfloat16*>(ws + dec->L.act);
  dec->part_o = reinterpret_cast<float*>(ws + dec->L.part_o);
  dec->part_ml = reinterpret_cast<float*>(ws + dec->L.part_ml);
  dec->attn_cnt = reinterpret_cast<unsigned*>(ws + dec->L.attn_cnt);
  dec->ss = reinterpret_cast<float*>(ws + dec->L.ss);
  dec->amax_val = reinterpret_cast<float*>(ws + dec->L.amax_val);
  dec->amax_idx = reinterpret_cast<int*>(ws + dec->L.amax_idx);
  dec->logits = reinterpret_cast<float*>(ws + dec->L.logits);
  dec->sk_part = reinterpret_cast<float*>(ws + dec->L.sk_part);
  dec->sk_flags = reinterpret_cast<unsigned*>(ws + dec->L.sk_flags);
  dec->chain_bar = reinterpret_cast<unsigned*>(ws + dec->L.chain_bar);
  dec->err = reinterpret_cast<unsigned*>(ws + dec->L.err);
  dec->gv_part = reinterpret_cast<float*>(ws + dec->L.gv_part);
  dec->gv_cnt = reinterpret_cast<unsigned*>(ws + dec->L.gv_cnt);
  dec->qkv_ready = reinterpret_cast<unsigned*>(ws + dec->L.qkv_ready);

  const SunDecoderDims& d = *dims;
  const int qd = d.n_q_heads * d.head_dim;
  dec->p_qkv = plan_gemm(qkv_rows(d), d.hidden);
  dec->p_o = plan_gemm(d.hidden, qd);
  dec->p_gu = plan_gemm(gu_rows(d), d.hidden);
  dec->p_down = plan_gemm(d.hidden, d.ffn);
  dec->p_lm = plan_gemm(d.vocab, d.hidden);
  if ((st = make_map_kv(&dec->tm_kv, d, *kv)) != SUN_OK) { delete dec; return st; }
  // zero the activation buffers once (K padding of SUN-ACT is never written) and
  // the attention split counters (self-resetting afterwards)
  cudaError_t e = cudaMemset(ws, 0, dec->L.part_o);
  if (e == cudaSuccess) e = cudaMemset(ws + dec->L.attn_cnt, 0, size_t(max_batch) * d_cnt_heads(*dims) * 4);
  if (e == cudaSuccess) e = cudaMemset(ws + dec->L.sk_flags, 0, kMaxGemmCtas * 4);
  if (e == cudaSuccess) e = cudaMemset(ws + dec->L.chain_bar, 0, 64 + size_t(kChainMaxPhases) * kChainReadyTiles * 4);
  if (e == cudaSuccess) e = cudaMemset(ws + dec->L.err, 0, 64);
  if (e == cudaSuccess) e = cudaMemset(ws + dec->L.gv_cnt, 0, kGvMaxTiles * 4);
  if (e == cudaSuccess) e = cudaMemset(ws + dec->L.qkv_ready, 0, size_t(d.n_layers) * kQkvReadyStride * 4);
  if (e != cudaSuccess) {
    delete dec;
    return fail(SUN_ERR_CUDA, "cudaMemset ws: %s", cudaGetErrorString(e));
  }
  *out = dec;
  return SUN_OK;
}

SunStatus sun_decoder_destroy(SunDecoder* dec) {
  delete dec;
  return SUN_OK;
}

SunStatus sun_decode_step(SunDecoder* dec, const int32_t* tokens, const int32_t* positions,
                          const int32_t* block_tables, int32_t bt_stride, int32_t batch,
                          int32_t pages_per_split, float* logits, int32_t* next_tokens, int32_t flags,
                          void* stream) {
  if (!dec) return fail(SUN_ERR_VALUE, "null decoder");
  if (batch < 1) return fail(SUN_ERR_VALUE, "decode batch must be non-empty");
  if (batch > dec->max_batch) return fail(SUN_ERR_CAPACITY, "batch %d > max_batch %d", batch, dec->max_batch);
  if (!tokens || !positions || !block_tables || !next_tokens) return fail(SUN_ERR_VALUE, "null buffer");
  const SunDecoderDims& d = dec->d;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool pdl = dec->pdl;
  const int bn = round16(batch);  // MMA N and the SUN-ACT row count of this step
  SunStatus s;
  const int qd = d.n_q_heads * d.head_dim;
  const int max_pages = (d.max_context + kPageTokens - 1) / kPageTokens;
  const int pps = pages_per_split > 0 ? std::min(pages_per_split, max_pages) : auto_pages_per_split(d, batch);
  float* lg = logits ? logits : dec->logits;
  const bool w4 = d.weight_bits == 4;
  // Timing experiments only (SUN_SKIP_KERNELS bitmask: 1 QKV, 2 attention, 8 O, 16
  // gate_up, 32 down): leave a kernel class out of the step to read its effective
  // cost inside the PDL-overlapped graph. Results are then meaningless.
  static const int skip = [] { const char* e = getenv("SUN_SKIP_KERNELS"); return e ? atoi(e) : 0; }();

  AttnArgs aa;
  memset(&aa, 0, sizeof(aa));
  aa.q = dec->q;
  aa.positions = positions;
  aa.block_tables = block_tables;
  aa.bt_stride = bt_stride;
  aa.n_q_heads = d.n_q_heads;
  aa.n_kv_heads = d.n_kv_heads;
  aa.pages_per_split = pps;
  aa.max_splits = (max_pages + pps - 1) / pps;
  aa.scale_log2 = 1.4426950408889634f / sqrtf(float(d.head_dim));
  aa.part_o = dec->part_o;
  aa.part_ml = dec->part_ml;
  aa.out = dec->attn;
  aa.ld_out = qd;
  aa.act_rows = bn;
  aa.counters = dec->attn_cnt;
  aa.fused_combine = attn_fused_combine();
  aa.max_ctx = d.max_context;
  static const int prestage_env = [] { const char* e = getenv("SUN_ATTN_PRESTAGE"); return e ? atoi(e) : 1; }();
  aa.prestage = (flags & SUN_STEP_DISTINCT_ROWS) && g_groups.start == nullptr && prestage_env ? 1 : 0;

  // RMSNorm is factored into the GEMMs: a producer writes xg = bf16(x * g) and
  // per-tile sums of squares, the consumer GEMM scales row b of its result by
  // r_b = rsqrt(mean(x_b^2) + eps) (W.(x*g*r) = r * W.(x*g)); no norm launches.
  const int ss_tiles = (d.hidden + kTileM - 1) / kTileM;
  auto consume_norm = [&](GemmArgs& g) {
    g.ss_in = dec->ss;
    g.ss_tiles = ss_tiles;
    g.norm_h = d.hidden;
    g.norm_eps = d.rms_eps;
  };
  auto produce_norm = [&](GemmArgs& g, const void* gain) {
    g.norm_w = static_cast<const __nv_bfloat16*>(gain);
    g.xg_out = dec->xn;
    g.ss_out = dec->ss;
  };
  // embedding gather + the first (attention) norm's operand
  StepCheck chk{positions, block_tables, bt_stride, d.vocab, d.max_context, (long long)dec->kv.num_pages, dec->err};
  SUN_CUDA(launch(embed_norm_kernel, dim3(batch), dim3(kRowThreads), 0, st, pdl, tokens,
                  static_cast<const __nv_bfloat16*>(dec->w.embed), dec->resid,
                  static_cast<const __nv_bfloat16*>(dec->layers[0].attn_norm), dec->xn, dec->ss, d.hidden, bn,
                  ss_tiles, chk));
  auto qkv_args = [&](int l) {  // QKV (* r_b) + bias + RoPE + KV append
    const SunLayerWeights& lw = dec->layers[l];
    GemmArgs a = base_args(dec->p_qkv, qkv_rows(d), d.hidden, batch, bn, dec->xn, dec->sk_part, dec->sk_flags);
    consume_norm(a);
    a.out_bf16 = dec->q;
    a.ldb = qd;
    a.bias = static_cast<const __nv_bfloat16*>(lw.b_qkv);
    a.rope_cos = dec->w.rope_cos;
    a.rope_sin = dec->w.rope_sin;
    a.positions = positions;
    a.block_tables = block_tables;
    a.bt_stride = bt_stride;
    a.kv_base = static_cast<__nv_bfloat16*>(dec->kv.base);
    a.page_stride = dec->page_stride;
    a.layer = l;
    a.n_q_heads = d.n_q_heads;
    a.n_kv_heads = d.n_kv_heads;
    a.head_dim = d.head_dim;
    a.page_size = d.page_size;
    a.max_pos = d.max_context;
    a.kv_pages = dec->kv.num_pages;
    return a;
  };
  auto o_args = [&](int l) {  // O projection + residual; emits the FFN norm's operand
    GemmArgs a = base_args(dec->p_o, d.hidden, qd, batch, bn, dec->attn, dec->sk_part, dec->sk_flags);
    a.out_f32 = dec->resid;
    a.ldo = d.hidden;
    produce_norm(a, dec->layers[l].ffn_norm);
    return a;
  };
  auto gu_args = [&](int l) {  // gate/up (* r_b) + SwiGLU
    GemmArgs a = base_args(dec->p_gu, gu_rows(d), d.hidden, batch, bn, dec->xn, dec->sk_part, dec->sk_flags);
    consume_norm(a);
    a.out_bf16 = dec->act;
    a.ldb = d.ffn;
    a.n_valid_out = d.ffn;
    return a;
  };
  auto down_args = [&](int l) {  // down + residual; emits the next attention norm's (or the final norm's) operand
    GemmArgs a = base_args(dec->p_down, d.hidden, d.ffn, batch, bn, dec->act, dec->sk_part, dec->sk_flags);
    a.out_f32 = dec->resid;
    a.ldo = d.hidden;
    produce_norm(a, l + 1 < d.n_layers ? dec->layers[l + 1].attn_norm : dec->w.final_norm);
    return a;
  };
  // QSUN small batches: the W4 GEMV, as separate launches (default) or as the GEMV layer
  // chain (SUN_W4_GEMV_CHAIN=1: measured slower, 2.56 vs 2.36 ms at B=1 — the split phases'
  // L2 reduction tails, 7-10 us, bound each phase either way and the chain adds the grid count)
  static const int gvchain_env = [] { const char* e = getenv("SUN_W4_GEMV_CHAIN"); return e ? atoi(e) : 0; }();
  const bool gemv = use_gemv(w4, batch);
  const bool chain = use_chain(flags, w4, bn) && (gemv ? gvchain_env != 0 : (w4 ? dec->chain_w4_ok : dec->chain_ok));
  auto w4_gemm = [&](auto epi_tag, const void* pk, const void* sc, const GemmArgs& ga, const GemmPlan& p,
                     const void* next_pk = nullptr, const GemmPlan* next_p = nullptr) {
    constexpr int E = decltype(epi_tag)::value;
    if (!gemv) return run_gemm<E>(nullptr, pk, sc, ga, p, st, pdl);
    GemmArgs g = ga;
    g.pf_w = nullptr;  // (the tcgen05 path's prefetch target: not this kernel's)
    if (next_p) gv_set_prefetch(g, next_pk, *next_p, dec->num_sms);
    return run_gemv_w4<E>(pk, sc, g, p, dec->gv_part, dec->gv_cnt, st, pdl, dec->num_sms);
  };
  const bool tile_ho = attn_tile_ready() && chain && !w4 && !gemv && aa.prestage;
  int qkv_writers = 0;  // writers per QKV tile of the chain that precedes the next attention
  using QkvT = std::integral_constant<int, EPI_QKV_ROPE>;
  using ResT = std::integral_constant<int, EPI_RESID_ADD>;
  using SwiT = std::integral_constant<int, EPI_SWIGLU>;
  for (int l = 0; l < d.n_layers; ++l) {
    const SunLayerWeights& lw = dec->layers[l];
    GemmArgs a;
    if (!chain || l == 0) {
      a = qkv_args(l);
      set_prefetch(a, lw.w_o, dec->p_o, bn, w4);  // O-proj weights, through the attention kernel
      if (!(skip & 1)) s = w4 ? w4_gemm(QkvT{}, lw.w_qkv, lw.s_qkv, a, dec->p_qkv, lw.w_o, &dec->p_o)
             : run_gemm<EPI_QKV_ROPE>(lw.w_qkv, nullptr, nullptr, a, dec->p_qkv, st, pdl);
      if (s != SUN_OK) return s;
    }
    // paged attention
    aa.layer = l;
    aa.qkv_ready = (chain && tile_ho && l > 0 && qkv_writers > 0) ? dec->qkv_ready + size_t(l) * kQkvReadyStride : nullptr;
    aa.ready_writers = static_cast<unsigned>(qkv_writers);
    if (!(skip & 2) && (s = run_attention(d, dec->tm_kv, aa, batch, st, pdl)) != SUN_OK) return s;
    if (chain) {  // O -> gate_up -> down (-> next layer's QKV) in one persistent launch
      GemmArgs ph[4] = {o_args(l), gu_args(l), down_args(l), GemmArgs{}};
      int epi[4] = {EPI_RESID_ADD, EPI_SWIGLU, EPI_RESID_ADD, EPI_QKV_ROPE};
      GemmPlan plans[4] = {dec->p_o, dec->p_gu, dec->p_down, dec->p_qkv};
      const void* wb[4] = {lw.w_o, lw.w_gate_up, lw.w_down, nullptr};
      const void* sc[4] = {lw.s_o, lw.s_gate_up, lw.s_down, nullptr};
      int nph = 3;
      if (l + 1 < d.n_layers) {
        ph[3] = qkv_args(l + 1);
        wb[3] = dec->layers[l + 1].w_qkv;
        sc[3] = dec->layers[l + 1].s_qkv;
        nph = 4;
      }
      s = gemv ? run_gemv_chain_w4(ph, plans, wb, sc, nph, dec->gv_part, dec->gv_cnt, dec->chain_bar, st, pdl,
                                   dec->num_sms)
          : w4 ? run_chain_w4(ph, epi, plans, wb, sc, nph, dec->chain_bar, st, pdl, dec->num_sms)
               : run_chain(ph, epi, plans, wb, nph, dec->chain_bar, st, pdl, dec->num_sms,
                           tile_ho && nph == 4 ? dec->qkv_ready + size_t(l + 1) * kQkvReadyStride : nullptr,
                           tile_ho && l > 0 ? dec->qkv_ready + size_t(l) * kQkvReadyStride : nullptr, &qkv_writers);
      if (s != SUN_OK) return s;
      continue;
    }
    a = o_args(l);
    set_prefetch(a, lw.w_gate_up, dec->p_gu, bn, w4);
    if (!(skip & 8)) s = w4 ? w4_gemm(ResT{}, lw.w_o, lw.s_o, a, dec->p_o, lw.w_gate_up, &dec->p_gu)
           : run_gemm<EPI_RESID_ADD>(lw.w_o, nullptr, nullptr, a, dec->p_o, st, pdl);
    if (s != SUN_OK) return s;
    a = gu_args(l);
    set_prefetch(a, lw.w_down, dec->p_down, bn, w4);
    if (!(skip & 16)) s = w4 ? w4_gemm(SwiT{}, lw.w_gate_up, lw.s_gate_up, a, dec->p_gu, lw.w_down, &dec->p_down)
           : run_gemm<EPI_SWIGLU>(lw.w_gate_up, nullptr, nullptr, a, dec->p_gu, st, pdl);
    if (s != SUN_OK) return s;
    a = down_args(l);
    if (l + 1 < d.n_layers) set_prefetch(a, dec->layers[l + 1].w_qkv, dec->p_qkv, bn, w4);
    else set_prefetch(a, dec->w.lm_head, dec->p_lm, bn, false);
    if (!(skip & 32)) s = w4 ? w4_gemm(ResT{}, lw.w_down, lw.s_down, a, dec->p_down,
                                       l + 1 < d.n_layers ? dec->layers[l + 1].w_qkv : nullptr, &dec->p_qkv)
           : run_gemm<EPI_RESID_ADD>(lw.w_down, nullptr, nullptr, a, dec->p_down, st, pdl);
    if (s != SUN_OK) return s;
  }
  // lm_head (* r_b) with per-tile argmax partials, then greedy sampling
  GemmArgs a = base_args(dec->p_lm, d.vocab, d.hidden, batch, bn, dec->xn, dec->sk_part, dec->sk_flags);
  consume_norm(a);
  a.out_f32 = lg;
  a.ldo = d.vocab;
  a.amax_val = dec->amax_val;
  a.amax_idx = dec->amax_idx;
  if ((s = run_gemm<EPI_LOGITS>(dec->w.lm_head, nullptr, nullptr, a, dec->p_lm, st, pdl)) != SUN_OK) return s;
  SUN_CUDA(launch(argmax_reduce_kernel, dim3(batch), dim3(kRowThreads), 0, st, pdl, (const float*)dec->amax_val,
                  (const int*)dec->amax_idx, dec->p_lm.m_tiles, bn, next_tokens,
                  (flags & SUN_STEP_FEEDBACK) ? const_cast<int*>(tokens) : (int*)nullptr,
                  const_cast<int*>(positions), dec->err));
  return SUN_OK;
}

SunStatus sun_launch_count(int64_t* launches) {
  if (!launches) return fail(SUN_ERR_VALUE, "null argument");
  *launches = g_trace.launches;
  return SUN_OK;
}

SunStatus sun_decode_step_profile(SunDecoder* dec, const int32_t* tokens, const int32_t* positions,
                                  const int32_t* block_tables, int32_t bt_stride, int32_t batch,
                                  int32_t pages_per_split, float* logits, int32_t* next_tokens, void* stream,
                                  float* kernel_ms, int32_t capacity, int32_t* n_kernels) {
  if (!dec || !kernel_ms || !n_kernels) return fail(SUN_ERR_VALUE, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<cudaEvent_t> evs;
  cudaEvent_t start;
  SUN_CUDA(cudaEventCreate(&start));
  SUN_CUDA(cudaEventRecord(start, st));
  const bool pdl = dec->pdl;
  dec->pdl = false;  // serialise kernels so event deltas attribute time to one kernel
  g_trace.events = &evs;
  SunStatus s = sun_decode_step(dec, tokens, positions, block_tables, bt_stride, batch, pages_per_split, logits,
                                next_tokens, SUN_STEP_DISTINCT_ROWS, stream);
  g_trace.events = nullptr;
  dec->pdl = pdl;
  if (s != SUN_OK) return s;
  SUN_CUDA(cudaStreamSynchronize(st));
  const int n = int(evs.size());
  *n_kernels = n;
  cudaEvent_t prev = start;
  for (int i = 0; i < n && i < capacity; ++i) {
    SUN_CUDA(cudaEventElapsedTime(&kernel_ms[i], prev, evs[i]));
    prev = evs[i];
  }
  cudaEventDestroy(start);
  for (auto e : evs) cudaEventDestroy(e);
  return SUN_OK;
}

SunStatus sun_decode_step_grouped(SunDecoder* dec, const int32_t* tokens, const int32_t* positions,
                                  const int32_t* block_tables, int32_t bt_stride, int32_t batch,
                                  int32_t pages_per_split, float* logits, int32_t* next_tokens, int32_t flags,
                                  void* stream, const int32_t* group_start, const int32_t* group_len,
                                  int32_t n_groups) {
  if (!group_start || !group_len || n_groups < 1 || n_groups > batch) return fail(SUN_ERR_VALUE, "bad row groups");
  g_groups.start = group_start;
  g_groups.len = group_len;
  g_groups.n = n_groups;
  SunStatus s = sun_decode_step(dec, tokens, positions, block_tables, bt_stride, batch, pages_per_split, logits,
                                next_tokens, flags, stream);
  g_groups = RowGroups{};
  return s;
}

SunStatus sun_decode_step_timeline(SunDecoder* dec, const int32_t* tokens, const int32_t* positions,
                                   const int32_t* block_tables, int32_t bt_stride, int32_t batch,
                                   int32_t pages_per_split, int32_t* next_tokens, void* stream, uint64_t* timeline,
                                   int32_t capacity, int32_t* n_launches, uint64_t* stamps, int32_t stamp_launch) {
  if (!dec || !timeline || !n_launches || capacity < 1) return fail(SUN_ERR_VALUE, "null argument");
  g_tl.tl = reinterpret_cast<unsigned long long*>(timeline);
  g_tl.next = 0;
  g_tl.capacity = capacity;
  g_tl.stamps = reinterpret_cast<unsigned long long*>(stamps);
  g_tl.stamp_idx = stamp_launch;
  SunStatus s = sun_decode_step(dec, tokens, positions, block_tables, bt_stride, batch, pages_per_split, nullptr,
                                next_tokens, SUN_STEP_DISTINCT_ROWS, stream);
  *n_launches = g_tl.next;
  g_tl = TimelineState{};
  return s;
}

SunStatus sun_gemm_workspace_bytes(int64_t n_out, int64_t k, int32_t batch, size_t* bytes) {
  if (n_out < 1 || k < 1 || batch < 1 || batch > 256) return fail(SUN_ERR_VALUE, "bad gemm shape");
  const size_t act = align_up(size_t(round16(batch)) * size_t((k + 63) / 64) * 128, 1024);  // SUN-ACT copy of X
  // + stream-K partials (or the W4 GEMV's two slots per CTA) and flags / per-tile counters
  *bytes = act + std::max(sk_part_bytes(round16(batch)), gv_part_bytes()) + kGvMaxTiles * 4;
  return SUN_OK;
}

extern "C++" {
namespace {
template <int EPI>
SunStatus gemm_api(const void* wblk, const void* packed, const void* scales, int64_t n_out, int64_t k, const void* x,
                   int64_t ldx, int64_t x_rows, int32_t batch, float* out, int64_t ldo, void* workspace,
                   size_t workspace_bytes, void* stream, uint64_t* stamps, bool gemv = false) {
  if (batch < 1) return fail(SUN_ERR_VALUE, "empty batch");
  if (k % 8 != 0) return fail(SUN_ERR_UNSUPPORTED, "k must be a multiple of 8");
  size_t need = 0;
  SunStatus s = sun_gemm_workspace_bytes(n_out, k, batch, &need);
  if (s != SUN_OK) return s;
  if (workspace_bytes < need) return fail(SUN_ERR_CAPACITY, "gemm workspace too small");
  const int bn = round16(batch);
  if (x_rows < batch) return fail(SUN_ERR_VALUE, "x has fewer rows than batch");
  init_kernel_attrs();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SUN_CUDA(launch(block_activations_kernel, dim3(148), dim3(256), 0, st, false, static_cast<const __nv_bfloat16*>(x),
                  int(batch), (long long)k, (long long)ldx, bn, static_cast<uint8_t*>(workspace)));
  GemmPlan p = plan_gemm(n_out, k);
  const size_t act = align_up(size_t(bn) * size_t((k + 63) / 64) * 128, 1024);
  uint8_t* wsb = static_cast<uint8_t*>(workspace);
  float* part = reinterpret_cast<float*>(wsb + act);
  unsigned* flags = reinterpret_cast<unsigned*>(wsb + act + std::max(sk_part_bytes(bn), gv_part_bytes()));
  GemmArgs a = base_args(p, n_out, k, batch, bn, workspace, part, flags);
  a.out_f32 = out;
  a.ldo = ldo;
  a.stamps = reinterpret_cast<unsigned long long*>(stamps);
  if (gemv) return run_gemv_w4<EPI>(packed, scales, a, p, part, flags, st, false, device_sms());
  return run_gemm<EPI>(wblk, packed, scales, a, p, st, false);
}
}  // namespace
}  // extern "C++"

SunStatus sun_gemm_bf16(const void* w, int64_t n_out, int64_t k, const void* x, int64_t ldx, int64_t x_rows,
                        int32_t batch, float* out, int64_t ldo, int32_t accumulate, void* workspace,
                        size_t workspace_bytes, void* stream) {
  return accumulate ? gemm_api<EPI_RESID_ADD>(w, nullptr, nullptr, n_out, k, x, ldx, x_rows, batch, out, ldo,
                                              workspace, workspace_bytes, stream, nullptr)
                    : gemm_api<EPI_STORE_F32>(w, nullptr, nullptr, n_out, k, x, ldx, x_rows, batch, out, ldo,
                                              workspace, workspace_bytes, stream, nullptr);
}

SunStatus sun_gemm_bf16_stamped(const void* w, int64_t n_out, int64_t k, const void* x, int64_t ldx,
                                int64_t x_rows, int32_t batch, float* out, int64_t ldo, int32_t accumulate,
                                void* workspace, size_t workspace_bytes, void* stream, uint64_t* stamps) {
  return accumulate ? gemm_api<EPI_RESID_ADD>(w, nullptr, nullptr, n_out, k, x, ldx, x_rows, batch, out, ldo,
                                              workspace, workspace_bytes, stream, stamps)
                    : gemm_api<EPI_STORE_F32>(w, nullptr, nullptr, n_out, k, x, ldx, x_rows, batch, out, ldo,
                                              workspace, workspace_bytes, stream, stamps);
}

SunStatus sun_gemm_w4(const void* packed, const void* scales, int64_t n_out, int64_t k, const void* x, int64_t ldx,
                      int64_t x_rows, int32_t batch, float* out, int64_t ldo, int32_t accumulate, void* workspace,
                      size_t workspace_bytes, void* stream) {
  if (k % 128 != 0) return fail(SUN_ERR_UNSUPPORTED, "W4 needs k multiple of 128");
  return accumulate ? gemm_api<EPI_RESID_ADD>(nullptr, packed, scales, n_out, k, x, ldx, x_rows, batch, out, ldo,
                                              workspace, workspace_bytes, stream, nullptr)
                    : gemm_api<EPI_STORE_F32>(nullptr, packed, scales, n_out, k, x, ldx, x_rows, batch, out, ldo,
                                              workspace, workspace_bytes, stream, nullptr);
}

SunStatus sun_gemv_w4(const void* packed, const void* scales, int64_t n_out, int64_t k, const void* x, int64_t ldx,
                      int64_t x_rows, int32_t batch, float* out, int64_t ldo, int32_t accumulate, void* workspace,
                      size_t workspace_bytes, void* stream) {
  if (k % 128 != 0) return fail(SUN_ERR_UNSUPPORTED, "W4 needs k multiple of 128");
  if (batch > kGemvKernelMaxBatch) return fail(SUN_ERR_VALUE, "W4 GEMV takes batches of <= %d rows", kGemvKernelMaxBatch);
  return accumulate ? gemm_api<EPI_RESID_ADD>(nullptr, packed, scales, n_out, k, x, ldx, x_rows, batch, out, ldo,
                                              workspace, workspace_bytes, stream, nullptr, true)
                    : gemm_api<EPI_STORE_F32>(nullptr, packed, scales, n_out, k, x, ldx, x_rows, batch, out, ldo,
                                              workspace, workspace_bytes, stream, nullptr, true);
}

SunStatus sun_gemv_w4_stamped(const void* packed, const void* scales, int64_t n_out, int64_t k, const void* x,
                              int64_t ldx, int64_t x_rows, int32_t batch, float* out, int64_t ldo, void* workspace,
                              size_t workspace_bytes, void* stream, uint64_t* stamps) {
  if (k % 128 != 0) return fail(SUN_ERR_UNSUPPORTED, "W4 needs k multiple of 128");
  if (batch > kGemvKernelMaxBatch) return fail(SUN_ERR_VALUE, "W4 GEMV takes batches of <= %d rows", kGemvKernelMaxBatch);
  return gemm_api<EPI_STORE_F32>(nullptr, packed, scales, n_out, k, x, ldx, x_rows, batch, out, ldo, workspace,
                                 workspace_bytes, stream, stamps, true);
}

SunStatus sun_gemm_w4_stamped(const void* packed, const void* scales, int64_t n_out, int64_t k, const void* x,
                              int64_t ldx, int64_t x_rows, int32_t batch, float* out, int64_t ldo, void* workspace,
                              size_t workspace_bytes, void* stream, uint64_t* stamps) {
  if (k % 128 != 0) return fail(SUN_ERR_UNSUPPORTED, "W4 needs k multiple of 128");
  return gemm_api<EPI_STORE_F32>(nullptr, packed, scales, n_out, k, x, ldx, x_rows, batch, out, ldo, workspace,
                                 workspace_bytes, stream, stamps);
}

SunStatus sun_attention_decode(const SunDecoderDims* dims, const SunKvPool* kv, int32_t layer, const void* q,
                               const int32_t* positions, const int32_t* block_tables, int32_t bt_stride,
                               int32_t batch, int32_t pages_per_split, void* out, void* workspace,
                               size_t workspace_bytes, void* stream) {
  SunStatus s = check_dims(dims);
  if (s != SUN_OK) return s;
  if (batch < 1) return fail(SUN_ERR_VALUE, "empty batch");
  init_kernel_attrs();
  const SunDecoderDims& d = *dims;
  const int max_pages = (d.max_context + kPageTokens - 1) / kPageTokens;
  const int pps = pages_per_split > 0 ? std::min(pages_per_split, max_pages) : auto_pages_per_split(d, batch);
  AttnArgs aa;
  memset(&aa, 0, sizeof(aa));
  aa.q = static_cast<const __nv_bfloat16*>(q);
  aa.positions = positions;
  aa.block_tables = block_tables;
  aa.bt_stride = bt_stride;
  aa.layer = layer;
  aa.n_q_heads = d.n_q_heads;
  aa.n_kv_heads = d.n_kv_heads;
  aa.pages_per_split = pps;
  aa.max_splits = (max_pages + pps - 1) / pps;
  aa.scale_log2 = 1.4426950408889634f / sqrtf(float(d.head_dim));
  const size_t po = size_t(batch) * d.n_q_heads * aa.max_splits * d.head_dim * 4;
  const size_t pm = size_t(batch) * d.n_q_heads * aa.max_splits * 2 * 4;
  const size_t pc = size_t(batch) * d.n_kv_heads * 4;
  if (workspace_bytes < align_up(po, 1024) + align_up(pm, 1024) + pc)
    return fail(SUN_ERR_CAPACITY, "attention workspace too small");
  aa.part_o = static_cast<float*>(workspace);
  aa.part_ml = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + align_up(po, 1024));
  aa.counters = reinterpret_cast<unsigned*>(static_cast<uint8_t*>(workspace) + align_up(po, 1024) + align_up(pm, 1024));
  aa.fused_combine = attn_fused_combine();
  aa.max_ctx = d.max_context;
  aa.out = static_cast<__nv_bfloat16*>(out);
  aa.ld_out = d.n_q_heads * d.head_dim;
  CUtensorMap tm;
  if ((s = make_map_kv(&tm, d, *kv)) != SUN_OK) return s;
  return run_attention(d, tm, aa, batch, static_cast<cudaStream_t>(stream), false);
}

SunStatus sun_decoder_status(SunDecoder* dec, uint32_t* flags, int32_t clear, void* stream) {
  if (!dec || !flags) return fail(SUN_ERR_VALUE, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned v = 0;
  SUN_CUDA(cudaMemcpyAsync(&v, dec->err, 4, cudaMemcpyDeviceToHost, st));
  if (clear) SUN_CUDA(cudaMemsetAsync(dec->err, 0, 4, st));
  SUN_CUDA(cudaStreamSynchronize(st));
  *flags = v;
  return SUN_OK;
}

SunStatus sun_decoder_uses_chain(SunDecoder* dec, int32_t flags, int32_t* uses) {
  if (!dec || !uses) return fail(SUN_ERR_VALUE, "null argument");
  const bool w4 = dec->d.weight_bits == 4;  // QSUN: for batches up to kW4ChainMaxBn
  *uses = (use_chain(flags, w4) && (w4 ? dec->chain_w4_ok : dec->chain_ok)) ? 1 : 0;
  return SUN_OK;
}

SunStatus sun_kv_page_bytes(const SunKvPool* kv, size_t* bytes) {
  if (!kv || !bytes || kv->n_layers < 1 || kv->n_kv_heads < 1 || kv->head_dim < 1 || kv->page_size < 1)
    return fail(SUN_ERR_VALUE, "bad KV pool geometry");
  *bytes = kv_page_bytes(*kv);
  return SUN_OK;
}

// ---- K8 hand-off by peer copy -------------------------------------------------
SunStatus sun_kv_pool_export(const SunKvPool* kv, SunKvPoolHandle* out) {
  if (!kv || !out || !kv->base) return fail(SUN_ERR_VALUE, "null argument");
  const PFN_getAddressRange_t range_fn = address_range_fn();
  if (!range_fn) return fail(SUN_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(kv->base)) != CUDA_SUCCESS)
    return fail(SUN_ERR_CUDA, "cuMemGetAddressRange failed for the KV pool");
  cudaIpcMemHandle_t h;
  SUN_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) <= sizeof(out->ipc), "IPC handle size");
  memset(out, 0, sizeof(*out));
  memcpy(out->ipc, &h, sizeof(h));
  out->offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(kv->base) - base);
  out->geometry = *kv;
  out->geometry.base = nullptr;
  return SUN_OK;
}

SunStatus sun_kv_pool_import(const SunKvPoolHandle* handle, SunKvPool* out) {
  if (!handle || !out) return fail(SUN_ERR_VALUE, "null argument");
  int here = 0;
  SUN_CUDA(cudaGetDevice(&here));
  const int peer = handle->geometry.device;
  if (peer != here) {  // copy engines reach the peer's HBM over NVLink
    int can = 0;
    SUN_CUDA(cudaDeviceCanAccessPeer(&can, here, peer));
    if (!can) return fail(SUN_ERR_UNSUPPORTED, "device %d cannot access device %d's memory", here, peer);
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) SUN_CUDA(e);
    cudaGetLastError();
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle->ipc, sizeof(h));
  void* base = nullptr;
  SUN_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *out = handle->geometry;
  out->base = static_cast<uint8_t*>(base) + handle->offset;
  return SUN_OK;
}

SunStatus sun_kv_pool_close(SunKvPool* imported) {
  if (!imported || !imported->base) return fail(SUN_ERR_VALUE, "null argument");
  // the mapping starts `offset` bytes before page 0: close the mapped allocation's base
  CUdeviceptr base = 0;
  size_t size = 0;
  if (address_range_fn() == nullptr ||
      address_range_fn()(&base, &size, reinterpret_cast<CUdeviceptr>(imported->base)) != CUDA_SUCCESS)
    return fail(SUN_ERR_CUDA, "cuMemGetAddressRange failed for the imported pool");
  SUN_CUDA(cudaIpcCloseMemHandle(reinterpret_cast<void*>(base)));
  imported->base = nullptr;
  return SUN_OK;
}

SunStatus sun_kv_handoff_copy(const SunKvPool* src, const int32_t* src_pages, const SunKvPool* dst,
                              const int32_t* dst_pages, int32_t n_pages, void* stream) {
  if (!src || !dst || (n_pages > 0 && (!src_pages || !dst_pages))) return fail(SUN_ERR_VALUE, "null argument");
  if (n_pages < 0) return fail(SUN_ERR_VALUE, "negative page count");
  if (src->n_layers != dst->n_layers || src->n_kv_heads != dst->n_kv_heads || src->head_dim != dst->head_dim ||
      src->page_size != dst->page_size || src->rope_theta != dst->rope_theta)
    return fail(SUN_ERR_MIXED_DECODER, "hand-off between KV pools of different geometry (not decoder-compatible)");
  const size_t pb = kv_page_bytes(*src);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < n_pages; ++i)  // validate everything before the first copy
    if (src_pages[i] < 0 || src_pages[i] >= src->num_pages || dst_pages[i] < 0 || dst_pages[i] >= dst->num_pages)
      return fail(SUN_ERR_VALUE, "hand-off page %d -> %d outside the pools", src_pages[i], dst_pages[i]);
  for (int i = 0; i < n_pages;) {
    const int s0 = src_pages[i], d0 = dst_pages[i];
    int n = 1;  // maximal run consecutive on both sides: one copy
    while (i + n < n_pages && src_pages[i + n] == s0 + n && dst_pages[i + n] == d0 + n) ++n;
    SUN_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(dst->base) + size_t(d0) * pb,
                             static_cast<const uint8_t*>(src->base) + size_t(s0) * pb, size_t(n) * pb,
                             cudaMemcpyDefault, st));
    i += n;
  }
  return SUN_OK;
}

SunStatus sun_blocked_bytes(int64_t rows, int64_t k, size_t* bytes) {
  if (rows < 1 || k < 1 || !bytes) return fail(SUN_ERR_VALUE, "bad shape");
  *bytes = size_t((rows + kTileM - 1) / kTileM) * size_t((k + kTileK - 1) / kTileK) * kTileWBytes;
  return SUN_OK;
}

SunStatus sun_block_weights_bf16(const void* w, int64_t rows, int64_t k, void* out, void* stream) {
  if (rows < 1 || k < 1 || k % 8 != 0) return fail(SUN_ERR_VALUE, "block_weights: k must be a multiple of 8");
  const long long m_tiles = (rows + kTileM - 1) / kTileM;
  const int kb64 = int((k + kTileK - 1) / kTileK);
  SUN_CUDA(launch(block_weights_kernel, dim3(unsigned(m_tiles * kb64)), dim3(256), 0, static_cast<cudaStream_t>(stream),
                  false, static_cast<const __nv_bfloat16*>(w), (long long)rows, (long long)k, kb64,
                  static_cast<uint8_t*>(out)));
  return SUN_OK;
}

SunStatus sun_rmsnorm(const float* x, const void* w, void* y, int32_t batch, int32_t h, float eps, void* stream) {
  if (batch < 1 || h % 4 != 0) return fail(SUN_ERR_VALUE, "bad rmsnorm shape");
  SUN_CUDA(launch(rmsnorm_kernel, dim3(batch), dim3(kRowThreads), 0, static_cast<cudaStream_t>(stream), false,
                  (const int*)nullptr, (const __nv_bfloat16*)nullptr, const_cast<float*>(x),
                  static_cast<const __nv_bfloat16*>(w), static_cast<__nv_bfloat16*>(y), h, (long long)h, eps, 0));
  return SUN_OK;
}

SunStatus sun_quantize_w4(const void* w, int64_t rows, int64_t k, int32_t group, void* packed, void* scales,
                          void* stream) {
  if (rows < 1 || k < 1 || group != 128 || k % group != 0) return fail(SUN_ERR_VALUE, "bad quantize shape");
  const long long groups = rows * (k / group);
  SUN_CUDA(launch(quantize_w4_kernel, dim3(unsigned((groups + 7) / 8)), dim3(256), 0,
                  static_cast<cudaStream_t>(stream), false, static_cast<const __nv_bfloat16*>(w), (long long)rows,
                  (long long)((rows + 127) / 128 * 128), (long long)k,
                  static_cast<uint8_t*>(packed), static_cast<__nv_bfloat16*>(scales)));
  return SUN_OK;
}

SunStatus sun_import_w4_ct(const void* ct_packed, const void* ct_scales, int64_t rows, int64_t k, int32_t group,
                           void* packed, void* scales, void* stream) {
  if (rows < 1 || k < 1 || group != 128 || k % group != 0) return fail(SUN_ERR_VALUE, "bad import_w4_ct shape");
  if (!ct_packed || !ct_scales || !packed || !scales) return fail(SUN_ERR_VALUE, "import_w4_ct: null pointer");
  const long long groups = rows * (k / group);
  SUN_CUDA(launch(import_w4_ct_kernel, dim3(unsigned((groups + 127) / 128)), dim3(128), 0,
                  static_cast<cudaStream_t>(stream), false, static_cast<const uint32_t*>(ct_packed),
                  static_cast<const __nv_bfloat16*>(ct_scales), (long long)rows, (long long)k,
                  static_cast<uint8_t*>(packed), static_cast<__nv_bfloat16*>(scales)));
  return SUN_OK;
}

}  // extern "C"
