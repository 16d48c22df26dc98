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
  int m_tiles, kb_total, kb_per_split, splits;
};

GemmPlan plan_gemm(int64_t n_out, int64_t k) {
  GemmPlan p;
  p.m_tiles = int((n_out + kTileM - 1) / kTileM);
  p.kb_total = int((k + kTileK - 1) / kTileK);
  const int target = 2 * kNumSms;
  int splits = (target + p.m_tiles - 1) / p.m_tiles;
  splits = std::max(1, std::min(splits, std::max(1, p.kb_total / 4)));
  p.kb_per_split = (p.kb_total + splits - 1) / splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  return p;
}

int gemm_stages(int bn) {
  const int budget = 110 * 1024 - 1280;
  int st = budget / int(kTileWBytes + bn * 128);
  return std::max(2, std::min(8, st));
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int round16(int b) { return (b + 15) / 16 * 16; }

template <typename K>
void set_max_smem(K kern) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

std::once_flag g_attr_once;
void init_kernel_attrs() {
  std::call_once(g_attr_once, [] {
    set_max_smem(gemm_bf16_kernel<EPI_STORE_F32>);
    set_max_smem(gemm_bf16_kernel<EPI_RESID_ADD>);
    set_max_smem(gemm_bf16_kernel<EPI_QKV_ROPE>);
    set_max_smem(gemm_bf16_kernel<EPI_SWIGLU>);
    set_max_smem(gemm_bf16_kernel<EPI_LOGITS>);
    set_max_smem(gemm_w4_kernel<EPI_RESID_ADD>);
    set_max_smem(gemm_w4_kernel<EPI_QKV_ROPE>);
    set_max_smem(gemm_w4_kernel<EPI_SWIGLU>);
    set_max_smem(gemm_w4_kernel<EPI_STORE_F32>);
    set_max_smem(attn_decode_kernel<64>);
    set_max_smem(attn_decode_kernel<128>);
  });
}

template <typename... KArgs, typename... Args>
cudaError_t launch_raw(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Per-thread launch accounting + optional per-kernel event timing (profile mode).
struct LaunchTrace {
  long long launches = 0;
  std::vector<cudaEvent_t>* events = nullptr;  // record one event after each launch
};
thread_local LaunchTrace g_trace;

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

// Workspace layout shared by sizing and creation.
struct WsLayout {
  size_t resid, xn, q, attn, act, part_o, part_ml, gemm_part, counters, amax_val, amax_idx, logits, total;
  int max_splits;
};

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
  w.resid = take(size_t(max_batch) * d.hidden * 4);
  w.xn = take(size_t(bmp) * d.hidden * 2);
  w.q = take(size_t(max_batch) * qd * 2);
  w.attn = take(size_t(bmp) * qd * 2);
  w.act = take(size_t(bmp) * d.ffn * 2);
  w.part_o = take(size_t(max_batch) * d.n_q_heads * w.max_splits * d.head_dim * 4);
  w.part_ml = take(size_t(max_batch) * d.n_q_heads * w.max_splits * 2 * 4);
  size_t gp = 0;
  int max_tiles = 0;
  const int64_t shapes[5][2] = {{qkv_rows(d), d.hidden}, {d.hidden, qd}, {gu_rows(d), d.hidden},
                                {d.hidden, d.ffn}, {d.vocab, d.hidden}};
  for (auto& s : shapes) {
    GemmPlan p = plan_gemm(s[0], s[1]);
    if (p.splits > 1) gp = std::max(gp, size_t(p.m_tiles) * p.splits * bmp * kTileM * 4);
    max_tiles = std::max(max_tiles, p.m_tiles);
  }
  w.gemm_part = take(std::max<size_t>(gp, 4));
  w.counters = take(size_t(max_tiles) * 4);
  const int lm_tiles = (d.vocab + kTileM - 1) / kTileM;
  w.amax_val = take(size_t(lm_tiles) * bmp * 4);
  w.amax_idx = take(size_t(lm_tiles) * bmp * 4);
  w.logits = take(size_t(max_batch) * d.vocab * 4);
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

struct XMaps {
  CUtensorMap xn, attn, act;
};

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
  std::vector<CUtensorMap> tm_qkv, tm_o, tm_gu, tm_down;
  CUtensorMap tm_lm;
  std::map<int, XMaps> xmaps;
  WsLayout L;
  uint8_t* ws = nullptr;
  float* resid;
  __nv_bfloat16 *xn, *q, *attn, *act;
  float *part_o, *part_ml, *gemm_part, *amax_val, *logits;
  unsigned* counters;
  int* amax_idx;
  GemmPlan p_qkv, p_o, p_gu, p_down, p_lm;
};

namespace {

SunStatus get_xmaps(SunDecoder* dec, int bn, XMaps** out) {
  auto it = dec->xmaps.find(bn);
  if (it == dec->xmaps.end()) {
    XMaps m;
    const SunDecoderDims& d = dec->d;
    SunStatus st;
    if ((st = make_map_2d(&m.xn, dec->xn, dec->bmp, d.hidden, d.hidden, bn)) != SUN_OK) return st;
    if ((st = make_map_2d(&m.attn, dec->attn, dec->bmp, d.n_q_heads * d.head_dim, d.n_q_heads * d.head_dim, bn)) != SUN_OK) return st;
    if ((st = make_map_2d(&m.act, dec->act, dec->bmp, d.ffn, d.ffn, bn)) != SUN_OK) return st;
    it = dec->xmaps.emplace(bn, m).first;
  }
  *out = &it->second;
  return SUN_OK;
}

GemmArgs base_args(const GemmPlan& p, int64_t n_out, int64_t k, int batch, int bn, float* part, unsigned* counters) {
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.n_out = int(n_out);
  a.k = int(k);
  a.batch = batch;
  a.bn = bn;
  a.kb_total = p.kb_total;
  a.kb_per_split = p.kb_per_split;
  a.splits = p.splits;
  a.stages = gemm_stages(bn);
  a.weight_bits = 16;
  a.partial = part;
  a.counters = counters;
  return a;
}

template <int EPI>
SunStatus run_gemm(const CUtensorMap& tw, const CUtensorMap& tx, const GemmArgs& a, const GemmPlan& p,
                   cudaStream_t st, bool pdl) {
  const size_t smem = gemm_smem_bytes(a.bn, a.stages);
  SUN_CUDA(launch(gemm_bf16_kernel<EPI>, dim3(p.m_tiles, p.splits), dim3(kGemmThreads), smem, st, pdl, tw, tx, a));
  return SUN_OK;
}

template <int EPI>
SunStatus run_gemm_w4(const W4Weights& ww, const CUtensorMap& tx, const GemmArgs& a, const GemmPlan& p,
                      cudaStream_t st, bool pdl) {
  const size_t smem = w4_smem_bytes(a.bn, a.stages);
  SUN_CUDA(launch(gemm_w4_kernel<EPI>, dim3(p.m_tiles, p.splits), dim3(kW4Threads), smem, st, pdl, ww, tx, a));
  return SUN_OK;
}

int auto_pages_per_split(const SunDecoderDims& d, int batch) {
  // Enough (split, kv_head, seq) units for ~4 resident waves of 2 CTAs/SM at
  // the longest context the decoder admits; at least 8 pages (128 tokens) so a
  // unit amortises its TMA ramp.
  const int max_pages = (d.max_context + kPageTokens - 1) / kPageTokens;
  const long long pairs = (long long)batch * d.n_kv_heads;
  const long long want_units = 8LL * kNumSms;
  long long splits = (want_units + pairs - 1) / pairs;
  if (splits < 1) splits = 1;
  long long pps = (max_pages + splits - 1) / splits;
  if (pps < 8) pps = 8;
  if (pps > max_pages) pps = max_pages;
  return int(pps);
}

SunStatus run_attention(const SunDecoderDims& d, const CUtensorMap& tm_kv, const AttnArgs& aa, int batch,
                        cudaStream_t st, bool pdl) {
  dim3 grid(aa.max_splits, d.n_kv_heads, batch);
  if (d.head_dim == 128) {
    SUN_CUDA(launch(attn_decode_kernel<128>, grid, dim3(128), AttnCfg<128>::kSmem, st, pdl, tm_kv, aa));
    SUN_CUDA(launch(attn_combine_kernel<128>, dim3(d.n_q_heads, batch), dim3(128), 0, st, pdl, aa));
  } else {
    SUN_CUDA(launch(attn_decode_kernel<64>, grid, dim3(128), AttnCfg<64>::kSmem, st, pdl, tm_kv, aa));
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
  init_kernel_attrs();
  SunDecoder* dec = new SunDecoder();
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
  dec->gemm_part = reinterpret_cast<float*>(ws + dec->L.gemm_part);
  dec->counters = reinterpret_cast<unsigned*>(ws + dec->L.counters);
  dec->amax_val = reinterpret_cast<float*>(ws + dec->L.amax_val);
  dec->amax_idx = reinterpret_cast<int*>(ws + dec->L.amax_idx);
  dec->logits = reinterpret_cast<float*>(ws + dec->L.logits);

  const SunDecoderDims& d = *dims;
  const int qd = d.n_q_heads * d.head_dim;
  dec->p_qkv = plan_gemm(qkv_rows(d), d.hidden);
  dec->p_o = plan_gemm(d.hidden, qd);
  dec->p_gu = plan_gemm(gu_rows(d), d.hidden);
  dec->p_down = plan_gemm(d.hidden, d.ffn);
  dec->p_lm = plan_gemm(d.vocab, d.hidden);
  if ((st = make_map_kv(&dec->tm_kv, d, *kv)) != SUN_OK) { delete dec; return st; }
  if (d.weight_bits == 16) {
    dec->tm_qkv.resize(d.n_layers);
    dec->tm_o.resize(d.n_layers);
    dec->tm_gu.resize(d.n_layers);
    dec->tm_down.resize(d.n_layers);
    for (int l = 0; l < d.n_layers; ++l) {
      const SunLayerWeights& lw = dec->layers[l];
      if ((st = make_map_2d(&dec->tm_qkv[l], lw.w_qkv, qkv_rows(d), d.hidden, d.hidden, kTileM)) != SUN_OK ||
          (st = make_map_2d(&dec->tm_o[l], lw.w_o, d.hidden, qd, qd, kTileM)) != SUN_OK ||
          (st = make_map_2d(&dec->tm_gu[l], lw.w_gate_up, gu_rows(d), d.hidden, d.hidden, kTileM)) != SUN_OK ||
          (st = make_map_2d(&dec->tm_down[l], lw.w_down, d.hidden, d.ffn, d.ffn, kTileM)) != SUN_OK) {
        delete dec;
        return st;
      }
    }
  }
  if ((st = make_map_2d(&dec->tm_lm, weights->lm_head, d.vocab, d.hidden, d.hidden, kTileM)) != SUN_OK) {
    delete dec;
    return st;
  }
  cudaError_t e = cudaMemset(ws + dec->L.counters, 0, size_t(std::max(dec->p_lm.m_tiles, 1)) * 4);
  if (e != cudaSuccess) {
    delete dec;
    return fail(SUN_ERR_CUDA, "cudaMemset counters: %s", cudaGetErrorString(e));
  }
  // zero the padded activation rows once (rows >= batch are never written)
  e = cudaMemset(ws, 0, dec->L.part_o);
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
  const int bn = round16(batch);
  XMaps* xm = nullptr;
  SunStatus s;
  if ((s = get_xmaps(dec, bn, &xm)) != SUN_OK) return s;
  const int qd = d.n_q_heads * d.head_dim;
  const int max_pages = (d.max_context + kPageTokens - 1) / kPageTokens;
  const int pps = pages_per_split > 0 ? std::min(pages_per_split, max_pages) : auto_pages_per_split(d, batch);
  float* lg = logits ? logits : dec->logits;

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

  // embedding gather + first attention RMSNorm
  SUN_CUDA(launch(rmsnorm_kernel, dim3(batch), dim3(kRowThreads), 0, st, pdl, tokens,
                  static_cast<const __nv_bfloat16*>(dec->w.embed), dec->resid,
                  static_cast<const __nv_bfloat16*>(dec->layers[0].attn_norm), dec->xn, d.hidden,
                  (long long)d.hidden, d.rms_eps));
  for (int l = 0; l < d.n_layers; ++l) {
    const SunLayerWeights& lw = dec->layers[l];
    if (l > 0)
      SUN_CUDA(launch(rmsnorm_kernel, dim3(batch), dim3(kRowThreads), 0, st, pdl, (const int*)nullptr,
                      (const __nv_bfloat16*)nullptr, dec->resid, static_cast<const __nv_bfloat16*>(lw.attn_norm),
                      dec->xn, d.hidden, (long long)d.hidden, d.rms_eps));
    // QKV + bias + RoPE + KV append
    GemmArgs a = base_args(dec->p_qkv, qkv_rows(d), d.hidden, batch, bn, dec->gemm_part, dec->counters);
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
    if (d.weight_bits == 16) s = run_gemm<EPI_QKV_ROPE>(dec->tm_qkv[l], xm->xn, a, dec->p_qkv, st, pdl);
    else s = run_gemm_w4<EPI_QKV_ROPE>(W4Weights{lw.w_qkv, lw.s_qkv}, xm->xn, a, dec->p_qkv, st, pdl);
    if (s != SUN_OK) return s;
    // paged attention
    aa.layer = l;
    if ((s = run_attention(d, dec->tm_kv, aa, batch, st, pdl)) != SUN_OK) return s;
    // O projection + residual
    a = base_args(dec->p_o, d.hidden, qd, batch, bn, dec->gemm_part, dec->counters);
    a.out_f32 = dec->resid;
    a.ldo = d.hidden;
    if (d.weight_bits == 16) s = run_gemm<EPI_RESID_ADD>(dec->tm_o[l], xm->attn, a, dec->p_o, st, pdl);
    else s = run_gemm_w4<EPI_RESID_ADD>(W4Weights{lw.w_o, lw.s_o}, xm->attn, a, dec->p_o, st, pdl);
    if (s != SUN_OK) return s;
    // FFN RMSNorm
    SUN_CUDA(launch(rmsnorm_kernel, dim3(batch), dim3(kRowThreads), 0, st, pdl, (const int*)nullptr,
                    (const __nv_bfloat16*)nullptr, dec->resid, static_cast<const __nv_bfloat16*>(lw.ffn_norm),
                    dec->xn, d.hidden, (long long)d.hidden, d.rms_eps));
    // gate/up + SwiGLU
    a = base_args(dec->p_gu, gu_rows(d), d.hidden, batch, bn, dec->gemm_part, dec->counters);
    a.out_bf16 = dec->act;
    a.ldb = d.ffn;
    a.n_valid_out = d.ffn;
    if (d.weight_bits == 16) s = run_gemm<EPI_SWIGLU>(dec->tm_gu[l], xm->xn, a, dec->p_gu, st, pdl);
    else s = run_gemm_w4<EPI_SWIGLU>(W4Weights{lw.w_gate_up, lw.s_gate_up}, xm->xn, a, dec->p_gu, st, pdl);
    if (s != SUN_OK) return s;
    // down + residual
    a = base_args(dec->p_down, d.hidden, d.ffn, batch, bn, dec->gemm_part, dec->counters);
    a.out_f32 = dec->resid;
    a.ldo = d.hidden;
    if (d.weight_bits == 16) s = run_gemm<EPI_RESID_ADD>(dec->tm_down[l], xm->act, a, dec->p_down, st, pdl);
    else s = run_gemm_w4<EPI_RESID_ADD>(W4Weights{lw.w_down, lw.s_down}, xm->act, a, dec->p_down, st, pdl);
    if (s != SUN_OK) return s;
  }
  // final norm, lm_head (+ argmax partials), greedy sampling
  SUN_CUDA(launch(rmsnorm_kernel, dim3(batch), dim3(kRowThreads), 0, st, pdl, (const int*)nullptr,
                  (const __nv_bfloat16*)nullptr, dec->resid, static_cast<const __nv_bfloat16*>(dec->w.final_norm),
                  dec->xn, d.hidden, (long long)d.hidden, d.rms_eps));
  GemmArgs a = base_args(dec->p_lm, d.vocab, d.hidden, batch, bn, dec->gemm_part, dec->counters);
  a.out_f32 = lg;
  a.ldo = d.vocab;
  a.amax_val = dec->amax_val;
  a.amax_idx = dec->amax_idx;
  if ((s = run_gemm<EPI_LOGITS>(dec->tm_lm, xm->xn, a, dec->p_lm, st, pdl)) != SUN_OK) return s;
  SUN_CUDA(launch(argmax_reduce_kernel, dim3(batch), dim3(kRowThreads), 0, st, pdl, (const float*)dec->amax_val,
                  (const int*)dec->amax_idx, dec->p_lm.m_tiles, bn, next_tokens,
                  (flags & SUN_STEP_FEEDBACK) ? const_cast<int*>(tokens) : (int*)nullptr,
                  const_cast<int*>(positions)));
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
                                next_tokens, 0, stream);
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

SunStatus sun_gemm_workspace_bytes(int64_t n_out, int64_t k, int32_t batch, size_t* bytes) {
  if (n_out < 1 || k < 1 || batch < 1 || batch > 256) return fail(SUN_ERR_VALUE, "bad gemm shape");
  GemmPlan p = plan_gemm(n_out, k);
  const int bn = round16(batch);
  *bytes = align_up(size_t(p.m_tiles) * 4, 1024) + size_t(p.m_tiles) * p.splits * bn * kTileM * 4;
  return SUN_OK;
}

SunStatus sun_gemm_bf16(const void* w, int64_t n_out, int64_t k, const void* x, int64_t ldx, int64_t x_rows,
                        int32_t batch, float* out, int64_t ldo, int32_t accumulate, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (batch < 1) return fail(SUN_ERR_VALUE, "empty batch");
  size_t need = 0;
  SunStatus s = sun_gemm_workspace_bytes(n_out, k, batch, &need);
  if (s != SUN_OK) return s;
  if (workspace_bytes < need) return fail(SUN_ERR_CAPACITY, "gemm workspace too small");
  const int bn = round16(batch);
  if (x_rows < bn) return fail(SUN_ERR_VALUE, "x must have >= round_up(batch,16) rows");
  init_kernel_attrs();
  GemmPlan p = plan_gemm(n_out, k);
  CUtensorMap tw, tx;
  if ((s = make_map_2d(&tw, w, n_out, k, k, kTileM)) != SUN_OK) return s;
  if ((s = make_map_2d(&tx, x, x_rows, k, ldx, bn)) != SUN_OK) return s;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  unsigned* counters = reinterpret_cast<unsigned*>(ws);
  float* part = reinterpret_cast<float*>(ws + align_up(size_t(p.m_tiles) * 4, 1024));
  GemmArgs a = base_args(p, n_out, k, batch, bn, part, counters);
  a.out_f32 = out;
  a.ldo = ldo;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (accumulate) return run_gemm<EPI_RESID_ADD>(tw, tx, a, p, st, false);
  return run_gemm<EPI_STORE_F32>(tw, tx, a, p, st, false);
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
  if (workspace_bytes < align_up(po, 1024) + pm) return fail(SUN_ERR_CAPACITY, "attention workspace too small");
  aa.part_o = static_cast<float*>(workspace);
  aa.part_ml = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + align_up(po, 1024));
  aa.out = static_cast<__nv_bfloat16*>(out);
  aa.ld_out = d.n_q_heads * d.head_dim;
  CUtensorMap tm;
  if ((s = make_map_kv(&tm, d, *kv)) != SUN_OK) return s;
  return run_attention(d, tm, aa, batch, static_cast<cudaStream_t>(stream), false);
}

SunStatus sun_rmsnorm(const float* x, const void* w, void* y, int32_t batch, int32_t h, float eps, void* stream) {
  if (batch < 1 || h % 4 != 0) return fail(SUN_ERR_VALUE, "bad rmsnorm shape");
  SUN_CUDA(launch(rmsnorm_kernel, dim3(batch), dim3(kRowThreads), 0, static_cast<cudaStream_t>(stream), false,
                  (const int*)nullptr, (const __nv_bfloat16*)nullptr, const_cast<float*>(x),
                  static_cast<const __nv_bfloat16*>(w), static_cast<__nv_bfloat16*>(y), h, (long long)h, eps));
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

}  // extern "C"
