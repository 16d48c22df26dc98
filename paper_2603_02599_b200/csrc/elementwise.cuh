// elementwise.cuh — row kernels of the decode step: embedding gather fused with
// the first RMSNorm, RMSNorm producing the bf16 GEMM operand, and the final
// greedy argmax over the lm_head tiles' (max, index) partials.
#pragma once
#include "../../include/sun_b200.h"  // SUN_STEP_ERR_* bits
#include "gemm_tc.cuh"  // act_offset (SUN-ACT layout)

namespace sun {

constexpr int kRowThreads = 256;

// What embed_norm_kernel validates at the start of a step (SUN_STEP_ERR_* bits of
// include/sun_b200.h into err).
struct StepCheck {
  const int* positions;
  const int* block_tables;
  int bt_stride;
  int vocab;
  int max_ctx;
  long long num_pages;
  unsigned* err;
};

SUN_DEVICE float block_sum(float v, float* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// y = bf16(x * rsqrt(mean(x^2) + eps) * w), fp32 math, one rounding.
// If `tokens` is non-null the row is first gathered from the embedding table
// into the fp32 residual stream (x := float(embed[token])).
// act_rows > 0: the output goes to the SUN-ACT layout the GEMMs stream
// (gemm_tc.cuh), otherwise row-major with stride ld_out.
__global__ void __launch_bounds__(kRowThreads)
    rmsnorm_kernel(const int* __restrict__ tokens, const __nv_bfloat16* __restrict__ embed,
                   float* __restrict__ resid, const __nv_bfloat16* __restrict__ w,
                   __nv_bfloat16* __restrict__ out, int h, long long ld_out, float eps, int act_rows) {
  __shared__ float red[kRowThreads / 32];
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.x;
  float* x = resid + static_cast<long long>(b) * h;
  if (tokens != nullptr) {
    const __nv_bfloat16* e = embed + static_cast<long long>(tokens[b]) * h;
    for (int i = threadIdx.x * 2; i < h; i += kRowThreads * 2) {
      const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(e + i);
      x[i] = __bfloat162float(v.x);
      x[i + 1] = __bfloat162float(v.y);
    }
    __syncthreads();
  }
  float ss = 0.f;
  for (int i = threadIdx.x * 4; i < h; i += kRowThreads * 4) {
    const float4 v = *reinterpret_cast<const float4*>(x + i);
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  const float tot = block_sum(ss, red);
  const float r = rsqrtf(tot / static_cast<float>(h) + eps);
  __nv_bfloat16* y = out + static_cast<long long>(b) * ld_out;
  for (int i = threadIdx.x * 4; i < h; i += kRowThreads * 4) {
    const float4 v = *reinterpret_cast<const float4*>(x + i);
    const __nv_bfloat162 w01 = *reinterpret_cast<const __nv_bfloat162*>(w + i);
    const __nv_bfloat162 w23 = *reinterpret_cast<const __nv_bfloat162*>(w + i + 2);
    __nv_bfloat162 o01 = __floats2bfloat162_rn(v.x * r * __bfloat162float(w01.x), v.y * r * __bfloat162float(w01.y));
    __nv_bfloat162 o23 = __floats2bfloat162_rn(v.z * r * __bfloat162float(w23.x), v.w * r * __bfloat162float(w23.y));
    __nv_bfloat16* dst = act_rows > 0 ? reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(out) +
                                                                         act_offset(b, i, act_rows))
                                      : y + i;
    *reinterpret_cast<__nv_bfloat162*>(dst) = o01;  // 4 consecutive columns stay in one 16-byte chunk
    *reinterpret_cast<__nv_bfloat162*>(dst + 2) = o23;
  }
}

// Embedding gather fused with the first (factored) RMSNorm: resid = embed[tok],
// xg = bf16(resid * g) in SUN-ACT, ss[0][b] = sum(resid^2) (other tiles 0); the
// QKV GEMM applies r_b = rsqrt(mean + eps) in its epilogue (see gemm_tc.cuh).
__global__ void __launch_bounds__(kRowThreads)
    embed_norm_kernel(const int* __restrict__ tokens, const __nv_bfloat16* __restrict__ embed,
                      float* __restrict__ resid, const __nv_bfloat16* __restrict__ g, __nv_bfloat16* __restrict__ xg,
                      float* __restrict__ ss, int h, int act_rows, int ss_tiles, StepCheck chk) {
  __shared__ float red[kRowThreads / 32];
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.x;
  // input validation (the step's error word, sun_decoder_status): a bad token reads
  // embedding row 0; bad positions / pages are clamped / skipped by the consumers
  int tok = tokens[b];
  const int pos = chk.positions[b];
  unsigned bits = 0;
  if (tok < 0 || tok >= chk.vocab) {
    bits |= SUN_STEP_ERR_TOKEN;
    tok = 0;
  }
  if (pos < 0 || pos >= chk.max_ctx) {
    bits |= SUN_STEP_ERR_POSITION;
  } else {
    const int* bt = chk.block_tables + static_cast<long long>(b) * chk.bt_stride;
    for (int j = threadIdx.x; j <= (pos >> 4); j += kRowThreads)
      if (bt[j] < 0 || static_cast<long long>(bt[j]) >= chk.num_pages) bits |= SUN_STEP_ERR_PAGE;
  }
  if (bits) atomicOr(chk.err, bits);
  const __nv_bfloat16* e = embed + static_cast<long long>(tok) * h;
  float* x = resid + static_cast<long long>(b) * h;
  float acc = 0.f;
  for (int i = threadIdx.x * 4; i < h; i += kRowThreads * 4) {
    const __nv_bfloat162 e01 = *reinterpret_cast<const __nv_bfloat162*>(e + i);
    const __nv_bfloat162 e23 = *reinterpret_cast<const __nv_bfloat162*>(e + i + 2);
    const float4 v = make_float4(__bfloat162float(e01.x), __bfloat162float(e01.y), __bfloat162float(e23.x),
                                 __bfloat162float(e23.y));
    *reinterpret_cast<float4*>(x + i) = v;
    acc += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    const __nv_bfloat162 g01 = *reinterpret_cast<const __nv_bfloat162*>(g + i);
    const __nv_bfloat162 g23 = *reinterpret_cast<const __nv_bfloat162*>(g + i + 2);
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(xg) + act_offset(b, i, act_rows));
    *reinterpret_cast<__nv_bfloat162*>(dst) =
        __floats2bfloat162_rn(v.x * __bfloat162float(g01.x), v.y * __bfloat162float(g01.y));
    *reinterpret_cast<__nv_bfloat162*>(dst + 2) =
        __floats2bfloat162_rn(v.z * __bfloat162float(g23.x), v.w * __bfloat162float(g23.y));
  }
  const float tot = block_sum(acc, red);
  if (threadIdx.x == 0) {
    ss[b] = tot;
    for (int t = 1; t < ss_tiles; ++t) ss[static_cast<long long>(t) * act_rows + b] = 0.f;
  }
}

// next[b] = argmax over lm_head tiles (ties -> lowest vocabulary index). With
// feedback, also tokens[b] = next[b] and positions[b] += 1 (graph-replayable loop).
__global__ void __launch_bounds__(kRowThreads)
    argmax_reduce_kernel(const float* __restrict__ val, const int* __restrict__ idx, int m_tiles, int bn,
                         int* __restrict__ next, int* __restrict__ feedback_tokens, int* __restrict__ positions,
                         unsigned* __restrict__ err) {
  __shared__ float sv[kRowThreads / 32];
  __shared__ int si[kRowThreads / 32];
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.x;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = threadIdx.x; t < m_tiles; t += kRowThreads) {
    const float v = val[static_cast<long long>(t) * bn + b];
    const int i = idx[static_cast<long long>(t) * bn + b];
    if (v > bv || (v == bv && i < bi)) {
      bv = v;
      bi = i;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kRowThreads / 32; ++w) {
      if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) {
        bv = sv[w];
        bi = si[w];
      }
    }
    if (bi == 0x7fffffff) {  // no finite maximum (NaN / -inf logits): token 0, flagged
      bi = 0;
      if (err != nullptr) atomicOr(err, SUN_STEP_ERR_NAN);
    }
    next[b] = bi;
    if (feedback_tokens != nullptr) {  // device-resident autoregressive loop
      feedback_tokens[b] = bi;
      positions[b] += 1;
    }
  }
}

}  // namespace sun
