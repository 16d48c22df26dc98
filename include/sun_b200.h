/*
 * sun_b200.h — C ABI of the B200-native SUN shared decode path.
 *
 * The reference (arxiv 2603.02599 "SUN", code: poolsim) has no FFI: its decode
 * step is the analytic price `decode_step_time[_from_totals]`
 * (/root/reference/pkg/src/poolsim/costmodel.py:101-140) called once per step
 * from the decode worker (engine.py:427-429), and the KV hand-off is the
 * `KvHandle` value object (domain.py:96-113). This library is the real thing
 * behind those two extension points: the decode module's step on one B200, and
 * the paged KV pool the hand-off writes into. The Python mirror of the reference
 * API (paper_2603_02599_b200/) binds these symbols with ctypes; see
 * INTEGRATION.md for the binding a poolsim maintainer would add.
 *
 * Conventions
 *  - plain pointers and sizes only; every device buffer is caller-owned
 *    (torch allocates), the library never allocates on the step path;
 *  - calls are asynchronous on the given stream (`void*` = cudaStream_t) and
 *    graph-capturable; a decoder's workspace is not re-entrant — one decoder
 *    per decode worker / GPU, as each poolsim decode worker owns one GPU;
 *  - status codes map 1:1 onto the reference's exceptions (see SunStatus).
 */
#ifndef SUN_B200_H
#define SUN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SUN_ABI_VERSION 2

/* Error bits of a decoder's device error word (sun_decoder_status). Every step
 * validates its inputs on the device before any KV write: a bad token reads
 * embedding row 0, a bad position is clamped and its KV append skipped, an
 * out-of-range page is never written (attention reads it as zeros through the
 * TMA bounds), so a bad block table cannot corrupt another sequence's KV. */
#define SUN_STEP_ERR_TOKEN 1u    /* token outside [0, vocab)                                */
#define SUN_STEP_ERR_POSITION 2u /* position outside [0, max_context)                       */
#define SUN_STEP_ERR_PAGE 4u     /* a block-table entry for pages 0..pos/16 outside the pool */
#define SUN_STEP_ERR_NAN 8u      /* a row's logits had no finite maximum (argmax -> 0)      */

typedef enum SunStatus {
  SUN_OK = 0,
  SUN_ERR_VALUE = 1,         /* ValueError: empty batch (costmodel.py:130-131), bad sizes   */
  SUN_ERR_MIXED_DECODER = 2, /* MixedDecoderError: decoder geometry mismatch (costmodel.py:132-138,
                                shared-decoder invariant domain.py:266-279)                    */
  SUN_ERR_UNSUPPORTED = 3,   /* shape outside what the sm_100a kernels implement               */
  SUN_ERR_CUDA = 4,          /* CUDA runtime / driver failure (message via sun_last_error)      */
  SUN_ERR_CAPACITY = 5       /* workspace or KV pool too small (engine.py:394-401 OVER_CAPACITY) */
} SunStatus;

/* Geometry of the frozen shared decode module θ_d (Eq. 3). Every
 * task-specific prefill module θ_p^τ that feeds this decoder must produce KV
 * with the same (n_layers, n_kv_heads, head_dim, RoPE) — the analogue of the
 * reference's "shared_decoder models agree on decode bits and param_count". */
typedef struct SunDecoderDims {
  int32_t vocab;
  int32_t hidden;
  int32_t n_layers;
  int32_t n_q_heads;
  int32_t n_kv_heads;
  int32_t head_dim;    /* 64 or 128 */
  int32_t ffn;         /* SwiGLU width f */
  int32_t page_size;   /* tokens per KV page; 16 */
  int32_t max_context; /* tokens per sequence upper bound (rope table rows) */
  int32_t weight_bits; /* 16 = bf16; 4 = QSUN W4A16 (int4 symmetric, bf16 scale per group) */
  int32_t group_size;  /* 128 when weight_bits == 4 */
  int32_t qkv_bias;    /* 1 if the QKV projection has a bias (Qwen2.5) */
  float rms_eps;
  float rope_theta;    /* RoPE base of the K cache this decoder reads and writes */
} SunDecoderDims;

/* SUN-BLK weight layout (bf16 linear layers and the lm_head as passed to the
 * decoder and sun_gemm_bf16): W[rows][k] is stored as [ceil(rows/128)]
 * [ceil(k/64)] blocks of 128 x 64 elements, each block 16 KB contiguous with the
 * 16-byte chunk c of row r at chunk position c ^ (r & 7) (the SWIZZLE_128B shared
 * memory image), zero padded. Every pipeline stage is then one linear bulk copy. */
SunStatus sun_blocked_bytes(int64_t rows, int64_t k, size_t* bytes);
SunStatus sun_block_weights_bf16(const void* w, int64_t rows, int64_t k, void* out, void* stream);

/* Device pointers of one decoder layer (bf16 unless stated; matrices in SUN-BLK).
 *  w_qkv      [(nq + 2 nkv) * d][hidden]           rows: q heads, k heads, v heads
 *  w_o        [hidden][nq * d]
 *  w_gate_up  [ceil(f/64) * 128][hidden]           64-row blocks: gate rows j..j+63 then
 *                                                  up rows j..j+63 (zero rows pad f)
 *  w_down     [hidden][f]
 * For weight_bits == 4, w_* hold SUN-W4 packed int4 (8 KB per 128-row x 128-k block,
 * blocks [row tile][K block], each [4 chunks of 32 k][128 rows][16 B], offset-binary
 * nibbles in order [0,2,4,6,1,3,5,7] per 8-k word) and s_* the bf16 group scales
 * tile-major [row tile][K/128][128] (oracle/quant_ref.py restates both). */
typedef struct SunLayerWeights {
  const void* attn_norm;
  const void* w_qkv;
  const void* s_qkv;
  const void* b_qkv;
  const void* w_o;
  const void* s_o;
  const void* ffn_norm;
  const void* w_gate_up;
  const void* s_gate_up;
  const void* w_down;
  const void* s_down;
} SunLayerWeights;

typedef struct SunWeights {
  const void* embed;       /* [vocab][hidden] */
  const void* final_norm;  /* [hidden] */
  const void* lm_head;     /* [vocab][hidden] SUN-BLK, bf16 always */
  const float* rope_cos;   /* [max_context][head_dim/2] fp32 */
  const float* rope_sin;
  const SunLayerWeights* layers; /* host array, n_layers entries */
} SunWeights;

/* Paged KV pool shared by every prefill module (decoder-compatible by
 * construction). Page p holds page_size consecutive tokens of
 * one sequence for all layers: [n_layers][2 (K,V)][n_kv_heads][page_size][head_dim]
 * bf16; K is stored after RoPE. A sequence's pages are listed in its block-table
 * row (the physical form of KvHandle, domain.py:96-113).
 * The pool records the KV geometry it was laid out for: every decoder created over
 * it (the shared decode module and each task prefill module) and every hand-off
 * copy into it must match, else SUN_ERR_MIXED_DECODER — the device-side form of the
 * reference's shared-decoder invariant (domain.py:266-279, costmodel.py:132-138). */
typedef struct SunKvPool {
  void* base;
  int64_t num_pages;
  int32_t n_layers;
  int32_t n_kv_heads;
  int32_t head_dim;
  int32_t page_size;
  float rope_theta;
  int32_t device;      /* CUDA device ordinal the pages live on */
} SunKvPool;

/* Bytes of one page of a pool with this geometry. */
SunStatus sun_kv_page_bytes(const SunKvPool* kv, size_t* bytes);

typedef struct SunDecoder SunDecoder;

int32_t sun_abi_version(void);
const char* sun_last_error(void);

/* Bytes of device workspace a decoder needs for batches up to max_batch. */
SunStatus sun_decoder_workspace_bytes(const SunDecoderDims* dims, int32_t max_batch, size_t* bytes);

/* Build a decoder over caller-owned weights, KV pool and (zeroed) workspace.
 * Encodes every TMA descriptor once. Replaces poolsim's per-worker
 * `_DecodeWorker(weight_bytes, capacity)` (engine.py:148-212). */
SunStatus sun_decoder_create(const SunDecoderDims* dims, const SunWeights* weights, const SunKvPool* kv,
                             void* workspace, size_t workspace_bytes, int32_t max_batch, int32_t use_pdl,
                             SunDecoder** out);
SunStatus sun_decoder_destroy(SunDecoder* dec);

/* One decode step of the shared decode module D_θd (Eq. 3) over a
 * mixed-model batch: for each member b, consume tokens[b] at position
 * positions[b] (= resident KV tokens before the step), append its K/V into the
 * page block_tables[b*bt_stride + positions[b]/page_size], attend over
 * positions[b]+1 tokens, and write next_tokens[b] = argmax logits (greedy).
 * logits (fp32 [batch][vocab]) may be NULL (an internal buffer is used).
 * pages_per_split: attention split-K granularity in pages (0 = automatic).
 * This is the operator that replaces costmodel.decode_step_time_from_totals
 * at engine.py:427-429. Errors: batch < 1 -> SUN_ERR_VALUE. */
#define SUN_STEP_FEEDBACK 1 /* flags: also write tokens[b] = next_tokens[b], positions[b] += 1 on device */
/* flags: every row is a different sequence (a decode batch; not token-parallel prefill
 * rows of one prompt): the step's KV append then touches only each row's last page,
 * so the attention stages the other pages while the QKV kernel is still finishing */
#define SUN_STEP_DISTINCT_ROWS 2 /* (also selects the persistent layer GEMM chain — bf16, and
                                     QSUN for batches up to 128 — which needs the whole GPU: one
                                     such step in flight per GPU) */
SunStatus sun_decode_step(SunDecoder* dec, const int32_t* tokens, const int32_t* positions,
                          const int32_t* block_tables, int32_t bt_stride, int32_t batch,
                          int32_t pages_per_split, float* logits, int32_t* next_tokens, int32_t flags,
                          void* stream);

/* Same step (rows distinct), serialised, with a CUDA event after every kernel: kernel_ms[i] is the
 * device time of the i-th launch (order: embed+norm, then per layer qkv, attention
 * [combine], o, gate_up, down — or, with the bf16 layer chain, qkv once and then per
 * layer attention [combine], chain; lm_head, argmax).
 * Synchronises the stream. For measurement only. */
/* sun_decode_step whose rows are grouped for the attention (token-parallel
 * prefill, PrefillModule): group g is rows [group_start[g], group_start[g] +
 * group_len[g]) — positions of ONE sequence, ascending, same block-table row,
 * at most 16 / (n_q_heads / n_kv_heads) rows — and its KV pages are staged once
 * for all of them. group_start / group_len are DEVICE int32 arrays [n_groups]
 * covering every row. Same results as sun_decode_step. */
SunStatus sun_decode_step_grouped(SunDecoder* dec, const int32_t* tokens, const int32_t* positions,
                                  const int32_t* block_tables, int32_t bt_stride, int32_t batch,
                                  int32_t pages_per_split, float* logits, int32_t* next_tokens, int32_t flags,
                                  void* stream, const int32_t* group_start, const int32_t* group_len,
                                  int32_t n_groups);

SunStatus sun_decode_step_profile(SunDecoder* dec, const int32_t* tokens, const int32_t* positions,
                                  const int32_t* block_tables, int32_t bt_stride, int32_t batch,
                                  int32_t pages_per_split, float* logits, int32_t* next_tokens, void* stream,
                                  float* kernel_ms, int32_t capacity, int32_t* n_kernels);

/* One sun_decode_step (PDL as configured, not serialised, rows distinct) with a device-side
 * timeline of its GEMM and attention launches: timeline is a DEVICE uint64 array
 * [capacity][2] pre-filled with (~0, 0); launch i records the earliest CTA start
 * and the latest CTA end (%globaltimer ns). If stamps is non-null and launch
 * stamp_launch is a GEMM, its CTAs also write sun_gemm_bf16_stamped's per-CTA
 * phase stamps there ([grid][16]). Profiling only. */
SunStatus sun_decode_step_timeline(SunDecoder* dec, const int32_t* tokens, const int32_t* positions,
                                   const int32_t* block_tables, int32_t bt_stride, int32_t batch,
                                   int32_t pages_per_split, int32_t* next_tokens, void* stream, uint64_t* timeline,
                                   int32_t capacity, int32_t* n_launches, uint64_t* stamps, int32_t stamp_launch);

/* Number of kernels this thread has launched through the library so far. */
SunStatus sun_launch_count(int64_t* launches);

/* Read (and, if clear != 0, reset) the decoder's device error word: the OR of the
 * SUN_STEP_ERR_* bits raised by the steps since the last clear. Synchronises the
 * stream. *flags == 0: every step's inputs were valid. */
SunStatus sun_decoder_status(SunDecoder* dec, uint32_t* flags, int32_t clear, void* stream);

/* Whether sun_decode_step runs the persistent layer GEMM chain for these flags on
 * this decoder (SUN_STEP_DISTINCT_ROWS, and a grid that fits this device's SMs
 * co-resident — checked with the occupancy API at create; QSUN decoders: for batches
 * up to 128, larger ones use separate GEMM launches). */
SunStatus sun_decoder_uses_chain(SunDecoder* dec, int32_t flags, int32_t* uses_chain);

/* ---- K8: prefill -> decode KV hand-off by peer copy (replaces transfer_time,
 * costmodel.py:148-155; the transfer window engine.py:345-392) ----
 * The decode worker exports its pool once; a prefill worker in another process
 * (any GPU of the node, or the same GPU) imports it and copies a request's pages
 * straight into the pages the decode worker reserved, with the copy engines:
 * NVLink 5 / NVSwitch between GPUs, HBM within one. No SMs are taken from a
 * decode step running concurrently (its persistent layer chain needs the whole
 * GPU), unlike a kernel-based transport. */
typedef struct SunKvPoolHandle {
  uint8_t ipc[64];     /* cudaIpcMemHandle_t of the allocation holding the pages */
  int64_t offset;      /* byte offset of page 0 inside that allocation          */
  SunKvPool geometry;  /* base = NULL; num_pages, KV geometry, device             */
} SunKvPoolHandle;
SunStatus sun_kv_pool_export(const SunKvPool* kv, SunKvPoolHandle* out);
/* Map an exported pool into this process (peer access enabled when it lives on
 * another device); *out is a pool whose base is valid here. */
SunStatus sun_kv_pool_import(const SunKvPoolHandle* handle, SunKvPool* out);
SunStatus sun_kv_pool_close(SunKvPool* imported);
/* Copy n_pages pages src_pages[i] of src into dst_pages[i] of dst (host int32
 * arrays; consecutive runs on both sides become one copy each), asynchronously on
 * stream. The pools' KV geometries must match (else SUN_ERR_MIXED_DECODER). */
SunStatus sun_kv_handoff_copy(const SunKvPool* src, const int32_t* src_pages, const SunKvPool* dst,
                              const int32_t* dst_pages, int32_t n_pages, void* stream);

/* ---- kernel-level entry points (unit parity tests; same kernels as the step) ---- */

/* out[b][n] (=|+=) sum_k w[n][k] * x[b][k] for b < batch, bf16 in (w in SUN-BLK),
 * fp32 out, tcgen05 swap-AB GEMM. x has x_rows >= round_up(batch,16) allocated rows of
 * stride ldx elements. workspace >= sun_gemm_workspace_bytes(...), zeroed once. */
SunStatus sun_gemm_workspace_bytes(int64_t n_out, int64_t k, int32_t batch, size_t* bytes);
SunStatus sun_gemm_bf16(const void* w, int64_t n_out, int64_t k, const void* x, int64_t ldx, int64_t x_rows,
                        int32_t batch, float* out, int64_t ldo, int32_t accumulate, void* workspace,
                        size_t workspace_bytes, void* stream);

/* sun_gemm_bf16 with per-CTA %globaltimer stamps (stamps: uint64 [grid][16]; slots:
 * 0 start, 1 setup done, 2 first stage landed, 3 last MMA issued, 4 first
 * accumulator ready, 5 epilogue done, 6 exit, 8-11 cluster reduction phases). Profiling aid. */
SunStatus sun_gemm_bf16_stamped(const void* w, int64_t n_out, int64_t k, const void* x, int64_t ldx,
                                int64_t x_rows, int32_t batch, float* out, int64_t ldo, int32_t accumulate,
                                void* workspace, size_t workspace_bytes, void* stream, uint64_t* stamps);

/* Same with QSUN SUN-W4 weights (packed int4 + bf16 group scales, see gemm_w4.cuh),
 * dequantised in-kernel to bf16 tcgen05 operands. k must be a multiple of 128. */
SunStatus sun_gemm_w4(const void* packed, const void* scales, int64_t n_out, int64_t k, const void* x, int64_t ldx,
                      int64_t x_rows, int32_t batch, float* out, int64_t ldo, int32_t accumulate, void* workspace,
                      size_t workspace_bytes, void* stream);
/* Small-batch QSUN GEMV (batch <= 16): the same SUN-W4 operands on the legacy
 * tensor path (m16n8k16) with in-register dequantisation and a stream-K grid —
 * the kernel QSUN decode steps of <= 8 rows run (gemm_w4.cuh gemv_w4_kernel).
 * Result = sum over 128-k groups of s * sum(q * x) (fp32). */
SunStatus sun_gemv_w4(const void* packed, const void* scales, int64_t n_out, int64_t k, const void* x, int64_t ldx,
                      int64_t x_rows, int32_t batch, float* out, int64_t ldo, int32_t accumulate, void* workspace,
                      size_t workspace_bytes, void* stream);
/* sun_gemv_w4 (store) with per-CTA %globaltimer stamps [grid][16] (profiling only; 0 start,
 * 1 setup done, 2 first stage landed, 3 last stage consumed, 5 last epilogue done, 6 exit). */
SunStatus sun_gemv_w4_stamped(const void* packed, const void* scales, int64_t n_out, int64_t k, const void* x,
                              int64_t ldx, int64_t x_rows, int32_t batch, float* out, int64_t ldo, void* workspace,
                              size_t workspace_bytes, void* stream, uint64_t* stamps);
/* sun_gemm_w4 (store) with per-CTA %globaltimer stamps [grid][16] (profiling only;
 * slots as sun_gemm_bf16_stamped). */
SunStatus sun_gemm_w4_stamped(const void* packed, const void* scales, int64_t n_out, int64_t k, const void* x,
                              int64_t ldx, int64_t x_rows, int32_t batch, float* out, int64_t ldo, void* workspace,
                              size_t workspace_bytes, void* stream, uint64_t* stamps);

/* Paged split-K decode attention for one layer: q bf16 [batch][nq][d] (post-RoPE),
 * KV from the pool, out bf16 [batch][nq*d]. */
SunStatus sun_attention_decode(const SunDecoderDims* dims, const SunKvPool* kv, int32_t layer, const void* q,
                               const int32_t* positions, const int32_t* block_tables, int32_t bt_stride,
                               int32_t batch, int32_t pages_per_split, void* out, void* workspace,
                               size_t workspace_bytes, void* stream);

/* y[b] = bf16(x[b] * rsqrt(mean(x[b]^2) + eps) * w), x fp32 [batch][h]. */
SunStatus sun_rmsnorm(const float* x, const void* w, void* y, int32_t batch, int32_t h, float eps, void* stream);

/* QSUN: quantize bf16 W[rows][K] to SUN-W4 packed int4 + bf16 scales (group 128
 * along K), symmetric, q = clamp(round_half_even(w / s), -8, 7), s = bf16(amax / 7.5);
 * packed must be zeroed (padding rows are not written). */
SunStatus sun_quantize_w4(const void* w, int64_t rows, int64_t k, int32_t group, void* packed, void* scales,
                          void* stream);

/* QSUN checkpoint import: a compressed-tensors "pack-quantized" W4A16 tensor
 * (weight_packed int32 [rows][K/8], element 8j+i of a row in nibble i of word j as
 * q + 8; weight_scale bf16 [rows][K/128]; symmetric, group 128) re-laid out to
 * SUN-W4 without touching q or s. packed must be zeroed (padding rows are not
 * written). Replaces the quantisation step of QSUN's offline pipeline
 * (LLM Compressor AWQ checkpoint -> vLLM) on the load side. */
SunStatus sun_import_w4_ct(const void* ct_packed, const void* ct_scales, int64_t rows, int64_t k, int32_t group,
                           void* packed, void* scales, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SUN_B200_H */
