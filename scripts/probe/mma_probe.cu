// mma_probe.cu — cycles per tcgen05.mma (cta_group::1, kind::f16, M=128, K=16) for
// N in {16..256}, A from shared memory vs A from tensor memory; one CTA per SM,
// 512 back-to-back MMAs into one accumulator. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_02599_b200/csrc \
//        -o scripts/probe/mma_probe scripts/probe/mma_probe.cu
#include <cstdio>
#include "sun_common.cuh"
using namespace sun;

__global__ void __launch_bounds__(128, 1) probe(int n, int a_tmem, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* A = base;             // 128 x 64 bf16 SW128 atom (16 KB)
  uint8_t* B = base + 16384;     // 256 x 64 bf16 (32 KB)
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *slot;
  const uint32_t idesc = make_idesc_bf16(128, n);
  long long t = 0;
  if (threadIdx.x < 32) {
    if (elect_one()) {
      const long long t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        const uint32_t kk = i & 3;
        if (a_tmem)
          umma_bf16_ta(tm, tm + 384 + kk * 8, make_sw128_desc(smem_u32(B) + kk * 32), idesc, i > 0);
        else
          umma_bf16(tm, make_sw128_desc(smem_u32(A) + kk * 32), make_sw128_desc(smem_u32(B) + kk * 32), idesc, i > 0);
      }
      umma_commit(bar);
      mbar_wait(bar, 0);
      t = clock64() - t0;
      out[blockIdx.x] = t;
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512)); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 1024 + 16384 + 32768 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int at = 0; at < 2; ++at)
    for (int n : {16, 32, 64, 128, 256}) {
      for (int rep = 0; rep < 2; ++rep) probe<<<148, 128, smem>>>(n, at, 1024, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("A=%s N=%3d: %.1f cycles/MMA (%s)\n", at ? "tmem" : "smem", n, avg / 1024, cudaGetErrorString(e));
    }
  return 0;
}
