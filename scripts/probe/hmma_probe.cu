// Microbenchmark: legacy tensor path (mma.sync m16n8k16 bf16 -> fp32) throughput on
// this GPU: independent HMMA chains per warp, 1-16 warps per SM, 148 CTAs.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

template <int CHAINS>
__global__ void hmma_kernel(int iters, float* sink) {
  float d[CHAINS][4];
  for (int c = 0; c < CHAINS; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.f;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3f80, b1 = a0 ^ 0x3f00;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
void run(int warps) {
  float* sink;
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 4096;
  hmma_kernel<CHAINS><<<148, warps * 32>>>(16, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  hmma_kernel<CHAINS><<<148, warps * 32>>>(iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n = double(iters) * CHAINS * warps;  // HMMAs per SM
  const double cyc = ms * 1e-3 * 1.965e9;
  printf("chains %2d warps/SM %2d: %.2f cycles per HMMA per SM (%.1f per sub-partition), %.0f TFLOP/s (%s)\n", CHAINS,
         warps, cyc / n, cyc / n * 4, n * 148 * 4096 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

int main() {
  for (int w : {1, 4, 8, 16}) run<1>(w);
  for (int w : {1, 4, 8, 16}) run<4>(w);
  for (int w : {4, 8, 16}) run<8>(w);
  return 0;
}
