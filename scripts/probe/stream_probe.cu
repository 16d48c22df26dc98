// Microbenchmark: how fast can each SM stream HBM into shared memory with
// cp.async.bulk / TMA under various (chunk, stages, CTAs/SM) settings.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2603_02599_b200/csrc/sun_common.cuh"
using namespace sun;

__global__ void stream_kernel(const uint8_t* src, long long bytes_per_cta, int chunk, int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * chunk);
  const uint8_t* base = src + blockIdx.x * bytes_per_cta;
  const long long n = bytes_per_cta / chunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    for (long long j = 0; j < n; ++j) {
      int s = j % stages;
      if (j >= stages) mbar_wait(&full[s], ((j / stages) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], chunk);
      bulk_load_hint(smem + s * chunk, base + j * chunk, chunk, &full[s], kEvictFirst);
    }
    for (long long j = n - stages > 0 ? n - stages : 0; j < n; ++j) mbar_wait(&full[j % stages], (j / stages) & 1);
    sink[blockIdx.x] = smem[5];
  }
}

int main() {
  const long long total = 2LL << 30;
  uint8_t* src; cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  unsigned long long* sink; cudaMalloc(&sink, 4096 * 8);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int configs[][3] = {{16384, 8, 148}, {16384, 12, 148}, {32768, 6, 148}, {65536, 3, 148}, {16384, 6, 296},
                      {8192, 24, 148}, {32768, 4, 296}, {16384, 4, 592}, {4096, 48, 148}};
  for (auto& c : configs) {
    int chunk = c[0], stages = c[1], ctas = c[2];
    long long per = (total / ctas) / chunk * chunk;
    size_t sm = size_t(stages) * chunk + 1024;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 2; ++w) stream_kernel<<<ctas, 32, sm>>>(src, per, chunk, stages, sink);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) stream_kernel<<<ctas, 32, sm>>>(src, per, chunk, stages, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double gbs = 5.0 * per * ctas / (ms / 1e3) / 1e9;
    printf("chunk %6d stages %2d ctas %3d (inflight/SM %4d KB): %7.0f GB/s  (%s)\n", chunk, stages, ctas,
           stages * chunk * (ctas / 148) / 1024, gbs, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
