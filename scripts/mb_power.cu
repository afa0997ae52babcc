// Power of plain TMA streaming (HBM -> smem, no compute) vs the sketch kernel: each CTA
// streams its share of a 32 GiB buffer through a 3 x 64 KB ring; run back to back ~2 s
// while nvidia-smi samples power (scripts/gpu_power_mb.sh).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(128, 1) k_stream(const char* src, size_t tiles, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 3 * 65536);
  if (threadIdx.x == 0) {
    for (int b = 0; b < 3; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + b)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  size_t f = 0;
  auto issue = [&](size_t t, int b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 65536;" ::"r"(su(bar + b)) : "memory");
    for (int k = 0; k < 4; ++k)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                       su(sm + b * 65536 + k * 16384)),
                   "l"(src + t * 65536 + k * 16384), "r"(su(bar + b))
                   : "memory");
  };
  if (threadIdx.x == 0)
    for (int b = 0; b < 3; ++b)
      if (blockIdx.x + (size_t)b * gridDim.x < tiles) issue(blockIdx.x + (size_t)b * gridDim.x, b);
  for (size_t t = blockIdx.x; t < tiles; t += gridDim.x, ++f) {
    const int b = (int)(f % 3);
    const uint32_t par = (uint32_t)((f / 3) & 1);
    asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(
                     su(bar + b)),
                 "r"(par)
                 : "memory");
    acc += reinterpret_cast<const float*>(sm + b * 65536)[threadIdx.x];
    __syncthreads();
    const size_t nt = t + 3 * (size_t)gridDim.x;
    if (threadIdx.x == 0 && nt < tiles) issue(nt, b);
  }
  if (acc == 1.2345f) sink[0] = acc;
}
int main() {
  const size_t bytes = (size_t)32 << 30, tiles = bytes / 65536;
  char* src;
  float* sink;
  if (cudaMalloc(&src, bytes) != cudaSuccess) return 1;
  cudaMemset(src, 0, bytes);
  cudaMalloc(&sink, 64);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536 + 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    const int K = rep == 1 ? 250 : 5;
    for (int i = 0; i < K; ++i) k_stream<<<148, 128, 3 * 65536 + 64>>>(src, tiles, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s x%d: %.3f ms per pass, %.0f GB/s (%s)\n", rep == 1 ? "sustained" : "burst", K, ms / K,
           bytes / (ms / K) / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
