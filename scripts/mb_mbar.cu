// What does mbarrier.pending_count report for the state returned by mbarrier.arrive?
// Four warps arrive one after another (count 4) on one barrier, twice (two phases).
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out) {
  __shared__ __align__(8) uint64_t bar;
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(a));
  __syncthreads();
  for (int ph = 0; ph < 2; ++ph)
    for (int w = 0; w < 4; ++w) {
      if (threadIdx.x == 32 * w) {
        uint64_t st;
        uint32_t pend;
        asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(a) : "memory");
        asm volatile("mbarrier.pending_count.b64 %0, %1;" : "=r"(pend) : "l"(st));
        out[ph * 4 + w] = pend;
      }
      __syncthreads();
    }
}
int main() {
  uint32_t* d;
  cudaMalloc(&d, 64);
  k<<<1, 128>>>(d);
  uint32_t h[8];
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("pending_count after arrivals 1..4 (phase 0): %u %u %u %u; phase 1: %u %u %u %u  (%s)\n", h[0], h[1], h[2],
         h[3], h[4], h[5], h[6], h[7], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
