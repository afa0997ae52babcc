// TMEM load/store throughput with several tcgen05.ld in flight per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
#define LD32(r, addr) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
  : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), \
    "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(addr))
#define ST32(addr, r) asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" \
  :: "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), \
    "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))

template <int NLD, int MODE>  // MODE 0: ld only, 1: ld+st (read-modify-write)
__global__ void k(float* out, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int nw = blockDim.x >> 5;
  const int per_sub = nw / 4;                     // warps sharing a lane quarter
  const int cols = 512 / per_sub;                 // columns per warp
  const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * cols);
  uint32_t r[NLD][32];
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const uint32_t c0 = (uint32_t)((it * NLD * 32) % cols);
#pragma unroll
    for (int j = 0; j < NLD; ++j) LD32(r[j], base + ((c0 + 32 * j) % cols));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int j = 0; j < NLD; ++j) {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[j][i] += 1u;
    }
    if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < NLD; ++j) ST32(base + ((c0 + 32 * j) % cols), r[j]);
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    acc += __uint_as_float(r[0][it & 31]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
  if (acc == 1.2345f) out[0] = acc;
}
template <int NLD, int MODE>
void run(float* out, int sms, int clk, int tpb) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2048;
  k<NLD, MODE><<<sms, tpb>>>(out, iters);
  cudaEventRecord(a);
  k<NLD, MODE><<<sms, tpb>>>(out, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double words = (double)sms * tpb * iters * NLD * 32;
  printf("tpb=%d NLD=%d %s: %.1f words/clk/SM loaded (%s)\n", tpb, NLD, MODE ? "ld+st" : "ld", words / (ms * 1e-3) / sms / (clk * 1e3),
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 64);
  for (int tpb : {128, 256, 512}) {
    run<1, 0>(out, sms, clk, tpb); run<2, 0>(out, sms, clk, tpb); run<4, 0>(out, sms, clk, tpb);
    run<1, 1>(out, sms, clk, tpb); run<4, 1>(out, sms, clk, tpb);
  }
  return 0;
}
