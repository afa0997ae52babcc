// Microbenchmark: FP64 tensor-core MMA (mma.sync m8n8k4 f64, SASS DMMA) vs FP64 FMA (DFMA)
// throughput per SM on the B200 (Gram-kernel design evidence).  nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(a, b, c[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == -1.2345) out[0] = s;
}
int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  for (int kind = 0; kind < 2; ++kind) {
    for (int tpb : {128, 256, 512}) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0) k_dmma<<<sms * 4, tpb>>>(d, iters); else k_dfma<<<sms * 4, tpb>>>(d, iters * 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      // DMMA m8n8k4: 256 FMA per warp instruction; DFMA: 1 per thread
      const double fma = kind == 0 ? (double)sms * 4 * (tpb / 32) * iters * 8 * 256.0
                                   : (double)sms * 4 * tpb * iters * 4 * 8.0;
      printf("%s tpb=%d: %.3f ms, %.2f TFLOP/s, %.1f FMA/clk/SM (at %d MHz)\n", kind == 0 ? "DMMA" : "DFMA", tpb, best,
             2 * fma / (best * 1e-3) / 1e12, fma / (best * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
