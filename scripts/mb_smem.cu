// Shared-memory access width microbenchmark (words/clk/SM) for LDS/STS .32/.64/.128.
#include <cstdio>
#include <cuda_runtime.h>
template <int W, bool LOAD>
__global__ void k(float* out, int iters) {
  __shared__ __align__(16) float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float acc = 0.f;
  const int words = W / 4;
  int base = threadIdx.x * words;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = (base + k * blockDim.x * words + it * 32 * words) & (8192 - words);
      if (LOAD) {
        if (W == 4) acc += sm[idx];
        if (W == 8) { float2 v = *reinterpret_cast<float2*>(&sm[idx]); acc += v.x + v.y; }
        if (W == 16) { float4 v = *reinterpret_cast<float4*>(&sm[idx]); acc += v.x + v.w; }
      } else {
        if (W == 4) sm[idx] = acc + k;
        if (W == 8) *reinterpret_cast<float2*>(&sm[idx]) = make_float2(acc, k);
        if (W == 16) *reinterpret_cast<float4*>(&sm[idx]) = make_float4(acc, k, it, 1.f);
      }
    }
  }
  __syncthreads();
  if (LOAD ? acc == 1.2345f : sm[threadIdx.x] == 1.2345f) out[0] = acc;
}
template <int W, bool LOAD>
void run(float* out, int sms, int clk) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, tpb = 512, bps = 2;
  k<W, LOAD><<<sms * bps, tpb>>>(out, iters);
  cudaEventRecord(a);
  k<W, LOAD><<<sms * bps, tpb>>>(out, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double words = (double)sms * bps * tpb * iters * 8 * (W / 4);
  printf("%s.%d: %.1f words/clk/SM\n", LOAD ? "LDS" : "STS", W * 8, words / (ms * 1e-3) / sms / (clk * 1e3));
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 64);
  run<4, true>(out, sms, clk); run<8, true>(out, sms, clk); run<16, true>(out, sms, clk);
  run<4, false>(out, sms, clk); run<8, false>(out, sms, clk); run<16, false>(out, sms, clk);
  return 0;
}
