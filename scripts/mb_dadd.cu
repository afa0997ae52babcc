// Microbenchmark: FP64 add (DADD) and FP32 add (FADD / FADD2) throughput per SM per clock on the
// B200 (the peak of the FP64-accumulation kernel's "alu" roofline).  nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void k_add(T* out, int iters, T a) {
  T v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = (T)(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = v[i] + a;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = v[i] - a;
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == (T)-1.2345) out[0] = s;
}
__global__ void k_add2(float* out, int iters, float a) {
  float2 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = make_float2(threadIdx.x + i, i);
  const float2 a2 = make_float2(a, a), m2 = make_float2(-a, -a);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __fadd2_rn(v[i], a2);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __fadd2_rn(v[i], m2);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i].x + v[i].y;
  if (s == -1.2345f) out[0] = s;
}
int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d; float* f;
  cudaMalloc(&d, 8); cudaMalloc(&f, 8);
  const int iters = 20000, threads = 1024, blocks = sms * 2;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int kind = 0; kind < 3; ++kind) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) k_add<double><<<blocks, threads>>>(d, iters, 1.0);
      else if (kind == 1) k_add<float><<<blocks, threads>>>(f, iters, 1.0f);
      else k_add2<<<blocks, threads>>>(f, iters, 1.0f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double adds = (double)blocks * threads * iters * 16 * (kind == 2 ? 2 : 1);
    const double per_s = adds / (best * 1e-3);
    printf("%s: %.3f ms, %.2f Tadd/s, %.1f adds/clk/SM at %d MHz (max clock)\n",
           kind == 0 ? "DADD" : kind == 1 ? "FADD" : "FADD2", best, per_s / 1e12, per_s / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
