// Does SHFL or tcgen05.ld (TMEM) share throughput with LDS?  (kernel-v3 design question)
// 8 "A" warps run LDS loops, 8 "B" warps run SHFL or TMEM loads; each role timed with clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_xbar scripts/mb_xbar.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode bit 1: LDS warps active; bit 2: SHFL warps active; bit 4: TMEM-load warps active
__global__ void __launch_bounds__(512, 1) k(int iters, int mode, unsigned long long* clk, float* out) {
  __shared__ float sm[8192];
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 8192; i += 512) sm[i] = i;
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned long long t0 = clock64();
  float acc = 0.f;
  if (warp < 8) {
    if (mode & 1) {
      int idx = tid;
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += sm[(idx + q * 256) & 8191];
        idx = (idx + 32) & 8191;
      }
    }
  } else {
    if (mode & 2) {
      float a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = tid + i;
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 15));
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += a[i];
    }
    if (mode & 4) {
      const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(((warp - 8) >> 2) * 64);
      for (int it = 0; it < iters; ++it) {
        uint32_t r[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(base + (uint32_t)((it & 3) * 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += __uint_as_float(r[i]);
      }
    }
  }
  const unsigned long long t1 = clock64();
  if ((tid & 31) == 0) clk[blockIdx.x * 16 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(taddr_s));
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* clk;
  cudaMalloc(&clk, sizeof(unsigned long long) * sms * 16);
  float* out;
  cudaMalloc(&out, 64);
  unsigned long long* h = new unsigned long long[sms * 16];
  const int iters = 20000;
  const char* names[] = {"", "LDS", "SHFL", "LDS+SHFL", "TMEMld", "LDS+TMEMld"};
  for (int mode : {1, 2, 3, 4, 5}) {
    k<<<sms, 512>>>(iters, mode, clk, out);
    cudaError_t e = cudaDeviceSynchronize();
    k<<<sms, 512>>>(iters, mode, clk, out);
    e = cudaDeviceSynchronize();
    cudaMemcpy(h, clk, sizeof(unsigned long long) * sms * 16, cudaMemcpyDeviceToHost);
    double a = 0, b = 0;
    for (int c = 0; c < sms; ++c) {
      unsigned long long ma = 0, mb = 0;
      for (int w = 0; w < 8; ++w) ma = h[c * 16 + w] > ma ? h[c * 16 + w] : ma;
      for (int w = 8; w < 16; ++w) mb = h[c * 16 + w] > mb ? h[c * 16 + w] : mb;
      a += ma;
      b += mb;
    }
    a /= sms;
    b /= sms;
    const double words = 256.0 * 16 * iters;
    printf("%-11s LDS warps: %.1f words/clk/SM | B warps: %.1f words/clk/SM (%s)\n", names[mode],
           (mode & 1) ? words / a : 0.0, (mode & 6) ? words / b : 0.0, cudaGetErrorString(e));
  }
  return 0;
}
