// L1/shared-memory sharing microbenchmark (kernel-v3 design question, sm_100a):
//   does a TMA bulk fill (cp.async.bulk global->shared) or an LDG stream take
//   shared-memory bandwidth away from LDS/STS running on the same SM?
// Also: FADD2 butterfly throughput with 1 and 2 warps per SMSP (fwht128 on 128 registers).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_l1 scripts/mb_l1.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e));          \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int RING = 4;
constexpr int STAGE = 32768;                      // bytes per TMA stage
constexpr int LDS_WORDS = 8192;                   // 32 KB LDS scratch
constexpr int SMEM = 256 + RING * STAGE + LDS_WORDS * 4;

// mode bits: 1 = LDS warps run, 2 = TMA warp runs, 4 = LDG warps run, 8 = STS instead of LDS
// warps 0..7: LDS/STS workers; warp 8: TMA driver (one lane); warps 9..16: LDG streamers
__global__ void __launch_bounds__(544, 1) k_mix(const float* __restrict__ g, size_t per_cta_bytes, int lds_iters, int mode,
                                                unsigned long long* clk_out, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  unsigned char* ring = smem + 256;
  float* lds = reinterpret_cast<float*>(smem + 256 + RING * STAGE);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < LDS_WORDS; i += blockDim.x) lds[i] = (float)i;
  if (tid == 0) {
    for (int s = 0; s < RING; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  float acc = 0.f;
  const char* src = reinterpret_cast<const char*>(g) + (size_t)blockIdx.x * per_cta_bytes;
  if (warp < 8) {
    if (mode & 1) {
      int idx = tid;
      if (mode & 8) {
        for (int it = 0; it < lds_iters; ++it) {
#pragma unroll
          for (int k = 0; k < 16; ++k) lds[(idx + k * 256) & (LDS_WORDS - 1)] = (float)(it + k);
          idx = (idx + 32) & (LDS_WORDS - 1);
        }
      } else {
        for (int it = 0; it < lds_iters; ++it) {
#pragma unroll
          for (int k = 0; k < 16; ++k) acc += lds[(idx + k * 256) & (LDS_WORDS - 1)];
          idx = (idx + 32) & (LDS_WORDS - 1);
        }
      }
    }
  } else if (warp == 8) {
    if ((mode & 2) && lane == 0) {
      const int nst = (int)(per_cta_bytes / STAGE);
      for (int k = 0; k < nst; ++k) {
        const int s = k % RING;
        if (k >= RING) {
          const uint32_t ph = ((k / RING) - 1) & 1;
          asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(
                           smem_u32(&bars[s])),
                       "r"(ph));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(STAGE));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(ring + s * STAGE)),
                     "l"(src + (size_t)k * STAGE), "r"(STAGE), "r"(smem_u32(&bars[s]))
                     : "memory");
      }
      for (int k = nst - RING; k < nst; ++k) {
        if (k < 0) continue;
        const int s = k % RING;
        const uint32_t ph = (k / RING) & 1;
        asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(
                         smem_u32(&bars[s])),
                     "r"(ph));
      }
    }
  } else {
    if (mode & 4) {
      const float4* p4 = reinterpret_cast<const float4*>(src);
      const size_t n4 = per_cta_bytes / 16;
      const int t = tid - 9 * 32;  // 0..255
      for (size_t i = t; i + 7 * 256 < n4; i += 8 * 256) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(p4 + i + u * 256);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].w;
      }
    }
  }
  const unsigned long long t1 = clock64();
  if (lane == 0) clk_out[(size_t)blockIdx.x * 17 + warp] = t1 - t0;
  if (acc == 1.2345f) out[0] = acc;
}

// ---------------- FADD2 butterflies on 128 register values ----------------
__device__ __forceinline__ void fwht128(float2 (&v)[64]) {
#pragma unroll
  for (int m = 0; m < 64; ++m) v[m] = __ffma2_rn(v[m], make_float2(1.f, -1.f), make_float2(v[m].y, v[m].x));
#pragma unroll
  for (int s = 1; s < 64; s <<= 1) {
#pragma unroll
    for (int m = 0; m < 64; ++m) {
      if (!(m & s)) {
        const float2 a = v[m], b = v[m | s];
        v[m] = __fadd2_rn(a, b);
        v[m | s] = __fadd2_rn(a, make_float2(-b.x, -b.y));
      }
    }
  }
}
__global__ void __launch_bounds__(256, 1) k_bfly(float* out, int iters) {
  float2 v[64];
#pragma unroll
  for (int m = 0; m < 64; ++m) v[m] = make_float2(threadIdx.x * 1e-9f + m, 0.5f * m);
  for (int it = 0; it < iters; ++it) {
    fwht128(v);  // values overflow to inf/nan after a few iterations: irrelevant for FP32 pipe timing
  }
  float s = 0.f;
#pragma unroll
  for (int m = 0; m < 64; ++m) s += v[m].x + v[m].y;
  if (s == 1.2345f) out[0] = s;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const size_t per_cta = (size_t)48 << 20;  // 48 MB per CTA, 7.1 GB total: larger than L2
  float* g;
  CK(cudaMalloc(&g, per_cta * sms));
  CK(cudaMemset(g, 0, per_cta * sms));
  unsigned long long* clk_d;
  CK(cudaMalloc(&clk_d, sizeof(unsigned long long) * sms * 17));
  float* out;
  CK(cudaMalloc(&out, 64));
  CK(cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int lds_iters = 20000;
  unsigned long long* clk_h = new unsigned long long[sms * 17];
  const char* names[] = {"", "LDS", "TMA", "LDS+TMA", "LDG", "LDS+LDG", "TMA+LDG", "all", "",
                         "STS", "", "STS+TMA", "", "STS+LDG"};
  for (int mode : {1, 2, 4, 3, 5, 9, 11, 13}) {
    k_mix<<<sms, 544, SMEM>>>(g, per_cta, lds_iters, mode, clk_d, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    k_mix<<<sms, 544, SMEM>>>(g, per_cta, lds_iters, mode, clk_d, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    CK(cudaMemcpy(clk_h, clk_d, sizeof(unsigned long long) * sms * 17, cudaMemcpyDeviceToHost));
    double lds_cyc = 0, tma_cyc = 0, ldg_cyc = 0;
    for (int c = 0; c < sms; ++c) {
      unsigned long long m = 0;
      for (int w = 0; w < 8; ++w) m = clk_h[c * 17 + w] > m ? clk_h[c * 17 + w] : m;
      lds_cyc += m;
      tma_cyc += clk_h[c * 17 + 8];
      m = 0;
      for (int w = 9; w < 17; ++w) m = clk_h[c * 17 + w] > m ? clk_h[c * 17 + w] : m;
      ldg_cyc += m;
    }
    lds_cyc /= sms;
    tma_cyc /= sms;
    ldg_cyc /= sms;
    const double lds_words = 256.0 * 16 * lds_iters;
    printf("%-8s kernel %.3f ms | LDS/STS warps %.0f cyc -> %.1f words/clk/SM | TMA %.0f cyc -> %.1f B/clk/SM (%.0f GB/s chip)"
           " | LDG %.0f cyc -> %.1f B/clk/SM\n",
           names[mode], ms, lds_cyc, (mode & 1) ? lds_words / lds_cyc : 0.0, tma_cyc,
           (mode & 2) ? per_cta / tma_cyc : 0.0, (mode & 2) ? per_cta / tma_cyc * sms * clk * 1e3 / 1e9 : 0.0, ldg_cyc,
           (mode & 4) ? per_cta / ldg_cyc : 0.0);
  }
  // butterflies
  for (int wps : {1, 2}) {
    const int iters = 2000;
    k_bfly<<<sms, 128 * wps>>>(out, iters);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    k_bfly<<<sms, 128 * wps>>>(out, iters);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fadd2 = 448.0 * iters * 4 * wps;  // per SM warp-instructions (FFMA2+FADD2)
    printf("fwht128 %d warp(s)/SMSP: %.1f cyc per fwht128 per warp, %.2f FADD2-class instr/clk/SMSP\n", wps,
           ms * 1e-3 * clk * 1e3 / iters, fadd2 / 4 / (ms * 1e-3 * clk * 1e3));
  }
  return 0;
}
