// tcgen05.cp (shared -> tensor memory) microbenchmark for the kernel-v3 design question
// "can round 1 read its raw tile from TMEM instead of with LDS?" (sm_100a):
//  1. layout: 32 copies of 128 rows x 128 bits from a 64 KB tile whose 16-byte row p' of
//     chunk h' sits at byte 16 p' + 2048 h' (no-swizzle K-major canonical layout, 8-row core
//     matrices 128 B apart) land lane p', columns 4h'..4h'+3 == words 4p' + 512h' + 0..3?
//  2. throughput of back-to-back tile copies (bytes per SM clock), one issuing thread;
//  3. LDS words/clk of 8 warps alone and while the copies stream, and tcgen05.ld words/clk.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_tmemcp scripts/mb_tmemcp.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_nosw(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

constexpr int TILE = 65536;
constexpr int LDSW = 4096;  // 16 KB LDS scratch

// mode bit 1: copies run (warp 8 lane 0); bit 2: LDS warps run (warps 0..7); bit 4: TMEM-load warps (0..3) instead of LDS
__global__ void __launch_bounds__(288, 1) k_cp(int iters, int mode, unsigned long long* out, int* bad) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint32_t* tile = reinterpret_cast<uint32_t*>(smem);
  float* lds = reinterpret_cast<float*>(smem + TILE);
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < TILE / 4; i += blockDim.x) tile[i] = (uint32_t)i;
  for (int i = tid; i < LDSW; i += blockDim.x) lds[i] = (float)i;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = taddr_s;
  const uint32_t sbase = su(tile);
  // ---- 1. layout check (one round of copies) ----
  if (tid == 256) {
    for (int h = 0; h < 32; ++h)
      asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tbase + 4 * h), "l"(desc_nosw(sbase + 2048 * h, 0, 128)));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
  }
  asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra W_%=;\n}" ::"r"(su(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    int nb = 0;
    const int p = 32 * warp + lane;
    for (int h = 0; h < 32; ++h) {
      uint32_t v0, v1, v2, v3;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                   : "r"(tbase + ((uint32_t)(32 * warp) << 16) + 4 * h));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const uint32_t e = 4 * p + 512 * h;
      nb += (v0 != e) + (v1 != e + 1) + (v2 != e + 2) + (v3 != e + 3);
    }
    if (nb) atomicAdd(bad, nb);
  }
  __syncthreads();
  // ---- 2/3. streams ----
  const unsigned long long t0 = clock64();
  float acc = 0.f;
  if (warp == 8) {
    if ((mode & 1) && lane == 0) {
      for (int it = 0; it < iters; ++it) {
        for (int h = 0; h < 32; ++h)
          asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tbase + 4 * h), "l"(desc_nosw(sbase + 2048 * h, 0, 128)));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
        const uint32_t ph = (uint32_t)((it + 1) & 1);
        asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(
                         su(&bar)),
                     "r"(ph)
                     : "memory");
      }
    }
  } else if (mode & 2) {
    if ((mode & 4) && warp < 4) {
      uint32_t s = 0;
      for (int it = 0; it < iters * 8; ++it) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                       "=r"(v[15])
                     : "r"(tbase + ((uint32_t)(32 * warp) << 16) + 16 * (it & 7)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 16; ++k) s += v[k];
      }
      acc = (float)s;
    } else if (!(mode & 4)) {
      int idx = tid;
      for (int it = 0; it < iters * 4; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += lds[(idx + k * 256) & (LDSW - 1)];
        idx = (idx + 32) & (LDSW - 1);
      }
    }
  }
  const unsigned long long t1 = clock64();
  if (acc == 1.2345f) out[0] = 0;
  if (blockIdx.x == 0) out[1 + tid] = t1 - t0;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

int main() {
  unsigned long long* d_out;
  int* d_bad;
  cudaMalloc(&d_out, 2048 * 8);
  cudaMalloc(&d_bad, 4);
  const int smem = TILE + LDSW * 4;
  cudaFuncSetAttribute(k_cp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 400;
  const char* names[] = {"copies alone", "LDS alone", "LDS + copies", "TMEM ld alone", "TMEM ld + copies"};
  const int modes[] = {1, 2, 3, 6, 7};
  for (int m = 0; m < 5; ++m) {
    cudaMemset(d_bad, 0, 4);
    k_cp<<<148, 288, smem>>>(iters, modes[m], d_out, d_bad);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[289];
    int bad = 0;
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(&bad, d_bad, 4, cudaMemcpyDeviceToHost);
    const double cp_cyc = (double)h[1 + 256];  // warp 8 lane 0
    const double w_cyc = (double)h[1 + 0];     // warp 0 lane 0
    double line1 = 0, line2 = 0;
    if (modes[m] & 1) line1 = (double)iters * TILE / cp_cyc;  // bytes / clk
    if ((modes[m] & 2) && !(modes[m] & 4)) line2 = (double)iters * 4 * 16 * 256 / w_cyc;   // LDS words / clk (8 warps)
    if ((modes[m] & 2) && (modes[m] & 4)) line2 = (double)iters * 8 * 16 * 128 / w_cyc;    // TMEM words / clk (4 warps)
    printf("%-18s layout errors %d | copies %.1f B/clk/SM | %s %.1f words/clk/SM (%s)\n", names[m], bad, line1,
           (modes[m] & 4) ? "TMEM ld" : "LDS", line2, cudaGetErrorString(e));
  }
  return 0;
}
