// Calibration microbenchmarks for the SRHT kernel design on B200 (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

// ---------------- streaming read bandwidth ----------------
template <int UNROLL>
__global__ void k_read(const float4* __restrict__ p, size_t n4, float* out) {
  float acc = 0.f;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n4; i += UNROLL * stride) {
    float4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

// per-CTA contiguous chunks (like a column slab), 8 x LDG.128 per thread per iteration
__global__ void k_read_chunks(const float* __restrict__ p, size_t chunk, int nchunks, float* out) {
  float acc = 0.f;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const float* base = p + (size_t)c * chunk;
    for (size_t off = 0; off < chunk; off += (size_t)blockDim.x * 32) {
      float4 v[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) v[h] = __ldcs(reinterpret_cast<const float4*>(base + off + h * blockDim.x * 4 + threadIdx.x * 4));
#pragma unroll
      for (int h = 0; h < 8; ++h) acc += v[h].x + v[h].y + v[h].z + v[h].w;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

// bulk-copy (TMA 1D) ring: one elected thread issues cp.async.bulk into a ring of smem stages,
// all threads consume (read) each stage.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_read_bulk(const float* __restrict__ p, size_t chunk, int nchunks, int stage_bytes, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int S = 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  float* buf = reinterpret_cast<float*>(smem + 128);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  float acc = 0.f;
  const int per_stage = stage_bytes / 4;
  // flatten work: (chunk c, piece k)
  long total = 0;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) total += chunk / per_stage;
  long issued = 0, consumed = 0;
  int c_iss = blockIdx.x; size_t k_iss = 0;
  auto issue = [&](long it) {
    const int s = it % S;
    const float* src = p + (size_t)c_iss * chunk + k_iss * per_stage;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(stage_bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(buf + s * per_stage)), "l"(src), "r"(stage_bytes), "r"(smem_u32(&bars[s])) : "memory");
    k_iss++;
    if (k_iss * per_stage >= chunk) { k_iss = 0; c_iss += gridDim.x; }
  };
  if (tid == 0) for (; issued < S && issued < total; ++issued) issue(issued);
  for (; consumed < total; ++consumed) {
    const int s = consumed % S;
    const uint32_t phase = (consumed / S) & 1;
    asm volatile("{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}" ::"r"(smem_u32(&bars[s])), "r"(phase));
    const float4* b4 = reinterpret_cast<const float4*>(buf + s * per_stage);
    for (int i = tid; i < per_stage / 4; i += blockDim.x) { float4 v = b4[i]; acc += v.x + v.y + v.z + v.w; }
    __syncthreads();
    if (tid == 0 && issued < total) { issue(issued); ++issued; }
  }
  if (acc == 12345.f) out[0] = acc;
}

// ---------------- ALU throughput ----------------
__global__ void k_fadd2(float* out, int iters) {
  float2 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-7f + i, i * 0.5f);
  const float2 b = make_float2(1e-7f, -1e-7f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __fadd2_rn(a[i], b);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 12345.f) out[0] = s;
}
__global__ void k_fadd(float* out, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-7f + i;
  const float b = 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = a[i] + b;
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void k_ffma2_swz(float* out, int iters) {  // the within-pair butterfly form
  float2 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-7f + i, i * 0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], make_float2(0.5f, -0.5f), make_float2(a[i].y, a[i].x));
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 12345.f) out[0] = s;
}
__global__ void k_lop3(unsigned* out, int iters) {
  unsigned a[16];
  unsigned w = threadIdx.x * 2654435761u;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] ^= (w << (31 - i)) & 0x80000000u;  // sign flip: SHF + LOP3
    w = w * 3u + 1u;
  }
  unsigned s = 0; for (int i = 0; i < 16; ++i) s ^= a[i];
  if (s == 12345u) out[0] = s;
}

// ---------------- shared memory / shuffle ----------------
__global__ void k_lds(float* out, int iters) {
  __shared__ float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float acc = 0.f;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += sm[(idx + k * 256) & 8191];
    idx = (idx + 1) & 8191;
  }
  if (acc == 12345.f) out[0] = acc;
}
__global__ void k_sts(float* out, int iters) {
  __shared__ float sm[8192];
  int idx = threadIdx.x;
  float v = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) sm[(idx + k * 256) & 8191] = v + k;
    idx = (idx + 1) & 8191;
  }
  __syncthreads();
  if (sm[threadIdx.x] == 12345.f) out[0] = 1;
}
__global__ void k_lds128(float* out, int iters) {
  __shared__ float4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
  __syncthreads();
  float acc = 0.f;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { float4 v = sm[(idx + k * 256) & 2047]; acc += v.x + v.w; }
    idx = (idx + 1) & 2047;
  }
  if (acc == 12345.f) out[0] = acc;
}
__global__ void k_shfl(float* out, int iters) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 << (i % 5));
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}

// ---------------- TMEM ----------------
__global__ void k_tmem(float* out, int iters, int mode) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x + i;
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                     "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                     "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(base + (uint32_t)((it & 1) * 32)));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += __uint_as_float(r[it & 31]);
    } else {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   ::"r"(base + (uint32_t)((it & 1) * 32)), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                     "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
                     "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
                     "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
      r[it & 31] += 1;
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(taddr_s));
  if (acc == 12345.f) out[0] = acc;
}

template <typename F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b); if (t < best) best = t;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s SMs=%d smem/SM=%zu smem/block optin=%zu regs/SM=%d L2=%d clock=%d kHz\n", prop.name, prop.multiProcessorCount,
         prop.sharedMemPerMultiprocessor, prop.sharedMemPerBlockOptin, prop.regsPerMultiprocessor, prop.l2CacheSize, clk);
  const int SM = prop.multiProcessorCount;
  float* out; CK(cudaMalloc(&out, 64));
  const size_t bytes = (size_t)8 << 30;
  float* buf; CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 0, bytes));
  const size_t n4 = bytes / 16;
  for (int tpb : {256, 512, 1024}) for (int bps : {1, 2, 4, 8}) {
    if (tpb * bps > 2048) continue;
    float t = time_ms([&] { k_read<4><<<SM * bps, tpb>>>((const float4*)buf, n4, out); });
    printf("read LDG.128 u4 tpb=%d blocks/SM=%d: %.1f GB/s\n", tpb, bps, bytes / t / 1e6);
  }
  for (int tpb : {256, 512}) for (int bps : {1, 2, 4}) {
    if (tpb * bps > 2048) continue;
    float t = time_ms([&] { k_read<8><<<SM * bps, tpb>>>((const float4*)buf, n4, out); });
    printf("read LDG.128 u8 tpb=%d blocks/SM=%d: %.1f GB/s\n", tpb, bps, bytes / t / 1e6);
  }
  {
    const size_t chunk = 1 << 20;  // 4 MB chunks
    const int nch = bytes / 4 / chunk;
    for (int tpb : {256, 512}) for (int bps : {1, 2, 4}) {
      if (tpb * bps > 2048) continue;
      float t = time_ms([&] { k_read_chunks<<<SM * bps, tpb>>>(buf, chunk, nch, out); });
      printf("read chunks 8xLDG.128 tpb=%d blocks/SM=%d: %.1f GB/s\n", tpb, bps, bytes / t / 1e6);
    }
    for (int sb : {8192, 16384, 32768}) for (int bps : {1, 2}) {
      const int smem = 128 + 4 * sb;
      if (smem * bps > 220 * 1024) continue;
      cudaFuncSetAttribute(k_read_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      float t = time_ms([&] { k_read_bulk<<<SM * bps, 256, smem>>>(buf, chunk, nch, sb, out); });
      printf("read bulk-copy ring 4x%dB blocks/SM=%d: %.1f GB/s (%s)\n", sb, bps, bytes / t / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // ALU
  const int iters = 4096;
  auto rate = [&](const char* name, float ms, double ops) {
    printf("%s: %.1f ops/clk/SM (%.3f ms)\n", name, ops / (ms * 1e-3) / SM / (clk * 1e3), ms);
  };
  { float t = time_ms([&] { k_fadd2<<<SM * 4, 512>>>(out, iters); }); rate("FADD2 (adds, 2/instr)", t, 2.0 * 8 * iters * SM * 4 * 512); }
  { float t = time_ms([&] { k_fadd<<<SM * 4, 512>>>(out, iters); }); rate("FADD", t, 16.0 * iters * SM * 4 * 512); }
  { float t = time_ms([&] { k_ffma2_swz<<<SM * 4, 512>>>(out, iters); }); rate("FFMA2 swizzled butterfly (fma, 2/instr)", t, 2.0 * 8 * iters * SM * 4 * 512); }
  { float t = time_ms([&] { k_lop3<<<SM * 4, 512>>>((unsigned*)out, iters); }); rate("sign flip (elements)", t, 16.0 * iters * SM * 4 * 512); }
  { float t = time_ms([&] { k_lds<<<SM * 4, 256>>>(out, iters); }); rate("LDS.32 conflict-free (words)", t, 16.0 * iters * SM * 4 * 256); }
  { float t = time_ms([&] { k_sts<<<SM * 4, 256>>>(out, iters); }); rate("STS.32 conflict-free (words)", t, 16.0 * iters * SM * 4 * 256); }
  { float t = time_ms([&] { k_lds128<<<SM * 4, 256>>>(out, iters); }); rate("LDS.128 (words)", t, 32.0 * iters * SM * 4 * 256); }
  { float t = time_ms([&] { k_shfl<<<SM * 4, 512>>>(out, iters); }); rate("SHFL (words)", t, 8.0 * iters * SM * 4 * 512); }
  {
    float t = time_ms([&] { k_tmem<<<SM, 256>>>(out, iters, 0); });
    rate("TMEM ld 32x32b.x32 (words)", t, 32.0 * iters * SM * 256);
    printf("  tmem ld err: %s\n", cudaGetErrorString(cudaGetLastError()));
    t = time_ms([&] { k_tmem<<<SM, 256>>>(out, iters, 1); });
    rate("TMEM st 32x32b.x32 (words)", t, 32.0 * iters * SM * 256);
    printf("  tmem st err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}
