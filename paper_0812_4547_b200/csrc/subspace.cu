// Algorithm 2, SubspaceSampling, sm_100a.
//
// Row i of Phi (n x d) is kept with probability q_i = min(1, r p_i) and scaled by
// 1/sqrt(q_i): kept iff q_i >= 1 or u_i < floor(q_i 2^64), u_i = word i of the Philox
// stream (seed, 1) (reading R18; the same coins as the Bernoulli SRHT plan, so
// p_i = 1/N on H_N D [M; 0] / sqrt(N) reproduces it).  Two passes: per-block keep counts,
// then an order-preserving compaction writing the kept indices (ascending) and the scaled
// rows.  The threshold is formed exactly (q_i 2^64 is exact in FP64; rounded down to an
// integer), so the keep decisions are bit-identical to the oracle's.
#include <cuda_runtime.h>

#include "internal.cuh"
#include "philox.cuh"

namespace srht {
namespace {

constexpr int SS_T = 256;
constexpr int SS_PER = 16;                  // rows per thread (4 Philox blocks)
constexpr int SS_CHUNK = SS_T * SS_PER;     // rows per CTA

__device__ __forceinline__ bool keep_row(uint64_t u, double q) {
  if (q >= 1.0) return true;
  const unsigned long long T = __double2ull_rd(q * 18446744073709551616.0);  // floor(q 2^64), q < 1
  return u < T;
}

__device__ __forceinline__ uint32_t chunk_mask(uint64_t seed, int64_t n, double r, const double* __restrict__ p,
                                               int64_t i0) {
  uint32_t m = 0;
#pragma unroll
  for (int b = 0; b < SS_PER / 4; ++b) {
    const int64_t q = i0 / 4 + b;
    if (4 * q >= n) break;
    const u64x4 w = stream_block(seed, 1, (uint64_t)q);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t i = 4 * q + e;
      if (i < n) {
        const double qi = fmin(1.0, r * p[i]);
        m |= (uint32_t)keep_row(w.v[e], qi) << (4 * b + e);
      }
    }
  }
  return m;
}

__device__ int block_excl_scan_ss(int v, int* total) {
  __shared__ int wsum[SS_T / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int s = lane < SS_T / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    if (lane < SS_T / 32) wsum[lane] = s;
  }
  __syncthreads();
  const int base = wid ? wsum[wid - 1] : 0;
  *total = wsum[SS_T / 32 - 1];
  __syncthreads();
  return base + inc - v;
}

__global__ void k_ss_count(uint64_t seed, int64_t n, double r, const double* __restrict__ p, int32_t* __restrict__ cnt) {
  const int64_t i0 = blockIdx.x * (int64_t)SS_CHUNK + (int64_t)threadIdx.x * SS_PER;
  int tot;
  block_excl_scan_ss(__popc(chunk_mask(seed, n, r, p, i0)), &tot);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__global__ void k_ss_offsets(int64_t nblk, const int32_t* __restrict__ cnt, int64_t* __restrict__ off,
                             int64_t* __restrict__ total) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t acc = 0;
  for (int64_t b = 0; b < nblk; ++b) {
    off[b] = acc;
    acc += cnt[b];
  }
  *total = acc;
}

__global__ void k_ss_write(uint64_t seed, int64_t n, double r, const double* __restrict__ p,
                           const int64_t* __restrict__ off, int64_t cap, int32_t* __restrict__ K) {
  const int64_t i0 = blockIdx.x * (int64_t)SS_CHUNK + (int64_t)threadIdx.x * SS_PER;
  const uint32_t m = chunk_mask(seed, n, r, p, i0);
  int tot;
  int64_t pos = off[blockIdx.x] + block_excl_scan_ss(__popc(m), &tot);
  for (int e = 0; e < SS_PER; ++e) {
    if ((m >> e) & 1u) {
      if (pos < cap) K[pos] = (int32_t)(i0 + e);
      ++pos;
    }
  }
}

// Kept rows, scaled: 32 consecutive kept rows per CTA (lanes), warps stride over the d
// columns, so every store instruction writes 32 consecutive output rows of one column.
__global__ void k_ss_gather(int64_t cap, const int64_t* __restrict__ total, int64_t d, double r,
                            const double* __restrict__ p, const float* __restrict__ Phi, int64_t ldphi,
                            const int32_t* __restrict__ K, float* __restrict__ out, int64_t ldout) {
  const int64_t t = blockIdx.x * 32 + (threadIdx.x & 31);
  const int64_t kept = *total < cap ? *total : cap;  // rows written by k_ss_write
  if (t >= kept) return;
  const int64_t i = K[t];
  const double s = 1.0 / sqrt(fmin(1.0, r * p[i]));
  for (int64_t j = threadIdx.x >> 5; j < d; j += blockDim.x >> 5)
    out[t + j * ldout] = (float)((double)Phi[i + j * ldphi] * s);
}

}  // namespace

// kept != nullptr: count only (synchronous).  Otherwise write K / out (capacity cap rows).
cudaError_t launch_subspace(int64_t n, int64_t d, int64_t r, uint64_t seed, const double* p, const float* Phi,
                            int64_t ldphi, int32_t* K, float* out, int64_t ldout, int64_t cap, int64_t* kept,
                            cudaStream_t stream) {
  const int64_t nblk = (n + SS_CHUNK - 1) / SS_CHUNK;
  int32_t* cnt = nullptr;
  int64_t* off = nullptr;
  cudaError_t e = cudaMallocAsync(&cnt, nblk * sizeof(int32_t), stream);
  if (e == cudaSuccess) e = cudaMallocAsync(&off, (nblk + 1) * sizeof(int64_t), stream);
  if (e == cudaSuccess) {
    k_ss_count<<<(unsigned)nblk, SS_T, 0, stream>>>(seed, n, (double)r, p, cnt);
    k_ss_offsets<<<1, 32, 0, stream>>>(nblk, cnt, off, off + nblk);
    if (kept) {
      e = cudaMemcpyAsync(kept, off + nblk, sizeof(int64_t), cudaMemcpyDeviceToHost, stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    } else {
      k_ss_write<<<(unsigned)nblk, SS_T, 0, stream>>>(seed, n, (double)r, p, off, cap, K);
      // rows written: min(cap, kept); the caller sized cap from the count pass
      if (cap > 0 && d > 0)
        k_ss_gather<<<(unsigned)((cap + 31) / 32), 256, 0, stream>>>(cap, off + nblk, d, (double)r, p, Phi, ldphi, K,
                                                                    out, ldout);
    }
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaFreeAsync(cnt, stream);
  cudaFreeAsync(off, stream);
  return e;
}

}  // namespace srht
