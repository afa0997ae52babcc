// FP64-accumulation SRHT sketch (parity mode, plan flag SRHT_PLAN_ACCUM_FP64), sm_100a.
//
// Same output and the same decomposition as the FP32 kernels:
//   SM[t] = r^{-1/2} sum_s (-1)^{popc(k_slab & s)} sum_j (-1)^{popc(k_mid & j)} (H_B D x_{s,j})[k_lo],
// but every add after the FP32 load is done in FP64 (butterflies, the pruned accumulation,
// the slab partials and their reduction), and the result is rounded once to FP32.  This is
// the mode SURVEY.md reading C14 / DESIGN.md reading R14 asks for: the end-to-end NNLS gate
// of 1e-6 sits at the FP32 rounding floor for the nearly consistent configs 4 and 5, so
// parity at that gate is established with this mode; the FP32 kernels stay the throughput
// path.  It is written for clarity, not speed: one CTA per (column, slab, sample group), the
// tile in shared memory as doubles, radix-8 passes with a barrier between passes.
#include <cuda_runtime.h>

#include "internal.cuh"

namespace srht {
namespace {

constexpr int T64 = 256;   // threads per CTA
// CTAs per SM: three 64 KB tiles (B <= 2^13) fit in shared memory; occupancy beats registers here
// (config 4: 2 CTAs / 128 registers 9.0 ms, 3 CTAs / 80 registers 7.2 ms, 1 CTA unbounded 12.0 ms)
template <int LOG_B>
constexpr int f64_min_blocks() { return LOG_B >= 14 ? 1 : 3; }
#ifndef F64_RPT
#define F64_RPT 32
#endif
constexpr int RPT64 = F64_RPT;  // samples per thread per work item (8192 per CTA: one pass over the
                                // tiles serves every sample up to r = 8192)

// One radix-8 pass of the unnormalized natural-order WHT over bits [bit, bit + nb) of the
// tile index (nb <= 3): each group of 2^nb entries differing only in those bits is
// transformed in registers.
template <int LOG_B>
__device__ __forceinline__ void wht_pass(double* tile, int bit, int nb) {
  constexpr int B = 1 << LOG_B;
  const int gsize = 1 << nb;
  const int ngroups = B >> nb;
  for (int g = threadIdx.x; g < ngroups; g += T64) {
    const int lo = g & ((1 << bit) - 1);
    const int base = ((g >> bit) << (bit + nb)) | lo;  // insert nb zero bits at position bit
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < gsize) v[u] = tile[base + (u << bit)];
#pragma unroll
    for (int st = 1; st < 8; st <<= 1) {
      if (st >= gsize) break;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u < gsize && !(u & st)) {
          const double a = v[u], b = v[u | st];
          v[u] = a + b;
          v[u | st] = a - b;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < gsize) tile[base + (u << bit)] = v[u];
  }
}

template <int LOG_B>
__global__ void __launch_bounds__(T64, f64_min_blocks<LOG_B>()) k_sketch_f64(const __grid_constant__ SketchParams P, int64_t groups) {
  constexpr int B = 1 << LOG_B;
  extern __shared__ __align__(16) double tile64[];
  __shared__ int64_t s_ptr;
  const int tid = threadIdx.x;

  int64_t item = blockIdx.x;
  const int64_t g = item % groups;
  item /= groups;
  const int64_t sl = item % P.S_act;  // slab of this launch
  const int64_t s = P.s_lo + sl;      // global slab
  const int64_t col = item / P.S_act;
  const bool second = col >= P.ncols0;
  const ColSrc& cs = second ? P.src[1] : P.src[0];
  const int64_t lc = second ? col - P.ncols0 : col;
  const int64_t prob = col / P.cols_per_problem;
  const uint32_t* __restrict__ signs = P.signs + prob * P.words32;
  const int32_t* __restrict__ Kp = P.K + prob * P.r;

  uint32_t km[RPT64];  // k_lo | k_mid << 16 (k_lo < 2^14, k_mid < 2^16)
  double acc[RPT64];
  const int64_t t0 = g * (int64_t)RPT64 * T64;
#pragma unroll
  for (int q = 0; q < RPT64; ++q) {
    const int64_t t = t0 + (int64_t)q * T64 + tid;
    const int32_t k = t < P.r ? Kp[t] : 0;
    km[q] = (uint32_t)(k & (B - 1)) | (((uint32_t)(k >> LOG_B) & (uint32_t)(P.J - 1)) << 16);
    acc[q] = 0.0;
  }

  const int64_t j0 = s * P.J;
  const int64_t j1 = (j0 + P.J < P.n_sub) ? j0 + P.J : P.n_sub;
  const int64_t n = P.n;
  int64_t cptr = 0, cend = 0;
  if (cs.fmt == SRHT_CSC) {
    cend = cs.colptr[lc + 1];
    if (tid == 0) {
      int64_t a = cs.colptr[lc], b = cend;
      const int64_t target = j0 * (int64_t)B;
      while (a < b) {  // lower_bound(rowidx, target)
        const int64_t m = (a + b) >> 1;
        if ((int64_t)cs.rowidx[m] < target) a = m + 1; else b = m;
      }
      s_ptr = a;
    }
    __syncthreads();
    cptr = s_ptr;
  }

  for (int64_t j = j0; j < j1; ++j) {
    const int64_t row0 = j * (int64_t)B;
    // ---- D x into the tile (FP32 input, exact in FP64); rows >= n are zero ----
    if (cs.fmt == SRHT_DENSE) {
      const float* __restrict__ colp = cs.vals + lc * cs.ld;
      for (int i = tid; i < B; i += T64) {
        const int64_t row = row0 + i;
        double x = 0.0;
        if (row < n) {
          x = (double)colp[row];
          if ((__ldg(signs + (row >> 5)) >> (row & 31)) & 1u) x = -x;
        }
        tile64[i] = x;
      }
      __syncthreads();
    } else {
      for (int i = tid; i < B; i += T64) tile64[i] = 0.0;
      __syncthreads();
      const int64_t rowend = row0 + B;
      while (true) {
        const int64_t e = cptr + tid;
        bool in = false;
        if (e < cend) {
          const int64_t row = cs.rowidx[e];
          if (row < rowend) {
            in = true;
            double x = (double)cs.vals[e];
            if ((__ldg(signs + (row >> 5)) >> (row & 31)) & 1u) x = -x;
            atomicAdd(&tile64[row - row0], x);  // duplicates are summed
          }
        }
        const int cnt = __syncthreads_count(in);
        cptr += cnt;
        if (cnt < T64) break;
      }
    }
    // ---- z = H_B D x, radix-8 passes ----
    for (int bit = 0; bit < LOG_B; bit += 3) {
      wht_pass<LOG_B>(tile64, bit, LOG_B - bit < 3 ? LOG_B - bit : 3);
      __syncthreads();
    }
    // ---- pruned accumulate: acc_t += (-1)^{popc(k_mid & j)} z[k_lo] ----
    const uint32_t jl = (uint32_t)(j - j0);
#pragma unroll
    for (int q = 0; q < RPT64; ++q) {
      const double z = tile64[km[q] & 0xffffu];
      acc[q] += (__popc((km[q] >> 16) & jl) & 1) ? -z : z;
    }
    __syncthreads();
  }

  if (P.S_act == 1 && !P.part_out) {
#pragma unroll
    for (int q = 0; q < RPT64; ++q) {
      const int64_t t = t0 + (int64_t)q * T64 + tid;
      if (t < P.r) cs.out[lc * cs.ldo + t] = (float)(acc[q] * P.scale_f64);
    }
  } else {
    double* __restrict__ part = P.partials64 + (sl * P.total_cols + col) * P.r;
#pragma unroll
    for (int q = 0; q < RPT64; ++q) {
      const int64_t t = t0 + (int64_t)q * T64 + tid;
      if (t < P.r) part[t] = acc[q];
    }
  }
}

// Fixed-order signed sum of the FP64 slab partials, scaled by r^{-1/2} and rounded once.
__global__ void k_reduce_slabs_f64(const __grid_constant__ SketchParams P, int slab_shift) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t col = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (t >= P.r || col >= P.total_cols) return;
  const int64_t prob = col / P.cols_per_problem;
  const uint32_t ks = (uint32_t)(P.K[prob * P.r + t] >> slab_shift);
  double sum = 0.0;
  for (int64_t s = 0; s < P.S_act; ++s) {
    const double v = P.partials64[(s * P.total_cols + col) * P.r + t];
    sum += (__popc(ks & (uint32_t)(P.s_lo + s)) & 1) ? -v : v;
  }
  if (P.part_out) {  // row shard: unscaled partial
    P.part_out[col * P.ldp + t] = sum;
    return;
  }
  const bool second = col >= P.ncols0;
  const ColSrc& cs = second ? P.src[1] : P.src[0];
  const int64_t lc = second ? col - P.ncols0 : col;
  cs.out[lc * cs.ldo + t] = (float)(sum * P.scale_f64);
}

template <int LOG_B>
cudaError_t launch_b64(const SketchParams& sp, int64_t groups, cudaStream_t stream) {
  const size_t smem = ((size_t)1 << LOG_B) * sizeof(double);
  static std::atomic<uint64_t> attr_done{0};
  const cudaError_t e = set_max_dyn_smem_once(k_sketch_f64<LOG_B>, (int)smem, attr_done);
  if (e != cudaSuccess) return e;
  const int64_t items = sp.total_cols * sp.S_act * groups;
  for (int64_t done = 0; done < items;) {
    const int64_t cnt = items - done < 0x7fffffff ? items - done : 0x7fffffff;
    k_sketch_f64<LOG_B><<<(unsigned)cnt, T64, smem, stream>>>(sp, groups);
    done += cnt;
  }
  return cudaGetLastError();
}

}  // namespace

int64_t f64_groups(int64_t r) { return (r + (int64_t)RPT64 * T64 - 1) / ((int64_t)RPT64 * T64); }

cudaError_t launch_sketch_f64(const srht_plan* P, const SketchParams& sp, cudaStream_t stream) {
  if (sp.total_cols <= 0) return cudaSuccess;
  const int64_t groups = f64_groups(sp.r);
  cudaError_t e;
  const int slot = (g_prof.on && g_prof.used < g_prof.capacity) ? g_prof.used++ : -1;
  if (slot >= 0) cudaEventRecord(g_prof.ev[2 * slot], stream);
  switch (P->log_b) {
    case 10: e = launch_b64<10>(sp, groups, stream); break;
    case 11: e = launch_b64<11>(sp, groups, stream); break;
    case 12: e = launch_b64<12>(sp, groups, stream); break;
    case 13: e = launch_b64<13>(sp, groups, stream); break;
    case 14: e = launch_b64<14>(sp, groups, stream); break;
    default: return cudaErrorInvalidValue;
  }
  if (slot >= 0) cudaEventRecord(g_prof.ev[2 * slot + 1], stream);
  g_last_kernel = 4;
  if (e != cudaSuccess || (sp.S_act == 1 && !sp.part_out)) return e;
  const int64_t zc = (sp.total_cols + 65534) / 65535;
  dim3 grid((unsigned)((sp.r + 255) / 256), (unsigned)(sp.total_cols < 65535 ? sp.total_cols : 65535), (unsigned)zc);
  k_reduce_slabs_f64<<<grid, 256, 0, stream>>>(sp, P->log_b + P->log_j);
  return cudaGetLastError();
}

}  // namespace srht
