// Batched Lawson-Hanson NNLS on the Gram form (Algorithm 1 step 5 through the QP form of
// Section 3.4), sm_100a.
//
// For each problem p: x = argmin_{x >= 0} x^T Q x - 2 q^T x with G_p = [[Q, q], [q^T, .]]
// (srht_gram of the sketch [SA | Sb]), i.e. min ||SA x - Sb||.  The active-set rules are
// those of the oracle (reading R13, oracle/nnls.py): dual w = q - Q x; enter argmax w over
// the candidates (smallest index on ties), stop when max w <= 1e-10 max|q|; inner loop:
// z = passive-set solution, step back with alpha = min x_j / (x_j - z_j) (smallest index on
// ties) and drop every passive x_j <= 0; a degenerate entry (z_t <= 0 on entry) is skipped
// until x changes; at most 30 d outer iterations; x < 1e-14 snapped to 0.  The passive-set
// solve is Q_PP z_P = q_P by Cholesky (the normal equations of the LS solve the oracle does
// by QR; same solution for a full-column-rank SA, which r >= d+1 makes the generic case).
//
// One CTA (256 threads) per problem, FP64 throughout; the Cholesky factor lives in shared
// memory when d <= 160 and in the caller's workspace otherwise.  Q is read from G (L2).
#include <cuda_runtime.h>
#include <math.h>

#include "internal.cuh"

namespace srht {
namespace {

constexpr int NT = 256;

struct NnlsSmem {
  double red_v[NT / 32];
  int red_i[NT / 32];
  double alpha;
  int t, flag, m;
};

// Block-wide max of v over threads with ok, smallest index on ties; result in s.red_v[0] / s.red_i[0].
__device__ void block_argmax(double v, int i, bool ok, NnlsSmem& s) {
  if (!ok) {
    v = -INFINITY;
    i = 0x7fffffff;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, off);
    const int oi = __shfl_xor_sync(0xffffffffu, i, off);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    s.red_v[w] = v;
    s.red_i[w] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < NT / 32; ++k)
      if (s.red_v[k] > s.red_v[0] || (s.red_v[k] == s.red_v[0] && s.red_i[k] < s.red_i[0])) {
        s.red_v[0] = s.red_v[k];
        s.red_i[0] = s.red_i[k];
      }
  }
  __syncthreads();
}

// Block-wide min (smallest index on ties).
__device__ void block_argmin(double v, int i, bool ok, NnlsSmem& s) {
  block_argmax(ok ? -v : 0.0, i, ok, s);
  if (threadIdx.x == 0) s.red_v[0] = -s.red_v[0];
  __syncthreads();
}

__global__ void __launch_bounds__(NT) k_nnls_lh(int d, const double* __restrict__ Gall, int64_t ldg, int64_t stride_g,
                                               double* __restrict__ xall, int64_t stride_x, int32_t* __restrict__ iters,
                                               double* __restrict__ ws, int64_t batch, int fac_in_smem) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ NnlsSmem s;
  const int64_t p = blockIdx.x + (int64_t)blockIdx.y * 65535;
  if (p >= batch) return;
  const double* __restrict__ G = Gall + p * stride_g;  // Q[i][j] = G[i + j*ldg], q[i] = G[i + d*ldg]
  // shared: x, z, w (d each), P index list (d ints), flags; factor F (m x m, ld = d) in smem or ws
  double* x = dsm;
  double* z = x + d;
  double* w = z + d;
  int* idx = reinterpret_cast<int*>(w + d);
  unsigned char* passive = reinterpret_cast<unsigned char*>(idx + d);
  unsigned char* skipped = passive + d;
  double* F = fac_in_smem ? reinterpret_cast<double*>(dsm + 3 * d + (d * 6 + 15) / 8 + 1) : ws + p * (int64_t)d * d;
  const int tid = threadIdx.x;

  for (int i = tid; i < d; i += NT) {
    x[i] = 0.0;
    passive[i] = 0;
    skipped[i] = 0;
  }
  // tol = 1e-10 max|q|
  double qm = 0.0;
  for (int i = tid; i < d; i += NT) qm = fmax(qm, fabs(G[i + d * ldg]));
  block_argmax(qm, 0, true, s);
  const double tol = 1e-10 * fmax(s.red_v[0], 2.2250738585072014e-308);
  const int max_iter = 30 * (d > 1 ? d : 1);
  int it = 0;
  int status = 0;
  while (true) {
    // w = q - Q x
    for (int i = tid; i < d; i += NT) {
      double acc = G[i + d * ldg];
      for (int j = 0; j < d; ++j) acc -= G[i + j * ldg] * x[j];  // column i of G = row i of Q
      w[i] = acc;
    }
    __syncthreads();
    double bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = tid; i < d; i += NT)
      if (!passive[i] && !skipped[i] && (w[i] > bv || (w[i] == bv && i < bi))) {
        bv = w[i];
        bi = i;
      }
    block_argmax(bv, bi, bi != 0x7fffffff, s);
    if (s.red_i[0] == 0x7fffffff || s.red_v[0] <= tol) break;
    if (++it > max_iter) {
      status = -1;
      break;
    }
    const int t = s.red_i[0];
    if (tid == 0) passive[t] = 1;
    __syncthreads();
    int inner = 0;
    while (true) {
      ++inner;
      if (inner > 10 * d + 10) {
        status = -2;
        break;
      }
      // passive index list, ascending
      if (tid == 0) {
        int m = 0;
        for (int j = 0; j < d; ++j)
          if (passive[j]) idx[m++] = j;
        s.m = m;
      }
      __syncthreads();
      const int m = s.m;
      // F = Q_PP (lower triangle), then Cholesky in place: F F^T = Q_PP
      for (int e = tid; e < m * m; e += NT) {
        const int a = e / m, b = e % m;
        if (b <= a) F[a + b * d] = G[idx[a] + idx[b] * ldg];
      }
      __syncthreads();
      for (int k = 0; k < m; ++k) {
        if (tid == 0) {
          const double dk = F[k + k * d];
          s.flag = dk > 0.0 ? 0 : 1;
          F[k + k * d] = sqrt(dk > 0.0 ? dk : 1.0);
        }
        __syncthreads();
        if (s.flag) break;
        const double piv = F[k + k * d];
        for (int a = k + 1 + tid; a < m; a += NT) F[a + k * d] /= piv;
        __syncthreads();
        const int rest = m - k - 1;
        for (int e = tid; e < rest * rest; e += NT) {
          const int a = k + 1 + e / rest, b = k + 1 + e % rest;
          if (b <= a) F[a + b * d] -= F[a + k * d] * F[b + k * d];
        }
        __syncthreads();
      }
      if (s.flag) {  // Q_PP not positive definite: rank-deficient passive set
        status = -3;
        break;
      }
      // z_P: forward (F y = q_P) and back (F^T z = y) substitution, warp 0
      if (tid < 32) {
        for (int a = 0; a < m; ++a) {
          double acc = 0.0;
          for (int b = tid; b < a; b += 32) acc += F[a + b * d] * z[idx[b]];
#pragma unroll
          for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
          if (tid == 0) z[idx[a]] = (G[idx[a] + d * ldg] - acc) / F[a + a * d];
          __syncwarp();
        }
        for (int a = m - 1; a >= 0; --a) {
          double acc = 0.0;
          for (int b = a + 1 + tid; b < m; b += 32) acc += F[b + a * d] * z[idx[b]];
#pragma unroll
          for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
          if (tid == 0) z[idx[a]] = (z[idx[a]] - acc) / F[a + a * d];
          __syncwarp();
        }
      }
      __syncthreads();
      for (int j = tid; j < d; j += NT)
        if (!passive[j]) z[j] = 0.0;
      // all z_P > 0?
      int bad = 0;
      for (int a = tid; a < m; a += NT) bad |= z[idx[a]] <= 0.0;
      bad = __syncthreads_or(bad);
      if (!bad) {
        for (int j = tid; j < d; j += NT) {
          x[j] = z[j];
          skipped[j] = 0;
        }
        __syncthreads();
        break;
      }
      if (inner == 1 && z[t] <= 0.0) {  // degenerate entry: leave x, do not offer t until x changes
        if (tid == 0) {
          passive[t] = 0;
          skipped[t] = 1;
        }
        __syncthreads();
        break;
      }
      // step back: alpha = min over passive j with z_j <= 0 of x_j / (x_j - z_j)
      double rv = INFINITY;
      int ri = 0x7fffffff;
      for (int a = tid; a < m; a += NT) {
        const int j = idx[a];
        if (z[j] <= 0.0) {
          const double ratio = x[j] / (x[j] - z[j]);
          if (ratio < rv || (ratio == rv && j < ri)) {
            rv = ratio;
            ri = j;
          }
        }
      }
      block_argmin(rv, ri, ri != 0x7fffffff, s);
      const double alpha = s.red_v[0];
      const int jstar = s.red_i[0];
      for (int j = tid; j < d; j += NT) {
        double xj = x[j] + alpha * (z[j] - x[j]);
        if (passive[j] && (xj <= 0.0 || j == jstar)) {
          xj = 0.0;
          passive[j] = 0;
        }
        x[j] = xj;
      }
      int any = 0;
      for (int j = tid; j < d; j += NT) any |= passive[j];
      any = __syncthreads_or(any);
      if (!any) break;
    }
    if (status) break;
  }
  double* xo = xall + p * stride_x;
  for (int j = tid; j < d; j += NT) xo[j] = x[j] < 1e-14 ? 0.0 : x[j];
  if (tid == 0 && iters) iters[p] = status ? status : it;
}

}  // namespace

size_t nnls_smem_bytes(int64_t d, bool fac_in_smem) {
  size_t b = (size_t)(3 * d + (d * 6 + 15) / 8 + 1) * sizeof(double);
  if (fac_in_smem) b += (size_t)d * d * sizeof(double);
  return b;
}

bool nnls_factor_in_smem(int64_t d) { return nnls_smem_bytes(d, true) <= 200 * 1024; }

cudaError_t launch_nnls_gram(int64_t d, int64_t batch, const double* G, int64_t ldg, int64_t stride_g, double* x,
                             int64_t stride_x, int32_t* iters, double* ws, cudaStream_t stream) {
  if (d <= 0 || batch <= 0) return cudaSuccess;
  const bool fs = nnls_factor_in_smem(d);
  const size_t smem = nnls_smem_bytes(d, fs);
  cudaError_t e = cudaFuncSetAttribute(k_nnls_lh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)(batch < 65535 ? batch : 65535), (unsigned)((batch + 65534) / 65535));
  k_nnls_lh<<<grid, NT, smem, stream>>>((int)d, G, ldg, stride_g, x, stride_x, iters, ws, batch, fs ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace srht
