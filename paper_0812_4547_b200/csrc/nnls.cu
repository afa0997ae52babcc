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
// solve is Q_PP z_P = q_P with a Cholesky factor L of Q_PP (the normal equations of the LS
// solve the oracle does by QR; same solution for a full-column-rank SA, which r >= d+1 makes
// the generic case).  L is kept up to date instead of refactored: an entering index is
// appended (one forward substitution, O(m^2)), a dropped one is deleted and the trailing
// block restored by a rank-1 Cholesky update (O(m^2)); the passive set is stored in
// insertion order, which changes only the rounding, not the solution.
//
// One CTA (256 threads) per problem, FP64 throughout: all threads for the dual w = q - Q x
// and the argmax/argmin reductions, warp 0 for the factor updates and the triangular solves.
// This incremental form runs when L fits in shared memory (d <= 160); larger d uses
// k_nnls_lh_refactor below with the factor in the caller's workspace.  Q is read from G (L2).
#include <cuda_runtime.h>
#include <math.h>

#include "internal.cuh"

namespace srht {
namespace {

constexpr int NT = 256;
// x, z, w, zt (d doubles each) + order (d ints) + passive, skipped (d bytes each), in doubles
#define NNLS_VEC_DOUBLES(d) (4 * (int64_t)(d) + ((int64_t)(d) * 6 + 7) / 8 + 1)

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

// ---- warp-0 helpers on the factor L (column-major, ld = d: L[i][j] at F[i + j*d]) ----

// Append index t: row m of L = L^{-1} Q[order, t], diagonal sqrt(Q_tt - |row|^2).
// Returns false (L unchanged) when the new pivot is not positive.
__device__ bool chol_append(double* F, int d, int* order, int m, int t, const double* G, int64_t ldg) {
  const int lane = threadIdx.x & 31;
  for (int a = 0; a < m; ++a) {
    double acc = 0.0;
    for (int b = lane; b < a; b += 32) acc += F[a + b * d] * F[m + b * d];
#pragma unroll
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) F[m + a * d] = (G[order[a] + (int64_t)t * ldg] - acc) / F[a + a * d];
    __syncwarp();
  }
  double ss = 0.0;
  for (int b = lane; b < m; b += 32) ss += F[m + b * d] * F[m + b * d];
#pragma unroll
  for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  const double dd = G[t + (int64_t)t * ldg] - ss;
  if (!(dd > 0.0)) return false;
  if (lane == 0) {
    F[m + m * d] = sqrt(dd);
    order[m] = t;
  }
  __syncwarp();
  return true;
}

// Delete position k of the passive list (m entries): shift rows/columns, then restore the
// trailing block with the rank-1 update L' L'^T = L22 L22^T + x x^T, x = old L[k+1.., k].
__device__ void chol_delete(double* F, int d, int* order, int m, int k, double* xt) {
  const int lane = threadIdx.x & 31;
  const int p = m - 1 - k;
  for (int i = lane; i < p; i += 32) xt[i] = F[k + 1 + i + k * d];
  __syncwarp();
  for (int j = 0; j < k; ++j)  // columns left of k: rows k+1.. move up by one
    for (int i0 = k; i0 < m - 1; i0 += 32) {
      const int i = i0 + lane;
      const double v = i < m - 1 ? F[i + 1 + j * d] : 0.0;
      __syncwarp();
      if (i < m - 1) F[i + j * d] = v;
      __syncwarp();
    }
  for (int j = k; j < m - 1; ++j)  // trailing block: (i+1, j+1) -> (i, j), lower triangle
    for (int i0 = j; i0 < m - 1; i0 += 32) {
      const int i = i0 + lane;
      const double v = i < m - 1 ? F[i + 1 + (j + 1) * d] : 0.0;
      __syncwarp();
      if (i < m - 1) F[i + j * d] = v;
      __syncwarp();
    }
  for (int i = k + lane; i < m - 1; i += 32) {
    const int o = order[i + 1];
    __syncwarp();
    order[i] = o;
  }
  __syncwarp();
  for (int j = 0; j < p; ++j) {  // rank-1 update of rows/columns k..m-2
    const int jj = k + j;
    const double ljj = F[jj + jj * d], xj = xt[j];
    const double rr = sqrt(ljj * ljj + xj * xj);
    const double c = rr / ljj, s = xj / ljj;
    for (int i = j + 1 + lane; i < p; i += 32) {
      const double lij = (F[k + i + jj * d] + s * xt[i]) / c;
      xt[i] = c * xt[i] - s * lij;
      F[k + i + jj * d] = lij;
    }
    __syncwarp();
    if (lane == 0) F[jj + jj * d] = rr;
    __syncwarp();
  }
}

// z[order[a]] for L L^T z_P = q_P (forward then back substitution); y kept in zt.
__device__ void chol_solve(const double* F, int d, const int* order, int m, const double* G, int64_t ldg, double* zt,
                           double* z) {
  const int lane = threadIdx.x & 31;
  for (int a = 0; a < m; ++a) {
    double acc = 0.0;
    for (int b = lane; b < a; b += 32) acc += F[a + b * d] * zt[b];
#pragma unroll
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) zt[a] = (G[order[a] + (int64_t)d * ldg] - acc) / F[a + a * d];
    __syncwarp();
  }
  for (int a = m - 1; a >= 0; --a) {
    double acc = 0.0;
    for (int b = a + 1 + lane; b < m; b += 32) acc += F[b + a * d] * zt[b];
#pragma unroll
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) zt[a] = (zt[a] - acc) / F[a + a * d];
    __syncwarp();
  }
  for (int a = lane; a < m; a += 32) z[order[a]] = zt[a];
  __syncwarp();
}

__global__ void __launch_bounds__(NT) k_nnls_lh(int d, const double* __restrict__ Gall, int64_t ldg, int64_t stride_g,
                                               double* __restrict__ xall, int64_t stride_x, int32_t* __restrict__ iters,
                                               double* __restrict__ ws, int64_t batch, int fac_in_smem) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ NnlsSmem s;
  const int64_t p = blockIdx.x + (int64_t)blockIdx.y * 65535;
  if (p >= batch) return;
  const double* __restrict__ G = Gall + p * stride_g;  // Q[i][j] = G[i + j*ldg], q[i] = G[i + d*ldg]
  // shared: x, z, w, zt (d doubles each), order (d ints), passive / skipped (d bytes each)
  double* x = dsm;
  double* z = x + d;
  double* w = z + d;
  double* zt = w + d;
  int* order = reinterpret_cast<int*>(zt + d);
  unsigned char* passive = reinterpret_cast<unsigned char*>(order + d);
  unsigned char* skipped = passive + d;
  double* F = fac_in_smem ? dsm + NNLS_VEC_DOUBLES(d) : ws + p * (int64_t)d * d;
  const int tid = threadIdx.x;

  for (int i = tid; i < d; i += NT) {
    x[i] = 0.0;
    z[i] = 0.0;
    passive[i] = 0;
    skipped[i] = 0;
  }
  if (tid == 0) s.m = 0;
  double qm = 0.0;  // tol = 1e-10 max|q|
  for (int i = tid; i < d; i += NT) qm = fmax(qm, fabs(G[i + d * ldg]));
  block_argmax(qm, 0, true, s);
  const double tol = 1e-10 * fmax(s.red_v[0], 2.2250738585072014e-308);
  const int max_iter = 30 * (d > 1 ? d : 1);
  int it = 0;
  int status = 0;
  while (true) {
    for (int i = tid; i < d; i += NT) {  // w = q - Q x (column i of G = row i of Q)
      double acc = G[i + d * ldg];
      for (int j = 0; j < d; ++j) acc -= G[i + j * ldg] * x[j];
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
    if (tid < 32) {
      const bool ok = chol_append(F, d, order, s.m, t, G, ldg);
      if (tid == 0) {
        s.flag = ok ? 0 : 1;
        if (ok) {
          s.m += 1;
          passive[t] = 1;
        }
      }
    }
    __syncthreads();
    if (s.flag) {  // Q_PP not positive definite: rank-deficient passive set
      status = -3;
      break;
    }
    int inner = 0;
    while (true) {
      ++inner;
      if (inner > 10 * d + 10) {
        status = -2;
        break;
      }
      if (tid < 32) chol_solve(F, d, order, s.m, G, ldg, zt, z);
      __syncthreads();
      const int m = s.m;
      int bad = 0;
      for (int a = tid; a < m; a += NT) bad |= z[order[a]] <= 0.0;
      bad = __syncthreads_or(bad);
      if (!bad) {
        for (int j = tid; j < d; j += NT) {
          x[j] = passive[j] ? z[j] : 0.0;
          skipped[j] = 0;
        }
        __syncthreads();
        break;
      }
      if (inner == 1 && z[t] <= 0.0) {  // degenerate entry: t is the last appended; pop it
        if (tid == 0) {
          passive[t] = 0;
          skipped[t] = 1;
          s.m -= 1;
        }
        __syncthreads();
        break;
      }
      // step back: alpha = min over passive j with z_j <= 0 of x_j / (x_j - z_j)
      double rv = INFINITY;
      int ri = 0x7fffffff;
      for (int a = tid; a < m; a += NT) {
        const int j = order[a];
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
        if (!passive[j]) continue;
        double xj = x[j] + alpha * (z[j] - x[j]);
        if (xj <= 0.0 || j == jstar) xj = 0.0;
        x[j] = xj;
      }
      __syncthreads();
      if (tid < 32) {  // delete the dropped positions, highest first
        int mm = s.m;
        for (int a = mm - 1; a >= 0; --a) {
          const int j = order[a];
          if (x[j] == 0.0) {
            chol_delete(F, d, order, mm, a, zt);
            if (tid == 0) passive[j] = 0;
            --mm;
          }
        }
        if (tid == 0) s.m = mm;
      }
      __syncthreads();
      if (s.m == 0) break;
    }
    if (status) break;
  }
  double* xo = xall + p * stride_x;
  for (int j = tid; j < d; j += NT) xo[j] = x[j] < 1e-14 ? 0.0 : x[j];
  if (tid == 0 && iters) iters[p] = status ? status : it;
}

// Large d (factor in the workspace, L2): the passive-set system is refactored from scratch in
// every inner step (O(m^3) spread over the CTA); the incremental updates of k_nnls_lh would
// serialise O(m^2) dependent L2 round trips per step there.
__global__ void __launch_bounds__(NT) k_nnls_lh_refactor(int d, const double* __restrict__ Gall, int64_t ldg, int64_t stride_g,
                                               double* __restrict__ xall, int64_t stride_x, int32_t* __restrict__ iters,
                                               double* __restrict__ ws, int64_t batch) {
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
  double* F = ws + p * (int64_t)d * d;  // large d: the factor lives in the workspace
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
  size_t b = (size_t)NNLS_VEC_DOUBLES(d) * sizeof(double);
  if (fac_in_smem) b += (size_t)d * d * sizeof(double);
  return b;
}

bool nnls_factor_in_smem(int64_t d) { return nnls_smem_bytes(d, true) <= 200 * 1024; }

cudaError_t launch_nnls_gram(int64_t d, int64_t batch, const double* G, int64_t ldg, int64_t stride_g, double* x,
                             int64_t stride_x, int32_t* iters, double* ws, cudaStream_t stream) {
  if (d <= 0 || batch <= 0) return cudaSuccess;
  const bool fs = nnls_factor_in_smem(d);
  const dim3 grid((unsigned)(batch < 65535 ? batch : 65535), (unsigned)((batch + 65534) / 65535));
  if (!fs) {
    const size_t smem = (size_t)(3 * d + (d * 6 + 15) / 8 + 1) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_nnls_lh_refactor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_nnls_lh_refactor<<<grid, NT, smem, stream>>>((int)d, G, ldg, stride_g, x, stride_x, iters, ws, batch);
    return cudaGetLastError();
  }
  const size_t smem = nnls_smem_bytes(d, true);
  cudaError_t e = cudaFuncSetAttribute(k_nnls_lh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_nnls_lh<<<grid, NT, smem, stream>>>((int)d, G, ldg, stride_g, x, stride_x, iters, ws, batch, 1);
  return cudaGetLastError();
}

}  // namespace srht
