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
// One CTA (256 threads) per problem, FP64 throughout (k_nnls_lh_big): all threads for the
// dual w = q - Q x and the argmax/argmin reductions; the factor is row-major, in shared
// memory while it fits (d <= 156) else in the caller's workspace, and the triangular
// solves are blocked (32-row diagonal blocks in one warp's registers, the rest CTA-wide).
// Q is read from G (L2).
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>

#include "internal.cuh"

namespace srht {
namespace {

constexpr int NT = 256;

struct NnlsSmem {
  double red_v[NT / 32];
  int red_i[NT / 32];
  double alpha;
  int t, flag, m;
  int yok;  // y = L^{-1} q_P (yv) is current for the factor
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

// ---------------------------------------------------------------------------------------
// The incremental Lawson-Hanson with the factor ROW-major (L[a][b] at F[a*d + b], b <= a) and
// CTA-wide blocked triangular solves, so every L2 access is a coalesced row segment or a
// 32 x 32 diagonal block held in one warp's registers: O(m^2 / 32) sequential steps per
// solve instead of O(m^2) dependent round trips.  A deletion removes row/column k (in place
// in shared memory, else by copying into the second workspace slot), then restores the
// trailing block with Givens rotations.
constexpr int BK = 32;
// x, z, w, zt, bv, yv (d doubles each) + order (d ints) + passive, skipped (d bytes each), in doubles
#define NNLS_BIG_VEC_DOUBLES(d) (6 * (int64_t)(d) + ((int64_t)(d) * 6 + 7) / 8 + 1)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// y[0..m) = L^{-1} b[0..m)   (b, y, part in shared memory; y may not alias b)
__device__ void big_fwd(const double* __restrict__ F, int d, int m, const double* b, double* y, double* part) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int a0 = 0; a0 < m; a0 += BK) {
    const int nb = m - a0 < BK ? m - a0 : BK;
    for (int i = wid; i < nb; i += NT / 32) {  // part[i] = sum_{c < a0} L[a0+i][c] y[c]
      const double* row = F + (size_t)(a0 + i) * d;
      double acc = 0.0;
      for (int c = lane; c < a0; c += 32) acc += row[c] * y[c];
      acc = warp_sum(acc);
      if (lane == 0) part[i] = acc;
    }
    __syncthreads();
    if (wid == 0) {  // diagonal block: lane j holds row a0+j; column sweep
      const bool act = lane < nb;
      double Lr[BK];
#pragma unroll
      for (int i = 0; i < BK; ++i) Lr[i] = (act && i <= lane) ? F[(size_t)(a0 + lane) * d + a0 + i] : 1.0;
      double rj = act ? b[a0 + lane] - part[lane] : 0.0, yj = 0.0;
#pragma unroll
      for (int i = 0; i < BK; ++i) {
        if (i < nb) {
          const double yi = __shfl_sync(0xffffffffu, rj / Lr[i], i);
          if (lane == i) yj = yi;
          if (lane > i) rj -= Lr[i] * yi;
        }
      }
      if (act) y[a0 + lane] = yj;
    }
    __syncthreads();
  }
}

// z[0..m) = L^{-T} y[0..m)   (y is consumed)
__device__ void big_bwd(const double* __restrict__ F, int d, int m, double* y, double* z) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int a1 = m; a1 > 0;) {
    const int a0 = ((a1 - 1) / BK) * BK, nb = a1 - a0;
    if (wid == 0) {  // diagonal block: lane j holds column a0+j; column sweep from the bottom
      const bool act = lane < nb;
      double Lc[BK];
#pragma unroll
      for (int i = 0; i < BK; ++i) Lc[i] = (act && i < nb && i >= lane) ? F[(size_t)(a0 + i) * d + a0 + lane] : 1.0;
      double rj = act ? y[a0 + lane] : 0.0, zj = 0.0;
#pragma unroll
      for (int i = BK - 1; i >= 0; --i) {
        if (i < nb) {
          const double zi = __shfl_sync(0xffffffffu, rj / Lc[i], i);
          if (lane == i) zj = zi;
          if (lane < i) rj -= Lc[i] * zi;
        }
      }
      if (act) z[a0 + lane] = zj;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < a0; c += NT) {  // y[c] -= sum_{b in block} L[b][c] z[b]
      double acc = 0.0;
      for (int b = a0; b < a1; ++b) acc += F[(size_t)b * d + c] * z[b];
      y[c] -= acc;
    }
    __syncthreads();
    a1 = a0;
  }
}

template <bool SMEM_F>
__global__ void __launch_bounds__(NT) k_nnls_lh_big(int d, const double* __restrict__ Gall, int64_t ldg, int64_t stride_g,
                                                   double* __restrict__ xall, int64_t stride_x, int32_t* __restrict__ iters,
                                                   double* __restrict__ ws, int64_t batch) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ NnlsSmem s;
  __shared__ double part[BK];
  const int64_t p = blockIdx.x + (int64_t)blockIdx.y * 65535;
  if (p >= batch) return;
  const double* __restrict__ G = Gall + p * stride_g;  // Q[i][j] = G[i + j*ldg], q[i] = G[i + d*ldg]
  double* x = dsm;
  double* z = x + d;
  double* w = z + d;
  double* zt = w + d;
  double* bv = zt + d;
  double* yv = bv + d;  // y = L^{-1} q_P, kept across appends (one new entry per append)
  int* order = reinterpret_cast<int*>(yv + d);
  unsigned char* passive = reinterpret_cast<unsigned char*>(order + d);
  unsigned char* skipped = passive + d;
  // factor: shared memory after the vectors (SMEM_F, d <= 156), else two workspace slots
  // (a deletion copies between them)
  double* F = SMEM_F ? dsm + NNLS_BIG_VEC_DOUBLES(d) : ws + p * 2 * (int64_t)d * d;
  double* F2 = F + (int64_t)d * d;
  const int tid = threadIdx.x;

  for (int i = tid; i < d; i += NT) {
    x[i] = 0.0;
    z[i] = 0.0;
    passive[i] = 0;
    skipped[i] = 0;
  }
  if (tid == 0) {
    s.m = 0;
    s.yok = 1;
  }
  double qm = 0.0;  // tol = 1e-10 max|q|
  for (int i = tid; i < d; i += NT) qm = fmax(qm, fabs(G[i + d * ldg]));
  block_argmax(qm, 0, true, s);
  const double tol = 1e-10 * fmax(s.red_v[0], 2.2250738585072014e-308);
  const int max_iter = 30 * (d > 1 ? d : 1);
  int it = 0;
  int status = 0;
  while (true) {
    const int mp = s.m;
    for (int i = tid; i < d; i += NT) {  // w = q - Q x (column i of G = row i of Q)
      double acc = G[i + d * ldg];
      for (int a = 0; a < mp; ++a) {  // x is zero off the passive set
        const int j = order[a];
        acc -= G[i + j * ldg] * x[j];
      }
      w[i] = acc;
    }
    __syncthreads();
    double bvv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = tid; i < d; i += NT)
      if (!passive[i] && !skipped[i] && (w[i] > bvv || (w[i] == bvv && i < bi))) {
        bvv = w[i];
        bi = i;
      }
    block_argmax(bvv, bi, bi != 0x7fffffff, s);
    if (s.red_i[0] == 0x7fffffff || s.red_v[0] <= tol) break;
    if (++it > max_iter) {
      status = -1;
      break;
    }
    const int t = s.red_i[0];
    {  // append t: row m of L = L^{-1} Q[order, t], diagonal sqrt(Q_tt - |row|^2)
      const int m = s.m;
      for (int a = tid; a < m; a += NT) bv[a] = G[order[a] + (int64_t)t * ldg];
      __syncthreads();
      big_fwd(F, d, m, bv, zt, part);
      double ss = 0.0, sy = 0.0;  // |row|^2 and row . y (the new entry of y)
      for (int a = tid; a < m; a += NT) {
        ss += zt[a] * zt[a];
        sy += zt[a] * yv[a];
      }
      ss = warp_sum(ss);
      sy = warp_sum(sy);
      __syncthreads();
      if ((tid & 31) == 0) {
        s.red_v[tid >> 5] = ss;
        part[tid >> 5] = sy;
      }
      __syncthreads();
      if (tid == 0) {
        double tot = 0.0, toty = 0.0;
        for (int k = 0; k < NT / 32; ++k) {
          tot += s.red_v[k];
          toty += part[k];
        }
        const double dd = G[t + (int64_t)t * ldg] - tot;
        s.flag = dd > 0.0 ? 0 : 1;
        if (dd > 0.0) {
          const double lmm = sqrt(dd);
          F[(size_t)m * d + m] = lmm;
          if (s.yok) yv[m] = (G[t + (int64_t)d * ldg] - toty) / lmm;
          order[m] = t;
          passive[t] = 1;
          s.m = m + 1;
        }
      }
      for (int a = tid; a < m; a += NT) F[(size_t)m * d + a] = zt[a];
      __syncthreads();
    }
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
      const int m = s.m;
      if (s.yok) {  // forward half maintained incrementally: y = L^{-1} q_P
        for (int a = tid; a < m; a += NT) zt[a] = yv[a];
        __syncthreads();
      } else {
        for (int a = tid; a < m; a += NT) bv[a] = G[order[a] + (int64_t)d * ldg];
        __syncthreads();
        big_fwd(F, d, m, bv, zt, part);
        for (int a = tid; a < m; a += NT) yv[a] = zt[a];
        __syncthreads();
        if (tid == 0) s.yok = 1;
      }
      big_bwd(F, d, m, zt, bv);  // z_P (in order positions) -> bv
      for (int a = tid; a < m; a += NT) z[order[a]] = bv[a];
      __syncthreads();
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
      double rv = INFINITY;  // step back: alpha = min over passive j with z_j <= 0 of x_j / (x_j - z_j)
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
      // delete the dropped positions, highest first
      for (int k = s.m - 1; k >= 0; --k) {
        if (x[order[k]] != 0.0) continue;  // uniform (shared x, synchronised)
        const int mm = s.m, pp = mm - 1 - k;
        for (int i = tid; i < pp; i += NT) zt[i] = F[(size_t)(k + 1 + i) * d + k];  // old column k below k
        if (SMEM_F) {  // in place: rows k.. take the next row without column k, one row per step
          __syncthreads();
          for (int i = k; i < mm - 1; ++i) {
            double v0 = 0.0, v1 = 0.0;  // row i has i+1 <= 2 NT entries
            const int j0 = tid, j1 = tid + NT;
            if (j0 <= i) v0 = F[(size_t)(i + 1) * d + (j0 < k ? j0 : j0 + 1)];
            if (j1 <= i) v1 = F[(size_t)(i + 1) * d + (j1 < k ? j1 : j1 + 1)];
            __syncthreads();
            if (j0 <= i) F[(size_t)i * d + j0] = v0;
            if (j1 <= i) F[(size_t)i * d + j1] = v1;
          }
        } else
        for (int e = tid; e < (mm - 1) * mm / 2 + mm; e += NT) {  // copy without row/column k
          // e enumerates (i, j), j <= i < mm-1, row by row: i = floor((sqrt(8e+1)-1)/2)
          int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
          while ((i + 1) * (i + 2) / 2 <= e) ++i;
          while (i * (i + 1) / 2 > e) --i;
          const int j = e - i * (i + 1) / 2;
          if (i >= mm - 1) continue;
          const int si = i < k ? i : i + 1, sj = j < k ? j : j + 1;
          F2[(size_t)i * d + j] = F[(size_t)si * d + sj];
        }
        __syncthreads();
        if (tid == 0) {
          passive[order[k]] = 0;
          for (int a = k; a < mm - 1; ++a) order[a] = order[a + 1];
          s.m = mm - 1;
          s.yok = 0;  // the factor changed from row k on
        }
        if (!SMEM_F) {  // the copy is the factor now
          double* tmp = F;
          F = F2;
          F2 = tmp;
        }
        for (int j = 0; j < pp; ++j) {  // rank-1 update L22 L22^T + x x^T of rows/columns k..mm-2
          const int jj = k + j;
          __syncthreads();  // step j-1's updates (zt, column jj-1) are visible
          if (tid == 0) {
            const double ljj = F[(size_t)jj * d + jj], xj = zt[j];
            const double rr = sqrt(ljj * ljj + xj * xj);
            s.alpha = rr / ljj;  // c
            part[0] = xj / ljj;  // s
            F[(size_t)jj * d + jj] = rr;
          }
          __syncthreads();
          const double c = s.alpha, sn = part[0];
          for (int i = j + 1 + tid; i < pp; i += NT) {
            const double lij = (F[(size_t)(k + i) * d + jj] + sn * zt[i]) / c;
            zt[i] = c * zt[i] - sn * lij;
            F[(size_t)(k + i) * d + jj] = lij;
          }
        }
        __syncthreads();
      }
      if (s.m == 0) break;
    }
    if (status) break;
  }
  double* xo = xall + p * stride_x;
  for (int j = tid; j < d; j += NT) xo[j] = x[j] < 1e-14 ? 0.0 : x[j];
  if (tid == 0 && iters) iters[p] = status ? status : it;
}
// ---------------------------------------------------------------------------------------
// Block principal pivoting (Portugal, Judice & Vicente 1994; Kim & Park 2011) on the Gram form:
// the same NNLS optimum (unique for a full-column-rank SA, the generic case r >= d+1) reached in
// a few exchanges of whole index sets instead of one Lawson-Hanson step per entering index.
// With F the passive set: x_F = Q_FF^{-1} q_F, x = 0 off F, y = Q x - q (y = -w of Lawson-Hanson);
// infeasible V = {i in F: x_i < 0} U {i not in F: y_i < -tol}, tol = 1e-10 max|q| (the
// Lawson-Hanson stopping rule); V empty is the KKT point.  Exchange all of V while |V| keeps
// decreasing (or for up to 3 non-decreasing steps), else only the largest index of V (the backup
// rule that makes the method finite).  Each step refactors Q_FF (Cholesky, 32-column panels:
// warp-level diagonal block, row-parallel panel solve, 4 x 4 register tiles for the trailing
// update from the panel staged in shared memory); the factor lives in the workspace.
constexpr int PB = 34;  // panel row stride in doubles (16-byte aligned, 16-byte bank shift per row)

struct BppSmem {
  int m, nv, imax, ninf, pcnt, status, bad;
};

// Cholesky of the m x m symmetric matrix in F (row-major, stride ld, lower triangle used) in
// place; returns false if it is not (numerically) positive definite.  panel: (d + 36) x PB doubles
// (the diagonal block, its reciprocal pivots, then the staged panel rows).  Staged row i goes to
// physical row (i & 3) * R4 + (i >> 2), so the 4 x 4 tiles' column rows (4 tj + b, consecutive tj
// across a warp) are consecutive physical rows: conflict-free 16-byte loads.
__device__ bool bpp_cholesky(double* __restrict__ F, int ld, int m, double* __restrict__ panel, int* bad) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* __restrict__ rinv = panel + (size_t)BK * PB;  // 1 / L[c][c] of the diagonal block (32)
  double* __restrict__ P = rinv + PB;
  for (int k0 = 0; k0 < m; k0 += BK) {
    const int nb = m - k0 < BK ? m - k0 : BK, k1 = k0 + nb;
    const int mt = m - k1, R4 = (mt + 3) >> 2;
    if (wid == 0) {  // diagonal block: lane j holds row k0 + j, column sweep with shuffles
      double Lr[BK];
#pragma unroll
      for (int c = 0; c < BK; ++c) Lr[c] = (lane < nb && c <= lane) ? F[(size_t)(k0 + lane) * ld + k0 + c] : 0.0;
      int fail = 0;
#pragma unroll
      for (int c = 0; c < BK; ++c) {
        if (c < nb) {
          const double dg = __shfl_sync(0xffffffffu, Lr[c], c);
          fail |= !(dg > 0.0);
          // one rsqrt instead of sqrt + divide on the column-to-column dependency chain
          const double ip = rsqrt(fmax(dg, 1e-300)), piv = dg * ip;
          Lr[c] = lane == c ? piv : Lr[c] * ip;
          if (lane == c) rinv[c] = ip;
          double lec[BK];
#pragma unroll
          for (int e = c + 1; e < BK; ++e) lec[e] = __shfl_sync(0xffffffffu, Lr[c], e);
#pragma unroll
          for (int e = c + 1; e < BK; ++e)
            if (lane >= e && e < nb) Lr[e] -= Lr[c] * lec[e];
        }
      }
      if (lane < nb) {
#pragma unroll
        for (int c = 0; c < BK; ++c)
          if (c <= lane) {
            F[(size_t)(k0 + lane) * ld + k0 + c] = Lr[c];
            panel[(size_t)lane * PB + c] = Lr[c];  // the diagonal block, for the panel solve
          }
      }
      if (lane == 0 && fail) *bad = 1;
    }
    __syncthreads();
    if (*bad) return false;
    // panel solve: rows i >= k1, L[i, k0:k1] = F[i, k0:k1] L_kk^{-T} (one row per thread; two
    // partial sums per entry halve the dependent chain)
    for (int i = k1 + tid; i < m; i += NT) {
      double l[BK];
      double* row = F + (size_t)i * ld + k0;
#pragma unroll
      for (int c = 0; c < BK; ++c) l[c] = c < nb ? row[c] : 0.0;
#pragma unroll
      for (int c = 0; c < BK; ++c) {
        if (c < nb) {
          double a0 = l[c], a1 = 0.0;
#pragma unroll
          for (int e = 0; e < c; e += 2) {
            a0 -= l[e] * panel[(size_t)c * PB + e];
            if (e + 1 < c) a1 -= l[e + 1] * panel[(size_t)c * PB + e + 1];
          }
          l[c] = (a0 + a1) * rinv[c];
        }
      }
      const int ii = i - k1;
      double* pr = P + (size_t)((ii & 3) * R4 + (ii >> 2)) * PB;
#pragma unroll
      for (int c = 0; c < BK; ++c) {
        if (c < nb) row[c] = l[c];
        pr[c] = l[c];  // staged (zero-padded to 32 columns)
      }
    }
    // padding rows of the last tile row: zeros
    for (int ii = mt + tid; ii < 4 * R4; ii += NT) {
      double* pr = P + (size_t)((ii & 3) * R4 + (ii >> 2)) * PB;
#pragma unroll
      for (int c = 0; c < BK; ++c) pr[c] = 0.0;
    }
    __syncthreads();
    // trailing update: F[i][j] -= sum_c P[i][c] P[j][c], k1 <= j <= i < m, 4 x 4 tiles (rows
    // 4 ti + a, columns 4 tj + b); the 16 F values are loaded before the products
    const int ntiles = R4 * (R4 + 1) / 2;
    for (int tix = tid; tix < ntiles; tix += NT) {
      int ti = (int)((sqrtf(8.f * tix + 1.f) - 1.f) * 0.5f);
      while ((ti + 1) * (ti + 2) / 2 <= tix) ++ti;
      while (ti * (ti + 1) / 2 > tix) --ti;
      const int tj = tix - ti * (ti + 1) / 2;
      double fv[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = k1 + 4 * ti + a, j = k1 + 4 * tj + b;
          fv[a][b] = (i < m && j <= i) ? F[(size_t)i * ld + j] : 0.0;
        }
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
#pragma unroll 4
      for (int c = 0; c < BK; c += 2) {
        double2 pa[4], pb[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          pa[a] = *reinterpret_cast<const double2*>(P + (size_t)(a * R4 + ti) * PB + c);
          pb[a] = *reinterpret_cast<const double2*>(P + (size_t)(a * R4 + tj) * PB + c);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(pa[a].x, pb[b].x, fma(pa[a].y, pb[b].y, acc[a][b]));
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = k1 + 4 * ti + a;
        if (i >= m) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int j = k1 + 4 * tj + b;
          if (j <= i) F[(size_t)i * ld + j] = fv[a][b] - acc[a][b];
        }
      }
    }
    __syncthreads();
  }
  return true;
}

__global__ void __launch_bounds__(NT) k_nnls_bpp(int d, const double* __restrict__ Gall, int64_t ldg, int64_t stride_g,
                                                double* __restrict__ xall, int64_t stride_x, int32_t* __restrict__ iters,
                                                double* __restrict__ ws, int64_t batch) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ BppSmem s;
  __shared__ NnlsSmem rs;
  __shared__ double part[BK];
  const int64_t p = blockIdx.x + (int64_t)blockIdx.y * 65535;
  if (p >= batch) return;
  const double* __restrict__ G = Gall + p * stride_g;  // Q[i][j] = G[i + j*ldg], q[i] = G[i + d*ldg]
  double* x = dsm;          // d: current x
  double* xs = x + d;       // d: x_F in order positions
  double* bv = xs + d;      // d
  double* zt = bv + d;      // d
  double* panel = zt + d;   // (d + 40) x PB: diagonal block, reciprocal pivots, staged panel (4-row padded)
  int* order = reinterpret_cast<int*>(panel + (size_t)(d + BK + 8) * PB);
  unsigned char* inF = reinterpret_cast<unsigned char*>(order + d);
  unsigned char* vflag = inF + d;  // infeasible in this step
  double* F = ws + p * (int64_t)d * d;
  const int tid = threadIdx.x;
  for (int i = tid; i < d; i += NT) {
    x[i] = 0.0;
    inF[i] = 0;
  }
  double qm = 0.0;
  for (int i = tid; i < d; i += NT) qm = fmax(qm, fabs(G[i + d * ldg]));
  block_argmax(qm, 0, true, rs);
  const double tol = 1e-10 * fmax(rs.red_v[0], 2.2250738585072014e-308);
  if (tid == 0) {
    s.ninf = d + 1;
    s.pcnt = 3;
    s.status = 0;
  }
  __syncthreads();
  const int max_iter = 10 * d + 10;
  int it = 0;
  while (true) {
    // order = F ascending (block prefix count over inF)
    if (tid == 0) {
      int m = 0;
      for (int i = 0; i < d; ++i)
        if (inF[i]) order[m++] = i;
      s.m = m;
      s.bad = 0;
    }
    __syncthreads();
    const int m = s.m;
    // x_F = Q_FF^{-1} q_F (Cholesky in the workspace)
    {  // Q_FF into the factor storage: warp per row a, lanes over b <= a (Q symmetric: read
       // column order[a] of G, contiguous in b; write row a of F, contiguous)
      const int lane = tid & 31, wid = tid >> 5;
      for (int a = wid; a < m; a += NT / 32) {
        const double* gc = G + (int64_t)order[a] * ldg;
        double* fr = F + (size_t)a * d;
        for (int b = lane; b <= a; b += 32) fr[b] = gc[order[b]];
      }
    }
    __syncthreads();
    if (m > 0 && !bpp_cholesky(F, d, m, panel, &s.bad)) {
      if (tid == 0) s.status = -3;
      __syncthreads();
      break;
    }
    for (int a = tid; a < m; a += NT) bv[a] = G[order[a] + (int64_t)d * ldg];
    __syncthreads();
    if (m > 0) {
      big_fwd(F, d, m, bv, zt, part);
      big_bwd(F, d, m, zt, xs);
    }
    for (int i = tid; i < d; i += NT) x[i] = 0.0;
    __syncthreads();
    for (int a = tid; a < m; a += NT) x[order[a]] = xs[a];
    __syncthreads();
    // infeasible set: F with x < 0, the rest with y = Q x - q < -tol
    int nv = 0, imax = -1;
    for (int i = tid; i < d; i += NT) {
      bool v;
      if (inF[i]) {
        v = x[i] < 0.0;
      } else {
        double y = -G[i + d * ldg];
        for (int a = 0; a < m; ++a) y += G[i + (int64_t)order[a] * ldg] * xs[a];
        v = y < -tol;
      }
      vflag[i] = v;
      if (v) {
        ++nv;
        imax = i;
      }
    }
    // block reductions: count and largest index
    {
      int cnt = nv, mx = imax;
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      }
      if (tid == 0) {
        s.nv = 0;
        s.imax = -1;
      }
      __syncthreads();
      if ((tid & 31) == 0) {
        atomicAdd(&s.nv, cnt);
        atomicMax(&s.imax, mx);
      }
      __syncthreads();
    }
    const int NV = s.nv;
    if (NV == 0) break;
    if (++it > max_iter) {
      if (tid == 0) s.status = -1;
      __syncthreads();
      break;
    }
    bool all;
    if (NV < s.ninf) {
      all = true;
    } else {
      all = s.pcnt > 0;
    }
    __syncthreads();
    if (tid == 0) {
      if (NV < s.ninf) {
        s.ninf = NV;
        s.pcnt = 3;
      } else if (s.pcnt > 0) {
        s.pcnt -= 1;
      }
    }
    // exchange all of V, or only its largest index (backup rule)
    const int im = s.imax;
    for (int i = tid; i < d; i += NT)
      if (vflag[i] && (all || i == im)) inF[i] ^= 1;
    __syncthreads();
  }
  double* xo = xall + p * stride_x;
  for (int j = tid; j < d; j += NT) xo[j] = x[j] < 1e-14 ? 0.0 : x[j];
  if (tid == 0 && iters) iters[p] = s.status ? s.status : it;
}
// ---------------------------------------------------------------------------------------
// The same block principal pivoting for ONE large problem on a thread-block cluster (CS CTAs on
// CS SMs): the factorization's parallel parts -- gathering Q_FF, the panel solves, the trailing
// updates -- and the dual y are split over the cluster's CTAs; the diagonal blocks, the
// triangular solves and the exchange decisions run on rank 0.  The factor and every shared
// vector live in the workspace (L2); cluster barriers (release / acquire) order the phases.
// Identical arithmetic per element as k_nnls_bpp except the reduction order of nothing: each F
// entry and each y_i is still computed by exactly one thread with the same operation order.
// (release / acquire at cluster scope order the global-memory writes of the cluster's CTAs too)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

// workspace layout of the cluster solver (doubles): F (d*d), x, xs, bv, zt (d each), then ints:
// order (d), inF (d), vflag (d), ctrl (16)
struct BppClCtrl {
  int m, nv, imax, ninf, pcnt, status, bad, it;
};

#ifdef BPP_TRACE
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BPP_T(k) if (rank == 0 && tid == 0) { const unsigned long long t_ = gtime(); tacc[k] += t_ - tlast; tlast = t_; }
#else
#define BPP_T(k)
#endif
#ifdef BPP_TRACE
__device__ unsigned long long g_chol_t[4];
#define BPP_C(k) if (rank == 0 && tid == 0) { const unsigned long long t_ = gtime(); g_chol_t[k] += t_ - tl; tl = t_; }
#else
#define BPP_C(k)
#endif
// Diagonal block [k0, k0 + nb) of the factor in F, by one warp (lane j holds row k0 + j).
__device__ __forceinline__ void bpp_diag_warp(double* __restrict__ F, int ld, int k0, int nb, int* badg) {
  const int lane = threadIdx.x & 31;
  double Lr[BK];
#pragma unroll
  for (int c = 0; c < BK; ++c) Lr[c] = (lane < nb && c <= lane) ? F[(size_t)(k0 + lane) * ld + k0 + c] : 0.0;
  int fail = 0;
#pragma unroll
  for (int c = 0; c < BK; ++c) {
    if (c < nb) {
      const double dg = __shfl_sync(0xffffffffu, Lr[c], c);
      fail |= !(dg > 0.0);
      const double ip = rsqrt(fmax(dg, 1e-300)), piv = dg * ip;
      Lr[c] = lane == c ? piv : Lr[c] * ip;
      double lec[BK];
#pragma unroll
      for (int e = c + 1; e < BK; ++e) lec[e] = __shfl_sync(0xffffffffu, Lr[c], e);
#pragma unroll
      for (int e = c + 1; e < BK; ++e)
        if (lane >= e && e < nb) Lr[e] -= Lr[c] * lec[e];
    }
  }
  if (lane < nb) {
#pragma unroll
    for (int c = 0; c < BK; ++c)
      if (c <= lane) F[(size_t)(k0 + lane) * ld + k0 + c] = Lr[c];
  }
  if (lane == 0 && fail) *badg = 1;
}

// 4 x 4 tile (ti, tj) of the trailing update F[i][j] -= sum_c P[i][c] P[j][c] (rows k1 + 4 ti + a,
// columns k1 + 4 tj + b, j <= i < m) from the staged panel P (permuted rows, see bpp_cholesky)
__device__ __forceinline__ void bpp_trail_tile(double* __restrict__ F, int ld, int m, int k1, int R4,
                                               const double* __restrict__ P, int ti, int tj) {
  double fv[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = k1 + 4 * ti + a, j = k1 + 4 * tj + b;
      fv[a][b] = (i < m && j <= i) ? F[(size_t)i * ld + j] : 0.0;
    }
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
#pragma unroll 4
  for (int c = 0; c < BK; c += 2) {
    double2 pa[4], pb[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      pa[a] = *reinterpret_cast<const double2*>(P + (size_t)(a * R4 + ti) * PB + c);
      pb[a] = *reinterpret_cast<const double2*>(P + (size_t)(a * R4 + tj) * PB + c);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(pa[a].x, pb[b].x, fma(pa[a].y, pb[b].y, acc[a][b]));
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = k1 + 4 * ti + a;
    if (i >= m) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = k1 + 4 * tj + b;
      if (j <= i) F[(size_t)i * ld + j] = fv[a][b] - acc[a][b];
    }
  }
}

// Cluster Cholesky with look-ahead: while the other CTAs apply panel k's trailing update to the
// rest of the matrix, rank 0 updates the next diagonal block first and factors it, so the
// diagonal chain (a warp of dependent pivots, ~19k cycles per 32 x 32 block) leaves the critical
// path of all but the first panel.
__device__ bool bpp_cholesky_cl(double* __restrict__ F, int ld, int m, double* __restrict__ panel, int* badg,
                                int rank, int cs) {
#ifdef BPP_TRACE
  unsigned long long tl = gtime();
#endif
  const int tid = threadIdx.x, wid = tid >> 5;
  const int gt = rank * NT + tid, gstride = cs * NT;  // cluster-wide thread index / count
  double* __restrict__ rinv = panel + (size_t)BK * PB;
  double* __restrict__ P = rinv + PB;
  if (rank == 0 && wid == 0) bpp_diag_warp(F, ld, 0, m < BK ? m : BK, badg);
  cluster_sync_all();
  BPP_C(0)
  for (int k0 = 0; k0 < m; k0 += BK) {
    const int nb = m - k0 < BK ? m - k0 : BK, k1 = k0 + nb;
    const int mt = m - k1, R4 = (mt + 3) >> 2;
    if (*(volatile int*)badg) return false;
    // every CTA: the (factored) diagonal block and its reciprocal pivots into shared memory
    for (int e = tid; e < nb * BK; e += NT) {
      const int a = e / BK, c = e - a * BK;
      if (c <= a && a < nb) panel[(size_t)a * PB + c] = F[(size_t)(k0 + a) * ld + k0 + c];
    }
    __syncthreads();
    if (tid < nb) rinv[tid] = 1.0 / panel[(size_t)tid * PB + tid];  // (same on every CTA)
    __syncthreads();
    // panel solve, rows split over the cluster
    for (int i = k1 + gt; i < m; i += gstride) {
      double l[BK];
      double* row = F + (size_t)i * ld + k0;
#pragma unroll
      for (int c = 0; c < BK; ++c) l[c] = c < nb ? row[c] : 0.0;
#pragma unroll
      for (int c = 0; c < BK; ++c) {
        if (c < nb) {
          double a0 = l[c], a1 = 0.0;
#pragma unroll
          for (int e = 0; e < c; e += 2) {
            a0 -= l[e] * panel[(size_t)c * PB + e];
            if (e + 1 < c) a1 -= l[e + 1] * panel[(size_t)c * PB + e + 1];
          }
          l[c] = (a0 + a1) * rinv[c];
        }
      }
#pragma unroll
      for (int c = 0; c < BK; ++c)
        if (c < nb) row[c] = l[c];
    }
    cluster_sync_all();
    BPP_C(1)
    if (mt <= 0) break;
    // every CTA stages the whole panel (permuted rows, as bpp_cholesky)
    for (int e = tid; e < 4 * R4 * BK; e += NT) {
      const int ii = e / BK, c = e - ii * BK;
      double* pr = P + (size_t)((ii & 3) * R4 + (ii >> 2)) * PB;
      pr[c] = (ii < mt && c < nb) ? F[(size_t)(k1 + ii) * ld + k0 + c] : 0.0;
    }
    __syncthreads();
    BPP_C(2)
    // trailing update: tile rows ti < 8 (with tj <= ti) are the next diagonal block: rank 0 applies
    // them and factors that block; ranks 1.. take every other tile
    const int ND = 8, nd_tiles = ND * (ND + 1) / 2;
    const int ntiles = R4 * (R4 + 1) / 2;
    if (rank == 0) {
      for (int tix = tid; tix < nd_tiles && tix < ntiles; tix += NT) {
        int ti = 0;
        while ((ti + 1) * (ti + 2) / 2 <= tix) ++ti;
        bpp_trail_tile(F, ld, m, k1, R4, P, ti, tix - ti * (ti + 1) / 2);
      }
      __syncthreads();
      if (wid == 0) bpp_diag_warp(F, ld, k1, mt < BK ? mt : BK, badg);
    } else {
      for (int tix = nd_tiles + (rank - 1) * NT + tid; tix < ntiles; tix += (cs - 1) * NT) {
        int ti = (int)((sqrtf(8.f * tix + 1.f) - 1.f) * 0.5f);
        while ((ti + 1) * (ti + 2) / 2 <= tix) ++ti;
        while (ti * (ti + 1) / 2 > tix) --ti;
        bpp_trail_tile(F, ld, m, k1, R4, P, ti, tix - ti * (ti + 1) / 2);
      }
    }
    cluster_sync_all();
    BPP_C(3)
  }
  return !*(volatile int*)badg;
}

// order = the passive indices ascending (block-wide scan of the 0/1 flags in `flag`), m returned
__device__ int block_compact(const int* __restrict__ flag, int d, int* __restrict__ order, int* wsum) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int PER = 4;  // d <= NT * PER
  int f[PER], cnt = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = tid * PER + k;
    f[k] = i < d ? flag[i] : 0;
    cnt += f[k] != 0;
  }
  int incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  int base = 0, total = 0;
  for (int w = 0; w < NT / 32; ++w) {
    if (w < wid) base += wsum[w];
    total += wsum[w];
  }
  int pos = base + incl - cnt;
#pragma unroll
  for (int k = 0; k < PER; ++k)
    if (f[k]) order[pos++] = tid * PER + k;
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(NT) k_nnls_bpp_cl(int d, const double* __restrict__ G, int64_t ldg,
                                                   double* __restrict__ xo, int32_t* __restrict__ iters,
                                                   double* __restrict__ ws) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ NnlsSmem rs;
  __shared__ double part[BK];
  __shared__ int wsum[NT / 32];
  const int rank = (int)cluster_rank(), cs = (int)cluster_size();
  const int tid = threadIdx.x, gt = rank * NT + tid, gstride = cs * NT;
  double* F = ws;
  double* x = F + (size_t)d * d;     // global: x (written by rank 0)
  double* xsg = x + d;                // global: x_F in order positions (written by rank 0)
  int* inF = reinterpret_cast<int*>(xsg + 3 * d);
  int* vflag = inF + d;
  BppClCtrl* ctl = reinterpret_cast<BppClCtrl*>(vflag + 2 * d);
  // shared memory: panel staging, then per-CTA copies of order and x_F, rank 0's solve vectors
  double* panel = dsm;  // (d + 40) x PB
  double* xs = panel + (size_t)(d + BK + 8) * PB;
  double* bv = xs + d;
  double* zt = bv + d;
  int* order = reinterpret_cast<int*>(zt + d);
  for (int i = gt; i < d; i += gstride) {
    x[i] = 0.0;
    inF[i] = 0;
  }
  double qm = 0.0;
  for (int i = tid; i < d; i += NT) qm = fmax(qm, fabs(G[i + (int64_t)d * ldg]));
  block_argmax(qm, 0, true, rs);
  const double tol = 1e-10 * fmax(rs.red_v[0], 2.2250738585072014e-308);
  if (rank == 0 && tid == 0) {
    ctl->ninf = d + 1;
    ctl->pcnt = 3;
    ctl->status = 0;
    ctl->it = 0;
    ctl->bad = 0;
  }
  cluster_sync_all();
  const int max_iter = 10 * d + 10;
#ifdef BPP_TRACE
  unsigned long long tacc[6] = {0, 0, 0, 0, 0, 0}, tlast = gtime();
#endif
  while (true) {
    const int m = block_compact(inF, d, order, wsum);  // every CTA: its own copy of order
    {  // Q_FF rows split over the cluster's warps
      const int lane = tid & 31, gw = rank * (NT / 32) + (tid >> 5);
      for (int a = gw; a < m; a += cs * (NT / 32)) {
        const double* gc = G + (int64_t)order[a] * ldg;
        double* fr = F + (size_t)a * d;
        for (int b = lane; b <= a; b += 32) fr[b] = gc[order[b]];
      }
    }
    if (rank == 0 && tid == 0) {
      ctl->nv = 0;
      ctl->imax = -1;
    }
    cluster_sync_all();
    BPP_T(0)
    if (m > 0 && !bpp_cholesky_cl(F, d, m, panel, &ctl->bad, rank, cs)) {
      if (rank == 0 && tid == 0) ctl->status = -3;
      break;
    }
    BPP_T(1)
    if (rank == 0) {  // triangular solves on rank 0 (vectors in its shared memory)
      for (int a = tid; a < m; a += NT) bv[a] = G[order[a] + (int64_t)d * ldg];
      __syncthreads();
      if (m > 0) {
        big_fwd(F, d, m, bv, zt, part);
        big_bwd(F, d, m, zt, xs);
      }
      for (int i = tid; i < d; i += NT) x[i] = 0.0;
      __syncthreads();
      for (int a = tid; a < m; a += NT) {
        x[order[a]] = xs[a];
        xsg[a] = xs[a];
      }
    }
    cluster_sync_all();
    BPP_T(2)
    if (rank != 0)
      for (int a = tid; a < m; a += NT) xs[a] = xsg[a];
    __syncthreads();
    // infeasible set, split over the cluster
    int nv = 0, imax = -1;
    for (int i = gt; i < d; i += gstride) {
      bool v;
      if (inF[i]) {
        v = x[i] < 0.0;
      } else {
        double y = -G[i + (int64_t)d * ldg];
        for (int a = 0; a < m; ++a) y += G[i + (int64_t)order[a] * ldg] * xs[a];
        v = y < -tol;
      }
      vflag[i] = v;
      if (v) {
        ++nv;
        imax = i;
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      nv += __shfl_xor_sync(0xffffffffu, nv, off);
      imax = max(imax, __shfl_xor_sync(0xffffffffu, imax, off));
    }
    if ((tid & 31) == 0) {
      if (nv) atomicAdd(&ctl->nv, nv);
      atomicMax(&ctl->imax, imax);
    }
    cluster_sync_all();
    BPP_T(3)
    const int NV = *(volatile int*)&ctl->nv;
#ifdef BPP_TRACE
    if (rank == 0 && tid == 0) printf("bpp_cl step: m %d infeasible %d\n", m, NV);
#endif
    if (NV == 0) break;
    const int it = *(volatile int*)&ctl->it + 1;
    if (it > max_iter) {
      if (rank == 0 && tid == 0) ctl->status = -1;
      break;
    }
    const int ninf = *(volatile int*)&ctl->ninf, pcnt = *(volatile int*)&ctl->pcnt;
    const bool all = NV < ninf || pcnt > 0;
    const int im = *(volatile int*)&ctl->imax;
    cluster_sync_all();  // everyone has read the decision inputs
    if (rank == 0 && tid == 0) {
      ctl->it = it;
      if (NV < ninf) {
        ctl->ninf = NV;
        ctl->pcnt = 3;
      } else if (pcnt > 0) {
        ctl->pcnt = pcnt - 1;
      }
    }
    for (int i = gt; i < d; i += gstride)
      if (vflag[i] && (all || i == im)) inF[i] ^= 1;
    cluster_sync_all();
    BPP_T(4)
  }
  cluster_sync_all();
#ifdef BPP_TRACE
  if (rank == 0 && tid == 0)
    printf("bpp_cl phases us: gather %.1f chol %.1f (diag %.1f panel %.1f stage %.1f trailing %.1f) solves %.1f dual %.1f "
           "exchange %.1f\n", tacc[0] * 1e-3, tacc[1] * 1e-3, g_chol_t[0] * 1e-3, g_chol_t[1] * 1e-3, g_chol_t[2] * 1e-3,
           g_chol_t[3] * 1e-3, tacc[2] * 1e-3, tacc[3] * 1e-3, tacc[4] * 1e-3);
#endif
  if (rank == 0) {
    for (int j = tid; j < d; j += NT) xo[j] = x[j] < 1e-14 ? 0.0 : x[j];
    if (tid == 0 && iters) iters[0] = ctl->status ? ctl->status : ctl->it;
  }
}
}  // namespace

size_t nnls_bpp_cl_workspace_bytes(int64_t d) {
  return ((size_t)d * d + 4 * (size_t)d) * sizeof(double) + 4 * (size_t)d * sizeof(int) + sizeof(BppClCtrl) + 64;
}

// One problem on a cluster of `cs` CTAs (16: non-portable size, opt-in); returns the launch error
// (e.g. the cluster cannot be scheduled) so the caller can fall back.
cudaError_t launch_nnls_bpp_cl(int64_t d, const double* G, int64_t ldg, double* x, int32_t* iters, double* ws,
                               int cs, cudaStream_t stream) {
  const size_t smem = (size_t)(d + BK + 8) * PB * sizeof(double) + 3 * (size_t)d * sizeof(double) + (size_t)d * sizeof(int);
  cudaError_t e = cudaFuncSetAttribute(k_nnls_bpp_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(k_nnls_bpp_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cs, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_nnls_bpp_cl, (int)d, G, ldg, x, iters, ws);
}

size_t nnls_bpp_smem_bytes(int64_t d) {
  return (size_t)(4 * d + (d + BK + 8) * PB) * sizeof(double) + (size_t)d * sizeof(int) + 2 * (size_t)d + 16;
}
bool nnls_bpp_ok(int64_t d) { return nnls_bpp_smem_bytes(d) <= 200 * 1024; }

cudaError_t launch_nnls_bpp(int64_t d, int64_t batch, const double* G, int64_t ldg, int64_t stride_g, double* x,
                            int64_t stride_x, int32_t* iters, double* ws, cudaStream_t stream) {
  if (d <= 0 || batch <= 0) return cudaSuccess;
#ifndef BPP_CLUSTER_MIN_D
#define BPP_CLUSTER_MIN_D 128
#endif
  if (batch == 1 && d >= BPP_CLUSTER_MIN_D) {  // one large problem: a cluster of 16 (else 8) SMs
    for (int cs : {16, 8}) {
      if (launch_nnls_bpp_cl(d, G, ldg, x, iters, ws, cs, stream) == cudaSuccess) return cudaSuccess;
      (void)cudaGetLastError();  // not schedulable at this size: try the next
    }
  }
  const dim3 grid((unsigned)(batch < 65535 ? batch : 65535), (unsigned)((batch + 65534) / 65535));
  const size_t smem = nnls_bpp_smem_bytes(d);
  cudaError_t e = cudaFuncSetAttribute(k_nnls_bpp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_nnls_bpp<<<grid, NT, smem, stream>>>((int)d, G, ldg, stride_g, x, stride_x, iters, ws, batch);
  return cudaGetLastError();
}

size_t nnls_smem_bytes(int64_t d, bool fac_in_smem) {
  size_t b = (size_t)NNLS_BIG_VEC_DOUBLES(d) * sizeof(double);
  if (fac_in_smem) b += (size_t)d * d * sizeof(double);
  return b;
}

bool nnls_factor_in_smem(int64_t d) { return nnls_smem_bytes(d, true) <= 200 * 1024; }

cudaError_t launch_nnls_gram(int64_t d, int64_t batch, const double* G, int64_t ldg, int64_t stride_g, double* x,
                             int64_t stride_x, int32_t* iters, double* ws, cudaStream_t stream) {
  if (d <= 0 || batch <= 0) return cudaSuccess;
  const bool fs = nnls_factor_in_smem(d);
  const dim3 grid((unsigned)(batch < 65535 ? batch : 65535), (unsigned)((batch + 65534) / 65535));
  const size_t smem = nnls_smem_bytes(d, fs);
  cudaError_t e;
  if (fs) {
    e = cudaFuncSetAttribute(k_nnls_lh_big<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_nnls_lh_big<true><<<grid, NT, smem, stream>>>((int)d, G, ldg, stride_g, x, stride_x, iters, ws, batch);
  } else {
    e = cudaFuncSetAttribute(k_nnls_lh_big<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_nnls_lh_big<false><<<grid, NT, smem, stream>>>((int)d, G, ldg, stride_g, x, stride_x, iters, ws, batch);
  }
  return cudaGetLastError();
}

}  // namespace srht
