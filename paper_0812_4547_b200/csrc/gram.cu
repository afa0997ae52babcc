// Gram matrices of sketches: the QP form of Section 3.4, sm_100a.
//
//   G_p = SM_p^T SM_p  with SM_p = [SA | Sb] (r x c, FP32)  =  [[Q~, q~], [q~^T, Sb^T Sb]],
//   Q~ = (H~DA)^T H~DA,  q~ = (H~DA)^T (H~Db)  (reading R17: the paper's q~ = (H~DA)^T b
//   must use the sketched b for the dimensions to agree).
//
// Products of FP32 entries are exact in FP64 and are accumulated in FP64 (DFMA), so G is
// the exact Gram matrix of the FP32 sketch up to FP64 rounding.  One CTA per (problem,
// 64 x 64 block of the upper triangle), 4 x 4 outputs per thread (two DFMA per shared-memory
// load); the two 64-column slabs of SM_p are staged through shared memory as doubles, 16
// rows at a time; each element is written once with its mirror (exactly symmetric).
#include <cuda_runtime.h>

#include "internal.cuh"

namespace srht {
namespace {

constexpr int GT = 64;   // output block edge
constexpr int GK = 16;   // rows of SM staged per step
constexpr int GTH = 256; // 16 x 16 threads, 4 x 4 outputs each (rows ty + 16 i, columns tx + 16 j)

__global__ void __launch_bounds__(GTH) k_gram(int64_t r, int64_t c, int64_t batch, const float* __restrict__ SM,
                                              int64_t ldsm, int64_t stride_sm, double* __restrict__ G, int64_t ldg,
                                              int64_t stride_g, int nb) {
  __shared__ double As[GK][GT + 1];  // +1: the staging stores (16 rows of one column) hit distinct banks
  __shared__ double Bs[GK][GT + 1];
  // upper-triangular block pair (bi <= bj) from the linear block index
  int pair = blockIdx.x, bi = 0;
  while (pair >= nb - bi) {
    pair -= nb - bi;
    ++bi;
  }
  const int bj = bi + pair;
  const int64_t p = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (p >= batch) return;
  const float* __restrict__ S = SM + p * stride_sm;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  // staging: thread -> (row kk = tid & 15, column lc = tid >> 4 + 16 u): 16 consecutive rows
  // of one column per half-warp (64 B contiguous)
  const int kk = tid & 15, lc0 = tid >> 4;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t k0 = 0; k0 < r; k0 += GK) {
    const int64_t k = k0 + kk;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int lc = lc0 + 16 * u;
      const int64_t ca = (int64_t)bi * GT + lc, cb = (int64_t)bj * GT + lc;
      As[kk][lc] = (k < r && ca < c) ? (double)S[k + ca * ldsm] : 0.0;
      Bs[kk][lc] = (k < r && cb < c) ? (double)S[k + cb * ldsm] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < GK; ++q) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[q][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[q][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* __restrict__ Gp = G + p * stride_g;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gi = (int64_t)bi * GT + ty + 16 * i, gj = (int64_t)bj * GT + tx + 16 * j;
      if (gi < c && gj < c && (bi != bj || gi <= gj)) {  // each element once, mirrored exactly
        Gp[gi + gj * ldg] = acc[i][j];
        Gp[gj + gi * ldg] = acc[i][j];
      }
    }
}

// Small-work variant (few problems x blocks, e.g. one problem with c = 513): 32 x 32 blocks,
// four outputs per thread, more CTAs.
constexpr int GT32 = 32;

__global__ void __launch_bounds__(256) k_gram32(int64_t r, int64_t c, int64_t batch, const float* __restrict__ SM,
                                             int64_t ldsm, int64_t stride_sm, double* __restrict__ G, int64_t ldg,
                                             int64_t stride_g, int nb) {
  __shared__ double As[GT32][GT32 + 1];
  __shared__ double Bs[GT32][GT32 + 1];
  // upper-triangular block pair (bi <= bj) from the linear block index
  int pair = blockIdx.x, bi = 0;
  while (pair >= nb - bi) {
    pair -= nb - bi;
    ++bi;
  }
  const int bj = bi + pair;
  const int64_t p = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (p >= batch) return;
  const float* __restrict__ S = SM + p * stride_sm;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;  // ty in 0..7
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k0 = 0; k0 < r; k0 += GT32) {
    // stage rows k0..k0+31 of the two column slabs: a warp reads 32 consecutive rows of a column
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int lc = ty + 8 * m;  // local column
      const int64_t k = k0 + tx;
      const int64_t ca = (int64_t)bi * GT32 + lc, cb = (int64_t)bj * GT32 + lc;
      As[tx][lc] = (k < r && ca < c) ? (double)S[k + ca * ldsm] : 0.0;
      Bs[tx][lc] = (k < r && cb < c) ? (double)S[k + cb * ldsm] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GT32; ++kk) {
      const double b = Bs[kk][tx];
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[m] = fma(As[kk][ty + 8 * m], b, acc[m]);
    }
    __syncthreads();
  }
  double* __restrict__ Gp = G + p * stride_g;
  const int64_t j = (int64_t)bj * GT32 + tx;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int64_t i = (int64_t)bi * GT32 + ty + 8 * m;
    if (i < c && j < c) {
      Gp[i + j * ldg] = acc[m];
      Gp[j + i * ldg] = acc[m];  // mirror (same value on the diagonal block)
    }
  }
}


// Small c (<= 112, many problems: config 2's c = 101): one CTA per problem computes only the
// upper triangle, as 4 x 4 register tiles (i <= j over ceil(c/4) tile rows): one thread per
// tile, e.g. 351 threads for c = 101, 2.2x less work than 64 x 64 blocks of a padded G.
constexpr int GTRI_K = 32;     // rows of SM staged per step
constexpr int GTRI_PF = 12;    // staged elements per thread held in registers (next step's, prefetched)
constexpr int GTRI_MAXC = 112;  // <= 406 tiles: 13 warps, so 128 registers per thread fit

__global__ void __launch_bounds__(416) k_gram_tri(int64_t r, int64_t c, int64_t batch, const float* __restrict__ SM,
                                                  int64_t ldsm, int64_t stride_sm, double* __restrict__ G, int64_t ldg,
                                                  int64_t stride_g) {
  __shared__ __align__(16) double S[GTRI_K][GTRI_MAXC + 2];  // +2: staged rows land in distinct banks
  const int64_t p = blockIdx.x + (int64_t)blockIdx.y * 65535;
  if (p >= batch) return;
  const float* __restrict__ Sp = SM + p * stride_sm;
  const int nt = (int)((c + 3) / 4), ntiles = nt * (nt + 1) / 2;
  const int tid = threadIdx.x;
  // this thread's tile (ti <= tj) from its linear index
  int ti = 0, rem = tid;
  while (ti < nt && rem >= nt - ti) {
    rem -= nt - ti;
    ++ti;
  }
  const int tj = ti + rem;
  const bool act = tid < ntiles;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  // staging: element e = (row kk = e % 32, column cc = e / 32); a warp reads 32 consecutive rows
  // of one column.  The next step's elements are loaded into registers during this step.
  const int nel = GTRI_K * 4 * nt;  // including zero padding columns
  float pf[GTRI_PF];
#define GTRI_FETCH(K0)                                                     \
  _Pragma("unroll") for (int u = 0; u < GTRI_PF; ++u) {                     \
    const int e = tid + u * (int)blockDim.x;                               \
    const int kk = e % GTRI_K, cc = e / GTRI_K;                            \
    const int64_t k = (K0) + kk;                                           \
    pf[u] = (e < nel && cc < c && k < r) ? Sp[k + cc * ldsm] : 0.f;        \
  }
  GTRI_FETCH(0)
  for (int64_t k0 = 0; k0 < r; k0 += GTRI_K) {
#pragma unroll
    for (int u = 0; u < GTRI_PF; ++u) {
      const int e = tid + u * (int)blockDim.x;
      if (e < nel) S[e % GTRI_K][e / GTRI_K] = (double)pf[u];
    }
    __syncthreads();
    if (k0 + GTRI_K < r) {
      GTRI_FETCH(k0 + GTRI_K)
    }
    if (act) {
#pragma unroll
      for (int q = 0; q < GTRI_K; ++q) {
        // 16-byte loads: a warp's lanes mostly share ti (broadcast) and take consecutive tj
        const double2 a01 = *reinterpret_cast<const double2*>(&S[q][4 * ti]);
        const double2 a23 = *reinterpret_cast<const double2*>(&S[q][4 * ti + 2]);
        const double2 b01 = *reinterpret_cast<const double2*>(&S[q][4 * tj]);
        const double2 b23 = *reinterpret_cast<const double2*>(&S[q][4 * tj + 2]);
#define GTRI_ROW(U, AU)                                                          \
  acc[U][0] = fma(AU, b01.x, acc[U][0]);                                         \
  acc[U][1] = fma(AU, b01.y, acc[U][1]);                                         \
  acc[U][2] = fma(AU, b23.x, acc[U][2]);                                         \
  acc[U][3] = fma(AU, b23.y, acc[U][3]);
        GTRI_ROW(0, a01.x)
        GTRI_ROW(1, a01.y)
        GTRI_ROW(2, a23.x)
        GTRI_ROW(3, a23.y)
#undef GTRI_ROW
      }
    }
    __syncthreads();
  }
  if (!act) return;
  double* __restrict__ Gp = G + p * stride_g;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t gi = 4 * ti + u, gj = 4 * tj + v;
      if (gi < c && gj < c && (ti != tj || gi <= gj)) {  // each element once, mirrored exactly
        Gp[gi + gj * ldg] = acc[u][v];
        Gp[gj + gi * ldg] = acc[u][v];
      }
    }
}
// ---------------------------------------------------------------------------------------
// FP64 tensor-core Gram (mma.sync m8n8k4 f64 = SASS DMMA; the same 64 FMA/clk/SM as DFMA on the
// B200, scripts/mb_dmma.cu, but 256 FMA per warp instruction and two 8-byte fragment loads per
// 256 FMA).  Products of FP32 entries are exact in FP64 and accumulated in FP64, as above.
// CTA = one 64 x 64 block pair (bi <= bj) of one problem and one K-split; 4 warps, each a
// 32 x 32 region as 4 x 4 tiles of 8 x 8 (tiles below the diagonal of a diagonal pair and tiles
// beyond the last column are skipped).  SM rows stream through shared memory as doubles in
// [column][k] layout (row stride 36 doubles: the fragment loads are conflict-free), 32 rows per
// step, the next step's rows prefetched into registers.  K-splits write 64 x 64 partials that
// k_gram_reduce sums in split order, so results are deterministic.
// Each element is computed once in the upper triangle and mirrored (exactly symmetric).
constexpr int MB = 64, MKT = 32, MPK = MKT + 4;

#ifndef GRAM_MMA_MINB
#define GRAM_MMA_MINB 4
#endif
template <bool VEC>
__global__ void __launch_bounds__(128, GRAM_MMA_MINB) k_gram_mma(int64_t r, int64_t c, int64_t batch, const float* __restrict__ SM,
                                                  int64_t ldsm, int64_t stride_sm, double* __restrict__ G, int64_t ldg,
                                                  int64_t stride_g, int nb, int splits, int64_t kchunk,
                                                  double* __restrict__ part) {
  __shared__ __align__(16) double Si[MB][MPK];
  __shared__ __align__(16) double Sj[MB][MPK];
  const int npairs = nb * (nb + 1) / 2;
  const int pair = blockIdx.x / splits, split = blockIdx.x - pair * splits;
  int rem = pair, bi = 0;
  while (rem >= nb - bi) {
    rem -= nb - bi;
    ++bi;
  }
  const int bj = bi + rem;
  const bool diag = bi == bj;
  const int64_t p = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (p >= batch) return;
  const float* __restrict__ S = SM + p * stride_sm;
  const int wi = (int)(c - (int64_t)MB * bi < MB ? c - (int64_t)MB * bi : MB);
  const int wj = (int)(c - (int64_t)MB * bj < MB ? c - (int64_t)MB * bj : MB);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 1, wc = warp & 1, gid = lane >> 2, tig = lane & 3;
  const int64_t k_lo = (int64_t)split * kchunk, k_hi = k_lo + kchunk < r ? k_lo + kchunk : r;
  // tile (ti, tj) of this warp is live iff inside both widths and not below a diagonal block's diagonal
  bool live[4][4];
  bool any = false;
#pragma unroll
  for (int ti = 0; ti < 4; ++ti)
#pragma unroll
    for (int tj = 0; tj < 4; ++tj) {
      const int i8 = 32 * wr + 8 * ti, j8 = 32 * wc + 8 * tj;
      live[ti][tj] = i8 < wi && j8 < wj && (!diag || i8 <= j8);
      any |= live[ti][tj];
    }
  double acc[4][4][2];
#pragma unroll
  for (int ti = 0; ti < 4; ++ti)
#pragma unroll
    for (int tj = 0; tj < 4; ++tj) acc[ti][tj][0] = acc[ti][tj][1] = 0.0;
  // staging: element (column cc, rows 4 k4 .. 4 k4 + 3) for idx = tid + 128 u, cc = idx >> 3, k4 = idx & 7
  float4 pf[2][4];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && diag) break;
      const int64_t cb = (int64_t)MB * (h ? bj : bi);
      const int w = h ? wj : wi;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = tid + 128 * u, cc = idx >> 3, k4 = idx & 7;
        const int64_t k = k0 + 4 * k4;
        const float* src = S + (cb + cc) * ldsm + k;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (cc < w) {
          if (VEC && k + 3 < k_hi) {
            v = __ldg(reinterpret_cast<const float4*>(src));
          } else {
            if (k < k_hi) v.x = __ldg(src);
            if (k + 1 < k_hi) v.y = __ldg(src + 1);
            if (k + 2 < k_hi) v.z = __ldg(src + 2);
            if (k + 3 < k_hi) v.w = __ldg(src + 3);
          }
        }
        pf[h][u] = v;
      }
    }
  };
  fetch(k_lo);
  for (int64_t k0 = k_lo; k0 < k_hi; k0 += MKT) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && diag) break;
      double(*D)[MPK] = h ? Sj : Si;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = tid + 128 * u, cc = idx >> 3, k4 = idx & 7;
        *reinterpret_cast<double2*>(&D[cc][4 * k4]) = make_double2(pf[h][u].x, pf[h][u].y);
        *reinterpret_cast<double2*>(&D[cc][4 * k4 + 2]) = make_double2(pf[h][u].z, pf[h][u].w);
      }
    }
    __syncthreads();
    if (k0 + MKT < k_hi) fetch(k0 + MKT);
    const double(*B)[MPK] = diag ? Si : Sj;
    if (any) {
#pragma unroll
      for (int kk = 0; kk < MKT; kk += 4) {
        double a[4], b[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          a[t] = Si[32 * wr + 8 * t + gid][kk + tig];
          b[t] = B[32 * wc + 8 * t + gid][kk + tig];
        }
#pragma unroll
        for (int ti = 0; ti < 4; ++ti)
#pragma unroll
          for (int tj = 0; tj < 4; ++tj)
            if (live[ti][tj])
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(acc[ti][tj][0]), "+d"(acc[ti][tj][1])
                           : "d"(a[ti]), "d"(b[tj]));
      }
    }
    __syncthreads();
  }
  double* __restrict__ Gp = G + p * stride_g;
  if (splits == 1) {
#pragma unroll
    for (int ti = 0; ti < 4; ++ti)
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) {
        if (!live[ti][tj]) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int ii = 32 * wr + 8 * ti + gid, jj = 32 * wc + 8 * tj + 2 * tig + e;
          if (ii < wi && jj < wj && (!diag || ii <= jj)) {
            const int64_t gi = (int64_t)MB * bi + ii, gj = (int64_t)MB * bj + jj;
            Gp[gi + gj * ldg] = acc[ti][tj][e];
            Gp[gj + gi * ldg] = acc[ti][tj][e];
          }
        }
      }
    return;
  }
  // K-split: this split's 64 x 64 partial (k_gram_reduce sums the splits in order)
  double* __restrict__ mine = part + (((p * npairs + pair) * splits + split) * (MB * MB));
#pragma unroll
  for (int ti = 0; ti < 4; ++ti)
#pragma unroll
    for (int tj = 0; tj < 4; ++tj) {
      const int ii = 32 * wr + 8 * ti + gid, jj = 32 * wc + 8 * tj + 2 * tig;
      *reinterpret_cast<double2*>(mine + ii * MB + jj) = make_double2(acc[ti][tj][0], acc[ti][tj][1]);
    }
}

// Fixed-order sum of the K-split partials of every block pair (deterministic), upper triangle
// computed once and mirrored.  Thread = one element of one pair's 64 x 64 block.
__global__ void k_gram_reduce(int64_t c, int64_t batch, double* __restrict__ G, int64_t ldg, int64_t stride_g, int nb,
                              int splits, const double* __restrict__ part) {
  const int npairs = nb * (nb + 1) / 2;
  const int64_t gidx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t slot = gidx / (MB * MB);
  const int e = (int)(gidx - slot * (MB * MB));
  if (slot >= (int64_t)npairs * batch) return;
  const int64_t p = slot / npairs;
  int rem = (int)(slot - p * npairs), bi = 0;
  while (rem >= nb - bi) {
    rem -= nb - bi;
    ++bi;
  }
  const int bj = bi + rem;
  const int ii = e / MB, jj = e - ii * MB;
  const int64_t gi = (int64_t)MB * bi + ii, gj = (int64_t)MB * bj + jj;
  if (gi >= c || gj >= c || gi > gj) return;
  const double* __restrict__ src = part + slot * splits * (MB * MB) + e;
  double sum = 0.0;
  for (int s2 = 0; s2 < splits; ++s2) sum += src[(int64_t)s2 * (MB * MB)];
  double* __restrict__ Gp = G + p * stride_g;
  Gp[gi + gj * ldg] = sum;
  Gp[gj + gi * ldg] = sum;
}
}  // namespace

// Many small problems (c <= 128, e.g. config 2's 3000 x 101): one CTA per problem stages every
// column once per 32-row step (a 64 x 64 block pair would stage the columns of both blocks) and its
// warps share the upper-triangle 8 x 8 tiles row pair by row pair (rows t and nt-1-t: nt+1 tiles per
// warp, balanced); per k-step a warp loads the fragments of its two tile rows and of the columns it
// needs once, then issues one DMMA per tile.
constexpr int SMC = 128, SNT = SMC / 8;  // max columns, max tile rows

// GRAM_DB: the staged rows are double-buffered (dynamic shared memory, 2 x 36 KB): step k+1's
// rows are written into the other buffer after step k's DMMAs, so one barrier per step.
#ifndef GRAM_DB
#define GRAM_DB 1
#endif
#ifndef GRAM_SMALL_MINB
#define GRAM_SMALL_MINB 2  // 2 CTAs per SM at 128 registers, no spills (config 2: 2.16 -> 1.83 ms, bit-identical)
#endif
template <bool VEC>
__global__ void __launch_bounds__(256, GRAM_SMALL_MINB) k_gram_mma_small(int64_t r, int64_t c, int64_t batch,
                                                        const float* __restrict__ SM, int64_t ldsm,
                                                        int64_t stride_sm, double* __restrict__ G, int64_t ldg,
                                                        int64_t stride_g) {
  extern __shared__ __align__(16) double gsm[];
  double(*S)[MPK] = reinterpret_cast<double(*)[MPK]>(gsm);
  const int64_t p = blockIdx.x + (int64_t)blockIdx.y * 65535;
  if (p >= batch) return;
  const float* __restrict__ Sp = SM + p * stride_sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gid = lane >> 2, tig = lane & 3;
  const int nt = (int)((c + 7) >> 3), cp = 8 * nt;
  const int ra = warp, rb = nt - 1 - warp;  // this warp's tile rows (rb < ra: none; rb == ra: one)
  const bool has_a = ra < nt && ra <= rb, has_b = has_a && rb != ra;
  // accumulator slot s (static): s in [ra, nt) -> tile (ra, s); s < ra -> tile (rb, rb + s);
  // s == SNT -> tile (rb, nt - 1).  Row ra has nt - ra tiles, row rb has ra + 1.
  double acc[SNT + 1][2];
#pragma unroll
  for (int j = 0; j <= SNT; ++j) acc[j][0] = acc[j][1] = 0.0;
  // staging: (column cc, rows 4 k4 .. 4 k4 + 3) for idx = tid + 256 u < cp * 8
  constexpr int NU = SMC * 8 / 256;
  float4 pf[NU];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int idx = tid + 256 * u, cc = idx >> 3, k4 = idx & 7;
      const int64_t k = k0 + 4 * k4;
      const float* src = Sp + (int64_t)cc * ldsm + k;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (cc < c) {
        if (VEC && k + 3 < r) {
          v = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          if (k < r) v.x = __ldg(src);
          if (k + 1 < r) v.y = __ldg(src + 1);
          if (k + 2 < r) v.z = __ldg(src + 2);
          if (k + 3 < r) v.w = __ldg(src + 3);
        }
      }
      pf[u] = v;
    }
  };
  auto put = [&](double(*D)[MPK]) {
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int idx = tid + 256 * u, cc = idx >> 3, k4 = idx & 7;
      if (cc < cp) {
        *reinterpret_cast<double2*>(&D[cc][4 * k4]) = make_double2(pf[u].x, pf[u].y);
        *reinterpret_cast<double2*>(&D[cc][4 * k4 + 2]) = make_double2(pf[u].z, pf[u].w);
      }
    }
  };
  fetch(0);
  if (GRAM_DB) {
    put(S);
    __syncthreads();
  }
  int cur = 0;
  for (int64_t k0 = 0; k0 < r; k0 += MKT) {
    if (!GRAM_DB) {
      put(S);
      __syncthreads();
    }
    if (k0 + MKT < r) fetch(k0 + MKT);
    const double(*T)[MPK] = S + (GRAM_DB ? cur * SMC : 0);
    if (has_a) {
#pragma unroll
      for (int kk = 0; kk < MKT; kk += 4) {
        const double fa = T[8 * ra + gid][kk + tig];
        const double fb = T[8 * rb + gid][kk + tig];
#pragma unroll
        for (int sl = 0; sl <= SNT; ++sl) {
          int j;
          bool rowb;
          if (sl == SNT) { j = nt - 1; rowb = true; }
          else if (sl >= ra) { j = sl; rowb = false; }
          else { j = rb + sl; rowb = true; }
          if (j >= nt || (rowb && !has_b)) continue;
          const double fc = T[8 * j + gid][kk + tig];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[sl][0]), "+d"(acc[sl][1])
                       : "d"(rowb ? fb : fa), "d"(fc));
        }
      }
    }
    if (GRAM_DB) {
      cur ^= 1;
      if (k0 + MKT < r) put(S + cur * SMC);  // buffer cur was last read in the previous step
    }
    __syncthreads();
  }
  if (!has_a) return;
  double* __restrict__ Gp = G + p * stride_g;
#pragma unroll
  for (int sl = 0; sl <= SNT; ++sl) {
    int j, ti;
    if (sl == SNT) { j = nt - 1; ti = rb; }
    else if (sl >= ra) { j = sl; ti = ra; }
    else { j = rb + sl; ti = rb; }
    if (j >= nt || ((sl == SNT || sl < ra) && !has_b)) continue;  // row rb's slots exist only if rb != ra
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t gi = 8 * ti + gid, gj = 8 * j + 2 * tig + e;
      if (gi < c && gj < c && gi <= gj) {
        Gp[gi + gj * ldg] = acc[sl][e];
        Gp[gj + gi * ldg] = acc[sl][e];
      }
    }
  }
}

// K-split geometry of the tensor-core Gram: about 4 CTAs per SM (148 SMs), >= 256 rows per split.
void gram_splits(int64_t r, int64_t c, int64_t batch, int64_t* splits_out, int64_t* kchunk_out, int* npairs_out) {
  const int nb = (int)((c + MB - 1) / MB);
  const int npairs = nb * (nb + 1) / 2;
#ifndef GRAM_CTAS_PER_SM
#define GRAM_CTAS_PER_SM 8
#endif
  int64_t splits = (GRAM_CTAS_PER_SM * 148 + npairs * batch - 1) / (npairs * batch);
  const int64_t maxs = r / 256 > 1 ? r / 256 : 1;
  if (splits > maxs) splits = maxs;
  if (splits < 1) splits = 1;
  int64_t kchunk = (r + splits - 1) / splits;
  kchunk = (kchunk + MKT - 1) / MKT * MKT;
  *splits_out = (r + kchunk - 1) / kchunk;
  *kchunk_out = kchunk;
  *npairs_out = npairs;
}

size_t gram_workspace_bytes(int64_t r, int64_t c, int64_t batch) {
  if (c <= SMC && batch >= 2 * 148) return 0;  // one CTA per problem, no K-split
  int64_t splits, kchunk;
  int npairs;
  gram_splits(r, c, batch, &splits, &kchunk, &npairs);
  if (splits <= 1) return 0;
  return (size_t)npairs * batch * splits * MB * MB * sizeof(double);
}

// ws: gram_workspace_bytes bytes (K-split partials); NULL: allocated stream-ordered for this call.
cudaError_t launch_gram_mma(int64_t r, int64_t c, int64_t batch, const float* SM, int64_t ldsm, int64_t stride_sm,
                            double* G, int64_t ldg, int64_t stride_g, void* ws, cudaStream_t stream) {
  const bool vec = (ldsm % 4 == 0) && (stride_sm % 4 == 0) && ((reinterpret_cast<uintptr_t>(SM) & 15) == 0);
  if (c <= SMC && batch >= 2 * 148) {  // many small problems: one CTA per problem
    const dim3 grid((unsigned)(batch < 65535 ? batch : 65535), (unsigned)((batch + 65534) / 65535));
    const int smem = (GRAM_DB ? 2 : 1) * SMC * MPK * (int)sizeof(double);
    static std::atomic<uint64_t> attr_t{0}, attr_f{0};
    cudaError_t e = vec ? set_max_dyn_smem_once(k_gram_mma_small<true>, smem, attr_t)
                        : set_max_dyn_smem_once(k_gram_mma_small<false>, smem, attr_f);
    if (e != cudaSuccess) return e;
    if (vec)
      k_gram_mma_small<true><<<grid, 256, smem, stream>>>(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g);
    else
      k_gram_mma_small<false><<<grid, 256, smem, stream>>>(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g);
    return cudaGetLastError();
  }
  int64_t splits, kchunk;
  int npairs;
  gram_splits(r, c, batch, &splits, &kchunk, &npairs);
  const int nb = (int)((c + MB - 1) / MB);
  void* own = nullptr;
  if (splits > 1 && !ws) {
    const cudaError_t e = cudaMallocAsync(&own, gram_workspace_bytes(r, c, batch), stream);
    if (e != cudaSuccess) return e;
    ws = own;
  }
  double* part = static_cast<double*>(ws);
  const dim3 grid((unsigned)(npairs * splits), (unsigned)(batch < 65535 ? batch : 65535), (unsigned)((batch + 65534) / 65535));
  if (vec)
    k_gram_mma<true><<<grid, 128, 0, stream>>>(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g, nb, (int)splits,
                                               kchunk, part);
  else
    k_gram_mma<false><<<grid, 128, 0, stream>>>(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g, nb, (int)splits,
                                                kchunk, part);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && splits > 1) {
    const int64_t total = (int64_t)npairs * batch * MB * MB;
    k_gram_reduce<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(c, batch, G, ldg, stride_g, nb, (int)splits,
                                                                       part);
    e = cudaGetLastError();
  }
  if (own) cudaFreeAsync(own, stream);
  return e;
}

cudaError_t launch_gram(int64_t r, int64_t c, int64_t batch, const float* SM, int64_t ldsm, int64_t stride_sm,
                        double* G, int64_t ldg, int64_t stride_g, void* ws, cudaStream_t stream) {
  if (r <= 0 || c <= 0 || batch <= 0) return cudaSuccess;
#ifndef GRAM_MMA
#define GRAM_MMA 1
#endif
  if (GRAM_MMA) return launch_gram_mma(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g, ws, stream);
  const int nb = (int)((c + GT - 1) / GT);
  const int pairs = nb * (nb + 1) / 2;
  const int64_t zc = (batch + 65534) / 65535;
  const int nt4 = (int)((c + 3) / 4);
  if (c <= GTRI_MAXC && batch >= 296 &&
      GTRI_PF * ((nt4 * (nt4 + 1) / 2 + 31) / 32 * 32) >= GTRI_K * 4 * nt4) {  // many small problems
    const int nt = nt4, ntiles = nt * (nt + 1) / 2;
    const int threads = ((ntiles + 31) / 32) * 32;
    const dim3 grid((unsigned)(batch < 65535 ? batch : 65535), (unsigned)zc);
    k_gram_tri<<<grid, threads, 0, stream>>>(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g);
    return cudaGetLastError();
  }
  if ((int64_t)pairs * batch < 296) {  // under two CTAs per SM with 64-blocks: smaller blocks
    const int nb32 = (int)((c + GT32 - 1) / GT32);
    const dim3 grid((unsigned)(nb32 * (nb32 + 1) / 2), (unsigned)(batch < 65535 ? batch : 65535), (unsigned)zc);
    k_gram32<<<grid, 256, 0, stream>>>(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g, nb32);
    return cudaGetLastError();
  }
  const dim3 grid((unsigned)pairs, (unsigned)(batch < 65535 ? batch : 65535), (unsigned)zc);
  k_gram<<<grid, GTH, 0, stream>>>(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g, nb);
  return cudaGetLastError();
}

}  // namespace srht
