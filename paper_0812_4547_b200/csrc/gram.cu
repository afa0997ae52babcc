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
}  // namespace

cudaError_t launch_gram(int64_t r, int64_t c, int64_t batch, const float* SM, int64_t ldsm, int64_t stride_sm,
                        double* G, int64_t ldg, int64_t stride_g, cudaStream_t stream) {
  if (r <= 0 || c <= 0 || batch <= 0) return cudaSuccess;
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
