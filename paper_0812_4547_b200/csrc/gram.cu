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

}  // namespace

cudaError_t launch_gram(int64_t r, int64_t c, int64_t batch, const float* SM, int64_t ldsm, int64_t stride_sm,
                        double* G, int64_t ldg, int64_t stride_g, cudaStream_t stream) {
  if (r <= 0 || c <= 0 || batch <= 0) return cudaSuccess;
  const int nb = (int)((c + GT - 1) / GT);
  const int pairs = nb * (nb + 1) / 2;
  const int64_t zc = (batch + 65534) / 65535;
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
