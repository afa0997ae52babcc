// Gram matrices of sketches: the QP form of Section 3.4, sm_100a.
//
//   G_p = SM_p^T SM_p  with SM_p = [SA | Sb] (r x c, FP32)  =  [[Q~, q~], [q~^T, Sb^T Sb]],
//   Q~ = (H~DA)^T H~DA,  q~ = (H~DA)^T (H~Db)  (reading R17: the paper's q~ = (H~DA)^T b
//   must use the sketched b for the dimensions to agree).
//
// Products of FP32 entries are exact in FP64 and are accumulated in FP64 (DFMA), so G is
// the exact Gram matrix of the FP32 sketch up to FP64 rounding.  One CTA per (problem,
// 32 x 32 block of the upper triangle); the two 32-row slabs of SM_p are staged through
// shared memory as doubles, 32 rows at a time; the block and its mirror are written.
#include <cuda_runtime.h>

#include "internal.cuh"

namespace srht {
namespace {

constexpr int GT = 32;   // block edge
constexpr int GK = 32;   // rows of SM staged per step

__global__ void __launch_bounds__(256) k_gram(int64_t r, int64_t c, int64_t batch, const float* __restrict__ SM,
                                             int64_t ldsm, int64_t stride_sm, double* __restrict__ G, int64_t ldg,
                                             int64_t stride_g, int nb) {
  __shared__ double As[GK][GT + 1];
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
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;  // ty in 0..7
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k0 = 0; k0 < r; k0 += GK) {
    // stage rows k0..k0+31 of the two column slabs: a warp reads 32 consecutive rows of a column
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int lc = ty + 8 * m;  // local column
      const int64_t k = k0 + tx;
      const int64_t ca = (int64_t)bi * GT + lc, cb = (int64_t)bj * GT + lc;
      As[tx][lc] = (k < r && ca < c) ? (double)S[k + ca * ldsm] : 0.0;
      Bs[tx][lc] = (k < r && cb < c) ? (double)S[k + cb * ldsm] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GK; ++kk) {
      const double b = Bs[kk][tx];
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[m] = fma(As[kk][ty + 8 * m], b, acc[m]);
    }
    __syncthreads();
  }
  double* __restrict__ Gp = G + p * stride_g;
  const int64_t j = (int64_t)bj * GT + tx;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int64_t i = (int64_t)bi * GT + ty + 8 * m;
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
  const dim3 grid((unsigned)pairs, (unsigned)(batch < 65535 ? batch : 65535), (unsigned)zc);
  k_gram<<<grid, 256, 0, stream>>>(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g, nb);
  return cudaGetLastError();
}

}  // namespace srht
