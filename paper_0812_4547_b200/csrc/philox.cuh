// Philox4x64-10 for the plan builder (library copy; the oracle has its own).
// Salmon, Moraes, Dror, Shaw, SC'11.  Stream convention (R4):
//   word w of stream (k0, k1) = word (w & 3) of philox(ctr=(1 + w/4, 0, 0, 0), key=(k0, k1)).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define SRHT_HD __host__ __device__ __forceinline__
#else
#define SRHT_HD inline
#endif

namespace srht {

struct u64x4 {
  uint64_t v[4];
};

SRHT_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

SRHT_HD u64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                            uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int rnd = 0; rnd < 10; ++rnd) {
    if (rnd > 0) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t hi0 = mulhi64(M0, c0), lo0 = M0 * c0;
    const uint64_t hi1 = mulhi64(M1, c2), lo1 = M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  u64x4 r;
  r.v[0] = c0;
  r.v[1] = c1;
  r.v[2] = c2;
  r.v[3] = c3;
  return r;
}

// Block q (words 4q .. 4q+3) of stream (k0, k1).
SRHT_HD u64x4 stream_block(uint64_t k0, uint64_t k1, uint64_t q) {
  return philox4x64_10(q + 1, 0, 0, 0, k0, k1);
}

SRHT_HD uint64_t stream_word(uint64_t k0, uint64_t k1, uint64_t w) {
  return stream_block(k0, k1, w >> 2).v[w & 3];
}

}  // namespace srht
