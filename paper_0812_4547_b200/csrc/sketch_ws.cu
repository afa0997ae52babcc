// Warp-specialized SRHT tile kernel for dense FP32 columns (sm_100a).
//
// Same decomposition as sketch.cu (Ailon-Liberty pruning):
//   SM[t] = r^{-1/2} sum_slab (-1)^{popc(k_slab & s)} sum_j (-1)^{popc(k_mid & j)} (H_B D x_{s,j})[k_lo]
// with B = 2^14 rows per tile, but organised so that each element crosses the
// shared-memory crossbar only ~5 times:
//
//   producer warpgroup g (4 warps, 128 threads x 128 registers, two groups
//   alternate tiles): LDG.128 of the tile straight into registers (rows bits
//   0,1 in the vector, 9..13 in registers), D applied by XOR of the sign bit,
//   7 butterfly stages in registers (FFMA2/FADD2), STS.128 into tile buffer g;
//   group barrier; LDS of the transposed layout (bits 2..8 in registers),
//   7 more stages, STS of z = H_B D x in place.
//   consumer warps (8 warps): for every sampled row t, in a per-plan slot
//   order chosen so each warp-wide LDS hits 32 distinct banks, read
//   meta = (byte offset of k_lo | reversed k_mid bits) from shared memory and
//   z[k_lo] from the tile, and accumulate in registers.  Sub-blocks of a slab
//   are visited in Gray-code order, so the k_mid sign is carried as a "frame":
//   F <- (+-F) + z with one conditional sign flip per visit (the flipped bit of
//   the Gray code), fixed once at the end of the slab.
//
// Producer/consumer hand-off uses named barriers (bar.arrive / bar.sync):
// FULL_g (tile g holds z), EMPTY_g (tile g may be overwritten).
#include <cuda_runtime.h>

#include "internal.cuh"

namespace srht {
namespace ws {

constexpr int LOG_B = 14;
constexpr int B = 1 << LOG_B;
constexpr int ROW = 544;                 // 512 words + 32 pad: row stride = 0 mod 32 banks
constexpr int TILE_WORDS = 32 * ROW;     // 17408
constexpr int TILE_BYTES = TILE_WORDS * 4;
constexpr int NCONS = 256;
constexpr int NTHREADS = 512;

enum { BAR_FULL0 = 1, BAR_FULL1 = 2, BAR_EMPTY0 = 3, BAR_EMPTY1 = 4, BAR_GRP0 = 5, BAR_GRP1 = 6, BAR_CONS = 7 };

// Padded tile layout: row x>>9 of 512 words, rotated by 4*((x>>9)&7) words.
// Additive over disjoint bit sets, so phys(base + off) = phys(base) + phys(off).
__host__ __device__ constexpr int phys(int x) { return (x & 511) + (((x >> 9) & 7) << 2) + (x >> 9) * ROW; }

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ float flipf(float x, uint32_t mask) { return __uint_as_float(__float_as_uint(x) ^ mask); }

// Butterflies over all 7 bits of a 128-value register tile stored as 64 float2
// (value u at v[u >> 1].x/.y): natural-order H_128, unnormalized.
__device__ __forceinline__ void fwht128(float2 (&v)[64]) {
#pragma unroll
  for (int m = 0; m < 64; ++m) v[m] = __ffma2_rn(v[m], make_float2(1.f, -1.f), make_float2(v[m].y, v[m].x));
#pragma unroll
  for (int s = 1; s < 64; s <<= 1) {
#pragma unroll
    for (int m = 0; m < 64; ++m) {
      if (!(m & s)) {
        const float2 a = v[m], b = v[m | s];
        v[m] = __fadd2_rn(a, b);
        v[m | s] = __fadd2_rn(a, make_float2(-b.x, -b.y));
      }
    }
  }
}

struct Sched {
  int64_t S_act, J, n_sub;
  __device__ __forceinline__ void item(int64_t it, int64_t& col, int64_t& s, int64_t& cnt, int& L) const {
    col = it / S_act;
    s = it - col * S_act;
    const int64_t j0 = s * J;
    cnt = (n_sub - j0 < J) ? n_sub - j0 : J;
    L = 0;
    while ((int64_t(1) << L) < cnt) ++L;
  }
};

template <int RPT>
__global__ void __launch_bounds__(NTHREADS, 1) k_sketch_ws(const __grid_constant__ WsParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* tiles = reinterpret_cast<float*>(smem);
  uint32_t* meta_s = reinterpret_cast<uint32_t*>(smem + 2 * TILE_BYTES);
  const int tid = threadIdx.x;
  const Sched sc{P.S_act, P.J, P.n_sub};

  if (tid < 256) {
    // =========================== producers ===========================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;");
    const int g = tid >> 7;                 // producer group == tile buffer
    const int p = tid & 127, lane = p & 31, wg = p >> 5;
    float* tile = tiles + g * TILE_WORDS;
    const int base0 = (lane << 2) + (wg << 7);                                           // phys == identity
    const int base1 = phys((lane & 3) + ((lane >> 2) << 9) + (wg << 12));
    const int64_t n = P.n;
    int64_t produced = 0;
    for (int64_t it = blockIdx.x; it < P.n_items; it += gridDim.x) {
      int64_t col, s, cnt;
      int L;
      sc.item(it, col, s, cnt, L);
      const bool second = col >= P.ncols0;
      const ColSrc& cs = second ? P.src[1] : P.src[0];
      const int64_t lc = second ? col - P.ncols0 : col;
      const float* __restrict__ colp = cs.vals + lc * cs.ld;
      const int64_t j0 = s * P.J;
      for (int m = 0; m < (1 << L); ++m) {
        const int64_t j = m ^ (m >> 1);
        if (j >= cnt) continue;
        const bool mine = (produced & 1) == g;
        ++produced;
        if (!mine) continue;
        const int64_t row0 = (j0 + j) * (int64_t)B;
        float2 v[64];
        // ---- load D x: element x = v4 + 4*lane + 128*wg + 512*h ----
        if (cs.vec && row0 + B <= n) {
#pragma unroll
          for (int h = 0; h < 32; ++h) {
            const float4 f = __ldcs(reinterpret_cast<const float4*>(colp + row0 + base0 + (h << 9)));
            v[2 * h] = make_float2(f.x, f.y);
            v[2 * h + 1] = make_float2(f.z, f.w);
          }
        } else {
#pragma unroll
          for (int h = 0; h < 32; ++h) {
            const int64_t row = row0 + base0 + (h << 9);
            v[2 * h] = make_float2(row + 0 < n ? colp[row + 0] : 0.f, row + 1 < n ? colp[row + 1] : 0.f);
            v[2 * h + 1] = make_float2(row + 2 < n ? colp[row + 2] : 0.f, row + 3 < n ? colp[row + 3] : 0.f);
          }
        }
        const uint32_t* __restrict__ sg = P.signs + ((row0 + (wg << 7)) >> 5) + (lane >> 3);
        const int sh = (lane & 7) << 2;
#pragma unroll
        for (int h = 0; h < 32; ++h) {
          const uint32_t w = __ldg(sg + (h << 4)) >> sh;
          v[2 * h].x = flipf(v[2 * h].x, w << 31);
          v[2 * h].y = flipf(v[2 * h].y, (w << 30) & 0x80000000u);
          v[2 * h + 1].x = flipf(v[2 * h + 1].x, (w << 29) & 0x80000000u);
          v[2 * h + 1].y = flipf(v[2 * h + 1].y, (w << 28) & 0x80000000u);
        }
        fwht128(v);  // bits 0,1 (vector) and 9..13 (h)
        bar_sync(g ? BAR_EMPTY1 : BAR_EMPTY0, 384);
#pragma unroll
        for (int h = 0; h < 32; ++h)
          *reinterpret_cast<float4*>(tile + base0 + ((h & 7) << 2) + h * ROW) =
              make_float4(v[2 * h].x, v[2 * h].y, v[2 * h + 1].x, v[2 * h + 1].y);
        bar_sync(g ? BAR_GRP1 : BAR_GRP0, 128);
#pragma unroll
        for (int k = 0; k < 64; ++k) v[k] = make_float2(tile[base1 + 8 * k], tile[base1 + 8 * k + 4]);
        fwht128(v);  // bits 2..8
#pragma unroll
        for (int k = 0; k < 64; ++k) {
          tile[base1 + 8 * k] = v[k].x;
          tile[base1 + 8 * k + 4] = v[k].y;
        }
        bar_arrive(g ? BAR_FULL1 : BAR_FULL0, 384);
      }
    }
    bar_sync(g ? BAR_EMPTY1 : BAR_EMPTY0, 384);  // matches the consumers' last release
  } else {
    // =========================== consumers ===========================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
    const int c = tid - 256;
    for (int i = c; i < RPT * NCONS; i += NCONS) meta_s[i] = P.meta[i];
    bar_sync(BAR_CONS, NCONS);
    bar_arrive(BAR_EMPTY0, 384);
    bar_arrive(BAR_EMPTY1, 384);
    float acc[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) acc[q] = 0.f;
    int64_t consumed = 0;
    const uint32_t* mrow = meta_s + c;
    for (int64_t it = blockIdx.x; it < P.n_items; it += gridDim.x) {
      int64_t col, s, cnt;
      int L;
      sc.item(it, col, s, cnt, L);
      for (int m = 0; m < (1 << L); ++m) {
        const int64_t j = m ^ (m >> 1);
        const int qb = m ? __ffs(m) - 1 : 0;  // Gray-code bit flipped at step m
        if (j < cnt) {
          const int b = (int)(consumed & 1);
          ++consumed;
          bar_sync(b ? BAR_FULL1 : BAR_FULL0, 384);
          const char* tb = reinterpret_cast<const char*>(tiles) + b * TILE_BYTES;
          if (qb == 0) {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
              const uint32_t mw = mrow[q * NCONS];
              const float z = *reinterpret_cast<const float*>(tb + (mw & 0x1ffffu));
              acc[q] = flipf(acc[q], mw & 0x80000000u) + z;
            }
          } else {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
              const uint32_t mw = mrow[q * NCONS];
              const float z = *reinterpret_cast<const float*>(tb + (mw & 0x1ffffu));
              acc[q] = flipf(acc[q], (mw << qb) & 0x80000000u) + z;
            }
          }
          bar_arrive(b ? BAR_EMPTY1 : BAR_EMPTY0, 384);
        } else {
#pragma unroll
          for (int q = 0; q < RPT; ++q) acc[q] = flipf(acc[q], (mrow[q * NCONS] << qb) & 0x80000000u);
        }
      }
      // ---- slab epilogue: undo the frame sign of the last Gray step, write ----
      const uint32_t jlast = (uint32_t)(((1 << L) - 1) ^ (((1 << L) - 1) >> 1));
      const bool second = col >= P.ncols0;
      const ColSrc& cs = second ? P.src[1] : P.src[0];
      const int64_t lc = second ? col - P.ncols0 : col;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int t = P.perm[q * NCONS + c];
        if (t >= 0) {
          const uint32_t kmid = __brev(mrow[q * NCONS]) & (uint32_t)(P.J - 1);
          const float a = flipf(acc[q], (uint32_t)(__popc(kmid & jlast) & 1) << 31);
          if (P.S_act == 1) cs.out[lc * cs.ldo + t] = a * P.scale;
          else P.partials[(s * P.total_cols + col) * P.r + t] = a;
        }
        acc[q] = 0.f;
      }
    }
  }
}

template <int RPT>
cudaError_t launch_rpt(const WsParams& wp, int grid, cudaStream_t stream) {
  const size_t smem = 2 * (size_t)TILE_BYTES + (size_t)RPT * NCONS * 4;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(k_sketch_ws<RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_sketch_ws<RPT><<<grid, NTHREADS, smem, stream>>>(wp);
  return cudaGetLastError();
}

}  // namespace ws

int ws_phys(int x) { return ws::phys(x); }

cudaError_t launch_sketch_ws(const srht_plan* P, const WsParams& wp, cudaStream_t stream) {
  if (wp.total_cols <= 0) return cudaSuccess;
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(wp.n_items < sms ? wp.n_items : sms);
  switch (P->rpt2) {
    case 8: return ws::launch_rpt<8>(wp, grid, stream);
    case 16: return ws::launch_rpt<16>(wp, grid, stream);
    case 32: return ws::launch_rpt<32>(wp, grid, stream);
    case 64: return ws::launch_rpt<64>(wp, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace srht
