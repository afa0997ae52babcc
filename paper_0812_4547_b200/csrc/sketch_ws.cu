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

enum { BAR_FULL0 = 1, BAR_FULL1 = 2, BAR_EMPTY0 = 3, BAR_EMPTY1 = 4, BAR_GRP0 = 5, BAR_GRP1 = 6, BAR_CONS = 7,
       BAR_TOK0 = 8, BAR_TOK1 = 9 };

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

// Schedule.  A CTA walks items blockIdx.x, +gridDim.x, ... (item = (column, slab)).
// A slab of cnt tiles is visited as pairs p = 0 .. npairs-1 of tiles
// j_a = 2 gray(p), j_b = j_a + 1 (Gray code over the tile bits >= 1, so
// consecutive pairs differ in one k_mid bit >= 1, and the two tiles of a pair
// differ in k_mid bit 0).  Producer group 0 makes j_a, group 1 makes j_b;
// tiles with j >= cnt (all padding) are skipped.
// The same transform, ordered so that each quarter of the tile (pairs 16q..16q+15)
// gets its first 5 stages as soon as its own loads land; the 2 stages across
// quarters (pair strides 16, 32) come last.  Lets the butterflies of quarter 0
// run while quarters 1-3 are still in flight.
__device__ __forceinline__ void fwht128_quarter(float2 (&v)[64], int q) {
#pragma unroll
  for (int m = 16 * q; m < 16 * q + 16; ++m)
    v[m] = __ffma2_rn(v[m], make_float2(1.f, -1.f), make_float2(v[m].y, v[m].x));
#pragma unroll
  for (int s = 1; s < 16; s <<= 1) {
#pragma unroll
    for (int m = 16 * q; m < 16 * q + 16; ++m) {
      if (!(m & s)) {
        const float2 a = v[m], b = v[m | s];
        v[m] = __fadd2_rn(a, b);
        v[m | s] = __fadd2_rn(a, make_float2(-b.x, -b.y));
      }
    }
  }
}
__device__ __forceinline__ void fwht128_cross(float2 (&v)[64]) {
#pragma unroll
  for (int s = 16; s < 64; s <<= 1) {
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

struct Cursor {
  int it, p, np, cnt, s, col;
  bool valid;
};

__device__ __forceinline__ void cursor_item(const WsParams& P, Cursor& c) {
  c.valid = c.it < P.n_items;
  if (!c.valid) return;
  c.col = (int)(c.it / P.S_act);
  c.s = (int)(P.s_lo + c.it - (int64_t)c.col * P.S_act);  // global slab
  const int64_t j0 = (int64_t)c.s * P.J;
  c.cnt = (int)((P.n_sub - j0 < P.J) ? P.n_sub - j0 : P.J);
  int L = 0;
  while ((1 << L) < c.cnt) ++L;
  c.np = L ? (1 << (L - 1)) : 1;
  c.p = 0;
}

__device__ __forceinline__ int pair_tile(const Cursor& c, int g) { return 2 * (c.p ^ (c.p >> 1)) + g; }

// Advance to the next pair whose tile g is active (g = -1: any active pair).
__device__ __forceinline__ bool cursor_next(const WsParams& P, Cursor& c, int g) {
  while (c.valid) {
    ++c.p;
    if (c.p >= c.np) {
      c.it += gridDim.x;
      cursor_item(P, c);
      if (!c.valid) return false;
    }
    if (pair_tile(c, g < 0 ? 0 : g) < c.cnt) return true;
  }
  return false;
}

__device__ __forceinline__ void cursor_start(const WsParams& P, Cursor& c, int g) {
  c.it = blockIdx.x;
  cursor_item(P, c);
  if (c.valid && pair_tile(c, g < 0 ? 0 : g) >= c.cnt) cursor_next(P, c, g);
}

__device__ __forceinline__ const float* col_ptr(const WsParams& P, int col) {
  const bool second = col >= P.ncols0;
  const float* base = second ? P.src[1].vals : P.src[0].vals;
  const int64_t ld = second ? P.src[1].ld : P.src[0].ld;
  const int64_t lc = second ? col - P.ncols0 : col;
  return base + lc * ld;
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  // bulk prefetch needs a 16-byte aligned address and a multiple-of-16 size
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t a16 = (a + 15) & ~uintptr_t(15);
  const uint32_t skip = (uint32_t)(a16 - a);
  if (bytes <= skip + 16) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a16), "r"((bytes - skip) & ~15u) : "memory");
}

__device__ __forceinline__ void prefetch_pair(const WsParams& P, const Cursor& c, int n) {
  for (int g = 0; g < 2; ++g) {
    const int j = pair_tile(c, g);
    if (j >= c.cnt) continue;
    const int row0 = (int)(((int64_t)c.s * P.J + j) * B);
    const int rows = n - row0 < B ? n - row0 : B;
    prefetch_l2(col_ptr(P, c.col) + row0, (uint32_t)(rows * 4) & ~15u);
  }
}

#define TRACE(k)                                                                              \
  if ((DBG & 8) && blockIdx.x == 0 && (p & 31) == 0 && ntr < 64)                             \
    P.trace[((size_t)(g * 4 + wg) * 64 + ntr) * 10 + (k)] = clock64();

template <int RPT, int DBG>
__global__ void __launch_bounds__(NTHREADS, 1) k_sketch_ws(const __grid_constant__ WsParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* tiles = reinterpret_cast<float*>(smem);
  uint32_t* meta_s = reinterpret_cast<uint32_t*>(smem + 2 * TILE_BYTES);
  const int tid = threadIdx.x;

  if (tid < 256) {
    // =========================== producers ===========================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;");
    const int g = tid >> 7;                 // producer group == tile buffer == tile within a pair
    const int p = tid & 127, lane = p & 31, wg = p >> 5;
    const int base0 = (lane << 2) + (wg << 7);                                           // phys == identity
    const int base1 = phys((lane & 3) + ((lane >> 2) << 9) + (wg << 12));
    const int n = (int)P.n;
    const bool vec_ok = P.src[0].vec && (P.total_cols == P.ncols0 || P.src[1].vec);
    // ALT: the two groups alternate their butterfly phases (token barriers
    // TOK0/TOK1), so one group's shared-memory phases overlap the other's FADD2s.
    constexpr bool ALT = (DBG & 16) != 0;
    const int cg = ALT ? -1 : g;  // ALT: both groups walk every active pair
    // SOLO (experiment): group 0 produces every tile, group 1 idles.
    constexpr bool SOLO = (DBG & 32) != 0;
    Cursor cur;
    cursor_start(P, cur, SOLO ? -1 : cg);
    int ntr = 0;
    if (ALT && g == 1) bar_arrive(BAR_TOK0, 256);
    auto produce = [&](const int row0, const float* __restrict__ colp, const int bs) {
      float* tile = tiles + bs * TILE_WORDS;
        float2 v[64];
        // ---- load D x: element x = v4 + 4*lane + 128*wg + 512*h ----
        const uint4 sgn = __ldg(P.signs_ws + ((size_t)(row0 >> LOG_B) << 7) + p);
        if (DBG & 1) {
#pragma unroll
          for (int h = 0; h < 32; ++h) {
            v[2 * h] = make_float2((float)h, (float)row0);
            v[2 * h + 1] = make_float2((float)base0, 1.f);
          }
        } else if (vec_ok && row0 + B <= n) {
#pragma unroll
          for (int h = 0; h < 32; ++h) {
            const float4 f = __ldcs(reinterpret_cast<const float4*>(colp + row0 + base0 + (h << 9)));
            v[2 * h] = make_float2(f.x, f.y);
            v[2 * h + 1] = make_float2(f.z, f.w);
          }
        } else {
#pragma unroll
          for (int h = 0; h < 32; ++h) {
            const int row = row0 + base0 + (h << 9);
            v[2 * h] = make_float2(row + 0 < n ? colp[row + 0] : 0.f, row + 1 < n ? colp[row + 1] : 0.f);
            v[2 * h + 1] = make_float2(row + 2 < n ? colp[row + 2] : 0.f, row + 3 < n ? colp[row + 3] : 0.f);
          }
        }
        if (DBG & 8) {
          float acc = 0.f;
#pragma unroll
          for (int h = 0; h < 64; ++h) acc += v[h].x;
          if (acc == 1234.5f) v[0].y = 0.f;
        }
        TRACE(1)
        TRACE(2)
        if (ALT) bar_sync(g ? BAR_TOK1 : BAR_TOK0, 256);
        // D (sign XOR) and the butterflies over bits 0,1 (vector) and 9..13 (h),
        // quarter by quarter in load order.
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const uint32_t w = (qq == 0 ? sgn.x : qq == 1 ? sgn.y : qq == 2 ? sgn.z : sgn.w);
#pragma unroll
          for (int h = 8 * qq; h < 8 * qq + 8; ++h) {  // sign of (h, v) = bit ((h & 7) << 2) + v of word h >> 3
            const int b = (h & 7) << 2;
            v[2 * h].x = flipf(v[2 * h].x, (w << (31 - b)) & 0x80000000u);
            v[2 * h].y = flipf(v[2 * h].y, (w << (30 - b)) & 0x80000000u);
            v[2 * h + 1].x = flipf(v[2 * h + 1].x, (w << (29 - b)) & 0x80000000u);
            v[2 * h + 1].y = flipf(v[2 * h + 1].y, (w << (28 - b)) & 0x80000000u);
          }
          if (!(DBG & 4)) fwht128_quarter(v, qq);
        }
        if (!(DBG & 4)) fwht128_cross(v);
        if (ALT) bar_arrive(g ? BAR_TOK0 : BAR_TOK1, 256);
        TRACE(3)
        bar_sync(bs ? BAR_EMPTY1 : BAR_EMPTY0, 384);
        TRACE(4)
#pragma unroll
        for (int h = 0; h < 32; ++h)
          *reinterpret_cast<float4*>(tile + base0 + ((h & 7) << 2) + h * ROW) =
              make_float4(v[2 * h].x, v[2 * h].y, v[2 * h + 1].x, v[2 * h + 1].y);
        TRACE(5)
        bar_sync(g ? BAR_GRP1 : BAR_GRP0, 128);
        TRACE(6)
#pragma unroll
        for (int k = 0; k < 64; ++k) v[k] = make_float2(tile[base1 + 8 * k], tile[base1 + 8 * k + 4]);
        if (DBG & 8) {
          float acc = 0.f;
#pragma unroll
          for (int h = 0; h < 64; ++h) acc += v[h].x;
          if (acc == 1234.5f) v[0].y = 0.f;
        }
        TRACE(7)
        if (ALT) bar_sync(g ? BAR_TOK1 : BAR_TOK0, 256);
        if (!(DBG & 4)) {  // bits 2..8, quarter by quarter in LDS order
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) fwht128_quarter(v, qq);
          fwht128_cross(v);
        }
        if (ALT) bar_arrive(g ? BAR_TOK0 : BAR_TOK1, 256);
        TRACE(8)
#pragma unroll
        for (int k = 0; k < 64; ++k) {
          tile[base1 + 8 * k] = v[k].x;
          tile[base1 + 8 * k + 4] = v[k].y;
        }
        bar_arrive(bs ? BAR_FULL1 : BAR_FULL0, 384);
        TRACE(9)
        if (DBG & 8) ++ntr;
    };
    if (SOLO && g == 1) cur.valid = false;
    while (cur.valid) {
      TRACE(0)
      if (SOLO) {
        const Cursor c0 = cur;
        cursor_next(P, cur, -1);
        for (int sub = 0; sub < 2; ++sub) {
          const int jt = pair_tile(c0, sub);
          if (jt < c0.cnt) produce((int)(((int64_t)c0.s * P.J + jt) * B), col_ptr(P, c0.col), sub);
        }
        continue;
      }
      const int jt = pair_tile(cur, g);
      const bool active = jt < cur.cnt;
      const int row0 = (int)(((int64_t)cur.s * P.J + jt) * B);
      const float* __restrict__ colp = col_ptr(P, cur.col);
      cursor_next(P, cur, cg);
      if (ALT && !active) {  // keep the token sequence balanced
        bar_sync(BAR_TOK1, 256);
        bar_arrive(BAR_TOK0, 256);
        bar_sync(BAR_TOK1, 256);
        bar_arrive(BAR_TOK0, 256);
        continue;
      }
      produce(row0, colp, g);
    }
    if (SOLO) {
      if (g == 0) {
        bar_sync(BAR_EMPTY0, 384);
        bar_sync(BAR_EMPTY1, 384);
      }
    } else {
      bar_sync(g ? BAR_EMPTY1 : BAR_EMPTY0, 384);  // matches the consumers' last release
    }
    if (ALT && g == 0) bar_sync(BAR_TOK0, 256);   // matches group 1's initial token
  } else {
    // =========================== consumers ===========================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
    const int c = tid - 256;
    for (int i = c; i < RPT * NCONS; i += NCONS) meta_s[i] = P.meta[i];
    // L2 prefetch cursor: one thread keeps the HBM stream PREF pairs ahead.
    constexpr int PREF = 4;
    Cursor pf;
    const bool pf_thread = (c == 0);
    const int n = (int)P.n;
    if (pf_thread) {
      cursor_start(P, pf, -1);
      for (int k = 0; k < PREF && pf.valid; ++k) {
        prefetch_pair(P, pf, n);
        cursor_next(P, pf, -1);
      }
    }
    bar_sync(BAR_CONS, NCONS);
    bar_arrive(BAR_EMPTY0, 384);
    bar_arrive(BAR_EMPTY1, 384);
    float acc[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) acc[q] = 0.f;
    const uint32_t* mrow = meta_s + c;
    const char* tb0 = reinterpret_cast<const char*>(tiles);
    const char* tb1 = tb0 + TILE_BYTES;
    for (int64_t it = blockIdx.x; it < P.n_items; it += gridDim.x) {
      const int col = (int)(it / P.S_act);
      const int s = (int)(P.s_lo + it - (int64_t)col * P.S_act);  // global slab
      const int64_t j0 = (int64_t)s * P.J;
      const int cnt = (int)((P.n_sub - j0 < P.J) ? P.n_sub - j0 : P.J);
      int L = 0;
      while ((1 << L) < cnt) ++L;
      const int np = L ? (1 << (L - 1)) : 1;
      for (int pp = 0; pp < np; ++pp) {
        const int ja = 2 * (pp ^ (pp >> 1));
        const int sh = pp ? __ffs(pp) : 1;  // pair step flips k_mid bit (ctz(pp) + 1): meta bit 31 - sh
        if (ja < cnt) {
          const bool both = ja + 1 < cnt;
          if (pf_thread && pf.valid) {
            prefetch_pair(P, pf, n);
            cursor_next(P, pf, -1);
          }
          bar_sync(BAR_FULL0, 384);
          if (both) bar_sync(BAR_FULL1, 384);
          if (DBG & 2) {
          } else if (both) {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
              const uint32_t mw = mrow[q * NCONS];
              const uint32_t off = mw & 0x1ffffu;
              const float za = *reinterpret_cast<const float*>(tb0 + off);
              const float zb = flipf(*reinterpret_cast<const float*>(tb1 + off), mw & 0x80000000u);
              acc[q] = flipf(acc[q], (mw << sh) & 0x80000000u) + (za + zb);
            }
          } else {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
              const uint32_t mw = mrow[q * NCONS];
              const float za = *reinterpret_cast<const float*>(tb0 + (mw & 0x1ffffu));
              acc[q] = flipf(acc[q], (mw << sh) & 0x80000000u) + za;
            }
          }
          bar_arrive(BAR_EMPTY0, 384);
          if (both) bar_arrive(BAR_EMPTY1, 384);
        } else {
#pragma unroll
          for (int q = 0; q < RPT; ++q) acc[q] = flipf(acc[q], (mrow[q * NCONS] << sh) & 0x80000000u);
        }
      }
      // ---- slab epilogue: undo the frame sign of the last pair, write ----
      const uint32_t jlast = (uint32_t)(2 * ((np - 1) ^ ((np - 1) >> 1)));
      const bool second = col >= P.ncols0;
      float* __restrict__ outp = second ? P.src[1].out : P.src[0].out;
      const int64_t ldo = second ? P.src[1].ldo : P.src[0].ldo;
      const int64_t lc = second ? col - P.ncols0 : col;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int t = __ldg(P.perm + q * NCONS + c);  // read-only: may be batched ahead of the stores
        if (t >= 0) {
          const uint32_t kmid = __brev(mrow[q * NCONS]) & (uint32_t)(P.J - 1);
          const float a = flipf(acc[q], (uint32_t)(__popc(kmid & jlast) & 1) << 31);
          if (P.direct) outp[lc * ldo + t] = a * P.scale;
          else P.partials[((int64_t)(s - P.s_lo) * P.total_cols + col) * P.r + t] = a;
        }
        acc[q] = 0.f;
      }
    }
  }
}

template <int RPT, int DBG>
cudaError_t launch_dbg(const WsParams& wp, int grid, cudaStream_t stream) {
  const size_t smem = 2 * (size_t)TILE_BYTES + (size_t)RPT * NCONS * 4;
  static std::atomic<uint64_t> attr{0};
  const cudaError_t e = set_max_dyn_smem_once(k_sketch_ws<RPT, DBG>, (int)smem, attr);
  if (e != cudaSuccess) return e;
  k_sketch_ws<RPT, DBG><<<grid, NTHREADS, smem, stream>>>(wp);
  return cudaGetLastError();
}

template <int RPT>
cudaError_t launch_rpt(const WsParams& wp, int grid, cudaStream_t stream) {
#ifdef SRHT_WS_DEBUG
  switch (wp.debug) {
    case 1: return launch_dbg<RPT, 1>(wp, grid, stream);
    case 2: return launch_dbg<RPT, 2>(wp, grid, stream);
    case 3: return launch_dbg<RPT, 3>(wp, grid, stream);
    case 4: return launch_dbg<RPT, 4>(wp, grid, stream);
    case 5: return launch_dbg<RPT, 5>(wp, grid, stream);
    case 6: return launch_dbg<RPT, 6>(wp, grid, stream);
    case 7: return launch_dbg<RPT, 7>(wp, grid, stream);
    case 8: return launch_dbg<RPT, 8>(wp, grid, stream);
    case 9: return launch_dbg<RPT, 9>(wp, grid, stream);
    case 11: return launch_dbg<RPT, 11>(wp, grid, stream);
    case 24: return launch_dbg<RPT, 24>(wp, grid, stream);
    case 25: return launch_dbg<RPT, 25>(wp, grid, stream);
    case 16: return launch_dbg<RPT, 16>(wp, grid, stream);
    case 32: return launch_dbg<RPT, 32>(wp, grid, stream);
    case 40: return launch_dbg<RPT, 40>(wp, grid, stream);
    case 41: return launch_dbg<RPT, 41>(wp, grid, stream);
    case 43: return launch_dbg<RPT, 43>(wp, grid, stream);
    case 33: return launch_dbg<RPT, 33>(wp, grid, stream);
    case 35: return launch_dbg<RPT, 35>(wp, grid, stream);
    case 17: return launch_dbg<RPT, 17>(wp, grid, stream);
    case 20: return launch_dbg<RPT, 20>(wp, grid, stream);
    default: break;
  }
#endif
  return launch_dbg<RPT, 0>(wp, grid, stream);
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
