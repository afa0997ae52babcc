// FP64-accumulation mode on the TMA pipeline (plan flag SRHT_PLAN_ACCUM_FP64; sm_100a).
//
// Same output as the FP32 path and the same decomposition (Ailon-Liberty
// pruning):
//   SM[t] = r^{-1/2} sum_s (-1)^{popc(k_slab & s)} sum_j (-1)^{popc(k_mid & j)} (H_B D x_{s,j})[k_lo],
// with every add after the FP32 load done in FP64 (butterflies, pruned accumulation, slab
// partials and their reduction) and one rounding to FP32 at the end: the parity mode of
// DESIGN.md reading R14 (the north_star 1e-6 end-to-end gate sits at the FP32 rounding floor on
// the nearly consistent configs 4 and 5).  This kernel is the fast version of that mode for
// dense 16-byte aligned columns (k_sketch_f64 in sketch_f64.cu still serves CSC, batched and
// small inputs).  Structure, the FP64 counterpart of kernel v3:
//
//  * B = 2^12 rows per tile.  The raw FP32 tile (16 KB) and its 512 B of packed D bits arrive by
//    TMA bulk copy into a ring of five raw slots, separate from the z buffers: the producer group
//    that has read a slot (round 1) refills it with the tile five ahead at once, so loads run a
//    whole production time ahead (a ring shared with the z buffers, refilled only when the
//    consumers are done with a tile, left the producers waiting on the loads: 2.0 ms on config 4).
//    The tile three beyond the next ring turn is prefetched into L2.
//  * Four producer groups of 64 threads (two warps) take the tiles in turn.  Thread p holds 64
//    doubles.  Round 1: rows x = e + 2p + 128h (e < 2, h < 32) read as float2 (a warp reads
//    256 consecutive bytes), D applied by XOR on the FP32 sign bit, widened to FP64, 6 butterfly
//    stages over row bits {0, 7..11}; stored into the group's own z buffer (once the consumers
//    are done with its previous tile: ZEMPTY mbarrier) in the mid layout
//        mid(x) = ((x >> 1) & 63) + 66 * ((x & 1) | ((x >> 7) << 1))   (doubles)
//    (a warp stores 32 consecutive doubles).  Round 2: thread p owns mid row p (64 doubles,
//    double2 loads; rows are 528 B apart, so 8 threads of a quarter-warp hit 8 distinct 16-byte
//    bank groups), the stages over bits 1..6, z = H_B D x stored in place.
//  * Eight consumer warps hold RPT FP64 accumulators per thread (RPT * 256 samples per sample
//    group; r > 8192 runs G = ceil(r / 8192) groups as separate items).  The byte offsets of the
//    samples' z values live in TMEM (loaded once per CTA, streamed per tile with tcgen05.ld);
//    the slot layout puts the 16 lanes of each half-warp on distinct 8-byte bank granules where
//    the sample counts allow.  Tiles of a slab are visited in Gray-code order with the k_mid sign
//    carried as a frame (one conditional flip of the high word per visit).  At the end of a slab
//    the accumulators go to FP64 partials in slot order; k_reduce64 maps slots to output rows and
//    sums the slabs in a fixed order.
#include <cuda_runtime.h>

#include "internal.cuh"

namespace srht {
namespace v64 {

constexpr int LOG_B = V64_LOG_B;
constexpr int B = 1 << LOG_B;
constexpr int ROW = 66;                       // mid-layout row stride in doubles
constexpr int Z_BYTES = 64 * ROW * 8;         // 33792: one z (mid-layout) buffer per producer group
constexpr int NGRP = 4;                       // producer groups of 64 threads
constexpr int NRAW = 5;                       // raw-tile ring (FP32 rows + D bits, TMA-filled)
constexpr int RAW_BYTES = B * 4;              // 16384
constexpr int SIGN_BYTES = 512;               // 64 threads x 64 bits of D per tile
constexpr int RAWSLOT = RAW_BYTES + SIGN_BYTES;
constexpr int NPROD = NGRP * 64;
constexpr int NCONS = 256;
constexpr int NTHREADS = NPROD + NCONS;
constexpr int RAW_OFF = NGRP * Z_BYTES;       // 135168
constexpr int CTRL_OFF = RAW_OFF + NRAW * RAWSLOT;
// control block: FULL[raw slot] mbarriers, ZEMPTY[group] mbarriers, TMEM address
constexpr int CTRL_FULL = 0, CTRL_ZEMPTY = 64, CTRL_TMEM = 128, CTRL_BYTES = 256;
constexpr int SMEM_BYTES = CTRL_OFF + CTRL_BYTES;
static_assert(SMEM_BYTES <= 232448, "shared memory");
#ifndef V64_PREG
#define V64_PREG 152
#endif
#ifndef V64_CREG
#define V64_CREG 96
#endif
static_assert(NPROD * V64_PREG + NCONS * V64_CREG <= 65536, "register split");
#ifndef V64_PFD
#define V64_PFD 3  // L2 prefetch of the tile this many active tiles beyond the one just loaded
#endif

enum { BAR_READY0 = 1, BAR_GRP0 = BAR_READY0 + NGRP, BAR_CONS = BAR_GRP0 + NGRP };  // 0 = __syncthreads
static_assert(BAR_CONS < 16, "named barriers");

__host__ __device__ constexpr int mid(int x) { return ((x >> 1) & 63) + ROW * ((x & 1) | ((x >> 7) << 1)); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float flipf(float x, uint32_t mask) { return __uint_as_float(__float_as_uint(x) ^ mask); }
// sign flip of a double: XOR of bit 31 of `mask` into the sign bit (high word only)
__device__ __forceinline__ double flipd(double x, uint32_t mask) {
  return __hiloint2double(__double2hiint(x) ^ (int)(mask & 0x80000000u), __double2loint(x));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int CH>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&w)[CH]) {
  if constexpr (CH == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "r"(taddr));
  } else {
    static_assert(CH == 4, "chunk");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "r"(taddr));
  }
}

// Natural-order H_64 on 64 register doubles (Sylvester order, H[k,i] = (-1)^popc(k&i)).
__device__ __forceinline__ void fwht64(double (&v)[64]) {
#pragma unroll
  for (int s = 1; s < 64; s <<= 1) {
#pragma unroll
    for (int m = 0; m < 64; ++m) {
      if (!(m & s)) {
        const double a = v[m], b = v[m | s];
        v[m] = a + b;
        v[m | s] = a - b;
      }
    }
  }
}

// Flat walk over a CTA's tiles: items blockIdx.x, +gridDim.x, ... with item = (group, column,
// slab); inside an item, Gray-code steps pp = 0 .. np-1 visit tile j = gray(pp) when j < cnt.
struct Cursor {
  int it, pp, np, cnt, s, col, gi;
};

__device__ __forceinline__ int gray(int pp) { return pp ^ (pp >> 1); }
__device__ __forceinline__ void cursor_item(const V64Params& P, Cursor& c) {
  if (c.it >= P.n_items32) return;
  const int per_g = P.cols32 * P.S_act32;
  c.gi = c.it / per_g;
  const int rem = c.it - c.gi * per_g;
  c.col = rem / P.S_act32;
  c.s = P.s_lo32 + rem - c.col * P.S_act32;
  const int rest = P.n_sub32 - c.s * P.J32;
  c.cnt = rest < P.J32 ? rest : P.J32;
  c.np = 1 << (32 - __clz(c.cnt - 1));
  c.pp = 0;
}
__device__ __forceinline__ void cursor_next_active(const V64Params& P, Cursor& c) {
  while (c.it < P.n_items32) {
    ++c.pp;
    if (c.pp >= c.np) {
      c.it += gridDim.x;
      cursor_item(P, c);
      if (c.it >= P.n_items32) return;
    }
    if (gray(c.pp) < c.cnt) return;
  }
}
__device__ __forceinline__ void cursor_start(const V64Params& P, Cursor& c) {
  c.it = blockIdx.x;
  cursor_item(P, c);
}
__device__ __forceinline__ const float* col_ptr(const V64Params& P, int col) {
  const bool second = col >= P.ncols0;
  const float* base = second ? P.src[1].vals : P.src[0].vals;
  const int64_t ld = second ? P.src[1].ld : P.src[0].ld;
  const int64_t lc = second ? col - P.ncols0 : col;
  return base + lc * ld;
}

// Load tile `c` into raw slot k (its D bits, and its rows unless it is the ragged tail tile,
// which the producers stage themselves), then prefetch the tile V64_PFD active tiles beyond the
// next ring turn into L2.
__device__ __forceinline__ void raw_issue(const V64Params& P, Cursor c, int k, unsigned char* smem) {
  if (c.it >= P.n_items32) return;
  const uint32_t bar = smem_u32(smem + CTRL_OFF + CTRL_FULL + 8 * k);
  const int tile = c.s * P.J32 + gray(c.pp);
  const int64_t row0 = (int64_t)tile * B;
  const bool full = row0 + B <= P.n;
  unsigned char* slot = smem + RAW_OFF + (size_t)k * RAWSLOT;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"((full ? RAW_BYTES : 0) + SIGN_BYTES)
               : "memory");
  uint64_t keep, stream;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(stream));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(slot + RAW_BYTES)),
      "l"(P.signs + (int64_t)tile * 64), "n"(SIGN_BYTES), "r"(bar), "l"(keep)
      : "memory");
  if (full)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(slot)),
        "l"(col_ptr(P, c.col) + row0), "n"(RAW_BYTES), "r"(bar), "l"(stream)
        : "memory");
  if (V64_PFD > 0) {
#pragma unroll 1
    for (int i = 0; i < NRAW + V64_PFD; ++i) cursor_next_active(P, c);
    if (c.it < P.n_items32) {
      const int64_t r1 = (int64_t)(c.s * P.J32 + gray(c.pp)) * B;
      if (r1 + B <= P.n)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(col_ptr(P, c.col) + r1), "n"(RAW_BYTES)
                     : "memory");
    }
  }
}

template <int RPT>
__global__ void __launch_bounds__(NTHREADS, 1) k_sketch_tma64(const __grid_constant__ V64Params P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + CTRL_OFF + CTRL_TMEM);
  const int tid = threadIdx.x;
  const int MWT = P.G * RPT;  // TMEM columns per consumer warp half (offsets of every group)
  const int tcols = (2 * MWT) <= 32 ? 32 : (2 * MWT) <= 64 ? 64 : (2 * MWT) <= 128 ? 128 : 256;

  if (tid == 0) {
    for (int k = 0; k < NRAW; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(smem + CTRL_OFF + CTRL_FULL + 8 * k)));
    for (int g = 0; g < NGRP; ++g)  // ZEMPTY[g]: one arrival per consumer warp
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(smem + CTRL_OFF + CTRL_ZEMPTY + 8 * g)),
                   "r"(NCONS / 32));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid >= NPROD && tid < NPROD + 32) {  // consumer warp 0 allocates TMEM
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  if (tid < NPROD) {
    // =========================== producers ===========================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(V64_PREG));
    const int g = tid >> 6;
    const int p = tid & 63;
    const int64_t n = P.n;
    Cursor cur;
    cursor_start(P, cur);
    if (tid == 0) {  // fill the raw ring: flat tiles 0 .. NRAW-1
      Cursor c0 = cur;
      for (int k = 0; k < NRAW; ++k) {
        raw_issue(P, c0, k, smem);
        cursor_next_active(P, c0);
      }
    }
    for (int k = 0; k < g; ++k) cursor_next_active(P, cur);
    int f = g;
    double* zb = reinterpret_cast<double*>(smem + (size_t)g * Z_BYTES);
    const uint32_t zempty = smem_u32(smem + CTRL_OFF + CTRL_ZEMPTY + 8 * g);
    while (cur.it < P.n_items32) {
      const int k = f % NRAW;
      const int64_t row0 = (int64_t)(cur.s * P.J32 + gray(cur.pp)) * B;
      unsigned char* slot = smem + RAW_OFF + (size_t)k * RAWSLOT;
      float* raw = reinterpret_cast<float*>(slot);
      mbar_wait(smem_u32(smem + CTRL_OFF + CTRL_FULL + 8 * k), (uint32_t)((f / NRAW) & 1));
      const uint2 sg = *reinterpret_cast<const uint2*>(slot + RAW_BYTES + 8 * p);
      if (row0 + B > n) {  // ragged tail tile (no TMA data): stage it, rows >= n read as zero
        const float* colp = col_ptr(P, cur.col);
#pragma unroll 4
        for (int h = 0; h < 32; ++h) {
          const int64_t row = row0 + 2 * p + 128 * h;
          *reinterpret_cast<float2*>(raw + 2 * p + 128 * h) =
              make_float2(row < n ? colp[row] : 0.f, row + 1 < n ? colp[row + 1] : 0.f);
        }
        bar_sync(BAR_GRP0 + g, 64);
      }
      double v[64];
      // ---- round 1: rows e + 2p + 128h -> v[e + 2h]; D = bit 2(h & 15) + e of word h >> 4 ----
#pragma unroll
      for (int h = 0; h < 32; ++h) {
        const float2 x = *reinterpret_cast<const float2*>(raw + 2 * p + 128 * h);
        const uint32_t w = h < 16 ? sg.x : sg.y;
        const int bt = (h & 15) << 1;
        v[2 * h] = (double)flipf(x.x, __funnelshift_l(w, w, 31 - bt) & 0x80000000u);
        v[2 * h + 1] = (double)flipf(x.y, __funnelshift_l(w, w, 30 - bt) & 0x80000000u);
      }
      bar_sync(BAR_GRP0 + g, 64);  // every raw row of slot k has been read: refill it (tile f + NRAW)
      if (p == 0) {
        Cursor cn = cur;
#pragma unroll 1
        for (int i = 0; i < NRAW; ++i) cursor_next_active(P, cn);
        raw_issue(P, cn, k, smem);
      }
      fwht64(v);  // row bits 0 and 7..11
      if (f >= NGRP) mbar_wait(zempty, (uint32_t)(((f / NGRP) - 1) & 1));  // consumers done with tile f - 4
#pragma unroll
      for (int u = 0; u < 64; ++u) zb[p + ROW * u] = v[u];
      bar_sync(BAR_GRP0 + g, 64);
      // ---- round 2: mid row p (row bits 1..6 in registers) ----
      double* rowp = zb + ROW * p;
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const double2 d2 = *reinterpret_cast<const double2*>(rowp + 2 * m);
        v[2 * m] = d2.x;
        v[2 * m + 1] = d2.y;
      }
      fwht64(v);
#pragma unroll
      for (int m = 0; m < 32; ++m) *reinterpret_cast<double2*>(rowp + 2 * m) = make_double2(v[2 * m], v[2 * m + 1]);
      bar_arrive(BAR_READY0 + g, 64 + NCONS);
#pragma unroll 1
      for (int i = 0; i < NGRP; ++i) cursor_next_active(P, cur);
      f += NGRP;
    }
  } else {
    // =========================== consumers ===========================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(V64_CREG));
    const int c = tid - NPROD;
    const int wc = c >> 5;
    const uint32_t tbase = *tmem_slot;
    const uint32_t taddr0 = tbase + ((uint32_t)(32 * (wc & 3)) << 16) + (uint32_t)((wc >> 2) * MWT);
    for (int gi = 0; gi < P.G; ++gi)  // gather offsets of every sample group -> TMEM (once)
#pragma unroll
      for (int k = 0; k < RPT; k += 4) {
        const uint4 m4 = __ldg(reinterpret_cast<const uint4*>(P.meta + ((size_t)gi * NCONS + c) * RPT + k));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr0 + gi * RPT + k),
                     "r"(m4.x), "r"(m4.y), "r"(m4.z), "r"(m4.w)
                     : "memory");
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    constexpr int CH = RPT >= 8 ? 8 : 4;
    double acc[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) acc[q] = 0.0;
    const int slots_n = RPT * NCONS;
    int f = 0;
    for (int it = blockIdx.x; it < P.n_items32; it += gridDim.x) {
      Cursor ci;
      ci.it = it;
      cursor_item(P, ci);
      const int col = ci.col, s = ci.s, cnt = ci.cnt, np = ci.np, gi = ci.gi;
      const uint32_t taddr = taddr0 + gi * RPT;
      const uint32_t* __restrict__ mrow = P.masks + (size_t)gi * P.log_j * NCONS + c;
      for (int pp = 0; pp < np; ++pp) {
        const uint32_t mk = pp ? __ldg(mrow + (__ffs(pp) - 1) * NCONS) : 0u;
        if (gray(pp) < cnt) {
          const int zg = f % NGRP;
          const char* bb = reinterpret_cast<const char*>(smem + (size_t)zg * Z_BYTES);
          uint32_t w[2][CH];
          tmem_ld<CH>(taddr, w[0]);  // in flight while waiting for the tile
          bar_sync(BAR_READY0 + zg, 64 + NCONS);
#pragma unroll
          for (int k = 0; k < RPT; k += CH) {
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (k + CH < RPT) tmem_ld<CH>(taddr + k + CH, w[((k / CH) + 1) & 1]);
            const uint32_t* wk = w[(k / CH) & 1];
#pragma unroll
            for (int i = 0; i < CH; ++i) {
              const int q = k + i;
              const double z = *reinterpret_cast<const double*>(bb + wk[i]);
              acc[q] = flipd(acc[q], __funnelshift_l(mk, mk, 31 - q)) + z;
            }
          }
          __syncwarp();
          if ((c & 31) == 0)  // this warp is done reading z buffer zg
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(smem + CTRL_OFF + CTRL_ZEMPTY + 8 * zg))
                         : "memory");
          ++f;
        } else {
#pragma unroll
          for (int q = 0; q < RPT; ++q) acc[q] = flipd(acc[q], __funnelshift_l(mk, mk, 31 - q));
        }
      }
      // slab epilogue: undo the frame sign of the last step, store in slot order (coalesced)
      const uint32_t jlast = (uint32_t)gray(np - 1);
      uint32_t fm = 0u;
      for (int l = 0; l < P.log_j; ++l)
        if ((jlast >> l) & 1u) fm ^= __ldg(mrow + l * NCONS);
      double* __restrict__ dst =
          P.partials + (((int64_t)(s - P.s_lo32) * P.G + gi) * P.total_cols + col) * slots_n + c;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        dst[q * NCONS] = flipd(acc[q], __funnelshift_l(fm, fm, 31 - q));
        acc[q] = 0.0;
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    bar_sync(BAR_CONS, NCONS);
    if (wc == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(tcols));
    }
  }
}

// Fixed-order slab reduction of the slot-order FP64 partials: thread j = slot (q, c) of group gi
// finds its output row t, sums the slabs in increasing order with the slab sign of K[t], scales
// by r^{-1/2} in FP64 and rounds once (reading R10); row shards get the unscaled sum.
__global__ void k_reduce64(const __grid_constant__ SketchParams P, const int32_t* __restrict__ ttab, int rpt, int G,
                           int slab_shift) {
  const int64_t slots = (int64_t)rpt * 256;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t cg = blockIdx.y + (int64_t)blockIdx.z * 65535;  // (group, column)
  const int64_t gi = cg / P.total_cols, col = cg - gi * P.total_cols;
  if (j >= slots || gi >= G) return;
  const int q = (int)(j >> 8), c = (int)(j & 255);
  const int32_t t = ttab[((size_t)gi * 256 + c) * rpt + q];
  if (t < 0) return;
  const uint32_t ks = (uint32_t)(P.K[t] >> slab_shift);
  double sum = 0.0;
  for (int64_t s = 0; s < P.S_act; ++s) {
    const double v = P.partials64[((s * G + gi) * P.total_cols + col) * slots + j];
    sum += (__popc(ks & (uint32_t)(P.s_lo + s)) & 1) ? -v : v;
  }
  if (P.part_out) {
    P.part_out[col * P.ldp + t] = sum;
    return;
  }
  const bool second = col >= P.ncols0;
  const ColSrc& cs = second ? P.src[1] : P.src[0];
  const int64_t lc = second ? col - P.ncols0 : col;
  cs.out[lc * cs.ldo + t] = (float)(sum * P.scale_f64);
}

template <int RPT>
cudaError_t launch_rpt(const V64Params& vp, int grid, cudaStream_t stream) {
  static std::atomic<uint64_t> attr{0};
  const cudaError_t e = set_max_dyn_smem_once(k_sketch_tma64<RPT>, SMEM_BYTES, attr);
  if (e != cudaSuccess) return e;
  k_sketch_tma64<RPT><<<grid, NTHREADS, SMEM_BYTES, stream>>>(vp);
  return cudaGetLastError();
}

}  // namespace v64

int v64_mid(int x) { return v64::mid(x); }

cudaError_t launch_sketch_tma64(const srht_plan* P, const V64Params& vp, cudaStream_t stream) {
  if (vp.total_cols <= 0 || vp.n_items32 <= 0) return cudaSuccess;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = vp.n_items32 < sms ? vp.n_items32 : sms;
  switch (P->rpt64) {
    case 4: return v64::launch_rpt<4>(vp, grid, stream);
    case 8: return v64::launch_rpt<8>(vp, grid, stream);
    case 16: return v64::launch_rpt<16>(vp, grid, stream);
    case 32: return v64::launch_rpt<32>(vp, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_reduce64(const SketchParams& sp, const int32_t* ttab, int rpt, int G, int slab_shift,
                            cudaStream_t stream) {
  const int64_t cg = sp.total_cols * G;
  const dim3 grid((unsigned)rpt, (unsigned)(cg < 65535 ? cg : 65535), (unsigned)((cg + 65534) / 65535));
  v64::k_reduce64<<<grid, 256, 0, stream>>>(sp, ttab, rpt, G, slab_shift);
  return cudaGetLastError();
}

}  // namespace srht
