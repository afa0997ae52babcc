// Kernel v3: TMA-fed, warp-specialized SRHT tile kernel for dense FP32 columns (sm_100a).
//
// Same decomposition as kernels v1/v2 (Ailon-Liberty pruning):
//   SM[t] = r^{-1/2} sum_slab (-1)^{popc(k_slab & s)} sum_j (-1)^{popc(k_mid & j)} (H_B D x_{s,j})[k_lo]
// with B = 2^14 rows per tile.  What changes against v2:
//
//  * Tiles arrive by TMA bulk copy (cp.async.bulk, four 16 KB quarters per tile, each
//    with its own FULL mbarrier) into a ring of three shared-memory buffers, L2-prefetched
//    three tiles ahead.  Measured on B200 (profiles/r01_mb_l1_sharing.txt): a TMA fill
//    does not take shared-memory bandwidth from LDS/STS, while an LDG stream costs ~1.3
//    crossbar words per word loaded.  The last consumer warp done with a buffer (its
//    EMPTY mbarrier arrival is the one that leaves a pending count of 1) copies quarter
//    0 and the tile's D bits; the producer thread that sees quarter 0 land copies
//    quarters 1..3 (a lone quarter lands ~4x sooner than four concurrent ones).
//  * Producer thread p of group g (two groups of 4 warps, alternate tiles) holds
//    128 values.  Round 1 reads its raw rows x = e + 2p + 256h (e = 0,1; h < 64)
//    with LDS.64 (half-warps read 32 consecutive words: conflict-free), applies D,
//    and runs the 7 butterfly stages over row bits {0, 8..13} in registers, quarter by
//    quarter as the quarters land.  After a group barrier it writes the results into
//    the "mid" layout
//        mid(x) = col(x) + 130 row(x),  col = bits 1..7 of x,  row = bit 0 | bits 8..13 << 1
//    (STS.32; a warp writes 32 consecutive words).  Round 2: thread p owns mid row p,
//    reads it with LDS.64 (rows are 130 words apart, so a half-warp hits 16 distinct
//    bank pairs), runs the stages over bits 1..7 and writes z = H_B D x back in place.
//  * Consumer warps (8 x 32 threads, 64 accumulators each at r = 16384) gather
//    z[k_lo] for their samples.  The byte offsets of the samples' z values live in
//    tensor memory (TMEM) and are streamed per tile with tcgen05.ld one chunk ahead, so
//    they use no shared-memory bandwidth and no registers between tiles.  Tiles of a
//    slab are visited in Gray-code order; the k_mid sign is carried as a frame (one
//    conditional flip per visit, from a per-thread bit mask in shared memory).  At the
//    end of a slab the accumulators go to the partials in slot order (coalesced);
//    k_reduce_v3 maps slots to output rows.
//
// Hand-off: mbarriers FULL[b][q] (quarter q of buffer b landed, or tail tile released)
// and EMPTY[b] (consumer warps done with buffer b); named barriers READY_b (z of buffer
// b written: 128 producer arrivals + 256 consumer syncs), GRP_g (producer group), CONS
// (consumers, before TMEM is released).
#include <cuda_runtime.h>

#include <cstring>

#include "internal.cuh"

namespace srht {
namespace v3 {

constexpr int LOG_B = 14;
constexpr int B = 1 << LOG_B;
constexpr int ROWW = 130;                  // mid-layout row stride in words
constexpr int BUF_WORDS = 128 * ROWW;      // 16640 (raw tile needs 16384)
constexpr int BUF_BYTES = BUF_WORDS * 4;   // 66560
constexpr int NBUF = 3;
constexpr int NCONS = 256;
constexpr int NTHREADS = 512;
constexpr int SIGN_OFF = NBUF * BUF_BYTES;            // per buffer: 128 threads x 16 B of D bits
constexpr int MASK_OFF = SIGN_OFF + NBUF * 2048;
constexpr int CTRL_OFF = MASK_OFF + V3_MAX_LOGJ * NCONS * 8;
// Register split (per thread): producers V3_PREG, consumers V3_CREG; 256 x (P + C) <= 64K.
#ifndef V3_PREG
#define V3_PREG 152
#endif
#ifndef V3_CREG
#define V3_CREG 96
#endif
static_assert(256 * (V3_PREG + V3_CREG) <= 65536, "register split");
#ifndef V3_EMPTY_MBAR
#define V3_EMPTY_MBAR 1
#endif
#ifndef V3_QSPLIT
#define V3_QSPLIT 1
#endif
// FULL mbarriers: NQ per buffer, one per contiguous 1/NQ of the tile (round 1 reads the
// tile quarter by quarter, so it starts as soon as the first quarter has landed).
constexpr int NQ = V3_QSPLIT ? 4 : 1;
// Split issue: the refill copies quarter 0 (and the D bits) only; the producer thread that
// sees quarter 0 land copies quarters 1..3 (a lone quarter lands ~4x sooner than four
// concurrent ones, and the later quarters are needed ~700 cycles apart).
#ifndef V3_SPLIT_ISSUE
#define V3_SPLIT_ISSUE 1
#endif
constexpr bool SPLIT = V3_SPLIT_ISSUE && NQ == 4;
// Quarters copied by the refill (the producer copies the rest): one for r = 16384 (RPT 64: config 5,
// 7.08 vs 7.33 ms with two), two for smaller r (RPT <= 32: config 4, 0.434 vs 0.447 ms back to back;
// profiles/r02c_ab_params.jsonl).
#ifndef V3_REFILL_Q
#define V3_REFILL_Q 0  // 0: by RPT as above
#endif
__host__ __device__ constexpr int nref_for(int rpt) {
  return !SPLIT ? NQ : V3_REFILL_Q > 0 ? V3_REFILL_Q : (rpt >= 64 ? 1 : 2);
}
// control block: FULL mbarriers [0, 8 NQ NBUF), TMEM address [96,100), EMPTY mbarriers
// [104,128), slot states [128,..)
constexpr int CTRL_TMEM = 96, CTRL_EMPTY = 104, CTRL_SLOTS = 128, CTRL_TFULL = 384, CTRL_BYTES = 512;
static_assert(8 * NQ * NBUF <= CTRL_TMEM, "FULL mbarriers overflow");
constexpr int SMEM_BYTES = CTRL_OFF + CTRL_BYTES;

enum { BAR_READY0 = 1, BAR_GRP0 = 4, BAR_CONS = 6 };  // named barriers (0 = __syncthreads)

// V3_TMEM_RAW (internal.cuh): round 1 reads the TMA-landed raw tile from tensor memory
// (tcgen05.cp smem -> TMEM, then tcgen05.ld) instead of with LDS; round 1 then owns row bits
// {0, 1, 9..13} (thread p = bits 2..8: TMEM lane p holds the 16-byte rows 4p + 512h') and the mid
// layout's rows/columns follow.
#if V3_TMEM_RAW
__host__ __device__ constexpr int mid(int x) { return ((x >> 2) & 127) + ROWW * ((x & 3) | ((x >> 9) << 2)); }
#else
__host__ __device__ constexpr int mid(int x) { return ((x >> 1) & 127) + ROWW * ((x & 1) | ((x >> 8) << 1)); }
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float flipf(float x, uint32_t mask) { return __uint_as_float(__float_as_uint(x) ^ mask); }

template <int CH>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&w)[CH]) {
  if constexpr (CH == 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]),
          "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
        : "r"(taddr));
  } else if constexpr (CH == 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(taddr));
  } else if constexpr (CH == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "r"(taddr));
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "r"(taddr));
  }
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Natural-order H_128 on 128 register values stored as 64 float2 (value u at v[u >> 1].x/.y).
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

// The same transform split for software pipelining inside one warp: the pair stage and
// the stages over m-bits 0..3 touch only the 16 float2 of quarter q (m in [16q, 16q+16)),
// so they can run as soon as that quarter's loads land; stage_m(S) is one cross stage.
__device__ __forceinline__ void fwht_quarter(float2 (&v)[64], int q) {
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
template <int S>
__device__ __forceinline__ void bfly(float2 (&v)[64], int m) {
  const float2 a = v[m], b = v[m | S];
  v[m] = __fadd2_rn(a, b);
  v[m | S] = __fadd2_rn(a, make_float2(-b.x, -b.y));
}

// Walk over the CTA's tiles: items blockIdx.x, +gridDim.x, ... (item = (column, slab));
// inside an item, Gray-code steps pp = 0 .. np-1 visit tile j = gray(pp) when j < cnt.
struct Cursor {
  int it, pp, np, cnt, s, col;  // valid while it < n_items
};

__device__ __forceinline__ void cursor_item(const V3Params& P, Cursor& c) {
  if (c.it >= P.n_items32) return;
  c.col = c.it / P.S_act32;
  c.s = P.s_lo32 + c.it - c.col * P.S_act32;  // global slab
  const int rest = P.n_sub32 - c.s * P.J32;
  c.cnt = rest < P.J32 ? rest : P.J32;
  c.np = 1 << (32 - __clz(c.cnt - 1));  // next power of two >= cnt (cnt >= 1)
  c.pp = 0;
}
__device__ __forceinline__ int gray(int pp) { return pp ^ (pp >> 1); }
// Advance to the next ACTIVE tile (j < cnt).
__device__ __forceinline__ void cursor_next_active(const V3Params& P, Cursor& c) {
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
__device__ __forceinline__ void cursor_start(const V3Params& P, Cursor& c) {
  c.it = blockIdx.x;
  cursor_item(P, c);  // pp = 0: tile 0 is always active (cnt >= 1)
}

__device__ __forceinline__ const float* col_ptr(const V3Params& P, int col) {
  const bool second = col >= P.ncols0;
  const float* base = second ? P.src[1].vals : P.src[0].vals;
  const int64_t ld = second ? P.src[1].ld : P.src[0].ld;
  const int64_t lc = second ? col - P.ncols0 : col;
  return base + lc * ld;
}

// TMA issue.  Buffer slot b (tiles f = b, b+3, ...) keeps its own cursor: the next tile to
// load into it.  The consumer warp that finishes tile f last (EMPTY[b] election; the
// shared-memory counter is the V3_EMPTY_MBAR=0 variant) refills the slot: tile f+3's 2 KB of
// packed D bits (L2 evict-last: the sign words are re-read for every column) and its first
// 16 KB quarter of rows (L2 evict-first; all four quarters with V3_SPLIT_ISSUE=0, the
// producer copies quarters 1..3 otherwise); then it advances the slot cursor by three
// active tiles and prefetches the tile V3_PFD tiles beyond f+3 into L2.  The cursors live
// in shared memory and cost the consumers no registers.
struct SlotState {
  Cursor cur;   // next tile for this slot
  int count;    // consumer warps done with the slot's current tile (atomic refill)
  int f;        // flat index of that tile (trace builds)
};
#ifndef V3_L2_HINTS
#define V3_L2_HINTS 1
#endif
static_assert(CTRL_SLOTS + NBUF * sizeof(SlotState) <= CTRL_TFULL, "control block overflows");
static_assert(CTRL_TFULL + 8 * NQ * NBUF <= CTRL_BYTES, "control block overflows");
// TMEM columns: [0, 3 x 128) raw tiles of the three buffers (TMEM_RAW), then the consumers' gather offsets
constexpr int TRAW_COLS = V3_TMEM_RAW ? NBUF * 128 : 0;
// V3_META_PER_BUF: the gather offsets are held once per tile buffer with the buffer's base already
// added, so a gather is one LDS [offset + smem base] (no per-sample IMAD of b x BUF_BYTES).
#ifndef V3_META_PER_BUF
#define V3_META_PER_BUF 1
#endif
constexpr bool META_PER_BUF = V3_META_PER_BUF && !V3_TMEM_RAW;
__host__ __device__ constexpr int pow2_at_least(int x) { return x <= 32 ? 32 : 2 * pow2_at_least((x + 1) / 2); }

// shared-memory matrix descriptor, no swizzle, K-major canonical layout (8-row core matrices):
// start address, leading byte offset, stride byte offset 128 (8 rows x 16 B), sm100 version bit
__device__ __forceinline__ uint64_t desc_nosw(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ void tile_src(const V3Params& P, const Cursor& c, int& tile, const float*& src, bool& full) {
  tile = c.s * P.J32 + gray(c.pp);
  const int64_t row0 = (int64_t)tile * B;
  full = row0 + B <= P.n;
  src = col_ptr(P, c.col) + row0;
}

// Flat tile f of this CTA when every slab of the launch is full (P.uniform: J tiles per item,
// no inactive Gray-code steps): item f >> log_j, step f & (J - 1).  False past the last item.
__device__ __forceinline__ bool flat_tile(const V3Params& P, int f, int& tile, const float*& src, bool& full) {
  const int it = blockIdx.x + (f >> P.log_j) * gridDim.x;
  if (it >= P.n_items32) return false;
  const int col = it / P.S_act32;
  const int s = P.s_lo32 + it - col * P.S_act32;
  tile = s * P.J32 + gray(f & (P.J32 - 1));
  const int64_t row0 = (int64_t)tile * B;
  full = row0 + B <= P.n;
  src = col_ptr(P, col) + row0;
  return true;
}

template <int DBG, int NREF>
__device__ __forceinline__ void tma_issue(const V3Params& P, SlotState& st, int b, unsigned char* smem) {
  Cursor c = st.cur;
  int tile;
  const float* src;
  bool full;
  const int f_load = st.f;
#ifndef V3_UNIFORM
#define V3_UNIFORM 0
#endif
  if (V3_UNIFORM && P.uniform) {
    if (!flat_tile(P, f_load, tile, src, full)) return;
  } else {
    if (c.it >= P.n_items32) return;
    tile_src(P, c, tile, src, full);
  }
  const Cursor st_loaded = c;
  if ((DBG & 1) && blockIdx.x == 0 && st.f < 4096) P.trace[((size_t)2 * 4096 + st.f) * 8 + 6] = clock64();
  st.f += NBUF;
  const uint32_t bar = smem_u32(smem + CTRL_OFF + 8 * NQ * b);  // quarter q: bar + 8 q
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
  for (int q = 0; q < NREF; ++q) {  // signs ride with the first part; a tail tile has no data parts
    const int bytes = (full ? B * 4 / NQ : 0) + (q == 0 ? 2048 : 0);
    if (bytes)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar + 8 * q), "r"(bytes) : "memory");
    else
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar + 8 * q) : "memory");
  }
  uint64_t keep, stream;
  if (V3_L2_HINTS) {
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(stream));
  } else {
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(keep));
    stream = keep;
  }
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], 2048, [%2], %3;" ::"r"(
          smem_u32(smem + SIGN_OFF + 2048 * b)),
      "l"(P.signs + ((int64_t)tile << 7)), "r"(bar), "l"(keep)
      : "memory");
  if (full) {  // a tail tile is loaded by the producers themselves (guarded)
    const uint32_t dst = smem_u32(smem + (size_t)b * BUF_BYTES);
#pragma unroll
    for (int k = 0; k < (SPLIT ? NREF : 4); ++k)  // 16 KB each
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], 16384, [%2], %3;" ::"r"(
              dst + k * 16384),
          "l"(reinterpret_cast<const char*>(src) + k * 16384), "r"(bar + 8 * (k * NQ / 4)), "l"(stream)
          : "memory");
  }
#ifndef V3_PFD
#define V3_PFD 3  // L2 prefetch of the tile V3_PFD active tiles beyond the one just loaded (0: none)
#endif
  if (V3_UNIFORM && P.uniform) {
    if (V3_PFD > 0 && flat_tile(P, f_load + V3_PFD, tile, src, full) && full)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(B * 4) : "memory");
    return;
  }
#pragma unroll
  for (int k = 0; k < NBUF; ++k) cursor_next_active(P, c);
  st.cur = c;
  if (V3_PFD > 0) {
    Cursor pc = V3_PFD >= NBUF ? c : st_loaded;
#pragma unroll
    for (int k = 0; k < (V3_PFD >= NBUF ? V3_PFD - NBUF : V3_PFD); ++k) cursor_next_active(P, pc);
    c = pc;
  }
  if (V3_PFD > 0 && c.it < P.n_items32) {
    tile_src(P, c, tile, src, full);
    if (full) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(B * 4) : "memory");
  }
}

// Experiment variants (DBG != 0 only for srht_debug_set_trace / srht_debug_set_mode; results
// are wrong for the knock-outs): bit 0 = clock64 at phase boundaries of CTA 0 for flat tiles
// 0..4095 (scripts/v3_trace.py); bit 1 = consumers skip the gather loads; bit 2 = producers
// skip the butterflies; bit 3 = producers skip the shared-memory loads/stores of both rounds;
// bit 4 = producers skip the whole transform (data movement only).
#define V3_TRACE_TILES 4096  // CTA 0, flat tiles 0..4095; trace buffer 3 x 4096 x 8 int64
#define V3_TRACE(role, k, pt)                                                            \
  if ((DBG & 1) && blockIdx.x == 0 && (k) < V3_TRACE_TILES)                              \
    P.trace[((size_t)(role) * V3_TRACE_TILES + (k)) * 8 + (pt)] = clock64();

// Meta words per TMEM load: the largest of V3_CH, 8, 4, 2 that divides the load slots.
#ifndef V3_CH
#define V3_CH 8
#endif
__host__ __device__ constexpr int pick_ch(int mw) {
  return (mw % V3_CH == 0 && mw >= V3_CH) ? V3_CH : (mw % 8 == 0) ? 8 : (mw % 4 == 0) ? 4 : 2;
}

// RPT accumulators per consumer thread; the first PAIRS load slots each feed an accumulator
// pair (two samples with the same k_lo: one LDS, one FADD2 with a broadcast operand), the other
// RPT - 2 PAIRS accumulators one load slot each (plan layout: api.cu deal_v3_pairs).
template <int RPT, int PAIRS, int DBG>
__global__ void __launch_bounds__(NTHREADS, 1) k_sketch_tma(const __grid_constant__ V3Params P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint2* masks_s = reinterpret_cast<uint2*>(smem + MASK_OFF);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + CTRL_OFF + CTRL_TMEM);
  SlotState* slots = reinterpret_cast<SlotState*>(smem + CTRL_OFF + CTRL_SLOTS);
  static_assert(PAIRS % 2 == 0 && 2 * PAIRS <= RPT && (RPT - PAIRS) % 4 == 0, "pair slots");
  constexpr int MW = RPT - PAIRS;                    // gather byte offsets (TMEM columns) per consumer thread
  constexpr int NREF = nref_for(RPT);
  // TMEM columns allocated: raw tiles (TMEM_RAW) + gather offsets (two consumer warps per lane quarter)
#ifndef V3_TCOLS_ALL
#define V3_TCOLS_ALL 0  // experiment: allocate all 512 TMEM columns for every RPT
#endif
  constexpr int TCOLS = (V3_TMEM_RAW || V3_TCOLS_ALL) ? 512 : META_PER_BUF ? pow2_at_least(2 * NBUF * MW) : ((2 * MW) < 32 ? 32 : 2 * MW);
  const int tid = threadIdx.x;

  // ---------------- setup (all threads) ----------------
  if (tid == 0) {
    for (int b = 0; b < NQ * NBUF; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(smem + CTRL_OFF + 8 * b)));
    for (int b = 0; b < NBUF; ++b)  // EMPTY[b]: one arrival per consumer warp
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(smem + CTRL_OFF + CTRL_EMPTY + 8 * b)),
                   "r"(NCONS / 32));
    if (V3_TMEM_RAW)
      for (int b = 0; b < NQ * NBUF; ++b)  // TFULL[b][q]: the copies of quarter q into TMEM completed
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(smem + CTRL_OFF + CTRL_TFULL + 8 * b)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid >= 256 && tid < 288) {  // consumer warp 0 allocates TMEM
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid >= 256)
    for (int i = tid - 256; i < P.log_j * NCONS; i += NCONS) masks_s[i] = P.masks[i];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  if (tid < 256) {
    // =========================== producers ===========================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(V3_PREG));
    const int g = tid >> 7;
    const int p = tid & 127;
    const int n = (int)P.n;
    Cursor cur;
    cursor_start(P, cur);
    int f = 0;
    if (g == 1) {
      cursor_next_active(P, cur);
      f = 1;
    }
    while (cur.it < P.n_items32) {
      const int b = f % NBUF;
      const uint32_t parity = (uint32_t)((f / NBUF) & 1);
      const int row0 = (cur.s * P.J32 + gray(cur.pp)) * B;
      const float* __restrict__ colp = col_ptr(P, cur.col);
      float* buf = reinterpret_cast<float*>(smem + (size_t)b * BUF_BYTES);
      if (p == 0) { V3_TRACE(g, f, 0) }
      const uint32_t fullb = smem_u32(smem + CTRL_OFF + 8 * NQ * b);
      mbar_wait(fullb, parity);  // first part (and the signs)
      if (p == 0) { V3_TRACE(g, f, 6) }
#ifndef V3_QSPREAD
#define V3_QSPREAD 1
#endif
      // quarters NREF..3 (data-less for a tail tile): with V3_QSPREAD, lane 0 of warp q of the
      // group issues quarter q, so no single warp carries all three issues into the group barrier
      if (SPLIT && (V3_QSPREAD ? ((p & 31) == 0 && (p >> 5) >= NREF) : p == 0)) {
        const bool full_tile = row0 + B <= n;
        uint64_t stream;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(stream));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t dst = smem_u32(buf);
        const int q0 = V3_QSPREAD ? (p >> 5) : NREF, q1 = V3_QSPREAD ? (p >> 5) + 1 : 4;
        for (int q = q0; q < q1; ++q) {
          if (full_tile) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(fullb + 8 * q) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], 16384, [%2], %3;" ::"r"(
                    dst + q * 16384),
                "l"(colp + row0 + q * 4096), "r"(fullb + 8 * q), "l"(stream)
                : "memory");
          } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fullb + 8 * q) : "memory");
          }
        }
      }
      if (DBG & 16) {  // knock-out: data movement only (no transform at all)
        for (int q = 1; q < NQ; ++q) mbar_wait(fullb + 8 * q, parity);
        bar_arrive(BAR_READY0 + b, 384);
        cursor_next_active(P, cur);
        cursor_next_active(P, cur);
        f += 2;
        continue;
      }
      const uint4 sg = *reinterpret_cast<const uint4*>(smem + SIGN_OFF + 2048 * b + 16 * p);
      float2 v[64];
#if V3_TMEM_RAW
      // ---- round 1 from TMEM: rows x = e2 + 4p + 512h' (e2 < 4, h' < 32) = register u = e2 + 4h',
      // pair m = u >> 1; quarter q = h' in [8q, 8q+8) = m in [16q, 16q+16) ----
      {
        const bool tail = row0 + B > n;
        const uint32_t tq = smem_u32(smem + CTRL_OFF + CTRL_TFULL + 8 * NQ * b);
        const uint32_t traw = *reinterpret_cast<const uint32_t*>(smem + CTRL_OFF + CTRL_TMEM) + (uint32_t)(128 * b) +
                              ((uint32_t)(32 * (p >> 5)) << 16);
        const float* __restrict__ colp = col_ptr(P, cur.col);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q > 0) mbar_wait(fullb + 8 * q, parity);
          if (p == 0) {
            if (!tail) {  // quarter q (h' = 8q .. 8q+7) -> TMEM columns 4h' .. 4h'+3 of buffer b
              const uint32_t t0 = *reinterpret_cast<const uint32_t*>(smem + CTRL_OFF + CTRL_TMEM) + (uint32_t)(128 * b);
              const uint32_t s0 = smem_u32(smem + (size_t)b * BUF_BYTES);
#pragma unroll
              for (int hh = 0; hh < 8; ++hh) {
                const int hp = 8 * q + hh;
                asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(t0 + 4 * hp), "l"(desc_nosw(s0 + 2048 * hp)));
              }
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tq + 8 * q)
                           : "memory");
            } else {
              asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tq + 8 * q) : "memory");  // keep phases
            }
          }
          uint32_t w[32];
          if (!tail) {
            mbar_wait(tq + 8 * q, parity);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
                  "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]),
                  "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]),
                  "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
                : "r"(traw + 32 * q));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          } else {  // ragged tail tile (no TMA data): rows >= n read as zero
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int row = row0 + 4 * p + 512 * (8 * q + (i >> 2)) + (i & 3);
              w[i] = __float_as_uint(row < n ? colp[row] : 0.f);
            }
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) v[16 * q + i] = make_float2(__uint_as_float(w[2 * i]), __uint_as_float(w[2 * i + 1]));
          const uint32_t wsg = q == 0 ? sg.x : q == 1 ? sg.y : q == 2 ? sg.z : sg.w;
#pragma unroll
          for (int h = 16 * q; h < 16 * q + 16; ++h) {
            const int bt = (h & 15) << 1;
            v[h].x = flipf(v[h].x, __funnelshift_l(wsg, wsg, 31 - bt) & 0x80000000u);
            v[h].y = flipf(v[h].y, __funnelshift_l(wsg, wsg, 30 - bt) & 0x80000000u);
          }
          fwht_quarter(v, q);  // row bits 0, 1 (pair, m bit 0) and 9..11 (m bits 1..3)
        }
      }
#else
      // ---- round 1: rows x = e + 2p + 256h; quarter q = h in [16q, 16q+16) ----
      if (row0 + B > n) {
        // tail tile (not copied by TMA): the group stages it in the raw layout itself,
        // zero-filling rows >= n, then reads it back like any other tile
        for (int q = 1; q < NQ; ++q) mbar_wait(fullb + 8 * q, parity);  // (data-less parts)
#pragma unroll 4
        for (int h = 0; h < 64; ++h) {
          const int row = row0 + 2 * p + 256 * h;
          *reinterpret_cast<float2*>(buf + 2 * p + 256 * h) =
              make_float2(row < n ? colp[row] : 0.f, row + 1 < n ? colp[row + 1] : 0.f);
        }
        bar_sync(BAR_GRP0 + g, 128);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (NQ == 4 && q > 0) mbar_wait(fullb + 8 * q, parity);
#pragma unroll
        for (int h = 16 * q; h < 16 * q + 16; ++h)
          v[h] = (DBG & 8) ? make_float2((float)h, (float)p) : *reinterpret_cast<const float2*>(buf + 2 * p + 256 * h);
        // D: sign of (h, e) = bit 2(h & 15) + e of word h >> 4 (= word q).  Funnel shifts
        // keep the bit moves on the ALU pipe (IMAD.SHL would take FMA slots).
        const uint32_t w = q == 0 ? sg.x : q == 1 ? sg.y : q == 2 ? sg.z : sg.w;
#pragma unroll
        for (int h = 16 * q; h < 16 * q + 16; ++h) {
          const int bt = (h & 15) << 1;
          v[h].x = flipf(v[h].x, __funnelshift_l(w, w, 31 - bt) & 0x80000000u);
          v[h].y = flipf(v[h].y, __funnelshift_l(w, w, 30 - bt) & 0x80000000u);
        }
        if (!(DBG & 4)) fwht_quarter(v, q);  // row bit 0 (pair) and bits 8..11 (h bits 0..3)
      }
#endif
      if (p == 0) { V3_TRACE(g, f, 1) }
#pragma unroll
      for (int m = 0; m < 64; ++m)
        if (!(m & 16) && !(DBG & 4)) bfly<16>(v, m);  // row bit 12
      if (p == 0) { V3_TRACE(g, f, 2) }
      bar_sync(BAR_GRP0 + g, 128);  // every raw row of the tile has been read
      // row bit 13, each result stored as soon as it is final: mid(x) = p + 130 (2h + e)
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        if (!(DBG & 4)) bfly<32>(v, m);
        if (!(DBG & 8)) {
          buf[p + ROWW * (2 * m)] = v[m].x;
          buf[p + ROWW * (2 * m + 1)] = v[m].y;
          buf[p + ROWW * (2 * (m + 32))] = v[m + 32].x;
          buf[p + ROWW * (2 * (m + 32) + 1)] = v[m + 32].y;
        }
      }
      if (p == 0) { V3_TRACE(g, f, 3) }
      bar_sync(BAR_GRP0 + g, 128);
      // ---- round 2: mid row p, cols 2m + e; quarter-ordered like round 1 ----
      float* rowp = buf + ROWW * p;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int m = 16 * q; m < 16 * q + 16; ++m)
          v[m] = (DBG & 8) ? make_float2(v[m].y, v[m].x) : *reinterpret_cast<const float2*>(rowp + 2 * m);
        if (!(DBG & 4)) fwht_quarter(v, q);  // row bit 1 (pair) and bits 2..5 (m bits 0..3)
      }
#pragma unroll
      for (int m = 0; m < 64; ++m)
        if (!(m & 16) && !(DBG & 4)) bfly<16>(v, m);  // row bit 6
      if (p == 0) { V3_TRACE(g, f, 4) }
#pragma unroll
      for (int m = 0; m < 32; ++m) {  // row bit 7, then z = H_B D x stored in place
        if (!(DBG & 4)) bfly<32>(v, m);
        if (!(DBG & 8)) {
          *reinterpret_cast<float2*>(rowp + 2 * m) = v[m];
          *reinterpret_cast<float2*>(rowp + 2 * (m + 32)) = v[m + 32];
        } else if (v[m].x == 1.2345f) {  // keep the values live
          rowp[m] = v[m + 32].y;
        }
      }
      bar_arrive(BAR_READY0 + b, 384);
      if (p == 0) { V3_TRACE(g, f, 5) }
      // next tile of this group: two active tiles ahead
      cursor_next_active(P, cur);
      cursor_next_active(P, cur);
      f += 2;
    }
  } else {
    // =========================== consumers ===========================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(V3_CREG));
    const int c = tid - 256;
    const int wc = c >> 5;
    const uint32_t tbase = *tmem_slot;
    const uint32_t taddr = tbase + ((uint32_t)(32 * (wc & 3)) << 16) + (uint32_t)(TRAW_COLS + (wc >> 2) * MW);
    // gather offsets of buffer b (META_PER_BUF: one copy per buffer, base added)
    auto tmeta = [&](int b) -> uint32_t { return META_PER_BUF ? taddr + (uint32_t)(2 * MW * b) : taddr; };
    // meta -> TMEM (once)
#pragma unroll
    for (int k = 0; k < MW; k += 4) {
      const uint4 m4 = __ldg(reinterpret_cast<const uint4*>(P.meta + (size_t)c * MW + k));
#pragma unroll
      for (int b = 0; b < (META_PER_BUF ? NBUF : 1); ++b) {
        const uint32_t o = META_PER_BUF ? (uint32_t)(b * BUF_BYTES) : 0u;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tmeta(b) + k), "r"(m4.x + o),
                     "r"(m4.y + o), "r"(m4.z + o), "r"(m4.w + o)
                     : "memory");
      }
    }
    // the TMEM stores must complete before the gather loads read the offsets back
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    if (c == 0) {  // slot b starts at active tile b; fill the ring, prefetch tiles 3..5
      Cursor c0;
      cursor_start(P, c0);
      for (int b = 0; b < NBUF; ++b) {
        slots[b].cur = c0;
        slots[b].count = 0;
        slots[b].f = b;
        cursor_next_active(P, c0);
      }
      for (int b = 0; b < NBUF; ++b) tma_issue<DBG, NREF>(P, slots[b], b, smem);
    }
    float acc[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) acc[q] = 0.f;
    // Gather offsets are the same for every tile, so their TMEM loads run one chunk ahead
    // across tile boundaries too (chunk 0 of the next tile lands in w[NCH & 1]; with an odd
    // chunk count it is moved to w[0] at the end of the tile).
    constexpr int CH = pick_ch(MW);
    constexpr int NCH = MW / CH;
    static_assert(MW % CH == 0 && CH % 2 == 0, "chunking");
    uint32_t w[2][CH];
    tmem_ld<CH>(taddr, w[0]);
    int f = 0;
    for (int it = blockIdx.x; it < P.n_items32; it += gridDim.x) {
      Cursor ci;
      ci.it = it;
      cursor_item(P, ci);
      const int col = ci.col, s = ci.s, cnt = ci.cnt, np = ci.np;
      for (int pp = 0; pp < np; ++pp) {
        uint2 mk = make_uint2(0u, 0u);
        if (pp) mk = masks_s[(__ffs(pp) - 1) * NCONS + c];
        if (gray(pp) < cnt) {
          const int b = f % NBUF;
          const float* buf = reinterpret_cast<const float*>(smem + (META_PER_BUF ? 0 : (size_t)b * BUF_BYTES));
          const uint32_t tb = tmeta(b), tnext = tmeta(b == NBUF - 1 ? 0 : b + 1);
          if (c == 0) { V3_TRACE(2, f, 0) }
          bar_sync(BAR_READY0 + b, 384);
#pragma unroll
          for (int k = 0; k < MW; k += CH) {
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            // next chunk in flight (after the last chunk: chunk 0 of the next tile)
            tmem_ld<CH>(k + CH < MW ? tb + k + CH : tnext, w[((k / CH) + 1) & 1]);
            if (k == 0 && c == 0) { V3_TRACE(2, f, 1) }
            const uint32_t* wk = w[(k / CH) & 1];
#pragma unroll
            for (int i = 0; i < CH; i += 2) {
              const int l = k + i;  // load slots l, l + 1
              // one byte offset per slot (no address arithmetic); a pair of accumulators is
              // updated by one FADD2
              const char* bb = reinterpret_cast<const char*>(buf);
              const float z0 = (DBG & 2) ? __uint_as_float(wk[i] & 0x3fffffffu) : *reinterpret_cast<const float*>(bb + wk[i]);
              const float z1 =
                  (DBG & 2) ? __uint_as_float(wk[i + 1] & 0x3fffffffu) : *reinterpret_cast<const float*>(bb + wk[i + 1]);
              // frame flip of accumulators q, q+1 (bits q, q+1 of the step's k_mid mask)
              auto flip2 = [&](int q) {
                const uint32_t mw = q < 32 ? mk.x : mk.y;
                return make_float2(flipf(acc[q], __funnelshift_l(mw, mw, 31 - (q & 31)) & 0x80000000u),
                                   flipf(acc[q + 1], __funnelshift_l(mw, mw, 30 - (q & 31)) & 0x80000000u));
              };
              if (l < PAIRS) {  // shared gathers: accumulators (2l, 2l+1) and (2l+2, 2l+3)
                const float2 s0 = __fadd2_rn(flip2(2 * l), make_float2(z0, z0));
                const float2 s1 = __fadd2_rn(flip2(2 * l + 2), make_float2(z1, z1));
                acc[2 * l] = s0.x;
                acc[2 * l + 1] = s0.y;
                acc[2 * l + 2] = s1.x;
                acc[2 * l + 3] = s1.y;
              } else {  // one accumulator per slot: PAIRS + l, PAIRS + l + 1
                const int q = PAIRS + l;
                const float2 sum = __fadd2_rn(flip2(q), make_float2(z0, z1));
                acc[q] = sum.x;
                acc[q + 1] = sum.y;
              }
            }
          }
          if constexpr (NCH & 1) {  // the next tile's chunk 0 was loaded into w[1]
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < CH; ++i) w[0][i] = w[1][i];
          }
          if (c == 0) { V3_TRACE(2, f, 2) }
          // the last consumer warp done with buffer b refills it (no consumer-wide barrier)
          __syncwarp();
          if ((c & 31) == 0) {
#if V3_EMPTY_MBAR
            // arrive on EMPTY[b]; the state returned is the barrier's state before this
            // arrival, so a pending count of 1 identifies the last warp (exactly one)
            uint64_t st;
            uint32_t pend;
            asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];"
                         : "=l"(st)
                         : "r"(smem_u32(smem + CTRL_OFF + CTRL_EMPTY + 8 * b))
                         : "memory");
            asm volatile("mbarrier.pending_count.b64 %0, %1;" : "=r"(pend) : "l"(st));
            if (pend == 1) {
              // acquire the other warps' arrivals (their reads of buffer b) before the
              // refill overwrites it: the phase is complete, so this wait returns at once
              mbar_wait(smem_u32(smem + CTRL_OFF + CTRL_EMPTY + 8 * b), (uint32_t)((f / NBUF) & 1));
              tma_issue<DBG, NREF>(P, slots[b], b, smem);
            }
#else
            const int done = atomicAdd(&slots[b].count, 1);
            if (done == NCONS / 32 - 1) {
              slots[b].count = 0;
              tma_issue<DBG, NREF>(P, slots[b], b, smem);
            }
#endif
          }
          if (c == 0) { V3_TRACE(2, f, 3) }
          ++f;
        } else {
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const uint32_t mw = q < 32 ? mk.x : mk.y;
            acc[q] = flipf(acc[q], __funnelshift_l(mw, mw, 31 - (q & 31)) & 0x80000000u);
          }
        }
      }
      // ---- slab epilogue: undo the frame sign of the last step; write the partial in slot
      // order (coalesced; k_reduce_v3 maps slots to output rows).  Writing rows t here
      // directly would scatter 32 lines per store instruction (measured 8 us per slab).
      if (c == 0 && f > 0) { V3_TRACE(2, f - 1, 4) }
      const uint32_t jlast = (uint32_t)gray(np - 1);
      // frame sign of slot q: popc(k_mid & jlast) odd = XOR of the k_mid bit masks of jlast's bits
      uint2 fm = make_uint2(0u, 0u);
      for (int l = 0; l < P.log_j; ++l)
        if ((jlast >> l) & 1u) {
          const uint2 m = masks_s[l * NCONS + c];
          fm.x ^= m.x;
          fm.y ^= m.y;
        }
      float* __restrict__ dst = P.partials + ((int64_t)(s - P.s_lo32) * P.total_cols + col) * (RPT * NCONS) + c;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const uint32_t mw = q < 32 ? fm.x : fm.y;
        dst[q * NCONS] = flipf(acc[q], __funnelshift_l(mw, mw, 31 - (q & 31)) & 0x80000000u);
        acc[q] = 0.f;
      }
      if (c == 0 && f > 0) { V3_TRACE(2, f - 1, 5) }
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");  // the last look-ahead load
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    bar_sync(BAR_CONS, NCONS);
    if (wc == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(TCOLS));
    }
  }
}

template <int RPT, int PAIRS, int DBG>
cudaError_t launch_dbg(const V3Params& vp, int grid, cudaStream_t stream) {
  static std::atomic<uint64_t> attr{0};
  const cudaError_t e = set_max_dyn_smem_once(k_sketch_tma<RPT, PAIRS, DBG>, SMEM_BYTES, attr);
  if (e != cudaSuccess) return e;
  k_sketch_tma<RPT, PAIRS, DBG><<<grid, NTHREADS, SMEM_BYTES, stream>>>(vp);
  return cudaGetLastError();
}
template <int RPT, int PAIRS>
cudaError_t launch_pairs(const V3Params& vp, int grid, cudaStream_t stream) {
  const int dbg = (vp.trace ? 1 : 0) | (vp.debug << 1);
#ifdef SRHT_WS_DEBUG
  if constexpr (RPT >= 32) {
    switch (dbg) {
      case 2: return launch_dbg<RPT, PAIRS, 2>(vp, grid, stream);
      case 4: return launch_dbg<RPT, PAIRS, 4>(vp, grid, stream);
      case 6: return launch_dbg<RPT, PAIRS, 6>(vp, grid, stream);
      case 8: return launch_dbg<RPT, PAIRS, 8>(vp, grid, stream);
      case 10: return launch_dbg<RPT, PAIRS, 10>(vp, grid, stream);
      case 12: return launch_dbg<RPT, PAIRS, 12>(vp, grid, stream);
      case 14: return launch_dbg<RPT, PAIRS, 14>(vp, grid, stream);
      case 16: return launch_dbg<RPT, PAIRS, 16>(vp, grid, stream);
      case 18: return launch_dbg<RPT, PAIRS, 18>(vp, grid, stream);
      default: break;
    }
  }
#endif
  return dbg & 1 ? launch_dbg<RPT, PAIRS, 1>(vp, grid, stream) : launch_dbg<RPT, PAIRS, 0>(vp, grid, stream);
}
template <int RPT>
cudaError_t launch_rpt(const V3Params& vp, int grid, cudaStream_t stream) {
  if constexpr (RPT >= 16)  // (RPT - PAIRS) % 4 == 0: 16-byte meta rows
    if (vp.pairs == RPT / 4) return launch_pairs<RPT, RPT / 4>(vp, grid, stream);
  if constexpr (RPT >= 32)
    if (vp.pairs == RPT / 8) return launch_pairs<RPT, RPT / 8>(vp, grid, stream);
  if (vp.pairs == 0) return launch_pairs<RPT, 0>(vp, grid, stream);
  return cudaErrorInvalidValue;
}

}  // namespace v3

int v3_mid(int x) { return v3::mid(x); }

namespace {
// Fixed-order slab reduction of kernel v3's slot-order partials: thread j = slot (q, c)
// = q * 256 + c finds its output row t in the plan's t table, then sums the slab
// partials exactly like k_reduce_slabs (FP64, slabs in order, slab sign of K[t]; DESIGN.md
// reading R10), so results do not depend on the slot layout.
__global__ void k_reduce_v3(const __grid_constant__ SketchParams P, const uint32_t* __restrict__ ttab, int rpt,
                            int slab_shift) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t col = blockIdx.y + (int64_t)blockIdx.z * 65535;
  const int64_t slots = (int64_t)rpt * 256;
  if (j >= slots || col >= P.total_cols) return;
  const int q = (int)(j >> 8), c = (int)(j & 255);
  const uint32_t t = (ttab[(size_t)c * (rpt / 2) + (q >> 1)] >> (16 * (q & 1))) & 0xffffu;
  if (t == 0xffffu) return;  // empty slot
  const uint32_t ks = (uint32_t)(P.K[t] >> slab_shift);
  double sum = 0.0;
  for (int64_t s = 0; s < P.S_act; ++s) {
    const uint32_t v = __float_as_uint(P.partials[(s * P.total_cols + col) * slots + j]);
    sum += (double)__uint_as_float(v ^ ((uint32_t)(__popc(ks & (uint32_t)(P.s_lo + s)) & 1) << 31));
  }
  if (P.part_out) {  // row shard: unscaled partial, summed across shards by the caller
    P.part_out[col * P.ldp + t] = sum;
    return;
  }
  const bool second = col >= P.ncols0;
  const ColSrc& cs = second ? P.src[1] : P.src[0];
  const int64_t lc = second ? col - P.ncols0 : col;
  const float y = (float)(sum * P.scale_f64);
  cs.out[lc * cs.ldo + t] = y;
  for (int k = 1; k < P.n_peers; ++k)  // fused gather: the same value into every peer's output (NVLink)
    P.peers[k][(P.peer_col0 + col) * P.peer_ld + t] = y;
}
}  // namespace

namespace {
// Copy of an r x cols block into peers[1..n) (the peer pointers ride in the parameter block).
__global__ void k_peer_copy(const float* __restrict__ src, int64_t src_ld, int64_t r, int64_t cols, int n_peers,
                            int64_t col0, int64_t peer_ld, const __grid_constant__ SketchParams pp) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    if (t >= r) continue;
    const float v = src[j * src_ld + t];
    for (int k = 1; k < n_peers; ++k) pp.peers[k][(col0 + j) * peer_ld + t] = v;
  }
}

// The same reduction with one CTA per column: slot sums (coalesced partial reads, slabs in
// order) are placed at their output rows in shared memory, then written out coalesced --
// k_reduce_v3's stores to rows t scatter 4-byte writes over the column (config 4: step 0.490 ->
// 0.482 ms).  Identical arithmetic, so identical results.
template <bool PART>
__global__ void __launch_bounds__(512) k_reduce_v3_col(const __grid_constant__ SketchParams P,
                                                      const uint32_t* __restrict__ ttab, int rpt, int slab_shift) {
  extern __shared__ __align__(16) unsigned char red_smem[];
  const int64_t col = blockIdx.x + (int64_t)blockIdx.y * 65535;
  if (col >= P.total_cols) return;
  const int64_t slots = (int64_t)rpt * 256;
  for (int64_t j = threadIdx.x; j < slots; j += blockDim.x) {
    const int q = (int)(j >> 8), c = (int)(j & 255);
    const uint32_t t = (ttab[(size_t)c * (rpt / 2) + (q >> 1)] >> (16 * (q & 1))) & 0xffffu;
    if (t == 0xffffu) continue;  // empty slot
    const uint32_t ks = (uint32_t)(P.K[t] >> slab_shift);
    double sum = 0.0;
    for (int64_t s = 0; s < P.S_act; ++s) {
      const uint32_t v = __float_as_uint(P.partials[(s * P.total_cols + col) * slots + j]);
      sum += (double)__uint_as_float(v ^ ((uint32_t)(__popc(ks & (uint32_t)(P.s_lo + s)) & 1) << 31));
    }
    if (PART) reinterpret_cast<double*>(red_smem)[t] = sum;
    else reinterpret_cast<float*>(red_smem)[t] = (float)(sum * P.scale_f64);
  }
  __syncthreads();
  if (PART) {
    for (int64_t t = threadIdx.x; t < P.r; t += blockDim.x) P.part_out[col * P.ldp + t] = reinterpret_cast<double*>(red_smem)[t];
  } else {
    const bool second = col >= P.ncols0;
    const ColSrc& cs = second ? P.src[1] : P.src[0];
    const int64_t lc = second ? col - P.ncols0 : col;
    float* __restrict__ o = cs.out + lc * cs.ldo;
    for (int64_t t = threadIdx.x; t < P.r; t += blockDim.x) o[t] = reinterpret_cast<float*>(red_smem)[t];
    for (int k = 1; k < P.n_peers; ++k) {  // fused gather: coalesced stores into every peer's output
      float* __restrict__ po = P.peers[k] + (P.peer_col0 + col) * P.peer_ld;
      for (int64_t t = threadIdx.x; t < P.r; t += blockDim.x) po[t] = reinterpret_cast<float*>(red_smem)[t];
    }
  }
}
}  // namespace

cudaError_t launch_peer_copy(const float* src, int64_t src_ld, int64_t r, int64_t cols, float* const* peers,
                             int n_peers, int64_t col0, int64_t peer_ld, cudaStream_t stream) {
  if (n_peers <= 1 || r <= 0 || cols <= 0) return cudaSuccess;
  SketchParams pp;
  memset(&pp, 0, sizeof(pp));
  for (int k = 0; k < n_peers && k < SRHT_MAX_PEERS; ++k) pp.peers[k] = peers[k];
  const dim3 grid((unsigned)((r + 255) / 256), (unsigned)(cols < 65535 ? cols : 65535));
  k_peer_copy<<<grid, 256, 0, stream>>>(src, src_ld, r, cols, n_peers, col0, peer_ld, pp);
  return cudaGetLastError();
}

cudaError_t launch_reduce_v3(const SketchParams& sp, const uint32_t* ttab, int rpt, int slab_shift,
                             cudaStream_t stream) {
#ifndef V3_REDUCE_COL
#define V3_REDUCE_COL 1
#endif
  const int64_t zc = (sp.total_cols + 65534) / 65535;
  if (V3_REDUCE_COL && sp.S_act <= 4) {  // few slabs (config 4: one); with many (config 5: 64) one CTA per
                                         // column reads too little in parallel (8.47 vs 8.27 ms per step)
    const dim3 grid((unsigned)(sp.total_cols < 65535 ? sp.total_cols : 65535), (unsigned)zc);
    const bool part = sp.part_out != nullptr;
    const size_t smem = (size_t)sp.r * (part ? sizeof(double) : sizeof(float));
    static std::atomic<uint64_t> attr_f{0}, attr_d{0};
    cudaError_t e = part ? set_max_dyn_smem_once(k_reduce_v3_col<true>, (int)(16384 * sizeof(double)), attr_d)
                         : set_max_dyn_smem_once(k_reduce_v3_col<false>, (int)(16384 * sizeof(float)), attr_f);
    if (e != cudaSuccess) return e;
    if (part) k_reduce_v3_col<true><<<grid, 512, smem, stream>>>(sp, ttab, rpt, slab_shift);
    else k_reduce_v3_col<false><<<grid, 512, smem, stream>>>(sp, ttab, rpt, slab_shift);
    return cudaGetLastError();
  }
  const dim3 grid((unsigned)rpt, (unsigned)(sp.total_cols < 65535 ? sp.total_cols : 65535), (unsigned)zc);
  k_reduce_v3<<<grid, 256, 0, stream>>>(sp, ttab, rpt, slab_shift);
  return cudaGetLastError();
}

cudaError_t launch_sketch_tma(const srht_plan* P, const V3Params& vp, cudaStream_t stream) {
  if (vp.total_cols <= 0) return cudaSuccess;
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = vp.n_items32 < sms ? vp.n_items32 : sms;
  switch (P->rpt2) {
    case 8: return v3::launch_rpt<8>(vp, grid, stream);
    case 16: return v3::launch_rpt<16>(vp, grid, stream);
    case 32: return v3::launch_rpt<32>(vp, grid, stream);
    case 64: return v3::launch_rpt<64>(vp, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace srht
