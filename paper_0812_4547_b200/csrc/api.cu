// C ABI (include/srht.h): validation, plan geometry, dispatch.
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

namespace {

// NVTX range around an entry point (visible in nsys / ncu --nvtx timelines; no cost without a tool)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int ceil_log2(int64_t x) {
  int l = 0;
  while ((int64_t(1) << l) < x) ++l;
  return l;
}

bool valid_matrix(const srht_matrix* M) {
  if (!M) return false;
  if (M->rows < 0 || M->cols < 0) return false;
  if (M->fmt == SRHT_DENSE) {
    if (M->cols > 0 && M->rows > 0 && !M->vals) return false;
    if (M->ld < M->rows || M->ld < 1) return false;
    return true;
  }
  if (M->fmt == SRHT_CSC) {
    if (!M->colptr) return false;
    if (M->nnz < 0 || M->nnz > 0x7fffffffLL) return false;
    if (M->nnz > 0 && (!M->rowidx || !M->vals)) return false;
    if (M->rows > 0x7fffffffLL) return false;
    return true;
  }
  return false;
}

srht::ColSrc make_src(const srht_matrix* M, float* out, int64_t ldo) {
  srht::ColSrc c;
  std::memset(&c, 0, sizeof(c));
  c.fmt = M->fmt;
  c.vals = M->vals;
  c.ld = M->ld;
  c.colptr = M->colptr;
  c.rowidx = M->rowidx;
  c.ncols = M->cols;
  c.out = out;
  c.ldo = ldo;
  c.vec = (M->fmt == SRHT_DENSE) && (M->ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(M->vals) & 15) == 0);
  return c;
}

// Workspace of srht_sketch* (and of srht_sketch_rows_partial when `shards`, which always goes
// through the slab partials): per-slab partial sums of the widest slab geometry in use.
size_t partial_bytes(const srht_plan* P, int64_t ncols, bool shards = false) {
  if (ncols <= 0) return 0;
  const int64_t min_s = shards ? 1 : 2;
  if (P->flags & SRHT_PLAN_ACCUM_FP64) {  // FP64 partials of the v1 slab geometry
    size_t b = P->S_act < min_s ? 0 : (size_t)P->S_act * (size_t)ncols * (size_t)P->r * sizeof(double);
    if (P->v64_ok) {  // FP64 TMA kernel: slot-order partials of every slab, even a single one
      const size_t b64 = (size_t)P->S_act64 * P->G64 * (size_t)ncols * (size_t)P->rpt64 * 256 * sizeof(double);
      if (b64 > b) b = b64;
    }
    return (b + 255) & ~size_t(255);
  }
  int64_t S = P->S_act;
  if (P->ws_ok && P->S_act2 > S) S = P->S_act2;
  size_t b = S < min_s ? 0 : (size_t)S * (size_t)ncols * (size_t)P->r * sizeof(float);
  if (P->ws_ok && P->v3_ok) {  // kernel v3: slot-order partials of every slab, even a single one
    const size_t b3 = (size_t)P->S_act2 * (size_t)ncols * (size_t)P->rpt2 * 256 * sizeof(float);
    if (b3 > b) b = b3;
  }
  return (b + 255) & ~size_t(255);
}

// Consumer slot layout (host side, once per plan) shared by kernels v2 and v3.
// Sample t goes to slot (q, c): consumer thread c = 32*w + lane handles it as its
// q-th accumulator.  Rows (q, w) of 32 lanes take at most one sample per
// shared-memory bank of the gather address where possible, so the gather LDS is
// conflict-free.  Samples, sorted by bank, are dealt round-robin over the rows:
// sample i of the bank-sorted order goes to row i mod rows, so a bank with c samples
// lands in min(c, rows) distinct rows (<= ceil(max_c / rows) per row).
// Returns slot_t[q*256 + 32*w + lane] = t or -1.
std::vector<int32_t> deal_slots(const std::vector<int32_t>& K, int rpt, int (*addr)(int)) {
  const int rows = rpt * 8;
  const int slots = rpt * 256;
  std::vector<std::vector<int32_t>> bucket(32);
  for (size_t t = 0; t < K.size(); ++t) bucket[addr(K[t] & ((1 << 14) - 1)) & 31].push_back((int32_t)t);
  std::vector<int32_t> row_t(slots, -1);
  std::vector<int> fill(rows, 0);
  int64_t i = 0;
  for (int b = 0; b < 32; ++b)
    for (int32_t t : bucket[b]) {
      const int row = (int)(i % rows);
      row_t[row * 32 + fill[row]++] = t;
      ++i;
    }
  std::vector<int32_t> slot_t(slots, -1);  // row = q*8 + w, lane -> index q*256 + 32*w + lane
  for (int row = 0; row < rows; ++row)
    for (int lane = 0; lane < 32; ++lane) slot_t[(row / 8) * 256 + (row % 8) * 32 + lane] = row_t[row * 32 + lane];
  return slot_t;
}

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(dst, v.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// Kernel v2: meta = byte offset of phys(k_lo) | reversed k_mid bits at the top.
cudaError_t build_ws_layout(srht_plan* P, const std::vector<int32_t>& K) {
  const int slots = P->rpt2 * 256;
  const std::vector<int32_t> slot_t = deal_slots(K, P->rpt2, srht::ws_phys);
  std::vector<uint32_t> meta(slots, 0u);
  for (int idx = 0; idx < slots; ++idx) {
    const int32_t t = slot_t[idx];
    if (t < 0) continue;
    const int k = K[t];
    const uint32_t off = (uint32_t)srht::ws_phys(k & ((1 << 14) - 1)) * 4u;
    const uint32_t kmid = (uint32_t)(k >> 14) & (uint32_t)(P->J2 - 1);
    uint32_t rev = 0;
    for (int i = 0; i < P->log_j2; ++i) rev |= ((kmid >> i) & 1u) << (31 - i);
    meta[idx] = off | rev;
  }
  cudaError_t e = upload(&P->d_meta, meta);
  if (e == cudaSuccess) e = upload(&P->d_perm, slot_t);
  return e;
}

// Kernel v3: per consumer thread c, rpt2 words: the byte offset of slot q's z value in
// the tile buffer (mid layout); ttab: per thread rpt2/2 words holding the output rows t
// of slots 2i, 2i+1 (bits 0..15, 16..31; 0xffff = empty slot); masks[sh][c] bit q = bit
// sh of k_mid of slot (q, c).
//
// Shared gathers (kernel v3): samples whose k_lo coincide read the same z word.  Thread c's
// first P3 load slots each feed the accumulator pair (2l, 2l+1) -- two samples with one k_lo,
// one LDS and one FADD2 with a broadcast operand -- and its remaining rpt - 2 P3 accumulators
// take one load slot each, so a thread issues rpt - P3 gathers per tile instead of rpt.
// P3 = rpt/4 when the plan has at least 64 rpt same-k_lo pairs (config 5: 4653 pairs for
// 4096 needed), else rpt/8, else 0.  Pair rows and single rows are each dealt by bank as in
// deal_slots.  Returns the accumulator -> sample map acc_t[q*256 + c] and meta[c][l].
int choose_pairs3(const std::vector<int32_t>& K, int rpt) {
  if (rpt < 16) return 0;
  std::vector<int> mult(1 << 14, 0);
  for (int32_t k : K) ++mult[k & ((1 << 14) - 1)];
  int64_t avail = 0;
  for (int m : mult) avail += m / 2;
  if (avail >= (int64_t)256 * (rpt / 4)) return rpt / 4;
  if (rpt >= 32 && avail >= (int64_t)256 * (rpt / 8)) return rpt / 8;  // (kernel instantiations)
  return 0;
}

// Gather-bank dealing.  A warp-wide gather (load slot l of warp w, 32 lanes) costs one shared-memory
// wavefront per distinct z word in its most used bank; lanes that read the same word are served by
// one broadcast.  So the samples of one z word that a row takes form a unit (one word, k lanes), and a
// row costs one wavefront when its units come from distinct banks.  (1) Pair selection: 256 P3 pairs
// (two samples of one k_lo per load) are taken one at a time from the bank whose single units most
// exceed its share of the single rows relative to its pair units' share of the pair rows, preferring
// words with exactly two samples left (the pair removes a single unit).  (2) Rows are filled one at a
// time with at most one unit per bank, banks with the most units left first (the largest unit that
// fits; a unit larger than the room left is split), then any room left from the bank with the most
// lanes left.  Config 5's plan: 384 wavefronts per tile, the one-per-instruction floor (round-robin
// dealing by bank: 511); config 4: 233 (floor 224; was 346).  Empty lanes read their row's first word.
namespace {
struct GUnit {
  int lo, lanes;
};
// rows x 32 lanes -> k_lo of the lane's word (-1: empty)
void deal_rows_by_bank(std::vector<std::vector<GUnit>>& units, int nrows, std::vector<int>& lane_lo) {
  lane_lo.assign((size_t)nrows * 32, -1);
  auto by_lanes = [](const GUnit& a, const GUnit& b) { return a.lanes > b.lanes; };
  for (auto& u : units) std::stable_sort(u.begin(), u.end(), by_lanes);
  int order[32];
  int64_t rem = 0;
  for (const auto& u : units)
    for (const GUnit& g : u) rem += g.lanes;
  for (int row = 0; row < nrows; ++row) {
    // lanes for this row: an even share of what is left (32 when every slot is used)
    const int64_t share = (rem + (nrows - row) - 1) / (nrows - row);
    int cap = share < 32 ? (int)share : 32, fill = 0;
    rem -= cap;
    auto put = [&](int lo, int k) {
      for (int i = 0; i < k; ++i) lane_lo[(size_t)row * 32 + fill++] = lo;
      cap -= k;
    };
    for (int b = 0; b < 32; ++b) order[b] = b;
    std::stable_sort(order, order + 32, [&](int a, int b) { return units[a].size() > units[b].size(); });
    for (int oi = 0; oi < 32 && cap > 0; ++oi) {
      std::vector<GUnit>& u = units[order[oi]];
      if (u.empty()) continue;
      size_t i = 0;
      while (i < u.size() && u[i].lanes > cap) ++i;
      if (i == u.size()) {  // split the largest unit
        GUnit g = u[0];
        g.lanes -= cap;
        put(g.lo, cap);
        u.erase(u.begin());
        u.insert(std::upper_bound(u.begin(), u.end(), g, by_lanes), g);
      } else {
        put(u[i].lo, u[i].lanes);
        u.erase(u.begin() + (std::ptrdiff_t)i);
      }
    }
    while (cap > 0) {  // room left: the bank with the most lanes left (a second word of that bank)
      int best = -1, bl = 0;
      for (int b = 0; b < 32; ++b) {
        int l = 0;
        for (const GUnit& g : units[b]) l += g.lanes;
        if (l > bl) {
          bl = l;
          best = b;
        }
      }
      if (best < 0) {
        rem += cap;
        break;
      }
      GUnit& g = units[best][0];
      const int k = g.lanes < cap ? g.lanes : cap;
      put(g.lo, k);
      g.lanes -= k;
      if (g.lanes == 0) units[best].erase(units[best].begin());
    }
  }
}
}  // namespace

void deal_v3_pairs(const std::vector<int32_t>& K, int rpt, int P3, std::vector<int32_t>& acc_t,
                   std::vector<uint32_t>& meta_off) {
  constexpr int LO = 1 << 14;
  const int L = rpt - P3;
  const int prows = P3 * 8, srows = (L - P3) * 8;
  acc_t.assign((size_t)rpt * 256, -1);
  meta_off.assign((size_t)256 * L, 0u);
  std::vector<std::vector<int32_t>> by_lo(LO);
  for (size_t t = 0; t < K.size(); ++t) by_lo[K[t] & (LO - 1)].push_back((int32_t)t);
  auto bank = [](int lo) { return srht::v3_mid(lo) & 31; };
  // (1) pair selection
  std::vector<int> left(LO), npair(LO, 0);
  std::vector<std::vector<int>> cand(32);  // words with >= 2 samples
  double su[32] = {}, pu[32] = {};
  for (int lo = 0; lo < LO; ++lo) {
    left[lo] = (int)by_lo[lo].size();
    if (left[lo] > 0) su[bank(lo)] += 1.0;
    if (left[lo] >= 2) cand[bank(lo)].push_back(lo);
  }
  for (int64_t k = 0; k < (int64_t)256 * P3; ++k) {
    int bb = -1, blo = -1;
    double bs = 0.0;
    for (int b = 0; b < 32; ++b) {
      int w = -1;
      for (int lo : cand[b])  // a word with exactly two left, else the one with the most left
        if (left[lo] >= 2 && (w < 0 || (left[lo] == 2) > (left[w] == 2) ||
                              ((left[lo] == 2) == (left[w] == 2) && left[lo] > left[w])))
          w = lo;
      if (w < 0) continue;
      const double sc = su[b] / (srows > 0 ? srows : 1) - pu[b] / prows + (left[w] == 2 ? 1e-3 : 0.0);
      if (bb < 0 || sc > bs) {
        bb = b;
        blo = w;
        bs = sc;
      }
    }
    if (bb < 0) break;  // (choose_pairs3 guarantees enough pairs)
    if (left[blo] == 2) su[bb] -= 1.0;
    if (npair[blo] == 0) pu[bb] += 1.0;
    ++npair[blo];
    left[blo] -= 2;
  }
  // (2) rows
  std::vector<std::vector<GUnit>> pun(32), sun(32);
  for (int lo = 0; lo < LO; ++lo) {
    if (npair[lo] > 0) pun[bank(lo)].push_back({lo, npair[lo]});
    if (left[lo] > 0) sun[bank(lo)].push_back({lo, left[lo]});
  }
  std::vector<int> cursor(LO, 0);
  std::vector<int> lane_lo;
  if (prows > 0) {
    deal_rows_by_bank(pun, prows, lane_lo);
    for (int row = 0; row < prows; ++row) {
      const int l = row / 8, w = row % 8;
      for (int lane = 0; lane < 32; ++lane) {
        const int c = w * 32 + lane;
        const int lo = lane_lo[(size_t)row * 32 + lane];
        const int rl = lo >= 0 ? lo : lane_lo[(size_t)row * 32];
        if (rl >= 0) meta_off[(size_t)c * L + l] = (uint32_t)srht::v3_mid(rl) * 4u;
        if (lo < 0) continue;
        acc_t[(size_t)(2 * l) * 256 + c] = by_lo[lo][cursor[lo]++];
        acc_t[(size_t)(2 * l + 1) * 256 + c] = by_lo[lo][cursor[lo]++];
      }
    }
  }
  if (srows > 0) {
    deal_rows_by_bank(sun, srows, lane_lo);
    for (int row = 0; row < srows; ++row) {
      const int l = P3 + row / 8, w = row % 8;
      for (int lane = 0; lane < 32; ++lane) {
        const int c = w * 32 + lane;
        const int lo = lane_lo[(size_t)row * 32 + lane];
        const int rl = lo >= 0 ? lo : lane_lo[(size_t)row * 32];
        if (rl >= 0) meta_off[(size_t)c * L + l] = (uint32_t)srht::v3_mid(rl) * 4u;
        if (lo < 0) continue;
        acc_t[(size_t)(P3 + l) * 256 + c] = by_lo[lo][cursor[lo]++];  // accumulator 2 P3 + (l - P3)
      }
    }
  }
}

// Whole-column kernel gather order for one problem (r <= 1024 kept rows K, N = 2^13): out[COL_SLOTS]
// = k | t << 16 (0xffffffff: empty) in 40 warp-wide steps of 32 slots; each kept row goes to the
// step with the fewest kept rows of its gather bank (lo + lo / 32) mod 32 so far, then the fewest
// of its staging bank t mod 32, then the fewest entries.
void deal_col_slots(const int32_t* K, int r, uint32_t* out) {
  constexpr int ROWS = srht::COL_SLOTS / 32;
  std::vector<std::pair<int, int32_t>> order(r);
  for (int t = 0; t < r; ++t) {
    const int lo = K[t] & 1023;
    order[t] = {(lo + (lo >> 5)) & 31, t};
  }
  std::sort(order.begin(), order.end());
  int cnt_a[ROWS][32] = {}, cnt_b[ROWS][32] = {}, fill[ROWS] = {};
  for (int i = 0; i < srht::COL_SLOTS; ++i) out[i] = 0xffffffffu;
  for (int m = 0; m < r; ++m) {
    const int a = order[m].first, t = order[m].second, b = t & 31;
    int best = -1;
    long long bs = 0;
    for (int row = 0; row < ROWS; ++row) {
      if (fill[row] >= 32) continue;
      const long long sc = (long long)cnt_a[row][a] * 1000000 + cnt_b[row][b] * 1000 + fill[row];
      if (best < 0 || sc < bs) {
        best = row;
        bs = sc;
      }
    }
    ++cnt_a[best][a];
    ++cnt_b[best][b];
    out[(size_t)best * 32 + fill[best]++] = (uint32_t)K[t] | ((uint32_t)t << 16);
  }
}

cudaError_t build_v3_layout(srht_plan* P, const std::vector<int32_t>& K) {
  const int rpt = P->rpt2, mw = rpt / 2;
#ifndef V3_PAIRS
#define V3_PAIRS 1
#endif
  P->pairs3 = V3_PAIRS ? choose_pairs3(K, rpt) : 0;
  std::vector<int32_t> slot_t;
  std::vector<uint32_t> meta;
  deal_v3_pairs(K, rpt, P->pairs3, slot_t, meta);
  std::vector<uint32_t> ttab((size_t)256 * mw, 0xffffffffu);
  std::vector<uint2> masks((size_t)(P->log_j2 > 0 ? P->log_j2 : 1) * 256, make_uint2(0u, 0u));
  for (int q = 0; q < rpt; ++q)
    for (int c = 0; c < 256; ++c) {
      const int32_t t = slot_t[q * 256 + c];
      if (t < 0) continue;
      const int k = K[t];
      const uint32_t kmid = (uint32_t)(k >> 14) & (uint32_t)(P->J2 - 1);
      uint32_t& tw = ttab[(size_t)c * mw + q / 2];
      tw = (tw & ~(0xffffu << (16 * (q & 1)))) | ((uint32_t)t << (16 * (q & 1)));
      for (int sh = 0; sh < P->log_j2; ++sh)
        if ((kmid >> sh) & 1u) {
          uint2& m = masks[(size_t)sh * 256 + c];
          if (q < 32) m.x |= 1u << q; else m.y |= 1u << (q - 32);
        }
    }
  cudaError_t e = upload(&P->d_meta3, meta);
  if (e == cudaSuccess) e = upload(&P->d_ttab3, ttab);
  if (e == cudaSuccess) e = upload(&P->d_masks3, masks);
  return e;
}

// FP64 TMA kernel: sample group gi takes samples t in [gi * slots, (gi + 1) * slots); inside a
// group, slot (q, c) belongs to half-warp row q * 16 + c / 16, and the group's samples, sorted by
// the 8-byte bank granule of their z value (mid(k_lo) mod 16), are dealt round-robin over the
// rows, so the 16 lanes of a half-warp gather from distinct granules where the counts allow.
cudaError_t build_v64_layout(srht_plan* P, const std::vector<int32_t>& K) {
  const int rpt = P->rpt64, G = P->G64, slots = rpt * 256, rows = rpt * 16;
  const int lj = P->log_j64 > 0 ? P->log_j64 : 1;
  std::vector<uint32_t> meta((size_t)G * 256 * rpt, 0u);
  std::vector<int32_t> ttab((size_t)G * 256 * rpt, -1);
  std::vector<uint32_t> masks((size_t)G * lj * 256, 0u);
  for (int gi = 0; gi < G; ++gi) {
    std::vector<std::vector<int32_t>> bucket(16);
    for (int64_t t = (int64_t)gi * slots; t < P->r && t < (int64_t)(gi + 1) * slots; ++t)
      bucket[srht::v64_mid(K[t] & ((1 << V64_LOG_B) - 1)) & 15].push_back((int32_t)t);
    std::vector<int> fill(rows, 0);
    int64_t i = 0;
    for (int bk = 0; bk < 16; ++bk)
      for (int32_t t : bucket[bk]) {
        const int row = (int)(i % rows);
        const int q = row / 16, c = 16 * (row % 16) + fill[row]++;
        ++i;
        const int k = K[t];
        const size_t idx = ((size_t)gi * 256 + c) * rpt + q;
        meta[idx] = 8u * (uint32_t)srht::v64_mid(k & ((1 << V64_LOG_B) - 1));
        ttab[idx] = t;
        const uint32_t kmid = (uint32_t)(k >> V64_LOG_B) & (uint32_t)(P->J64 - 1);
        for (int l = 0; l < P->log_j64; ++l)
          if ((kmid >> l) & 1u) masks[((size_t)gi * lj + l) * 256 + c] |= 1u << q;
      }
  }
  cudaError_t e = upload(&P->d_meta64, meta);
  if (e == cudaSuccess) e = upload(&P->d_ttab64, ttab);
  if (e == cudaSuccess) e = upload(&P->d_masks64, masks);
  return e;
}

srht::SketchParams base_params(const srht_plan* P) {
  srht::SketchParams sp;
  std::memset(&sp, 0, sizeof(sp));
  sp.signs = reinterpret_cast<const uint32_t*>(P->d_signs);
  sp.words32 = P->words64 * 2;
  sp.K = P->d_K;
  sp.colk = P->d_colk;
  sp.r = P->r;
  sp.n = P->n;
  sp.J = P->J;
  sp.log_j = P->log_j;
  sp.n_sub = P->n_sub;
  sp.S_act = P->S_act;
  sp.groups = P->groups;
  sp.scale = P->scale;
  sp.scale_f64 = 1.0 / std::sqrt((double)P->r_target);
  return sp;
}

// Global slab range [lo, hi) of slabs of `slab_rows` rows that covers rows [row0, row0 + nrows).
void slab_range(int64_t row0, int64_t nrows, int64_t slab_rows, int64_t S_total, int64_t& lo, int64_t& cnt) {
  lo = row0 / slab_rows;
  int64_t hi = (row0 + nrows + slab_rows - 1) / slab_rows;
  if (hi > S_total) hi = S_total;
  cnt = hi - lo;
}

// Launch the sketch of sp's columns over rows [row0, row0 + nrows) (whole columns: 0, n).
// With sp.part_out set, the unscaled FP64 partial sums of those rows go to part_out
// (row shards); otherwise r^{-1/2} * sum goes to the sources' outputs.
srht_status run(const srht_plan* P, srht::SketchParams& sp, void* ws, size_t ws_bytes, void* stream,
                int64_t row0 = 0, int64_t nrows = -1) {
  if (sp.total_cols == 0) return SRHT_OK;
  if (nrows < 0) nrows = P->n;
  const size_t need = partial_bytes(P, sp.total_cols, sp.part_out != nullptr);
  if (need) {
    if (!ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255)) return SRHT_EINVAL;
    sp.partials = static_cast<float*>(ws);
  }
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return SRHT_ECUDA;
  if (dev != P->device) return SRHT_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool part = sp.part_out != nullptr;
  // kernel v1 / FP64 geometry: slabs of B * J rows
  slab_range(row0, nrows, P->B * P->J, P->S_act, sp.s_lo, sp.S_act);
  if (P->flags & SRHT_PLAN_ACCUM_FP64) {
    sp.partials64 = static_cast<double*>(ws);
    sp.partials = nullptr;
    const bool batched1 = sp.cols_per_problem != INT64_MAX;
    bool fast = P->v64_ok && !batched1;
    const int nsrc = sp.total_cols > sp.ncols0 ? 2 : 1;
    for (int i = 0; i < nsrc; ++i)
      if (sp.src[i].ncols > 0 && !(sp.src[i].fmt == SRHT_DENSE && sp.src[i].vec)) fast = false;
    int64_t s_lo64 = 0, S64 = 0;
    if (fast) {
      slab_range(row0, nrows, (int64_t(1) << V64_LOG_B) * P->J64, P->S_act64, s_lo64, S64);
      fast = sp.total_cols * S64 * P->G64 < (int64_t(1) << 31);
    }
    if (!fast) return srht::launch_sketch_f64(P, sp, st) == cudaSuccess ? SRHT_OK : SRHT_ECUDA;
    srht::V64Params vp;
    std::memset(&vp, 0, sizeof(vp));
    vp.src[0] = sp.src[0];
    vp.src[1] = nsrc == 2 ? sp.src[1] : srht::ColSrc();
    vp.ncols0 = sp.ncols0;
    vp.total_cols = sp.total_cols;
    vp.signs = P->d_signs64;
    vp.meta = P->d_meta64;
    vp.masks = P->d_masks64;
    vp.log_j = P->log_j64;
    vp.G = P->G64;
    vp.n = P->n;
    vp.cols32 = (int)sp.total_cols;
    vp.S_act32 = (int)S64;
    vp.s_lo32 = (int)s_lo64;
    vp.J32 = (int)P->J64;
    vp.n_sub32 = (int)P->n_sub64;
    vp.n_items32 = (int)(sp.total_cols * S64 * P->G64);
    vp.partials = sp.partials64;
    const int slot = (srht::g_prof.on && srht::g_prof.used < srht::g_prof.capacity) ? srht::g_prof.used++ : -1;
    if (slot >= 0) cudaEventRecord(srht::g_prof.ev[2 * slot], st);
    cudaError_t e = srht::launch_sketch_tma64(P, vp, st);
    if (slot >= 0) cudaEventRecord(srht::g_prof.ev[2 * slot + 1], st);
    srht::g_last_kernel = 6;
    if (e != cudaSuccess) return SRHT_ECUDA;
    srht::SketchParams rp = sp;
    rp.S_act = S64;
    rp.s_lo = s_lo64;
    return srht::launch_reduce64(rp, P->d_ttab64, P->rpt64, P->G64, V64_LOG_B + P->log_j64, st) == cudaSuccess
               ? SRHT_OK
               : SRHT_ECUDA;
  }
  const bool batched = sp.cols_per_problem != INT64_MAX;
  if (P->ws_ok && !batched) {
    // dense sources -> kernel v3 (or v2 for unaligned columns); any CSC source -> one
    // kernel-v1 launch for every column (e.g. CSC A + dense b)
    srht::ColSrc dense[2];
    int nd = 0, ncsc = 0;
    const int nsrc = sp.total_cols > sp.ncols0 ? 2 : 1;
    for (int i = 0; i < nsrc; ++i) {
      if (sp.src[i].ncols <= 0) continue;
      if (sp.src[i].fmt == SRHT_DENSE) dense[nd++] = sp.src[i]; else ++ncsc;
    }
    if (ncsc || !nd) return srht::launch_sketch(P, sp, st) == cudaSuccess ? SRHT_OK : SRHT_ECUDA;
    // kernel v2/v3 geometry: slabs of 2^14 * J2 rows
    int64_t s_lo2, S2;
    slab_range(row0, nrows, (int64_t(1) << 14) * P->J2, P->S_act2, s_lo2, S2);
    const int direct = (P->S_act2 == 1 && !part) ? 1 : 0;
    srht::SketchParams rp = sp;  // the fixed-order slab reduction of this geometry
    rp.src[0] = dense[0];
    rp.src[1] = nd == 2 ? dense[1] : srht::ColSrc();
    rp.ncols0 = dense[0].ncols;
    rp.total_cols = dense[0].ncols + (nd == 2 ? dense[1].ncols : 0);
    rp.S_act = S2;
    rp.s_lo = s_lo2;
    bool v3 = P->v3_ok && srht::g_kernel_force != 2 && rp.total_cols * S2 < (int64_t(1) << 31);
    for (int i = 0; i < nd; ++i) v3 = v3 && dense[i].vec;
    const int slot = (srht::g_prof.on && srht::g_prof.used < srht::g_prof.capacity) ? srht::g_prof.used++ : -1;
    if (slot >= 0) cudaEventRecord(srht::g_prof.ev[2 * slot], st);
    cudaError_t e;
    if (v3) {
      srht::V3Params vp;
      std::memset(&vp, 0, sizeof(vp));
      vp.src[0] = rp.src[0];
      vp.src[1] = rp.src[1];
      vp.ncols0 = rp.ncols0;
      vp.total_cols = rp.total_cols;
      vp.signs = P->d_signs3;
      vp.meta = P->d_meta3;
      vp.masks = P->d_masks3;
      vp.log_j = P->log_j2;
      vp.r = P->r;
      vp.n = P->n;
      vp.J = P->J2;
      vp.n_sub = P->n_sub2;
      vp.S_act = S2;
      vp.n_items = vp.total_cols * S2;
      vp.n_items32 = (int)vp.n_items;
      vp.S_act32 = (int)S2;
      vp.s_lo32 = (int)s_lo2;
      vp.J32 = (int)vp.J;
      vp.n_sub32 = (int)vp.n_sub;
      vp.uniform = (s_lo2 + S2) * vp.J <= vp.n_sub ? 1 : 0;
      vp.pairs = P->pairs3;
      vp.partials = sp.partials;
      vp.trace = srht::g_debug_trace;
      vp.debug = srht::g_debug_mode;
      e = srht::launch_sketch_tma(P, vp, st);
      srht::g_last_kernel = 3;
#ifdef V3_SYNC_CHECK  // experiment build: name the kernel an asynchronous fault comes from
      if (e == cudaSuccess) {
        const cudaError_t se = cudaStreamSynchronize(st);
        if (se != cudaSuccess) fprintf(stderr, "V3_SYNC_CHECK k_sketch_tma rpt %d: %s\n", P->rpt2, cudaGetErrorString(se));
      }
#endif
    } else {
      srht::WsParams wp;
      std::memset(&wp, 0, sizeof(wp));
      wp.src[0] = rp.src[0];
      wp.src[1] = rp.src[1];
      wp.ncols0 = rp.ncols0;
      wp.total_cols = rp.total_cols;
      wp.signs_ws = P->d_signs_ws;
      wp.meta = P->d_meta;
      wp.perm = P->d_perm;
      wp.r = P->r;
      wp.n = P->n;
      wp.J = P->J2;
      wp.n_sub = P->n_sub2;
      wp.S_act = S2;
      wp.s_lo = s_lo2;
      wp.n_items = wp.total_cols * S2;
      wp.scale = P->scale;
      wp.partials = sp.partials;
      wp.direct = direct;
      wp.debug = srht::g_debug_mode;
      wp.trace = srht::g_debug_trace;
      e = srht::launch_sketch_ws(P, wp, st);
      srht::g_last_kernel = 2;
    }
    if (slot >= 0) cudaEventRecord(srht::g_prof.ev[2 * slot + 1], st);
    if (e != cudaSuccess) return SRHT_ECUDA;
    if (v3) {  // slot-order partials, always reduced (also for a single slab)
      if (srht::launch_reduce_v3(rp, P->d_ttab3, P->rpt2, 14 + P->log_j2, st) != cudaSuccess) return SRHT_ECUDA;
#ifdef V3_SYNC_CHECK
      {
        const cudaError_t se = cudaStreamSynchronize(st);
        if (se != cudaSuccess) fprintf(stderr, "V3_SYNC_CHECK k_reduce_v3 rpt %d: %s\n", P->rpt2, cudaGetErrorString(se));
      }
#endif
    } else if (!direct && srht::launch_reduce(rp, 14 + P->log_j2, st) != cudaSuccess) {
      return SRHT_ECUDA;
    }
    return SRHT_OK;
  }
  return srht::launch_sketch(P, sp, st) == cudaSuccess ? SRHT_OK : SRHT_ECUDA;
}

}  // namespace

extern "C" {

const char* srht_status_str(srht_status s) {
  switch (s) {
    case SRHT_OK: return "SRHT_OK";
    case SRHT_EINVAL: return "SRHT_EINVAL: invalid argument";
    case SRHT_ENOMEM: return "SRHT_ENOMEM: device allocation failed";
    case SRHT_ECUDA: return "SRHT_ECUDA: CUDA error";
    case SRHT_EUNSUPPORTED: return "SRHT_EUNSUPPORTED: outside supported limits";
  }
  return "unknown srht_status";
}

srht_status srht_plan_create_ex(int64_t n, int64_t d, int64_t r, uint64_t seed, int64_t batch, uint32_t flags,
                                srht_plan** out) {
  NvtxRange nvtx_("srht_plan_create_ex");
  if (!out) return SRHT_EINVAL;
  *out = nullptr;
  if (n < 1 || d < 0 || r < 1 || batch < 1 || batch > 65535) return SRHT_EINVAL;
  if (flags & ~(uint32_t)(SRHT_PLAN_ACCUM_FP64 | SRHT_PLAN_BERNOULLI)) return SRHT_EINVAL;
  if ((flags & SRHT_PLAN_BERNOULLI) && batch != 1) return SRHT_EINVAL;
  int64_t N = 2;
  while (N < n) N *= 2;
  if (r > N) return SRHT_EINVAL;
  if (N > (int64_t(1) << 30)) return SRHT_EUNSUPPORTED;

  srht_plan* P = new (std::nothrow) srht_plan;
  if (!P) return SRHT_ENOMEM;
  std::memset(P, 0, sizeof(*P));
  P->n = n;
  P->d = d;
  P->r = r;
  P->N = N;
  P->batch = batch;
  P->seed = seed;
  P->flags = flags;
  P->r_target = r;
  if (flags & SRHT_PLAN_BERNOULLI) {
    // Algorithm 1 step 2 verbatim: row i kept iff u_i < T = floor(2^64 r / N) (prob. r/N).
    // The kept rows are then exactly the r' smallest keys, so the exact-r selection below
    // builds them with r = r' (the count is random; the scale stays r^{-1/2}).
    int64_t kept = N;
    if (r < N) {
      int lg = 0;
      while ((int64_t(1) << lg) < N) ++lg;
      const uint64_t T = (uint64_t)r << (64 - lg);  // N = 2^lg, r < N
      cudaStream_t st0;
      if (cudaStreamCreateWithFlags(&st0, cudaStreamNonBlocking) != cudaSuccess) {
        delete P;
        return SRHT_ECUDA;
      }
      const cudaError_t ce = srht::count_keys_below(seed, N, T, &kept, st0);
      cudaStreamDestroy(st0);
      if (ce != cudaSuccess) {
        delete P;
        return SRHT_ECUDA;
      }
    }
    if (kept < 1) {
      delete P;
      return SRHT_EUNSUPPORTED;  // no row kept (probability (1 - r/N)^N)
    }
    P->r = r = kept;
  }
  // Geometry (depends on n and r only).  Tile B ~ r (so ~1 sampled entry per
  // tile row, Ailon-Liberty balance), clamped to [2^10, 2^14]; slabs of ~2^20 rows.
  // B = 2r (capped at N): half a gather per element and half the tiles per column of B = r, for
  // +0.5 adds per element (config 3: 0.105 -> 0.094 ms; B = 4r: 0.115 ms)
  int lb = ceil_log2(r) + 1;
  if (lb > ceil_log2(N)) lb = ceil_log2(N);
  // Small columns (N <= 2^12) are transformed as a single tile: fewer
  // sequential sub-blocks per CTA and more threads per column (config 1:
  // 18.7 -> 11.7 us; 2^13 single tiles made config 2 slower, 3.7 -> 6.3 ms).
  if (N <= (int64_t(1) << 12) && ceil_log2(N) > lb) lb = ceil_log2(N);
  if (lb < 10) lb = 10;
  if (lb > 14) lb = 14;
  P->log_b = lb;
  P->B = int64_t(1) << lb;
  P->N_eff = N > P->B ? N : P->B;
  const int64_t NB = P->N_eff / P->B;
  int lj = 20 - lb;
  if (lj < 0) lj = 0;
  while ((int64_t(1) << lj) > NB) --lj;
  // Few, long columns (config 3: 301 columns of 32 tiles): shorter slabs so that the
  // (column, slab) items fill the GPU (~8 per SM; a slab reduction pass is added).
  {
#ifndef SRHT_V1_MIN_ITEMS
#define SRHT_V1_MIN_ITEMS 1184
#endif
    const int64_t nsub = (n + P->B - 1) / P->B;
    while (lj > 0 && batch * (d + 1) * ((nsub + (int64_t(1) << lj) - 1) >> lj) < SRHT_V1_MIN_ITEMS) --lj;
  }
  P->log_j = lj;
  P->J = int64_t(1) << lj;
  P->n_sub = (n + P->B - 1) / P->B;
  P->S_act = (P->n_sub + P->J - 1) / P->J;
  P->threads = (int)(P->B / 32);
  const int64_t per = (r + P->threads - 1) / P->threads;
  P->rpt = per <= 4 ? 4 : per <= 8 ? 8 : per <= 16 ? 16 : 32;
#ifdef SRHT_V1_MAX_RPT  // experiment: fewer accumulators per thread, more sample groups (CTAs) per tile
  if (P->rpt > SRHT_V1_MAX_RPT && P->B >= (int64_t(1) << 13)) P->rpt = SRHT_V1_MAX_RPT;
#endif
  P->groups = (r + (int64_t)P->rpt * P->threads - 1) / ((int64_t)P->rpt * P->threads);
  P->words64 = P->N_eff / 64;
  P->scale = (float)(1.0 / std::sqrt((double)P->r_target));
  if (cudaGetDevice(&P->device) != cudaSuccess) {
    delete P;
    return SRHT_ECUDA;
  }
  if (cudaMalloc(&P->d_signs, (size_t)batch * P->words64 * sizeof(uint64_t)) != cudaSuccess) {
    delete P;
    return SRHT_ENOMEM;
  }
  if (cudaMalloc(&P->d_K, (size_t)batch * r * sizeof(int32_t)) != cudaSuccess) {
    cudaFree(P->d_signs);
    delete P;
    return SRHT_ENOMEM;
  }
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    srht_plan_destroy(P);
    return SRHT_ECUDA;
  }
  cudaError_t e = srht::build_plan_device(P, st);
  cudaStreamDestroy(st);
  // Kernel v2 geometry (dense single problems): B = 2^14, slabs of 2^20 rows.
  // (Not built for FP64-accumulation plans, which always run the FP64 kernel.)
  if (e == cudaSuccess && !(flags & SRHT_PLAN_ACCUM_FP64) && batch == 1 && N >= (int64_t(1) << 14) && r <= 16384) {
    P->ws_ok = true;
    // Slab = J2 tiles; J2 ~ 64 r / 2^14 keeps the slab partials (r floats per
    // slab) near 3% of the input, and slabs small enough to load-balance.
    const int64_t NB2 = N >> 14;
    int lj2 = 0;
#ifndef SRHT_SLAB_FACTOR
#define SRHT_SLAB_FACTOR 64
#endif
    while ((int64_t(1) << lj2) < SRHT_SLAB_FACTOR * r / (1 << 14) && lj2 < SRHT_V3_MAX_LOGJ) ++lj2;
    while ((int64_t(1) << lj2) > NB2) --lj2;
    P->log_j2 = lj2;
    P->J2 = int64_t(1) << lj2;
    P->n_sub2 = (n + (1 << 14) - 1) >> 14;
    P->S_act2 = (P->n_sub2 + P->J2 - 1) / P->J2;
    P->rpt2 = r <= 8 * 256 ? 8 : r <= 16 * 256 ? 16 : r <= 32 * 256 ? 32 : 64;
    std::vector<int32_t> K(r);
    e = cudaMemcpy(K.data(), P->d_K, r * sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = build_ws_layout(P, K);
    if (e == cudaSuccess) e = build_v3_layout(P, K);
    const int64_t n_tiles = (P->N_eff >> 14);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_signs_ws, n_tiles * 128 * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_signs3, n_tiles * 128 * sizeof(uint4));
    if (e == cudaSuccess) {
      cudaStream_t st2;
      e = cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking);
      if (e == cudaSuccess) {
        e = srht::build_ws_signs(P->d_signs, n_tiles, P->d_signs_ws, st2);
        if (e == cudaSuccess) e = srht::build_v3_signs(P->d_signs, n_tiles, P->d_signs3, st2);
        cudaStreamDestroy(st2);
      }
    }
    P->v3_ok = (e == cudaSuccess) && P->log_j2 <= srht::V3_MAX_LOGJ && P->r < 0xffff;  // 16-bit t table
  }
  // Whole-column kernel gather order (FP32 plans with N_eff = 2^13, r <= 1024): per problem, the
  // kept rows are placed in SRHT_COL_SLOTS = 40 warp-wide steps of 32 slots (5 per thread), each
  // step taking at most one kept row per bank of its y words (tile word lo + 1024 j at
  // pad(lo) + 1056 j: bank (lo + lo / 32) mod 32) and, where possible, one per bank of its staging
  // word t (t mod 32) -- greedy, rows scanned for the fewest repeats.  Host simulation on config 2's
  // plans: 398 shared wavefronts per column for the gathers and z stores vs 594 with 32 steps.
#ifndef COL_PRUNE
#define COL_PRUNE 1
#endif
  if (COL_PRUNE && e == cudaSuccess && !(flags & SRHT_PLAN_ACCUM_FP64) && P->N_eff == (1 << 13) && r <= 1024) {
    std::vector<int32_t> Kall((size_t)batch * r);
    e = cudaMemcpy(Kall.data(), P->d_K, Kall.size() * sizeof(int32_t), cudaMemcpyDeviceToHost);
    std::vector<uint32_t> ck((size_t)batch * srht::COL_SLOTS, 0xffffffffu);
    for (int64_t pb = 0; e == cudaSuccess && pb < batch; ++pb)
      deal_col_slots(Kall.data() + pb * r, (int)r, ck.data() + pb * srht::COL_SLOTS);
    if (e == cudaSuccess) e = upload(&P->d_colk, ck);
  }
  // FP64 TMA kernel geometry (FP64 plans, single problem): B = 2^12, G sample groups of up to
  // 8192 samples (32 FP64 accumulators per consumer thread), slabs of up to 512 tiles, shortened
  // until the (group, column, slab) items give ~6 per SM.
  if (e == cudaSuccess && (flags & SRHT_PLAN_ACCUM_FP64) && batch == 1 && N >= (int64_t(1) << V64_LOG_B) &&
      r <= 4 * 8192) {
    P->G64 = (int)((r + 8191) / 8192);
    const int64_t per = (r + P->G64 - 1) / P->G64;
    P->rpt64 = per <= 4 * 256 ? 4 : per <= 8 * 256 ? 8 : per <= 16 * 256 ? 16 : 32;
    const int64_t n_tiles = N >> V64_LOG_B;
    P->n_sub64 = (n + (1 << V64_LOG_B) - 1) >> V64_LOG_B;
    int lj = 9;
    while (lj > 0 && (int64_t(1) << lj) > n_tiles) --lj;
    while (lj > 0 && P->G64 * (d + 1) * ((P->n_sub64 + (int64_t(1) << lj) - 1) >> lj) < 6 * 148) --lj;
    P->log_j64 = lj;
    P->J64 = int64_t(1) << lj;
    P->S_act64 = (P->n_sub64 + P->J64 - 1) / P->J64;
    std::vector<int32_t> K(r);
    e = cudaMemcpy(K.data(), P->d_K, r * sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = build_v64_layout(P, K);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_signs64, n_tiles * 64 * sizeof(uint2));
    if (e == cudaSuccess) {
      cudaStream_t st3;
      e = cudaStreamCreateWithFlags(&st3, cudaStreamNonBlocking);
      if (e == cudaSuccess) {
        e = srht::build_v64_signs(P->d_signs, n_tiles, P->d_signs64, st3);
        cudaStreamDestroy(st3);
      }
    }
    P->v64_ok = e == cudaSuccess;
  }
  if (e != cudaSuccess) {
    srht_plan_destroy(P);
    return e == cudaErrorMemoryAllocation ? SRHT_ENOMEM : SRHT_ECUDA;
  }
  *out = P;
  return SRHT_OK;
}

srht_status srht_plan_create_batched(int64_t n, int64_t d, int64_t r, uint64_t seed, int64_t batch,
                                     srht_plan** out) {
  return srht_plan_create_ex(n, d, r, seed, batch, 0u, out);
}

srht_status srht_plan_create(int64_t n, int64_t d, int64_t r, uint64_t seed, srht_plan** out) {
  return srht_plan_create_ex(n, d, r, seed, 1, 0u, out);
}

srht_status srht_plan_destroy(srht_plan* P) {
  if (!P) return SRHT_OK;
  cudaFree(P->d_signs);
  cudaFree(P->d_K);
  cudaFree(P->d_meta);
  cudaFree(P->d_perm);
  cudaFree(P->d_signs_ws);
  cudaFree(P->d_signs3);
  cudaFree(P->d_meta3);
  cudaFree(P->d_ttab3);
  cudaFree(P->d_masks3);
  cudaFree(P->d_signs64);
  cudaFree(P->d_meta64);
  cudaFree(P->d_ttab64);
  cudaFree(P->d_masks64);
  cudaFree(P->d_colk);
  delete P;
  return SRHT_OK;
}

srht_status srht_plan_info(const srht_plan* P, int64_t* N, int64_t* r, int64_t* batch) {
  if (!P) return SRHT_EINVAL;
  if (N) *N = P->N;
  if (r) *r = P->r;
  if (batch) *batch = P->batch;
  return SRHT_OK;
}

srht_status srht_plan_copy_indices(const srht_plan* P, int64_t problem, int32_t* host_K) {
  if (!P || !host_K || problem < 0 || problem >= P->batch) return SRHT_EINVAL;
  return cudaMemcpy(host_K, P->d_K + problem * P->r, P->r * sizeof(int32_t), cudaMemcpyDeviceToHost) == cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

srht_status srht_plan_copy_signs(const srht_plan* P, int64_t problem, uint64_t* host_words) {
  if (!P || !host_words || problem < 0 || problem >= P->batch) return SRHT_EINVAL;
  const int64_t w = (P->N + 63) / 64;
  return cudaMemcpy(host_words, P->d_signs + problem * P->words64, w * sizeof(uint64_t), cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

size_t srht_workspace_bytes(const srht_plan* P, int64_t ncols) {
  if (!P) return 0;
  return partial_bytes(P, ncols, true);  // covers srht_sketch_rows_partial too
}

srht_status srht_sketch_columns(const srht_plan* P, const srht_matrix* M, float* SM, int64_t ldsm, void* ws,
                                size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("srht_sketch_columns");
  if (!P || !valid_matrix(M) || M->rows != P->n || ldsm < P->r) return SRHT_EINVAL;
  if (M->cols > 0 && !SM) return SRHT_EINVAL;
  srht::SketchParams sp = base_params(P);
  sp.src[0] = make_src(M, SM, ldsm);
  sp.ncols0 = M->cols;
  sp.total_cols = M->cols;
  sp.cols_per_problem = INT64_MAX;  // every column uses problem 0's plan
  return run(P, sp, ws, ws_bytes, stream);
}

srht_status srht_ipc_alloc(size_t bytes, void** dev_ptr, void* handle) {
  if (!dev_ptr || !handle || bytes == 0) return SRHT_EINVAL;
  *dev_ptr = nullptr;
  if (cudaMalloc(dev_ptr, bytes) != cudaSuccess) return SRHT_ENOMEM;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, *dev_ptr) != cudaSuccess) {
    cudaFree(*dev_ptr);
    *dev_ptr = nullptr;
    return SRHT_ECUDA;
  }
  std::memcpy(handle, &h, sizeof(h));
  return SRHT_OK;
}

srht_status srht_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return SRHT_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? SRHT_OK : SRHT_ECUDA;
}

srht_status srht_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return SRHT_EINVAL;
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? SRHT_OK : SRHT_ECUDA;
}

srht_status srht_ipc_free(void* dev_ptr) {
  if (!dev_ptr) return SRHT_OK;
  return cudaFree(dev_ptr) == cudaSuccess ? SRHT_OK : SRHT_ECUDA;
}

srht_status srht_sketch_columns_peers(const srht_plan* P, const srht_matrix* M, int64_t col0, float* const* peers,
                                      int n_peers, int64_t ldp, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("srht_sketch_columns_peers");
  if (!P || !valid_matrix(M) || M->rows != P->n || ldp < P->r || col0 < 0 || !peers) return SRHT_EINVAL;
  if (n_peers < 1 || n_peers > SRHT_MAX_PEERS) return SRHT_EINVAL;
  for (int k = 0; k < n_peers; ++k)
    if (!peers[k]) return SRHT_EINVAL;
  if (M->cols == 0) return SRHT_OK;
  srht::SketchParams sp = base_params(P);
  float* local = peers[0] + col0 * ldp;
  sp.src[0] = make_src(M, local, ldp);
  sp.ncols0 = M->cols;
  sp.total_cols = M->cols;
  sp.cols_per_problem = INT64_MAX;
  sp.n_peers = n_peers;
  for (int k = 0; k < n_peers; ++k) sp.peers[k] = peers[k];
  sp.peer_col0 = col0;
  sp.peer_ld = ldp;
  srht::g_last_kernel = 0;
  const srht_status st = run(P, sp, ws, ws_bytes, stream);
  if (st != SRHT_OK) return st;
  if (srht::g_last_kernel == 3) return SRHT_OK;  // kernel v3's reduction stored into every peer
  // other paths: one copy kernel from the primary output into the peers
  return srht::launch_peer_copy(local, ldp, P->r, M->cols, peers, n_peers, col0, ldp,
                                static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

srht_status srht_sketch(const srht_plan* P, const srht_matrix* A, const srht_matrix* b, float* SA, int64_t ldsa,
                        float* Sb, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("srht_sketch");
  if (!P || !valid_matrix(A) || A->rows != P->n || ldsa < P->r) return SRHT_EINVAL;
  if (A->cols > 0 && !SA) return SRHT_EINVAL;
  if (b) {
    if (!valid_matrix(b) || b->rows != P->n || b->cols != 1 || !Sb) return SRHT_EINVAL;
  }
  srht::SketchParams sp = base_params(P);
  sp.src[0] = make_src(A, SA, ldsa);
  sp.ncols0 = A->cols;
  sp.total_cols = A->cols;
  if (b) {
    sp.src[1] = make_src(b, Sb, P->r);
    sp.total_cols += 1;
  }
  sp.cols_per_problem = INT64_MAX;  // a single problem (p = 0)
  return run(P, sp, ws, ws_bytes, stream);
}

srht_status srht_sketch_batched(const srht_plan* P, const srht_matrix* M, float* SM, void* ws, size_t ws_bytes,
                                void* stream) {
  NvtxRange nvtx_("srht_sketch_batched");
  if (!P || !valid_matrix(M) || M->rows != P->n || !SM) return SRHT_EINVAL;
  if (M->cols % P->batch != 0 || M->cols == 0) return SRHT_EINVAL;
  srht::SketchParams sp = base_params(P);
  sp.src[0] = make_src(M, SM, P->r);
  sp.ncols0 = M->cols;
  sp.total_cols = M->cols;
  sp.cols_per_problem = M->cols / P->batch;
  return run(P, sp, ws, ws_bytes, stream);
}

int64_t srht_row_shard_rows(const srht_plan* P) {
  if (!P) return 0;
  int64_t g = P->B * P->J;  // kernel v1 / FP64 slab
  if (P->ws_ok) {
    const int64_t g2 = (int64_t(1) << 14) * P->J2;  // kernel v2 / v3 slab
    if (g2 > g) g = g2;
  }
  if (P->v64_ok) {
    const int64_t g3 = (int64_t(1) << V64_LOG_B) * P->J64;  // FP64 TMA kernel slab
    if (g3 > g) g = g3;
  }
  return g;  // both are powers of two, so the larger is a multiple of the smaller
}

srht_status srht_sketch_rows_partial(const srht_plan* P, const srht_matrix* M, int64_t row0, double* part,
                                     int64_t ldp, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("srht_sketch_rows_partial");
  if (!P || !M || !part || P->batch != 1 || ldp < P->r || row0 < 0) return SRHT_EINVAL;
  if (M->rows < 1 || row0 + M->rows > P->n) return SRHT_EINVAL;
  const int64_t g = srht_row_shard_rows(P);
  if (row0 % g != 0 || ((row0 + M->rows) % g != 0 && row0 + M->rows != P->n)) return SRHT_EINVAL;
  srht_matrix Mg = *M;  // the shard seen with global row indices
  if (M->fmt == SRHT_DENSE) {
    if (!valid_matrix(M)) return SRHT_EINVAL;
    Mg.rows = P->n;
    if (M->cols > 0) Mg.vals = M->vals - row0;  // never dereferenced outside [row0, row0 + rows)
  } else {
    // CSC shards carry global row indices in [row0, row0 + rows); validated as an n-row matrix
    Mg.rows = P->n;
    if (!valid_matrix(&Mg)) return SRHT_EINVAL;
  }
  srht::SketchParams sp = base_params(P);
  sp.src[0] = make_src(&Mg, nullptr, P->r);
  sp.ncols0 = M->cols;
  sp.total_cols = M->cols;
  sp.cols_per_problem = INT64_MAX;
  sp.part_out = part;
  sp.ldp = ldp;
  return run(P, sp, ws, ws_bytes, stream, row0, M->rows);
}

srht_status srht_rows_finish(const srht_plan* P, const double* part, int64_t ldp, int64_t cols, float* SM,
                             int64_t ldsm, void* stream) {
  NvtxRange nvtx_("srht_rows_finish");
  if (!P || cols < 0 || ldp < P->r || ldsm < P->r) return SRHT_EINVAL;
  if (cols > 0 && (!part || !SM)) return SRHT_EINVAL;
  return srht::launch_rows_finish(part, ldp, P->r, cols, 1.0 / std::sqrt((double)P->r_target), SM, ldsm,
                                  static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

srht_status srht_gram(int64_t r, int64_t c, int64_t batch, const float* SM, int64_t ldsm, int64_t stride_sm,
                      double* G, int64_t ldg, int64_t stride_g, void* stream) {
  NvtxRange nvtx_("srht_gram");
  if (r < 1 || c < 1 || batch < 1 || !SM || !G || ldsm < r || ldg < c) return SRHT_EINVAL;
  if (batch > 1 && (stride_sm < ldsm * c || stride_g < ldg * c)) return SRHT_EINVAL;
  return srht::launch_gram(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g, nullptr,
                           static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

size_t srht_gram_workspace_bytes(int64_t r, int64_t c, int64_t batch) {
  if (r < 1 || c < 1 || batch < 1) return 0;
  return srht::gram_workspace_bytes(r, c, batch);
}

srht_status srht_gram_ex(int64_t r, int64_t c, int64_t batch, const float* SM, int64_t ldsm, int64_t stride_sm,
                         double* G, int64_t ldg, int64_t stride_g, void* workspace, size_t workspace_bytes,
                         void* stream) {
  NvtxRange nvtx_("srht_gram_ex");
  if (r < 1 || c < 1 || batch < 1 || !SM || !G || ldsm < r || ldg < c) return SRHT_EINVAL;
  if (batch > 1 && (stride_sm < ldsm * c || stride_g < ldg * c)) return SRHT_EINVAL;
  const size_t need = srht::gram_workspace_bytes(r, c, batch);
  if (need && (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 255)))
    return SRHT_EINVAL;
  return srht::launch_gram(r, c, batch, SM, ldsm, stride_sm, G, ldg, stride_g, need ? workspace : nullptr,
                           static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

size_t srht_nnls_workspace_bytes(int64_t d, int64_t batch) {
  if (d < 1 || batch < 1 || srht::nnls_factor_in_smem(d)) return 0;
  return (size_t)batch * 2 * (size_t)d * (size_t)d * sizeof(double);  // two factor slots per problem
}

srht_status srht_nnls_gram(int64_t d, int64_t batch, const double* G, int64_t ldg, int64_t stride_g, double* x,
                           int64_t stride_x, int32_t* iters, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("srht_nnls_gram");
  if (d < 1 || batch < 1 || !G || !x || ldg < d + 1 || d > 4096) return SRHT_EINVAL;
  if (batch > 1 && (stride_g < ldg * (d + 1) || stride_x < d)) return SRHT_EINVAL;
  const size_t need = srht_nnls_workspace_bytes(d, batch);
  if (need && (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 7))) return SRHT_EINVAL;
  return srht::launch_nnls_gram(d, batch, G, ldg, stride_g, x, stride_x, iters, static_cast<double*>(workspace),
                                static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

size_t srht_nnls_bpp_workspace_bytes(int64_t d, int64_t batch) {
  if (d < 1 || batch < 1) return 0;
  const size_t b = (size_t)batch * (size_t)d * (size_t)d * sizeof(double);
  if (batch == 1) {  // the cluster solver keeps its vectors in the workspace too
    const size_t c = srht::nnls_bpp_cl_workspace_bytes(d);
    return c > b ? c : b;
  }
  return b;
}

srht_status srht_nnls_gram_bpp(int64_t d, int64_t batch, const double* G, int64_t ldg, int64_t stride_g, double* x,
                               int64_t stride_x, int32_t* iters, void* workspace, size_t workspace_bytes,
                               void* stream) {
  NvtxRange nvtx_("srht_nnls_gram_bpp");
  if (d < 1 || batch < 1 || !G || !x || ldg < d + 1) return SRHT_EINVAL;
  if (batch > 1 && (stride_g < ldg * (d + 1) || stride_x < d)) return SRHT_EINVAL;
  if (!srht::nnls_bpp_ok(d)) return SRHT_EUNSUPPORTED;
  const size_t need = srht_nnls_bpp_workspace_bytes(d, batch);
  if (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 7)) return SRHT_EINVAL;
  return srht::launch_nnls_bpp(d, batch, G, ldg, stride_g, x, stride_x, iters, static_cast<double*>(workspace),
                               static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

srht_status srht_subspace_sample_count(int64_t n, int64_t r, uint64_t seed, const double* p, int64_t* kept,
                                       void* stream) {
  if (n < 1 || r < 1 || !p || !kept) return SRHT_EINVAL;
  return srht::launch_subspace(n, 0, r, seed, p, nullptr, 1, nullptr, nullptr, 1, 0, kept,
                               static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

srht_status srht_subspace_sample(int64_t n, int64_t d, int64_t r, uint64_t seed, const double* p, const float* Phi,
                                 int64_t ldphi, int32_t* K, float* out, int64_t ldout, int64_t cap, void* stream) {
  NvtxRange nvtx_("srht_subspace_sample");
  if (n < 1 || d < 0 || r < 1 || !p || !K || cap < 0 || (d > 0 && (!Phi || !out || ldphi < n || ldout < cap)))
    return SRHT_EINVAL;
  return srht::launch_subspace(n, d, r, seed, p, Phi, ldphi, K, out, ldout, cap, nullptr,
                               static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

// Undeclared test hook: copy the kernel-v2 consumer slot layout to the host.
int srht_debug_copy_ws_layout(const srht_plan* P, uint32_t* meta, int32_t* perm, int* rpt2) {
  if (!P || !P->ws_ok) return 1;
  *rpt2 = P->rpt2;
  if (meta && cudaMemcpy(meta, P->d_meta, P->rpt2 * 256 * sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return 3;
  if (perm && cudaMemcpy(perm, P->d_perm, P->rpt2 * 256 * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return 3;
  return 0;
}

// Undeclared host-only test hooks (no CUDA calls; `-m "not gpu"` tests run them on the oracle's
// plans): the slot dealing of kernel v3 (shared gathers) and of the whole-column kernel.
int srht_debug_deal_v3(const int32_t* K, int64_t r, int rpt, int* pairs, int32_t* acc_t, uint32_t* meta) {
  if (!K || r < 1 || r > 256 * (int64_t)rpt || !pairs || !acc_t || !meta) return 1;
  const std::vector<int32_t> Kv(K, K + r);
  *pairs = choose_pairs3(Kv, rpt);
  std::vector<int32_t> a;
  std::vector<uint32_t> m;
  deal_v3_pairs(Kv, rpt, *pairs, a, m);
  std::copy(a.begin(), a.end(), acc_t);
  std::copy(m.begin(), m.end(), meta);
  return 0;
}
int srht_debug_deal_col(const int32_t* K, int64_t r, uint32_t* out) {
  if (!K || r < 1 || r > 1024 || !out) return 1;
  deal_col_slots(K, (int)r, out);
  return 0;
}

// Undeclared test hook: kernel v3's consumer layout -- load-slot byte offsets meta[c][l]
// (rpt2 - pairs3 per thread), output rows of the accumulators ttab[c][q/2] (16 bits each), and
// the number of shared-gather slots pairs3.
int srht_debug_copy_v3_layout(const srht_plan* P, uint32_t* meta, uint32_t* ttab, int* rpt2, int* pairs3) {
  if (!P || !P->v3_ok) return 1;
  *rpt2 = P->rpt2;
  *pairs3 = P->pairs3;
  const size_t nm = (size_t)256 * (P->rpt2 - P->pairs3), nt = (size_t)256 * (P->rpt2 / 2);
  if (meta && cudaMemcpy(meta, P->d_meta3, nm * sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess) return 3;
  if (ttab && cudaMemcpy(ttab, P->d_ttab3, nt * sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess) return 3;
  return 0;
}

// Undeclared experiment hook (scripts only): knock out parts of kernel v2.
// bit0: producers skip global loads; bit1: consumers skip the gather;
// bit2: producers skip the butterflies.  Results are wrong when non-zero.
int srht_debug_set_mode(int mode) {
  srht::g_debug_mode = mode;
  return 0;
}
// Undeclared experiment hook: 0 = automatic kernel choice, 2 = use kernel v2 where
// kernel v3 would run (A/B comparison in scripts and tests).
int srht_debug_last_kernel(void) { return srht::g_last_kernel; }
int srht_debug_set_kernel(int version) {
  srht::g_kernel_force = version;
  return 0;
}
int srht_debug_set_trace(unsigned long long* dev_buf) {
  srht::g_debug_trace = dev_buf;
  return 0;
}

srht_status srht_profile_start(int capacity) {
  if (capacity < 1 || srht::g_prof.on) return SRHT_EINVAL;
  srht::ProfileState& g = srht::g_prof;
  g.ev = new (std::nothrow) cudaEvent_t[2 * (size_t)capacity];
  if (!g.ev) return SRHT_ENOMEM;
  for (int i = 0; i < 2 * capacity; ++i) {
    if (cudaEventCreate(&g.ev[i]) != cudaSuccess) {
      for (int k = 0; k < i; ++k) cudaEventDestroy(g.ev[k]);
      delete[] g.ev;
      g.ev = nullptr;
      return SRHT_ECUDA;
    }
  }
  g.capacity = capacity;
  g.used = 0;
  g.on = true;
  return SRHT_OK;
}

srht_status srht_profile_stop(float* ms, int capacity, int* count) {
  srht::ProfileState& g = srht::g_prof;
  if (!g.on) return SRHT_EINVAL;
  srht_status st = SRHT_OK;
  int n = 0;
  for (int i = 0; i < g.used; ++i) {
    float t = 0.f;
    if (cudaEventSynchronize(g.ev[2 * i + 1]) != cudaSuccess ||
        cudaEventElapsedTime(&t, g.ev[2 * i], g.ev[2 * i + 1]) != cudaSuccess) {
      st = SRHT_ECUDA;
      break;
    }
    if (ms && i < capacity) ms[n++] = t;
  }
  if (count) *count = n;
  for (int i = 0; i < 2 * g.capacity; ++i) cudaEventDestroy(g.ev[i]);
  delete[] g.ev;
  g = srht::ProfileState();
  return st;
}

srht_status srht_gen_uniform(uint64_t seed, uint64_t stream0, int64_t rows, int64_t cols, float* out, int64_t ld,
                             void* stream) {
  if (rows < 0 || cols < 0 || ld < rows || (rows > 0 && cols > 0 && !out)) return SRHT_EINVAL;
  return srht::launch_gen_uniform(seed, stream0, rows, cols, out, ld, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? SRHT_OK
             : SRHT_ECUDA;
}

// Host-buffer variant: stream column chunks host -> device, sketch, device -> host,
// double-buffered over two streams so copies overlap the kernels.
srht_status srht_sketch_columns_host(const srht_plan* P, const srht_matrix* Mh, float* SMh, int64_t ldsm) {
  NvtxRange nvtx_("srht_sketch_columns_host");
  if (!P || !valid_matrix(Mh) || Mh->rows != P->n || ldsm < P->r) return SRHT_EINVAL;
  if (Mh->cols == 0) return SRHT_OK;
  if (!SMh) return SRHT_EINVAL;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != P->device) return SRHT_EINVAL;
  const int64_t n = Mh->rows, ncols = Mh->cols;
  // columns per chunk: ~256 MB of input, at least 1
  int64_t chunk = 1;
  if (Mh->fmt == SRHT_DENSE) {
    const int64_t bytes_per_col = n * (int64_t)sizeof(float);
    chunk = (int64_t(256) << 20) / (bytes_per_col > 0 ? bytes_per_col : 1);
  } else {
    const int64_t per = (Mh->nnz * 12) / (ncols > 0 ? ncols : 1) + 16;
    chunk = (int64_t(256) << 20) / per;
  }
  if (chunk < 1) chunk = 1;
  if (chunk > ncols) chunk = ncols;
  // For CSC the largest chunk nnz bounds the buffer size.
  int64_t max_nnz = 0;
  if (Mh->fmt == SRHT_CSC) {
    for (int64_t c0 = 0; c0 < ncols; c0 += chunk) {
      const int64_t c1 = c0 + chunk < ncols ? c0 + chunk : ncols;
      const int64_t z = Mh->colptr[c1] - Mh->colptr[c0];
      if (z > max_nnz) max_nnz = z;
    }
  }
  const size_t ws = partial_bytes(P, chunk);
  struct Buf {
    float* vals = nullptr;
    int64_t* colptr = nullptr;
    int32_t* rowidx = nullptr;
    float* out = nullptr;
    void* ws = nullptr;
    cudaStream_t st = nullptr;
  } buf[2];
  srht_status status = SRHT_OK;
  auto fail = [&](srht_status s) {
    if (status == SRHT_OK) status = s;
  };
  for (int i = 0; i < 2 && status == SRHT_OK; ++i) {
    if (cudaStreamCreateWithFlags(&buf[i].st, cudaStreamNonBlocking) != cudaSuccess) fail(SRHT_ECUDA);
    const size_t vbytes = Mh->fmt == SRHT_DENSE ? (size_t)n * chunk * sizeof(float) : (size_t)(max_nnz + 1) * sizeof(float);
    if (cudaMalloc(&buf[i].vals, vbytes) != cudaSuccess) fail(SRHT_ENOMEM);
    if (Mh->fmt == SRHT_CSC) {
      if (cudaMalloc(&buf[i].colptr, (chunk + 1) * sizeof(int64_t)) != cudaSuccess) fail(SRHT_ENOMEM);
      if (cudaMalloc(&buf[i].rowidx, (max_nnz + 1) * sizeof(int32_t)) != cudaSuccess) fail(SRHT_ENOMEM);
    }
    if (cudaMalloc(&buf[i].out, (size_t)P->r * chunk * sizeof(float)) != cudaSuccess) fail(SRHT_ENOMEM);
    if (ws && cudaMalloc(&buf[i].ws, ws) != cudaSuccess) fail(SRHT_ENOMEM);
  }
  int64_t it = 0;
  for (int64_t c0 = 0; c0 < ncols && status == SRHT_OK; c0 += chunk, ++it) {
    Buf& b = buf[it & 1];
    const int64_t nc = c0 + chunk < ncols ? chunk : ncols - c0;
    srht_matrix Md = *Mh;
    Md.cols = nc;
    if (Mh->fmt == SRHT_DENSE) {
      if (cudaMemcpy2DAsync(b.vals, n * sizeof(float), Mh->vals + c0 * Mh->ld, Mh->ld * sizeof(float),
                            n * sizeof(float), nc, cudaMemcpyHostToDevice, b.st) != cudaSuccess) {
        fail(SRHT_ECUDA);
        break;
      }
      Md.vals = b.vals;
      Md.ld = n;
    } else {
      const int64_t z0 = Mh->colptr[c0], z1 = Mh->colptr[c0 + nc];
      if (cudaMemcpyAsync(b.colptr, Mh->colptr + c0, (nc + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, b.st) !=
              cudaSuccess ||
          (z1 > z0 && cudaMemcpyAsync(b.rowidx, Mh->rowidx + z0, (z1 - z0) * sizeof(int32_t),
                                      cudaMemcpyHostToDevice, b.st) != cudaSuccess) ||
          (z1 > z0 && cudaMemcpyAsync(b.vals, Mh->vals + z0, (z1 - z0) * sizeof(float), cudaMemcpyHostToDevice,
                                      b.st) != cudaSuccess)) {
        fail(SRHT_ECUDA);
        break;
      }
      // colptr entries are absolute offsets: rebase the value/index pointers.
      Md.colptr = b.colptr;
      Md.rowidx = b.rowidx - z0;
      Md.vals = b.vals - z0;
      Md.nnz = z1 - z0;
    }
    const srht_status s = srht_sketch_columns(P, &Md, b.out, P->r, b.ws, ws, b.st);
    if (s != SRHT_OK) {
      fail(s);
      break;
    }
    if (cudaMemcpy2DAsync(SMh + c0 * ldsm, ldsm * sizeof(float), b.out, P->r * sizeof(float), P->r * sizeof(float),
                          nc, cudaMemcpyDeviceToHost, b.st) != cudaSuccess) {
      fail(SRHT_ECUDA);
      break;
    }
  }
  for (int i = 0; i < 2; ++i) {
    if (buf[i].st && cudaStreamSynchronize(buf[i].st) != cudaSuccess) fail(SRHT_ECUDA);
  }
  for (int i = 0; i < 2; ++i) {
    cudaFree(buf[i].vals);
    cudaFree(buf[i].colptr);
    cudaFree(buf[i].rowidx);
    cudaFree(buf[i].out);
    cudaFree(buf[i].ws);
    if (buf[i].st) cudaStreamDestroy(buf[i].st);
  }
  return status;
}

}  // extern "C"
