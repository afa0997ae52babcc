// Internal declarations shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>

#include "../../include/srht.h"

struct srht_plan {
  int64_t n, d, r, N, batch;
  uint64_t seed;
  uint32_t flags;   // SRHT_PLAN_ACCUM_FP64: every sketch runs the FP64-accumulation kernel;
                    // SRHT_PLAN_BERNOULLI: r is the random kept count, r_target the requested r
  int64_t r_target; // requested r (the scale is r_target^{-1/2})
  // Tile / slab geometry: depends on (n, r) only.
  int log_b;        // tile bits; B = 2^log_b rows per sub-block
  int64_t B;
  int64_t N_eff;    // max(N, B)
  int log_j;        // sub-blocks per slab J = 2^log_j
  int64_t J;
  int64_t n_sub;    // sub-blocks holding rows < n: ceil(n / B)
  int64_t S_act;    // slabs holding rows < n: ceil(n_sub / J)
  int threads;      // CTA size = B / 32
  int rpt;          // accumulators per thread
  int64_t groups;   // sample groups = ceil(r / (rpt * threads))
  int64_t words64;  // sign words per problem = N_eff / 64
  float scale;      // r^{-1/2} rounded to FP32
  int device;
  uint64_t* d_signs;  // [batch][words64]
  int32_t* d_K;       // [batch][r], ascending
  // Kernel v2 (dense, warp-specialized, B = 2^14): geometry + consumer slot layout.
  bool ws_ok;         // single problem, N >= 2^14, r <= 16384
  int log_j2;
  int64_t J2, n_sub2, S_act2;
  int rpt2;           // consumer accumulators per thread (8/16/32/64)
  uint4* d_signs_ws;  // [N/2^14][128] sign bits in producer-thread order
  uint32_t* d_meta;   // [rpt2*256]: byte offset of phys(k_lo) | reversed k_mid << 17
  int32_t* d_perm;    // [rpt2*256]: sample index t or -1
  // Kernel v3 (TMA-fed, same geometry as v2): layouts for its own tile order.
  bool v3_ok;
  uint4* d_signs3;    // [N/2^14][128] sign bits of rows e + 2p + 256h, bit 2h+e
  int pairs3;          // kernel v3: load slots per consumer thread that feed two accumulators
  uint32_t* d_meta3;  // [256][rpt2 - pairs3]: byte offset of load slot l's z value (mid layout)
  uint32_t* d_ttab3;  // [256][rpt2/2]: output rows t of slots (2i, 2i+1), 16 bits each (0xffff: empty)
  uint2* d_masks3;    // [log_j2][256]: bit q = bit sh of k_mid of slot (q, c)
  // FP64-accumulation TMA kernel (sketch_tma64.cu; FP64 plans, single problem, N >= 2^12,
  // r <= 32768): B = 2^12 tiles, slabs of J64 tiles, G64 sample groups of rpt64 * 256 slots.
  bool v64_ok;
  int log_j64;
  int64_t J64, n_sub64, S_act64;
  int rpt64, G64;
  uint2* d_signs64;   // [N/2^12][64] D bits of rows e + 2p + 128h, bit 2(h & 15) + e of word h >> 4
  uint32_t* d_meta64; // [G][256][rpt64]: byte offset of slot (q, c)'s z value (mid layout)
  int32_t* d_ttab64;  // [G][256][rpt64]: output row t of the slot, -1 if empty
  uint32_t* d_masks64;// [G][log_j64][256]: bit q = bit l of k_mid of slot (q, c)
  // Whole-column kernel (N_eff = 2^13, r <= 1024): per problem the kept rows in gather order,
  // k | (output row t) << 16 (0xffffffff: empty slot), in srht::COL_SLOTS slots = 40 warp-wide
  // steps of 32, dealt so a step's gathers (and where possible its staging stores) hit distinct banks.
  uint32_t* d_colk;   // [batch][COL_SLOTS]
};

namespace srht {
constexpr int COL_SLOTS = 5 * 256;  // whole-column kernel: kept-row slots per problem (5 per thread)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) holds per device: set it once per device
// a kernel runs on (bit per device ordinal), safely from several host threads.
template <typename K>
cudaError_t set_max_dyn_smem_once(K* kernel, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}


// Plan builder (plan.cu): fills d_signs and d_K; synchronous on `stream`.
cudaError_t build_plan_device(srht_plan* P, cudaStream_t stream);
cudaError_t count_keys_below(uint64_t seed, int64_t N, uint64_t T, int64_t* count, cudaStream_t stream);
cudaError_t build_ws_signs(const uint64_t* signs, int64_t n_tiles, uint4* out, cudaStream_t stream);
cudaError_t build_v3_signs(const uint64_t* signs, int64_t n_tiles, uint4* out, cudaStream_t stream);

// One column source of a sketch launch.
struct ColSrc {
  int fmt;                // SRHT_DENSE / SRHT_CSC
  int vec;                // dense: 16-byte vector loads allowed
  const float* vals;
  int64_t ld;
  const int64_t* colptr;
  const int32_t* rowidx;
  int64_t ncols;
  float* out;             // column j of this source -> out + j * ldo
  int64_t ldo;
};

#define SRHT_MAX_PEERS 8
struct SketchParams {
  ColSrc src[2];
  int64_t ncols0;             // columns of src[0]; src[1] follows
  int64_t total_cols;
  int64_t cols_per_problem;   // problem of global column g = g / cols_per_problem
  const uint32_t* signs;      // sign words viewed as uint32
  int64_t words32;            // per problem
  const int32_t* K;
  int64_t r;
  int64_t n;
  int64_t J;
  int log_j;
  int64_t n_sub;
  int64_t S_act;              // slabs of this launch: global slabs s_lo .. s_lo + S_act - 1
  int64_t s_lo;               // first global slab (row shards, srht_sketch_rows_partial); else 0
  int64_t groups;
  float scale;
  double scale_f64;           // r^{-1/2} in FP64 (slab reduction)
  float* partials;            // [S_act][total_cols][r] when S_act > 1 or part_out
  double* partials64;         // FP64 mode: [S_act][total_cols][r] when S_act > 1 or part_out
  double* part_out;           // row-shard mode: unscaled FP64 partial sums, column j at part_out + j*ldp
  int64_t ldp;
  // fused gather (srht_sketch_columns_peers): kernel v3's reduction also stores output column j at
  // column peer_col0 + j of every peer buffer (ld peer_ld); peers[0] is the primary output
  float* peers[SRHT_MAX_PEERS];
  int n_peers;
  int64_t peer_col0, peer_ld;
  const uint32_t* colk;       // whole-column kernel: plan d_colk (null: full last round + gather)
};
// FP64-accumulation parity mode (sketch_f64.cu), v1 slab geometry.
cudaError_t launch_sketch_f64(const srht_plan* P, const SketchParams& sp, cudaStream_t stream);

cudaError_t launch_sketch(const srht_plan* P, const SketchParams& sp, cudaStream_t stream);

// Kernel v2 (sketch_ws.cu): dense columns only.
struct WsParams {
  ColSrc src[2];
  int64_t ncols0, total_cols;
  const uint4* signs_ws;  // problem 0, producer-thread order
  const uint32_t* meta;
  const int32_t* perm;
  int64_t r, n;
  int64_t J, n_sub, S_act;  // S_act: slabs of this launch, global slabs s_lo ..
  int64_t s_lo;
  int64_t n_items;        // total_cols * S_act
  float scale;
  float* partials;        // [S_act][total_cols][r] when S_act > 1 or direct == 0
  int direct;             // 1: single slab, write r^{-1/2} * sum straight to the output
  int debug;              // experiment knock-outs (srht_debug_set_mode); 0 in production
  unsigned long long* trace;  // experiment phase timestamps (debug build only)
};
extern int g_debug_mode;
extern unsigned long long* g_debug_trace;
cudaError_t launch_sketch_ws(const srht_plan* P, const WsParams& wp, cudaStream_t stream);
int ws_phys(int x);  // tile layout of kernel v2 (host side, for the slot layout)
// Kernel v3 (sketch_tma.cu): dense columns with 16-byte aligned columns (TMA bulk copies).
#ifndef V3_TMEM_RAW
#define V3_TMEM_RAW 0  // 1: kernel v3 round 1 reads the raw tile through TMEM (measured slower, DESIGN 11)
#endif
#ifndef SRHT_V3_MAX_LOGJ
#define SRHT_V3_MAX_LOGJ 6
#endif
constexpr int V3_MAX_LOGJ = SRHT_V3_MAX_LOGJ;
struct V3Params {
  ColSrc src[2];
  int64_t ncols0, total_cols;
  const uint4* signs;     // plan d_signs3
  const uint32_t* meta;   // plan d_meta3
  const uint2* masks;     // plan d_masks3
  int log_j;
  int64_t r, n;
  int64_t J, n_sub, S_act;  // S_act: slabs of this launch, global slabs s_lo ..
  int64_t n_items;        // total_cols * S_act
  int n_items32, S_act32, J32, n_sub32, s_lo32;  // the same, 32-bit (checked on the host)
  int uniform;            // every slab of the launch is full (J tiles): closed-form tile order
  int pairs;              // load slots per consumer thread that feed two accumulators (plan pairs3)
  float* partials;        // [S_act][total_cols][rpt2 * 256], slot order (k_reduce_v3 finishes)
  unsigned long long* trace;  // experiment phase timestamps (srht_debug_set_trace), else null
  int debug;                  // experiment knock-outs (srht_debug_set_mode, debug build), else 0
};
cudaError_t launch_sketch_tma(const srht_plan* P, const V3Params& vp, cudaStream_t stream);
// FP64-accumulation TMA kernel (sketch_tma64.cu).
#define V64_LOG_B 12
struct V64Params {
  ColSrc src[2];
  int64_t ncols0, total_cols;
  const uint2* signs;     // plan d_signs64
  const uint32_t* meta;   // plan d_meta64
  const uint32_t* masks;  // plan d_masks64
  int log_j, G;
  int64_t n;
  int n_items32, cols32, S_act32, J32, n_sub32, s_lo32;  // items = G * cols * S_act (checked < 2^31)
  double* partials;       // [S_act][G][total_cols][rpt64 * 256], slot order (k_reduce64 finishes)
};
cudaError_t launch_sketch_tma64(const srht_plan* P, const V64Params& vp, cudaStream_t stream);
cudaError_t launch_reduce64(const SketchParams& sp, const int32_t* ttab, int rpt, int G, int slab_shift,
                            cudaStream_t stream);
int v64_mid(int x);  // kernel z layout (host side, for the slot layout)
cudaError_t build_v64_signs(const uint64_t* signs, int64_t n_tiles, uint2* out, cudaStream_t stream);
// Slab reduction of kernel v3's slot-order partials (sp.partials, S_act, s_lo, outputs).
cudaError_t launch_reduce_v3(const SketchParams& sp, const uint32_t* ttab, int rpt, int slab_shift,
                             cudaStream_t stream);
// Copy r x cols FP32 (column-major, ld src_ld) to every peer buffer at column col0 (ld peer_ld).
cudaError_t launch_peer_copy(const float* src, int64_t src_ld, int64_t r, int64_t cols, float* const* peers,
                             int n_peers, int64_t col0, int64_t peer_ld, cudaStream_t stream);
int v3_mid(int x);  // kernel-v3 z layout (host side, for the slot layout)
extern int g_kernel_force;  // 0 auto, 2 = kernel v2 instead of v3 (srht_debug_set_kernel)
extern int g_last_kernel;   // tile kernel of the last srht_sketch* call (bench labels): 1 tiles, 2 ws,
                            // 3 tma, 4 f64, 5 col, 6 tma64
// Gram matrices of sketches (gram.cu): G_p = SM_p^T SM_p in FP64.
cudaError_t launch_gram(int64_t r, int64_t c, int64_t batch, const float* SM, int64_t ldsm, int64_t stride_sm,
                        double* G, int64_t ldg, int64_t stride_g, void* ws, cudaStream_t stream);
size_t gram_workspace_bytes(int64_t r, int64_t c, int64_t batch);

// Batched Lawson-Hanson NNLS on the Gram form (nnls.cu).
bool nnls_factor_in_smem(int64_t d);
// Block principal pivoting NNLS on the Gram form (nnls.cu): d x d FP64 factor per problem in ws.
bool nnls_bpp_ok(int64_t d);
size_t nnls_bpp_cl_workspace_bytes(int64_t d);  // single large problem on a cluster (batch 1)
cudaError_t launch_nnls_bpp(int64_t d, int64_t batch, const double* G, int64_t ldg, int64_t stride_g, double* x,
                            int64_t stride_x, int32_t* iters, double* ws, cudaStream_t stream);
cudaError_t launch_nnls_gram(int64_t d, int64_t batch, const double* G, int64_t ldg, int64_t stride_g, double* x,
                             int64_t stride_x, int32_t* iters, double* ws, cudaStream_t stream);

// Algorithm 2 SubspaceSampling (subspace.cu).
cudaError_t launch_subspace(int64_t n, int64_t d, int64_t r, uint64_t seed, const double* p, const float* Phi,
                            int64_t ldphi, int32_t* K, float* out, int64_t ldout, int64_t cap, int64_t* kept,
                            cudaStream_t stream);

// Fixed-order slab reduction shared by every kernel.
cudaError_t launch_reduce(const SketchParams& sp, int slab_shift, cudaStream_t stream);
// Row-partition finish: SM = (float)(part * scale), r x cols (srht_rows_finish).
cudaError_t launch_rows_finish(const double* part, int64_t ldp, int64_t r, int64_t cols, double scale, float* SM,
                               int64_t ldsm, cudaStream_t stream);

// Profiling (srht_profile_start/stop): event pairs around the tile kernel.
struct ProfileState {
  bool on = false;
  int capacity = 0, used = 0;
  cudaEvent_t* ev = nullptr;  // 2 * capacity
};
extern ProfileState g_prof;

cudaError_t launch_gen_uniform(uint64_t seed, uint64_t stream0, int64_t rows, int64_t cols,
                               float* out, int64_t ld, cudaStream_t stream);

}  // namespace srht
