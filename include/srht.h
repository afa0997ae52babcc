/*
 * srht.h -- C ABI of the B200 SRHT sketch (hot path of RandomizedNNLS,
 * arXiv 0812.4547, "Random projections for the nonnegative least-squares
 * problem").
 *
 * What it computes (Algorithm 1, and the proof's
 * Phi = [H_n D A, -H_n D b]):
 *
 *     SM[t, j] = sqrt(N/r) * (H_N/sqrt(N) * D * [M ; 0])[k_t, j]
 *              = r^{-1/2} * sum_{i<n} (-1)^{popc(k_t & i)} * sigma_i * M[i, j]
 *
 * for every column j of M = [A | b] (n x (d+1)), with
 *   N        = smallest power of two >= max(n, 2) (zero padding),
 *   sigma_i  = +-1 diagonal of D (Algorithm 1 step 4),
 *   k_0<...<k_{r-1} = the kept rows of S H_N (steps 2-3),
 *   H_N[k,i] = (-1)^{popc(k & i)} (Sylvester recursion of P:154-165).
 * The same D and the same kept rows act on every column.
 *
 * Readings where the paper is silent (R1-R14): exactly r distinct
 * rows (R1); the padded N is the n of sqrt(n/r) (R2); Philox4x64-10 streams
 * (R4): word w of stream (seed, 2p + tag) is word (w mod 4) of
 * philox4x64_10(ctr = (1 + w/4, 0, 0, 0), key = (seed, 2p + tag)); sigma_i = -1
 * iff bit (i mod 64) of word i/64 of tag 0 is set (R5); k = the r indices with
 * the smallest (word i of tag 1, i), sorted ascending (R6).  p is the problem
 * index (0 for a single problem).
 *
 * Conventions for every entry point:
 *   - Matrix/vector pointers passed to srht_sketch* are DEVICE pointers owned by
 *     the caller; inputs are read-only, outputs write-only.  The plan owns only
 *     its own device buffers (sign words, kept rows).
 *   - srht_sketch* enqueue work on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream) and return without synchronizing.
 *     Asynchronous faults surface at the caller's next synchronization.
 *   - srht_plan_create* are synchronous on the current CUDA device.
 *   - Scratch memory is caller-provided (srht_workspace_bytes); srht_sketch*
 *     never allocate, so concurrent calls on different streams with different
 *     workspaces are safe.  A plan is immutable after creation.
 *   - Invalid arguments return SRHT_EINVAL before any launch; launch failures
 *     return SRHT_ECUDA.  Non-finite input values are not checked.
 *   - Arithmetic: FP32 inputs, FP32 adds (round to nearest), FP32 outputs;
 *     the final r^{-1/2} is applied once, in FP32, to the FP32 sum.
 */
#ifndef SRHT_H_
#define SRHT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct srht_plan srht_plan; /* opaque, immutable after create */

typedef enum {
  SRHT_OK = 0,
  SRHT_EINVAL = 1,       /* bad argument (checked before any launch)        */
  SRHT_ENOMEM = 2,       /* device allocation failed (plan creation only)   */
  SRHT_ECUDA = 3,        /* a CUDA call or kernel launch failed             */
  SRHT_EUNSUPPORTED = 4  /* valid but outside this build's limits           */
} srht_status;

enum { SRHT_DENSE = 0, SRHT_CSC = 1 };

/* A device matrix with `rows` rows and `cols` columns.
 * SRHT_DENSE: column-major FP32, element (i, j) at vals[i + j*ld], ld >= rows.
 * SRHT_CSC:   column j holds entries colptr[j] .. colptr[j+1]-1 of
 *             (rowidx, vals); colptr has cols+1 int64 entries (colptr[0] may be
 *             non-zero); rowidx is int32, sorted ascending within a column,
 *             0 <= rowidx < rows; duplicate row indices are summed.          */
typedef struct {
  int32_t fmt;
  int64_t rows, cols;
  const float* vals;
  int64_t ld;
  const int64_t* colptr;
  const int32_t* rowidx;
  int64_t nnz;
} srht_matrix;

/* Build the plan of one problem (p = 0): n rows, d columns of A (the sketch
 * accepts any column count; d is recorded for srht_sketch), r kept rows,
 * Philox seed.  Requires n >= 1, d >= 0, 1 <= r <= N, N <= 2^30.
 * Algorithm 1 steps 2 and 4, computed on the device.            */
srht_status srht_plan_create(int64_t n, int64_t d, int64_t r, uint64_t seed,
                             srht_plan** out);

/* `batch` independent problems of the same shape; problem p uses streams
 * (seed, 2p) and (seed, 2p+1), i.e. its own D and kept rows.                 */
srht_status srht_plan_create_batched(int64_t n, int64_t d, int64_t r,
                                     uint64_t seed, int64_t batch,
                                     srht_plan** out);

/* Plan flags for srht_plan_create_ex. */
enum {
  /* Every sketch of this plan accumulates in FP64: FP32 inputs are widened,
   * the Hadamard butterflies, the pruned accumulation and the slab sums run
   * in FP64, and each output is rounded once to FP32 (close to the correctly
   * rounded FP32 sketch).  This is the parity mode of DESIGN.md reading R14
   * (the 1e-6 end-to-end NNLS gate of BASELINE.json's north_star sits at the
   * FP32 rounding floor); it is several times slower than the
   * default FP32 path, which it does not replace.  Workspace: FP64 partials
   * (srht_workspace_bytes accounts for it).                                  */
  SRHT_PLAN_ACCUM_FP64 = 1,
  /* Algorithm 1 step 2 read verbatim: every row of S H_N is
   * kept independently with probability r/N -- row i iff u_i < floor(2^64 r/N)
   * (u_i = word i of stream (seed, 1), the same keys as the exact-r
   * selection) -- so the kept count r' is random with mean r.  srht_plan_info
   * reports r' (the sketches have r' rows); the scale stays r^{-1/2} for the
   * requested r.  Single-problem plans only (batch = 1); r' = 0 is
   * SRHT_EUNSUPPORTED.                                                      */
  SRHT_PLAN_BERNOULLI = 2
};

/* srht_plan_create_batched with flags (an OR of SRHT_PLAN_ACCUM_FP64 and
 * SRHT_PLAN_BERNOULLI); any other bit is SRHT_EINVAL.  Same requirements and
 * errors otherwise.                                                          */
srht_status srht_plan_create_ex(int64_t n, int64_t d, int64_t r, uint64_t seed,
                                int64_t batch, uint32_t flags,
                                srht_plan** out);

srht_status srht_plan_destroy(srht_plan* plan); /* NULL is a no-op */

/* N (padded size), r and batch of a plan; any output pointer may be NULL.    */
srht_status srht_plan_info(const srht_plan* plan, int64_t* N, int64_t* r,
                           int64_t* batch);

/* Kept rows of problem p, ascending, into host memory (r int32 values).     */
srht_status srht_plan_copy_indices(const srht_plan* plan, int64_t problem,
                                   int32_t* host_K);

/* Sign words of problem p into host memory: ceil(N/64) uint64 words, bit
 * (i mod 64) of word i/64 set iff sigma_i = -1.                              */
srht_status srht_plan_copy_signs(const srht_plan* plan, int64_t problem,
                                 uint64_t* host_words);

/* Device scratch bytes needed by srht_sketch* for `ncols` columns: the
 * per-slab partial sums that the fixed-order slab reduction finishes (the
 * dense TMA kernel always writes them, in its slot order, even for a single
 * slab; 0 when no path needs them).  The workspace must be 256-byte aligned. */
size_t srht_workspace_bytes(const srht_plan* plan, int64_t ncols);

/* Sketch one problem: SA (r x A->cols, column-major, ldsa >= r) = H~ D A and
 * Sb (r) = H~ D b (Algorithm 1 step 5 inputs).  A->rows and b->rows
 * must equal the plan's n; b must have exactly one column.  b may be NULL
 * (then Sb is ignored).  A and b may be dense or CSC independently.          */
srht_status srht_sketch(const srht_plan* plan, const srht_matrix* A,
                        const srht_matrix* b, float* SA, int64_t ldsa,
                        float* Sb, void* workspace, size_t workspace_bytes,
                        void* stream);

/* Sketch every column of M (rows == n, any column count) into SM (r x cols,
 * ldsm >= r).  Columns are independent, so a column range of [A | b] is the
 * multi-GPU shard primitive; results do not depend on the range (the tile and
 * slab geometry depend only on n and r).                                     */
srht_status srht_sketch_columns(const srht_plan* plan, const srht_matrix* M,
                                float* SM, int64_t ldsm, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Column shard with the gather fused in (replaces the NCCL all-gather): the sketch of
 * M's columns (the same values srht_sketch_columns writes) is stored at columns [col0, col0 +
 * M->cols) of EVERY buffer peers[0..n_peers) (column-major, ld ldp >= r; 1 <= n_peers <= 8).
 * peers[0] is this rank's own r x c output; peers[1..] are the other ranks' outputs mapped into this
 * process (CUDA IPC handles or peer access over NVLink).  On the dense TMA path the slab reduction
 * kernel itself stores every output element into all peers (one kernel: reduce + gather over peer
 * memory); other paths write peers[0] and one copy kernel stores the block into the others.  The
 * caller orders the ranks (stream sync + barrier) before reading.  `peers` is a HOST array of device
 * pointers.  EINVAL on bad arguments (null pointers, n_peers out of range, ldp < r, col0 < 0).
 * Asynchronous on `stream`.                                                  */
srht_status srht_sketch_columns_peers(const srht_plan* plan, const srht_matrix* M,
                                      int64_t col0, float* const* peers,
                                      int n_peers, int64_t ldp, void* workspace,
                                      size_t workspace_bytes, void* stream);

/* Buffers for srht_sketch_columns_peers shared across processes (CUDA IPC):
 * srht_ipc_alloc: device allocation of `bytes` on the current device and its 64-byte IPC handle
 * (written to `handle`, host memory) for the other ranks; srht_ipc_open: map another process's
 * allocation from its handle (peer access enabled lazily; NVLink between GPUs); srht_ipc_close:
 * unmap it; srht_ipc_free: free an srht_ipc_alloc buffer (NULL: no-op).  Synchronous.      */
srht_status srht_ipc_alloc(size_t bytes, void** dev_ptr, void* handle);
srht_status srht_ipc_open(const void* handle, void** dev_ptr);
srht_status srht_ipc_close(void* dev_ptr);
srht_status srht_ipc_free(void* dev_ptr);

/* Batched mode: M has batch*c columns (problem p owns columns p*c .. p*c+c-1,
 * c = M->cols / batch); output SM is batch blocks of r x c, column-major and
 * contiguous (column g of M lands at SM + g*r).  Problem p uses its own plan.  */
srht_status srht_sketch_batched(const srht_plan* plan, const srht_matrix* M,
                                float* SM, void* workspace,
                                size_t workspace_bytes, void* stream);

/* ---- Row shards (data partitioned by rows across ranks) ----
 * srht_row_shard_rows: the row granularity G of row shards for this plan (a
 * power of two: the slab size of the kernels).
 * srht_sketch_rows_partial: M holds rows [row0, row0 + M->rows) of the n-row
 * matrix [A | b] (all of its columns); row0 must be a multiple of G and the
 * shard must end at a multiple of G or at n.  Dense M is column-major with
 * M->rows rows (ld >= M->rows); CSC M carries GLOBAL row indices in
 * [row0, row0 + M->rows).  Writes the UNSCALED partial sums over these rows,
 *     part[t + j*ldp] = sum_{row0 <= i < row0+rows} (-1)^{popc(k_t & i)} sigma_i M[i, j]
 * in FP64 (ldp >= r), for every column j.  By linearity the sketch is
 * r^{-1/2} * (sum of the partials of a row partition), e.g. after one
 * all-reduce (paper_0812_4547_b200.dist.sketch_row_sharded).  Single-problem
 * plans only; EINVAL otherwise or on misaligned shards.  Workspace as for
 * srht_sketch (srht_workspace_bytes covers both).  Asynchronous on `stream`. */
int64_t srht_row_shard_rows(const srht_plan* plan);
srht_status srht_sketch_rows_partial(const srht_plan* plan,
                                     const srht_matrix* M, int64_t row0,
                                     double* part, int64_t ldp,
                                     void* workspace, size_t workspace_bytes,
                                     void* stream);

/* Finish of a row partition (the step after the all-reduce of the partials):
 *     SM[t + j*ldsm] = (float)(part[t + j*ldp] * r^{-1/2}),   t < r, j < cols,
 * i.e. Algorithm 1's scale sqrt(N/r) on the normalized H_N/sqrt(N) (P:298,
 * P:166-168), applied once in FP64 to the summed FP64 partials, then one
 * rounding to FP32 -- the same arithmetic as the single-GPU slab reduction, so
 * a row-sharded sketch equals srht_sketch_columns up to the FP64 association
 * order of the partial sums.  `part` (FP64, ldp >= r) and SM (FP32, ldsm >= r)
 * are device pointers owned by the caller; r is the plan's kept count and the
 * scale uses the requested r (Bernoulli plans).  EINVAL on null pointers,
 * cols < 0 or short leading dimensions.  Asynchronous on `stream`.          */
srht_status srht_rows_finish(const srht_plan* plan, const double* part,
                             int64_t ldp, int64_t cols, float* SM,
                             int64_t ldsm, void* stream);

/* ---- Gram matrices of sketches: the QP form of Section 3.4 ----
 * For p < batch: G_p = SM_p^T SM_p (c x c, FP64, column-major, both triangles,
 * G_p[i + j*ldg] at G + p*stride_g, ldg >= c) where SM_p is the r x c FP32
 * column-major block at SM + p*stride_sm (ldsm >= r; for batch > 1 the strides
 * must separate the blocks).  With SM_p = [SA | Sb] (srht_sketch*):
 *     G_p = [[Q~, q~], [q~^T, Sb^T Sb]],  Q~ = (H~DA)^T H~DA,  q~ = (H~DA)^T H~Db,
 * so min_{x>=0} ||SA x - Sb||^2 = min x^T Q~ x - 2 q~^T x + Sb^T Sb.  Products of
 * the FP32 entries are exact in FP64 and accumulated in FP64.  All pointers are
 * device pointers; asynchronous on `stream` (cudaStream_t as void*).         */
srht_status srht_gram(int64_t r, int64_t c, int64_t batch, const float* SM,
                      int64_t ldsm, int64_t stride_sm, double* G, int64_t ldg,
                      int64_t stride_g, void* stream);

/* srht_gram with caller-provided scratch (no allocation inside the call).  The products run on
 * the FP64 tensor cores (DMMA, exact FP32 products, FP64 sums) over 64 x 64 block pairs of the
 * upper triangle; when a problem has few block pairs the rows are split into K ranges whose
 * partial blocks are summed in a fixed order (deterministic).  srht_gram_workspace_bytes: the
 * bytes those partials need (0: none); the workspace must be 256-byte aligned (its contents
 * on entry do not matter).  srht_gram allocates the same scratch stream-ordered per call.     */
size_t srht_gram_workspace_bytes(int64_t r, int64_t c, int64_t batch);
srht_status srht_gram_ex(int64_t r, int64_t c, int64_t batch, const float* SM,
                         int64_t ldsm, int64_t stride_sm, double* G, int64_t ldg,
                         int64_t stride_g, void* workspace, size_t workspace_bytes,
                         void* stream);

/* ---- NNLS on the Gram form (Algorithm 1 step 5, via P:570-590) ----
 * For p < batch: x_p = argmin_{x >= 0} x^T Q x - 2 q^T x, i.e. the NNLS solution
 * of min ||SA x - Sb|| when G_p = [[Q, q], [q^T, .]] = srht_gram([SA | Sb]) is
 * (d+1) x (d+1) FP64 column-major at G + p*stride_g (ldg >= d+1).  Lawson-Hanson
 * active set with the oracle's rules (reading R13: argmax dual entry,
 * smallest-index ties, tol 1e-10 max|q|, degenerate entries skipped, <= 30 d
 * outer iterations, x < 1e-14 snapped to 0); the passive-set solve is a
 * Cholesky factorization of Q_PP (needs a full-column-rank SA, the generic case
 * for r >= d+1).  x_p (d FP64) at x + p*stride_x; iters[p] (device, may be NULL)
 * = outer iterations, or -1 (iteration cap), -2 (inner loop cap), -3 (Q_PP not
 * positive definite).  One CTA per problem; the factor is updated
 * incrementally (append / delete with Givens rotations), in shared memory for
 * d <= 156, else in the workspace (two d x d FP64 slots per problem, row-major,
 * blocked 32-row triangular solves; srht_nnls_workspace_bytes; 0 for d <= 156),
 * 8-byte aligned.
 * Device pointers; asynchronous on `stream`.                                  */
size_t srht_nnls_workspace_bytes(int64_t d, int64_t batch);
srht_status srht_nnls_gram(int64_t d, int64_t batch, const double* G,
                           int64_t ldg, int64_t stride_g, double* x,
                           int64_t stride_x, int32_t* iters, void* workspace,
                           size_t workspace_bytes, void* stream);

/* ---- NNLS on the Gram form by block principal pivoting (same problem, faster for large d) ----
 * Same inputs, outputs and iters codes as srht_nnls_gram (Algorithm 1 step 5 via the QP form,
 * P:311-314 and P:570-590) -- "any standard NNLS solver": the optimum of a
 * full-column-rank SA is unique, so both solvers return it up to FP64 rounding.  Method
 * (Portugal, Judice & Vicente 1994; Kim & Park 2011): with F the passive set, x_F solves
 * Q_FF x_F = q_F, y = Q x - q; the infeasible set V = {i in F: x_i < 0} U {i not in F:
 * y_i < -tol} (tol = 1e-10 max|q|, the Lawson-Hanson stopping rule) is exchanged whole while
 * |V| decreases (3 extra tries), else only its largest index; V empty is the KKT point.  Each
 * step refactors Q_FF (Cholesky); iters[p] = exchange steps, or -1 (cap of 10 d + 10 steps),
 * -3 (Q_FF not positive definite).  One CTA per problem; a single problem with d >= 128 runs on a
 * thread-block cluster of 16 (else 8) SMs (factorization, panel solves and the dual split over the
 * cluster).  d <= 580 (EUNSUPPORTED above).  Workspace: srht_nnls_bpp_workspace_bytes (d x d FP64
 * per problem, plus O(d) vectors for a single problem), 8-byte aligned.
 * Device pointers; asynchronous on `stream`.                                  */
size_t srht_nnls_bpp_workspace_bytes(int64_t d, int64_t batch);
srht_status srht_nnls_gram_bpp(int64_t d, int64_t batch, const double* G,
                               int64_t ldg, int64_t stride_g, double* x,
                               int64_t stride_x, int32_t* iters, void* workspace,
                               size_t workspace_bytes, void* stream);

/* ---- Algorithm 2, SubspaceSampling ----
 * Row i of Phi (n x d, FP32 column-major, ldphi >= n) is kept with probability
 * q_i = min(1, r p_i) (p: n FP64 probabilities) and scaled by 1/sqrt(q_i): kept
 * iff q_i >= 1 or u_i < floor(q_i 2^64), u_i = word i of the Philox stream
 * (seed, 1) -- the coins of SRHT_PLAN_BERNOULLI, so p_i = 1/N applied to
 * H_N D [M; 0] / sqrt(N) is the Bernoulli SRHT sketch.
 * srht_subspace_sample_count: the number of kept rows into *kept (host;
 * synchronous on `stream`).  srht_subspace_sample: kept row indices, ascending,
 * into K (device int32, capacity cap) and the scaled rows into out (cap x d,
 * ldout >= cap); rows beyond cap are dropped.  Temporaries are allocated
 * stream-ordered (cudaMallocAsync).                                          */
srht_status srht_subspace_sample_count(int64_t n, int64_t r, uint64_t seed,
                                       const double* p, int64_t* kept,
                                       void* stream);
srht_status srht_subspace_sample(int64_t n, int64_t d, int64_t r, uint64_t seed,
                                 const double* p, const float* Phi,
                                 int64_t ldphi, int32_t* K, float* out,
                                 int64_t ldout, int64_t cap, void* stream);

/* Same as srht_sketch_columns, but M's values, column pointers, row indices
 * and SM are HOST buffers (pinned or pageable).  Host->device copies, the
 * sketch and the device->host copy run inside the call, pipelined over column
 * chunks on internal streams; returns after SM is written (synchronous).
 * Device memory is allocated internally per call.                            */
srht_status srht_sketch_columns_host(const srht_plan* plan,
                                     const srht_matrix* M_host, float* SM_host,
                                     int64_t ldsm);

const char* srht_status_str(srht_status s);

/* ---- Profiling (benchmark instrumentation) ----
 * srht_profile_start(capacity): from now on, every srht_sketch* call records a
 * pair of CUDA events on its own stream immediately around the main tile
 * kernel (k_sketch_tiles), for up to `capacity` calls (later calls are not
 * recorded).  srht_profile_stop(ms, capacity, &count): waits for the recorded
 * events, writes the per-call tile-kernel durations in milliseconds to host
 * array `ms` (up to `capacity` values), sets *count, frees the events and
 * disables recording.  Process-global and not thread-safe; EINVAL if
 * start is called twice without stop or capacity < 1.                        */
srht_status srht_profile_start(int capacity);
srht_status srht_profile_stop(float* ms, int capacity, int* count);

/* ---- Workload generator (benchmark / test input only; not the method) ----
 * out[i + j*ld] = (word i of stream (seed, 2^32 + stream0 + j) >> 40) * 2^-24,
 * i.e. exact FP32 Uniform[0,1) values from the same Philox stream convention,
 * for i < rows, j < cols (device pointer, async on stream).                 */
srht_status srht_gen_uniform(uint64_t seed, uint64_t stream0, int64_t rows,
                             int64_t cols, float* out, int64_t ld,
                             void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SRHT_H_ */
