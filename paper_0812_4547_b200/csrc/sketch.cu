// SRHT sketch kernels for sm_100a.
//
// Output (Algorithm 1 step 5 inputs; Phi of P:461-465):
//   SM[t, j] = r^{-1/2} * sum_{i<n} (-1)^{popc(k_t & i)} sigma_i M[i, j].
//
// Decomposition (Ailon-Liberty-style pruning).  Split a row index
// i = (i_slab, i_mid, i_lo) with i_lo the low b bits (tile of B = 2^b rows),
// i_mid the next log J bits (sub-block inside a slab) and i_slab the rest; the
// same split of a kept row k gives (k_slab, k_mid, k_lo).  Because
// popc(k & i) = popc(k_lo & i_lo) + popc(k_mid & i_mid) + popc(k_slab & i_slab),
//
//   SM[t] = r^{-1/2} sum_s (-1)^{popc(k_slab & s)}
//                      sum_j (-1)^{popc(k_mid & j)} (H_B D x_{s,j})[k_lo],
//
// so a CTA streams the sub-blocks x_{s,j} of one (column, slab), transforms
// each tile completely on chip (z = H_B D x, b stages), and accumulates only
// the r sampled entries z[k_lo(t)] with the k_mid sign: ~b + r/B adds per
// element instead of log2 N.  The slab sum (k_slab signs, r^{-1/2}) is done by
// k_reduce_slabs in a fixed order, so results do not depend on how columns are
// split across launches or GPUs.
//
// In-tile FWHT of B = 2^b FP32 values by T = B/32 threads, 32 values each,
// in 2-3 rounds of up to 5 bits (registers) with XOR-swizzled shared-memory
// exchanges in between; butterflies use packed FADD2/FFMA2 (sm_100).
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.cuh"

namespace srht {
namespace {

// Bank-conflict-free swizzle of the tile: word x lives at phys(x).  It is
// linear over GF(2), so phys(base | off) = phys(base) ^ phys(off).
__host__ __device__ constexpr int phys(int x) { return x ^ ((x >> 5) & 31); }

// Round 2 register bit k (LOG_B > 10): bits 7.. are transformed, the rest fill.
__host__ __device__ constexpr int reg2_bit(int LOG_B, int k) {
  return k < LOG_B - 10 ? 7 + k
                        : (k - (LOG_B - 10) == 0   ? LOG_B - 3
                           : k - (LOG_B - 10) == 1 ? LOG_B - 2
                           : k - (LOG_B - 10) == 2 ? LOG_B - 1
                           : k - (LOG_B - 10) == 3 ? 6
                                                   : 5);
}

template <int LOG_B>
__host__ __device__ constexpr int off0(int u) {  // round 0: bits {0,1,b-3,b-2,b-1}
  return (u & 3) | ((u >> 2) << (LOG_B - 3));
}
__host__ __device__ constexpr int off1(int u) { return u << 2; }  // round 1: bits 2..6
template <int LOG_B>
__host__ __device__ constexpr int off2(int u) {
  return (((u >> 0) & 1) << reg2_bit(LOG_B, 0)) | (((u >> 1) & 1) << reg2_bit(LOG_B, 1)) |
         (((u >> 2) & 1) << reg2_bit(LOG_B, 2)) | (((u >> 3) & 1) << reg2_bit(LOG_B, 3)) |
         (((u >> 4) & 1) << reg2_bit(LOG_B, 4));
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }

// Unnormalized Walsh-Hadamard butterflies over the low NB bits of the register
// index u (value u lives in v[u >> 1].x / .y).  Natural order: (a, b) -> (a+b, a-b).
template <int NB>
__device__ __forceinline__ void fwht_regs(float2 (&v)[16]) {
  if constexpr (NB >= 1) {
#pragma unroll
    for (int m = 0; m < 16; ++m)  // within-pair bit: one FFMA2 per pair
      v[m] = __ffma2_rn(v[m], make_float2(1.f, -1.f), make_float2(v[m].y, v[m].x));
  }
#pragma unroll
  for (int s = 1; s < NB; ++s) {
    const int st = 1 << (s - 1);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      if (!(m & st)) {
        const float2 a = v[m], b = v[m | st];
        v[m] = add2(a, b);
        v[m | st] = sub2(a, b);
      }
    }
  }
}

__device__ __forceinline__ float flip(float x, uint32_t bit) {
  return __uint_as_float(__float_as_uint(x) ^ (bit << 31));
}

// RPT = 32: the sample metadata lives in shared memory (re-read per tile, conflict-free)
// instead of 32 registers, so the kernel fits its register budget without spilling.
#ifndef V1_META_SMEM
#define V1_META_SMEM 1
#endif
template <int RPT>
__host__ __device__ constexpr bool meta_in_smem() { return V1_META_SMEM && RPT == 32; }
#ifndef V1_CSC_STAGE
#define V1_CSC_STAGE 1024  // CSC entries staged in shared memory per CTA (>= threads per CTA)
#endif

#ifndef V1_THREADS_PER_SM
#define V1_THREADS_PER_SM 512
#endif
template <int LOG_B, int RPT>
#ifndef V1_TPS_OTHER
#define V1_TPS_OTHER 512  // threads per SM the register budget targets when RPT != 32
#endif
__global__ void __launch_bounds__((1 << LOG_B) / 32, (meta_in_smem<RPT>() ? V1_THREADS_PER_SM : V1_TPS_OTHER) / ((1 << LOG_B) / 32))
    k_sketch_tiles(const __grid_constant__ SketchParams P) {
  constexpr int B = 1 << LOG_B;
  constexpr int T = B / 32;
  extern __shared__ __align__(16) float tile[];
  __shared__ int64_t s_ptr;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- decode the work item: (column, slab, sample group) ----
  int64_t item = blockIdx.x;
  const int64_t g = item % P.groups;
  item /= P.groups;
  const int64_t sl = item % P.S_act;  // slab of this launch
  const int64_t s = P.s_lo + sl;      // global slab
  const int64_t col = item / P.S_act;
  const bool second = col >= P.ncols0;
  const ColSrc& cs = second ? P.src[1] : P.src[0];
  const int64_t lc = second ? col - P.ncols0 : col;
  const int64_t prob = col / P.cols_per_problem;
  const uint32_t* __restrict__ signs = P.signs + prob * P.words32;
  const int32_t* __restrict__ Kp = P.K + prob * P.r;

  // ---- per-thread bases of the three exchange layouts (swizzled) ----
  const int pb0 = phys((lane << 2) | (warp << 7));
  const int pb1 = phys((lane & 3) | ((lane >> 2) << 7) | (warp << 10));
  int b2 = lane;
  {
    int w = warp, k = 0;
    for (int bit = 5; bit < LOG_B; ++bit) {
      bool is_reg = false;
#pragma unroll
      for (int q = 0; q < 5; ++q) is_reg |= (reg2_bit(LOG_B, q) == bit);
      if (LOG_B > 10 && !is_reg) {
        b2 |= ((w >> k) & 1) << bit;
        ++k;
      }
    }
  }
  const int pb2 = phys(b2);

  // ---- sample metadata: byte offset of phys(k_lo) | k_mid << 16 ----
  constexpr bool MS = meta_in_smem<RPT>();
  uint32_t meta[MS ? 1 : RPT];
  uint32_t* meta_s = reinterpret_cast<uint32_t*>(tile + B);  // [RPT][T] when MS
  float acc[RPT];
  const int64_t t0 = g * (int64_t)RPT * T;
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int64_t t = t0 + (int64_t)q * T + tid;
    uint32_t m = 0;
    if (t < P.r) {
      const int32_t k = Kp[t];
      const int lo = k & (B - 1);
      const uint32_t mid = (uint32_t)(k >> LOG_B) & (uint32_t)(P.J - 1);
      m = ((uint32_t)phys(lo) << 2) | (mid << 16);
    }
    if constexpr (MS) meta_s[q * T + tid] = m; else meta[q] = m;
    acc[q] = 0.f;
  }

  const int64_t j0 = s * P.J;
  const int64_t j1 = (j0 + P.J < P.n_sub) ? j0 + P.J : P.n_sub;
  const int64_t n = P.n;

  // CSC: the slab's entries [gbase, gend) are staged in shared memory (row, signed value), up to
  // V1_CSC_STAGE at a time, so the per-tile scatter reads no global memory (config 3: the per-tile
  // global loads put a DRAM round trip on every tile's critical path)
  __shared__ int64_t s_end;
  int* srow = reinterpret_cast<int*>(meta_s + (MS ? RPT * T : 0));
  float* sval = reinterpret_cast<float*>(srow + V1_CSC_STAGE);
  int64_t cptr = 0, gbase = 0, gend = 0;
  int nst = 0;
  auto stage = [&](int64_t from) {
    gbase = from;
    const int64_t left = gend - from;
    nst = (int)(left < V1_CSC_STAGE ? left : V1_CSC_STAGE);
    for (int i = tid; i < nst; i += T) {
      const int row = cs.rowidx[from + i];
      srow[i] = row;
      sval[i] = flip(cs.vals[from + i], (__ldg(signs + (row >> 5)) >> (row & 31)) & 1u);
    }
  };
  if (cs.fmt == SRHT_CSC) {
    if (tid < 2) {  // lower_bound(rowidx, slab start / slab end)
      int64_t lo = cs.colptr[lc], hi = cs.colptr[lc + 1];
      const int64_t target = (tid == 0 ? j0 : j1) * (int64_t)B;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)cs.rowidx[mid] < target) lo = mid + 1; else hi = mid;
      }
      if (tid == 0) s_ptr = lo; else s_end = lo;
    }
    __syncthreads();
    cptr = s_ptr;
    gend = s_end;
    stage(cptr);
  }

  for (int64_t j = j0; j < j1; ++j) {
    const int64_t row0 = j * (int64_t)B;
    float2 v[16];
    // ---- round 0: load D x (bits 0,1 and the top three bits in registers) ----
    if (cs.fmt == SRHT_DENSE) {
      const float* __restrict__ colp = cs.vals + lc * cs.ld;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const int64_t row = row0 + ((lane << 2) | (warp << 7) | (h << (LOG_B - 3)));
        float4 f;
        if (cs.vec && row + 3 < n) {
          f = __ldcs(reinterpret_cast<const float4*>(colp + row));
        } else {
          f.x = row + 0 < n ? colp[row + 0] : 0.f;
          f.y = row + 1 < n ? colp[row + 1] : 0.f;
          f.z = row + 2 < n ? colp[row + 2] : 0.f;
          f.w = row + 3 < n ? colp[row + 3] : 0.f;
        }
        const uint32_t sw = __ldg(signs + (row >> 5)) >> (row & 31);
        v[2 * h] = make_float2(flip(f.x, sw & 1u), flip(f.y, (sw >> 1) & 1u));
        v[2 * h + 1] = make_float2(flip(f.z, (sw >> 2) & 1u), flip(f.w, (sw >> 3) & 1u));
      }
    } else {
      // CSC: densify the sub-block into the tile from the staged entries, then read it.
#pragma unroll
      for (int i = tid; i < B / 4; i += T) reinterpret_cast<float4*>(tile)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncthreads();
      const int rowend = (int)(row0 + B);
      while (true) {
        if (cptr + T > gbase + nst && gbase + nst < gend) {  // uniform: restage from cptr
          stage(cptr);
          __syncthreads();
        }
        const int64_t e = cptr + tid;
        bool in = false;
        if (e < gbase + nst) {
          const int row = srow[e - gbase];
          if (row < rowend) {
            in = true;
            atomicAdd(&tile[phys(row - (int)row0)], sval[e - gbase]);  // duplicates are summed
          }
        }
        const int cnt = __syncthreads_count(in);
        cptr += cnt;
        if (cnt < T) break;
      }
#pragma unroll
      for (int u = 0; u < 32; u += 2) v[u >> 1] = make_float2(tile[pb0 ^ phys(off0<LOG_B>(u))],
                                                             tile[pb0 ^ phys(off0<LOG_B>(u + 1))]);
    }
    fwht_regs<5>(v);
#pragma unroll
    for (int u = 0; u < 32; u += 2) {
      tile[pb0 ^ phys(off0<LOG_B>(u))] = v[u >> 1].x;
      tile[pb0 ^ phys(off0<LOG_B>(u + 1))] = v[u >> 1].y;
    }
    __syncthreads();
    // ---- round 1: bits 2..6 ----
#pragma unroll
    for (int u = 0; u < 32; u += 2)
      v[u >> 1] = make_float2(tile[pb1 ^ phys(off1(u))], tile[pb1 ^ phys(off1(u + 1))]);
    fwht_regs<5>(v);
#pragma unroll
    for (int u = 0; u < 32; u += 2) {
      tile[pb1 ^ phys(off1(u))] = v[u >> 1].x;
      tile[pb1 ^ phys(off1(u + 1))] = v[u >> 1].y;
    }
    __syncthreads();
    // ---- round 2: bits 7 .. b-4 ----
    if constexpr (LOG_B > 10) {
#pragma unroll
      for (int u = 0; u < 32; u += 2)
        v[u >> 1] = make_float2(tile[pb2 ^ phys(off2<LOG_B>(u))], tile[pb2 ^ phys(off2<LOG_B>(u + 1))]);
      fwht_regs<LOG_B - 10>(v);
#pragma unroll
      for (int u = 0; u < 32; u += 2) {
        tile[pb2 ^ phys(off2<LOG_B>(u))] = v[u >> 1].x;
        tile[pb2 ^ phys(off2<LOG_B>(u + 1))] = v[u >> 1].y;
      }
      __syncthreads();
    }
    // ---- pruned accumulate: acc_t += (-1)^{popc(k_mid & j)} z[k_lo] ----
    const uint32_t jl = (uint32_t)(j - j0);
    const char* tb = reinterpret_cast<const char*>(tile);
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      uint32_t m;
      if constexpr (MS) m = meta_s[q * T + tid]; else m = meta[q];
      const float z = *reinterpret_cast<const float*>(tb + (m & 0xffffu));
      acc[q] += flip(z, __popc((m >> 16) & jl) & 1u);
    }
    __syncthreads();
  }

  // ---- epilogue ----
  if (P.S_act == 1 && !P.part_out) {
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int64_t t = t0 + (int64_t)q * T + tid;
      if (t < P.r) cs.out[lc * cs.ldo + t] = acc[q] * P.scale;
    }
  } else {
    float* __restrict__ part = P.partials + (sl * P.total_cols + col) * P.r;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int64_t t = t0 + (int64_t)q * T + tid;
      if (t < P.r) part[t] = acc[q];
    }
  }
}

// Fixed-order signed sum over slabs, scale, and write (one thread per output).
__global__ void k_reduce_slabs(const __grid_constant__ SketchParams P, int slab_shift) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t col = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (t >= P.r || col >= P.total_cols) return;
  const int64_t prob = col / P.cols_per_problem;
  const uint32_t ks = (uint32_t)(P.K[prob * P.r + t] >> slab_shift);
  // FP32 slab partials, summed in FP64 (fixed order) and scaled by r^{-1/2} once
  // before the single rounding to FP32 (reading R10).
  double sum = 0.0;
  for (int64_t s = 0; s < P.S_act; ++s) {
    const float v = P.partials[(s * P.total_cols + col) * P.r + t];
    sum += (double)flip(v, __popc(ks & (uint32_t)(P.s_lo + s)) & 1u);
  }
  if (P.part_out) {  // row shard: unscaled partial, summed across shards by the caller
    P.part_out[col * P.ldp + t] = sum;
    return;
  }
  const bool second = col >= P.ncols0;
  const ColSrc& cs = second ? P.src[1] : P.src[0];
  const int64_t lc = second ? col - P.ncols0 : col;
  cs.out[lc * cs.ldo + t] = (float)(sum * P.scale_f64);
}

template <int LOG_B, int RPT>
cudaError_t launch_t(const SketchParams& sp, int64_t items, cudaStream_t stream) {
  constexpr int B = 1 << LOG_B;
  const size_t smem = (size_t)B * sizeof(float) + (meta_in_smem<RPT>() ? (size_t)RPT * (B / 32) * 4 : 0) +
                      (size_t)V1_CSC_STAGE * 8;
  static std::atomic<uint64_t> attr_done{0};
  const cudaError_t e = set_max_dyn_smem_once(k_sketch_tiles<LOG_B, RPT>, (int)smem, attr_done);
  if (e != cudaSuccess) return e;
  for (int64_t done = 0; done < items;) {
    // one launch covers at most 2^31-1 items (never reached in practice)
    const int64_t cnt = items - done < 0x7fffffff ? items - done : 0x7fffffff;
    k_sketch_tiles<LOG_B, RPT><<<(unsigned)cnt, B / 32, smem, stream>>>(sp);
    done += cnt;
  }
  return cudaGetLastError();
}

template <int LOG_B>
cudaError_t launch_b(int rpt, const SketchParams& sp, int64_t items, cudaStream_t stream) {
  switch (rpt) {
    case 4: return launch_t<LOG_B, 4>(sp, items, stream);
    case 8: return launch_t<LOG_B, 8>(sp, items, stream);
    case 16: return launch_t<LOG_B, 16>(sp, items, stream);
    case 32: return launch_t<LOG_B, 32>(sp, items, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

ProfileState g_prof;
int g_debug_mode = 0;
int g_kernel_force = 0;
int g_last_kernel = 0;
unsigned long long* g_debug_trace = nullptr;

namespace {
// ---------------------------------------------------------------------------------------
// Whole-column kernel for N = 2^13 (config 2's batched CSC problems): one CTA of 256 threads
// transforms a full column (8192 rows) in three register rounds of 5 + 5 + 3 bits, then
// gathers the r kept rows of z = H_N D x.  Against the tiled kernel (8 tiles of 1024 rows,
// one warp each, plus the pruned accumulate over the tiles) this halves the instructions
// per column and runs 8 warps per CTA.  The tile is padded (word x at x + x/32), which
// keeps every round's shared-memory accesses conflict-free with immediate offsets.
constexpr int COL_N = 1 << 13, COL_T = 256;
__device__ __forceinline__ int cpad(int x) { return x + (x >> 5); }
// Zero source for the tile fill: a bulk copy (TMA engine) instead of 264 wavefronts of STS on
// the LSU data path, which bounds this kernel.  Device globals start zeroed.
__device__ __align__(128) float g_col_zeros[COL_N + COL_N / 32];
#ifndef COL_TMA_ZERO
#define COL_TMA_ZERO 1
#endif

#ifndef COL_MINB
#define COL_MINB 5
#endif
__global__ void __launch_bounds__(COL_T, COL_MINB) k_sketch_col(const __grid_constant__ SketchParams P) {
  __shared__ __align__(16) float tile[COL_N + COL_N / 32];
  const int tid = threadIdx.x;
  const int64_t col = blockIdx.x + (int64_t)blockIdx.y * 65535;
  if (col >= P.total_cols) return;
  const bool second = col >= P.ncols0;
  const ColSrc& cs = second ? P.src[1] : P.src[0];
  const int64_t lc = second ? col - P.ncols0 : col;
  const int64_t prob = col / P.cols_per_problem;
  const uint32_t* __restrict__ signs = P.signs + prob * P.words32;
  const int32_t* __restrict__ Kp = P.K + prob * P.r;
  const int n = (int)P.n;
  // kept rows of the pruned last three bits (plan gather order), loaded now: their latency is
  // hidden behind the tile's fill and rounds A and B
  constexpr int ZPT = COL_SLOTS / COL_T;  // kept-row slots per thread
  const bool pruned = P.colk && P.r <= 4 * COL_T;
  uint32_t ckw[ZPT];
#pragma unroll
  for (int q = 0; q < ZPT; ++q)
    ckw[q] = pruned ? __ldg(P.colk + prob * COL_SLOTS + tid + COL_T * q) : 0xffffffffu;
  // ---- D x into the padded tile (rows >= n stay 0) ----
  if (cs.fmt == SRHT_CSC) {
    // The zero fill (bulk copy from a zeroed L2-resident buffer: no LSU wavefronts) is issued
    // first, and each thread's first CSC entry (row, value, neighbours' rows, sign word) is
    // loaded while it lands, so the two latencies overlap.
    __shared__ __align__(8) uint64_t zbar;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&zbar);
    if (COL_TMA_ZERO && tid == 0) {
      constexpr uint32_t bytes = (COL_N + COL_N / 32) * 4;
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(tile)),
                   "l"(g_col_zeros), "r"(bytes), "r"(bar)
                   : "memory");
    }
    const int64_t cbeg = cs.colptr[lc], cend = cs.colptr[lc + 1];
    const int64_t e0 = cbeg + tid;
    int r0 = -1, rprev = -1, rnext = -1;
    float v0 = 0.f;
    uint32_t sw0 = 0u;
    if (e0 < cend) {
      r0 = cs.rowidx[e0];
      v0 = cs.vals[e0];
      if (e0 > cbeg) rprev = cs.rowidx[e0 - 1];
      if (e0 + 1 < cend) rnext = cs.rowidx[e0 + 1];
      sw0 = __ldg(signs + (r0 >> 5));
    }
    if (COL_TMA_ZERO) {
      __syncthreads();  // the barrier is initialised before anyone waits on it
      asm volatile(
          "{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra W_%=;\n}" ::"r"(bar)
          : "memory");
    } else {
      for (int i = tid; i < (COL_N + COL_N / 32) / 4; i += COL_T)
        reinterpret_cast<float4*>(tile)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncthreads();
    }
    // scatter D x: rows are sorted within a column, so duplicates are adjacent; the first entry of
    // each run of equal rows sums the run (in entry order: deterministic) and stores it once.
    // (Shared FP32 atomicAdd compiles to a CAS loop: ncu put 13% of this kernel's shared-memory
    // wavefronts in it.)
    if (e0 < cend && rprev != r0) {
      float v = v0;
      if (rnext == r0)
        for (int64_t e2 = e0 + 1; e2 < cend && cs.rowidx[e2] == r0; ++e2) v += cs.vals[e2];
      tile[cpad(r0)] = flip(v, (sw0 >> (r0 & 31)) & 1u);
    }
    for (int64_t e = e0 + COL_T; e < cend; e += COL_T) {
      const int row = cs.rowidx[e];
      if (cs.rowidx[e - 1] == row) continue;  // not the first of its run
      float v = cs.vals[e];
      for (int64_t e2 = e + 1; e2 < cend && cs.rowidx[e2] == row; ++e2) v += cs.vals[e2];
      const uint32_t sb = (__ldg(signs + (row >> 5)) >> (row & 31)) & 1u;
      tile[cpad(row)] = flip(v, sb);
    }
  } else {
    const float* __restrict__ colp = cs.vals + lc * cs.ld;
    for (int x = tid; x < COL_N; x += COL_T) {
      const uint32_t sb = (__ldg(signs + (x >> 5)) >> (x & 31)) & 1u;
      tile[cpad(x)] = x < n ? flip(colp[x], sb) : 0.f;
    }
  }
  __syncthreads();
  float2 v[16];
  // ---- round A: bits 0..4 in registers; thread = bits 5..12.  x = 32 tid + u ----
  {
    float* base = tile + cpad(tid << 5);
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = make_float2(base[2 * m], base[2 * m + 1]);
    fwht_regs<5>(v);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      base[2 * m] = v[m].x;
      base[2 * m + 1] = v[m].y;
    }
  }
  __syncthreads();
  // ---- round B: bits 5..9; thread = bits 0..4 | bits 10..12 << 5.  x = lane + 32 u + 1024 h ----
  {
    float* base = tile + cpad((tid & 31) | ((tid >> 5) << 10));
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = make_float2(base[33 * (2 * m)], base[33 * (2 * m + 1)]);
    fwht_regs<5>(v);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      base[33 * (2 * m)] = v[m].x;
      base[33 * (2 * m + 1)] = v[m].y;
    }
  }
  __syncthreads();
  if (pruned) {
    // ---- pruned last three row bits: only the kept rows of z are formed.  Kept row
    // k = lo | hi << 10 needs z[k] = sum_j (-1)^popc(hi & j) y[lo + 1024 j] (y = the tile after
    // rounds A and B): eight reads and seven adds instead of round C over all 8192 rows plus the
    // gather.  The plan's gather order (d_colk, 5 slots per thread) puts distinct banks in each
    // warp-wide step where the bank counts allow. ----
    float zr[ZPT];
    int zd[ZPT];
#pragma unroll
    for (int q = 0; q < ZPT; ++q) {
      zd[q] = -1;
      zr[q] = 0.f;
      if (ckw[q] != 0xffffffffu) {
        const uint32_t w = ckw[q];
        const int k = (int)(w & 0xffffu), lo = k & 1023;
        const uint32_t hi = (uint32_t)k >> 10;
        const float* y = tile + cpad(lo);  // y[lo + 1024 j] at offset 1056 j
        const uint32_t s0 = (hi & 1u) << 31, s1 = ((hi >> 1) & 1u) << 31, s2 = (hi >> 2) << 31;
        const float2 a = __fadd2_rn(make_float2(y[0], y[4 * 1056]),
                                    make_float2(__uint_as_float(__float_as_uint(y[1056]) ^ s0),
                                                __uint_as_float(__float_as_uint(y[5 * 1056]) ^ s0)));
        const float2 b = __fadd2_rn(make_float2(y[2 * 1056], y[6 * 1056]),
                                    make_float2(__uint_as_float(__float_as_uint(y[3 * 1056]) ^ s0),
                                                __uint_as_float(__float_as_uint(y[7 * 1056]) ^ s0)));
        const float2 c = __fadd2_rn(a, make_float2(__uint_as_float(__float_as_uint(b.x) ^ s1),
                                                   __uint_as_float(__float_as_uint(b.y) ^ s1)));
        zr[q] = c.x + __uint_as_float(__float_as_uint(c.y) ^ s2);
        zd[q] = (int)(w >> 16);
      }
    }
    __syncthreads();  // every y read before z overwrites the tile
#pragma unroll
    for (int q = 0; q < ZPT; ++q)
      if (zd[q] >= 0) tile[zd[q]] = zr[q];
    __syncthreads();
    float* __restrict__ o = cs.out + lc * cs.ldo;
    for (int64_t t = tid; t < P.r; t += COL_T) o[t] = tile[t] * P.scale;
    return;
  }
  // ---- round C: bits 10..12 (u bits 0..2) with bits 0, 1 carried along (u bits 3, 4);
  // thread = bits 2..9.  x = f + 4 tid + 1024 g, u = g + 8 f ----
  {
    float* base = tile + cpad(tid << 2);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int u0 = 2 * m, u1 = 2 * m + 1;
      v[m] = make_float2(base[(u0 >> 3) + 1056 * (u0 & 7)], base[(u1 >> 3) + 1056 * (u1 & 7)]);
    }
    fwht_regs<3>(v);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int u0 = 2 * m, u1 = 2 * m + 1;
      base[(u0 >> 3) + 1056 * (u0 & 7)] = v[m].x;
      base[(u1 >> 3) + 1056 * (u1 & 7)] = v[m].y;
    }
  }
  __syncthreads();
  // ---- the kept rows of z, scaled (coalesced stores) ----
  float* __restrict__ o = cs.out + lc * cs.ldo;
  for (int64_t t = tid; t < P.r; t += COL_T) o[t] = tile[cpad(Kp[t])] * P.scale;
}
}  // namespace

// Finish of a row partition: one FP64 scale and one rounding per entry (srht_rows_finish).
__global__ void k_rows_finish(const double* __restrict__ part, int64_t ldp, int64_t r, int64_t cols, double scale,
                              float* __restrict__ SM, int64_t ldsm) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
    if (t < r) SM[j * ldsm + t] = (float)(part[j * ldp + t] * scale);
}

cudaError_t launch_rows_finish(const double* part, int64_t ldp, int64_t r, int64_t cols, double scale, float* SM,
                               int64_t ldsm, cudaStream_t stream) {
  if (r <= 0 || cols <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((r + 255) / 256), (unsigned)(cols < 65535 ? cols : 65535));
  k_rows_finish<<<grid, 256, 0, stream>>>(part, ldp, r, cols, scale, SM, ldsm);
  return cudaGetLastError();
}

// Whole-column path: N = 2^13 (the padded tile is 33 KB), one slab per column, outputs
// written directly (no row shards).
bool use_col_kernel(const srht_plan* P, const SketchParams& sp) {
  return P->N_eff == COL_N && sp.S_act == 1 && sp.s_lo == 0 && !sp.part_out && P->r <= COL_N;
}

cudaError_t launch_sketch(const srht_plan* P, const SketchParams& sp, cudaStream_t stream) {
  if (sp.total_cols <= 0) return cudaSuccess;
  const int64_t items = sp.total_cols * sp.S_act * sp.groups;
  cudaError_t e;
  const int slot = (g_prof.on && g_prof.used < g_prof.capacity) ? g_prof.used++ : -1;
  if (slot >= 0) cudaEventRecord(g_prof.ev[2 * slot], stream);
  if (use_col_kernel(P, sp)) {
    const int64_t zc = (sp.total_cols + 65534) / 65535;
    k_sketch_col<<<dim3((unsigned)(sp.total_cols < 65535 ? sp.total_cols : 65535), (unsigned)zc), COL_T, 0, stream>>>(sp);
    if (slot >= 0) cudaEventRecord(g_prof.ev[2 * slot + 1], stream);
    g_last_kernel = 5;
    return cudaGetLastError();
  }
  switch (P->log_b) {
    case 10: e = launch_b<10>(P->rpt, sp, items, stream); break;
    case 11: e = launch_b<11>(P->rpt, sp, items, stream); break;
    case 12: e = launch_b<12>(P->rpt, sp, items, stream); break;
    case 13: e = launch_b<13>(P->rpt, sp, items, stream); break;
    case 14: e = launch_b<14>(P->rpt, sp, items, stream); break;
    default: return cudaErrorInvalidValue;
  }
  if (slot >= 0) cudaEventRecord(g_prof.ev[2 * slot + 1], stream);
  g_last_kernel = 1;
  if (e != cudaSuccess || (sp.S_act == 1 && !sp.part_out)) return e;
  return launch_reduce(sp, P->log_b + P->log_j, stream);
}

cudaError_t launch_reduce(const SketchParams& sp, int slab_shift, cudaStream_t stream) {
  const int64_t zc = (sp.total_cols + 65534) / 65535;
  dim3 grid((unsigned)((sp.r + 255) / 256), (unsigned)(sp.total_cols < 65535 ? sp.total_cols : 65535),
            (unsigned)zc);
  k_reduce_slabs<<<grid, 256, 0, stream>>>(sp, slab_shift);
  return cudaGetLastError();
}

}  // namespace srht
