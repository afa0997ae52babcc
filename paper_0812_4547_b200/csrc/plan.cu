// Plan builder: Algorithm 1 steps 2 and 4 on the device.
//
//  * D: sign words = Philox stream (seed, 2p + 0), word w for w < N_eff/64 (R4, R5).
//  * S: the r indices with the smallest (u_i, i), u_i = word i of stream
//    (seed, 2p + 1), i < N (R1, R6).  Found by an 8-pass MSB radix select of
//    the r-th smallest key (keys are regenerated each pass, never stored),
//    then an index-ordered compaction, so K comes out sorted ascending.
#include "internal.cuh"
#include "philox.cuh"

namespace srht {
namespace {

constexpr int kHistThreads = 256;
constexpr int kChunkThreads = 256;
constexpr int kKeysPerThread = 16;                          // 4 Philox blocks
constexpr int64_t kChunk = kChunkThreads * kKeysPerThread;  // keys per chunk

__global__ void k_gen_signs(uint64_t seed, int64_t batch, int64_t words, uint64_t* out) {
  const int64_t bpp = (words + 3) / 4;
  const int64_t total = batch * bpp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / bpp, q = idx % bpp;
    const u64x4 w = stream_block(seed, 2 * (uint64_t)p + 0, (uint64_t)q);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t wi = 4 * q + e;
      if (wi < words) out[p * words + wi] = w.v[e];
    }
  }
}

// Histogram of byte `shift/8` over keys matching the prefix of problem blockIdx.y.
__global__ void k_hist(uint64_t seed, int64_t N, int shift, uint64_t mask,
                       const uint64_t* __restrict__ prefix, uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[256];
  const int64_t p = blockIdx.y;
  for (int b = threadIdx.x; b < 256; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const uint64_t pre = prefix[p];
  const int64_t nblk = (N + 3) / 4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nblk;
       q += (int64_t)gridDim.x * blockDim.x) {
    const u64x4 w = stream_block(seed, 2 * (uint64_t)p + 1, (uint64_t)q);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t u = w.v[e];
      if (4 * q + e < N && (u & mask) == pre) atomicAdd(&sh[(u >> shift) & 255u], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[p * 256 + b], sh[b]);
}

// Pick the bucket holding the need-th smallest matching key; one thread per problem.
__global__ void k_select(int64_t batch, int shift, uint64_t* prefix, int64_t* need, uint32_t* hist) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= batch) return;
  int64_t cum = 0;
  const int64_t nd = need[p];
  int chosen = 255;
  int64_t before = 0;
  for (int b = 0; b < 256; ++b) {
    const int64_t h = hist[p * 256 + b];
    if (cum + h >= nd) {
      chosen = b;
      before = cum;
      break;
    }
    cum += h;
  }
  prefix[p] |= (uint64_t)chosen << shift;
  need[p] = nd - before;
  for (int b = 0; b < 256; ++b) hist[p * 256 + b] = 0;
}

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Exclusive scan over the block (blockDim.x == kChunkThreads); also returns the total.
__device__ int block_excl_scan(int v, int* total) {
  __shared__ int wsum[kChunkThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int s = lane < kChunkThreads / 32 ? wsum[lane] : 0;
    s = warp_incl_scan(s);
    if (lane < kChunkThreads / 32) wsum[lane] = s;
  }
  __syncthreads();
  const int base = wid ? wsum[wid - 1] : 0;
  *total = wsum[kChunkThreads / 32 - 1];
  __syncthreads();
  return base + inc - v;
}

// Per (problem, chunk): number of keys < T and == T.
__global__ void k_count(uint64_t seed, int64_t N, int64_t chunks, const uint64_t* __restrict__ thr,
                        int32_t* __restrict__ n_less, int32_t* __restrict__ n_eq) {
  const int64_t p = blockIdx.y, c = blockIdx.x;
  const uint64_t T = thr[p];
  int less = 0, eq = 0;
  const int64_t i0 = c * kChunk + (int64_t)threadIdx.x * kKeysPerThread;
#pragma unroll
  for (int b = 0; b < kKeysPerThread / 4; ++b) {
    const int64_t q = i0 / 4 + b;
    if (4 * q >= N) break;
    const u64x4 w = stream_block(seed, 2 * (uint64_t)p + 1, (uint64_t)q);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (4 * q + e < N) {
        less += w.v[e] < T;
        eq += w.v[e] == T;
      }
    }
  }
  int tl, te;
  block_excl_scan(less, &tl);
  block_excl_scan(eq, &te);
  if (threadIdx.x == 0) {
    n_less[p * chunks + c] = tl;
    n_eq[p * chunks + c] = te;
  }
}

// Per problem (one thread each): chunk offsets of equal keys and of selected keys.
__global__ void k_offsets(int64_t batch, int64_t chunks, const int64_t* __restrict__ need_eq,
                          const int32_t* __restrict__ n_less, const int32_t* __restrict__ n_eq,
                          int64_t* __restrict__ eq_off, int64_t* __restrict__ sel_off) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= batch) return;
  const int64_t ne = need_eq[p];
  int64_t eq_before = 0, sel_before = 0;
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t e = n_eq[p * chunks + c];
    eq_off[p * chunks + c] = eq_before;
    sel_off[p * chunks + c] = sel_before;
    int64_t take = ne - eq_before;
    take = take < 0 ? 0 : (take > e ? e : take);
    sel_before += n_less[p * chunks + c] + take;
    eq_before += e;
  }
}

__global__ void k_write(uint64_t seed, int64_t N, int64_t r, int64_t chunks,
                        const uint64_t* __restrict__ thr, const int64_t* __restrict__ need_eq,
                        const int64_t* __restrict__ eq_off, const int64_t* __restrict__ sel_off,
                        int32_t* __restrict__ K) {
  const int64_t p = blockIdx.y, c = blockIdx.x;
  const uint64_t T = thr[p];
  const int64_t i0 = c * kChunk + (int64_t)threadIdx.x * kKeysPerThread;
  uint32_t is_less = 0, is_eq = 0;
#pragma unroll
  for (int b = 0; b < kKeysPerThread / 4; ++b) {
    const int64_t q = i0 / 4 + b;
    if (4 * q >= N) break;
    const u64x4 w = stream_block(seed, 2 * (uint64_t)p + 1, (uint64_t)q);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (4 * q + e < N) {
        is_less |= (uint32_t)(w.v[e] < T) << (4 * b + e);
        is_eq |= (uint32_t)(w.v[e] == T) << (4 * b + e);
      }
    }
  }
  int tot;
  const int eq_rank0 = block_excl_scan(__popc(is_eq), &tot);
  const int64_t eq_base = eq_off[p * chunks + c] + eq_rank0;
  const int64_t ne = need_eq[p];
  uint32_t sel = is_less;
  int er = 0;
  for (int e = 0; e < kKeysPerThread; ++e) {
    if ((is_eq >> e) & 1u) {
      if (eq_base + er < ne) sel |= 1u << e;
      ++er;
    }
  }
  const int pos0 = block_excl_scan(__popc(sel), &tot);
  int64_t pos = sel_off[p * chunks + c] + pos0;
  for (int e = 0; e < kKeysPerThread; ++e) {
    if ((sel >> e) & 1u) {
      if (pos < r) K[p * r + pos] = (int32_t)(i0 + e);
      ++pos;
    }
  }
}

template <typename T>
cudaError_t dev_alloc(T** p, size_t count) {
  return cudaMalloc((void**)p, count * sizeof(T) + 16);
}

}  // namespace

// Number of keys u_i < T (i < N) of problem 0's sampling stream: the kept count of the
// Bernoulli(r/N) plan (T = floor(2^64 r / N)), computed with the selection's count pass.
cudaError_t count_keys_below(uint64_t seed, int64_t N, uint64_t T, int64_t* count, cudaStream_t stream) {
  const int64_t chunks = (N + kChunk - 1) / kChunk;
  uint64_t* thr = nullptr;
  int32_t *n_less = nullptr, *n_eq = nullptr;
  cudaError_t err;
  do {
    if ((err = dev_alloc(&thr, 1)) != cudaSuccess) break;
    if ((err = dev_alloc(&n_less, chunks)) != cudaSuccess) break;
    if ((err = dev_alloc(&n_eq, chunks)) != cudaSuccess) break;
    if ((err = cudaMemcpyAsync(thr, &T, sizeof(T), cudaMemcpyHostToDevice, stream)) != cudaSuccess) break;
    k_count<<<dim3((unsigned)chunks, 1u), kChunkThreads, 0, stream>>>(seed, N, chunks, thr, n_less, n_eq);
    if ((err = cudaGetLastError()) != cudaSuccess) break;
    int32_t* h = new int32_t[chunks];
    err = cudaMemcpyAsync(h, n_less, chunks * sizeof(int32_t), cudaMemcpyDeviceToHost, stream);
    if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
    int64_t tot = 0;
    for (int64_t c = 0; c < chunks; ++c) tot += h[c];
    delete[] h;
    *count = tot;
  } while (0);
  cudaFree(thr);
  cudaFree(n_less);
  cudaFree(n_eq);
  return err;
}

cudaError_t build_plan_device(srht_plan* P, cudaStream_t stream) {
  cudaError_t err = cudaSuccess;
  const int64_t batch = P->batch, N = P->N;
  // --- D (Algorithm 1 step 4) ---
  {
    const int64_t blocks = (batch * ((P->words64 + 3) / 4) + 255) / 256;
    const int grid = (int)(blocks < 65535 * 16 ? blocks : 65535 * 16);
    k_gen_signs<<<grid, 256, 0, stream>>>(P->seed, batch, P->words64, P->d_signs);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
  }
  // --- S (steps 2-3): radix select of the r-th smallest key per problem ---
  uint64_t* prefix = nullptr;
  int64_t* need = nullptr;
  uint32_t* hist = nullptr;
  int32_t *n_less = nullptr, *n_eq = nullptr;
  int64_t *eq_off = nullptr, *sel_off = nullptr;
  const int64_t chunks = (N + kChunk - 1) / kChunk;
  do {
    if ((err = dev_alloc(&prefix, batch)) != cudaSuccess) break;
    if ((err = dev_alloc(&need, batch)) != cudaSuccess) break;
    if ((err = dev_alloc(&hist, batch * 256)) != cudaSuccess) break;
    if ((err = dev_alloc(&n_less, batch * chunks)) != cudaSuccess) break;
    if ((err = dev_alloc(&n_eq, batch * chunks)) != cudaSuccess) break;
    if ((err = dev_alloc(&eq_off, batch * chunks)) != cudaSuccess) break;
    if ((err = dev_alloc(&sel_off, batch * chunks)) != cudaSuccess) break;
    if ((err = cudaMemsetAsync(prefix, 0, batch * sizeof(uint64_t), stream)) != cudaSuccess) break;
    if ((err = cudaMemsetAsync(hist, 0, batch * 256 * sizeof(uint32_t), stream)) != cudaSuccess) break;
    {
      // need = r for every problem
      int64_t* h = new int64_t[batch];
      for (int64_t p = 0; p < batch; ++p) h[p] = P->r;
      err = cudaMemcpyAsync(need, h, batch * sizeof(int64_t), cudaMemcpyHostToDevice, stream);
      if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
      delete[] h;
      if (err != cudaSuccess) break;
    }
    const int64_t nblk = (N + 3) / 4;
    int64_t gx = (nblk + kHistThreads - 1) / kHistThreads;
    if (gx > 2048) gx = 2048;
    const int sel_grid = (int)((batch + 127) / 128);
    for (int shift = 56; shift >= 0; shift -= 8) {
      const uint64_t mask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
      k_hist<<<dim3((unsigned)gx, (unsigned)batch), kHistThreads, 0, stream>>>(P->seed, N, shift, mask,
                                                                               prefix, hist);
      k_select<<<sel_grid, 128, 0, stream>>>(batch, shift, prefix, need, hist);
    }
    if ((err = cudaGetLastError()) != cudaSuccess) break;
    // After 8 passes: prefix = threshold value T_p, need = how many keys equal to
    // T_p are taken (lowest indices first, R6).
    k_count<<<dim3((unsigned)chunks, (unsigned)batch), kChunkThreads, 0, stream>>>(P->seed, N, chunks, prefix,
                                                                                  n_less, n_eq);
    k_offsets<<<sel_grid, 128, 0, stream>>>(batch, chunks, need, n_less, n_eq, eq_off, sel_off);
    k_write<<<dim3((unsigned)chunks, (unsigned)batch), kChunkThreads, 0, stream>>>(
        P->seed, N, P->r, chunks, prefix, need, eq_off, sel_off, P->d_K);
    if ((err = cudaGetLastError()) != cudaSuccess) break;
    err = cudaStreamSynchronize(stream);
  } while (0);
  cudaFree(prefix);
  cudaFree(need);
  cudaFree(hist);
  cudaFree(n_less);
  cudaFree(n_eq);
  cudaFree(eq_off);
  cudaFree(sel_off);
  return err;
}

// ---------------------------------------------------------------------------
// Kernel-v2 sign layout: for tile T (2^14 rows) and producer thread p
// (lane = p & 31, wg = p >> 5), the 128 sign bits of its round-0 elements
// x = v + 4*lane + 128*wg + 512*h (v < 4, h < 32) packed as bit 4h+v of a uint4,
// so one 16-byte load gives a thread all its signs for the tile.
// ---------------------------------------------------------------------------
namespace {
__global__ void k_permute_signs_ws(const uint32_t* __restrict__ signs32, int64_t n_tiles, uint4* __restrict__ out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n_tiles * 128) return;
  const int64_t T = idx >> 7;
  const int p = (int)(idx & 127), lane = p & 31, wg = p >> 5;
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  for (int h = 0; h < 32; ++h) {
    for (int v = 0; v < 4; ++v) {
      const int64_t row = (T << 14) + v + 4 * lane + 128 * wg + 512 * h;
      const uint32_t bit = (signs32[row >> 5] >> (row & 31)) & 1u;
      w[h >> 3] |= bit << (((h & 7) << 2) + v);
    }
  }
  out[idx] = make_uint4(w[0], w[1], w[2], w[3]);
}
// Kernel v3 order: producer thread p of tile T owns rows e + 2p + 256h (e < 2, h < 64);
// bit 2(h & 15) + e of word h >> 4.
__global__ void k_permute_signs_v3(const uint32_t* __restrict__ signs32, int64_t n_tiles, uint4* __restrict__ out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n_tiles * 128) return;
  const int64_t T = idx >> 7;
  const int p = (int)(idx & 127);
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  for (int h = 0; h < 64; ++h)
    for (int e = 0; e < 2; ++e) {
      // register u = e + 2h of producer thread p: rows e + 2p + 256h, or with V3_TMEM_RAW rows
      // (u & 3) + 4p + 512 (u >> 2)
      const int u = e + 2 * h;
      const int64_t row = V3_TMEM_RAW ? (T << 14) + (u & 3) + 4 * p + 512 * (u >> 2) : (T << 14) + e + 2 * p + 256 * h;
      const uint32_t bit = (signs32[row >> 5] >> (row & 31)) & 1u;
      w[h >> 4] |= bit << (((h & 15) << 1) + e);
    }
  out[idx] = make_uint4(w[0], w[1], w[2], w[3]);
}
// FP64 TMA kernel order: producer thread p of tile T (2^12 rows) owns rows e + 2p + 128h
// (e < 2, h < 32); bit 2(h & 15) + e of word h >> 4.
__global__ void k_permute_signs_v64(const uint32_t* __restrict__ signs32, int64_t n_tiles, uint2* __restrict__ out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n_tiles * 64) return;
  const int64_t T = idx >> 6;
  const int p = (int)(idx & 63);
  uint32_t w[2] = {0u, 0u};
  for (int h = 0; h < 32; ++h)
    for (int e = 0; e < 2; ++e) {
      const int64_t row = (T << 12) + e + 2 * p + 128 * h;
      const uint32_t bit = (signs32[row >> 5] >> (row & 31)) & 1u;
      w[h >> 4] |= bit << (((h & 15) << 1) + e);
    }
  out[idx] = make_uint2(w[0], w[1]);
}
}  // namespace

cudaError_t build_v64_signs(const uint64_t* signs, int64_t n_tiles, uint2* out, cudaStream_t stream) {
  const int64_t total = n_tiles * 64;
  k_permute_signs_v64<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(reinterpret_cast<const uint32_t*>(signs),
                                                                           n_tiles, out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  return e;
}

cudaError_t build_v3_signs(const uint64_t* signs, int64_t n_tiles, uint4* out, cudaStream_t stream) {
  const int64_t total = n_tiles * 128;
  k_permute_signs_v3<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(reinterpret_cast<const uint32_t*>(signs),
                                                                         n_tiles, out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  return e;
}

cudaError_t build_ws_signs(const uint64_t* signs, int64_t n_tiles, uint4* out, cudaStream_t stream) {
  const int64_t total = n_tiles * 128;
  k_permute_signs_ws<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(reinterpret_cast<const uint32_t*>(signs),
                                                                         n_tiles, out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  return e;
}

// ---------------------------------------------------------------------------
// Workload generator (benchmark/test inputs only): exact FP32 Uniform[0,1).
// ---------------------------------------------------------------------------
namespace {
__global__ void k_gen_uniform(uint64_t seed, uint64_t stream0, int64_t rows, int64_t cols, float* out,
                              int64_t ld) {
  const int64_t nblk = (rows + 3) / 4;
  const int64_t j = blockIdx.y;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nblk;
       q += (int64_t)gridDim.x * blockDim.x) {
    const u64x4 w = stream_block(seed, (1ull << 32) + stream0 + (uint64_t)j, (uint64_t)q);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t i = 4 * q + e;
      if (i < rows) out[i + j * ld] = (float)(w.v[e] >> 40) * 0x1p-24f;
    }
  }
}
}  // namespace

cudaError_t launch_gen_uniform(uint64_t seed, uint64_t stream0, int64_t rows, int64_t cols, float* out,
                               int64_t ld, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  for (int64_t c0 = 0; c0 < cols; c0 += 65535) {
    const int64_t nc = cols - c0 < 65535 ? cols - c0 : 65535;
    int64_t gx = ((rows + 3) / 4 + 255) / 256;
    if (gx > 4096) gx = 4096;
    k_gen_uniform<<<dim3((unsigned)gx, (unsigned)nc), 256, 0, stream>>>(seed, stream0 + c0, rows, nc,
                                                                         out + c0 * ld, ld);
  }
  return cudaGetLastError();
}

}  // namespace srht
