// sl_build.cu — index build on the device (SPEC.md [MODULE] index, build_index).
//
// Token ids arrive flat, doc-major (u32[T] + u64 offsets[N+1]). The reference's two
// passes (pass 1: count_terms + DF + lengths, tokenizer.cpp:162-168 /
// vocabulary.hpp:38; pass 2: S^Δ per nonzero, scoring.cpp:116-145) become:
//   K1  doc expansion + stable LSD radix sort of (token, doc) by token   -> (t,d) order
//   K1' run-length encoding of equal (t,d) runs -> doc ids, run starts (tf), indptr
//   K2  df = row lengths (+ NCCL all-reduce of df, Σ|D|, N across shards)
//   K3  idf(t), S^θ(t) in f64 (scoring.cpp:60-79, 125-145)
//   K4  values[p] = f32(idf * tf_component - S^θ)  (scoring.cpp:81-123)
// followed by the query-side structures (dense copies of the highest-df rows and
// per-tile skip offsets) that sl_query.cu consumes.
// Everything is HBM-streaming integer work; no tensor cores are involved.
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "sl_index.cuh"

namespace sl {

// ============================================================== scan (u32, exclusive)
namespace {
constexpr int kScanThreads = 256;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// exclusive block scan; sw needs 33 entries
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sw, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t incl = warp_incl_scan(v);
  if (lane == 31) sw[w] = incl;
  __syncthreads();
  if (w == 0) {
    const uint32_t x = lane < nw ? sw[lane] : 0u;
    const uint32_t xi = warp_incl_scan(x);
    if (lane < nw) sw[lane] = xi - x;
    if (lane == 31) sw[32] = xi;
  }
  __syncthreads();
  const uint32_t r = sw[w] + incl - v;
  if (total) *total = sw[32];
  __syncthreads();
  return r;
}

}  // namespace

namespace {
// Single-pass exclusive scan (decoupled look-back, Merrill & Garland): a block takes the next
// tile in launch order from a ticket, scans it, publishes its aggregate in a status word
// (flag << 32 | value: 1 = aggregate, 2 = inclusive prefix), and warp 0 sums its predecessors'
// words back to the nearest inclusive prefix, 32 tiles per step. One launch per scan.
constexpr int kLbIPT = 16, kLbTile = kScanThreads * kLbIPT;
constexpr unsigned long long kLbAgg = 1ull << 32, kLbPre = 2ull << 32;

__device__ __forceinline__ uint32_t lookback_warp(unsigned long long* status, uint32_t tile, uint32_t agg) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) atomicExch(status + tile, (tile == 0 ? 2ull << 32 : 1ull << 32) | agg);
  if (tile == 0) return 0;
  uint32_t excl = 0;
  int64_t base = (int64_t)tile - 1;
  for (;;) {
    const int64_t t = base - lane;
    const unsigned long long v = t >= 0 ? *(volatile unsigned long long*)(status + t) : (unsigned long long)(2ull << 32);
    const uint32_t flag = (uint32_t)(v >> 32);
    const uint32_t pm = __ballot_sync(0xffffffffu, flag == 2u);
    const uint32_t zm = __ballot_sync(0xffffffffu, flag == 0u);
    const uint32_t low = pm & (0u - pm);
    const uint32_t need = pm ? (low | (low - 1u)) : 0xffffffffu;  // lanes up to the nearest prefix
    if (zm & need) continue;                                      // a predecessor has not published
    excl += __reduce_add_sync(0xffffffffu, ((need >> lane) & 1u) ? (uint32_t)v : 0u);
    if (pm) break;
    base -= 32;
  }
  if (lane == 0) atomicExch(status + tile, kLbPre | (excl + agg));
  return excl;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_1p(const uint32_t* in, uint32_t* out, uint64_t n,
                                                          unsigned long long* status, uint32_t* ticket,
                                                          uint32_t* total) {
  __shared__ uint32_t sw[33];
  __shared__ uint32_t s_tile, s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * kLbTile + (uint64_t)threadIdx.x * kLbIPT;
  uint32_t v[kLbIPT];
  uint32_t s = 0;
  if (base + kLbIPT <= n && ((reinterpret_cast<uintptr_t>(in + base) & 15) == 0)) {
#pragma unroll
    for (int j = 0; j < kLbIPT; j += 4) {
      const uint4 q = *reinterpret_cast<const uint4*>(in + base + j);
      v[j] = q.x; v[j + 1] = q.y; v[j + 2] = q.z; v[j + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kLbIPT; ++j) v[j] = base + j < n ? in[base + j] : 0u;
  }
#pragma unroll
  for (int j = 0; j < kLbIPT; ++j) s += v[j];
  uint32_t agg;
  const uint32_t excl = block_excl_scan(s, sw, &agg);
  if (threadIdx.x < 32) {
    const uint32_t pre = lookback_warp(status, tile, agg);
    if (threadIdx.x == 0) {
      s_prefix = pre;
      if ((uint64_t)(tile + 1) * kLbTile >= n) *total = pre + agg;  // the last tile
    }
  }
  __syncthreads();
  uint32_t run = s_prefix + excl;
#pragma unroll
  for (int j = 0; j < kLbIPT; ++j) {
    if (base + j < n) out[base + j] = run;
    run += v[j];
  }
}
}  // namespace

// in-place safe (each block reads its whole tile before writing it)
int32_t exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t st,
                           uint32_t* total_host) {
  if (n == 0) {
    if (total_host) *total_host = 0;
    return SL_OK;
  }
  const uint64_t nb = (n + kLbTile - 1) / kLbTile;
  if (nb > 0xFFFFFFFFull) SL_FAIL(SL_EUNSUPPORTED, "scan: too many tiles");
  // status words [nb] | ticket | total (one stream-ordered allocation, zeroed)
  unsigned long long* status = nullptr;
  const uint64_t bytes = nb * 8 + 8;
  SL_CUDA_TRY(cudaMallocAsync(&status, bytes, st));
  SL_CUDA_TRY(cudaMemsetAsync(status, 0, bytes, st));
  uint32_t* ticket = reinterpret_cast<uint32_t*>(status + nb);
  k_scan_1p<<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, n, status, ticket, ticket + 1); ++t_launches;
  SL_CUDA_TRY(cudaGetLastError());
  if (total_host) {
    SL_CUDA_TRY(cudaMemcpyAsync(total_host, ticket + 1, 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaStreamSynchronize(st));
  }
  SL_CUDA_TRY(cudaFreeAsync(status, st));
  return SL_OK;
}

// ============================================================== build kernels
namespace {

constexpr uint32_t kErrOffsets = 1u, kErrToken = 2u, kErrDocLen = 4u;

// doc id per token position (warp per document) + |D| (tokenizer.cpp:166)
__global__ void k_doc_expand(const uint64_t* __restrict__ off, uint32_t N, uint64_t o0,
                             uint32_t* __restrict__ docs, uint32_t* __restrict__ doclens,
                             uint32_t* err) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t d = gw; d < N; d += nw) {
    const uint64_t b = off[d], e = off[d + 1];
    if (e < b) {
      if (lane == 0) atomicOr(err, kErrOffsets);
      continue;
    }
    if (lane == 0) {
      if (e - b > 0xFFFFFFFFull) atomicOr(err, kErrDocLen);
      doclens[d] = (uint32_t)(e - b);
    }
    for (uint64_t i = b - o0 + lane; i < e - o0; i += 32) docs[i] = (uint32_t)d;
  }
}

// |D| per document, offset validation, and tile_doc[k] = the document holding the first
// position of radix-sort tile k (the first sort pass derives every position's document from
// it instead of reading a materialised doc-id array)
__global__ void k_doc_meta(const uint64_t* __restrict__ off, uint32_t N, uint64_t o0, uint32_t tile,
                           uint32_t n_tiles, uint32_t* __restrict__ doclens, uint32_t* __restrict__ tile_doc,
                           uint32_t* err) {
  for (uint64_t d = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; d < N; d += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = off[d], e = off[d + 1];
    if (e < b || b < o0) {
      atomicOr(err, kErrOffsets);
      doclens[d] = 0;
      continue;
    }
    if (e - b > 0xFFFFFFFFull) atomicOr(err, kErrDocLen);
    doclens[d] = (uint32_t)(e - b);
    if (e == b) continue;
    const uint64_t k0 = (b - o0 + tile - 1) / tile, k1 = min((e - o0 - 1) / tile, (uint64_t)n_tiles - 1);
    for (uint64_t k = k0; k <= k1; ++k) tile_doc[k] = (uint32_t)d;
  }
}

__global__ void k_check_tokens(const uint32_t* __restrict__ keys, uint64_t n, uint32_t V,
                               uint32_t* err) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (keys[i] >= V) atomicOr(err, kErrToken);
}

#ifndef SL_SORT_THREADS
#define SL_SORT_THREADS 128
#endif
#ifndef SL_SORT_MINB
#define SL_SORT_MINB 6
#endif
constexpr int kSortThreads = SL_SORT_THREADS;
constexpr int kSortIPT = 16;
constexpr int kSortTile = kSortThreads * kSortIPT;
constexpr int kSortMaxBits = 7;  // digit width cap: rank counters take 2^(bits+1) x 256 B of shared memory

// per-tile digit histogram, digit-major output (hist[digit * n_tiles + tile]). One shared
// atomic per element into per-warp copies (a hot Zipf digit contends within one warp only).
__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const uint32_t* __restrict__ keys,
                                                             uint64_t n, int shift, uint32_t mask,
                                                             uint32_t* __restrict__ hist,
                                                             uint32_t n_tiles, uint32_t V,
                                                             uint32_t* err) {
  constexpr int NW = kSortThreads / 32;
  __shared__ uint32_t sh[NW][1 << kSortMaxBits];
  const int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NW * (1 << kSortMaxBits); i += kSortThreads) (&sh[0][0])[i] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kSortTile + threadIdx.x;
  uint32_t kk[kSortIPT];
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j) {
    const uint64_t i = base + (uint64_t)j * kSortThreads;
    kk[j] = i < n ? keys[i] : 0xFFFFFFFFu;
  }
  bool bad = false;
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j) {
    const bool valid = base + (uint64_t)j * kSortThreads < n;
    bad |= valid && kk[j] >= V;
    if (valid) atomicAdd(&sh[w][(kk[j] >> shift) & mask], 1u);
  }
  if (err && bad) atomicOr(err, kErrToken);
  __syncthreads();
  for (uint32_t dg = threadIdx.x; dg <= mask; dg += kSortThreads) {
    uint32_t c = 0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) c += sh[ww][dg];
    hist[(uint64_t)dg * n_tiles + blockIdx.x] = c;
  }
}

// Stable scatter of one tile (kSortTile elements, 16 consecutive per thread) by digit
// ranking with per-thread counters (the counting scheme of Merrill & Grimshaw's GPU radix
// sort): every thread counts its own elements per digit in private 16-bit shared counters
// (two digits per word: digits [0, ND/2) in the low halves, [ND/2, ND) in the high halves),
// one raking scan over the counters in (digit, thread) order turns them into exclusive
// ranks, and an element's rank = its counter's scanned value + the earlier elements of the
// same digit in its own thread. The tile is then staged in shared memory in rank order and
// every digit's run written to its global offset (coalesced). No warp votes per element.
template <int LOGD, bool DOCS>
__global__ void __launch_bounds__(kSortThreads, SL_SORT_MINB) k_radix_scatter(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, uint64_t n, int shift, uint32_t mask, const uint32_t* __restrict__ offs,
    uint32_t n_tiles, DocSrc ds) {
  constexpr int ND = 1 << LOGD, LANES = ND / 2;
  constexpr int R = LANES;                        // counter words per thread in the raking scan
  constexpr int NWORDS = LANES * kSortThreads;
  constexpr int NPAD = NWORDS + NWORDS / 32;      // one pad word per 32 (conflict-free raking)
  static_assert(NPAD >= 2 * kSortTile, "staging aliases the counters");
  extern __shared__ uint32_t smem[];
  uint32_t* cw = smem;                            // packed counters, then the staged tile
  __shared__ uint32_t delta[ND], sw[33];  // per digit: global start - tile-local start
  const int tid = threadIdx.x;
  for (int i = tid; i < NPAD; i += kSortThreads) cw[i] = 0;
  const uint64_t tile0 = (uint64_t)blockIdx.x * kSortTile;
  const uint64_t b = tile0 + (uint64_t)tid * kSortIPT;
  const uint32_t cnt = (uint32_t)min((uint64_t)kSortTile, n - tile0);
  uint32_t kk[kSortIPT], vv[kSortIPT];
  if constexpr (DOCS) {
    // document of every position: the last document starting at or before the thread's first
    // position (binary search between the tile's and the next tile's first documents), then
    // walked forward (empty documents are skipped)
    const uint32_t tdoc = ds.tile_doc[blockIdx.x];
    uint32_t lo = min(tdoc, ds.N - 1);
    uint32_t hi = blockIdx.x + 1 < n_tiles ? min(ds.tile_doc[blockIdx.x + 1], ds.N - 1) : ds.N - 1;
    if (hi < lo) hi = lo;
    const uint64_t pb = ds.o0 + b;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (__ldg(ds.off + mid) <= pb) lo = mid; else hi = mid - 1;
    }
    uint32_t d = lo;
    uint64_t nxt = __ldg(ds.off + d + 1);
#pragma unroll
    for (int j = 0; j < kSortIPT; ++j) {
      while (nxt <= pb + j && d + 1 < ds.N) nxt = __ldg(ds.off + (++d) + 1);
      vv[j] = d;
    }
  }
  const bool full = cnt == kSortTile && ((((uintptr_t)(kin + b)) | (DOCS ? 0 : ((uintptr_t)(vin + b)))) & 15) == 0;
  if (full) {
#pragma unroll
    for (int j = 0; j < kSortIPT; j += 4) {
      const uint4 a = *reinterpret_cast<const uint4*>(kin + b + j);
      kk[j] = a.x; kk[j + 1] = a.y; kk[j + 2] = a.z; kk[j + 3] = a.w;
      if constexpr (!DOCS) {
        const uint4 c = *reinterpret_cast<const uint4*>(vin + b + j);
        vv[j] = c.x; vv[j + 1] = c.y; vv[j + 2] = c.z; vv[j + 3] = c.w;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kSortIPT; ++j) {
      const bool valid = b + j < n;
      kk[j] = valid ? kin[b + j] : 0u;
      if constexpr (!DOCS) vv[j] = valid ? vin[b + j] : 0u;
    }
  }
  __syncthreads();
  auto cptr = [&](uint32_t dg) {  // this thread's 16-bit counter of digit dg
    const uint32_t w = (dg & (LANES - 1)) * kSortThreads + tid;
    return reinterpret_cast<uint16_t*>(cw + w + (w >> 5)) + (dg >> (LOGD - 1));
  };
  uint32_t pre[kSortIPT];
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j) {
    if (b + j < n) {
      uint16_t* c = cptr((kk[j] >> shift) & mask);
      pre[j] = *c;
      *c = (uint16_t)(pre[j] + 1);
    }
  }
  __syncthreads();
  // raking exclusive scan of the packed counters in (digit lane, thread) order
  uint32_t* seg = cw + tid * R + ((tid * R) >> 5);
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) s += seg[i + (i >> 5)];
  uint32_t tot;
  uint32_t run = block_excl_scan(s, sw, &tot);
  run += (tot & 0xFFFFu) << 16;  // high-half digits follow every low-half digit
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const uint32_t c = seg[i + (i >> 5)];
    seg[i + (i >> 5)] = run;
    run += c;
  }
  __syncthreads();
  for (uint32_t dg = tid; dg < ND; dg += kSortThreads) {
    const uint32_t w = (dg & (LANES - 1)) * kSortThreads;  // thread 0's counter
    const uint32_t ds = reinterpret_cast<const uint16_t*>(cw + w + (w >> 5))[dg >> (LOGD - 1)];
    delta[dg] = (dg <= mask ? offs[(uint64_t)dg * n_tiles + blockIdx.x] : 0u) - ds;
  }
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j)
    if (b + j < n) pre[j] += *cptr((kk[j] >> shift) & mask);
  __syncthreads();
  // (key, value) staged as one 8-byte word in rank order
  uint64_t* stage = reinterpret_cast<uint64_t*>(cw);
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j)
    if (b + j < n) stage[pre[j]] = ((uint64_t)vv[j] << 32) | kk[j];
  __syncthreads();
  for (uint32_t i = tid; i < cnt; i += kSortThreads) {
    const uint64_t e = stage[i];
    const uint32_t k = (uint32_t)e;
    const uint32_t pos = delta[(k >> shift) & mask] + i;
    kout[pos] = k;
    vout[pos] = (uint32_t)(e >> 32);
  }
}

template <int LOGD>
constexpr size_t scatter_smem() {
  return ((size_t)(1 << (LOGD - 1)) * kSortThreads * 33 / 32) * 4;
}

// Run-length encoding of the sorted (token, doc) stream in two passes over 4096-element
// tiles (16 consecutive elements per thread): k_rle_count counts run heads per tile, an
// exclusive scan of the tile counts gives every tile's first nonzero, k_rle_emit writes each
// run's doc id, row and start (tf = distance to the next run's start) and the row starts
// into indptr.
constexpr int kRleThreads = 256, kRleIPT = 16, kRleTile = kRleThreads * kRleIPT;

struct RleItems {
  uint32_t k[kRleIPT], v[kRleIPT];
  uint32_t pk, pv;  // element before the thread's first (pk = 0xFFFFFFFF at i = 0)
  uint32_t heads;   // bit j: element j starts a run
};

__device__ __forceinline__ void rle_load(const uint32_t* __restrict__ k, const uint32_t* __restrict__ v,
                                         uint64_t n, RleItems& it) {
  const uint64_t b = (uint64_t)blockIdx.x * kRleTile + (uint64_t)threadIdx.x * kRleIPT;
  if (b + kRleIPT <= n && ((((uintptr_t)(k + b)) | ((uintptr_t)(v + b))) & 15) == 0) {
#pragma unroll
    for (int j = 0; j < kRleIPT; j += 4) {
      const uint4 a = *reinterpret_cast<const uint4*>(k + b + j);
      const uint4 c = *reinterpret_cast<const uint4*>(v + b + j);
      it.k[j] = a.x; it.k[j + 1] = a.y; it.k[j + 2] = a.z; it.k[j + 3] = a.w;
      it.v[j] = c.x; it.v[j + 1] = c.y; it.v[j + 2] = c.z; it.v[j + 3] = c.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kRleIPT; ++j) {
      const bool valid = b + j < n;
      it.k[j] = valid ? k[b + j] : 0xFFFFFFFFu;
      it.v[j] = valid ? v[b + j] : 0xFFFFFFFFu;
    }
  }
  it.pk = b == 0 || b > n ? 0xFFFFFFFFu : k[b - 1];
  it.pv = b == 0 || b > n ? 0xFFFFFFFFu : v[b - 1];
  uint32_t h = 0, pk = it.pk, pv = it.pv;
#pragma unroll
  for (int j = 0; j < kRleIPT; ++j) {
    if (b + j < n && (b + j == 0 || it.k[j] != pk || it.v[j] != pv)) h |= 1u << j;
    pk = it.k[j];
    pv = it.v[j];
  }
  it.heads = h;
}

__global__ void __launch_bounds__(kRleThreads) k_rle_count(const uint32_t* __restrict__ k,
                                                           const uint32_t* __restrict__ v, uint64_t n,
                                                           uint32_t* __restrict__ tile_counts) {
  __shared__ uint32_t sw[33];
  RleItems it;
  rle_load(k, v, n, it);
  uint32_t tot;
  block_excl_scan(__popc(it.heads), sw, &tot);
  if (threadIdx.x == 0) tile_counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kRleThreads) k_rle_emit(const uint32_t* __restrict__ k,
                                                          const uint32_t* __restrict__ v, uint64_t n,
                                                          const uint32_t* __restrict__ tile_offs, uint64_t nnz,
                                                          uint32_t V, uint32_t* __restrict__ docids,
                                                          uint32_t* __restrict__ rows, uint32_t* __restrict__ runstart,
                                                          uint64_t* __restrict__ indptr) {
  // the tile's runs are staged in shared memory and written as one contiguous range
  __shared__ uint32_t sw[33];
  extern __shared__ uint32_t s_runs[];  // 3 x kRleTile
  uint32_t *s_doc = s_runs, *s_row = s_runs + kRleTile, *s_start = s_runs + 2 * kRleTile;
  RleItems it;
  rle_load(k, v, n, it);
  uint32_t tile_runs;
  uint32_t q = block_excl_scan(__popc(it.heads), sw, &tile_runs);
  const uint32_t p0 = tile_offs[blockIdx.x];
  const uint64_t b = (uint64_t)blockIdx.x * kRleTile + (uint64_t)threadIdx.x * kRleIPT;
  uint32_t pk = it.pk;
#pragma unroll
  for (int j = 0; j < kRleIPT; ++j) {
    if ((it.heads >> j) & 1u) {
      const uint32_t t = it.k[j];
      s_doc[q] = it.v[j];
      s_row[q] = t;
      s_start[q] = (uint32_t)(b + j);
      if (b + j == 0 || pk != t) {  // row start: rows (previous row, t] begin here
        const int64_t prev = b + j == 0 ? -1 : (int64_t)pk;
        for (int64_t x = prev + 1; x <= (int64_t)t; ++x) indptr[x] = p0 + q;
      }
      ++q;
    }
    if (b + j == n - 1) {
      for (uint64_t x = (uint64_t)it.k[j] + 1; x <= V; ++x) indptr[x] = nnz;
      runstart[nnz] = (uint32_t)n;
    }
    pk = it.k[j];
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < tile_runs; i += kRleThreads) {
    docids[p0 + i] = s_doc[i];
    rows[p0 + i] = s_row[i];
    runstart[p0 + i] = s_start[i];
  }
}

__global__ void k_df_from_indptr(const uint64_t* __restrict__ indptr, uint32_t V, uint32_t* __restrict__ df) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < V; t += gridDim.x * blockDim.x)
    df[t] = (uint32_t)(indptr[t + 1] - indptr[t]);
}

// K3: idf and S^θ per token (df = 0 -> empty row, theta 0)
__global__ void k_token_stats(const uint32_t* __restrict__ df, uint32_t V, uint32_t Ng, sl_params p,
                              double* __restrict__ idf64, double* __restrict__ theta64,
                              float* __restrict__ theta) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < V; t += gridDim.x * blockDim.x) {
    const uint32_t d = df[t];
    double i = 0.0, th = 0.0;
    if (d > 0) {
      i = d_idf(p.variant, (double)Ng, (double)d);
      if (!is_sparse_variant(p.variant)) th = d_nonoccurrence(p.variant, i, p.k1, p.delta);
    }
    idf64[t] = i;
    theta64[t] = th;
    theta[t] = (float)th;
  }
}

// K4: S^Δ = idf * tf_component - S^θ in f64, narrowed to f32 (SPEC index pass 2); tf is the
// run length of the (t, d) run (kept for export when tf_out != nullptr). Four consecutive
// nonzeros per thread (vector loads: more bytes in flight per thread).
__device__ __forceinline__ float value_of(const sl_params& p, double avg, uint32_t t, uint32_t tf, uint32_t dl,
                                          const double* __restrict__ idf64, const double* __restrict__ theta64) {
  const double tfc = d_tf_component(p.variant, (double)tf, (double)dl, avg, p.k1, p.b, p.delta);
  const double s = __dmul_rn(idf64[t], tfc);
  return __double2float_rn(__dsub_rn(s, theta64[t]));
}

__global__ void k_values(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ docids,
                         const uint32_t* __restrict__ runstart, const uint32_t* __restrict__ doclens,
                         const double* __restrict__ idf64, const double* __restrict__ theta64,
                         uint64_t nnz, sl_params p, double avg, float* __restrict__ values,
                         uint32_t* __restrict__ tf_out) {
  const uint64_t n4 = nnz / 4;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 t = reinterpret_cast<const uint4*>(rows)[q];
    const uint4 d = reinterpret_cast<const uint4*>(docids)[q];
    const uint4 r = reinterpret_cast<const uint4*>(runstart)[q];
    const uint32_t r4 = runstart[4 * q + 4];
    const uint4 tf = make_uint4(r.y - r.x, r.z - r.y, r.w - r.z, r4 - r.w);
    const uint32_t l0 = doclens[d.x], l1 = doclens[d.y], l2 = doclens[d.z], l3 = doclens[d.w];
    if (tf_out) reinterpret_cast<uint4*>(tf_out)[q] = tf;
    float4 o;
    o.x = value_of(p, avg, t.x, tf.x, l0, idf64, theta64);
    o.y = value_of(p, avg, t.y, tf.y, l1, idf64, theta64);
    o.z = value_of(p, avg, t.z, tf.z, l2, idf64, theta64);
    o.w = value_of(p, avg, t.w, tf.w, l3, idf64, theta64);
    reinterpret_cast<float4*>(values)[q] = o;
  }
  for (uint64_t i = 4 * n4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t tf = runstart[i + 1] - runstart[i];
    if (tf_out) tf_out[i] = tf;
    values[i] = value_of(p, avg, rows[i], tf, doclens[docids[i]], idf64, theta64);
  }
}

__global__ void k_dense_fill(const uint64_t* __restrict__ indptr, const uint32_t* __restrict__ docids,
                             const float* __restrict__ values, const uint32_t* __restrict__ slot_tok,
                             uint32_t n_slots, uint32_t n_pad, float* __restrict__ dense) {
  for (uint32_t s = blockIdx.y; s < n_slots; s += gridDim.y) {
    const uint32_t t = slot_tok[s];
    const uint64_t b = indptr[t], e = indptr[t + 1];
    float* row = dense + (uint64_t)s * n_pad;
    for (uint64_t i = b + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
         i += (uint64_t)gridDim.x * blockDim.x)
      row[docids[i]] = values[i];
  }
}

// pair rows P_ab = r_a + r_b (a < b < m) of the leading dense slots: a run whose dense
// signature starts with a and b starts its dense sum from P_ab — the same f32 addition the
// scoring kernel would do first, so every sum stays bit-identical
__global__ void k_dense_pairs(float* __restrict__ dense, uint32_t n_dense, uint32_t m, uint32_t n_pad) {
  const uint32_t np = m * (m - 1) / 2;
  for (uint32_t pr = blockIdx.y; pr < np; pr += gridDim.y) {
    uint32_t a = 0, r = pr;
    while (r >= m - 1 - a) {
      r -= m - 1 - a;
      ++a;
    }
    const uint32_t b = a + 1 + r;
    const float4* ra = reinterpret_cast<const float4*>(dense + (uint64_t)a * n_pad);
    const float4* rb = reinterpret_cast<const float4*>(dense + (uint64_t)b * n_pad);
    float4* out = reinterpret_cast<float4*>(dense + (uint64_t)dense_pair_row(n_dense, m, a, b) * n_pad);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_pad / 4; i += gridDim.x * blockDim.x) {
      const float4 x = ra[i], y = rb[i];
      out[i] = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
    }
  }
}

// triple rows T_abc = P_ab + r_c (a < b < c < m3 <= m2): the kernel's next addition after P_ab
__global__ void k_dense_triples(float* __restrict__ dense, uint32_t n_dense, uint32_t m2, uint32_t m3,
                                uint32_t n_pad) {
  const uint32_t nt = m3 * (m3 - 1) * (m3 - 2) / 6;
  for (uint32_t tr = blockIdx.y; tr < nt; tr += gridDim.y) {
    uint32_t c = 2;
    while ((c + 1) * c * (c - 1) / 6 <= tr) ++c;
    uint32_t r = tr - c * (c - 1) * (c - 2) / 6, b = 1;
    while ((b + 1) * b / 2 <= r) ++b;
    const uint32_t a = r - b * (b - 1) / 2;
    const float4* pab = reinterpret_cast<const float4*>(dense + (uint64_t)dense_pair_row(n_dense, m2, a, b) * n_pad);
    const float4* rc = reinterpret_cast<const float4*>(dense + (uint64_t)c * n_pad);
    float4* out = reinterpret_cast<float4*>(dense + (uint64_t)dense_triple_row(n_dense, m2, a, b, c) * n_pad);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_pad / 4; i += gridDim.x * blockDim.x) {
      const float4 x = pab[i], y = rc[i];
      out[i] = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
    }
  }
}

// skip[s][tile] = first row-relative posting with doc >= tile * kTileDocs; one CTA per row
// (grid-stride over rows), four postings per thread per step
__global__ void __launch_bounds__(256) k_skip_fill(const uint64_t* __restrict__ indptr,
                                                   const uint32_t* __restrict__ docids,
                                                   const uint32_t* __restrict__ slot_tok, uint32_t n_slots,
                                                   uint32_t n_tiles, uint32_t* __restrict__ skip) {
  for (uint32_t s = blockIdx.x; s < n_slots; s += gridDim.x) {
    const uint32_t t = slot_tok[s];
    const uint64_t b = indptr[t];
    const uint32_t len = (uint32_t)(indptr[t + 1] - b);
    const uint32_t* row = docids + b;
    uint32_t* tab = skip + (uint64_t)s * (n_tiles + 1);
    for (uint32_t j0 = threadIdx.x * 4; j0 < len; j0 += 256 * 4) {
      uint32_t tl[5];
      tl[0] = j0 == 0 ? 0xFFFFFFFFu : row[j0 - 1] / kTileDocs;
#pragma unroll
      for (int u = 0; u < 4; ++u) tl[u + 1] = j0 + u < len ? row[j0 + u] / kTileDocs : 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t j = j0 + u;
        if (j < len) {
          const int64_t prev = j == 0 ? -1 : (int64_t)tl[u];
          for (int64_t x = prev + 1; x <= (int64_t)tl[u + 1]; ++x) tab[x] = j;
          if (j == len - 1)
            for (int64_t x = (int64_t)tl[u + 1] + 1; x <= (int64_t)n_tiles; ++x) tab[x] = len;
        }
      }
    }
  }
}

// planning candidates: rows with df >= dthr or row length >= sthr ({t, df, len} triples,
// appended in any order; out == nullptr only counts)
__global__ void k_plan_count(const uint64_t* __restrict__ indptr, const uint32_t* __restrict__ df, uint32_t V,
                             uint32_t dthr, uint32_t sthr, uint32_t* __restrict__ cnt, uint32_t* __restrict__ out) {
  for (uint32_t t0 = blockIdx.x * blockDim.x; t0 < V; t0 += gridDim.x * blockDim.x) {
    const uint32_t t = t0 + threadIdx.x;
    bool c = false;
    uint32_t f = 0, dl = 0;
    if (t < V) {
      dl = (uint32_t)(indptr[t + 1] - indptr[t]);
      f = df[t];
      c = dl && f && (f >= dthr || dl >= sthr);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, c);
    if (!m) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(cnt, (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (c && out) {
      const uint32_t i = base + __popc(m & ((1u << lane) - 1u));
      out[3 * i] = t;
      out[3 * i + 1] = f;
      out[3 * i + 2] = dl;
    }
  }
}

// planning fast path: per-token class flags (dense copy / skip table) under the thresholds
__global__ void k_plan_flags(const uint64_t* __restrict__ indptr, const uint32_t* __restrict__ df, uint32_t V,
                             uint32_t dthr, uint32_t sthr, uint32_t* __restrict__ fd, uint32_t* __restrict__ fs) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < V; t += gridDim.x * blockDim.x) {
    const uint32_t dl = (uint32_t)(indptr[t + 1] - indptr[t]), f = df[t];
    const bool dn = dl && f && f >= dthr;
    fd[t] = dn;
    fs[t] = dl && f && !dn && dl >= sthr;
  }
}

// slots in token order from the scanned flags; tokinfo for every token
__global__ void k_plan_assign(const uint32_t* __restrict__ fd, const uint32_t* __restrict__ pd,
                              const uint32_t* __restrict__ fs, const uint32_t* __restrict__ ps, uint32_t V,
                              uint32_t n_dense, uint32_t* __restrict__ slot_tok, int32_t* __restrict__ info) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < V; t += gridDim.x * blockDim.x) {
    int32_t v = -1;
    if (fd[t]) {
      v = (int32_t)pd[t];
      slot_tok[pd[t]] = t;
    } else if (fs[t]) {
      v = -2 - (int32_t)ps[t];
      slot_tok[n_dense + ps[t]] = t;
    }
    info[t] = v;
  }
}

// tokinfo[t] = dense slot (>= 0) or -2 - skip slot
__global__ void k_set_tokinfo(const uint32_t* __restrict__ slot_tok, uint32_t n_dense, uint32_t n_skip,
                              int32_t* __restrict__ info) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_dense + n_skip; s += gridDim.x * blockDim.x)
    info[slot_tok[s]] = s < n_dense ? (int32_t)s : -2 - (int32_t)(s - n_dense);
}

// max(0, v) as order-preserving bits (non-negative floats order like their bit patterns)
__device__ __forceinline__ uint32_t pos_bits(float v) { return __float_as_uint(v > 0.f ? v : 0.f); }

// rowmax[t] = max(0, max S^Δ in row t); the row of posting p by binary search on indptr
__global__ void k_row_max(const uint64_t* __restrict__ indptr, uint32_t V, const float* __restrict__ values,
                          uint64_t nnz, uint32_t* __restrict__ rowmax_bits) {
  const uint32_t full = 0xffffffffu;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < nnz; base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = base + threadIdx.x;
    const bool valid = p < nnz;
    uint32_t row = 0xFFFFFFFFu, bits = 0;
    if (valid) {
      uint32_t lo = 0, hi = V;  // last t with indptr[t] <= p
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (indptr[mid] <= p) lo = mid; else hi = mid;
      }
      row = lo;
      bits = pos_bits(values[p]);
    }
    const uint32_t peers = __match_any_sync(full, row);
    const uint32_t m = __reduce_max_sync(peers, bits);
    if (valid && (threadIdx.x & 31) == __ffs(peers) - 1 && m) atomicMax(rowmax_bits + row, m);
  }
}

// per-tile maxima of the dense copies: warp per (slot, tile)
__global__ void k_dense_tile_max(const float* __restrict__ dense, uint32_t n_slots, uint32_t n_tiles, uint32_t n_pad,
                                 float* __restrict__ dmax) {
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (uint64_t)n_slots * n_tiles) return;
  const uint32_t slot = (uint32_t)(w / n_tiles), tile = (uint32_t)(w % n_tiles);
  const float* p = dense + (uint64_t)slot * n_pad + (uint64_t)tile * kTileDocs;
  float m = 0.f;
  for (int i = lane; i < kTileDocs; i += 32) m = fmaxf(m, p[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) dmax[w] = m;
}

// per-tile maxima of the skip rows' slices (warp-aggregated by tile)
__global__ void k_skip_tile_max(const uint64_t* __restrict__ indptr, const uint32_t* __restrict__ docids,
                                const float* __restrict__ values, const uint32_t* __restrict__ slot_tok,
                                uint32_t n_slots, uint32_t n_tiles, uint32_t* __restrict__ smax_bits) {
  for (uint32_t s = blockIdx.y; s < n_slots; s += gridDim.y) {
    const uint32_t t = slot_tok[s];
    const uint64_t b = indptr[t];
    const uint32_t len = (uint32_t)(indptr[t + 1] - b);
    for (uint32_t base = blockIdx.x * blockDim.x; base < len; base += gridDim.x * blockDim.x) {
      const uint32_t j = base + threadIdx.x;
      const bool valid = j < len;
      const uint32_t tile = valid ? docids[b + j] / kTileDocs : 0xFFFFFFFFu;
      const uint32_t bits = valid ? pos_bits(values[b + j]) : 0u;
      const uint32_t peers = __match_any_sync(0xffffffffu, tile);
      const uint32_t m = __reduce_max_sync(peers, bits);
      if (valid && (threadIdx.x & 31) == __ffs(peers) - 1 && m)
        atomicMax(smax_bits + (uint64_t)s * n_tiles + tile, m);
    }
  }
}

// SMs of the current device (queried once per device; grids are sized in multiples of it)
int dev_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
  return cache[dev] > 0 ? cache[dev] : 1;
}

int grid_for(uint64_t n, int threads, int max_blocks = 0) {
  if (max_blocks <= 0) max_blocks = 32 * dev_sms();
  uint64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > (uint64_t)max_blocks) b = max_blocks;
  return (int)b;
}

// BM25Params::validate (scoring.cpp:47-58) — one implementation, in sl_bm25.cpp
int32_t host_validate(const sl_params& p) { return sl_params_validate(&p); }

// RAII set of stream-ordered temporaries
struct Temps {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Temps(cudaStream_t s) : st(s) {}
  template <class T>
  int32_t alloc(T** p, uint64_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMallocAsync((void**)p, count * sizeof(T), st);
    if (e != cudaSuccess) {
      set_error(std::string("device allocation of ") + std::to_string(count * sizeof(T)) +
                " bytes failed: " + cudaGetErrorString(e));
      return SL_ENOMEM;
    }
    ptrs.push_back(*p);
    return SL_OK;
  }
  void release(void* p) {
    for (auto& q : ptrs)
      if (q == p) {
        cudaFreeAsync(q, st);
        q = nullptr;
      }
  }
  ~Temps() {
    for (void* p : ptrs)
      if (p) cudaFreeAsync(p, st);
  }
};

}  // namespace

// Stable LSD radix sort of u32 (key, value) pairs by the low `bits` key bits (<= 7-bit
// digits, widths balanced over the passes). Pass p reads the previous output and writes
// k{p&1}/v{p&1}; kin/vin are only read by the first pass, so v1 may alias vin. When
// v_check != 0, keys >= v_check set err bit 2 during the first histogram pass.
int sort_tile_elems() { return kSortTile; }

int32_t radix_sort_pairs(const uint32_t* kin, const uint32_t* vin, uint64_t n, int bits, uint32_t* k0, uint32_t* k1,
                         uint32_t* v0, uint32_t* v1, cudaStream_t st, const uint32_t** kout, const uint32_t** vout,
                         uint32_t v_check, uint32_t* err, const DocSrc* docs) {
  *kout = kin;
  *vout = vin;
  if (bits <= 0 || n == 0) return SL_OK;
  const int passes = (bits + kSortMaxBits - 1) / kSortMaxBits;
  const int width = (bits + passes - 1) / passes;
  const uint32_t mask = (1u << width) - 1u;
  const int logd = width <= 6 ? 6 : 7;  // counter layout: at least 64 digits
  const uint64_t n_tiles = (n + kSortTile - 1) / kSortTile;
  if (n_tiles > 0x7FFFFFFFull) SL_FAIL(SL_EUNSUPPORTED, "radix sort: too many tiles");
  static bool attr_set = false;
  if (!attr_set) {
    SL_CUDA_TRY(cudaFuncSetAttribute(k_radix_scatter<6, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)scatter_smem<6>()));
    SL_CUDA_TRY(cudaFuncSetAttribute(k_radix_scatter<7, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)scatter_smem<7>()));
    SL_CUDA_TRY(cudaFuncSetAttribute(k_radix_scatter<6, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)scatter_smem<6>()));
    SL_CUDA_TRY(cudaFuncSetAttribute(k_radix_scatter<7, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)scatter_smem<7>()));
    attr_set = true;
  }
  uint32_t* hist;
  SL_CUDA_TRY(cudaMallocAsync(&hist, n_tiles * (uint64_t)(mask + 1) * 4, st));
  uint32_t* kb[2] = {k0, k1};
  uint32_t* vb[2] = {v0, v1};
  const uint32_t* ki = kin;
  const uint32_t* vi = vin;
  for (int p = 0; p < passes; ++p) {
    const int shift = p * width;
    k_radix_hist<<<(unsigned)n_tiles, kSortThreads, 0, st>>>(ki, n, shift, mask, hist, (uint32_t)n_tiles,
                                                             v_check ? v_check : 0xFFFFFFFFu,
                                                             p == 0 && v_check ? err : nullptr); ++t_launches;
    SL_TRY(exclusive_scan_u32(hist, hist, n_tiles * (uint64_t)(mask + 1), st, nullptr));
    const bool from_docs = p == 0 && docs;
    const DocSrc ds = from_docs ? *docs : DocSrc{};
    const unsigned g = (unsigned)n_tiles;
    if (logd == 6 && from_docs)
      k_radix_scatter<6, true><<<g, kSortThreads, scatter_smem<6>(), st>>>(ki, vi, kb[p & 1], vb[p & 1], n, shift,
                                                                           mask, hist, (uint32_t)n_tiles, ds);
    else if (logd == 6)
      k_radix_scatter<6, false><<<g, kSortThreads, scatter_smem<6>(), st>>>(ki, vi, kb[p & 1], vb[p & 1], n, shift,
                                                                            mask, hist, (uint32_t)n_tiles, ds);
    else if (from_docs)
      k_radix_scatter<7, true><<<g, kSortThreads, scatter_smem<7>(), st>>>(ki, vi, kb[p & 1], vb[p & 1], n, shift,
                                                                           mask, hist, (uint32_t)n_tiles, ds);
    else
      k_radix_scatter<7, false><<<g, kSortThreads, scatter_smem<7>(), st>>>(ki, vi, kb[p & 1], vb[p & 1], n, shift,
                                                                            mask, hist, (uint32_t)n_tiles, ds);
    ++t_launches;
    ki = kb[p & 1];
    vi = vb[p & 1];
  }
  SL_CUDA_TRY(cudaFreeAsync(hist, st));
  SL_CUDA_TRY(cudaGetLastError());
  *kout = ki;
  *vout = vi;
  return SL_OK;
}

int32_t nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SL_OK;
  set_error(std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
  return SL_ENCCL;
}

int32_t comm_agree(sl_comm* c, int32_t status) {
  if (!c || c->nranks <= 1) return status;
  const std::string own = get_error();
  int32_t worst = status;
  const bool ok = cudaMemcpyAsync(c->dflag, &worst, 4, cudaMemcpyHostToDevice, c->st) == cudaSuccess &&
                  nccl().AllReduce(c->dflag, c->dflag, 1, ncclInt32, ncclMax, c->comm, c->st) == ncclSuccess &&
                  cudaMemcpyAsync(&worst, c->dflag, 4, cudaMemcpyDeviceToHost, c->st) == cudaSuccess &&
                  cudaStreamSynchronize(c->st) == cudaSuccess;
  if (status != SL_OK) {
    set_error(own);
    return status;
  }
  if (!ok) SL_FAIL(SL_ENCCL, "status agreement with the peer ranks failed");
  if (worst != SL_OK)
    SL_FAIL(worst, std::string("a peer rank failed (") + sl_status_string(worst) + "); see that rank's error");
  return SL_OK;
}

void free_index(sl_index* ix) {
  if (!ix) return;
  cudaSetDevice(ix->device);
  void* ps[] = {ix->indptr, ix->docids, ix->values, ix->df_global, ix->theta, ix->doclens, ix->tf,
                ix->tokinfo, ix->dense, ix->skiptab, ix->rowmax, ix->dmax, ix->smax};
  for (void* p : ps)
    if (p) cudaFreeAsync(p, 0);  // back to the stream-ordered pool
  cudaStreamSynchronize(0);
  delete ix;
}

namespace {
// persistent index arrays come from the device's stream-ordered pool (kept mapped across
// builds by the release threshold set in get_stream), so rebuilding does not pay page mapping
thread_local cudaStream_t t_build_stream = nullptr;
thread_local cudaStream_t t_side_stream[64][2] = {};

// side build streams of the current device (work that overlaps the build stream's):
// 0 = per-nonzero values, 1 = skip tables
int32_t side_stream(cudaStream_t* out, int which = 1) {
  int dev = 0;
  SL_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) SL_FAIL(SL_EUNSUPPORTED, "device ordinal out of range");
  cudaStream_t& s = t_side_stream[dev][which & 1];
  if (!s) SL_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = s;
  return SL_OK;
}

template <class T>
int32_t dalloc(sl_index* ix, T** p, uint64_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMallocAsync((void**)p, count * sizeof(T), t_build_stream);
  if (e != cudaSuccess) {
    *p = nullptr;
    set_error(std::string("device allocation of ") + std::to_string(count * sizeof(T)) +
              " bytes failed: " + cudaGetErrorString(e));
    return SL_ENOMEM;
  }
  ix->device_bytes += count * sizeof(T);
  return SL_OK;
}

// Query-side access structures from a finished CSC (ix->indptr/docids/values/df_global):
// dense copies of the rows with global df >= density * N_global, per-tile skip offsets of
// long rows, and the per-token dispatch table. Used by the build and by index loading.
int32_t build_query_structures(sl_index* ix, float dense_min_density, cudaStream_t st,
                               cudaEvent_t values_ready = nullptr) {
  Temps tmp(st);
  const uint32_t N = ix->N, V = ix->V;
  ix->num_tiles = (N + kTileDocs - 1) / kTileDocs;
  ix->n_pad = ix->num_tiles * kTileDocs;
  const double density = dense_min_density > 0.f ? (double)dense_min_density : 0.125;
  double dense_thr = density > 1.0 ? INFINITY : density * (double)ix->N_global;
#ifndef SL_SKIP_PER_TILE
#define SL_SKIP_PER_TILE 0.25
#endif
  uint64_t skip_thr = std::max<uint64_t>(1, (uint64_t)(SL_SKIP_PER_TILE * ix->num_tiles));
  const uint32_t dthr = dense_thr >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)std::ceil(dense_thr);
  const uint32_t sthr = skip_thr >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)skip_thr;
  // Dense copies: rows with global df >= N/8 (c2 top-10: N/4 -> N/8 +2.4%, N/16 worse). By
  // default their global footprint is capped at 12 GB (at most 12 GB / (4 N) rows, highest df
  // first): c5's 50M docs would otherwise take 141 rows, whose chunks crowd L2 (c5 shard
  // top-100 -8% against the 59 rows of N/4). The cap uses only global quantities, so every
  // shard of any sharding classifies the same rows (identical per-document summation order).
  uint64_t dense_cap = UINT64_MAX;
  if (!(dense_min_density > 0.f) && ix->N_global) {
    dense_cap = (12ull << 30) / (4ull * ix->N_global);
    if (const char* e = std::getenv("SL_DENSE_MAX_ROWS"))  // bench: a one-GPU stand-in for one shard
      if (*e) dense_cap = std::strtoull(e, nullptr, 10);    // of a larger corpus uses the corpus's cap
  }
  // Per-tile skip tables for rows with >= SL_SKIP_PER_TILE postings per tile on average: a
  // prefetched table entry beats probing the row's doc ids from one posting per few tiles on
  // (c2 top-10: 4 -> 0.25 postings/tile +4.5%). Tables cost (tiles+1) x 4 B per row, so they
  // are held to 4 B per nonzero (at least 64 MB): beyond that budget only the longest rows
  // get one.
  const uint64_t skip_row_bytes = ((uint64_t)ix->num_tiles + 1) * 4;
  const uint64_t skip_cap = std::max<uint64_t>(4 * ix->nnz, 64ull << 20) / skip_row_bytes;
  std::vector<uint32_t> dense_tok, skip_tok;
  uint32_t* slot_tok = nullptr;
  bool planned = false;
  {
    // fast path (no cap binds): class flags, ordered slots and tokinfo on the device; only
    // the two counts travel to the host
    uint32_t *f, *pf;
    SL_TRY(tmp.alloc(&f, 2ull * V));
    SL_TRY(tmp.alloc(&pf, 2ull * V));
    k_plan_flags<<<grid_for(V, 256), 256, 0, st>>>(ix->indptr, ix->df_global, V, dthr, sthr, f, f + V); ++t_launches;
    SL_TRY(exclusive_scan_u32(f, pf, V, st, nullptr));
    SL_TRY(exclusive_scan_u32(f + V, pf + V, V, st, nullptr));
    uint32_t h[4];
    SL_CUDA_TRY(cudaMemcpyAsync(h, f + V - 1, 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(h + 1, pf + V - 1, 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(h + 2, f + 2ull * V - 1, 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(h + 3, pf + 2ull * V - 1, 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaStreamSynchronize(st));
    const uint32_t nd = h[0] + h[1], ns = h[2] + h[3];
    if (nd <= dense_cap && ns <= skip_cap) {
      ix->dense_rows = nd;
      ix->skip_rows = ns;
      SL_TRY(dalloc(ix, &ix->tokinfo, V));
      SL_TRY(tmp.alloc(&slot_tok, (uint64_t)nd + ns));
      k_plan_assign<<<grid_for(V, 256), 256, 0, st>>>(f, pf, f + V, pf + V, V, nd, slot_tok, ix->tokinfo);
      ++t_launches;
      planned = true;
    }
  }
  // Capped path: candidates (rows that can get a dense copy or a skip table under the
  // thresholds before the caps, which only raise them) are compacted on the device; only they
  // travel to the host, sorted there so slot order is token order.
  std::vector<uint32_t> cand;  // {t, df, row length} triples
  if (!planned) {
    uint32_t* d_cand;
    uint32_t* d_cnt;
    SL_TRY(tmp.alloc(&d_cnt, 1));
    SL_CUDA_TRY(cudaMemsetAsync(d_cnt, 0, 4, st));
    k_plan_count<<<grid_for(V, 256), 256, 0, st>>>(ix->indptr, ix->df_global, V, dthr, sthr, d_cnt, nullptr); ++t_launches;
    uint32_t nc = 0;
    SL_CUDA_TRY(cudaMemcpyAsync(&nc, d_cnt, 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaStreamSynchronize(st));
    if (nc) {
      SL_TRY(tmp.alloc(&d_cand, 3ull * nc));
      SL_CUDA_TRY(cudaMemsetAsync(d_cnt, 0, 4, st));
      k_plan_count<<<grid_for(V, 256), 256, 0, st>>>(ix->indptr, ix->df_global, V, dthr, sthr, d_cnt, d_cand); ++t_launches;
      cand.resize(3ull * nc);
      SL_CUDA_TRY(cudaMemcpyAsync(cand.data(), d_cand, 12ull * nc, cudaMemcpyDeviceToHost, st));
      SL_CUDA_TRY(cudaStreamSynchronize(st));
    }
  }
  if (!planned) {
    const size_t nc = cand.size() / 3;
    std::vector<uint32_t> order(nc);
    for (size_t i = 0; i < nc; ++i) order[i] = (uint32_t)i;
    std::sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return cand[3 * x] < cand[3 * y]; });
    auto c_t = [&](size_t i) { return cand[3 * order[i]]; };
    auto c_df = [&](size_t i) { return cand[3 * order[i] + 1]; };
    auto c_dl = [&](size_t i) { return (uint64_t)cand[3 * order[i] + 2]; };
    if (dense_cap != UINT64_MAX) {  // highest df first within the cap
      std::vector<uint32_t> dc;
      for (size_t i = 0; i < nc; ++i)
        if ((double)c_df(i) >= dense_thr) dc.push_back(c_df(i));
      if (dc.size() > dense_cap) {
        if (dense_cap == 0) {
          dense_thr = INFINITY;
        } else {
          std::nth_element(dc.begin(), dc.begin() + (dense_cap - 1), dc.end(), std::greater<uint32_t>());
          dense_thr = (double)dc[dense_cap - 1] + 1.0;  // strictly above: ties past the cap stay sparse
        }
      }
    }
    {  // longest rows first within the skip-table budget
      std::vector<uint64_t> sc;
      for (size_t i = 0; i < nc; ++i)
        if (c_dl(i) >= skip_thr && (double)c_df(i) < dense_thr) sc.push_back(c_dl(i));
      if (sc.size() > skip_cap) {
        if (skip_cap == 0) {
          skip_thr = UINT64_MAX;
        } else {
          std::nth_element(sc.begin(), sc.begin() + (skip_cap - 1), sc.end(), std::greater<uint64_t>());
          skip_thr = sc[skip_cap - 1] + 1;  // strictly above: ties beyond the budget are dropped
        }
      }
    }
    for (size_t i = 0; i < nc; ++i) {
      if ((double)c_df(i) >= dense_thr) dense_tok.push_back(c_t(i));
      else if (c_dl(i) >= skip_thr) skip_tok.push_back(c_t(i));
    }
    ix->dense_rows = (uint32_t)dense_tok.size();
    ix->skip_rows = (uint32_t)skip_tok.size();
    SL_TRY(dalloc(ix, &ix->tokinfo, V));
    SL_CUDA_TRY(cudaMemsetAsync(ix->tokinfo, 0xFF, (uint64_t)V * 4, st));  // -1: short row
    SL_TRY(tmp.alloc(&slot_tok, dense_tok.size() + skip_tok.size()));
    if (!dense_tok.empty())
      SL_CUDA_TRY(cudaMemcpyAsync(slot_tok, dense_tok.data(), dense_tok.size() * 4, cudaMemcpyHostToDevice, st));
    if (!skip_tok.empty())
      SL_CUDA_TRY(cudaMemcpyAsync(slot_tok + dense_tok.size(), skip_tok.data(), skip_tok.size() * 4,
                                  cudaMemcpyHostToDevice, st));
    if (ix->dense_rows + ix->skip_rows) {
      k_set_tokinfo<<<grid_for(ix->dense_rows + ix->skip_rows, 256), 256, 0, st>>>(slot_tok, ix->dense_rows,
                                                                                  ix->skip_rows, ix->tokinfo);
      ++t_launches;
    }
  }
  // skip tables on a side stream: their fill is latency-bound (one CTA per row), the dense
  // copies below are bandwidth-bound, so the two overlap
  cudaEvent_t fork = nullptr, join = nullptr;
  struct EvGuard {  // on every exit: the build stream waits for the side stream before the
    cudaStream_t s;  // temporaries it reads (slot_tok) are freed on the build stream
    cudaEvent_t* a;
    cudaEvent_t* b;
    ~EvGuard() {
      if (*b) cudaStreamWaitEvent(s, *b, 0);
      if (*a) cudaEventDestroy(*a);
      if (*b) cudaEventDestroy(*b);
    }
  } evg{st, &fork, &join};
  if (ix->skip_rows) {
    SL_TRY(dalloc(ix, &ix->skiptab, (uint64_t)ix->skip_rows * (ix->num_tiles + 1)));
    cudaStream_t side;
    SL_TRY(side_stream(&side));
    SL_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    SL_CUDA_TRY(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    SL_CUDA_TRY(cudaEventRecord(fork, st));
    SL_CUDA_TRY(cudaStreamWaitEvent(side, fork, 0));
    k_skip_fill<<<std::min<uint32_t>(ix->skip_rows, 8 * dev_sms()), 256, 0, side>>>(
        ix->indptr, ix->docids, slot_tok + ix->dense_rows, ix->skip_rows, ix->num_tiles, ix->skiptab); ++t_launches;
    SL_CUDA_TRY(cudaEventRecord(join, side));
  }
  // the dense copies read the per-nonzero values (computed on a side stream during a build)
  if (values_ready) SL_CUDA_TRY(cudaStreamWaitEvent(st, values_ready, 0));
  if (ix->dense_rows) {
    // pair rows for the leading m dense slots, within 2 GB (c2: 120 rows, 480 MB; c4: 55 rows)
    // — SL_DENSE_PAIRS=m overrides, 0: none
    uint32_t m = std::min<uint32_t>(16, ix->dense_rows);
    const uint64_t row_bytes = (uint64_t)ix->n_pad * 4;
    while (m > 1 && (uint64_t)m * (m - 1) / 2 * row_bytes > (2ull << 30)) --m;
    if (const char* e = std::getenv("SL_DENSE_PAIRS"))
      if (*e) m = std::min<uint32_t>((uint32_t)std::atoi(e), ix->dense_rows);
    if (m < 2) m = 0;
    ix->pair_m = m;
    // triple rows for the leading m3 <= m slots within 512 MB (c2: 56 rows, 224 MB). Larger
    // dense arrays fragmented the allocator's pool between rebuilds (c4 with 3.7 GB of pairs
    // and 2 GB of triples rebuilt in 84-259 ms instead of 21) — SL_DENSE_TRIPLES=m3 overrides
    uint32_t m3 = std::min<uint32_t>(8, m);
    while (m3 > 2 && (uint64_t)m3 * (m3 - 1) * (m3 - 2) / 6 * row_bytes > (512ull << 20)) --m3;
    if (const char* e = std::getenv("SL_DENSE_TRIPLES"))
      if (*e) m3 = std::min<uint32_t>((uint32_t)std::atoi(e), m);
    if (m3 < 3) m3 = 0;
    ix->triple_m = m3;
    const uint64_t rows = (uint64_t)ix->dense_rows + (m ? (uint64_t)m * (m - 1) / 2 : 0) +
                          (m3 ? (uint64_t)m3 * (m3 - 1) * (m3 - 2) / 6 : 0);
    SL_TRY(dalloc(ix, &ix->dense, rows * ix->n_pad));
    SL_CUDA_TRY(cudaMemsetAsync(ix->dense, 0, (uint64_t)ix->dense_rows * ix->n_pad * 4, st));
    dim3 g(grid_for(N, 256, 1024), std::min<uint32_t>(ix->dense_rows, 65535));
    k_dense_fill<<<g, 256, 0, st>>>(ix->indptr, ix->docids, ix->values, slot_tok, ix->dense_rows, ix->n_pad,
                                    ix->dense); ++t_launches;
    if (m) {
      dim3 gp(grid_for(ix->n_pad / 4, 256, 256), std::min<uint32_t>(m * (m - 1) / 2, 65535));
      k_dense_pairs<<<gp, 256, 0, st>>>(ix->dense, ix->dense_rows, m, ix->n_pad); ++t_launches;
    }
    if (m3) {
      dim3 gt(grid_for(ix->n_pad / 4, 256, 256), std::min<uint32_t>(m3 * (m3 - 1) * (m3 - 2) / 6, 65535));
      k_dense_triples<<<gt, 256, 0, st>>>(ix->dense, ix->dense_rows, m, m3, ix->n_pad); ++t_launches;
    }
  }
  if (ix->skip_rows) SL_CUDA_TRY(cudaStreamWaitEvent(st, join, 0));  // the skip tables (side stream) are done
  // block-max bounds for exact pruning (opt-in: SL_BLOCKMAX=1; measured slower at 512-doc tiles,
  // DESIGN.md §8)
  const char* bm = std::getenv("SL_BLOCKMAX");
  if (!bm || std::atoi(bm) == 0) {
    SL_CUDA_TRY(cudaGetLastError());
    return SL_OK;
  }
  SL_TRY(dalloc(ix, &ix->rowmax, V));
  SL_CUDA_TRY(cudaMemsetAsync(ix->rowmax, 0, (uint64_t)V * 4, st));
  if (ix->nnz)
    k_row_max<<<grid_for(ix->nnz, 256), 256, 0, st>>>(ix->indptr, V, ix->values, ix->nnz, (uint32_t*)ix->rowmax); ++t_launches;
  if (ix->dense_rows) {
    SL_TRY(dalloc(ix, &ix->dmax, (uint64_t)ix->dense_rows * ix->num_tiles));
    const uint64_t warps = (uint64_t)ix->dense_rows * ix->num_tiles;
    k_dense_tile_max<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(ix->dense, ix->dense_rows, ix->num_tiles,
                                                                         ix->n_pad, ix->dmax); ++t_launches;
  }
  if (ix->skip_rows) {
    SL_TRY(dalloc(ix, &ix->smax, (uint64_t)ix->skip_rows * ix->num_tiles));
    SL_CUDA_TRY(cudaMemsetAsync(ix->smax, 0, (uint64_t)ix->skip_rows * ix->num_tiles * 4, st));
    dim3 g(8, std::min<uint32_t>(ix->skip_rows, 65535));
    k_skip_tile_max<<<g, 256, 0, st>>>(ix->indptr, ix->docids, ix->values, slot_tok + ix->dense_rows,
                                       ix->skip_rows, ix->num_tiles, (uint32_t*)ix->smax); ++t_launches;
  }
  SL_CUDA_TRY(cudaGetLastError());
  return SL_OK;
}


int32_t build_body(const sl_build_desc* d, sl_index* ix, cudaStream_t st, bool* agreed) {
  PhaseTrace tr(st, "SL_BUILD_TRACE", "build");
  const uint32_t N = d->num_docs, V = d->vocab_size;
  // ---- inputs on the device
  uint64_t o0 = 0, oN = 0;
  if (d->mem == SL_MEM_HOST) {
    o0 = d->doc_offsets[0];
    oN = d->doc_offsets[N];
  } else {
    SL_CUDA_TRY(cudaMemcpyAsync(&o0, d->doc_offsets, 8, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(&oN, d->doc_offsets + N, 8, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (oN < o0) SL_FAIL(SL_EINVAL, "build_index: doc offsets must be non-decreasing");
  const uint64_t T = oN - o0;
  if (T == 0) SL_FAIL(SL_EINVAL, "build_index: degenerate corpus (all documents empty)");
  if (T >= 0xFFFFFFFFull)
    SL_FAIL(SL_EUNSUPPORTED, "build_index: a shard must hold fewer than 2^32-1 tokens; shard further");

  Temps tmp(st);
  const uint64_t* off = d->doc_offsets;
  const uint32_t* tokens = d->token_ids + o0;
  if (d->mem == SL_MEM_HOST) {
    uint64_t* doff;
    uint32_t* dtok;
    SL_TRY(tmp.alloc(&doff, (uint64_t)N + 1));
    SL_TRY(tmp.alloc(&dtok, T));
    SL_CUDA_TRY(cudaMemcpyAsync(doff, off, ((uint64_t)N + 1) * 8, cudaMemcpyHostToDevice, st));
    SL_CUDA_TRY(cudaMemcpyAsync(dtok, tokens, T * 4, cudaMemcpyHostToDevice, st));
    off = doff;
    tokens = dtok;
  }

  cudaEvent_t ev0, ev1;
  SL_CUDA_TRY(cudaEventCreate(&ev0));
  SL_CUDA_TRY(cudaEventCreate(&ev1));
  SL_CUDA_TRY(cudaEventRecord(ev0, st));
  tr.mark("start");

  uint32_t* err;
  SL_TRY(tmp.alloc(&err, 1));
  SL_CUDA_TRY(cudaMemsetAsync(err, 0, 4, st));

  // ---- K1: stable LSD radix sort of (token, doc) by token; the first pass takes every
  // position's doc id from the offsets (k_doc_meta), later passes from the ping-pong buffers
  int bits = 0;
  while (bits < 32 && (V - 1) >> bits) ++bits;
  uint32_t *docs, *kb0, *kb1, *vb1;
  SL_TRY(tmp.alloc(&docs, T));
  SL_TRY(dalloc(ix, &ix->doclens, N));
  const uint32_t* ksorted = tokens;
  const uint32_t* vsorted = docs;
  if (bits == 0) {
    k_doc_expand<<<grid_for((uint64_t)N * 32, 256), 256, 0, st>>>(off, N, o0, docs, ix->doclens, err); ++t_launches;
    k_check_tokens<<<grid_for(T, 256), 256, 0, st>>>(tokens, T, V, err); ++t_launches;
  } else {
    const uint64_t n_tiles = (T + kSortTile - 1) / kSortTile;
    uint32_t* tile_doc;
    SL_TRY(tmp.alloc(&tile_doc, n_tiles));
    SL_CUDA_TRY(cudaMemsetAsync(tile_doc, 0, n_tiles * 4, st));
    k_doc_meta<<<grid_for(N, 256), 256, 0, st>>>(off, N, o0, kSortTile, (uint32_t)n_tiles, ix->doclens, tile_doc,
                                                 err); ++t_launches;
    tr.mark("doc_meta");
    SL_TRY(tmp.alloc(&kb0, T));
    SL_TRY(tmp.alloc(&kb1, T));
    SL_TRY(tmp.alloc(&vb1, T));
    const DocSrc ds{off, o0, N, tile_doc};
    // values ping-pong between vb1 and docs
    SL_TRY(radix_sort_pairs(tokens, nullptr, T, bits, kb0, kb1, vb1, docs, st, &ksorted, &vsorted, V, err, &ds));
  }
  SL_CUDA_TRY(cudaGetLastError());
  tr.mark("sort");
  uint32_t herr = 0;  // checked after the run-count sync below (one host round trip)
  SL_CUDA_TRY(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));

  // ---- K1': run-length encode (t,d) runs
  const uint64_t rle_tiles = (T + kRleTile - 1) / kRleTile;
  uint32_t* tile_offs;
  SL_TRY(tmp.alloc(&tile_offs, rle_tiles));
  k_rle_count<<<(unsigned)rle_tiles, kRleThreads, 0, st>>>(ksorted, vsorted, T, tile_offs); ++t_launches;
  uint32_t nnz32 = 0;
  SL_TRY(exclusive_scan_u32(tile_offs, tile_offs, rle_tiles, st, &nnz32));
  if (herr & kErrOffsets) SL_FAIL(SL_EINVAL, "build_index: doc offsets must be non-decreasing");
  if (herr & kErrToken) SL_FAIL(SL_EINVAL, "build_index: token id >= vocab size");
  if (herr & kErrDocLen) SL_FAIL(SL_EUNSUPPORTED, "build_index: document longer than 2^32-1 tokens");
  const uint64_t nnz = nnz32;
  ix->nnz = nnz;
  tr.mark("rle_count+sync");
  uint32_t *rows, *runstart;
  SL_TRY(tmp.alloc(&rows, nnz));
  SL_TRY(tmp.alloc(&runstart, nnz + 1));
  SL_TRY(dalloc(ix, &ix->docids, nnz));
  SL_TRY(dalloc(ix, &ix->indptr, (uint64_t)V + 1));
  SL_CUDA_TRY(cudaFuncSetAttribute(k_rle_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * kRleTile * 4));
  k_rle_emit<<<(unsigned)rle_tiles, kRleThreads, 3 * kRleTile * 4, st>>>(ksorted, vsorted, T, tile_offs, nnz, V, ix->docids, rows,
                                                          runstart, ix->indptr); ++t_launches;
  tr.mark("rle_emit");
  if (d->keep_tf) SL_TRY(dalloc(ix, &ix->tf, nnz));
  if (bits > 0) {
    tmp.release(kb0);
    tmp.release(kb1);
    tmp.release(vb1);
  }
  tmp.release(docs);

  // ---- K2: df (global via NCCL), N, Σ|D|
  SL_TRY(dalloc(ix, &ix->df_global, V));
  k_df_from_indptr<<<grid_for(V, 256), 256, 0, st>>>(ix->indptr, V, ix->df_global); ++t_launches;
  uint64_t stats[2] = {T, N};
  if (d->global_df) {
    // caller-supplied global statistics (virtual shards / external transport)
    SL_CUDA_TRY(cudaMemcpyAsync(ix->df_global, d->global_df, (uint64_t)V * 4, cudaMemcpyHostToDevice, st));
    stats[0] = d->global_total_len;
    stats[1] = d->global_num_docs;
    if (stats[1] < N || stats[0] < T) SL_FAIL(SL_EINVAL, "build_index: global statistics smaller than the shard's");
  } else if (d->comm) {
    uint64_t* dstats;
    SL_TRY(tmp.alloc(&dstats, 2));
    *agreed = true;  // from here on every rank takes part in the collectives below
    SL_TRY(comm_agree(d->comm, SL_OK));
    SL_CUDA_TRY(cudaMemcpyAsync(dstats, stats, 16, cudaMemcpyHostToDevice, st));
    SL_TRY(nccl_check(nccl().AllReduce(ix->df_global, ix->df_global, V, ncclUint32, ncclSum, d->comm->comm, st),
                      "ncclAllReduce(df)"));
    SL_TRY(nccl_check(nccl().AllReduce(dstats, dstats, 2, ncclUint64, ncclSum, d->comm->comm, st),
                      "ncclAllReduce(sum_len, N)"));
    SL_CUDA_TRY(cudaMemcpyAsync(stats, dstats, 16, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (stats[1] > 0xFFFFFFFFull) SL_FAIL(SL_EUNSUPPORTED, "build_index: more than 2^32-1 documents");
  ix->total_len = stats[0];
  ix->N_global = (uint32_t)stats[1];
  ix->avg_len = (double)stats[0] / (double)stats[1];  // SPEC L_avg = Σ|D| / N

  // ---- K3 + K4
  double *idf64, *theta64;
  SL_TRY(tmp.alloc(&idf64, V));
  SL_TRY(tmp.alloc(&theta64, V));
  SL_TRY(dalloc(ix, &ix->theta, V));
  k_token_stats<<<grid_for(V, 256), 256, 0, st>>>(ix->df_global, V, ix->N_global, d->params, idf64, theta64,
                                                 ix->theta); ++t_launches;
  SL_TRY(dalloc(ix, &ix->values, nnz));
  // the values run on a side stream while the access structures are planned and the skip
  // tables filled (they need only indptr / docids / df); the dense copies wait for them
  cudaStream_t vside;
  SL_TRY(side_stream(&vside, 0));
  cudaEvent_t vfork = nullptr, vjoin = nullptr;
  struct VGuard {  // on every exit the build stream waits for the values before its temporaries
    cudaStream_t s;  // (rows, runstart, idf64, theta64) are freed
    cudaEvent_t* a;
    cudaEvent_t* b;
    ~VGuard() {
      if (*b) cudaStreamWaitEvent(s, *b, 0);
      if (*a) cudaEventDestroy(*a);
      if (*b) cudaEventDestroy(*b);
    }
  } vg{st, &vfork, &vjoin};
  SL_CUDA_TRY(cudaEventCreateWithFlags(&vfork, cudaEventDisableTiming));
  SL_CUDA_TRY(cudaEventCreateWithFlags(&vjoin, cudaEventDisableTiming));
  SL_CUDA_TRY(cudaEventRecord(vfork, st));
  SL_CUDA_TRY(cudaStreamWaitEvent(vside, vfork, 0));
  k_values<<<grid_for(nnz / 4 + 1, 256), 256, 0, vside>>>(rows, ix->docids, runstart, ix->doclens, idf64, theta64,
                                                         nnz, d->params, ix->avg_len, ix->values, ix->tf);
  ++t_launches;
  SL_CUDA_TRY(cudaGetLastError());
  SL_CUDA_TRY(cudaEventRecord(vjoin, vside));
  tr.mark("df+stats+values");

  SL_TRY(build_query_structures(ix, d->dense_min_density, st, vjoin));
  SL_CUDA_TRY(cudaStreamWaitEvent(st, vjoin, 0));
  tr.mark("structures");
  SL_CUDA_TRY(cudaEventRecord(ev1, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  SL_CUDA_TRY(cudaEventElapsedTime(&ix->build_ms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  return SL_OK;
}
}  // namespace

int32_t build_index_impl(const sl_build_desc* d, sl_index** out) {
  if (!d || !out) SL_FAIL(SL_EINVAL, "sl_index_build: null argument");
  *out = nullptr;
  SL_TRY(host_validate(d->params));
  if (d->num_docs == 0) SL_FAIL(SL_EINVAL, "build_index: empty corpus");
  if (d->vocab_size == 0) SL_FAIL(SL_EINVAL, "build_index: empty vocabulary");
  if (!d->doc_offsets || !d->token_ids) SL_FAIL(SL_EINVAL, "build_index: null corpus pointers");
  if (d->mem != SL_MEM_HOST && d->mem != SL_MEM_DEVICE) SL_FAIL(SL_EINVAL, "build_index: bad mem kind");
  if ((uint64_t)d->doc_base + d->num_docs > 0xFFFFFFFFull)
    SL_FAIL(SL_EUNSUPPORTED, "build_index: global doc ids must fit in 32 bits");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    SL_FAIL(SL_ECUDA, "sl_index_build: no CUDA device available (there is no CPU fallback)");
  SL_CUDA_TRY(cudaSetDevice(d->device));
  auto* ix = new sl_index();
  ix->device = d->device;
  ix->params = d->params;
  ix->N = d->num_docs;
  ix->V = d->vocab_size;
  ix->doc_base = d->doc_base;
  ix->comm = d->comm;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    delete ix;
    SL_FAIL(SL_ECUDA, "sl_index_build: stream creation failed");
  }
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d->device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  t_build_stream = st;
  bool agreed = false;
  int32_t rc = build_body(d, ix, st, &agreed);
  // a rank that failed before the statistics all-reduce still takes part in the agreement
  if (rc != SL_OK && d->comm && !d->global_df && !agreed) rc = comm_agree(d->comm, rc);
  t_build_stream = nullptr;
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc != SL_OK) {
    free_index(ix);
    return rc;
  }
  *out = ix;
  return SL_OK;
}

// Device index from host CSC arrays (index loading, SPEC load_index): validates the
// ScoreMatrix invariants on the device, uploads, rebuilds the query-side structures.
namespace {
__global__ void k_row_starts(const uint64_t* __restrict__ indptr, uint32_t V, uint8_t* __restrict__ start) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < V; t += gridDim.x * blockDim.x)
    if (indptr[t] < indptr[t + 1]) start[indptr[t]] = 1;
}
__global__ void k_check_rows(const uint32_t* __restrict__ docids, const uint8_t* __restrict__ start, uint64_t nnz,
                             uint32_t N, uint32_t* err) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = docids[p];
    if (d >= N || (!start[p] && p > 0 && d <= docids[p - 1])) atomicOr(err, 1u);
  }
}
}  // namespace

int32_t load_index_from_host(const HostIndex& h, int device, float dense_min_density, sl_index** out) {
  *out = nullptr;
  SL_TRY(host_validate(h.params));
  const uint32_t V = h.V, N = h.N;
  const uint64_t nnz = h.indptr.empty() ? 0 : h.indptr.back();
  if (h.indptr.size() != (size_t)V + 1 || h.indptr[0] != 0)
    SL_FAIL(SL_ECORRUPT, "load_index: corrupt matrix (indptr length/origin)");
  for (uint32_t t = 0; t < V; ++t)
    if (h.indptr[t + 1] < h.indptr[t]) SL_FAIL(SL_ECORRUPT, "load_index: corrupt matrix (indptr decreasing)");
  if (h.docids.size() != nnz || h.values.size() != nnz)
    SL_FAIL(SL_ECORRUPT, "load_index: corrupt matrix (indptr[V] != number of stored entries)");
  if (h.df.size() != V || h.theta.size() != V || h.doclens.size() != N)
    SL_FAIL(SL_ECORRUPT, "load_index: corrupt matrix (array length mismatch)");
  for (uint32_t t = 0; t < V; ++t) {
    const uint64_t rl = h.indptr[t + 1] - h.indptr[t];
    if (h.df[t] < rl || (h.N_global == N && h.df[t] != rl))
      SL_FAIL(SL_ECORRUPT, "load_index: corrupt matrix (df does not match row lengths)");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    SL_FAIL(SL_ECUDA, "load_index: no CUDA device available (there is no CPU fallback)");
  SL_CUDA_TRY(cudaSetDevice(device));
  auto* ix = new sl_index();
  ix->device = device;
  ix->params = h.params;
  ix->N = N;
  ix->V = V;
  ix->doc_base = h.doc_base;
  ix->N_global = h.N_global;
  ix->total_len = h.total_len;
  ix->avg_len = h.avg_len;
  ix->nnz = nnz;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    delete ix;
    SL_FAIL(SL_ECUDA, "load_index: stream creation failed");
  }
  t_build_stream = st;
  auto body = [&]() -> int32_t {
    SL_TRY(dalloc(ix, &ix->indptr, (uint64_t)V + 1));
    SL_TRY(dalloc(ix, &ix->docids, nnz));
    SL_TRY(dalloc(ix, &ix->values, nnz));
    SL_TRY(dalloc(ix, &ix->df_global, V));
    SL_TRY(dalloc(ix, &ix->theta, V));
    SL_TRY(dalloc(ix, &ix->doclens, N));
    SL_CUDA_TRY(cudaMemcpyAsync(ix->indptr, h.indptr.data(), ((uint64_t)V + 1) * 8, cudaMemcpyHostToDevice, st));
    if (nnz) {
      SL_CUDA_TRY(cudaMemcpyAsync(ix->docids, h.docids.data(), nnz * 4, cudaMemcpyHostToDevice, st));
      SL_CUDA_TRY(cudaMemcpyAsync(ix->values, h.values.data(), nnz * 4, cudaMemcpyHostToDevice, st));
    }
    SL_CUDA_TRY(cudaMemcpyAsync(ix->df_global, h.df.data(), (uint64_t)V * 4, cudaMemcpyHostToDevice, st));
    SL_CUDA_TRY(cudaMemcpyAsync(ix->theta, h.theta.data(), (uint64_t)V * 4, cudaMemcpyHostToDevice, st));
    SL_CUDA_TRY(cudaMemcpyAsync(ix->doclens, h.doclens.data(), (uint64_t)N * 4, cudaMemcpyHostToDevice, st));
    if (nnz) {  // strictly increasing doc ids per row, all < N (SPEC ScoreMatrix invariants)
      Temps tmp(st);
      uint8_t* start;
      uint32_t* err;
      SL_TRY(tmp.alloc(&start, nnz));
      SL_TRY(tmp.alloc(&err, 1));
      SL_CUDA_TRY(cudaMemsetAsync(start, 0, nnz, st));
      SL_CUDA_TRY(cudaMemsetAsync(err, 0, 4, st));
      k_row_starts<<<grid_for(V, 256), 256, 0, st>>>(ix->indptr, V, start); ++t_launches;
      k_check_rows<<<grid_for(nnz, 256), 256, 0, st>>>(ix->docids, start, nnz, N, err); ++t_launches;
      uint32_t herr = 0;
      SL_CUDA_TRY(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));
      SL_CUDA_TRY(cudaStreamSynchronize(st));
      if (herr) SL_FAIL(SL_ECORRUPT, "load_index: corrupt matrix (doc ids not strictly increasing or >= num_docs)");
    }
    ix->build_ms = 0.f;
    return build_query_structures(ix, dense_min_density, st);
  };
  const int32_t rc = body();
  cudaStreamSynchronize(st);
  t_build_stream = nullptr;
  cudaStreamDestroy(st);
  if (rc != SL_OK) {
    free_index(ix);
    return rc;
  }
  *out = ix;
  return SL_OK;
}

}  // namespace sl
