// sl_query.cu — batched query scoring + top-k on the device (SPEC.md [MODULE] retrieval).
//
// Reference semantics (SPEC retrieval): score_query accumulates each query token's
// contiguous slice into a zeroed |C| accumulator and adds Σ S^θ; top_k selects the k
// best with ties -> smaller doc index; retrieve_batch runs both per query.
//
// B200 design:
//   * doc-tiled scoring: a CTA owns (query, contiguous run of 2048-doc tiles). The
//     tile's scores live in shared memory (8 KB) and never touch HBM; the |C| vector of
//     the reference is never materialised.
//   * rows with global df >= density*N have a dense f32 copy: their contribution is a
//     coalesced float4 stream accumulated in registers (no indirection, no atomics);
//   * remaining rows are gathered per tile from the CSC slice [s, e) found through a
//     per-tile skip table (long rows) or a warp ballot over a cursor (short rows), and
//     added to the shared accumulator one token at a time (doc ids are unique within a
//     row, so no atomics are needed). Every document sums its terms in query order
//     whatever the dense/gathered split, tile split or GPU count: bit-identical results;
//   * fused top-k: each CTA keeps its running best keys (u64 = orderable(score)<<32 |
//     ~doc) in shared memory behind a threshold; overflow triggers an in-CTA MSD radix
//     select; the per-split winners are merged per query by k_merge (also the rank-0
//     merge of the G x k candidates gathered over NCCL).
#include <algorithm>
#include <cstring>
#include <vector>

#include "sl_index.cuh"

namespace sl {
namespace {

constexpr int NT = kScoreThreads;
constexpr int NW = NT / 32;
constexpr int TILE = kTileDocs;
constexpr int F4 = TILE / (4 * NT);  // float4 per thread per tile
static_assert(F4 * 4 * NT == TILE, "tile must be a multiple of 4*threads");

enum Mode { MODE_TOPK = 0, MODE_DENSE = 1, MODE_VECTOR = 2 };

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

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
  *total = sw[32];
  __syncthreads();
  return r;
}

// MSD radix select over u64 keys (8-bit digits): returns tau such that exactly k of the
// visited keys are >= tau. Requires more than k keys. `visit(f)` calls f(key) for every
// key this thread owns. hist: 256 u32, bc: 3 u32 (shared).
template <class Visit>
__device__ uint64_t block_select_kth(Visit visit, uint32_t k, uint32_t* hist, uint32_t* bc) {
  uint64_t prefix = 0, mask = 0;
  uint32_t need = k;
  const int lane = threadIdx.x & 31;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    visit([&](uint64_t x) {
      if ((x & mask) == prefix) atomicAdd(&hist[(uint32_t)(x >> shift) & 255u], 1u);
    });
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t c[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[255 - (8 * lane + j)];
        s += c[j];
      }
      const uint32_t incl = warp_incl_scan(s), excl = incl - s;
      if (excl < need && need <= incl) {
        uint32_t run = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (run + c[j] >= need) {
            bc[0] = 255u - (8u * lane + j);
            bc[1] = run;
            bc[2] = c[j];
            break;
          }
          run += c[j];
        }
      }
    }
    __syncthreads();
    const uint32_t b = bc[0], above = bc[1], cnt = bc[2];
    need -= above;
    prefix |= (uint64_t)b << shift;
    mask |= 0xFFull << shift;
    __syncthreads();
    if (cnt == need) break;
  }
  return prefix;
}

// descending bitonic sort of n (power of two) keys in shared memory
__device__ void block_bitonic_desc(uint64_t* buf, uint32_t n) {
  for (uint32_t size = 2; size <= n; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const uint32_t lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const uint64_t a = buf[lo], b = buf[hi];
        if ((a < b) == desc) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

__host__ __device__ inline uint32_t next_pow2(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

__host__ __device__ inline uint32_t kept_capacity(uint32_t k) {
  const uint32_t c = 2 * next_pow2(k);
  return c < 512 ? 512 : c;
}

// dynamic shared memory layout of the scoring kernel
struct Smem {
  float* acc;          // [TILE]
  uint64_t* kept[2];   // [C] each
  uint64_t* row_start; // [qmax]
  uint32_t* hist;      // [256]
  uint32_t* sw;        // [40]
  int32_t* dslot;      // [qmax]
  uint32_t* row_len;   // [qmax]
  int32_t* skip;       // [qmax]
  uint32_t* cursor;    // [qmax]
  uint32_t* rs;        // [qmax]
  uint32_t* re;        // [qmax]
  int32_t* counts;     // [4] nd, ns
};

__host__ __device__ inline size_t smem_bytes(uint32_t C, uint32_t qmax) {
  return (size_t)TILE * 4 + 2 * (size_t)C * 8 + (size_t)qmax * 8 + 256 * 4 + 40 * 4 +
         (size_t)qmax * 4 * 6 + 16;
}

__device__ inline Smem carve(unsigned char* base, uint32_t C, uint32_t qmax) {
  Smem s;
  unsigned char* p = base;
  s.acc = (float*)p; p += (size_t)TILE * 4;
  s.kept[0] = (uint64_t*)p; p += (size_t)C * 8;
  s.kept[1] = (uint64_t*)p; p += (size_t)C * 8;
  s.row_start = (uint64_t*)p; p += (size_t)qmax * 8;
  s.hist = (uint32_t*)p; p += 256 * 4;
  s.sw = (uint32_t*)p; p += 40 * 4;
  s.dslot = (int32_t*)p; p += (size_t)qmax * 4;
  s.row_len = (uint32_t*)p; p += (size_t)qmax * 4;
  s.skip = (int32_t*)p; p += (size_t)qmax * 4;
  s.cursor = (uint32_t*)p; p += (size_t)qmax * 4;
  s.rs = (uint32_t*)p; p += (size_t)qmax * 4;
  s.re = (uint32_t*)p; p += (size_t)qmax * 4;
  s.counts = (int32_t*)p;
  return s;
}

struct QueryArgs {
  const uint64_t* q_off;   // [B+1] (absolute offsets into q_tok)
  const uint32_t* q_tok;
  const double* qconst;    // [B] Σ S^θ
  uint32_t B;
  uint32_t k;
  uint32_t C;              // kept capacity
  uint32_t qmax;
  uint32_t n_splits;
  uint64_t* cand;          // [B][n_splits][k] (MODE_TOPK / MODE_VECTOR)
  float* dense_out;        // [N] (MODE_DENSE)
  const float* vec;        // [n] input scores (MODE_VECTOR)
  uint32_t vec_n;
};

// Score one tile of one query into s.acc (local doc d0 .. d0+TILE).
// Entries are the query's tokens in QUERY ORDER: dense copies (dslot >= 0) are streamed
// as float4 and accumulated in registers; a CSC-gathered token (dslot < 0) spills the
// registers to the shared accumulator, scatters its slice, and reloads. Every document
// therefore sums its terms in query order, whatever the dense/gathered split, tile split
// or GPU count (bit-identical results across all of them).
__device__ __forceinline__ void score_tile(const IndexView& ix, const Smem& s, int ne, uint32_t tile,
                                           uint32_t d0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t d1 = d0 + TILE;
  // slice [rs, re) of every gathered row within this tile (one warp per row)
  for (int e = warp; e < ne; e += NW) {
    if (s.dslot[e] >= 0) continue;
    uint32_t sb, se;
    const int32_t sk = s.skip[e];
    if (sk >= 0) {
      const uint32_t* tab = ix.skiptab + (uint64_t)sk * (ix.num_tiles + 1);
      sb = tab[tile];
      se = tab[tile + 1];
    } else {
      uint32_t cur = s.cursor[e];
      const uint32_t len = s.row_len[e];
      const uint32_t* ids = ix.docids + s.row_start[e];
      sb = cur;
      while (true) {
        const uint32_t idx = cur + lane;
        const bool in = idx < len && __ldg(ids + idx) < d1;
        const uint32_t c = __popc(__ballot_sync(0xffffffffu, in));
        cur += c;
        if (c < 32) break;
      }
      se = cur;
      if (lane == 0) s.cursor[e] = cur;
    }
    if (lane == 0) {
      s.rs[e] = sb;
      s.re[e] = se;
    }
  }
  float4 a[F4];
#pragma unroll
  for (int r = 0; r < F4; ++r) a[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  float4* acc4 = reinterpret_cast<float4*>(s.acc);
  bool in_smem = false;
  for (int e = 0; e < ne; ++e) {
    const int32_t slot = s.dslot[e];
    if (slot >= 0) {
      if (in_smem) {
#pragma unroll
        for (int r = 0; r < F4; ++r) a[r] = acc4[threadIdx.x + r * NT];
        in_smem = false;
      }
      const float4* row = reinterpret_cast<const float4*>(ix.dense + (uint64_t)slot * ix.n_pad + d0);
#pragma unroll
      for (int r = 0; r < F4; ++r) {
        const float4 v = __ldg(row + threadIdx.x + r * NT);
        a[r].x += v.x;
        a[r].y += v.y;
        a[r].z += v.z;
        a[r].w += v.w;
      }
    } else {
      if (!in_smem) {
#pragma unroll
        for (int r = 0; r < F4; ++r) acc4[threadIdx.x + r * NT] = a[r];
        in_smem = true;
        __syncthreads();
      }
      const uint32_t sb = s.rs[e], se = s.re[e];
      if (sb == se) continue;
      const uint64_t base = s.row_start[e];
      // doc ids are unique within a row: plain shared-memory RMW, no atomics
      for (uint32_t p = sb + threadIdx.x; p < se; p += NT) {
        const uint32_t doc = __ldg(ix.docids + base + p);
        s.acc[doc - d0] += __ldg(ix.values + base + p);
      }
      __syncthreads();
    }
  }
  if (!in_smem) {
#pragma unroll
    for (int r = 0; r < F4; ++r) acc4[threadIdx.x + r * NT] = a[r];
  }
  __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(NT) k_score_topk(IndexView ix, QueryArgs qa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Smem s = carve(smem_raw, qa.C, qa.qmax);
  const uint32_t q = blockIdx.x / qa.n_splits;
  const uint32_t split = blockIdx.x % qa.n_splits;
  const uint32_t n_docs = MODE == MODE_VECTOR ? qa.vec_n : ix.N;
  const uint32_t n_tiles = (n_docs + TILE - 1) / TILE;
  const uint32_t t0 = (uint32_t)((uint64_t)split * n_tiles / qa.n_splits);
  const uint32_t t1 = (uint32_t)((uint64_t)(split + 1) * n_tiles / qa.n_splits);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  int ne = 0;
  if constexpr (MODE != MODE_VECTOR) {
    // the query's tokens in query order (OOV / locally empty rows dropped)
    if (threadIdx.x == 0) {
      const uint64_t qb = qa.q_off[q], qe = qa.q_off[q + 1];
      int c = 0;
      for (uint64_t j = qb; j < qe; ++j) {
        const uint32_t t = qa.q_tok[j];
        if (t >= ix.V || ix.df_global[t] == 0) continue;  // OOV drop (SPEC tokenizer decisions)
        const uint64_t rb = ix.indptr[t], re = ix.indptr[t + 1];
        if (rb == re) continue;  // no local postings
        const int32_t info = ix.tokinfo[t];
        s.dslot[c] = info >= 0 ? info : -1;
        s.row_start[c] = rb;
        s.row_len[c] = (uint32_t)(re - rb);
        s.skip[c] = info <= -2 ? -2 - info : -1;
        ++c;
      }
      s.counts[0] = c;
    }
    __syncthreads();
    ne = s.counts[0];
    // cursors of short rows at the split's first doc (lower_bound, one lane per row)
    const uint32_t dstart = t0 * TILE;
    for (int e = warp; e < ne; e += NW) {
      if (lane == 0 && s.dslot[e] < 0 && s.skip[e] < 0) {
        const uint32_t* ids = ix.docids + s.row_start[e];
        uint32_t lo = 0, hi = s.row_len[e];
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (ids[mid] < dstart) lo = mid + 1; else hi = mid;
        }
        s.cursor[e] = lo;
      }
    }
    __syncthreads();
  }

  uint32_t n_kept = 0;
  uint64_t tau = 0;
  int cur = 0;
  const double qc = (MODE == MODE_VECTOR) ? 0.0 : qa.qconst[q];

  for (uint32_t tile = t0; tile < t1; ++tile) {
    const uint32_t d0 = tile * TILE;
    const uint32_t nvalid = min((uint32_t)TILE, n_docs - d0);
    if constexpr (MODE == MODE_VECTOR) {
      for (uint32_t i = threadIdx.x; i < TILE; i += NT) s.acc[i] = i < nvalid ? qa.vec[d0 + i] : 0.f;
      __syncthreads();
    } else {
      score_tile(ix, s, ne, tile, d0);
    }
    if constexpr (MODE == MODE_DENSE) {
      for (uint32_t i = threadIdx.x; i < nvalid; i += NT)
        qa.dense_out[d0 + i] = __double2float_rn((double)s.acc[i] + qc);
      __syncthreads();
      continue;
    }
    const uint32_t gdoc0 = (MODE == MODE_VECTOR ? 0u : ix.doc_base) + d0;
    // candidates of this tile that clear the running threshold
    auto tile_visit = [&](uint64_t thr, auto&& f) {
#pragma unroll
      for (int r = 0; r < F4; ++r) {
        const uint32_t dl = 4 * (threadIdx.x + r * NT);
        const float4 v = reinterpret_cast<const float4*>(s.acc)[threadIdx.x + r * NT];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (dl + c < nvalid) {
            const float x = c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
            const uint64_t key = make_key(x, gdoc0 + dl + c);
            if (key >= thr) f(key);
          }
        }
      }
    };
    uint32_t mine = 0;
    tile_visit(tau, [&](uint64_t) { ++mine; });
    uint32_t P;
    uint32_t off = block_excl_scan(mine, s.sw, &P);
    if (n_kept + P <= qa.C) {
      uint64_t* dst = s.kept[cur] + n_kept + off;
      tile_visit(tau, [&](uint64_t key) { *dst++ = key; });
      n_kept += P;
      __syncthreads();
    } else {
      const uint64_t* kb = s.kept[cur];
      const uint32_t nk = n_kept;
      const uint64_t old = tau;
      tau = block_select_kth(
          [&](auto&& f) {
            for (uint32_t i = threadIdx.x; i < nk; i += NT) f(kb[i]);
            tile_visit(old, f);
          },
          qa.k, s.hist, s.sw + 36);
      uint32_t m2 = 0;
      for (uint32_t i = threadIdx.x; i < nk; i += NT) m2 += kb[i] >= tau;
      tile_visit(tau, [&](uint64_t) { ++m2; });
      uint32_t tot;
      const uint32_t o2 = block_excl_scan(m2, s.sw, &tot);
      uint64_t* dst = s.kept[cur ^ 1] + o2;
      for (uint32_t i = threadIdx.x; i < nk; i += NT)
        if (kb[i] >= tau) *dst++ = kb[i];
      tile_visit(tau, [&](uint64_t key) { *dst++ = key; });
      n_kept = tot;
      cur ^= 1;
      __syncthreads();
    }
  }
  if constexpr (MODE == MODE_DENSE) return;
  else {

  // emit this split's best min(k, n_kept) keys, sorted descending
  if (n_kept > qa.k) {
    const uint64_t* kb = s.kept[cur];
    const uint32_t nk = n_kept;
    const uint64_t t2 = block_select_kth(
        [&](auto&& f) {
          for (uint32_t i = threadIdx.x; i < nk; i += NT) f(kb[i]);
        },
        qa.k, s.hist, s.sw + 36);
    uint32_t m2 = 0;
    for (uint32_t i = threadIdx.x; i < nk; i += NT) m2 += kb[i] >= t2;
    uint32_t tot;
    const uint32_t o2 = block_excl_scan(m2, s.sw, &tot);
    uint64_t* dst = s.kept[cur ^ 1] + o2;
    for (uint32_t i = threadIdx.x; i < nk; i += NT)
      if (kb[i] >= t2) *dst++ = kb[i];
    n_kept = tot;
    cur ^= 1;
    __syncthreads();
  }
  const uint32_t m = min(n_kept, qa.k);
  const uint32_t p2 = next_pow2(max(m, 2u));
  uint64_t* buf = s.kept[cur];
  for (uint32_t i = m + threadIdx.x; i < p2; i += NT) buf[i] = kInvalidKey;
  __syncthreads();
  block_bitonic_desc(buf, p2);
  uint64_t* out = qa.cand + ((uint64_t)q * qa.n_splits + split) * qa.k;
  for (uint32_t i = threadIdx.x; i < qa.k; i += NT) out[i] = i < m ? buf[i] : kInvalidKey;
  }
}

// Per query: top-k over n_splits x k candidate keys (invalid = 0), sorted, decoded.
__global__ void __launch_bounds__(256) k_merge(const uint64_t* __restrict__ cand, uint32_t n_splits,
                                               uint64_t split_stride, uint64_t query_stride, uint32_t k,
                                               const double* __restrict__ qconst, uint32_t* out_ids,
                                               float* out_scores, uint64_t* out_keys) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* buf = (uint64_t*)smem_raw;  // [p2]
  const uint32_t p2 = next_pow2(max(k, 2u));
  uint32_t* hist = (uint32_t*)(buf + p2);
  uint32_t* sw = hist + 256;
  const uint32_t q = blockIdx.x;
  const uint64_t* base = cand + (uint64_t)q * query_stride;
  const uint64_t total = (uint64_t)n_splits * k;
  auto at = [&](uint64_t i) { return base[(i / k) * split_stride + (i % k)]; };

  uint32_t mine = 0;
  for (uint64_t i = threadIdx.x; i < total; i += blockDim.x) mine += at(i) != kInvalidKey;
  uint32_t nvalid;
  block_excl_scan(mine, sw, &nvalid);
  uint64_t tau = 1;
  if (nvalid > k) {
    tau = block_select_kth(
        [&](auto&& f) {
          for (uint64_t i = threadIdx.x; i < total; i += blockDim.x) {
            const uint64_t x = at(i);
            if (x != kInvalidKey) f(x);
          }
        },
        k, hist, sw + 36);
  }
  uint32_t m2 = 0;
  for (uint64_t i = threadIdx.x; i < total; i += blockDim.x) m2 += at(i) >= tau;
  uint32_t m;
  const uint32_t o = block_excl_scan(m2, sw, &m);
  uint64_t* dst = buf + o;
  for (uint64_t i = threadIdx.x; i < total; i += blockDim.x) {
    const uint64_t x = at(i);
    if (x >= tau) *dst++ = x;
  }
  for (uint32_t i = m + threadIdx.x; i < p2; i += blockDim.x) buf[i] = kInvalidKey;
  __syncthreads();
  block_bitonic_desc(buf, p2);
  const double qc = qconst ? qconst[q] : 0.0;
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
    const uint64_t key = i < m ? buf[i] : kInvalidKey;
    if (out_keys) out_keys[(uint64_t)q * k + i] = key;
    if (out_ids) out_ids[(uint64_t)q * k + i] = i < m ? key_doc(key) : 0xFFFFFFFFu;
    if (out_scores)
      out_scores[(uint64_t)q * k + i] =
          i < m ? __double2float_rn((double)key_score(key) + qc) : -INFINITY;
  }
}

// Per query: validation, Σ S^θ (f64, query order), max length, algorithmic posting bytes.
__global__ void k_query_prep(const uint64_t* __restrict__ q_off, const uint32_t* __restrict__ q_tok,
                             uint32_t B, IndexView ix, double* __restrict__ qconst,
                             uint32_t* __restrict__ info /*[0]=err [1]=qmax*/,
                             unsigned long long* __restrict__ bytes) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < B; q += gridDim.x * blockDim.x) {
    const uint64_t b = q_off[q], e = q_off[q + 1];
    if (e < b) {
      atomicOr(&info[0], 2u);
      qconst[q] = 0.0;
      continue;
    }
    atomicMax(&info[1], (uint32_t)min(e - b, (uint64_t)0xFFFFFFFFu));
    double c = 0.0;
    unsigned long long pb = 0;
    for (uint64_t j = b; j < e; ++j) {
      const uint32_t t = q_tok[j];
      if (t >= ix.V) {
        atomicOr(&info[0], 1u);
        continue;
      }
      if (ix.df_global[t] == 0) continue;
      c += (double)ix.theta[t];
      pb += 8ull * (ix.indptr[t + 1] - ix.indptr[t]);
    }
    qconst[q] = c;
    if (bytes && pb) atomicAdd(bytes, pb);
  }
}

struct StreamCache {
  int device = -1;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[4] = {};
};
thread_local StreamCache t_stream[16];

int32_t get_stream(int device, StreamCache** out) {
  if (device < 0 || device >= 16) SL_FAIL(SL_EINVAL, "device ordinal out of range");
  StreamCache& c = t_stream[device];
  if (!c.st) {
    SL_CUDA_TRY(cudaSetDevice(device));
    SL_CUDA_TRY(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
    for (auto& e : c.ev) SL_CUDA_TRY(cudaEventCreate(&e));
    c.device = device;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  SL_CUDA_TRY(cudaSetDevice(device));
  *out = &c;
  return SL_OK;
}

struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <class T>
  int32_t alloc(T** p, uint64_t count) {
    if (count == 0) count = 1;
    cudaError_t e = cudaMallocAsync((void**)p, count * sizeof(T), st);
    if (e != cudaSuccess) {
      *p = nullptr;
      set_error(std::string("scratch allocation failed: ") + cudaGetErrorString(e));
      return SL_ENOMEM;
    }
    ptrs.push_back(*p);
    return SL_OK;
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

int num_sms(int device) {
  static int cache[16] = {0};
  if (!cache[device]) cudaDeviceGetAttribute(&cache[device], cudaDevAttrMultiProcessorCount, device);
  return cache[device];
}

template <int MODE>
int32_t launch_score(const IndexView& ix, QueryArgs& qa, cudaStream_t st, int device, uint32_t n_docs,
                     uint32_t n_blocks_per_item_hint) {
  const size_t smem = smem_bytes(qa.C, qa.qmax);
  if (smem > 227 * 1024) SL_FAIL(SL_EUNSUPPORTED, "top-k / query length too large for shared memory");
  SL_CUDA_TRY(cudaFuncSetAttribute(k_score_topk<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const uint32_t n_tiles = (n_docs + TILE - 1) / TILE;
  if (n_blocks_per_item_hint) {
    qa.n_splits = std::min(n_blocks_per_item_hint, std::max(1u, n_tiles));
  } else {
    int per_sm = 0;
    SL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_score_topk<MODE>, NT, smem));
    const uint64_t target = (uint64_t)std::max(1, per_sm) * num_sms(device) * 2;
    uint64_t ns = (target + qa.B - 1) / qa.B;
    ns = std::max<uint64_t>(1, std::min<uint64_t>(ns, std::max(1u, n_tiles)));
    qa.n_splits = (uint32_t)ns;
  }
  const uint64_t grid = (uint64_t)qa.B * qa.n_splits;
  if (grid > 0x7FFFFFFFull) SL_FAIL(SL_EUNSUPPORTED, "query batch too large");
  k_score_topk<MODE><<<(unsigned)grid, NT, smem, st>>>(ix, qa);
  SL_CUDA_TRY(cudaGetLastError());
  return SL_OK;
}

int32_t launch_merge(const uint64_t* cand, uint32_t B, uint32_t n_splits, uint64_t split_stride,
                     uint64_t query_stride, uint32_t k, const double* qconst, uint32_t* ids, float* scores,
                     uint64_t* keys, cudaStream_t st) {
  const size_t smem = (size_t)next_pow2(std::max(k, 2u)) * 8 + 256 * 4 + 40 * 4;
  SL_CUDA_TRY(cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_merge<<<B, 256, smem, st>>>(cand, n_splits, split_stride, query_stride, k, qconst, ids, scores, keys);
  SL_CUDA_TRY(cudaGetLastError());
  return SL_OK;
}

}  // namespace

// ------------------------------------------------------------------ entry points
int32_t retrieve_impl(const sl_index* ix, const uint64_t* q_offsets, const uint32_t* q_tokens, uint32_t B,
                      uint32_t k, int32_t mem, uint32_t* out_ids, float* out_scores, sl_retrieve_stats* stats) {
  if (!ix) SL_FAIL(SL_EINVAL, "retrieve_batch: null index");
  if (k == 0) SL_FAIL(SL_EINVAL, "top_k: k must be >= 1");
  if (k > kMaxK) SL_FAIL(SL_EUNSUPPORTED, "retrieve_batch: k > 4096 is not supported by the fused top-k");
  if (mem != SL_MEM_HOST && mem != SL_MEM_DEVICE) SL_FAIL(SL_EINVAL, "retrieve_batch: bad mem kind");
  const bool dist = ix->comm && ix->comm->nranks > 1;
  const bool want_out = !dist || ix->comm->rank == 0;
  if (B == 0) return SL_OK;
  if (!q_offsets || !q_tokens) SL_FAIL(SL_EINVAL, "retrieve_batch: null query pointers");
  if (want_out && (!out_ids || !out_scores)) SL_FAIL(SL_EINVAL, "retrieve_batch: null output pointers");
  StreamCache* sc;
  SL_TRY(get_stream(ix->device, &sc));
  cudaStream_t st = sc->st;
  Scratch scr(st);

  // queries on the device
  const uint64_t* d_off = q_offsets;
  const uint32_t* d_tok = q_tokens;
  uint64_t ntok = 0;
  if (mem == SL_MEM_HOST) {
    ntok = q_offsets[B];
    uint64_t* o;
    uint32_t* t;
    SL_TRY(scr.alloc(&o, (uint64_t)B + 1));
    SL_TRY(scr.alloc(&t, ntok));
    SL_CUDA_TRY(cudaMemcpyAsync(o, q_offsets, ((uint64_t)B + 1) * 8, cudaMemcpyHostToDevice, st));
    if (ntok) SL_CUDA_TRY(cudaMemcpyAsync(t, q_tokens, ntok * 4, cudaMemcpyHostToDevice, st));
    d_off = o;
    d_tok = t;
  }
  SL_CUDA_TRY(cudaEventRecord(sc->ev[0], st));
  const IndexView v = ix->view();
  double* qconst;
  uint32_t* info;
  unsigned long long* bytes;
  SL_TRY(scr.alloc(&qconst, B));
  SL_TRY(scr.alloc(&info, 4));
  SL_TRY(scr.alloc(&bytes, 1));
  SL_CUDA_TRY(cudaMemsetAsync(info, 0, 16, st));
  SL_CUDA_TRY(cudaMemsetAsync(bytes, 0, 8, st));
  k_query_prep<<<(B + 255) / 256, 256, 0, st>>>(d_off, d_tok, B, v, qconst, info, bytes);
  SL_CUDA_TRY(cudaGetLastError());
  uint32_t h_info[4];
  SL_CUDA_TRY(cudaMemcpyAsync(h_info, info, 16, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_info[0] & 2u) SL_FAIL(SL_EINVAL, "retrieve_batch: query offsets must be non-decreasing");
  if (h_info[0] & 1u) SL_FAIL(SL_EINVAL, "score_query: token id >= vocab size");
  if (h_info[1] > (uint32_t)kQMax) SL_FAIL(SL_EUNSUPPORTED, "retrieve_batch: queries longer than 256 tokens are not supported");

  QueryArgs qa{};
  qa.q_off = d_off;
  qa.q_tok = d_tok;
  qa.qconst = qconst;
  qa.B = B;
  qa.k = k;
  qa.C = kept_capacity(k);
  qa.qmax = std::max(1u, h_info[1]);
  SL_CUDA_TRY(cudaEventRecord(sc->ev[1], st));
  // split count is known only inside launch_score; allocate for the worst case first
  {
    const size_t smem = smem_bytes(qa.C, qa.qmax);
    if (smem > 227 * 1024) SL_FAIL(SL_EUNSUPPORTED, "top-k / query length too large for shared memory");
  }
  int per_sm = 0;
  {
    const size_t smem = smem_bytes(qa.C, qa.qmax);
    SL_CUDA_TRY(cudaFuncSetAttribute(k_score_topk<MODE_TOPK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_score_topk<MODE_TOPK>, NT, smem));
  }
  const uint32_t n_tiles = std::max(1u, ix->num_tiles);
  const uint64_t target = (uint64_t)std::max(1, per_sm) * num_sms(ix->device) * 2;
  const uint32_t n_splits = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((target + B - 1) / B, n_tiles));
  uint64_t* cand;
  SL_TRY(scr.alloc(&cand, (uint64_t)B * n_splits * k));
  qa.cand = cand;
  SL_TRY(launch_score<MODE_TOPK>(v, qa, st, ix->device, ix->N, n_splits));
  SL_CUDA_TRY(cudaEventRecord(sc->ev[2], st));

  uint32_t* ids_dev = nullptr;
  float* sc_dev = nullptr;
  if (want_out) {
    if (mem == SL_MEM_DEVICE) {
      ids_dev = out_ids;
      sc_dev = out_scores;
    } else {
      SL_TRY(scr.alloc(&ids_dev, (uint64_t)B * k));
      SL_TRY(scr.alloc(&sc_dev, (uint64_t)B * k));
    }
  }
  if (!dist) {
    SL_TRY(launch_merge(cand, B, qa.n_splits, k, (uint64_t)qa.n_splits * k, k, qconst, ids_dev, sc_dev,
                        nullptr, st));
  } else {
    // local merge -> keys, gather the G x k candidates on rank 0 (NCCL), merge there
    const sl_comm* cm = ix->comm;
    uint64_t* local;
    SL_TRY(scr.alloc(&local, (uint64_t)B * k));
    SL_TRY(launch_merge(cand, B, qa.n_splits, k, (uint64_t)qa.n_splits * k, k, nullptr, nullptr, nullptr, local,
                        st));
    uint64_t* gathered = nullptr;
    if (cm->rank == 0) SL_TRY(scr.alloc(&gathered, (uint64_t)cm->nranks * B * k));
    const size_t cnt = (size_t)B * k;
    SL_TRY(nccl_check(nccl().GroupStart(), "ncclGroupStart"));
    if (cm->rank == 0) {
      for (int r = 0; r < cm->nranks; ++r)
        SL_TRY(nccl_check(nccl().Recv(gathered + (uint64_t)r * cnt, cnt, ncclUint64, r, cm->comm, st), "ncclRecv"));
    }
    SL_TRY(nccl_check(nccl().Send(local, cnt, ncclUint64, 0, cm->comm, st), "ncclSend"));
    SL_TRY(nccl_check(nccl().GroupEnd(), "ncclGroupEnd"));
    if (cm->rank == 0)
      SL_TRY(launch_merge(gathered, B, (uint32_t)cm->nranks, cnt, k, k, qconst, ids_dev, sc_dev, nullptr, st));
  }
  SL_CUDA_TRY(cudaEventRecord(sc->ev[3], st));
  if (want_out && mem == SL_MEM_HOST) {
    SL_CUDA_TRY(cudaMemcpyAsync(out_ids, ids_dev, (uint64_t)B * k * 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(out_scores, sc_dev, (uint64_t)B * k * 4, cudaMemcpyDeviceToHost, st));
  }
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  if (stats) {
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, sc->ev[0], sc->ev[3]);
    cudaEventElapsedTime(&b, sc->ev[1], sc->ev[2]);
    cudaEventElapsedTime(&c, sc->ev[2], sc->ev[3]);
    unsigned long long hb = 0;
    cudaMemcpy(&hb, bytes, 8, cudaMemcpyDeviceToHost);
    stats->total_ms = a;
    stats->score_kernel_ms = b;
    stats->merge_ms = c;
    stats->posting_bytes = hb;
    stats->scorevec_bytes = 4ull * ix->N * B;
    stats->unique_posting_bytes = 0;
    stats->kernels_launched = dist ? (ix->comm->rank == 0 ? 4 : 3) : 3;
  }
  return SL_OK;
}

int32_t score_query_impl(const sl_index* ix, const uint32_t* q_tokens, uint32_t q_len, int32_t mem, float* out) {
  if (!ix || !out) SL_FAIL(SL_EINVAL, "score_query: null argument");
  if (q_len > (uint32_t)kQMax) SL_FAIL(SL_EUNSUPPORTED, "score_query: query longer than 256 tokens");
  StreamCache* sc;
  SL_TRY(get_stream(ix->device, &sc));
  cudaStream_t st = sc->st;
  Scratch scr(st);
  uint64_t h_off[2] = {0, q_len};
  uint64_t* d_off;
  uint32_t* d_tok;
  float* d_out = out;
  SL_TRY(scr.alloc(&d_off, 2));
  SL_TRY(scr.alloc(&d_tok, std::max(1u, q_len)));
  SL_CUDA_TRY(cudaMemcpyAsync(d_off, h_off, 16, cudaMemcpyHostToDevice, st));
  if (q_len)
    SL_CUDA_TRY(cudaMemcpyAsync(d_tok, q_tokens, (uint64_t)q_len * 4,
                                mem == SL_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
  if (mem == SL_MEM_HOST) SL_TRY(scr.alloc(&d_out, ix->N));
  const IndexView v = ix->view();
  double* qconst;
  uint32_t* info;
  SL_TRY(scr.alloc(&qconst, 1));
  SL_TRY(scr.alloc(&info, 4));
  SL_CUDA_TRY(cudaMemsetAsync(info, 0, 16, st));
  k_query_prep<<<1, 32, 0, st>>>(d_off, d_tok, 1, v, qconst, info, nullptr);
  uint32_t h_info[4];
  SL_CUDA_TRY(cudaMemcpyAsync(h_info, info, 16, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_info[0] & 1u) SL_FAIL(SL_EINVAL, "score_query: token id >= vocab size");
  QueryArgs qa{};
  qa.q_off = d_off;
  qa.q_tok = d_tok;
  qa.qconst = qconst;
  qa.B = 1;
  qa.k = 1;
  qa.C = kept_capacity(1);
  qa.qmax = std::max(1u, q_len);
  qa.dense_out = d_out;
  SL_TRY(launch_score<MODE_DENSE>(v, qa, st, ix->device, ix->N, std::max(1u, ix->num_tiles)));
  if (mem == SL_MEM_HOST)
    SL_CUDA_TRY(cudaMemcpyAsync(out, d_out, (uint64_t)ix->N * 4, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  return SL_OK;
}

int32_t top_k_impl(const float* scores, uint32_t n, uint32_t k, int32_t mem, int32_t device, uint32_t* out_ids,
                   float* out_scores) {
  if (k == 0) SL_FAIL(SL_EINVAL, "top_k: k must be >= 1");
  if (k > kMaxK) SL_FAIL(SL_EUNSUPPORTED, "top_k: k > 4096 is not supported");
  if (!out_ids || !out_scores || (!scores && n)) SL_FAIL(SL_EINVAL, "top_k: null argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    SL_FAIL(SL_ECUDA, "top_k: no CUDA device available (there is no CPU fallback)");
  StreamCache* sc;
  SL_TRY(get_stream(device, &sc));
  cudaStream_t st = sc->st;
  Scratch scr(st);
  const float* d_in = scores;
  if (mem == SL_MEM_HOST && n) {
    float* t;
    SL_TRY(scr.alloc(&t, n));
    SL_CUDA_TRY(cudaMemcpyAsync(t, scores, (uint64_t)n * 4, cudaMemcpyHostToDevice, st));
    d_in = t;
  }
  uint32_t* ids_dev = out_ids;
  float* sc_dev = out_scores;
  if (mem == SL_MEM_HOST) {
    SL_TRY(scr.alloc(&ids_dev, k));
    SL_TRY(scr.alloc(&sc_dev, k));
  }
  IndexView v{};
  QueryArgs qa{};
  qa.B = 1;
  qa.k = k;
  qa.C = kept_capacity(k);
  qa.qmax = 1;
  qa.vec = d_in;
  qa.vec_n = n;
  const uint32_t n_tiles = std::max(1u, (n + TILE - 1) / TILE);
  const uint32_t n_splits = std::min<uint32_t>(n_tiles, 148 * 4);
  uint64_t* cand;
  SL_TRY(scr.alloc(&cand, (uint64_t)n_splits * k));
  qa.cand = cand;
  if (n) {
    SL_TRY(launch_score<MODE_VECTOR>(v, qa, st, device, n, n_splits));
  } else {
    qa.n_splits = 1;
    SL_CUDA_TRY(cudaMemsetAsync(cand, 0, (uint64_t)k * 8, st));
  }
  SL_TRY(launch_merge(cand, 1, qa.n_splits, k, (uint64_t)qa.n_splits * k, k, nullptr, ids_dev, sc_dev, nullptr, st));
  if (mem == SL_MEM_HOST) {
    SL_CUDA_TRY(cudaMemcpyAsync(out_ids, ids_dev, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(out_scores, sc_dev, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
  }
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  return SL_OK;
}

}  // namespace sl
