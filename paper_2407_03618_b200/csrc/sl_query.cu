// sl_query.cu — batched query scoring + top-k on the device (SPEC.md [MODULE] retrieval).
//
// Reference semantics (SPEC retrieval): score_query accumulates each query token's
// contiguous slice into a zeroed |C| accumulator and adds Σ S^θ; top_k selects the k
// best with ties -> smaller doc index; retrieve_batch runs both per query.
//
// B200 design. k_score_runs: queries are grouped by their DENSE SIGNATURE
// (the rows with a dense f32 copy, i.e. global df >= density*N) — sorted by a signature
// hash and cut into runs of <= R identical signatures. One WARP owns (run, doc split) and
// walks 1024-doc tiles with no CTA-level synchronisation:
//   1. the run's dense signature is summed once per tile, in registers, ascending slot
//      order, every lane streaming 8 float4 per row with all loads in flight;
//   2. per query of the run: lane j locates token j's CSC slice in the tile (per-tile skip
//      table for long rows, forward cursor for short rows); if the query has postings in
//      the tile, the dense sum is spilled to the warp's 4 KB shared accumulator and the
//      postings are flattened across tokens, loaded 4 x 32 at a time, and applied in
//      token order (same-doc postings inside a round serialised with match.any);
//   3. running top-k: float pre-test against the threshold, exact 64-bit keys
//      (orderable(score) << 32 | ~doc) for survivors into a per-query shared buffer;
//      overflow -> warp-level MSD radix select.
// The reference's |C| score vector is never materialised. Per document the sum is the
// dense terms (ascending slot) then the gathered terms (query order): a fixed function of
// the query and the global df classification — identical for any grouping, doc split or
// GPU count. k_merge selects the final top-k per query from the per-split candidates (and
// is the rank-0 merge of the G x k candidates gathered over NCCL).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_pipeline.h>

#include "sl_index.cuh"

namespace sl {
namespace {

constexpr int NT = 256;
#ifndef SL_DYN_WSMEM
#define SL_DYN_WSMEM (SL_TILE_DOCS > 512)  // per-warp layouts above 48 KB per CTA need dynamic smem
#endif
#ifndef SL_MINB
#define SL_MINB 4  // resident CTAs per SM the scoring kernel is register-budgeted for
#endif
constexpr int NW = NT / 32;
constexpr int TILE = kTileDocs;      // 512
constexpr int F4L = TILE / 4 / 32;   // float4 per lane when a warp scans one tile
static_assert(F4L * 128 == TILE, "a warp covers a tile with whole float4 per lane");

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

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

// Locate the bucket holding the need-th largest key from a 256-bin histogram (bins read
// high to low). Executed by one full warp; returns (bucket, count above, bucket count).
__device__ __forceinline__ void warp_pick_bucket(const uint32_t* hist, uint32_t need, uint32_t& b,
                                                 uint32_t& above, uint32_t& cnt) {
  const int lane = threadIdx.x & 31;
  uint32_t c[8], s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    c[j] = hist[255 - (8 * lane + j)];
    s += c[j];
  }
  const uint32_t incl = warp_incl_scan(s), excl = incl - s;
  const bool mine = excl < need && need <= incl;
  uint32_t lb = 0, la = 0, lc = 0;
  if (mine) {
    uint32_t run = excl;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (run + c[j] >= need) {
        lb = 255u - (8u * lane + j);
        la = run;
        lc = c[j];
        break;
      }
      run += c[j];
    }
  }
  const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
  b = __shfl_sync(0xffffffffu, lb, src);
  above = __shfl_sync(0xffffffffu, la, src);
  cnt = __shfl_sync(0xffffffffu, lc, src);
}

// MSD radix select over u64 keys (8-bit digits): returns tau such that exactly k of the
// visited keys are >= tau (keys are distinct). Requires more than k keys.
template <class Visit>
__device__ uint64_t block_select_kth(Visit visit, uint32_t k, uint32_t* hist, uint32_t* bc) {
  uint64_t prefix = 0, mask = 0;
  uint32_t need = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    visit([&](uint64_t x) {
      if ((x & mask) == prefix) atomicAdd(&hist[(uint32_t)(x >> shift) & 255u], 1u);
    });
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t b, a, c;
      warp_pick_bucket(hist, need, b, a, c);
      if (threadIdx.x == 0) {
        bc[0] = b;
        bc[1] = a;
        bc[2] = c;
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

#ifndef SL_DENSE_ASYNC
#define SL_DENSE_ASYNC 1
#endif
#ifndef SL_DCH
#define SL_DCH 4  // float4 per lane of one dense row in registers at a time (the dense pass's chunk)
#endif
#ifndef SL_TMA_EARLY
#define SL_TMA_EARLY 1  // the first dense row's bulk copy starts at the top of the tile
#endif
#ifndef SL_DENSE_TMA
#define SL_DENSE_TMA 1  // first dense row of a tile by one bulk copy (cp.async.bulk + mbarrier) per warp
#endif

// ---- 1-D bulk copy global -> shared completing on an mbarrier (Hopper+ TMA engine, no tensor map)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one lane: arm the barrier for `bytes` and start the copy (dst, src, bytes: 16-byte multiples)
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

// warp-level variant with 4-bit digits (16-bin warp-private histogram, 64 bytes)
template <class Visit>
__device__ uint64_t warp_select_kth(Visit visit, uint32_t k, uint32_t* hist) {
  const int lane = threadIdx.x & 31;
  uint64_t prefix = 0, mask = 0;
  uint32_t need = k;
  for (int shift = 60; shift >= 0; shift -= 4) {
    if (lane < 16) hist[lane] = 0;
    __syncwarp();
    visit([&](uint64_t x) {
      if ((x & mask) == prefix) atomicAdd(&hist[(uint32_t)(x >> shift) & 15u], 1u);
    });
    __syncwarp();
    const uint32_t c = lane < 16 ? hist[15 - lane] : 0u;  // buckets high -> low
    const uint32_t incl = warp_incl_scan(c), excl = incl - c;
    const bool mine = lane < 16 && excl < need && need <= incl;
    const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
    const uint32_t above = __shfl_sync(0xffffffffu, excl, src);
    const uint32_t cnt = __shfl_sync(0xffffffffu, c, src);
    __syncwarp();
    need -= above;
    prefix |= (uint64_t)(15 - src) << shift;
    mask |= 0xFull << shift;
    if (cnt == need) break;
  }
  return prefix;
}

#ifndef SL_BALLOT_SELECT
#define SL_BALLOT_SELECT 0  // measured: c2 top-10 -2.6%, c4 top-1000 -2.5% (register allocation)
#endif

// The exact k-th largest among the keys kept[0, nk) and this lane's tile candidates (bits of pm
// over buf, keys >= lo): MSD radix select with 4-bit digits like warp_select_kth, but the bin
// counts of each pass come from ballots instead of shared-memory atomics (lane b < 16 counts
// bin b from the four digit-bit ballots), so a pass costs a few warp-wide instructions per 32
// keys however skewed the digits are. Warp-synchronous: every lane runs the same trip counts.
__device__ __forceinline__ uint64_t warp_select_kth_tile(const uint64_t* kept, uint32_t nk, uint32_t pm,
                                                         const float* bf, uint32_t gdoc0, uint64_t lo, uint32_t k) {
  const int lane = threadIdx.x & 31;
  const uint32_t tile_iters = __reduce_max_sync(0xffffffffu, (uint32_t)__popc(pm));
  uint64_t prefix = 0, mask = 0;
  uint32_t need = k;
  for (int shift = 60; shift >= 0; shift -= 4) {
    uint32_t cnt = 0;
    auto add = [&](bool v, uint64_t x) {
      const bool m = v && (x & mask) == prefix;
      const uint32_t bm = __ballot_sync(0xffffffffu, m);
      if (!bm) return;
      const uint32_t d = (uint32_t)(x >> shift) & 15u;
      const uint32_t b0 = __ballot_sync(0xffffffffu, d & 1u), b1 = __ballot_sync(0xffffffffu, d & 2u);
      const uint32_t b2 = __ballot_sync(0xffffffffu, d & 4u), b3 = __ballot_sync(0xffffffffu, d & 8u);
      const uint32_t sel = bm & ((lane & 1) ? b0 : ~b0) & ((lane & 2) ? b1 : ~b1) & ((lane & 4) ? b2 : ~b2) &
                           ((lane & 8) ? b3 : ~b3);
      cnt += __popc(sel);
    };
    for (uint32_t base = 0; base < nk; base += 32) {
      const uint32_t i = base + lane;
      add(i < nk, i < nk ? kept[i] : 0ull);
    }
    uint32_t m = pm;
    for (uint32_t it = 0; it < tile_iters; ++it) {
      bool v = m != 0;
      uint64_t key = 0;
      if (v) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t dl = 4 * (lane + 32 * (bit >> 2)) + (bit & 3);
        key = make_key(bf[dl], gdoc0 + dl);
        v = key >= lo;
      }
      add(v, key);
    }
    // buckets high -> low: lane j < 16 takes bin 15 - j
    const uint32_t cj = __shfl_sync(0xffffffffu, cnt, 15 - (lane & 15));
    const uint32_t c = lane < 16 ? cj : 0u;
    const uint32_t incl = warp_incl_scan(c), excl = incl - c;
    const bool mine = lane < 16 && excl < need && need <= incl;
    const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
    const uint32_t above = __shfl_sync(0xffffffffu, excl, src);
    const uint32_t cb = __shfl_sync(0xffffffffu, c, src);
    need -= above;
    prefix |= (uint64_t)(15 - src) << shift;
    mask |= 0xFull << shift;
    if (cb == need) break;
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

// candidate buffer per (query, split)
__host__ __device__ inline uint32_t kept_capacity(uint32_t k) {
  const uint32_t c = 2 * next_pow2(k);
  return c < 64 ? 64 : c;
}

// float lower bound of every key >= tau (for the cheap pre-test)
// x > tau_float(tau) <=> orderable(x) > hi(tau). hi = 0x7FFFFFFF (a split threshold published
// one ordinal below a score of 0) is no float's ordinal since -0 and +0 share one: its float
// would be -0.0, and +0 > -0 is false, so it maps to the largest negative float instead.
__device__ __forceinline__ float tau_float(uint64_t tau) {
  const uint32_t hi = (uint32_t)(tau >> 32);
  if (hi == 0x7FFFFFFFu) return __uint_as_float(0x80000001u);
  return hi < 0x00800000u ? -INFINITY : ord_to_float(hi);
}

__device__ __forceinline__ float f4c(const float4& v, int c) {
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}

enum GroupMode { GM_TOPK = 0, GM_DENSE = 1 };

#ifndef SL_ULOG
#define SL_ULOG 8
#endif
constexpr int ULOG = SL_ULOG;  // undo-log capacity in gather slots
#ifndef SL_RMAX_CT
#define SL_RMAX_CT 4  // up to four queries of one dense signature per warp item (all but the last via the undo log)
#endif
constexpr int RMAX = SL_RMAX_CT;  // queries per run (same dense signature) handled by one warp
#ifndef SL_UNROLL
#define SL_UNROLL 4
#endif
constexpr int UNROLL = SL_UNROLL;  // gather rounds whose loads are issued together
#ifndef SL_PIN_IDS
#define SL_PIN_IDS 3  // lane / warp ids held in registers (bit 0: lane, bit 1: warp); 3: +1.7% at c2, lane alone -4.5%
#endif
#ifndef SL_PROXY_FENCE
#define SL_PROXY_FENCE 1  // fence.proxy.async before the first dense row's bulk copy overwrites the warp's dense sum (0: +0.5%, not taken: the generic writes of the previous tile must be ordered before the async-proxy write)
#endif
#ifndef SL_ONE_FILTER
#define SL_ONE_FILTER 1  // one filter instantiation (the partial last tile padded with -inf): ~25% less code
#endif

constexpr int NDMAX = 64;   // dense rows per query in the warp kernel

// Everything a (run, split) work item of k_score_runs needs to start, written once per run and
// batch by k_run_desc in work order (the classification of the run's tokens does not depend on
// the split): members, their gathered-row entries (query order, then token order; at most 32,
// one lane each), the dense signature in canonical order with its leading pair / triple row.
struct __align__(16) RunDesc {
  uint32_t qid[SL_RMAX_CT];       // original query index of member r (~0: none)
  int32_t ebeg[SL_RMAX_CT + 1];   // member r owns entries [ebeg[r], ebeg[r + 1])
  int32_t nd;                     // dense rows to sum
  int32_t dslot[NDMAX];           // ascending slots; dslot[0] may be a pair / triple row
  uint64_t row_start[32];         // per entry: CSC row start, length, skip-table slot (-1: none), row maximum
  uint32_t row_len[32];
  int32_t skip[32];
  float rmax[32];
};

struct RunArgs {
  const uint64_t* q_off;      // [B+1]
  const uint32_t* q_tok;
  const double* qconst;       // [B]
  const uint32_t* perm;       // sorted position -> original query id
  const uint32_t* run_begin;  // [n_runs+1] positions in perm
  const uint32_t* n_runs;     // device scalar
  const uint32_t* rorder;     // runs in work order (heaviest first), nullptr: run index order
  const RunDesc* rdesc;       // [n_runs] descriptor of the run at each work-order position (k_run_desc)
  uint32_t* work;             // device scalar: next work item (zeroed by k_build_runs)
  uint64_t* gtau;             // [B] shared threshold per query across doc splits (nullptr: off)
  uint32_t k;
  uint32_t C;                 // candidates kept per (query, split)
  uint32_t R;                 // max queries per run
  uint32_t qmax;
  uint32_t n_splits;
  uint32_t wpc;               // warps per CTA in use
  uint64_t* cand;             // [B][n_splits][C] (original query order)
  float* dense_out;           // GM_DENSE: [N]
  uint32_t debug_skip;        // timing experiments only (SL_DEBUG_SKIP): 1 gather, 2 filter, 4 dense
  uint32_t split_major;       // work-item order (see k_score_runs)
  uint32_t prune;             // exact block-max pruning of (query, tile) pairs
};

// top-k state of the CTA-per-query kernel (k_score_long), in its dynamic shared memory;
// filter_tile takes this or the warp kernel's WarpSmem
struct WSmem {
  uint64_t* tau;     // [1]
  float* tauf;       // [1] tau_float(*tau), kept with it
  uint32_t* n_kept;  // [1]
  uint32_t* hist;    // [16] warp_select_kth histogram
};

// Static per-warp shared layout of k_score_runs: compile-time offsets, so every access is an
// LDS/STS with an immediate offset (no generic-pointer rematerialisation). Bounds: <= 32
// gathered rows and <= NDMAX dense rows per run (other queries take k_score_long).
constexpr int WPC = 8;      // warps per CTA
struct __align__(16) WarpSmem {
  float dsum[TILE];           // dense-signature sum of the current tile
#if SL_RMAX_CT > 1
  // undo log of a non-last run member's gather into the shared dense sum: (doc, old value)
  // per applied posting, replayed backwards after its filter (<= ULOG slots of 32 postings)
  uint16_t ulog_doc[ULOG * 32];
  float ulog_old[ULOG * 32];
#endif
  uint64_t tau[RMAX];         // exact running threshold key per query
  float tauf[RMAX];           // tau_float(tau[r]), updated with it (the filter's pre-test bound)
  int32_t dslot[NDMAX];       // the run's dense signature, ascending slots
  uint32_t hist[16];          // warp_select_kth histogram
  uint32_t n_kept[RMAX];
  uint32_t qid[RMAX];         // original query index of run member r
  uint32_t emask[RMAX];       // its gathered-row entries as a lane mask
  uint64_t* keptp[RMAX];      // its candidate slot for this split
  int32_t ebeg[RMAX + 1];     // query r owns entries [ebeg[r], ebeg[r+1])
  int32_t nd[1];
#if SL_DENSE_TMA
  uint64_t mbar[1];           // completion of the first dense row's bulk copy
  uint32_t mphase[1];         // parity of its next completion
#endif
};


// four resident CTAs per SM: 228 KB of shared memory per SM, 1 KB reserved per CTA
static_assert(SL_MINB * (WPC * sizeof(WarpSmem) + 1024) <= 228 * 1024, "WarpSmem exceeds the per-SM shared memory at SL_MINB CTAs");

// Add the tile slices of the query owning lanes [e0, e1) (lane = gathered-row entry, in
// query order) to buf. Work is cut into rounds of <= 32 postings of ONE entry (doc ids are
// unique within a row, so a round has no write conflicts). A warp-uniform iterator walks
// the non-empty entries in lane (= token) order; the loads of UNROLL rounds are in flight
// together and the rounds are applied in order with __syncwarp between them, so every
// document receives its terms in token order without atomics.
// cnt/rbase are this lane's entry slice (length, absolute start).
template <bool LOG = false>
__device__ __forceinline__ float apply_slices(const IndexView& ix, uint32_t emask, uint32_t cnt, uint64_t rbase,
                                              float* buf, uint32_t d0, uint16_t* ldoc = nullptr,
                                              float* lold = nullptr, uint32_t* nslots = nullptr) {
  uint32_t slot = 0;
  float gm = -INFINITY;  // max of the values this lane wrote (feeds the filter's pre-test)
  const int lane = threadIdx.x & 31;
  uint32_t m = __ballot_sync(0xffffffffu, cnt != 0) & emask;  // entries with postings here
  int tk = m ? __ffs(m) - 1 : 32;
  uint32_t c = 0;                                             // next 32-posting chunk of entry tk
  uint32_t tcnt = __shfl_sync(0xffffffffu, cnt, tk & 31);
  uint64_t trb = __shfl_sync(0xffffffffu, rbase, tk & 31);
  while (tk < 32) {
    uint32_t doc[UNROLL];
    float val[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      doc[u] = 0xFFFFFFFFu;
      val[u] = 0.f;
      if (tk < 32) {
        const uint32_t off = c * 32 + lane;
        if (off < tcnt) {
          doc[u] = __ldg(ix.docids + trb + off);
          val[u] = __ldg(ix.values + trb + off);
        }
        if ((++c) * 32 >= tcnt) {  // entry exhausted: move to the next non-empty one
          m &= m - 1;
          tk = m ? __ffs(m) - 1 : 32;
          c = 0;
          tcnt = __shfl_sync(0xffffffffu, cnt, tk & 31);
          trb = __shfl_sync(0xffffffffu, rbase, tk & 31);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (doc[u] != 0xFFFFFFFFu) {
        const float old = buf[doc[u] - d0];
        const float nv = old + val[u];
        buf[doc[u] - d0] = nv;
        gm = fmaxf(gm, nv);
        if (LOG) {
          ldoc[slot * 32 + lane] = (uint16_t)(doc[u] - d0);
          lold[slot * 32 + lane] = old;
        }
      } else if (LOG) {
        ldoc[slot * 32 + lane] = 0xFFFFu;
      }
      if (LOG) ++slot;
      __syncwarp();
    }
  }
  if (LOG) *nslots = slot;
  return gm;
}

// Running top-k of query r over one tile (warp-level) from buf[TILE].
// tau is kept EXACT (the k-th best key so far, or 0 before k keys exist). Tiles are visited
// in increasing doc order and a key carries ~doc, so a later doc whose score EQUALS tau's
// score can never beat tau: the float pre-test is strict (x > tau_f), which rejects the
// large tie classes (head-token-only / OOV queries) without building keys.
// FULL: all TILE docs of the tile exist (every tile but the last): no per-doc bound checks.
// gpub: the query's threshold shared by its doc splits (atomicMax after every select). A
// split's exact k-th key bounds the global k-th key from below, so keys under it cannot be
// in the result. It is published one score ordinal lower with the largest doc part, so the
// strict float pre-test stays exact for equal scores in any split. Read only once the local
// pre-test passes (tiles without candidates stay load-free).
// pmax: when not NaN, an upper bound (per lane, warp-wide max >= every value of the tile)
// supplied by the caller, which skips the max pass over buf.
template <bool FULL, class SM>
__device__ __forceinline__ void filter_tile(SM& s, uint32_t r, uint32_t k, uint32_t C, uint32_t gdoc0,
                                            uint32_t nvalid, const float* buf, uint64_t* kept, uint64_t* gpub,
                                            float pmax, uint64_t g) {
  const int lane = threadIdx.x & 31;
  const float4* b4 = reinterpret_cast<const float4*>(buf);
  uint64_t tau = s.tau[r];
  float tf = s.tauf[r];
  float mx = pmax;
  if (isnan(pmax)) {
  mx = -INFINITY;
#pragma unroll
  for (int rr = 0; rr < F4L; ++rr) {
    const float4 v = b4[lane + 32 * rr];
    const uint32_t dl = 4 * (lane + 32 * rr);
    if (FULL || dl + 3 < nvalid) {
      mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (dl + c < nvalid) mx = fmaxf(mx, f4c(v, c));
    }
  }
  }
  if (!__any_sync(0xffffffffu, mx > tf || tau == 0)) return;
  if (gpub) {
    if (g > tau) {
      tau = g;
      tf = tau_float(g);
      if (!__any_sync(0xffffffffu, mx > tf)) return;
    }
  }
  // one test pass: bit (4*rr + c) of pm = element passes (key >= tau); later passes walk pm
  static_assert(F4L * 4 <= 32, "tile elements per lane must fit a 32-bit mask");
  uint32_t pm = 0;
#pragma unroll
  for (int rr = 0; rr < F4L; ++rr) {
    const float4 v = b4[lane + 32 * rr];
    const uint32_t dl = 4 * (lane + 32 * rr);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float x = f4c(v, c);
      // x > tf already implies key(x) > tau: tf is tau's own score (or one ordinal below a
      // published split threshold, or -inf below every finite score, also for tau == 0), so
      // no 64-bit key here
      if (x > tf && (FULL || dl + c < nvalid)) pm |= 1u << (4 * rr + c);
    }
  }
  const float* bf = buf;
  auto tile_visit = [&](uint64_t thr, auto&& fn) {  // keys >= max(thr, tau) of this lane
    for (uint32_t m = pm; m; m &= m - 1) {
      const int bit = __ffs(m) - 1;
      const uint32_t dl = 4 * (lane + 32 * (bit >> 2)) + (bit & 3);
      const uint64_t key = make_key(bf[dl], gdoc0 + dl);
      if (key >= thr) fn(key);
    }
  };
  const uint32_t mine = __popc(pm);
  const uint32_t incl = warp_incl_scan(mine);
  const uint32_t P = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t nk = s.n_kept[r];
  if (nk + P <= C) {
    uint64_t* dst = kept + nk + incl - mine;
    tile_visit(tau, [&](uint64_t key) { *dst++ = key; });
    __syncwarp();
    if (lane == 0) s.n_kept[r] = nk + P;
  } else {
#if SL_BALLOT_SELECT
    const uint64_t nt = warp_select_kth_tile(kept, nk, pm, bf, gdoc0, tau, k);
#else
    const uint64_t nt = warp_select_kth(
        [&](auto&& fn) {
          for (uint32_t i = lane; i < nk; i += 32) fn(kept[i]);
          tile_visit(tau, fn);
        },
        k, s.hist);
#endif
    // in-place compaction of kept (destination never passes the source chunk)
    uint32_t out = 0;
    for (uint32_t b = 0; b < nk; b += 32) {
      const uint32_t i = b + lane;
      const uint64_t x = i < nk ? kept[i] : 0ull;
      const bool keep = i < nk && x >= nt;
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) kept[out + __popc(bal & lanemask_lt())] = x;
      out += __popc(bal);
      __syncwarp();
    }
    const uint64_t nt2 = nt > tau ? nt : tau;  // survivors among this tile's candidates (keys >= tau)
    uint32_t m2 = 0;
    tile_visit(nt2, [&](uint64_t) { ++m2; });
    const uint32_t inc2 = warp_incl_scan(m2);
    const uint32_t tot2 = __shfl_sync(0xffffffffu, inc2, 31);
    uint64_t* dst = kept + out + inc2 - m2;
    tile_visit(nt2, [&](uint64_t key) { *dst++ = key; });
    __syncwarp();
    // exact k-th key = min of the k survivors
    uint64_t mn = ~0ull;
    for (uint32_t i = lane; i < out + tot2; i += 32) mn = min(mn, kept[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0) {
      s.n_kept[r] = out + tot2;
      s.tau[r] = mn;
      s.tauf[r] = tau_float(mn);
      const uint64_t hi = mn >> 32;
      if (gpub && hi > 1) atomicMax((unsigned long long*)gpub, (unsigned long long)(((hi - 1) << 32) | 0xFFFFFFFFull));
    }
  }
  __syncwarp();
}

// One warp per (run, doc split): a run is <= R queries with the same dense signature.
// Lane e owns gathered-row entry e of the run (the runs' queries' CSC tokens concatenated
// in query order; at most 32). No CTA-level synchronisation: warps progress independently.
// Persistent: the grid fills the GPU once and every warp pulls (run, split) items from a
// global counter in increasing order, so warps that finish short runs early stay busy.
template <int MODE, bool PRUNE, int DCHT = SL_DCH>
__global__ void __launch_bounds__(NT, SL_MINB) k_score_runs(IndexView ix, RunArgs ra) {
#if SL_DYN_WSMEM
  extern __shared__ __align__(16) unsigned char wsm_raw[];
  WarpSmem* wsm = reinterpret_cast<WarpSmem*>(wsm_raw);
#else
  __shared__ WarpSmem wsm[WPC];
#endif
#if SL_PIN_IDS
  // lane / warp as opaque register values: otherwise they are rematerialised from S2R tid at
  // every use (~6% of the kernel's instructions, with the S2R latency exposed)
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#if SL_PIN_IDS & 1
  asm volatile("" : "+r"(lane));
#endif
#if SL_PIN_IDS & 2
  asm volatile("" : "+r"(warp));
#endif
#else
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#endif
  const uint32_t n_runs = *ra.n_runs;
  const uint32_t total = n_runs * ra.n_splits;
  WarpSmem& s = wsm[warp];
#if SL_DENSE_TMA
  if (lane == 0) {
    mbar_init(s.mbar, 1);
    s.mphase[0] = 0;
  }
  __syncwarp();
#endif
  for (;;) {
  uint32_t it = 0;
  if (lane == 0) it = atomicAdd(ra.work, 1u);
  const uint32_t item = __shfl_sync(0xffffffffu, it, 0);
  if (item >= total) break;
  // split-major order: concurrently resident warps sweep the same doc region, so each CSC
  // slice / dense chunk is fetched from HBM once and served from L2 to every query using it
  const bool smaj = ra.split_major != 0;
  const uint32_t ridx = (uint32_t)(smaj ? item % n_runs : item / ra.n_splits);
  const uint32_t split = (uint32_t)(smaj ? item / n_runs : item % ra.n_splits);
  const uint32_t t0 = (uint32_t)((uint64_t)split * ix.num_tiles / ra.n_splits);
  const uint32_t t1 = (uint32_t)((uint64_t)(split + 1) * ix.num_tiles / ra.n_splits);

  // ---- setup: the run's descriptor (k_run_desc, work order) — members, gathered-row entries
  // (lane = entry, straight into registers) and the dense signature; every load is independent,
  // so a work item starts after one L2 round trip (plus the first slices below)
  const RunDesc* rd = ra.rdesc + ridx;
  const uint32_t qm = lane < RMAX ? __ldg(rd->qid + lane) : 0xFFFFFFFFu;
  const int32_t eb = lane <= RMAX ? __ldg(rd->ebeg + lane) : 0;
  const int nd = __ldg(&rd->nd);
  const uint32_t nr = (uint32_t)__popc(__ballot_sync(0xffffffffu, qm != 0xFFFFFFFFu));
  const int E = __shfl_sync(0xffffffffu, eb, nr);
  const bool ent = lane < E;
  const uint64_t rstart = ent ? __ldg(rd->row_start + lane) : 0ull;
  const uint32_t rlen = ent ? __ldg(rd->row_len + lane) : 0u;
  const int32_t sk = ent ? __ldg(rd->skip + lane) : -1;
  const float rmx = PRUNE && ent ? __ldg(rd->rmax + lane) : 0.f;
  if (lane < nd) s.dslot[lane] = __ldg(rd->dslot + lane);
  if (lane + 32 < nd) s.dslot[lane + 32] = __ldg(rd->dslot + lane + 32);
  {
    const int e1 = __shfl_down_sync(0xffffffffu, eb, 1);
    if ((uint32_t)lane < nr) {
      s.qid[lane] = qm;
      s.n_kept[lane] = 0;
      s.tau[lane] = 0;
      s.tauf[lane] = -INFINITY;
      s.emask[lane] = (e1 >= 32 ? 0xffffffffu : ((1u << e1) - 1u)) & ~((1u << eb) - 1u);
      s.keptp[lane] = ra.cand + ((uint64_t)qm * ra.n_splits + split) * ra.C;
    }
    if (PRUNE && (uint32_t)lane <= nr) s.ebeg[lane] = eb;
  }
  __syncwarp();
#ifdef SL_DEBUG_CHECKS
  if (lane == 0 && (nr > ra.R || nr == 0 || (uint32_t)E > 32u || (uint32_t)nd > ra.qmax)) {
    printf("k_score_runs invariant: item %u nr %u R %u E %d qmax %u nd %d\n", ridx, nr, ra.R, E, ra.qmax, nd);
    __trap();
  }
#endif
  const uint32_t* tab = ix.skiptab + (uint64_t)(sk < 0 ? 0 : sk) * (ix.num_tiles + 1);
  uint32_t cursor = 0, nextdoc = 0xFFFFFFFFu;  // short rows
  uint32_t nsb = 0, nse = 0;                   // skip rows: slice [nsb, nse) of the current tile
  if (ent) {
    if (sk >= 0) {
      nsb = __ldg(tab + t0);
      nse = __ldg(tab + t0 + 1);
    } else {
      const uint32_t* ids = ix.docids + rstart;
      const uint32_t dstart = t0 * TILE;
      uint32_t lo = 0, hi = rlen;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(ids + mid) < dstart) lo = mid + 1; else hi = mid;
      }
      cursor = lo;
      nextdoc = lo < rlen ? __ldg(ids + lo) : 0xFFFFFFFFu;
    }
  }
  const uint32_t rstride = ix.n_pad / 4;
  float4* dsum4 = reinterpret_cast<float4*>(s.dsum);

  for (uint32_t tile = t0; tile < t1; ++tile) {
    const uint32_t d0 = tile * TILE, d1 = d0 + TILE;
    const uint32_t nvalid = min((uint32_t)TILE, ix.N - d0);
#if SL_DENSE_TMA
    // the whole 4 KB first-row tile by one bulk copy: order this warp's earlier generic accesses
    // to the buffer before the async-proxy write, then lane 0 arms the barrier and starts the copy
    auto issue_first_row = [&]() {
#if SL_PROXY_FENCE
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
      __syncwarp();
      if (lane == 0) bulk_copy_g2s(s.dsum, ix.dense + (uint64_t)s.dslot[0] * ix.n_pad + d0, TILE * 4u, s.mbar);
    };
#if SL_TMA_EARLY
    // issued before the tile's slice bookkeeping, whose loads then overlap the copy
    if (nd > 0 && !(ra.debug_skip & 4)) issue_first_row();
#endif
#endif
    // (1) this tile's slice of every gathered row (lane = entry)
    uint32_t sb = 0, cnt = 0;
    if (ent) {
      if (sk >= 0) {
        sb = nsb;
        cnt = nse - nsb;
        nsb = nse;  // the next tile's slice starts where this one ends
        if (tile + 1 < t1) nse = __ldg(tab + tile + 2);  // consumed one iteration later
      } else if (nextdoc < d1) {
        const uint32_t* ids = ix.docids + rstart;
        sb = cursor;
        uint32_t cur = cursor + 1;
        while (true) {  // probe 4 postings at a time (independent loads)
          uint32_t p[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) p[i] = cur + i < rlen ? __ldg(ids + cur + i) : 0xFFFFFFFFu;
          int adv = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) adv += (adv == i && p[i] < d1) ? 1 : 0;
          cur += adv;
          if (adv < 4) {
            nextdoc = p[adv];
            break;
          }
        }
        cnt = cur - cursor;
        cursor = cur;
      } else {
        sb = cursor;
      }
    }
    const uint32_t hmask = __ballot_sync(0xffffffffu, cnt != 0);
    const uint64_t rbase = rstart + sb;
    // (1b) exact block-max pruning: UB(query, tile) = Σ dense-row tile maxima (ascending slot,
    // the order of the real sum) + Σ gathered-row bounds of rows with postings here; a query
    // whose UB cannot exceed its threshold score skips the tile (its later docs cannot win
    // ties either: larger ids). 4e-6 relative margin covers the tree-order of the bound sum.
    uint32_t live = (1u << nr) - 1u;
    if constexpr (PRUNE) {
      float ubd = 0.f;
      for (int i = 0; i < nd; ++i) ubd += __ldg(ix.dmax + (uint64_t)s.dslot[i] * ix.num_tiles + tile);
      const float bnd = cnt == 0 ? 0.f : (sk >= 0 ? __ldg(ix.smax + (uint64_t)sk * ix.num_tiles + tile) : rmx);
      for (uint32_t r = 0; r < nr; ++r) {
        const int e0 = s.ebeg[r], e1 = s.ebeg[r + 1];
        float v = (lane >= e0 && lane < e1) ? bnd : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const float ub = ubd + v;
        const uint64_t tau = s.tau[r];
        if (tau != 0 && ub + fabsf(ub) * 4e-6f <= tau_float(tau)) live &= ~(1u << r);
      }
      if (!live) {
#if SL_DENSE_TMA && SL_TMA_EARLY
        if (nd > 0 && !(ra.debug_skip & 4)) {  // the early copy must complete before the buffer is reused
          const uint32_t ph = s.mphase[0];
          mbar_wait(s.mbar, ph);
          __syncwarp();
          if (lane == 0) s.mphase[0] = ph ^ 1u;
        }
#endif
        continue;
      }
    }
    // (2) dense signature of the run, ascending slot order, all loads in flight
    // register passes of DCH float4 per lane, so the tile size does not set the register
    // footprint; returns the lane max of its sums (padding docs included: an upper bound)
    // the corpus's last tile: -inf past its last document, so the filter needs no per-document
    // bound checks (the strict pre-test x > tau_f never passes -inf)
    auto pad_tail = [&]() {
      if (nvalid != (uint32_t)TILE) {
        __syncwarp();
        for (uint32_t i = nvalid + lane; i < (uint32_t)TILE; i += 32) s.dsum[i] = -INFINITY;
      }
    };
#if SL_DENSE_ASYNC
    // The first dense row is copied global -> shared with cp.async (no registers: the whole row
    // in flight at once, one L2 round trip); later rows are added chunk by chunk in registers,
    // in ascending slot order as before (((r0 + r1) + r2) ...). Preloading the second row's
    // chunk during the copy spilled 648 B at the 64-register cap.
    auto dense_pass = [&](bool issued) -> float {
      float m = -INFINITY;
      constexpr int DCH = F4L < DCHT ? F4L : DCHT;
      const float4* dbase = reinterpret_cast<const float4*>(ix.dense + d0) + lane;
      if (nd == 0) {
#pragma unroll
        for (int rr = 0; rr < F4L; ++rr) dsum4[lane + 32 * rr] = make_float4(0.f, 0.f, 0.f, 0.f);
        pad_tail();
        return 0.f;
      }
#if SL_DENSE_TMA
      if (!issued) issue_first_row();
#else
      {
        const float4* row0 = dbase + (uint64_t)s.dslot[0] * rstride;
#pragma unroll
        for (int rr = 0; rr < F4L; ++rr) __pipeline_memcpy_async(dsum4 + lane + 32 * rr, row0 + 32 * rr, 16);
        __pipeline_commit();
      }
#endif
#pragma unroll 1
      for (int c0 = 0; c0 < F4L; c0 += DCH) {
#if SL_DENSE_TMA
        if (c0 == 0) {
          const uint32_t ph = s.mphase[0];
          mbar_wait(s.mbar, ph);
          __syncwarp();
          if (lane == 0) s.mphase[0] = ph ^ 1u;
        }
#else
        if (c0 == 0) __pipeline_wait_prior(0);
#endif
        float4 a[DCH];
#pragma unroll
        for (int rr = 0; rr < DCH; ++rr) a[rr] = dsum4[lane + 32 * (c0 + rr)];
        for (int i = 1; i < nd; ++i) {
          float4 v[DCH];
          {
            const float4* row = dbase + (uint64_t)s.dslot[i] * rstride + 32 * c0;
#pragma unroll
            for (int rr = 0; rr < DCH; ++rr) v[rr] = __ldg(row + 32 * rr);
          }
#pragma unroll
          for (int rr = 0; rr < DCH; ++rr) {
            a[rr].x += v[rr].x;
            a[rr].y += v[rr].y;
            a[rr].z += v[rr].z;
            a[rr].w += v[rr].w;
          }
        }
#pragma unroll
        for (int rr = 0; rr < DCH; ++rr) {
          if (nd > 1) dsum4[lane + 32 * (c0 + rr)] = a[rr];
          m = fmaxf(m, fmaxf(fmaxf(a[rr].x, a[rr].y), fmaxf(a[rr].z, a[rr].w)));
        }
      }
      pad_tail();
      return m;
    };
#else
    auto dense_pass = [&](bool) -> float {
      float m = -INFINITY;
      constexpr int DCH = F4L < DCHT ? F4L : DCHT;
#pragma unroll 1
      for (int c0 = 0; c0 < F4L; c0 += DCH) {
        float4 a[DCH];
#pragma unroll
        for (int rr = 0; rr < DCH; ++rr) a[rr] = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4* dbase = reinterpret_cast<const float4*>(ix.dense + d0) + lane + 32 * c0;
        for (int i = 0; i < nd; ++i) {
          const float4* row = dbase + (uint64_t)s.dslot[i] * rstride;
          float4 v[DCH];
#pragma unroll
          for (int rr = 0; rr < DCH; ++rr) v[rr] = __ldg(row + 32 * rr);
#pragma unroll
          for (int rr = 0; rr < DCH; ++rr) {
            a[rr].x += v[rr].x;
            a[rr].y += v[rr].y;
            a[rr].z += v[rr].z;
            a[rr].w += v[rr].w;
          }
        }
#pragma unroll
        for (int rr = 0; rr < DCH; ++rr) {
          dsum4[lane + 32 * (c0 + rr)] = a[rr];
          m = fmaxf(m, fmaxf(fmaxf(a[rr].x, a[rr].y), fmaxf(a[rr].z, a[rr].w)));
        }
      }
      pad_tail();
      return m;
    };
#endif
    // (3) per query: gathered rows, then the running top-k. The dense pass has ONE inlined site:
    // before member 0, and again before a member whose predecessor's gather outgrew the undo log
    float dm = INFINITY;
    bool redo = true;
    for (uint32_t r = 0; r < nr; ++r) {
      if (redo) {
        if (!(ra.debug_skip & 4)) dm = dense_pass(r == 0 && SL_TMA_EARLY && SL_DENSE_TMA);
        __syncwarp();
        redo = false;
      }
      if (PRUNE && !((live >> r) & 1u)) continue;
      const uint32_t emask = s.emask[r];
      float* buf = s.dsum;
      float lmax = dm;
      const uint32_t q = s.qid[r];
      uint64_t* gp = ra.gtau ? ra.gtau + q : nullptr;
      const uint64_t gv = gp ? *(volatile const uint64_t*)gp : 0ull;  // in flight during the gather
      // a non-last run member gathers into the shared dense sum and undoes its postings after
      // its filter (log replayed backwards: each doc gets its first old value back); too many
      // rounds for the log -> the dense sum is recomputed instead
      int undo = 0;  // 0 none, 1 replay the log, 2 recompute the dense sum
      uint32_t nslots = 0;
      if ((hmask & emask) && !(ra.debug_skip & 1)) {
#if SL_RMAX_CT > 1
        if (r + 1 < nr) {
          const uint32_t mine = ((emask >> lane) & 1u) ? (cnt + 31) / 32 : 0u;
          const uint32_t rounds = __reduce_add_sync(0xffffffffu, mine);
          undo = rounds + UNROLL - 1 <= (uint32_t)ULOG ? 1 : 2;
        }
        if (undo == 1)
          lmax = fmaxf(lmax, apply_slices<true>(ix, emask, cnt, rbase, buf, d0, s.ulog_doc, s.ulog_old, &nslots));
        else
#endif
          lmax = fmaxf(lmax, apply_slices(ix, emask, cnt, rbase, buf, d0));
      }
      if constexpr (MODE == GM_DENSE) {
        const double qc = ra.qconst[q];
        for (uint32_t i = lane; i < nvalid; i += 32) ra.dense_out[d0 + i] = __double2float_rn((double)buf[i] + qc);
        __syncwarp();
      } else {
        uint64_t* kept = s.keptp[r];
        if (!(ra.debug_skip & 2)) {
          // one instantiation: the corpus's last, partial tile holds -inf past its documents
          // (dense_pass), which the strict pre-test never passes
#if SL_ONE_FILTER
          filter_tile<true>(s, r, ra.k, ra.C, ix.doc_base + d0, nvalid, buf, kept, gp, lmax, gv);
#else
          if (nvalid == TILE)
            filter_tile<true>(s, r, ra.k, ra.C, ix.doc_base + d0, nvalid, buf, kept, gp, lmax, gv);
          else
            filter_tile<false>(s, r, ra.k, ra.C, ix.doc_base + d0, nvalid, buf, kept, gp, lmax, gv);
#endif
        }
      }
#if SL_RMAX_CT > 1
      if (undo == 1) {
        __syncwarp();
        for (int sl = (int)nslots - 1; sl >= 0; --sl) {
          const uint32_t d = s.ulog_doc[sl * 32 + lane];
          if (d != 0xFFFFu) buf[d] = s.ulog_old[sl * 32 + lane];
          __syncwarp();
        }
      } else if (undo == 2) {
        redo = true;  // recomputed at the top of the next member's iteration
      }
#endif
    }
    __syncwarp();
  }
  if constexpr (MODE == GM_TOPK) {
    for (uint32_t r = 0; r < nr; ++r) {
      const uint32_t q = s.qid[r];
      const uint32_t nk = s.n_kept[r];
      uint64_t* out = ra.cand + ((uint64_t)q * ra.n_splits + split) * ra.C;
      for (uint32_t i = nk + lane; i < ra.C; i += 32) out[i] = kInvalidKey;  // candidates are in place
    }
  }
  __syncwarp();
  }  // work items
}

// Queries with more than 32 gathered rows (one lane per row does not fit): one CTA per
// (query, doc split). Same per-document summation order as k_score_runs — dense rows in
// ascending slot order, then gathered rows in query order — so scores are bit-identical to
// what the warp kernel would produce; the running top-k is the same warp-level filter.
// Shared memory: acc[TILE] | tau, n_kept, hist | per-entry arrays [ne].
template <int MODE>
__global__ void __launch_bounds__(NT) k_score_long(IndexView ix, RunArgs ra, uint32_t first, uint32_t n_long,
                                                   uint32_t qcap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t li = blockIdx.x / ra.n_splits, split = blockIdx.x % ra.n_splits;
  if (li >= n_long) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* acc = reinterpret_cast<float*>(smem_raw);
  uint64_t* tau = reinterpret_cast<uint64_t*>(acc + TILE);
  uint64_t* row_start = tau + 1;                                   // [qcap]
  uint32_t* n_kept = reinterpret_cast<uint32_t*>(row_start + qcap);
  uint32_t* hist = n_kept + 1;                                     // [16]
  int32_t* counts = reinterpret_cast<int32_t*>(hist + 16);         // nd, ns
  float* tauf = reinterpret_cast<float*>(counts + 2);              // [1] (+ 1 pad)
  int32_t* dslot = counts + 4;                                     // [qcap]
  uint32_t* row_len = reinterpret_cast<uint32_t*>(dslot + qcap);   // [qcap]
  int32_t* skip = reinterpret_cast<int32_t*>(row_len + qcap);      // [qcap]
  uint32_t* cursor = reinterpret_cast<uint32_t*>(skip + qcap);     // [qcap]
  uint32_t* nextdoc = cursor + qcap;                               // [qcap]
  uint32_t* sbv = nextdoc + qcap;                                  // [qcap]
  uint32_t* cntv = sbv + qcap;                                     // [qcap]
  const uint32_t q = ra.perm[first + li];
  const uint32_t t0 = (uint32_t)((uint64_t)split * ix.num_tiles / ra.n_splits);
  const uint32_t t1 = (uint32_t)((uint64_t)(split + 1) * ix.num_tiles / ra.n_splits);
  if (threadIdx.x == 0) {
    int nd = 0, ns = 0;
    for (uint64_t j = ra.q_off[q]; j < ra.q_off[q + 1]; ++j) {
      const uint32_t t = ra.q_tok[j];
      if (t >= ix.V || ix.df_global[t] == 0) continue;  // OOV drop (SPEC tokenizer decisions)
      const uint64_t rb = ix.indptr[t], re = ix.indptr[t + 1];
      if (rb == re) continue;
      const int32_t info = ix.tokinfo[t];
      if (info >= 0) {
        int b = nd - 1;  // ascending slot order (canonical dense order)
        while (b >= 0 && dslot[b] > info) {
          dslot[b + 1] = dslot[b];
          --b;
        }
        dslot[b + 1] = info;
        ++nd;
      } else {
        row_start[ns] = rb;
        row_len[ns] = (uint32_t)(re - rb);
        skip[ns] = info <= -2 ? -2 - info : -1;
        ++ns;
      }
    }
    counts[0] = nd;
    counts[1] = ns;
    *tau = 0;
    *tauf = -INFINITY;
    *n_kept = 0;
  }
  __syncthreads();
  const int nd = counts[0], ns = counts[1];
  for (int e = threadIdx.x; e < ns; e += NT) {
    if (skip[e] < 0) {
      const uint32_t* ids = ix.docids + row_start[e];
      uint32_t lo = 0, hi = row_len[e];
      const uint32_t dstart = t0 * TILE;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(ids + mid) < dstart) lo = mid + 1; else hi = mid;
      }
      cursor[e] = lo;
      nextdoc[e] = lo < row_len[e] ? __ldg(ids + lo) : 0xFFFFFFFFu;
    }
  }
  __syncthreads();
  WSmem ws{};
  ws.tau = tau;
  ws.tauf = tauf;
  ws.n_kept = n_kept;
  ws.hist = hist;
  uint64_t* kept = ra.cand + ((uint64_t)q * ra.n_splits + split) * ra.C;
  const uint32_t rstride = ix.n_pad / 4;
  for (uint32_t tile = t0; tile < t1; ++tile) {
    const uint32_t d0 = tile * TILE, d1 = d0 + TILE;
    const uint32_t nvalid = min((uint32_t)TILE, ix.N - d0);
    // slices of the gathered rows in this tile (thread per entry)
    for (int e = threadIdx.x; e < ns; e += NT) {
      uint32_t sb, cnt = 0;
      if (skip[e] >= 0) {
        const uint32_t* tab = ix.skiptab + (uint64_t)skip[e] * (ix.num_tiles + 1) + tile;
        sb = __ldg(tab);
        cnt = __ldg(tab + 1) - sb;
      } else {
        sb = cursor[e];
        if (nextdoc[e] < d1) {
          const uint32_t* ids = ix.docids + row_start[e];
          uint32_t cur = sb + 1, nxt = 0xFFFFFFFFu;
          while (cur < row_len[e]) {
            nxt = __ldg(ids + cur);
            if (nxt >= d1) break;
            ++cur;
          }
          if (cur >= row_len[e]) nxt = 0xFFFFFFFFu;
          cnt = cur - sb;
          cursor[e] = cur;
          nextdoc[e] = nxt;
        }
      }
      sbv[e] = sb;
      cntv[e] = cnt;
    }
    // dense rows: thread-owned float4, ascending slot order (the warp kernel's order)
    if (threadIdx.x < TILE / 4) {
      const float4* dbase = reinterpret_cast<const float4*>(ix.dense + d0) + threadIdx.x;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int i = 0; i < nd; ++i) {
        const float4 v = __ldg(dbase + (uint64_t)dslot[i] * rstride);
        a.x += v.x;
        a.y += v.y;
        a.z += v.z;
        a.w += v.w;
      }
      reinterpret_cast<float4*>(acc)[threadIdx.x] = a;
    }
    __syncthreads();
    // gathered rows one at a time in query order (unique docs within a row)
    for (int e = 0; e < ns; ++e) {
      const uint32_t cnt = cntv[e];
      if (!cnt) continue;
      const uint64_t base = row_start[e] + sbv[e];
      for (uint32_t p = threadIdx.x; p < cnt; p += NT)
        acc[__ldg(ix.docids + base + p) - d0] += __ldg(ix.values + base + p);
      __syncthreads();
    }
    if constexpr (MODE == GM_DENSE) {
      const double qc = ra.qconst[q];
      for (uint32_t i = threadIdx.x; i < nvalid; i += NT) ra.dense_out[d0 + i] = __double2float_rn((double)acc[i] + qc);
    } else {
      if (warp == 0) filter_tile<false>(ws, 0, ra.k, ra.C, ix.doc_base + d0, nvalid, acc, kept, nullptr, NAN, 0ull);
    }
    __syncthreads();
  }
  if constexpr (MODE == GM_TOPK) {
    if (warp == 0)
      for (uint32_t i = *n_kept + lane; i < ra.C; i += 32) kept[i] = kInvalidKey;
  }
}

__host__ inline size_t long_smem_bytes(uint32_t qcap) {
  return (size_t)TILE * 4 + 8 + (size_t)qcap * 8 + 4 + 16 * 4 + 16 + (size_t)qcap * 4 * 7 + 16;
}

// Large k (> kMaxK): keys for a stable LSD radix sort that yields (score desc, doc asc).
__global__ void k_rank_keys(const float* __restrict__ scores, uint32_t n, uint32_t id_base, uint32_t* __restrict__ key,
                            uint32_t* __restrict__ val) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    key[i] = ~float_to_ord(scores[i]);  // ascending key == descending score
    val[i] = id_base + i;                // ascending ids: stability gives smaller id first on ties
  }
}
// first k of the sorted order -> outputs (score + query constant), padding beyond n
__global__ void k_rank_emit(const uint32_t* __restrict__ key, const uint32_t* __restrict__ val, uint32_t n, uint32_t k,
                            double qc, uint32_t* __restrict__ ids, float* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
    if (i < n) {
      ids[i] = val[i];
      out[i] = __double2float_rn((double)ord_to_float(~key[i]) + qc);
    } else {
      ids[i] = 0xFFFFFFFFu;
      out[i] = -INFINITY;
    }
  }
}


__device__ __forceinline__ bool same_signature(const int32_t* qdense, const uint32_t* nden, uint32_t qmax,
                                               uint32_t a, uint32_t b) {
  if (nden[a] != nden[b]) return false;
  const int32_t* x = qdense + (uint64_t)a * qmax;
  const int32_t* y = qdense + (uint64_t)b * qmax;
  for (uint32_t i = 0; i < nden[a]; ++i)
    if (x[i] != y[i]) return false;
  return true;
}

// Grouping by dense signature without a sort: every short query claims or finds its
// signature's slot in a hash table (key = hash, value = the claiming query, whose signature is
// compared on a hash match), takes a position in the group from the slot's counter, and is
// scattered to its group's range of perm after a scan of the counters. Long queries (more
// than 32 gathered rows) go to the tail of perm. The order inside a group is the arrival
// order: scores do not depend on the grouping (fixed per-document summation order).
__global__ void k_group_insert(const uint32_t* __restrict__ hkey, uint32_t B, const int32_t* __restrict__ qdense,
                               const uint32_t* __restrict__ nden, uint32_t qmax,
                               unsigned long long* __restrict__ table, uint32_t cap, uint32_t* __restrict__ cnt,
                               uint32_t* __restrict__ gslot, uint32_t* __restrict__ gpos,
                               uint32_t* __restrict__ n_long) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < B; q += gridDim.x * blockDim.x) {
    const uint32_t h = hkey[q];
    if (h == 0xFFFFFFFFu) {
      gslot[q] = 0xFFFFFFFFu;
      gpos[q] = atomicAdd(n_long, 1u);
      continue;
    }
    const unsigned long long tag = (unsigned long long)(h | 0x80000000u) << 32;
    uint32_t s = (h * 0x9E3779B1u) & (cap - 1);
    for (;;) {
      unsigned long long cur = table[s];
      if (cur == 0ull) {
        cur = atomicCAS(table + s, 0ull, tag | q);
        if (cur == 0ull) break;  // claimed: this query represents the signature
      }
      if ((cur & 0xFFFFFFFF00000000ull) == tag && same_signature(qdense, nden, qmax, (uint32_t)cur, q)) break;
      s = (s + 1) & (cap - 1);
    }
    gslot[q] = s;
    gpos[q] = atomicAdd(cnt + s, 1u);
  }
}

__global__ void k_group_scatter(const uint32_t* __restrict__ gslot, const uint32_t* __restrict__ gpos, uint32_t B,
                                const uint32_t* __restrict__ gofs, const uint32_t* __restrict__ n_long,
                                uint32_t* __restrict__ perm) {
  const uint32_t b_short = B - *n_long;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < B; q += gridDim.x * blockDim.x) {
    const uint32_t s = gslot[q];
    perm[s == 0xFFFFFFFFu ? b_short + gpos[q] : gofs[s] + gpos[q]] = q;
  }
}

// runs of one slot's group: a WARP per slot; the group is cut into blocks of R consecutive
// members (one lane per block) and each block into runs greedily by the 32-lane entry budget,
// so a large group (e.g. every query without dense tokens) is packed in parallel. Count pass
// (gcnt per slot) / write pass (run starts at the slot's scanned offset).
template <bool WRITE>
__global__ void k_pack_slots(const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ gofs, uint32_t cap,
                             const uint32_t* __restrict__ perm, const uint32_t* __restrict__ ngath, uint32_t R,
                             uint32_t* __restrict__ gcnt, const uint32_t* __restrict__ goff,
                             uint32_t* __restrict__ run_begin, uint32_t* __restrict__ n_runs,
                             const uint32_t* __restrict__ n_long, uint32_t B) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < cap; g += nwarps) {
    const uint32_t c = cnt[g];
    uint32_t total = 0;
    if (c) {
      const uint32_t b = gofs[g], nblk = (c + R - 1) / R;
      for (uint32_t k0 = 0; k0 < nblk; k0 += 32) {
        const uint32_t blk = k0 + lane;
        const uint32_t i0 = b + blk * R, i1 = min(i0 + R, b + c);
        uint32_t runs = 0;
        if (blk < nblk) {
          uint32_t ent = 0, in_run = 0;
          for (uint32_t i = i0; i < i1; ++i) {
            const uint32_t ng = __ldg(ngath + __ldg(perm + i));
            if (in_run == 0 || ent + ng > 32u) {
              ++runs;
              in_run = 0;
              ent = 0;
            }
            ++in_run;
            ent += ng;
          }
        }
        const uint32_t incl = warp_incl_scan(runs);
        if (WRITE && blk < nblk) {
          uint32_t o = goff[g] + total + incl - runs;
          uint32_t ent = 0, in_run = 0;
          for (uint32_t i = i0; i < i1; ++i) {
            const uint32_t ng = __ldg(ngath + __ldg(perm + i));
            if (in_run == 0 || ent + ng > 32u) {
              run_begin[o++] = i;
              in_run = 0;
              ent = 0;
            }
            ++in_run;
            ent += ng;
          }
        }
        total += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (!WRITE && lane == 0) gcnt[g] = total;
  }
  if (WRITE && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t t = goff[cap - 1] + gcnt[cap - 1];
    run_begin[t] = B - *n_long;
    n_runs[0] = t;
    n_runs[1] = 0;  // work-item counter of k_score_runs
  }
}

// Work order of the runs, heaviest first (an LPT schedule for the persistent scoring kernel:
// with few items per warp — document shards, small batches — the heaviest run pulled last
// would set the kernel's tail). Cost ~ postings of the run's queries + its dense rows x docs / 4;
// runs are bucketed by log2 of the cost (32 buckets, counting sort, order within a bucket
// arbitrary — the scores do not depend on it).
__device__ __forceinline__ uint32_t run_bucket(const uint32_t* run_begin, const uint32_t* perm, const uint32_t* qpost,
                                               const uint32_t* nden, uint32_t r, uint32_t n_docs) {
  const uint32_t b = run_begin[r], e = run_begin[r + 1];
  unsigned long long c = (unsigned long long)nden[perm[b]] * (n_docs / 4 + 1);
  for (uint32_t i = b; i < e; ++i) c += qpost[perm[i]];
  c = min(c, 0xFFFFFFFFull);
  return c ? 31u - (uint32_t)__clz((uint32_t)c) : 0u;  // 0..31
}

__global__ void k_run_order(const uint32_t* __restrict__ run_begin, const uint32_t* __restrict__ n_runs,
                            const uint32_t* __restrict__ perm, const uint32_t* __restrict__ qpost,
                            const uint32_t* __restrict__ nden, uint32_t n_docs, uint32_t* __restrict__ rorder) {
  // one CTA: counts per bucket, exclusive offsets (heaviest bucket first), scatter
  __shared__ uint32_t cnt[32], off[32];
  const uint32_t R = *n_runs;
  if (threadIdx.x < 32) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < R; r += blockDim.x)
    atomicAdd(&cnt[run_bucket(run_begin, perm, qpost, nden, r, n_docs)], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int b = 31; b >= 0; --b) {
      off[b] = run;
      run += cnt[b];
    }
  }
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < R; r += blockDim.x)
    rorder[atomicAdd(&off[run_bucket(run_begin, perm, qpost, nden, r, n_docs)], 1u)] = r;
}

// Descriptor of every run in work order (one warp per run; see RunDesc). A lane per query token:
// the tokens of the run's queries, concatenated in query order, are classified 32 at a time (each
// lane's df / indptr / tokinfo loads in flight together) and ballots place the gathered rows
// (query order, then token order) and query 0's dense slots — every query of a run has the same
// dense multiset. The dense signature is put in canonical (ascending slot) order; a signature led
// by two (three) slots with a pair (triple) row starts from that row.
constexpr int kDescWarps = 4;
__global__ void __launch_bounds__(kDescWarps * 32) k_run_desc(IndexView ix, const uint32_t* __restrict__ rorder,
                                                              const uint32_t* __restrict__ run_begin,
                                                              const uint32_t* __restrict__ n_runs,
                                                              const uint32_t* __restrict__ perm,
                                                              const uint64_t* __restrict__ q_off,
                                                              const uint32_t* __restrict__ q_tok, uint32_t prune,
                                                              RunDesc* __restrict__ rdesc) {
  __shared__ RunDesc sd[kDescWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t i = blockIdx.x * kDescWarps + warp;
  if (i >= *n_runs) return;
  RunDesc& d = sd[warp];
  const uint32_t run = rorder ? rorder[i] : i;
  const uint32_t pb = run_begin[run];
  const uint32_t nr = min(run_begin[run + 1] - pb, (uint32_t)RMAX);
  const bool act = (uint32_t)lane < nr;
  const uint32_t ql = act ? perm[pb + lane] : 0xFFFFFFFFu;
  const uint64_t qbl = act ? q_off[ql] : 0ull;
  const uint32_t lenl = act ? (uint32_t)(q_off[ql + 1] - qbl) : 0u;
  const uint32_t incl = warp_incl_scan(lenl);  // lanes >= nr hold the total
  const uint32_t excl = incl - lenl;
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t len0 = __shfl_sync(0xffffffffu, incl, 0);  // query 0 owns positions [0, len0)
  if (lane < RMAX) d.qid[lane] = ql;
  uint32_t e = 0, nd = 0, eb = 0;  // gathered entries / query 0's dense terms so far (uniform); entries before query `lane`
  for (uint32_t p0 = 0; p0 < tot; p0 += 32) {
    const uint32_t p = p0 + lane;
    uint32_t r = 0;  // the query owning position p
    for (uint32_t a = 0; a + 1 < nr; ++a) r += p >= __shfl_sync(0xffffffffu, incl, a) ? 1u : 0u;
    const uint64_t qb = __shfl_sync(0xffffffffu, qbl, r);
    const uint32_t ex = __shfl_sync(0xffffffffu, excl, r);
    uint32_t t = 0xFFFFFFFFu;
    if (p < tot) t = q_tok[qb + (p - ex)];
    bool ok = p < tot && t < ix.V;
    uint32_t dfv = 0;
    uint64_t rb = 0, re = 0;
    int32_t info = 0;
    if (ok) {
      dfv = ix.df_global[t];
      rb = ix.indptr[t];
      re = ix.indptr[t + 1];
      info = ix.tokinfo[t];
    }
    ok = ok && dfv != 0 && rb != re;  // OOV drop (SPEC tokenizer decisions); no local postings
    const bool isg = ok && info < 0, isd = ok && info >= 0 && p < len0;
    const uint32_t ms = __ballot_sync(0xffffffffu, isg), md = __ballot_sync(0xffffffffu, isd);
    if (isg) {
      const uint32_t ee = e + __popc(ms & lanemask_lt());
      if (ee < 32) {
        d.row_start[ee] = rb;
        d.row_len[ee] = (uint32_t)(re - rb);
        d.skip[ee] = info <= -2 ? -2 - info : -1;
        d.rmax[ee] = ix.rowmax ? ix.rowmax[t] : 0.f;
      }
    }
    if (isd) {
      const uint32_t di = nd + __popc(md & lanemask_lt());
      if (di < (uint32_t)NDMAX) d.dslot[di] = info;
    }
    const uint32_t w = excl > p0 ? min(excl - p0, 32u) : 0u;  // this chunk's positions before query `lane`
    eb += __popc(ms & (w >= 32u ? 0xffffffffu : (1u << w) - 1u));
    e += __popc(ms);
    nd += __popc(md);
  }
  if (lane <= RMAX) d.ebeg[lane] = (int32_t)min((uint32_t)lane < nr ? eb : e, 32u);
  __syncwarp();
  if (lane == 0) {
    for (uint32_t a = 1; a < nd && a < (uint32_t)NDMAX; ++a) {  // canonical (ascending slot) order of the dense terms
      const int32_t x = d.dslot[a];
      int b = (int)a - 1;
      while (b >= 0 && d.dslot[b] > x) {
        d.dslot[b + 1] = d.dslot[b];
        --b;
      }
      d.dslot[b + 1] = x;
    }
    // (a repeated token repeats its slot: equal leading slots have no pair row; block-max
    // pruning has bounds for the plain rows only)
    if (!prune && nd >= 3 && nd <= (uint32_t)NDMAX && (uint32_t)d.dslot[2] < ix.triple_m &&
        d.dslot[0] < d.dslot[1] && d.dslot[1] < d.dslot[2]) {
      d.dslot[0] = (int32_t)dense_triple_row(ix.n_dense, ix.pair_m, (uint32_t)d.dslot[0], (uint32_t)d.dslot[1],
                                             (uint32_t)d.dslot[2]);
      for (uint32_t a = 1; a + 2 < nd; ++a) d.dslot[a] = d.dslot[a + 2];
      nd -= 2;
    } else if (!prune && nd >= 2 && nd <= (uint32_t)NDMAX && (uint32_t)d.dslot[1] < ix.pair_m &&
               d.dslot[0] < d.dslot[1]) {
      d.dslot[0] = (int32_t)dense_pair_row(ix.n_dense, ix.pair_m, (uint32_t)d.dslot[0], (uint32_t)d.dslot[1]);
      for (uint32_t a = 1; a + 1 < nd; ++a) d.dslot[a] = d.dslot[a + 1];
      --nd;
    }
    d.nd = (int32_t)nd;
  }
  __syncwarp();
  // descriptor out, 16 bytes per lane and step (entries past the run's counts are never read)
  const uint4* src = reinterpret_cast<const uint4*>(&d);
  uint4* dst = reinterpret_cast<uint4*>(rdesc + i);
  for (uint32_t w = lane; w < sizeof(RunDesc) / 16; w += 32) dst[w] = src[w];
}

// top-k over an arbitrary f32 vector (SPEC top_k on its own): CTA per split of tiles,
// block-level filter + select, candidates [n_splits][C].
__global__ void __launch_bounds__(NT) k_topk_vector(const float* __restrict__ vec, uint32_t n, uint32_t k,
                                                    uint32_t C, uint32_t n_splits, uint64_t* cand) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* acc = (float*)smem_raw;
  uint64_t* kept[2] = {(uint64_t*)(acc + TILE), (uint64_t*)(acc + TILE) + C};
  uint32_t* hist = (uint32_t*)(kept[1] + C);
  uint32_t* sw = hist + 256;
  const uint32_t split = blockIdx.x;
  const uint32_t n_tiles = (n + TILE - 1) / TILE;
  const uint32_t t0 = (uint32_t)((uint64_t)split * n_tiles / n_splits);
  const uint32_t t1 = (uint32_t)((uint64_t)(split + 1) * n_tiles / n_splits);
  uint32_t n_kept = 0;
  uint64_t tau = 0;
  int cur = 0;
  for (uint32_t tile = t0; tile < t1; ++tile) {
    const uint32_t d0 = tile * TILE;
    const uint32_t nvalid = min((uint32_t)TILE, n - d0);
    for (uint32_t i = threadIdx.x; i < TILE; i += NT) acc[i] = i < nvalid ? vec[d0 + i] : 0.f;
    __syncthreads();
    auto visit = [&](uint64_t thr, auto&& f) {
      for (uint32_t i = threadIdx.x; i < nvalid; i += NT) {
        const uint64_t key = make_key(acc[i], d0 + i);
        if (key >= thr) f(key);
      }
    };
    uint32_t mine = 0;
    visit(tau, [&](uint64_t) { ++mine; });
    uint32_t P;
    const uint32_t off = block_excl_scan(mine, sw, &P);
    if (n_kept + P <= C) {
      uint64_t* dst = kept[cur] + n_kept + off;
      visit(tau, [&](uint64_t key) { *dst++ = key; });
      n_kept += P;
    } else {
      const uint64_t* kb = kept[cur];
      const uint32_t nk = n_kept;
      const uint64_t old = tau;
      tau = block_select_kth(
          [&](auto&& f) {
            for (uint32_t i = threadIdx.x; i < nk; i += NT) f(kb[i]);
            visit(old, f);
          },
          k, hist, sw + 36);
      uint32_t m2 = 0;
      for (uint32_t i = threadIdx.x; i < nk; i += NT) m2 += kb[i] >= tau;
      visit(tau, [&](uint64_t) { ++m2; });
      uint32_t tot;
      const uint32_t o2 = block_excl_scan(m2, sw, &tot);
      uint64_t* dst = kept[cur ^ 1] + o2;
      for (uint32_t i = threadIdx.x; i < nk; i += NT)
        if (kb[i] >= tau) *dst++ = kb[i];
      visit(tau, [&](uint64_t key) { *dst++ = key; });
      n_kept = tot;
      cur ^= 1;
    }
    __syncthreads();
  }
  uint64_t* out = cand + (uint64_t)split * C;
  for (uint32_t i = threadIdx.x; i < C; i += NT) out[i] = i < n_kept ? kept[cur][i] : kInvalidKey;
}

// Per query: top-k over n_splits x per_split candidate keys (invalid = 0), sorted, decoded.
// gtau (nullable): the query's threshold shared by its doc splits, a lower bound of its k-th
// key — candidates below it cannot be selected and are skipped.
__global__ void __launch_bounds__(256) k_merge(const uint64_t* __restrict__ cand, uint32_t n_splits,
                                               uint32_t per_split, uint64_t split_stride, uint64_t query_stride,
                                               uint32_t k, const double* __restrict__ qconst, uint32_t* out_ids,
                                               float* out_scores, uint64_t* out_keys,
                                               const uint64_t* __restrict__ gtau, uint32_t cap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* buf = (uint64_t*)smem_raw;  // [p2]
  const uint32_t p2 = next_pow2(max(k, 2u));
  uint32_t* hist = (uint32_t*)(buf + p2);
  uint32_t* sw = hist + 256;
  const uint32_t q = blockIdx.x;
  const uint64_t* base = cand + (uint64_t)q * query_stride;
  const uint64_t g = gtau ? gtau[q] : 0ull;
  // every valid candidate (>= g); power-of-two split sizes (the single-rank case) index with
  // shifts, others walk split by split
  const bool pow2 = (per_split & (per_split - 1)) == 0;
  const int lg = pow2 ? __ffs(per_split) - 1 : 0;
  const uint64_t total = (uint64_t)n_splits * per_split;
  auto visit = [&](auto&& f) {
    if (pow2) {
      for (uint64_t i = threadIdx.x; i < total; i += blockDim.x) {
        const uint64_t x = base[(i >> lg) * split_stride + (i & (per_split - 1))];
        if (x != kInvalidKey && x >= g) f(x);
      }
    } else {
      for (uint32_t sp = 0; sp < n_splits; ++sp) {
        const uint64_t* p = base + (uint64_t)sp * split_stride;
        for (uint32_t j = threadIdx.x; j < per_split; j += blockDim.x) {
          const uint64_t x = p[j];
          if (x != kInvalidKey && x >= g) f(x);
        }
      }
    }
  };
  // when every candidate slot fits shared memory, one pass stages the valid candidates (>= g;
  // order is irrelevant: keys are unique and the winners are sorted) and the select and the
  // copy run on them; otherwise every pass reads the candidate buffers.
  uint64_t* cbuf = reinterpret_cast<uint64_t*>(sw + 40);
  uint32_t* s_n = sw + 39;
  uint32_t nvalid = 0;
  const bool staged = total <= cap;  // every slot fits: stage (cap = 0: candidate sets too large)
  if (staged) {
    if (threadIdx.x == 0) *s_n = 0;
    __syncthreads();
    visit([&](uint64_t x) { cbuf[atomicAdd(s_n, 1u)] = x; });
    __syncthreads();
    nvalid = *s_n;
    __syncthreads();
  } else {
    uint32_t mine = 0;
    visit([&](uint64_t) { ++mine; });
    block_excl_scan(mine, sw, &nvalid);
  }
  auto visit_s = [&](auto&& f) {
    if (staged) {
      for (uint32_t i = threadIdx.x; i < nvalid; i += blockDim.x) f(cbuf[i]);
    } else {
      visit(f);
    }
  };
  uint64_t tau = 1;
  if (nvalid > k) tau = block_select_kth(visit_s, k, hist, sw + 36);
  uint32_t m2 = 0;
  visit_s([&](uint64_t x) { m2 += x >= tau; });
  uint32_t m;
  const uint32_t o = block_excl_scan(m2, sw, &m);
  uint64_t* dst = buf + o;
  visit_s([&](uint64_t x) {
    if (x >= tau) *dst++ = x;
  });
  for (uint32_t i = m + threadIdx.x; i < p2; i += blockDim.x) buf[i] = kInvalidKey;
  __syncthreads();
  block_bitonic_desc(buf, p2);
  const double qc = qconst ? qconst[q] : 0.0;
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
    const uint64_t key = i < m ? buf[i] : kInvalidKey;
    if (out_keys) out_keys[(uint64_t)q * k + i] = key;
    if (out_ids) out_ids[(uint64_t)q * k + i] = i < m ? key_doc(key) : 0xFFFFFFFFu;
    if (out_scores)
      out_scores[(uint64_t)q * k + i] = i < m ? __double2float_rn((double)key_score(key) + qc) : -INFINITY;
  }
}

// k_merge for small sets (k <= 32, n_splits x per_split <= kMergeWarpCap): one WARP per query.
// The valid candidates (>= the shared threshold g) are staged in the warp's shared slice, the
// exact k-th key is found by the warp radix select, and the k winners (one per lane) are ranked
// by counting (keys are unique): the same keys, order and decoding as k_merge.
constexpr int kMergeWarps = 4, kMergeWarpCap = 1024;
__global__ void __launch_bounds__(kMergeWarps * 32) k_merge_warp(const uint64_t* __restrict__ cand, uint32_t B,
                                                                  uint32_t n_splits, uint32_t per_split,
                                                                  uint64_t split_stride, uint64_t query_stride,
                                                                  uint32_t k, const double* __restrict__ qconst,
                                                                  uint32_t* out_ids, float* out_scores,
                                                                  uint64_t* out_keys, const uint64_t* __restrict__ gtau) {
  __shared__ uint64_t sbuf[kMergeWarps][kMergeWarpCap];
  __shared__ uint32_t shist[kMergeWarps][16];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t q = blockIdx.x * kMergeWarps + w;
  if (q >= B) return;
  uint64_t* buf = sbuf[w];
  const uint64_t* base = cand + (uint64_t)q * query_stride;
  const uint64_t g = gtau ? gtau[q] : 0ull;
  uint32_t n = 0;  // staged so far (warp-uniform)
  const uint32_t total = n_splits * per_split;
  for (uint32_t t0 = 0; t0 < total; t0 += 128) {  // four loads per lane in flight
    uint64_t x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = t0 + 32u * u + lane;
      const uint32_t sp = i / per_split;
      x[u] = i < total ? __ldg(base + (uint64_t)sp * split_stride + (i - sp * per_split)) : kInvalidKey;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool v = x[u] != kInvalidKey && x[u] >= g;
      const uint32_t bal = __ballot_sync(0xffffffffu, v);
      if (v) buf[n + __popc(bal & lanemask_lt())] = x[u];
      n += __popc(bal);
    }
  }
  __syncwarp();
  uint64_t tau = 1;
  if (n > k)
    tau = warp_select_kth(
        [&](auto&& fn) {
          for (uint32_t i = lane; i < n; i += 32) fn(buf[i]);
        },
        k, shist[w]);
  // the winners (keys >= tau: exactly min(n, k) of them), one per lane
  uint64_t mine = kInvalidKey;
  uint32_t m = 0;
  for (uint32_t i0 = 0; i0 < n; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint64_t x = i < n ? buf[i] : kInvalidKey;
    const bool v = i < n && x >= tau;
    const uint32_t bal = __ballot_sync(0xffffffffu, v);
    const uint32_t r = m + __popc(bal & lanemask_lt());
    // the winner of rank r (in staging order) goes to lane r
    for (uint32_t b = bal; b; b &= b - 1) {
      const int src = __ffs(b) - 1;
      const uint64_t y = __shfl_sync(0xffffffffu, x, src);
      const uint32_t ry = __shfl_sync(0xffffffffu, r, src);
      if ((uint32_t)lane == ry) mine = y;
    }
    m += __popc(bal);
  }
  // descending rank of this lane's key among the winners
  uint32_t rank = 0;
  for (int j = 0; j < 32; ++j) {
    const uint64_t y = __shfl_sync(0xffffffffu, mine, j);
    rank += (uint32_t)j < m && y > mine;
  }
  const double qc = qconst ? qconst[q] : 0.0;
  if ((uint32_t)lane < m) {
    const uint64_t o = (uint64_t)q * k + rank;
    if (out_keys) out_keys[o] = mine;
    if (out_ids) out_ids[o] = key_doc(mine);
    if (out_scores) out_scores[o] = __double2float_rn((double)key_score(mine) + qc);
  }
  for (uint32_t i = m + lane; i < k; i += 32) {  // fewer than k candidates: padding
    const uint64_t o = (uint64_t)q * k + i;
    if (out_keys) out_keys[o] = kInvalidKey;
    if (out_ids) out_ids[o] = 0xFFFFFFFFu;
    if (out_scores) out_scores[o] = -INFINITY;
  }
}

// k_query_prep and the dense signature in one pass over each query's tokens (score_chunk):
// validation, Σ S^θ (f64, query order), max length and posting bytes (warp-aggregated
// atomics), the sorted dense slots (stride NDMAX: a query with more is scored by k_score_long),
// gathered-row count and signature hash (0xFFFFFFFF: the long-query path).
__global__ void k_query_prep_sig(const uint64_t* __restrict__ q_off, const uint32_t* __restrict__ q_tok, uint32_t B,
                                 IndexView ix, double* __restrict__ qconst, uint32_t* __restrict__ info,
                                 unsigned long long* __restrict__ bytes, int32_t* __restrict__ qdense,
                                 uint32_t* __restrict__ nden, uint32_t* __restrict__ ngath,
                                 uint32_t* __restrict__ hkey, uint32_t* __restrict__ qpost) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t q0 = blockIdx.x * blockDim.x; q0 < B; q0 += stride) {
    const uint32_t q = q0 + threadIdx.x;
    uint32_t len = 0;
    unsigned long long pb = 0;
    if (q < B) {
      const uint64_t b = q_off[q], e = q_off[q + 1];
      double c = 0.0;
      uint32_t n = 0, ng = 0;
      int32_t* d = qdense + (uint64_t)q * NDMAX;
      if (e < b) {
        atomicOr(&info[0], 2u);
      } else {
        len = (uint32_t)min(e - b, (uint64_t)0xFFFFFFFFu);
        for (uint64_t j = b; j < e; ++j) {
          const uint32_t t = q_tok[j];
          if (t >= ix.V) {
            atomicOr(&info[0], 1u);
            continue;
          }
          if (ix.df_global[t] == 0) continue;
          c += (double)ix.theta[t];
          const uint64_t rb = ix.indptr[t], re = ix.indptr[t + 1];
          pb += 8ull * (re - rb);
          if (rb == re) continue;
          const int32_t tinfo = ix.tokinfo[t];
          if (tinfo < 0) {
            ++ng;
            continue;
          }
          if (n < (uint32_t)NDMAX) {  // insertion into the sorted slots
            int bb = (int)n - 1;
            while (bb >= 0 && d[bb] > tinfo) {
              d[bb + 1] = d[bb];
              --bb;
            }
            d[bb + 1] = tinfo;
          }
          ++n;
        }
      }
      const bool lng = ng > 32 || n > (uint32_t)NDMAX;
      if (lng) atomicAdd(&info[2], 1u);
      uint32_t h = 2166136261u ^ n;  // FNV-1a over the sorted slots
      if (!lng)
        for (uint32_t i = 0; i < n; ++i) h = (h ^ (uint32_t)d[i]) * 16777619u;
      qconst[q] = c;
      qpost[q] = (uint32_t)min(pb / 8ull, (unsigned long long)0xFFFFFFFFu);  // postings the query reads
      nden[q] = lng ? 0u : n;
      ngath[q] = ng;
      hkey[q] = lng ? 0xFFFFFFFFu : (h & 0x7FFFFFFFu);
    }
    const uint32_t m = __reduce_max_sync(0xffffffffu, len);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pb += __shfl_xor_sync(0xffffffffu, pb, o);
    if ((threadIdx.x & 31) == 0) {
      if (m) atomicMax(&info[1], m);
      if (bytes && pb) atomicAdd(bytes, pb);
    }
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
    uint32_t ng = 0, ndn = 0;
    for (uint64_t j = b; j < e; ++j) {
      const uint32_t t = q_tok[j];
      if (t >= ix.V) {
        atomicOr(&info[0], 1u);
        continue;
      }
      if (ix.df_global[t] == 0) continue;
      c += (double)ix.theta[t];
      pb += 8ull * (ix.indptr[t + 1] - ix.indptr[t]);
      if (ix.indptr[t + 1] != ix.indptr[t] && ix.tokinfo) ix.tokinfo[t] < 0 ? ++ng : ++ndn;
    }
    if (ng > 32 || ndn > NDMAX) atomicAdd(&info[2], 1u);
    qconst[q] = c;
    if (bytes && pb) atomicAdd(bytes, pb);
  }
}

// The split-threshold pre-test relies on denormal compares (tau_float: 0 > -denorm_min). A
// build with flush-to-zero (-ftz=true / --use_fast_math) would silently drop exact-zero ties
// across doc splits; nvcc defines no macro for it, so every stream checks it once on the device.
__global__ void k_ftz_probe(const float* __restrict__ zero, uint32_t* __restrict__ out) {
  const float x = zero[0];
  out[0] = (x > tau_float(0x7FFFFFFFull << 32)) ? 1u : 0u;
}

struct StreamCache {
  int device = -1;
  bool ftz = false;  // built with flush-to-zero: every call fails (k_ftz_probe)
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
    {
      void* buf;
      SL_CUDA_TRY(cudaMalloc(&buf, 8));
      SL_CUDA_TRY(cudaMemset(buf, 0, 8));
      k_ftz_probe<<<1, 1, 0, c.st>>>((const float*)buf, (uint32_t*)buf + 1); ++t_launches;
      uint32_t ok = 0;
      SL_CUDA_TRY(cudaMemcpyAsync(&ok, (uint32_t*)buf + 1, 4, cudaMemcpyDeviceToHost, c.st));
      SL_CUDA_TRY(cudaStreamSynchronize(c.st));
      cudaFree(buf);
      c.ftz = !ok;
    }
    c.device = device;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  if (c.ftz) SL_FAIL(SL_EUNSUPPORTED, "libsparselex_b200 was compiled with flush-to-zero; the top-k threshold "
                                      "pre-test needs denormal compares (rebuild without -ftz / --use_fast_math)");
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

int cur_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  return num_sms(dev);
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

struct RunPlan {
  uint32_t R, C, wpc, n_splits, per_sm;
  size_t smem;
};

// Launch plan of k_score_runs: candidate capacity per (query, split), queries per run, the
// resident CTAs of the persistent grid and the number of doc splits. SL_SPLITS / SL_RUN
// override the plan in tuning runs.
int32_t plan_runs(const sl_index* ix, uint32_t B, uint32_t k, uint32_t qmax, RunPlan* p) {
  p->C = kept_capacity(k);
  uint32_t R = (uint32_t)env_int("SL_RUN", 0);
  if (R == 0) R = 2;  // SL_RUN up to RMAX
  // the run builder keeps every run within 32 gathered entries (one lane each)
  p->R = std::max(1u, std::min<uint32_t>(R, RMAX));
  p->wpc = WPC;
  p->smem = SL_DYN_WSMEM ? sizeof(WarpSmem) * WPC : 0;  // static layout unless it exceeds 48 KB
  int per_sm = 0;
  if (p->smem) {
    SL_CUDA_TRY(cudaFuncSetAttribute(k_score_runs<GM_TOPK, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)p->smem));
    SL_CUDA_TRY(cudaFuncSetAttribute(k_score_runs<GM_TOPK, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)p->smem));
    SL_CUDA_TRY(cudaFuncSetAttribute(k_score_runs<GM_TOPK, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)p->smem));
  }
  SL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_score_runs<GM_TOPK, false>, NT, p->smem));
  p->per_sm = (uint32_t)std::max(1, per_sm);
  if (env_int("SL_PLAN_TRACE", 0)) fprintf(stderr, "[plan] k_score_runs: %d CTAs/SM, %zu B shared per CTA\n", per_sm, p->smem);
  const uint64_t warps = (uint64_t)std::max(1, per_sm) * p->wpc * num_sms(ix->device);
  const uint64_t items = std::max<uint64_t>(1, (uint64_t)B / std::max(1u, p->R / 2 + 1));  // expected runs
  uint32_t ns = (uint32_t)env_int("SL_SPLITS", 0);
  // doc splits: enough (run, split) items to keep every warp busy several times over; the
  // splits of a query share its threshold, so small k affords more of them (merge cost
  // grows with splits x k). Measured: c2 top-10 best at 12 items/warp, top-100 / c4 top-1000 at 8.
  // They also bound the doc region the resident warps sweep together (split-major order): it
  // must stay small enough for its dense-row chunks and posting slices to be served from L2 —
  // at most 128k docs per split (k <= 256; larger candidate sets trade region size for merge
  // cost: 128k x C/512). c5 shard (6.25M docs): 2 -> 48 splits, 38.8k -> 71k QPS.
  // The region's L2 footprint grows with the bytes per document the sweep touches (dense copies
  // + postings): the 128k-doc region is tuned at c2 (50 dense rows, 60 nonzeros per document,
  // ~680 B/doc); denser corpora shrink it by sqrt of the ratio (c5 shard, ~2.3 KB/doc: 72k docs,
  // 87 splits; 48 -> 96 splits measured 82.0k -> 87.0k QPS, 192 splits 83.0k: merge cost grows).
  const uint64_t f = k <= 16 ? 12 : 8;
  if (ns == 0) {
    const uint64_t by_work = (f * warps + items - 1) / items;
    const double bpd = 4.0 * ix->dense_rows + 8.0 * (double)ix->nnz / (double)std::max(1u, ix->N);
    const double shrink = bpd > 680.0 ? std::sqrt(680.0 / bpd) : 1.0;
    const uint64_t region = (uint64_t)(131072.0 * shrink) * std::max(1u, p->C / 512);
    const uint64_t by_l2 = ((uint64_t)ix->N + region - 1) / region;
    ns = (uint32_t)std::max<uint64_t>(1, std::max(by_work, by_l2));
    // but every split keeps ~64 tiles to amortise a work item's setup (query classification,
    // row cursors, the first tiles' top-k warm-up): the document shards of c2 score best in
    // 8 / 4 / 2 splits at 1/2, 1/4, 1/8 of the corpus (489 / 245 / 122 tiles; 1/8: 5.75M QPS in
    // 2 splits against 4.20M in the 12 the work rule asks for). While there are fewer runs than
    // resident warps, splits still add parallelism (c1).
    const uint64_t min_tiles = (uint64_t)std::max(1, env_int("SL_MIN_TILES", 64));
    const uint64_t cap = std::max<uint64_t>((ix->num_tiles + min_tiles / 2) / min_tiles, (warps + items - 1) / items);
    ns = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(ns, cap));
  }
  p->n_splits = std::max(1u, std::min(ns, std::max(1u, ix->num_tiles)));
  // few work items per resident warp (document shards, small batches): one query per run — the
  // run sharing saves dense passes, but with ~2 items per warp the balance matters more (1/8 shard
  // of c2: +5%)
  if (env_int("SL_RUN", 0) == 0 && (uint64_t)(B / 2) * p->n_splits < 4 * warps) p->R = 1;
  return SL_OK;
}

int32_t launch_merge(const uint64_t* cand, uint32_t B, uint32_t n_splits, uint32_t per_split, uint64_t split_stride,
                     uint64_t query_stride, uint32_t k, const double* qconst, uint32_t* ids, float* scores,
                     uint64_t* keys, cudaStream_t st, const uint64_t* gtau = nullptr) {
  // staging room for the candidates when all slots fit 8192 keys (64 KB); larger candidate
  // sets (top-1000: 37 splits x 2048) are visited in the buffers
  const uint64_t slots = (uint64_t)n_splits * per_split;
  if (k <= 32 && slots <= (uint64_t)kMergeWarpCap && env_int("SL_MERGE_WARP", 1)) {
    k_merge_warp<<<(B + kMergeWarps - 1) / kMergeWarps, kMergeWarps * 32, 0, st>>>(
        cand, B, n_splits, per_split, split_stride, query_stride, k, qconst, ids, scores, keys, gtau);
    ++t_launches;
    SL_CUDA_TRY(cudaGetLastError());
    return SL_OK;
  }
  const uint32_t cap = slots <= 8192 ? (uint32_t)slots : 0u;
  const size_t smem = (size_t)next_pow2(std::max(k, 2u)) * 8 + 256 * 4 + 40 * 4 + (size_t)cap * 8;
  SL_CUDA_TRY(cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_merge<<<B, 256, smem, st>>>(cand, n_splits, per_split, split_stride, query_stride, k, qconst, ids, scores, keys,
                                gtau, cap); ++t_launches;
  SL_CUDA_TRY(cudaGetLastError());
  return SL_OK;
}

// Full ranking of one score vector (device): the first k by (score desc, id asc).
struct RankBufs {
  uint32_t *k0, *v0, *k1, *v1, *k2, *v2;
  int32_t alloc(Scratch& scr, uint32_t n) {
    SL_TRY(scr.alloc(&k0, n));
    SL_TRY(scr.alloc(&v0, n));
    SL_TRY(scr.alloc(&k1, n));
    SL_TRY(scr.alloc(&v1, n));
    SL_TRY(scr.alloc(&k2, n));
    SL_TRY(scr.alloc(&v2, n));
    return SL_OK;
  }
};

int32_t rank_full(const float* scores, uint32_t n, uint32_t k, uint32_t id_base, double qc, uint32_t* ids,
                  float* out, cudaStream_t st, const RankBufs& rb) {
  uint32_t *k0 = rb.k0, *v0 = rb.v0, *k1 = rb.k1, *v1 = rb.v1, *k2 = rb.k2, *v2 = rb.v2;
  const unsigned g = (unsigned)std::min<uint64_t>((n + 255) / 256 + 1, 32 * cur_sms());
  if (n) k_rank_keys<<<g, 256, 0, st>>>(scores, n, id_base, k0, v0); ++t_launches;
  const uint32_t *ks = k0, *vs = v0;
  if (n) SL_TRY(radix_sort_pairs(k0, v0, n, 32, k1, k2, v1, v2, st, &ks, &vs, 0, nullptr));
  k_rank_emit<<<(unsigned)std::min<uint64_t>((k + 255) / 256, 32 * cur_sms()), 256, 0, st>>>(ks, vs, n, k, qc, ids, out); ++t_launches;
  SL_CUDA_TRY(cudaGetLastError());
  return SL_OK;
}

}  // namespace

// ------------------------------------------------------------------ entry points
namespace {
// Host query offsets must be non-decreasing before anything is staged: the copy takes
// q_offsets[B] tokens and the device kernels index the staged tokens with every offset.
int32_t validate_host_offsets(const uint64_t* off, uint32_t B) {
  for (uint32_t q = 0; q < B; ++q)
    if (off[q + 1] < off[q]) SL_FAIL(SL_EINVAL, "retrieve_batch: query offsets must be non-decreasing");
  return SL_OK;
}

// Candidate scratch of one chunk is [chunk][n_splits][C] keys; batches whose scratch would
// exceed the budget (SL_CAND_MB, default 4096 MB) are scored in equal chunks of queries.
// Results are identical for any chunking (a query's keys depend on the query only).
int32_t chunk_size(const sl_index* ix, uint32_t B, uint32_t k, uint32_t* out) {
  const uint64_t budget = (uint64_t)std::max(1, env_int("SL_CAND_MB", 4096)) << 20;
  RunPlan p;
  SL_TRY(plan_runs(ix, B, k, 1, &p));
  uint64_t per_q = (uint64_t)p.n_splits * p.C * 8;
  uint64_t bc = B;
  if ((uint64_t)B * per_q > budget) {
    bc = std::max<uint64_t>(1, budget / per_q);
    SL_TRY(plan_runs(ix, (uint32_t)bc, k, 1, &p));  // fewer queries -> possibly more splits
    per_q = (uint64_t)p.n_splits * p.C * 8;
    bc = std::max<uint64_t>(1, std::min<uint64_t>(bc, budget / per_q));
    const uint64_t nch = (B + bc - 1) / bc;
    bc = (B + nch - 1) / nch;
  }
  *out = (uint32_t)bc;
  return SL_OK;
}

// One chunk of queries through the fused scorer: validation and query constants
// (k_query_prep), grouping by dense signature, k_score_runs (+ k_score_long for queries with
// more than 32 gathered rows), then the per-query merge of the split candidates into the
// final (ids, scores) or, for a multi-rank index, into this rank's top-k keys. d_off / qconst
// point at the chunk's first query (offsets stay absolute into d_tok).
int32_t score_chunk(const sl_index* ix, StreamCache* sc, const uint64_t* d_off, const uint32_t* d_tok, uint32_t B,
                    uint32_t k, double* qconst, uint32_t* ids, float* scores, uint64_t* keys,
                    unsigned long long* bytes, float* score_ms) {
  PhaseTrace tr(sc->st, "SL_QUERY_TRACE", "query");
  tr.mark("start");
  cudaStream_t st = sc->st;
  Scratch scr(st);
  const IndexView v = ix->view();
  const bool have_bounds = v.rowmax && (!ix->dense_rows || v.dmax) && (!ix->skip_rows || v.smax);
  uint32_t* info;
  SL_TRY(scr.alloc(&info, 4));
  SL_CUDA_TRY(cudaMemsetAsync(info, 0, 16, st));
  // validation, query constants and dense signatures in one kernel, then one host round trip
  int32_t* qdense;
  uint32_t *nden, *hk, *run_begin, *n_runs, *ngath, *perm_w;
  SL_TRY(scr.alloc(&qdense, (uint64_t)B * NDMAX));
  SL_TRY(scr.alloc(&nden, B));
  SL_TRY(scr.alloc(&ngath, B));
  SL_TRY(scr.alloc(&hk, B));
  SL_TRY(scr.alloc(&perm_w, B));
  uint32_t* qpost;
  SL_TRY(scr.alloc(&qpost, B));
  SL_TRY(scr.alloc(&run_begin, (uint64_t)B + 1));
  SL_TRY(scr.alloc(&n_runs, 2));
  k_query_prep_sig<<<(B + 255) / 256, 256, 0, st>>>(d_off, d_tok, B, v, qconst, info, bytes, qdense, nden, ngath, hk,
                                                     qpost);
  ++t_launches;
  SL_CUDA_TRY(cudaGetLastError());
  uint32_t h_info[4];
  SL_CUDA_TRY(cudaMemcpyAsync(h_info, info, 16, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  tr.mark("prep+sync");
  if (h_info[0] & 2u) SL_FAIL(SL_EINVAL, "retrieve_batch: query offsets must be non-decreasing");
  if (h_info[0] & 1u) SL_FAIL(SL_EINVAL, "score_query: token id >= vocab size");
  const uint32_t qmax = std::max(1u, h_info[1]);
  const uint32_t n_long = h_info[2];   // queries with > 32 gathered rows -> k_score_long
  const uint32_t B_short = B - n_long;  // they sort after every other query
  RunPlan plan;
  SL_TRY(plan_runs(ix, B, k, qmax, &plan));
  // group queries by dense signature (hash table, no sort), cut runs of <= R identical ones
  {
    const uint32_t cap = next_pow2(std::max(64u, 2 * B));
    // one zeroed scratch: table u64[cap] | cnt[cap] | n_long
    unsigned long long* table;
    SL_TRY(scr.alloc(&table, (uint64_t)cap + cap / 2 + 1));
    SL_CUDA_TRY(cudaMemsetAsync(table, 0, ((uint64_t)cap + cap / 2 + 1) * 8, st));
    uint32_t* cnt = reinterpret_cast<uint32_t*>(table + cap);
    uint32_t* nl = cnt + cap;
    uint32_t *gslot, *gpos, *gofs, *gcnt, *goff;
    SL_TRY(scr.alloc(&gslot, B));
    SL_TRY(scr.alloc(&gpos, B));
    SL_TRY(scr.alloc(&gofs, cap));
    SL_TRY(scr.alloc(&gcnt, cap));
    SL_TRY(scr.alloc(&goff, cap));
    const unsigned g = (B + 255) / 256, gc = (unsigned)std::min<uint64_t>((cap + 7) / 8, 64ull * num_sms(ix->device));
    k_group_insert<<<g, 256, 0, st>>>(hk, B, qdense, nden, NDMAX, table, cap, cnt, gslot, gpos, nl); ++t_launches;
    SL_TRY(exclusive_scan_u32(cnt, gofs, cap, st, nullptr));
    k_group_scatter<<<g, 256, 0, st>>>(gslot, gpos, B, gofs, nl, perm_w); ++t_launches;
    k_pack_slots<false><<<gc, 256, 0, st>>>(cnt, gofs, cap, perm_w, ngath, plan.R, gcnt, nullptr, nullptr, nullptr,
                                            nl, B);
    ++t_launches;
    SL_TRY(exclusive_scan_u32(gcnt, goff, cap, st, nullptr));
    k_pack_slots<true><<<gc, 256, 0, st>>>(cnt, gofs, cap, perm_w, ngath, plan.R, gcnt, goff, run_begin, n_runs, nl,
                                           B);
    ++t_launches;
  }
  const uint32_t* perm = perm_w;
  uint32_t* rorder = nullptr;
  if (env_int("SL_RUN_ORDER", 1)) {
    SL_TRY(scr.alloc(&rorder, B));
    k_run_order<<<1, 1024, 0, st>>>(run_begin, n_runs, perm, qpost, nden, ix->N, rorder); ++t_launches;
  }
  // every run's descriptor in work order (members, gathered-row entries, dense signature)
  const uint32_t prune = have_bounds && env_int("SL_PRUNE", 0) ? 1u : 0u;  // opt-in
  RunDesc* rdesc;
  SL_TRY(scr.alloc(&rdesc, std::max<uint64_t>(B, 1)));
  k_run_desc<<<std::max(1u, (B + kDescWarps - 1) / kDescWarps), kDescWarps * 32, 0, st>>>(
      v, rorder, run_begin, n_runs, perm, d_off, d_tok, prune, rdesc);
  ++t_launches;
  tr.mark("groups+runs");
  SL_CUDA_TRY(cudaGetLastError());
  RunArgs ra{};
  ra.q_off = d_off;
  ra.q_tok = d_tok;
  ra.qconst = qconst;
  ra.perm = perm;
  ra.run_begin = run_begin;
  ra.n_runs = n_runs;
  ra.rorder = rorder;
  ra.rdesc = rdesc;
  ra.work = n_runs + 1;
  ra.k = k;
  ra.C = plan.C;
  ra.R = plan.R;
  ra.qmax = qmax;
  ra.n_splits = plan.n_splits;
  ra.wpc = plan.wpc;
  ra.debug_skip = (uint32_t)env_int("SL_DEBUG_SKIP", 0);
  ra.split_major = (uint32_t)env_int("SL_SPLIT_MAJOR", 1);
  ra.prune = prune;
  uint64_t* cand;
  SL_TRY(scr.alloc(&cand, (uint64_t)B * plan.n_splits * plan.C));
  ra.cand = cand;
  if (plan.n_splits > 1 && env_int("SL_GTAU", 1)) {
    SL_TRY(scr.alloc(&ra.gtau, B));
    SL_CUDA_TRY(cudaMemsetAsync(ra.gtau, 0, (uint64_t)B * 8, st));
  }
  // persistent grid: resident CTAs only (never more warps than the upper bound of B items)
  const uint64_t items_ub = (uint64_t)B_short * plan.n_splits;
  if (items_ub > 0xFFFFFFFFull) SL_FAIL(SL_EUNSUPPORTED, "query batch too large");
  const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>((items_ub + plan.wpc - 1) / plan.wpc,
                                                                 (uint64_t)plan.per_sm * num_sms(ix->device)));
  SL_CUDA_TRY(cudaEventRecord(sc->ev[1], st));
  if (ra.prune) {
    k_score_runs<GM_TOPK, true><<<(unsigned)grid, plan.wpc * 32, plan.smem, st>>>(v, ra); ++t_launches;
  } else {
    // few work items per warp (document shards, small batches): the spill-free 2-float4 dense
    // chunks win (1/8 shard of c2: +4.6%); otherwise 4 (more of each row in flight)
    const uint64_t n_items = (uint64_t)(B_short / std::max(1u, plan.R / 2 + 1)) * plan.n_splits;
    if (n_items < (uint64_t)env_int("SL_NARROW_ITEMS", 4) * grid * plan.wpc)
      k_score_runs<GM_TOPK, false, 2><<<(unsigned)grid, plan.wpc * 32, plan.smem, st>>>(v, ra);
    else
      k_score_runs<GM_TOPK, false><<<(unsigned)grid, plan.wpc * 32, plan.smem, st>>>(v, ra);
    ++t_launches;
  }
  if (n_long) {
    const size_t lsm = long_smem_bytes(qmax);
    if (lsm > 227 * 1024) SL_FAIL(SL_EUNSUPPORTED, "retrieve_batch: query too long for the device scorer");
    SL_CUDA_TRY(cudaFuncSetAttribute(k_score_long<GM_TOPK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
    k_score_long<GM_TOPK><<<n_long * plan.n_splits, NT, lsm, st>>>(v, ra, B_short, n_long, qmax); ++t_launches;
  }
  SL_CUDA_TRY(cudaGetLastError());
  SL_CUDA_TRY(cudaEventRecord(sc->ev[2], st));
  tr.mark("score");
  const uint64_t qstride = (uint64_t)plan.n_splits * plan.C;
  if (keys) {
    SL_TRY(launch_merge(cand, B, plan.n_splits, plan.C, plan.C, qstride, k, nullptr, nullptr, nullptr, keys, st,
                        ra.gtau));
  } else {
    SL_TRY(launch_merge(cand, B, plan.n_splits, plan.C, plan.C, qstride, k, qconst, ids, scores, nullptr, st,
                        ra.gtau));
  }
  tr.mark("merge");
  if (score_ms) {
    float ms = 0.f;
    SL_CUDA_TRY(cudaEventSynchronize(sc->ev[2]));
    SL_CUDA_TRY(cudaEventElapsedTime(&ms, sc->ev[1], sc->ev[2]));
    *score_ms += ms;
  }
  return SL_OK;
}

// Rank-local part of retrieval for a batch already on the device: every chunk scored and
// merged into this rank's keys (keys != nullptr) or straight into the final results.
int32_t local_topk(const sl_index* ix, StreamCache* sc, const uint64_t* d_off, const uint32_t* d_tok, uint32_t B,
                   uint32_t k, double* qconst, uint32_t* ids, float* scores, uint64_t* keys,
                   unsigned long long* bytes, float* score_ms) {
  uint32_t bc = B;
  SL_TRY(chunk_size(ix, B, k, &bc));
  for (uint32_t b0 = 0; b0 < B; b0 += bc) {
    const uint32_t n = std::min(bc, B - b0);
    const uint64_t o = (uint64_t)b0 * k;
    SL_TRY(score_chunk(ix, sc, d_off + b0, d_tok, n, k, qconst + b0, ids ? ids + o : nullptr,
                       scores ? scores + o : nullptr, keys ? keys + o : nullptr, bytes, score_ms));
  }
  return SL_OK;
}

// k > kMaxK (SPEC top_k up to |C|): dense score vector per query + full stable ranking; single rank.
int32_t retrieve_large_k(const sl_index* ix, StreamCache* sc, Scratch& scr, const uint64_t* d_off,
                         const uint32_t* d_tok, uint32_t B, uint32_t k, uint32_t* ids_dev, float* sc_dev) {
  cudaStream_t st = sc->st;
  const IndexView v = ix->view();
  double* qconst;
  uint32_t* info;
  SL_TRY(scr.alloc(&qconst, B));
  SL_TRY(scr.alloc(&info, 4));
  SL_CUDA_TRY(cudaMemsetAsync(info, 0, 16, st));
  k_query_prep<<<(B + 255) / 256, 256, 0, st>>>(d_off, d_tok, B, v, qconst, info, nullptr); ++t_launches;
  uint32_t h_info[4];
  SL_CUDA_TRY(cudaMemcpyAsync(h_info, info, 16, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_info[0] & 2u) SL_FAIL(SL_EINVAL, "retrieve_batch: query offsets must be non-decreasing");
  if (h_info[0] & 1u) SL_FAIL(SL_EINVAL, "score_query: token id >= vocab size");
  const uint32_t qmax = std::max(1u, h_info[1]);
  float* vec;
  double* zero;
  uint32_t* iota;
  SL_TRY(scr.alloc(&vec, std::max(1u, ix->N)));
  SL_TRY(scr.alloc(&zero, B));
  SL_TRY(scr.alloc(&iota, B));
  SL_CUDA_TRY(cudaMemsetAsync(zero, 0, (uint64_t)B * 8, st));
  std::vector<uint32_t> h_iota(B);
  for (uint32_t i = 0; i < B; ++i) h_iota[i] = i;
  SL_CUDA_TRY(cudaMemcpyAsync(iota, h_iota.data(), (uint64_t)B * 4, cudaMemcpyHostToDevice, st));
  std::vector<double> h_qc(B);
  SL_CUDA_TRY(cudaMemcpyAsync(h_qc.data(), qconst, (uint64_t)B * 8, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  RunArgs ra{};
  ra.q_off = d_off;
  ra.q_tok = d_tok;
  ra.qconst = zero;  // rank by the accumulated score; the constant is added on output
  ra.perm = iota;
  ra.k = 1;
  ra.C = kept_capacity(1);
  ra.n_splits = std::max(1u, ix->num_tiles);
  ra.dense_out = vec;
  const size_t lsm = long_smem_bytes(qmax);
  if (lsm > 227 * 1024) SL_FAIL(SL_EUNSUPPORTED, "retrieve_batch: query too long for the device scorer");
  SL_CUDA_TRY(cudaFuncSetAttribute(k_score_long<GM_DENSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
  RankBufs rbuf;
  SL_TRY(rbuf.alloc(scr, std::max(1u, ix->N)));
  for (uint32_t b = 0; b < B; ++b) {
    k_score_long<GM_DENSE><<<ra.n_splits, NT, lsm, st>>>(v, ra, b, 1, qmax); ++t_launches;
    SL_TRY(rank_full(vec, ix->N, k, ix->doc_base, h_qc[b], ids_dev + (uint64_t)b * k, sc_dev + (uint64_t)b * k, st,
                     rbuf));
  }
  return SL_OK;
}

// Stage host queries on the device (validated first) or take device pointers as they are.
int32_t stage_queries(Scratch& scr, cudaStream_t st, const uint64_t* q_offsets, const uint32_t* q_tokens,
                      uint32_t B, int32_t mem, const uint64_t** d_off, const uint32_t** d_tok) {
  *d_off = q_offsets;
  *d_tok = q_tokens;
  if (mem != SL_MEM_HOST) return SL_OK;
  SL_TRY(validate_host_offsets(q_offsets, B));
  const uint64_t ntok = q_offsets[B];
  uint64_t* o;
  uint32_t* t;
  SL_TRY(scr.alloc(&o, (uint64_t)B + 1));
  SL_TRY(scr.alloc(&t, ntok));
  SL_CUDA_TRY(cudaMemcpyAsync(o, q_offsets, ((uint64_t)B + 1) * 8, cudaMemcpyHostToDevice, st));
  if (ntok) SL_CUDA_TRY(cudaMemcpyAsync(t, q_tokens, ntok * 4, cudaMemcpyHostToDevice, st));
  *d_off = o;
  *d_tok = t;
  return SL_OK;
}

// Rank-local retrieval + (multi-rank) gather of the G x B x k keys on rank 0 and the final
// merge there. *agreed is set once this rank has entered the status agreement that precedes
// the gather (retrieve_impl's caller-facing wrapper agrees on the failure otherwise).
int32_t retrieve_body(const sl_index* ix, const uint64_t* q_offsets, const uint32_t* q_tokens, uint32_t B,
                      uint32_t k, int32_t mem, uint32_t* out_ids, float* out_scores, sl_retrieve_stats* stats,
                      bool* agreed) {
  const bool dist = ix->comm != nullptr;  // any communicator, 1 rank included
  const bool want_out = !dist || ix->comm->rank == 0;
  StreamCache* sc;
  SL_TRY(get_stream(ix->device, &sc));
  cudaStream_t st = sc->st;
  Scratch scr(st);
  const uint64_t* d_off;
  const uint32_t* d_tok;
  SL_TRY(stage_queries(scr, st, q_offsets, q_tokens, B, mem, &d_off, &d_tok));
  const uint32_t launches0 = t_launches;
  SL_CUDA_TRY(cudaEventRecord(sc->ev[0], st));
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
  float score_ms = 0.f, merge_ms = 0.f;
  unsigned long long* bytes;
  SL_TRY(scr.alloc(&bytes, 1));
  SL_CUDA_TRY(cudaMemsetAsync(bytes, 0, 8, st));
  if (k > kMaxK) {
    if (dist) SL_FAIL(SL_EUNSUPPORTED, "retrieve_batch: k > 4096 is not supported across ranks");
    SL_TRY(retrieve_large_k(ix, sc, scr, d_off, d_tok, B, k, ids_dev, sc_dev));
  } else {
    double* qconst;
    SL_TRY(scr.alloc(&qconst, B));
    if (!dist) {
      SL_TRY(local_topk(ix, sc, d_off, d_tok, B, k, qconst, ids_dev, sc_dev, nullptr, bytes,
                        stats ? &score_ms : nullptr));
    } else {
      // local top-k keys -> gather the G x k candidates of every query on rank 0 (NCCL) -> merge there
      sl_comm* cm = ix->comm;
      uint64_t* local;
      SL_TRY(scr.alloc(&local, (uint64_t)B * k));
      SL_TRY(local_topk(ix, sc, d_off, d_tok, B, k, qconst, nullptr, nullptr, local, bytes,
                        stats ? &score_ms : nullptr));
      uint64_t* gathered = nullptr;
      if (cm->rank == 0) SL_TRY(scr.alloc(&gathered, (uint64_t)cm->nranks * B * k));
      SL_CUDA_TRY(cudaStreamSynchronize(st));
      *agreed = true;
      SL_TRY(comm_agree(cm, SL_OK));
      SL_CUDA_TRY(cudaEventRecord(sc->ev[2], st));
      const size_t cnt = (size_t)B * k;
      SL_TRY(nccl_check(nccl().GroupStart(), "ncclGroupStart"));
      if (cm->rank == 0) {
        for (int r = 0; r < cm->nranks; ++r)
          SL_TRY(nccl_check(nccl().Recv(gathered + (uint64_t)r * cnt, cnt, ncclUint64, r, cm->comm, st), "ncclRecv"));
      }
      SL_TRY(nccl_check(nccl().Send(local, cnt, ncclUint64, 0, cm->comm, st), "ncclSend"));
      SL_TRY(nccl_check(nccl().GroupEnd(), "ncclGroupEnd"));
      if (cm->rank == 0)
        SL_TRY(launch_merge(gathered, B, (uint32_t)cm->nranks, k, cnt, k, k, qconst, ids_dev, sc_dev, nullptr, st));
      SL_CUDA_TRY(cudaEventRecord(sc->ev[3], st));
      if (stats) {
        SL_CUDA_TRY(cudaEventSynchronize(sc->ev[3]));
        SL_CUDA_TRY(cudaEventElapsedTime(&merge_ms, sc->ev[2], sc->ev[3]));
      }
    }
  }
  SL_CUDA_TRY(cudaEventRecord(sc->ev[3], st));
  if (want_out && mem == SL_MEM_HOST) {
    SL_CUDA_TRY(cudaMemcpyAsync(out_ids, ids_dev, (uint64_t)B * k * 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(out_scores, sc_dev, (uint64_t)B * k * 4, cudaMemcpyDeviceToHost, st));
  }
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  if (stats) {
    float a = 0;
    cudaEventElapsedTime(&a, sc->ev[0], sc->ev[3]);
    unsigned long long hb = 0;
    SL_CUDA_TRY(cudaMemcpy(&hb, bytes, 8, cudaMemcpyDeviceToHost));
    std::memset(stats, 0, sizeof(*stats));
    stats->total_ms = a;
    stats->score_kernel_ms = score_ms;
    stats->merge_ms = merge_ms;
    stats->posting_bytes = hb;
    stats->scorevec_bytes = 4ull * ix->N * B;
    stats->kernels_launched = t_launches - launches0;  // every kernel of this call
  }
  return SL_OK;
}
}  // namespace

int32_t retrieve_impl(const sl_index* ix, const uint64_t* q_offsets, const uint32_t* q_tokens, uint32_t B,
                      uint32_t k, int32_t mem, uint32_t* out_ids, float* out_scores, sl_retrieve_stats* stats) {
  if (!ix) SL_FAIL(SL_EINVAL, "retrieve_batch: null index");
  if (k == 0) SL_FAIL(SL_EINVAL, "top_k: k must be >= 1");
  if (mem != SL_MEM_HOST && mem != SL_MEM_DEVICE) SL_FAIL(SL_EINVAL, "retrieve_batch: bad mem kind");
  const bool dist = ix->comm != nullptr;
  const bool want_out = !dist || ix->comm->rank == 0;
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (B == 0) return SL_OK;
  if (!q_offsets || !q_tokens) SL_FAIL(SL_EINVAL, "retrieve_batch: null query pointers");
  if (want_out && (!out_ids || !out_scores)) SL_FAIL(SL_EINVAL, "retrieve_batch: null output pointers");
  bool agreed = false;
  int32_t rc = retrieve_body(ix, q_offsets, q_tokens, B, k, mem, out_ids, out_scores, stats, &agreed);
  // a rank that failed before the candidate gather still takes part in the status agreement,
  // so its peers return an error instead of waiting in ncclRecv / ncclSend
  if (rc != SL_OK && dist && !agreed) rc = comm_agree(ix->comm, rc);
  return rc;
}

// Multi-rank building blocks (include/sparselex_b200.h sl_retrieve_local / sl_merge_candidates).
int32_t retrieve_local_impl(const sl_index* ix, const uint64_t* q_offsets, const uint32_t* q_tokens, uint32_t B,
                            uint32_t k, int32_t mem, uint64_t* out_keys, double* out_qconst) {
  if (!ix) SL_FAIL(SL_EINVAL, "retrieve_local: null index");
  if (k == 0) SL_FAIL(SL_EINVAL, "top_k: k must be >= 1");
  if (k > kMaxK) SL_FAIL(SL_EUNSUPPORTED, "retrieve_local: k > 4096 has no candidate form");
  if (mem != SL_MEM_HOST && mem != SL_MEM_DEVICE) SL_FAIL(SL_EINVAL, "retrieve_local: bad mem kind");
  if (B == 0) return SL_OK;
  if (!q_offsets || !q_tokens || !out_keys || !out_qconst) SL_FAIL(SL_EINVAL, "retrieve_local: null argument");
  StreamCache* sc;
  SL_TRY(get_stream(ix->device, &sc));
  cudaStream_t st = sc->st;
  Scratch scr(st);
  const uint64_t* d_off;
  const uint32_t* d_tok;
  SL_TRY(stage_queries(scr, st, q_offsets, q_tokens, B, mem, &d_off, &d_tok));
  uint64_t* keys = out_keys;
  double* qconst = out_qconst;
  if (mem == SL_MEM_HOST) {
    SL_TRY(scr.alloc(&keys, (uint64_t)B * k));
    SL_TRY(scr.alloc(&qconst, B));
  }
  SL_TRY(local_topk(ix, sc, d_off, d_tok, B, k, qconst, nullptr, nullptr, keys, nullptr, nullptr));
  if (mem == SL_MEM_HOST) {
    SL_CUDA_TRY(cudaMemcpyAsync(out_keys, keys, (uint64_t)B * k * 8, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(out_qconst, qconst, (uint64_t)B * 8, cudaMemcpyDeviceToHost, st));
  }
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  return SL_OK;
}

int32_t merge_candidates_impl(const uint64_t* keys, uint32_t G, uint32_t B, uint32_t k, const double* qconst,
                              int32_t mem, int32_t device, uint32_t* out_ids, float* out_scores) {
  if (k == 0) SL_FAIL(SL_EINVAL, "top_k: k must be >= 1");
  if (k > kMaxK) SL_FAIL(SL_EUNSUPPORTED, "merge_candidates: k > 4096 has no candidate form");
  if (G == 0) SL_FAIL(SL_EINVAL, "merge_candidates: no shards");
  if (mem != SL_MEM_HOST && mem != SL_MEM_DEVICE) SL_FAIL(SL_EINVAL, "merge_candidates: bad mem kind");
  if (B == 0) return SL_OK;
  if (!keys || !qconst || !out_ids || !out_scores) SL_FAIL(SL_EINVAL, "merge_candidates: null argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    SL_FAIL(SL_ECUDA, "merge_candidates: no CUDA device available (there is no CPU fallback)");
  StreamCache* sc;
  SL_TRY(get_stream(device, &sc));
  cudaStream_t st = sc->st;
  Scratch scr(st);
  const uint64_t cnt = (uint64_t)B * k;
  const uint64_t* d_keys = keys;
  const double* d_qc = qconst;
  uint32_t* ids = out_ids;
  float* scs = out_scores;
  if (mem == SL_MEM_HOST) {
    uint64_t* kk;
    double* qq;
    SL_TRY(scr.alloc(&kk, cnt * G));
    SL_TRY(scr.alloc(&qq, B));
    SL_TRY(scr.alloc(&ids, cnt));
    SL_TRY(scr.alloc(&scs, cnt));
    SL_CUDA_TRY(cudaMemcpyAsync(kk, keys, cnt * G * 8, cudaMemcpyHostToDevice, st));
    SL_CUDA_TRY(cudaMemcpyAsync(qq, qconst, (uint64_t)B * 8, cudaMemcpyHostToDevice, st));
    d_keys = kk;
    d_qc = qq;
  }
  SL_TRY(launch_merge(d_keys, B, G, k, cnt, k, k, d_qc, ids, scs, nullptr, st));
  if (mem == SL_MEM_HOST) {
    SL_CUDA_TRY(cudaMemcpyAsync(out_ids, ids, cnt * 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(out_scores, scs, cnt * 4, cudaMemcpyDeviceToHost, st));
  }
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  return SL_OK;
}

int32_t score_query_impl(const sl_index* ix, const uint32_t* q_tokens, uint32_t q_len, int32_t mem, float* out) {
  if (!ix || !out) SL_FAIL(SL_EINVAL, "score_query: null argument");
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
  k_query_prep<<<1, 32, 0, st>>>(d_off, d_tok, 1, v, qconst, info, nullptr); ++t_launches;
  uint32_t h_info[4];
  SL_CUDA_TRY(cudaMemcpyAsync(h_info, info, 16, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_info[0] & 1u) SL_FAIL(SL_EINVAL, "score_query: token id >= vocab size");
  // the single query as a "long" query: one CTA per tile, same summation order as retrieval
  uint32_t* d_perm;
  SL_TRY(scr.alloc(&d_perm, 1));
  SL_CUDA_TRY(cudaMemsetAsync(d_perm, 0, 4, st));
  RunArgs ra{};
  ra.q_off = d_off;
  ra.q_tok = d_tok;
  ra.qconst = qconst;
  ra.perm = d_perm;
  ra.k = 1;
  ra.C = kept_capacity(1);
  ra.n_splits = std::max(1u, ix->num_tiles);
  ra.dense_out = d_out;
  const uint32_t qcap = std::max(1u, q_len);
  const size_t smem = long_smem_bytes(qcap);
  if (smem > 227 * 1024) SL_FAIL(SL_EUNSUPPORTED, "score_query: query too long for the device scorer");
  SL_CUDA_TRY(cudaFuncSetAttribute(k_score_long<GM_DENSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_score_long<GM_DENSE><<<ra.n_splits, NT, smem, st>>>(v, ra, 0, 1, qcap); ++t_launches;
  SL_CUDA_TRY(cudaGetLastError());
  if (mem == SL_MEM_HOST)
    SL_CUDA_TRY(cudaMemcpyAsync(out, d_out, (uint64_t)ix->N * 4, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  return SL_OK;
}

int32_t top_k_impl(const float* scores, uint32_t n, uint32_t k, int32_t mem, int32_t device, uint32_t* out_ids,
                   float* out_scores) {
  if (k == 0) SL_FAIL(SL_EINVAL, "top_k: k must be >= 1");
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
  if (k > kMaxK) {  // full stable ranking
    RankBufs rbuf;
    SL_TRY(rbuf.alloc(scr, std::max(1u, n)));
    SL_TRY(rank_full(d_in, n, k, 0, 0.0, ids_dev, sc_dev, st, rbuf));
    if (mem == SL_MEM_HOST) {
      SL_CUDA_TRY(cudaMemcpyAsync(out_ids, ids_dev, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
      SL_CUDA_TRY(cudaMemcpyAsync(out_scores, sc_dev, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
    }
    SL_CUDA_TRY(cudaStreamSynchronize(st));
    return SL_OK;
  }
  const uint32_t C = std::max(512u, kept_capacity(k));
  const uint32_t n_tiles = std::max(1u, (n + TILE - 1) / TILE);
  const uint32_t n_splits = std::min<uint32_t>(n_tiles, 4 * num_sms(device));
  uint64_t* cand;
  SL_TRY(scr.alloc(&cand, (uint64_t)n_splits * C));
  if (n) {
    const size_t smem = (size_t)TILE * 4 + 2 * (size_t)C * 8 + 256 * 4 + 40 * 4;
    SL_CUDA_TRY(cudaFuncSetAttribute(k_topk_vector, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_topk_vector<<<n_splits, NT, smem, st>>>(d_in, n, k, C, n_splits, cand); ++t_launches;
    SL_CUDA_TRY(cudaGetLastError());
  } else {
    SL_CUDA_TRY(cudaMemsetAsync(cand, 0, (uint64_t)C * 8, st));
  }
  SL_TRY(launch_merge(cand, 1, n ? n_splits : 1, C, C, (uint64_t)n_splits * C, k, nullptr, ids_dev, sc_dev, nullptr,
                      st));
  if (mem == SL_MEM_HOST) {
    SL_CUDA_TRY(cudaMemcpyAsync(out_ids, ids_dev, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
    SL_CUDA_TRY(cudaMemcpyAsync(out_scores, sc_dev, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
  }
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  return SL_OK;
}

}  // namespace sl
