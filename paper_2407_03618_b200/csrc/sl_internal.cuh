// sl_internal.cuh — shared device/host internals of libsparselex_b200.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "sl_bm25_math.h"
#include "sparselex_b200.h"

namespace sl {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
const std::string& get_error();

struct Status {
  int32_t code = SL_OK;
  bool ok() const { return code == SL_OK; }
};

#define SL_CUDA_TRY(expr)                                                                   \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess) {                                                                \
      ::sl::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                  \
      return _e == cudaErrorMemoryAllocation ? SL_ENOMEM : SL_ECUDA;                        \
    }                                                                                       \
  } while (0)

#define SL_TRY(expr)                 \
  do {                               \
    int32_t _s = (expr);             \
    if (_s != SL_OK) return _s;      \
  } while (0)

#define SL_FAIL(code, msg)     \
  do {                         \
    ::sl::set_error(msg);      \
    return (code);             \
  } while (0)

// kernels launched by this host thread (bench.py's gpu_launches evidence)
extern thread_local uint32_t t_launches;

// ---------------------------------------------------------------- constants
#ifndef SL_TILE_DOCS
#define SL_TILE_DOCS 1024
#endif
constexpr int kTileDocs = SL_TILE_DOCS;  // docs per scoring tile (f32 accumulator = 4 KB smem per warp)
constexpr int kScoreThreads = 256;     // threads per scoring CTA
constexpr int kQMax = 32;              // gathered rows per query in the warp kernel (one lane each); longer queries go to k_score_long
constexpr uint32_t kMaxK = 4096;       // max k for the fused top-k path
constexpr uint64_t kInvalidKey = 0ull; // never produced by a real (score, doc) key

// ---------------------------------------------------------------- BM25 math (f64)
// proj/src/scoring.cpp:60-145 as written once in sl_bm25_math.h; the device instantiation
// rounds every operation explicitly (no FMA contraction), matching the reference's C++
// expression trees. Preconditions are validated on the host.
__device__ __forceinline__ double d_idf(int v, double n, double d) { return bm25::idf<bm25::DevOps>(v, n, d); }

__device__ __forceinline__ double d_tf_component(int v, double tf, double dl, double avg, double k1,
                                                 double b, double delta) {
  return bm25::tf_component<bm25::DevOps>(v, tf, bm25::norm<bm25::DevOps>(dl, avg, b), k1, delta);
}

__device__ __forceinline__ double d_nonoccurrence(int v, double idf, double k1, double delta) {
  return bm25::nonoccurrence<bm25::DevOps>(v, idf, k1, delta);
}

__host__ __device__ __forceinline__ bool is_sparse_variant(int v) {
  return v == SL_ROBERTSON || v == SL_ATIRE || v == SL_LUCENE;
}

// ---------------------------------------------------------------- top-k keys
// key = orderable(score) << 32 | ~doc : larger key = better; equal scores -> smaller doc.
__host__ __device__ __forceinline__ uint32_t float_to_ord(float f) {
  f = f + 0.0f;  // -0 -> +0 so that both zeros tie
#ifdef __CUDA_ARCH__
  uint32_t u = __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
#endif
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float ord_to_float(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}
__host__ __device__ __forceinline__ uint64_t make_key(float score, uint32_t doc) {
  return ((uint64_t)float_to_ord(score) << 32) | (uint64_t)(~doc);
}
__host__ __device__ __forceinline__ uint32_t key_doc(uint64_t key) { return ~(uint32_t)key; }
__host__ __device__ __forceinline__ float key_score(uint64_t key) {
  return ord_to_float((uint32_t)(key >> 32));
}

// ---------------------------------------------------------------- device views
struct IndexView {
  const uint64_t* indptr;     // [V+1]
  const uint32_t* docids;     // [nnz] local doc ids
  const float* values;        // [nnz] S^Δ
  const uint32_t* df_global;  // [V]
  const float* theta;         // [V]
  const int32_t* tokinfo;     // [V] >=0 dense slot, -1 short row, <=-2 skip slot -(x+2)
  const float* dense;         // [dense_rows][n_pad]
  const uint32_t* skiptab;    // [skip_rows][num_tiles+1]
  const float* rowmax;        // [V]                       max(0, S^Δ) over the row
  const float* dmax;          // [dense_rows][num_tiles]   max(0, S^Δ) over a dense row's tile
  const float* smax;          // [skip_rows][num_tiles]    max(0, S^Δ) over a skip row's tile slice
  uint32_t V;
  uint32_t N;        // local docs
  uint32_t n_pad;    // num_tiles * kTileDocs
  uint32_t num_tiles;
  uint32_t doc_base;
  uint32_t n_dense;  // dense rows (pair rows follow them in `dense`)
  uint32_t pair_m;   // leading dense slots with pair rows
  uint32_t triple_m; // leading dense slots with triple rows (after the pair rows)
};

// row of the triple (a, b, c), a < b < c < m3 (colex order): triple rows follow the pair rows
__host__ __device__ __forceinline__ uint32_t dense_triple_row(uint32_t n_dense, uint32_t m2, uint32_t a, uint32_t b,
                                                              uint32_t c) {
  return n_dense + m2 * (m2 - 1) / 2 + c * (c - 1) * (c - 2) / 6 + b * (b - 1) / 2 + a;
}

// row of the pair (a, b), a < b < m, in the dense array: pair rows follow the n_dense single rows
__host__ __device__ __forceinline__ uint32_t dense_pair_row(uint32_t n_dense, uint32_t m, uint32_t a, uint32_t b) {
  return n_dense + a * (2 * m - a - 1) / 2 + (b - a - 1);
}

// host launchers shared between sl_build.cu and sl_query.cu
int32_t exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t st,
                           uint32_t* total_host);
// Values of the first pass taken from document offsets instead of vin (index build: the
// value of token position p is its document): tile_doc[k] = document holding the first
// position of sort tile k.
// SL_BUILD_TRACE=1 / SL_QUERY_TRACE=1: device time between phases (events on the stream), stderr
struct PhaseTrace {
  bool on = false;
  cudaStream_t st = nullptr;
  const char* tag = "";
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  PhaseTrace(cudaStream_t s, const char* env, const char* t) : st(s), tag(t) {
    const char* e = std::getenv(env);
    on = e && std::atoi(e);
  }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.emplace_back(name, e);
  }
  ~PhaseTrace() {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back().second);
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      fprintf(stderr, "[%s] %-14s %8.3f ms\n", tag, ev[i].first, ms);
    }
    for (auto& x : ev) cudaEventDestroy(x.second);
  }
};

struct DocSrc {
  const uint64_t* off;  // [N+1] absolute
  uint64_t o0;
  uint32_t N;
  const uint32_t* tile_doc;
};
int32_t radix_sort_pairs(const uint32_t* kin, const uint32_t* vin, uint64_t n, int bits, uint32_t* k0, uint32_t* k1,
                         uint32_t* v0, uint32_t* v1, cudaStream_t st, const uint32_t** kout, const uint32_t** vout,
                         uint32_t v_check, uint32_t* err, const DocSrc* docs = nullptr);
int sort_tile_elems();  // elements per radix-sort tile

}  // namespace sl
