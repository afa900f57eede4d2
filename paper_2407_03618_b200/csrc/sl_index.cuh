// sl_index.cuh — the device-resident SearchIndex shard behind the opaque sl_index handle.
#pragma once

#include <nccl.h>

#include "sl_nccl.cuh"

#include "sl_internal.cuh"

struct sl_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1;
  int rank = 0;
  int device = 0;
  cudaStream_t st = nullptr;  // the status agreement's stream (usable whatever state the caller's work is in)
  int32_t* dflag = nullptr;   // device word for the status agreement
};

// SPEC.md [MODULE] index, SearchIndex: matrix (indptr/docids/values), stats, params,
// theta; plus the query-side acceleration structures this design adds (dense copies of
// the highest-df rows, per-tile skip offsets for long rows).
struct sl_index {
  int device = 0;
  sl_params params{};
  uint32_t N = 0;          // local docs
  uint32_t N_global = 0;
  uint32_t V = 0;
  uint32_t doc_base = 0;
  uint64_t nnz = 0;        // local nonzeros
  uint64_t total_len = 0;  // global Σ|D|
  double avg_len = 0.0;
  sl_comm* comm = nullptr;  // borrowed

  uint64_t* indptr = nullptr;     // [V+1]
  uint32_t* docids = nullptr;     // [nnz]
  float* values = nullptr;        // [nnz]
  uint32_t* df_global = nullptr;  // [V]
  float* theta = nullptr;         // [V]
  uint32_t* doclens = nullptr;    // [N]
  uint32_t* tf = nullptr;         // [nnz] (keep_tf only)

  int32_t* tokinfo = nullptr;     // [V]
  float* dense = nullptr;         // [(dense_rows + pair rows) * n_pad]
  uint32_t dense_rows = 0;
  uint32_t pair_m = 0;            // dense slots [0, pair_m) also have pair rows r_a + r_b (a < b)
  uint32_t triple_m = 0;          // ... and [0, triple_m) triple rows (r_a + r_b) + r_c (a < b < c)
  uint32_t* skiptab = nullptr;    // [skip_rows * (num_tiles + 1)]
  // block-max bounds (exact top-k pruning): max(0, S^Δ) over a row / a row's tile slice
  float* rowmax = nullptr;        // [V]
  float* dmax = nullptr;          // [dense_rows * num_tiles]
  float* smax = nullptr;          // [skip_rows * num_tiles]
  uint32_t skip_rows = 0;
  uint32_t num_tiles = 0;
  uint32_t n_pad = 0;

  uint64_t device_bytes = 0;
  float build_ms = 0.f;

  sl::IndexView view() const {
    sl::IndexView v;
    v.indptr = indptr;
    v.docids = docids;
    v.values = values;
    v.df_global = df_global;
    v.theta = theta;
    v.tokinfo = tokinfo;
    v.dense = dense;
    v.skiptab = skiptab;
    v.rowmax = rowmax;
    v.dmax = dmax;
    v.smax = smax;
    v.V = V;
    v.N = N;
    v.n_pad = n_pad;
    v.n_dense = dense_rows;
    v.pair_m = pair_m;
    v.triple_m = triple_m;
    v.num_tiles = num_tiles;
    v.doc_base = doc_base;
    return v;
  }
};

#include <vector>

namespace sl {
// host copy of a SearchIndex shard (persistence)
struct HostIndex {
  sl_params params{};
  uint32_t N = 0, V = 0, doc_base = 0, N_global = 0;
  uint64_t total_len = 0;
  double avg_len = 0.0;
  std::vector<uint64_t> indptr;
  std::vector<uint32_t> docids, df, doclens;
  std::vector<float> values, theta;
};
int32_t load_index_from_host(const HostIndex& h, int device, float dense_min_density, sl_index** out);
int32_t build_index_impl(const sl_build_desc* desc, sl_index** out);
void free_index(sl_index* ix);
int32_t nccl_check(ncclResult_t r, const char* what);
// Status agreement before a data collective: every rank passes its own status (SL_OK or the
// error it hit) and gets back its own error, or, when it was fine but a peer was not, the
// largest peer status. A rank that fails before a collective calls this instead of returning
// straight away, so its peers fail too instead of blocking in the collective.
int32_t comm_agree(sl_comm* c, int32_t status);
}  // namespace sl
