// sl_capi.cu — the extern "C" boundary declared in include/sparselex_b200.h.
#include <cmath>
#include <cstring>
#include <string>

#include "sl_index.cuh"

namespace sl {
thread_local uint32_t t_launches = 0;
namespace {
thread_local std::string t_error;
}
void set_error(const std::string& msg) { t_error = msg; }
const std::string& get_error() { return t_error; }

int32_t retrieve_impl(const sl_index* ix, const uint64_t* q_offsets, const uint32_t* q_tokens, uint32_t B,
                      uint32_t k, int32_t mem, uint32_t* out_ids, float* out_scores, sl_retrieve_stats* stats);
int32_t score_query_impl(const sl_index* ix, const uint32_t* q_tokens, uint32_t q_len, int32_t mem, float* out);
int32_t retrieve_local_impl(const sl_index* ix, const uint64_t* q_offsets, const uint32_t* q_tokens, uint32_t B,
                            uint32_t k, int32_t mem, uint64_t* out_keys, double* out_qconst);
int32_t merge_candidates_impl(const uint64_t* keys, uint32_t G, uint32_t B, uint32_t k, const double* qconst,
                              int32_t mem, int32_t device, uint32_t* out_ids, float* out_scores);
int32_t top_k_impl(const float* scores, uint32_t n, uint32_t k, int32_t mem, int32_t device, uint32_t* out_ids,
                   float* out_scores);

}  // namespace sl

using namespace sl;

extern "C" {

int32_t sl_abi_version(void) { return SL_ABI_VERSION; }

const char* sl_last_error(void) { return get_error().c_str(); }

const char* sl_status_string(int32_t s) {
  switch (s) {
    case SL_OK: return "ok";
    case SL_EINVAL: return "invalid argument";
    case SL_ECUDA: return "CUDA error";
    case SL_ENCCL: return "NCCL error";
    case SL_ENOMEM: return "out of device memory";
    case SL_ECORRUPT: return "corrupt index";
    case SL_EUNSUPPORTED: return "unsupported";
    case SL_EIO: return "I/O error";
    default: return "unknown status";
  }
}

// sl_params_validate / sl_default_delta and the scoring functions live in sl_bm25.cpp.

int32_t sl_index_build(const sl_build_desc* desc, sl_index** out) { return build_index_impl(desc, out); }

void sl_index_destroy(sl_index* index) { free_index(index); }

int32_t sl_index_get_info(const sl_index* ix, sl_index_info* info) {
  if (!ix || !info) SL_FAIL(SL_EINVAL, "sl_index_get_info: null argument");
  info->num_docs_local = ix->N;
  info->num_docs_global = ix->N_global;
  info->vocab_size = ix->V;
  info->doc_base = ix->doc_base;
  info->nnz_local = ix->nnz;
  info->total_len_global = ix->total_len;
  info->avg_len = ix->avg_len;
  info->dense_rows = ix->dense_rows;
  info->skip_rows = ix->skip_rows;
  info->tile_docs = kTileDocs;
  info->num_tiles = ix->num_tiles;
  info->device_bytes = ix->device_bytes;
  info->build_ms = ix->build_ms;
  return SL_OK;
}

int32_t sl_index_export(const sl_index* ix, int32_t mem, uint64_t* indptr, uint32_t* docids, float* values,
                        uint32_t* df, float* theta, uint32_t* doclens, uint32_t* tf) {
  if (!ix) SL_FAIL(SL_EINVAL, "sl_index_export: null index");
  if (tf && !ix->tf) SL_FAIL(SL_EINVAL, "sl_index_export: tf requested but the index was built without keep_tf");
  SL_CUDA_TRY(cudaSetDevice(ix->device));
  const cudaMemcpyKind kind = mem == SL_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  struct {
    void* dst;
    const void* src;
    uint64_t bytes;
  } items[] = {{indptr, ix->indptr, ((uint64_t)ix->V + 1) * 8}, {docids, ix->docids, ix->nnz * 4},
               {values, ix->values, ix->nnz * 4},           {df, ix->df_global, (uint64_t)ix->V * 4},
               {theta, ix->theta, (uint64_t)ix->V * 4},     {doclens, ix->doclens, (uint64_t)ix->N * 4},
               {tf, ix->tf, ix->nnz * 4}};
  for (auto& it : items)
    if (it.dst && it.bytes) SL_CUDA_TRY(cudaMemcpy(it.dst, it.src, it.bytes, kind));
  return SL_OK;
}

int32_t sl_retrieve_batch(const sl_index* index, const uint64_t* q_offsets, const uint32_t* q_tokens,
                          uint32_t num_queries, uint32_t k, int32_t ordered, int32_t mem, uint32_t* out_ids,
                          float* out_scores) {
  (void)ordered;
  return retrieve_impl(index, q_offsets, q_tokens, num_queries, k, mem, out_ids, out_scores, nullptr);
}

int32_t sl_retrieve_batch_timed(const sl_index* index, const uint64_t* q_offsets, const uint32_t* q_tokens,
                                uint32_t num_queries, uint32_t k, int32_t mem, uint32_t* out_ids,
                                float* out_scores, sl_retrieve_stats* stats) {
  if (stats) std::memset(stats, 0, sizeof(*stats));
  return retrieve_impl(index, q_offsets, q_tokens, num_queries, k, mem, out_ids, out_scores, stats);
}

int32_t sl_score_query(const sl_index* index, const uint32_t* q_tokens, uint32_t q_len, int32_t mem,
                       float* out_scores) {
  return score_query_impl(index, q_tokens, q_len, mem, out_scores);
}

int32_t sl_top_k(const float* scores, uint32_t n, uint32_t k, int32_t ordered, int32_t mem, int32_t device,
                 uint32_t* out_ids, float* out_scores) {
  (void)ordered;
  return top_k_impl(scores, n, k, mem, device, out_ids, out_scores);
}

int32_t sl_comm_unique_id(uint8_t out_id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!nccl().ok) SL_FAIL(SL_ENCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  SL_TRY(nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId"));
  std::memcpy(out_id, &id, 128);
  return SL_OK;
}

int32_t sl_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device, sl_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) SL_FAIL(SL_EINVAL, "sl_comm_init: bad arguments");
  if (!nccl().ok) SL_FAIL(SL_ENCCL, "libnccl.so.2 could not be loaded");
  SL_CUDA_TRY(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  auto* c = new sl_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc((void**)&c->dflag, 4) != cudaSuccess) {
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
    SL_FAIL(SL_ECUDA, "sl_comm_init: stream / flag allocation failed");
  }
  const int32_t rc = nccl_check(nccl().CommInitRank(&c->comm, nranks, uid, rank), "ncclCommInitRank");
  if (rc != SL_OK) {
    cudaFree(c->dflag);
    cudaStreamDestroy(c->st);
    delete c;
    return rc;
  }
  *out = c;
  return SL_OK;
}

int32_t sl_retrieve_local(const sl_index* index, const uint64_t* q_offsets, const uint32_t* q_tokens,
                          uint32_t num_queries, uint32_t k, int32_t mem, uint64_t* out_keys, double* out_qconst) {
  return retrieve_local_impl(index, q_offsets, q_tokens, num_queries, k, mem, out_keys, out_qconst);
}

int32_t sl_merge_candidates(const uint64_t* keys, uint32_t num_shards, uint32_t num_queries, uint32_t k,
                            const double* qconst, int32_t mem, int32_t device, uint32_t* out_ids, float* out_scores) {
  return merge_candidates_impl(keys, num_shards, num_queries, k, qconst, mem, device, out_ids, out_scores);
}

void sl_comm_destroy(sl_comm* c) {
  if (!c) return;
  if (c->comm) nccl().CommDestroy(c->comm);
  cudaSetDevice(c->device);
  if (c->dflag) cudaFree(c->dflag);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
}

}  // extern "C"
