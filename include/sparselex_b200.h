/* sparselex_b200.h — C-ABI of the B200-native eager sparse BM25 path.
 *
 * The reference (paths relative to its root) has no index/retrieval code, only the
 * SPEC's C++ operations plus proj/include/sparselex/bm25.hpp. Each entry point
 * below replaces one of those operations for token-id input:
 *
 *   sl_index_build      <- build_index(corpus, BM25Params, TokenizerConfig)  SPEC.md [MODULE] index
 *                          (token ids instead of text; pass 1/2 on the GPU; DF + length
 *                          all-reduce over NCCL when a communicator is given)
 *   sl_index_export     <- the ScoreMatrix / SearchIndex fields                SPEC.md [MODULE] index
 *                          (indptr.bin u64, docids.bin u32, values.bin f32, df.bin u32,
 *                          theta.bin f32, doclens.bin u32 of "External Interfaces")
 *   sl_retrieve_batch   <- retrieve_batch(index, queries, k, ordered, workers) SPEC.md [MODULE] retrieval
 *                          = score_query + top_k per query, k x G candidates merged on rank 0
 *   sl_score_query      <- score_query(index, query) -> dense |C| vector       SPEC.md [MODULE] retrieval
 *   sl_top_k            <- top_k(scores, k, ordered)                           SPEC.md [MODULE] retrieval
 *   sl_params_validate  <- BM25Params::validate                                proj/src/scoring.cpp:47-58
 *   sl_index_save       <- save_index(index, directory)                        SPEC.md [MODULE] index
 *   sl_index_load       <- load_index(directory)                               SPEC.md [MODULE] index
 *   sl_retrieve_local / sl_merge_candidates <- retrieve_batch split at the rank boundary
 *                          (per-shard top-k keys; rank-0 merge), for callers with their own transport
 *   sl_index_destroy / sl_last_error : ownership + error plumbing (the reference throws
 *                          std::invalid_argument with fixed messages, scoring.cpp:15-138;
 *                          here a status code + thread-local message).
 *
 * Conventions: plain pointers and sizes only. `mem` says whether caller buffers live
 * in host memory (SL_MEM_HOST: the call copies in/out) or on the index's device
 * (SL_MEM_DEVICE). The index owns all device memory; inputs are borrowed for the
 * duration of the call. Built indexes are immutable and safe for concurrent
 * sl_retrieve_batch calls (each call uses its own scratch and stream).
 * Variant numbering follows proj/include/sparselex/bm25.hpp:16-23.
 * There is no CPU fallback: every compute entry point runs CUDA kernels for sm_100a
 * and fails with SL_ECUDA if no device is usable.
 */
#ifndef SPARSELEX_B200_H
#define SPARSELEX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SL_ABI_VERSION 1

typedef enum {
  SL_OK = 0,
  SL_EINVAL = 1,   /* contract violation (reference: std::invalid_argument) */
  SL_ECUDA = 2,    /* CUDA runtime / launch failure or no device */
  SL_ENCCL = 3,    /* NCCL failure */
  SL_ENOMEM = 4,   /* device allocation failed */
  SL_ECORRUPT = 5, /* structural invariant violated */
  SL_EUNSUPPORTED = 6,
  SL_EIO = 7       /* file I/O failure (message names the path) */
} sl_status;

typedef enum {
  SL_ROBERTSON = 0,
  SL_ATIRE = 1,
  SL_LUCENE = 2,
  SL_BM25L = 3,
  SL_BM25PLUS = 4,
  SL_TFLDP = 5
} sl_variant;

typedef enum { SL_MEM_HOST = 0, SL_MEM_DEVICE = 1 } sl_mem;

/* BM25Params (bm25.hpp:31-47). */
typedef struct {
  int32_t variant;
  double k1;
  double b;
  double delta;
} sl_params;

typedef struct sl_index sl_index;
typedef struct sl_comm sl_comm;

/* One rank's shard of a document-sharded corpus. With comm == NULL the
 * shard is the whole corpus. Documents are contiguous: this rank owns global doc ids
 * [doc_base, doc_base + num_docs). */
typedef struct {
  const uint64_t* doc_offsets; /* [num_docs + 1], token offsets; doc_offsets[0] may be nonzero */
  const uint32_t* token_ids;   /* token_ids[doc_offsets[0] .. doc_offsets[num_docs]) */
  uint32_t num_docs;           /* local |C_r| */
  uint32_t vocab_size;         /* |V| (global, identical on all ranks) */
  uint32_t doc_base;           /* global id of local doc 0 */
  int32_t mem;                 /* sl_mem of doc_offsets / token_ids */
  sl_params params;
  int32_t device;              /* CUDA device ordinal */
  int32_t keep_tf;             /* keep per-nonzero tf for sl_index_export (debug/parity) */
  float dense_min_density;     /* rows with global df >= density * N_global get a dense
                                  query-side copy; <= 0 selects the default (0.125) */
  sl_comm* comm;               /* NULL = single shard */
  /* Optional precomputed GLOBAL statistics (host memory). When global_df != NULL the
   * build uses them instead of its own counts / the NCCL all-reduce: df[V] summed over all
   * shards, N and Σ|D| over all shards. Lets a caller shard without NCCL (e.g. several
   * shards on one GPU, or statistics exchanged over another transport). */
  const uint32_t* global_df;
  uint32_t global_num_docs;
  uint64_t global_total_len;
} sl_build_desc;

/* Index statistics (global unless marked local). */
typedef struct {
  uint32_t num_docs_local;
  uint32_t num_docs_global;
  uint32_t vocab_size;
  uint32_t doc_base;
  uint64_t nnz_local;
  uint64_t total_len_global; /* Σ|D| */
  double avg_len;            /* L_avg = Σ|D| / N */
  uint32_t dense_rows;       /* rows with a dense query-side copy */
  uint32_t skip_rows;        /* rows with a per-tile skip table */
  uint32_t tile_docs;        /* docs per scoring tile */
  uint32_t num_tiles;
  uint64_t device_bytes;     /* device memory held by the index */
  float build_ms;            /* device time of the last build (CUDA events) */
} sl_index_info;

int32_t sl_abi_version(void);
const char* sl_last_error(void);
const char* sl_status_string(int32_t status);

int32_t sl_params_validate(const sl_params* p);
double sl_default_delta(int32_t variant); /* bm25.hpp:37-39 / scoring.cpp:34-41 */

/* The scoring functions of proj/include/sparselex/bm25.hpp:25-72 (scoring.cpp:8-145) as C:
 * the same arithmetic as the C++ symbols of include/sparselex/bm25.hpp (exported by this library
 * for reference code that links against them) and as the GPU build's per-nonzero math.
 * Contract violations return SL_EINVAL with the reference's std::invalid_argument message. */
int32_t sl_variant_from_string(const char* name, int32_t* out);  /* variant_from_string, scoring.cpp:8-16 */
const char* sl_variant_to_string(int32_t variant);              /* to_string, scoring.cpp:18-28; NULL if invalid */
int32_t sl_is_sparse_variant(int32_t variant);                  /* is_sparse_variant, scoring.cpp:30-32: 1 / 0 */
int32_t sl_idf(int32_t variant, uint32_t df, uint32_t num_docs, double* out);  /* idf, scoring.cpp:60-79 */
int32_t sl_tf_component(double tf, double doc_len, uint32_t num_docs, double avg_len, const sl_params* p,
                        double* out);                             /* tf_component, scoring.cpp:81-114 */
int32_t sl_score(double tf, uint32_t df, double doc_len, uint32_t num_docs, double avg_len, const sl_params* p,
                 double* out);                                    /* score, scoring.cpp:116-123 */
int32_t sl_nonoccurrence_score(uint32_t df, uint32_t num_docs, const sl_params* p,
                               double* out);                      /* nonoccurrence_score, scoring.cpp:125-145 */

/* Index build (SPEC build_index). Token ids must be < vocab_size; num_docs >= 1; the
 * corpus must not be all-empty ("degenerate corpus"). */
int32_t sl_index_build(const sl_build_desc* desc, sl_index** out);
void sl_index_destroy(sl_index* index);
int32_t sl_index_get_info(const sl_index* index, sl_index_info* info);

/* Export any subset of the SearchIndex arrays (NULL = skip). Sizes: indptr V+1,
 * docids/values/tf nnz_local, df/theta V, doclens num_docs_local. df is the GLOBAL
 * document frequency; docids are LOCAL (add doc_base for global ids). tf requires
 * keep_tf at build time. */
int32_t sl_index_export(const sl_index* index, int32_t mem, uint64_t* indptr, uint32_t* docids,
                        float* values, uint32_t* df, float* theta, uint32_t* doclens, uint32_t* tf);

/* SPEC save_index / load_index: the 9-file directory layout of SPEC.md [MODULE] index
 * "External Interfaces" (meta.json, vocab.json, df.bin, theta.bin, indptr.bin, docids.bin,
 * values.bin, doclens.bin, docs.json; little-endian). Token-id corpora store the id's decimal
 * string as the vocabulary token and the global doc id as the external id. load validates
 * every ScoreMatrix invariant: missing file -> SL_EIO (path in the message), corrupt lengths /
 * invariants -> SL_ECORRUPT, format version mismatch -> SL_EUNSUPPORTED. */
int32_t sl_index_save(const sl_index* index, const char* directory);
int32_t sl_index_load(const char* directory, int32_t device, float dense_min_density, sl_index** out);

/* Batched retrieval (SPEC retrieve_batch): for each query b, the min(k, N_global) best
 * documents by B(Q,D) = Σ S^Δ + Σ S^θ, score descending, ties -> smaller global doc id.
 * Outputs are [num_queries x k]; slots beyond min(k, N) hold id 0xFFFFFFFF, score -inf.
 * Query tokens with global df = 0 are dropped (SPEC OOV rule); ids >= |V| are an error.
 * Any k >= 1 (k > 4096: full per-query ranking, single rank only); any query length.
 * `ordered` is accepted for API parity; results are always sorted (a valid order for
 * ordered == 0 as well). With a communicator, every rank passes the same queries and
 * the merged result is written on rank 0 only (other ranks may pass NULL outputs). */
int32_t sl_retrieve_batch(const sl_index* index, const uint64_t* q_offsets, const uint32_t* q_tokens,
                          uint32_t num_queries, uint32_t k, int32_t ordered, int32_t mem,
                          uint32_t* out_ids, float* out_scores);

/* Device-timed variant used by the bench harness: same as sl_retrieve_batch with
 * mem == SL_MEM_DEVICE, and reports the device time of the scoring kernel and the whole
 * call (CUDA events on the call's stream) plus the algorithmic posting bytes read. */
typedef struct {
  float total_ms;
  float score_kernel_ms;
  float merge_ms;
  uint64_t posting_bytes;   /* Σ_q Σ_{t in q} 8 * nnz_local(t) */
  uint64_t scorevec_bytes;  /* Σ_q 4 * N_local */
  uint64_t unique_posting_bytes; /* 8 * Σ_{t in union of batch} nnz_local(t) */
  uint32_t kernels_launched;
} sl_retrieve_stats;

int32_t sl_retrieve_batch_timed(const sl_index* index, const uint64_t* q_offsets,
                                const uint32_t* q_tokens, uint32_t num_queries, uint32_t k,
                                int32_t mem, uint32_t* out_ids, float* out_scores,
                                sl_retrieve_stats* stats);

/* Dense score vector of one query over the LOCAL shard (SPEC score_query; f32).
 * out_scores has num_docs_local entries and includes the Σ S^θ constant. */
int32_t sl_score_query(const sl_index* index, const uint32_t* q_tokens, uint32_t q_len, int32_t mem,
                       float* out_scores);

/* SPEC top_k over an arbitrary f32 vector (GPU radix select). Returns min(k, n) results,
 * padded as in sl_retrieve_batch. */
int32_t sl_top_k(const float* scores, uint32_t n, uint32_t k, int32_t ordered, int32_t mem,
                 int32_t device, uint32_t* out_ids, float* out_scores);

/* Multi-rank building blocks for callers that move candidates over their own transport (the
 * library's NCCL path runs the same two steps internally):
 *   sl_retrieve_local   <- the per-rank half of retrieve_batch: this shard's best k candidates per
 *                          query as 64-bit keys [num_queries x k], key = (order-preserving bits of
 *                          the f32 accumulated score, query constant excluded) << 32 | ~global_doc_id,
 *                          larger key = better (ties -> smaller doc id), 0 = empty slot; plus the
 *                          query constant Σ S^θ (f64, identical on every shard) in out_qconst[B].
 *   sl_merge_candidates <- the rank-0 merge: keys of num_shards shards laid out
 *                          [num_shards][num_queries][k] -> the [num_queries x k] (ids, scores) that
 *                          sl_retrieve_batch on the unsharded index returns (same padding).
 * k <= 4096. With mem == SL_MEM_HOST every buffer is host memory; SL_MEM_DEVICE: all on `device`
 * (sl_retrieve_local: the index's device). */
int32_t sl_retrieve_local(const sl_index* index, const uint64_t* q_offsets, const uint32_t* q_tokens,
                          uint32_t num_queries, uint32_t k, int32_t mem, uint64_t* out_keys, double* out_qconst);
int32_t sl_merge_candidates(const uint64_t* keys, uint32_t num_shards, uint32_t num_queries, uint32_t k,
                            const double* qconst, int32_t mem, int32_t device, uint32_t* out_ids, float* out_scores);

/* Multi-GPU (one process per GPU). The unique id (128 bytes) is created on rank 0 and
 * shipped to every rank by the caller (any transport), then each rank joins. */
int32_t sl_comm_unique_id(uint8_t out_id[128]);
int32_t sl_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device,
                     sl_comm** out);
void sl_comm_destroy(sl_comm* comm);

/* ---- Text pipeline (SPEC.md [MODULE] tokenizer) ---------------
 *   sl_tokenize(build=1)  <- tokenize_build(text, TokenizerConfig, Vocabulary&) per document
 *                            proj/include/sparselex/tokenizer.hpp:36-39 (split -> lowercase ->
 *                            stopword filter -> stem -> id; unseen tokens get the next ids in
 *                            first-encounter order, vocabulary.hpp:26-33)
 *   sl_tokenize(build=0)  <- tokenize_query(text, TokenizerConfig, const Vocabulary&)
 *                            tokenizer.hpp:41-45 (out-of-vocabulary tokens dropped)
 *   sl_stem_batch         <- stem_english(word) stemmer.hpp:16-18, one call per word
 *   sl_vocab_*            <- Vocabulary (vocabulary.hpp:13-48): size, tokens in id order
 * Documents are byte ranges [doc_offsets[d], doc_offsets[d+1]) of `text` (doc_offsets[0]
 * must be 0), each tokenized on its own as the reference tokenizes one string. The output
 * batch is device-resident: its offsets/ids feed sl_index_build / sl_retrieve_batch with
 * mem = SL_MEM_DEVICE directly. Stopwords: newline-separated tokens, '#' lines ignored
 * (stopwords.hpp:13-15), compared with the lowercased pre-stem token. */
typedef enum { SL_STEMMER_NONE = 0, SL_STEMMER_SNOWBALL_ENGLISH = 1 } sl_stemmer;

typedef struct {
  int32_t lowercase;         /* TokenizerConfig.lowercase (tokenizer.hpp:17) */
  int32_t stemmer;           /* sl_stemmer (stemmer.hpp:8-11) */
  const char* stopwords;     /* NULL or newline-separated list (host memory) */
  uint64_t stopwords_bytes;
} sl_tokenizer_config;

typedef struct sl_vocab sl_vocab;
typedef struct sl_token_batch sl_token_batch;

int32_t sl_vocab_create(int32_t device, sl_vocab** out);
int32_t sl_vocab_destroy(sl_vocab* vocab);
int32_t sl_vocab_size(const sl_vocab* vocab, uint32_t* size);
/* tokens in id order: offsets[size+1] (NULL to skip), bytes (NULL to skip), total byte count */
int32_t sl_vocab_export(const sl_vocab* vocab, uint64_t* offsets, char* bytes, uint64_t* total_bytes);
/* fills an EMPTY vocabulary with n tokens in id order (load_index) */
int32_t sl_vocab_import(sl_vocab* vocab, const uint64_t* offsets, const char* bytes, uint32_t n);

int32_t sl_tokenize(sl_vocab* vocab, const sl_tokenizer_config* config, int32_t build, const char* text,
                    const uint64_t* doc_offsets, uint32_t num_docs, int32_t mem, sl_token_batch** out);
/* device pointers stay owned by the batch */
int32_t sl_token_batch_info(const sl_token_batch* batch, uint32_t* num_docs, uint64_t* num_tokens,
                            const uint64_t** d_offsets, const uint32_t** d_ids);
int32_t sl_token_batch_copy(const sl_token_batch* batch, uint64_t* host_offsets, uint32_t* host_ids);
int32_t sl_token_batch_destroy(sl_token_batch* batch);

/* Streaming tokenize of a HOST corpus (same output as sl_tokenize + sl_token_batch_copy): the
 * corpus is cut into document-aligned chunks of about chunk_bytes (0: 256 MiB); chunk i+1 is
 * copied to the device while chunk i is tokenized, and each chunk's ids / token offsets are
 * copied back while the next chunk runs (separate H2D and D2H streams). out_offsets:
 * u64[num_docs+1]; out_ids: room for ids_capacity ids (SL_EINVAL when the corpus has more
 * tokens); *num_tokens = total. Pinned host buffers give full PCIe bandwidth. */
int32_t sl_tokenize_stream(sl_vocab* vocab, const sl_tokenizer_config* config, int32_t build, const char* text,
                           const uint64_t* doc_offsets, uint32_t num_docs, uint64_t chunk_bytes,
                           uint64_t* out_offsets, uint32_t* out_ids, uint64_t ids_capacity, uint64_t* num_tokens);

/* ---- Text-level SearchIndex (SPEC.md [MODULE] index / retrieval over texts) -------------------
 *   sl_text_index_build    <- build_index(corpus: sequence of (external_id, text), params,
 *                             tokenizer_config) SPEC.md:201-209: tokenize_build on the device, then
 *                             sl_index_build on the device-resident ids. Errors (SL_EINVAL): empty
 *                             corpus, degenerate corpus (every document tokenizes to empty),
 *                             duplicate external ids. ids / texts: byte ranges [off[d], off[d+1]).
 *   sl_text_index_save/load<- save_index / load_index SPEC.md:210-227: the 9-file layout with the real
 *                             vocab.json {token: id}, docs.json [external ids] and meta.json tokenizer
 *                             {lowercase, stopwords_hash, stemmer} (+ the stopword list); load checks
 *                             the list against the hash (SL_ECORRUPT on mismatch).
 *   sl_text_index_retrieve <- retrieve / retrieve_batch over query texts SPEC.md:296-313: tokenize_query
 *                             with the index's config and frozen vocabulary, then score + top-k; host
 *                             outputs [num_queries x k] padded as sl_retrieve_batch.
 *   sl_text_index_external_id <- QueryResult.external_ids / SearchIndex.doc_external_ids (borrowed bytes)
 * The index, vocabulary and configuration returned by the accessors are borrowed from the text index. */
typedef struct sl_text_index sl_text_index;

int32_t sl_text_index_build(const char* ext_ids, const uint64_t* id_offsets, const char* text,
                            const uint64_t* text_offsets, uint32_t num_docs, const sl_params* params,
                            const sl_tokenizer_config* config, int32_t device, float dense_min_density,
                            sl_text_index** out);
void sl_text_index_destroy(sl_text_index* index);
int32_t sl_text_index_save(const sl_text_index* index, const char* directory);
int32_t sl_text_index_load(const char* directory, int32_t device, float dense_min_density, sl_text_index** out);
const sl_index* sl_text_index_index(const sl_text_index* index);
sl_vocab* sl_text_index_vocab(const sl_text_index* index);
int32_t sl_text_index_config(const sl_text_index* index, sl_tokenizer_config* out);
int32_t sl_text_index_num_docs(const sl_text_index* index, uint32_t* out);
int32_t sl_text_index_external_id(const sl_text_index* index, uint32_t doc, const char** id, uint64_t* len);
int32_t sl_text_index_retrieve(const sl_text_index* index, const char* text, const uint64_t* offsets,
                               uint32_t num_queries, uint32_t k, int32_t ordered, uint32_t* out_ids,
                               float* out_scores);

/* stem_english for n words (host buffers): out has the input's byte size, word i's stem is
 * out[offsets[i] .. offsets[i] + out_len[i]) */
int32_t sl_stem_batch(const char* words, const uint64_t* offsets, uint32_t n, int32_t device, char* out,
                      uint32_t* out_len);

#ifdef __cplusplus
}
#endif

#endif /* SPARSELEX_B200_H */
