// sparselex/b200.hpp — C++20 mirror of the reference's SPEC API over the C-ABI
// (include/sparselex_b200.h). Header-only; link with -lsparselex_b200.
//
// The reference declares its scoring types in proj/include/sparselex/bm25.hpp:16-72 and
// specifies build_index / score_query / top_k / retrieve / retrieve_batch in SPEC.md
// ([MODULE] index, [MODULE] retrieval) without shipping code for them. This header gives
// those operations for token-id input, computed on a B200:
//   build_index(TokenCorpus, BM25Params)                       SPEC index build_index
//   score_query(index, query) -> std::vector<float>[|C|]       SPEC retrieval score_query
//   top_k(scores, k, ordered) -> QueryResult                   SPEC retrieval top_k
//   retrieve(index, query, k, ordered) -> QueryResult          SPEC retrieval retrieve
//   retrieve_batch(index, queries, k, ordered, workers)        SPEC retrieval retrieve_batch
// Contract violations throw std::invalid_argument (as scoring.cpp does); CUDA / NCCL
// failures throw std::runtime_error.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "sparselex/bm25.hpp"
#include "sparselex_b200.h"

namespace sparselex::b200 {

// bm25.hpp:16-47: the reference's own scoring types (include/sparselex/bm25.hpp), implemented by
// this library — a BM25Params built by reference code is passed straight through.
using sparselex::BM25Params;
using sparselex::Variant;

inline void check(int32_t status) {
  if (status == SL_OK) return;
  const std::string msg = sl_last_error();
  if (status == SL_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(std::string(sl_status_string(status)) + ": " + msg);
}

inline sl_params to_c(const BM25Params& p) { return sl_params{static_cast<int32_t>(p.variant), p.k1, p.b, p.delta}; }

// A tokenised corpus: document d holds token_ids[doc_offsets[d] .. doc_offsets[d+1]).
struct TokenCorpus {
  std::span<const uint64_t> doc_offsets;  // num_docs + 1 entries
  std::span<const uint32_t> token_ids;
  uint32_t vocab_size = 0;
};

struct BuildOptions {
  int device = 0;
  bool keep_tf = false;
  float dense_min_density = 0.f;  // <= 0: library default
  uint32_t doc_base = 0;          // shard's first global doc id
  sl_comm* comm = nullptr;        // NCCL communicator for a document-sharded corpus
};

// SPEC retrieval QueryResult: doc indices with exact B(Q,D) scores, descending;
// external_ids for a text index.
struct QueryResult {
  std::vector<uint32_t> doc_indices;
  std::vector<std::string> external_ids;
  std::vector<float> scores;
};

// A device-resident index shard (move-only RAII over sl_index*).
class SearchIndex {
 public:
  SearchIndex() = default;
  explicit SearchIndex(sl_index* h) : h_(h) {}
  SearchIndex(SearchIndex&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  SearchIndex& operator=(SearchIndex&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  SearchIndex(const SearchIndex&) = delete;
  SearchIndex& operator=(const SearchIndex&) = delete;
  ~SearchIndex() { reset(); }

  sl_index* handle() const {
    if (!h_) throw std::invalid_argument("SearchIndex: empty handle");
    return h_;
  }
  sl_index_info info() const {
    sl_index_info i{};
    check(sl_index_get_info(handle(), &i));
    return i;
  }
  uint32_t num_docs() const { return info().num_docs_global; }
  uint32_t vocab_size() const { return info().vocab_size; }
  double avg_len() const { return info().avg_len; }

  // ScoreMatrix + statistics (SPEC index External Interfaces layout)
  struct Arrays {
    std::vector<uint64_t> indptr;
    std::vector<uint32_t> docids;
    std::vector<float> values;
    std::vector<uint32_t> df;
    std::vector<float> theta;
    std::vector<uint32_t> doclens;
  };
  Arrays export_arrays() const {
    const sl_index_info i = info();
    Arrays a;
    a.indptr.resize(i.vocab_size + 1ull);
    a.docids.resize(i.nnz_local);
    a.values.resize(i.nnz_local);
    a.df.resize(i.vocab_size);
    a.theta.resize(i.vocab_size);
    a.doclens.resize(i.num_docs_local);
    check(sl_index_export(handle(), SL_MEM_HOST, a.indptr.data(), a.docids.data(), a.values.data(), a.df.data(),
                          a.theta.data(), a.doclens.data(), nullptr));
    return a;
  }

 private:
  void reset() {
    if (h_) sl_index_destroy(h_);
    h_ = nullptr;
  }
  sl_index* h_ = nullptr;
};

inline SearchIndex build_index(const TokenCorpus& corpus, const BM25Params& params, const BuildOptions& opt = {}) {
  if (corpus.doc_offsets.size() < 2) throw std::invalid_argument("build_index: empty corpus");
  // the library copies tokens [doc_offsets[0], doc_offsets[N]) from the host pointer
  if (corpus.doc_offsets.back() > corpus.token_ids.size() || corpus.doc_offsets.front() > corpus.doc_offsets.back())
    throw std::invalid_argument("build_index: doc offsets exceed the token array");
  sl_build_desc d{};
  d.doc_offsets = corpus.doc_offsets.data();
  d.token_ids = corpus.token_ids.data();
  d.num_docs = static_cast<uint32_t>(corpus.doc_offsets.size() - 1);
  d.vocab_size = corpus.vocab_size;
  d.doc_base = opt.doc_base;
  d.mem = SL_MEM_HOST;
  d.params = to_c(params);
  d.device = opt.device;
  d.keep_tf = opt.keep_tf ? 1 : 0;
  d.dense_min_density = opt.dense_min_density;
  d.comm = opt.comm;
  sl_index* h = nullptr;
  check(sl_index_build(&d, &h));
  return SearchIndex(h);
}

// SPEC save_index / load_index (9-file layout)
inline void save_index(const SearchIndex& index, const std::string& directory) {
  check(sl_index_save(index.handle(), directory.c_str()));
}
inline SearchIndex load_index(const std::string& directory, int device = 0) {
  sl_index* h = nullptr;
  check(sl_index_load(directory.c_str(), device, 0.f, &h));
  return SearchIndex(h);
}

inline std::vector<float> score_query(const SearchIndex& index, std::span<const uint32_t> query) {
  std::vector<float> out(index.info().num_docs_local);
  check(sl_score_query(index.handle(), query.data(), static_cast<uint32_t>(query.size()), SL_MEM_HOST, out.data()));
  return out;
}

inline QueryResult top_k(std::span<const float> scores, uint32_t k, bool ordered = true, int device = 0) {
  if (k == 0) throw std::invalid_argument("top_k: k must be >= 1");
  QueryResult r;
  r.doc_indices.resize(k);
  r.scores.resize(k);
  check(sl_top_k(scores.data(), static_cast<uint32_t>(scores.size()), k, ordered ? 1 : 0, SL_MEM_HOST, device,
                 r.doc_indices.data(), r.scores.data()));
  const size_t m = k < scores.size() ? k : scores.size();
  r.doc_indices.resize(m);
  r.scores.resize(m);
  return r;
}

// workers: accepted for SPEC parity (results are identical for any value; the batch is
// one device launch sequence).
inline std::vector<QueryResult> retrieve_batch(const SearchIndex& index,
                                               const std::vector<std::vector<uint32_t>>& queries, uint32_t k,
                                               bool ordered = true, int workers = 1) {
  if (workers < 1) throw std::invalid_argument("retrieve_batch: workers must be >= 1");
  if (k == 0) throw std::invalid_argument("top_k: k must be >= 1");
  std::vector<uint64_t> off(queries.size() + 1, 0);
  for (size_t i = 0; i < queries.size(); ++i) off[i + 1] = off[i] + queries[i].size();
  std::vector<uint32_t> tok;
  tok.reserve(off.back());
  for (const auto& q : queries) tok.insert(tok.end(), q.begin(), q.end());
  if (tok.empty()) tok.push_back(0);
  const size_t B = queries.size();
  std::vector<uint32_t> ids(B * k);
  std::vector<float> sc(B * k);
  if (B) {
    check(sl_retrieve_batch(index.handle(), off.data(), tok.data(), static_cast<uint32_t>(B), k, ordered ? 1 : 0,
                            SL_MEM_HOST, ids.data(), sc.data()));
  }
  const uint32_t n = index.num_docs();
  const size_t m = k < n ? k : n;
  std::vector<QueryResult> out(B);
  for (size_t b = 0; b < B; ++b) {
    out[b].doc_indices.assign(ids.begin() + b * k, ids.begin() + b * k + m);
    out[b].scores.assign(sc.begin() + b * k, sc.begin() + b * k + m);
  }
  return out;
}

inline QueryResult retrieve(const SearchIndex& index, std::span<const uint32_t> query, uint32_t k,
                            bool ordered = true) {
  return std::move(retrieve_batch(index, {std::vector<uint32_t>(query.begin(), query.end())}, k, ordered)[0]);
}

// ---------------------------------------------------------------- text (SPEC [MODULE] tokenizer)
// stemmer.hpp:8-11
enum class StemmerKind : int32_t { none = SL_STEMMER_NONE, snowball_english = SL_STEMMER_SNOWBALL_ENGLISH };

// tokenizer.hpp:16-23; stopwords compared with the lowercased pre-stem token
struct TokenizerConfig {
  bool lowercase = true;
  std::vector<std::string> stopwords;
  StemmerKind stemmer = StemmerKind::none;
};

// vocabulary.hpp:13-48 on the device (ids in first-encounter order)
class Vocabulary {
 public:
  explicit Vocabulary(int device = 0) { check(sl_vocab_create(device, &h_)); }
  Vocabulary(Vocabulary&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  Vocabulary& operator=(Vocabulary&& o) noexcept {
    if (this != &o) {
      if (h_) sl_vocab_destroy(h_);
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  Vocabulary(const Vocabulary&) = delete;
  Vocabulary& operator=(const Vocabulary&) = delete;
  ~Vocabulary() {
    if (h_) sl_vocab_destroy(h_);
  }
  sl_vocab* handle() const { return h_; }
  uint32_t size() const {
    uint32_t n = 0;
    check(sl_vocab_size(h_, &n));
    return n;
  }
  std::vector<std::string> tokens() const {
    const uint32_t n = size();
    std::vector<uint64_t> off(n + 1ull);
    uint64_t total = 0;
    check(sl_vocab_export(h_, nullptr, nullptr, &total));
    std::string bytes(total, '\0');
    check(sl_vocab_export(h_, off.data(), bytes.data(), &total));
    std::vector<std::string> out(n);
    for (uint32_t i = 0; i < n; ++i) out[i] = bytes.substr(off[i], off[i + 1] - off[i]);
    return out;
  }

 private:
  sl_vocab* h_ = nullptr;
};

// Token ids per document (host copy of a device sl_token_batch)
struct TokenizedCorpus {
  std::vector<uint64_t> doc_offsets;
  std::vector<uint32_t> token_ids;
  std::vector<uint32_t> doc(size_t d) const {
    return {token_ids.begin() + doc_offsets[d], token_ids.begin() + doc_offsets[d + 1]};
  }
};

namespace detail {
struct CfgC {
  std::string blob;
  sl_tokenizer_config c{};
  explicit CfgC(const TokenizerConfig& t) {
    for (const auto& w : t.stopwords) blob += w + "\n";
    c.lowercase = t.lowercase ? 1 : 0;
    c.stemmer = static_cast<int32_t>(t.stemmer);
    c.stopwords = blob.empty() ? nullptr : blob.data();
    c.stopwords_bytes = blob.size();
  }
};
inline TokenizedCorpus tokenize(const std::vector<std::string>& texts, const TokenizerConfig& cfg, Vocabulary& v,
                                bool build) {
  std::string all;
  std::vector<uint64_t> off{0};
  for (const auto& t : texts) {
    all += t;
    off.push_back(all.size());
  }
  if (all.empty()) all.push_back('\0');
  CfgC c(cfg);
  sl_token_batch* b = nullptr;
  check(sl_tokenize(v.handle(), &c.c, build ? 1 : 0, all.data(), off.data(), static_cast<uint32_t>(texts.size()),
                    SL_MEM_HOST, &b));
  uint32_t n = 0;
  uint64_t T = 0;
  sl_token_batch_info(b, &n, &T, nullptr, nullptr);
  TokenizedCorpus out;
  out.doc_offsets.resize(n + 1ull);
  out.token_ids.resize(T);
  const int32_t rc = sl_token_batch_copy(b, out.doc_offsets.data(), out.token_ids.data());
  sl_token_batch_destroy(b);
  check(rc);
  return out;
}
}  // namespace detail

// tokenize_build / tokenize_query (tokenizer.hpp:36-45), every text a separate document
inline TokenizedCorpus tokenize_build(const std::vector<std::string>& texts, const TokenizerConfig& cfg,
                                      Vocabulary& vocab) {
  return detail::tokenize(texts, cfg, vocab, true);
}
inline TokenizedCorpus tokenize_query(const std::vector<std::string>& texts, const TokenizerConfig& cfg,
                                      Vocabulary& vocab) {
  return detail::tokenize(texts, cfg, vocab, false);
}

// tokenize_build / tokenize_query over a corpus already concatenated in host memory (text bytes
// + u64 doc offsets[N+1]): sl_tokenize_stream, document-aligned chunks with the copies to and
// from the device overlapping the device work (chunk_bytes 0: the library default)
inline TokenizedCorpus tokenize_stream(const std::string& text, const std::vector<uint64_t>& doc_offsets,
                                       const TokenizerConfig& cfg, Vocabulary& vocab, bool build,
                                       uint64_t chunk_bytes = 0) {
  if (doc_offsets.empty()) throw std::invalid_argument("tokenize_stream: doc_offsets needs N+1 entries");
  detail::CfgC c(cfg);
  const uint32_t n = static_cast<uint32_t>(doc_offsets.size() - 1);
  TokenizedCorpus out;
  out.doc_offsets.resize(doc_offsets.size());
  out.token_ids.resize(text.size() / 2 + 1);  // a token takes >= 2 bytes
  uint64_t T = 0;
  check(sl_tokenize_stream(vocab.handle(), &c.c, build ? 1 : 0, text.data(), doc_offsets.data(), n, chunk_bytes,
                           out.doc_offsets.data(), out.token_ids.data(), out.token_ids.size(), &T));
  out.token_ids.resize(T);
  return out;
}

// stem_english (stemmer.hpp:16-18), on the device
inline std::vector<std::string> stem_english(const std::vector<std::string>& words, int device = 0) {
  std::string all;
  std::vector<uint64_t> off{0};
  for (const auto& w : words) {
    all += w;
    off.push_back(all.size());
  }
  std::string out(all.size() + 1, '\0');
  std::vector<uint32_t> len(words.size());
  if (!words.empty())
    check(sl_stem_batch(all.data(), off.data(), static_cast<uint32_t>(words.size()), device, out.data(), len.data()));
  std::vector<std::string> r(words.size());
  for (size_t i = 0; i < words.size(); ++i) r[i] = out.substr(off[i], len[i]);
  return r;
}

// ---------------------------------------------------------------- text-level SearchIndex
// SPEC SearchIndex with vocabulary, tokenizer config and external document ids,
// move-only RAII over the library's sl_text_index.
class TextIndex {
 public:
  TextIndex() = default;
  explicit TextIndex(sl_text_index* h) : h_(h) {}
  TextIndex(TextIndex&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  TextIndex& operator=(TextIndex&& o) noexcept {
    if (this != &o) {
      if (h_) sl_text_index_destroy(h_);
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  TextIndex(const TextIndex&) = delete;
  TextIndex& operator=(const TextIndex&) = delete;
  ~TextIndex() {
    if (h_) sl_text_index_destroy(h_);
  }
  sl_text_index* handle() const {
    if (!h_) throw std::invalid_argument("TextIndex: empty handle");
    return h_;
  }
  uint32_t num_docs() const {
    uint32_t n = 0;
    check(sl_text_index_num_docs(handle(), &n));
    return n;
  }
  std::string external_id(uint32_t doc) const {
    const char* p = nullptr;
    uint64_t n = 0;
    check(sl_text_index_external_id(handle(), doc, &p, &n));
    return std::string(p, n);
  }
  std::vector<std::string> doc_external_ids() const {
    std::vector<std::string> out(num_docs());
    for (uint32_t d = 0; d < out.size(); ++d) out[d] = external_id(d);
    return out;
  }
  // vocabulary tokens in id order (vocabulary.hpp:13-48)
  std::vector<std::string> vocab_tokens() const {
    sl_vocab* v = sl_text_index_vocab(handle());
    uint32_t n = 0;
    check(sl_vocab_size(v, &n));
    std::vector<uint64_t> off(n + 1ull);
    uint64_t total = 0;
    check(sl_vocab_export(v, nullptr, nullptr, &total));
    std::string bytes(total, '\0');
    check(sl_vocab_export(v, off.data(), bytes.data(), &total));
    std::vector<std::string> out(n);
    for (uint32_t i = 0; i < n; ++i) out[i] = bytes.substr(off[i], off[i + 1] - off[i]);
    return out;
  }
  TokenizerConfig tokenizer_config() const {
    sl_tokenizer_config c{};
    check(sl_text_index_config(handle(), &c));
    TokenizerConfig t;
    t.lowercase = c.lowercase != 0;
    t.stemmer = static_cast<StemmerKind>(c.stemmer);
    std::string cur;
    for (uint64_t i = 0; i <= c.stopwords_bytes; ++i) {
      if (i == c.stopwords_bytes || c.stopwords[i] == '\n') {
        if (!cur.empty()) t.stopwords.push_back(cur);
        cur.clear();
      } else {
        cur += c.stopwords[i];
      }
    }
    return t;
  }
  // token-id level view of the same index (score_query / export_arrays); owned by this TextIndex
  const sl_index* index() const { return sl_text_index_index(handle()); }

 private:
  sl_text_index* h_ = nullptr;
};

// SPEC build_index(corpus: sequence of (external_id, text), params, tokenizer_config) SPEC.md:201-209;
// throws std::invalid_argument on an empty corpus, a degenerate corpus or duplicate external ids
inline TextIndex build_text_index(const std::vector<std::pair<std::string, std::string>>& corpus,
                                  const BM25Params& params, const TokenizerConfig& cfg, int device = 0,
                                  float dense_min_density = 0.f) {
  std::string ids, text;
  std::vector<uint64_t> ioff{0}, toff{0};
  for (const auto& [id, t] : corpus) {
    ids += id;
    ioff.push_back(ids.size());
    text += t;
    toff.push_back(text.size());
  }
  if (ids.empty()) ids.push_back('\0');
  if (text.empty()) text.push_back('\0');
  detail::CfgC c(cfg);
  const sl_params p = to_c(params);
  sl_text_index* h = nullptr;
  check(sl_text_index_build(ids.data(), ioff.data(), text.data(), toff.data(), static_cast<uint32_t>(corpus.size()),
                            &p, &c.c, device, dense_min_density, &h));
  return TextIndex(h);
}
// documents without ids of their own get their position ("0", "1", ...) as external id
inline TextIndex build_text_index(const std::vector<std::string>& docs, const BM25Params& params,
                                  const TokenizerConfig& cfg, int device = 0) {
  std::vector<std::pair<std::string, std::string>> corpus;
  corpus.reserve(docs.size());
  for (size_t i = 0; i < docs.size(); ++i) corpus.emplace_back(std::to_string(i), docs[i]);
  return build_text_index(corpus, params, cfg, device);
}

// SPEC save_index / load_index for a text index
inline void save_index(const TextIndex& t, const std::string& directory) {
  check(sl_text_index_save(t.handle(), directory.c_str()));
}
inline TextIndex load_text_index(const std::string& directory, int device = 0) {
  sl_text_index* h = nullptr;
  check(sl_text_index_load(directory.c_str(), device, 0.f, &h));
  return TextIndex(h);
}

// SPEC retrieve_batch(index, queries, k, ordered, workers) over query texts
inline std::vector<QueryResult> retrieve_batch(const TextIndex& t, const std::vector<std::string>& queries,
                                               uint32_t k, bool ordered = true, int workers = 1) {
  if (workers < 1) throw std::invalid_argument("retrieve_batch: workers must be >= 1");
  if (k == 0) throw std::invalid_argument("top_k: k must be >= 1");
  std::string all;
  std::vector<uint64_t> off{0};
  for (const auto& q : queries) {
    all += q;
    off.push_back(all.size());
  }
  if (all.empty()) all.push_back('\0');
  const size_t B = queries.size();
  std::vector<uint32_t> ids(B * k);
  std::vector<float> sc(B * k);
  if (B)
    check(sl_text_index_retrieve(t.handle(), all.data(), off.data(), static_cast<uint32_t>(B), k, ordered ? 1 : 0,
                                 ids.data(), sc.data()));
  const uint32_t n = t.num_docs();
  const size_t m = k < n ? k : n;
  std::vector<QueryResult> out(B);
  for (size_t b = 0; b < B; ++b) {
    out[b].doc_indices.assign(ids.begin() + b * k, ids.begin() + b * k + m);
    out[b].scores.assign(sc.begin() + b * k, sc.begin() + b * k + m);
    for (uint32_t d : out[b].doc_indices) out[b].external_ids.push_back(t.external_id(d));
  }
  return out;
}
// SPEC retrieve(index, text, k, ordered): frozen vocabulary, OOV tokens dropped, external ids mapped
inline QueryResult retrieve(const TextIndex& t, const std::string& text, uint32_t k, bool ordered = true) {
  return std::move(retrieve_batch(t, std::vector<std::string>{text}, k, ordered)[0]);
}

}  // namespace sparselex::b200
