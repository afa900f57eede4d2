// sl_textindex.cpp — the SPEC's text-level SearchIndex in the host language (C++), behind the C-ABI
// sl_text_index_* of include/sparselex_b200.h:
//   build_index(corpus: sequence of (external_id, text), params, tokenizer_config)
//     errors: empty corpus, degenerate corpus, duplicate external ids
//   SearchIndex.vocab / doc_external_ids / tokenizer_config
//   save_index / load_index of the 9-file layout with the real vocab.json, docs.json
//     and meta.json tokenizer fields
//   retrieve / retrieve_batch over query texts; QueryResult.external_ids via
//     sl_text_index_external_id
// Host plumbing only: tokenisation (sl_tokenize), the index build and retrieval all run on the
// GPU through the same entry points as the token-id path; nothing here computes scores.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include "sl_internal_host.h"
#include "sl_persist.h"
#include "sparselex_b200.h"

struct sl_text_index {
  sl_index* index = nullptr;
  sl_vocab* vocab = nullptr;
  int32_t device = 0;
  int32_t lowercase = 1;
  int32_t stemmer = SL_STEMMER_NONE;
  std::vector<std::string> stopwords;  // sorted, distinct
  std::string stop_blob;               // newline-separated (sl_tokenizer_config.stopwords)
  std::vector<std::string> ext_ids;    // SearchIndex.doc_external_ids

  ~sl_text_index() {
    if (index) sl_index_destroy(index);
    if (vocab) sl_vocab_destroy(vocab);
  }
  sl_tokenizer_config config() const {
    sl_tokenizer_config c{};
    c.lowercase = lowercase;
    c.stemmer = stemmer;
    c.stopwords = stop_blob.empty() ? nullptr : stop_blob.data();
    c.stopwords_bytes = stop_blob.size();
    return c;
  }
};

namespace {

#define TI_FAIL(code, msg)  \
  do {                      \
    sl::set_error(msg);     \
    return (code);          \
  } while (0)

// stopwords.hpp:17-19: order-independent hash of the set = Σ FNV-1a-64(word) mod 2^64
uint64_t stopwords_hash(const std::vector<std::string>& words) {
  uint64_t tot = 0;
  for (const auto& w : words) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (unsigned char c : w) h = (h ^ c) * 0x100000001B3ull;
    tot += h;
  }
  return tot;
}

// the stopword set of a config blob (newline-separated, '#' lines and blanks ignored,
// stopwords.hpp:13-15), sorted and distinct
std::vector<std::string> stopword_set(const sl_tokenizer_config* c) {
  std::vector<std::string> out;
  if (!c || !c->stopwords) return out;
  std::string cur;
  auto flush = [&] {
    while (!cur.empty() && (cur.back() == '\r' || cur.back() == ' ' || cur.back() == '\t')) cur.pop_back();
    size_t b = 0;
    while (b < cur.size() && (cur[b] == ' ' || cur[b] == '\t')) ++b;
    cur.erase(0, b);
    if (!cur.empty() && cur[0] != '#') out.push_back(cur);
    cur.clear();
  };
  for (uint64_t i = 0; i < c->stopwords_bytes; ++i) {
    if (c->stopwords[i] == '\n') flush();
    else cur += c->stopwords[i];
  }
  flush();
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

void set_stopwords(sl_text_index* t, std::vector<std::string> words) {
  t->stopwords = std::move(words);
  t->stop_blob.clear();
  for (size_t i = 0; i < t->stopwords.size(); ++i) {
    if (i) t->stop_blob += '\n';
    t->stop_blob += t->stopwords[i];
  }
}

int32_t vocab_tokens(const sl_vocab* v, std::vector<std::string>& out) {
  uint32_t n = 0;
  int32_t rc = sl_vocab_size(v, &n);
  if (rc) return rc;
  std::vector<uint64_t> off((size_t)n + 1);
  uint64_t total = 0;
  if ((rc = sl_vocab_export(v, nullptr, nullptr, &total))) return rc;
  std::string bytes(total, '\0');
  if ((rc = sl_vocab_export(v, off.data(), bytes.data(), &total))) return rc;
  out.resize(n);
  for (uint32_t i = 0; i < n; ++i) out[i] = bytes.substr(off[i], off[i + 1] - off[i]);
  return SL_OK;
}

}  // namespace

extern "C" {

int32_t sl_text_index_build(const char* ext_ids, const uint64_t* id_offsets, const char* text,
                            const uint64_t* text_offsets, uint32_t num_docs, const sl_params* params,
                            const sl_tokenizer_config* config, int32_t device, float dense_min_density,
                            sl_text_index** out) {
  if (!out || !params || !config || !id_offsets || !text_offsets) TI_FAIL(SL_EINVAL, "build_index: null argument");
  *out = nullptr;
  if (num_docs == 0) TI_FAIL(SL_EINVAL, "build_index: empty corpus");
  if ((id_offsets[num_docs] > id_offsets[0] && !ext_ids) || (text_offsets[num_docs] > text_offsets[0] && !text))
    TI_FAIL(SL_EINVAL, "build_index: null corpus bytes");
  if (int32_t rc = sl_params_validate(params)) return rc;
  auto* t = new sl_text_index();
  t->device = device;
  t->lowercase = config->lowercase ? 1 : 0;
  t->stemmer = config->stemmer;
  set_stopwords(t, stopword_set(config));
  t->ext_ids.resize(num_docs);
  {
    std::unordered_set<std::string> seen;
    seen.reserve(num_docs * 2ull);
    for (uint32_t d = 0; d < num_docs; ++d) {
      if (id_offsets[d + 1] < id_offsets[d]) {
        delete t;
        TI_FAIL(SL_EINVAL, "build_index: external id offsets must be non-decreasing");
      }
      t->ext_ids[d].assign(ext_ids + id_offsets[d], id_offsets[d + 1] - id_offsets[d]);
      if (!seen.insert(t->ext_ids[d]).second) {
        const std::string dup = t->ext_ids[d];
        delete t;
        TI_FAIL(SL_EINVAL, "build_index: duplicate external ids (\"" + dup + "\")");
      }
    }
  }
  int32_t rc = sl_vocab_create(device, &t->vocab);
  sl_token_batch* batch = nullptr;
  if (!rc) {
    const sl_tokenizer_config c = t->config();
    rc = sl_tokenize(t->vocab, &c, 1, text ? text : "", text_offsets, num_docs, SL_MEM_HOST, &batch);
  }
  if (!rc) {
    uint32_t n = 0, V = 0;
    uint64_t T = 0;
    const uint64_t* d_off = nullptr;
    const uint32_t* d_ids = nullptr;
    rc = sl_token_batch_info(batch, &n, &T, &d_off, &d_ids);
    if (!rc && T == 0) {
      sl::set_error("build_index: degenerate corpus (every document tokenizes to empty)");
      rc = SL_EINVAL;
    }
    if (!rc) rc = sl_vocab_size(t->vocab, &V);
    if (!rc) {
      sl_build_desc d{};
      d.doc_offsets = d_off;
      d.token_ids = d_ids;
      d.num_docs = n;
      d.vocab_size = V;
      d.mem = SL_MEM_DEVICE;
      d.params = *params;
      d.device = device;
      d.dense_min_density = dense_min_density;
      rc = sl_index_build(&d, &t->index);
    }
  }
  if (batch) {
    const std::string keep = sl::get_error();
    sl_token_batch_destroy(batch);
    sl::set_error(keep);
  }
  if (rc) {
    delete t;
    return rc;
  }
  *out = t;
  return SL_OK;
}

void sl_text_index_destroy(sl_text_index* t) { delete t; }

const sl_index* sl_text_index_index(const sl_text_index* t) { return t ? t->index : nullptr; }

sl_vocab* sl_text_index_vocab(const sl_text_index* t) { return t ? t->vocab : nullptr; }

int32_t sl_text_index_config(const sl_text_index* t, sl_tokenizer_config* out) {
  if (!t || !out) TI_FAIL(SL_EINVAL, "sl_text_index_config: null argument");
  *out = t->config();
  return SL_OK;
}

int32_t sl_text_index_num_docs(const sl_text_index* t, uint32_t* out) {
  if (!t || !out) TI_FAIL(SL_EINVAL, "sl_text_index_num_docs: null argument");
  *out = (uint32_t)t->ext_ids.size();
  return SL_OK;
}

int32_t sl_text_index_external_id(const sl_text_index* t, uint32_t doc, const char** id, uint64_t* len) {
  if (!t || !id || !len) TI_FAIL(SL_EINVAL, "sl_text_index_external_id: null argument");
  if (doc >= t->ext_ids.size()) TI_FAIL(SL_EINVAL, "sl_text_index_external_id: document index out of range");
  *id = t->ext_ids[doc].data();
  *len = t->ext_ids[doc].size();
  return SL_OK;
}

int32_t sl_text_index_save(const sl_text_index* t, const char* directory) {
  if (!t || !directory) TI_FAIL(SL_EINVAL, "save_index: null argument");
  std::vector<std::string> toks;
  if (int32_t rc = vocab_tokens(t->vocab, toks)) return rc;
  sl::TextMeta tm;
  tm.tokens = &toks;
  tm.ext_ids = &t->ext_ids;
  tm.stopwords = &t->stopwords;
  tm.lowercase = t->lowercase != 0;
  tm.stemmer = t->stemmer;
  tm.stopwords_hash = stopwords_hash(t->stopwords);
  return sl::save_index_impl(t->index, directory, &tm);
}

int32_t sl_text_index_load(const char* directory, int32_t device, float dense_min_density, sl_text_index** out) {
  if (!directory || !out) TI_FAIL(SL_EINVAL, "load_index: null argument");
  *out = nullptr;
  sl::LoadedText lt;
  auto* t = new sl_text_index();
  t->device = device;
  int32_t rc = sl::load_index_impl(directory, device, dense_min_density, &t->index, &lt);
  if (!rc && lt.has_hash && stopwords_hash(lt.stopwords) != lt.stopwords_hash) {
    sl::set_error("load_index: stopword configuration does not match the index (stopwords_hash)");
    rc = SL_ECORRUPT;
  }
  if (!rc) rc = sl_vocab_create(device, &t->vocab);
  if (!rc && !lt.tokens.empty()) {
    std::vector<uint64_t> off(lt.tokens.size() + 1, 0);
    std::string bytes;
    for (size_t i = 0; i < lt.tokens.size(); ++i) {
      bytes += lt.tokens[i];
      off[i + 1] = bytes.size();
    }
    if (bytes.empty()) bytes.push_back('\0');
    rc = sl_vocab_import(t->vocab, off.data(), bytes.data(), (uint32_t)lt.tokens.size());
  }
  if (rc) {
    delete t;
    return rc;
  }
  t->lowercase = lt.lowercase ? 1 : 0;
  t->stemmer = lt.stemmer;
  std::sort(lt.stopwords.begin(), lt.stopwords.end());
  lt.stopwords.erase(std::unique(lt.stopwords.begin(), lt.stopwords.end()), lt.stopwords.end());
  set_stopwords(t, std::move(lt.stopwords));
  t->ext_ids = std::move(lt.ext_ids);
  *out = t;
  return SL_OK;
}

int32_t sl_text_index_retrieve(const sl_text_index* t, const char* text, const uint64_t* offsets,
                               uint32_t num_queries, uint32_t k, int32_t ordered, uint32_t* out_ids,
                               float* out_scores) {
  if (!t || !offsets) TI_FAIL(SL_EINVAL, "retrieve_batch: null argument");
  if (k == 0) TI_FAIL(SL_EINVAL, "top_k: k must be >= 1");
  if (num_queries == 0) return SL_OK;
  if (!out_ids || !out_scores) TI_FAIL(SL_EINVAL, "retrieve_batch: null output pointers");
  // tokenize_query with the index's config and frozen vocabulary, on the device
  const sl_tokenizer_config c = t->config();
  sl_token_batch* batch = nullptr;
  int32_t rc = sl_tokenize(t->vocab, &c, 0, text ? text : "", offsets, num_queries, SL_MEM_HOST, &batch);
  if (rc) return rc;
  uint32_t n = 0;
  uint64_t T = 0;
  const uint64_t* d_off = nullptr;
  const uint32_t* d_ids = nullptr;
  rc = sl_token_batch_info(batch, &n, &T, &d_off, &d_ids);
  uint32_t* d_out_ids = nullptr;
  float* d_out_sc = nullptr;
  const uint64_t cnt = (uint64_t)num_queries * k;
  if (!rc && (cudaSetDevice(t->device) != cudaSuccess || cudaMalloc((void**)&d_out_ids, cnt * 4) != cudaSuccess ||
              cudaMalloc((void**)&d_out_sc, cnt * 4) != cudaSuccess)) {
    sl::set_error("retrieve_batch: device allocation of the results failed");
    rc = SL_ENOMEM;
  }
  if (!rc)
    rc = sl_retrieve_batch(t->index, d_off, d_ids ? d_ids : reinterpret_cast<const uint32_t*>(d_off), n, k, ordered,
                           SL_MEM_DEVICE, d_out_ids, d_out_sc);
  if (!rc && (cudaMemcpy(out_ids, d_out_ids, cnt * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
              cudaMemcpy(out_scores, d_out_sc, cnt * 4, cudaMemcpyDeviceToHost) != cudaSuccess)) {
    sl::set_error("retrieve_batch: copy of the results failed");
    rc = SL_ECUDA;
  }
  const std::string keep = sl::get_error();
  if (d_out_ids) cudaFree(d_out_ids);
  if (d_out_sc) cudaFree(d_out_sc);
  sl_token_batch_destroy(batch);
  sl::set_error(keep);
  return rc;
}

}  // extern "C"
