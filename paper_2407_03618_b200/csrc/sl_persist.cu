// sl_persist.cu — SPEC index persistence (save_index / load_index), SPEC.md [MODULE] index,
// "External Interfaces": a directory with
//   meta.json   {format_version, variant, k1, b, delta, num_docs, avg_len, num_tokens,
//                num_nonzeros, tokenizer: {lowercase, stopwords_hash, stemmer}}
//   vocab.json  {token: id}         (token-id corpora: the id's decimal string)
//   df.bin u32[V], theta.bin f32[V], indptr.bin u64[V+1], docids.bin u32[nnz],
//   values.bin f32[nnz], doclens.bin u32[N]  (little-endian)
//   docs.json   ordered external document ids (token-id corpora: global doc id strings)
// Extensions for document shards (ignored by a SPEC reader): num_docs_global, doc_base,
// vocab_size, total_len_global in meta.json. Saving copies straight from the device buffers;
// loading validates every ScoreMatrix invariant and rebuilds the query-side structures.
// Errors (SPEC load_index): missing file -> SL_EIO naming the path; corrupt lengths /
// invariants -> SL_ECORRUPT ("corrupt matrix"); format version mismatch -> SL_EUNSUPPORTED;
// vocabulary size != indptr length - 1 -> SL_ECORRUPT ("structural error").
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "sl_index.cuh"
#include "sl_json.h"
#include "sl_persist.h"

namespace sl {
namespace {

constexpr int kFormatVersion = 1;

const char* variant_name(int v) {
  static const char* n[] = {"robertson", "atire", "lucene", "bm25l", "bm25plus", "tfldp"};
  return v >= 0 && v < 6 ? n[v] : "?";
}
int variant_from_name(const std::string& s) {
  static const char* n[] = {"robertson", "atire", "lucene", "bm25l", "bm25plus", "tfldp"};
  for (int i = 0; i < 6; ++i)
    if (s == n[i]) return i;
  return -1;
}

std::string join(const std::string& dir, const char* f) { return dir + "/" + f; }

int32_t write_file(const std::string& path, const void* data, size_t bytes) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) SL_FAIL(SL_EIO, "save_index: cannot write " + path + ": " + std::strerror(errno));
  const size_t w = bytes ? std::fwrite(data, 1, bytes, f) : 0;
  const bool ok = w == bytes && std::fclose(f) == 0;
  if (!ok) SL_FAIL(SL_EIO, "save_index: short write to " + path);
  return SL_OK;
}

int32_t read_file(const std::string& path, std::string& out) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) SL_FAIL(SL_EIO, "load_index: missing file " + path);
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out.resize(n > 0 ? (size_t)n : 0);
  const size_t r = n > 0 ? std::fread(&out[0], 1, (size_t)n, f) : 0;
  std::fclose(f);
  if (r != out.size()) SL_FAIL(SL_EIO, "load_index: read error on " + path);
  return SL_OK;
}

template <class T>
int32_t read_array(const std::string& path, std::vector<T>& v, uint64_t expect, const char* what) {
  std::string raw;
  SL_TRY(read_file(path, raw));
  if (raw.size() != expect * sizeof(T))
    SL_FAIL(SL_ECORRUPT, std::string("load_index: corrupt matrix (") + what + " has " +
                             std::to_string(raw.size() / sizeof(T)) + " entries, expected " + std::to_string(expect) +
                             ")");
  v.resize(expect);
  if (expect) std::memcpy(v.data(), raw.data(), raw.size());
  return SL_OK;
}

template <class T>
int32_t d2h(std::vector<T>& v, const T* src, uint64_t n) {
  v.resize(n);
  if (n) SL_CUDA_TRY(cudaMemcpy(v.data(), src, n * sizeof(T), cudaMemcpyDeviceToHost));
  return SL_OK;
}

}  // namespace
}  // namespace sl

using namespace sl;

namespace sl {

int32_t save_index_impl(const sl_index* ix, const std::string& dir, const TextMeta* tm) {
  struct stat sb;
  if (stat(dir.c_str(), &sb) != 0 && mkdir(dir.c_str(), 0755) != 0)
    SL_FAIL(SL_EIO, "save_index: cannot create directory " + dir + ": " + std::strerror(errno));
  if (tm && ((tm->tokens && tm->tokens->size() != ix->V) || (tm->ext_ids && tm->ext_ids->size() != ix->N)))
    SL_FAIL(SL_EINVAL, "save_index: vocabulary / external ids do not match the index");
  SL_CUDA_TRY(cudaSetDevice(ix->device));
  std::vector<uint64_t> indptr;
  std::vector<uint32_t> docids, df, doclens;
  std::vector<float> values, theta;
  SL_TRY(d2h(indptr, ix->indptr, (uint64_t)ix->V + 1));
  SL_TRY(d2h(docids, ix->docids, ix->nnz));
  SL_TRY(d2h(values, ix->values, ix->nnz));
  SL_TRY(d2h(df, ix->df_global, ix->V));
  SL_TRY(d2h(theta, ix->theta, ix->V));
  SL_TRY(d2h(doclens, ix->doclens, ix->N));
  std::string tok;
  if (tm && tm->tokens) {
    tok = std::string("{\"lowercase\": ") + (tm->lowercase ? "true" : "false") +
          ", \"stopwords_hash\": " + std::to_string(tm->stopwords_hash) + ", \"stemmer\": \"" +
          (tm->stemmer == SL_STEMMER_SNOWBALL_ENGLISH ? "snowball-english" : "none") + "\"}";
  } else {
    tok = "{\"lowercase\": false, \"stopwords_hash\": \"none\", \"stemmer\": \"none\", \"input\": \"token-ids\"}";
  }
  char meta[2048];
  std::snprintf(meta, sizeof(meta),
                "{\n \"format_version\": %d,\n \"variant\": \"%s\",\n \"k1\": %.17g,\n \"b\": %.17g,\n"
                " \"delta\": %.17g,\n \"num_docs\": %u,\n \"avg_len\": %.17g,\n \"num_tokens\": %llu,\n"
                " \"num_nonzeros\": %llu,\n \"tokenizer\": %s,\n \"vocab_size\": %u,\n"
                " \"num_docs_global\": %u,\n \"doc_base\": %u,\n \"total_len_global\": %llu",
                kFormatVersion, variant_name(ix->params.variant), ix->params.k1, ix->params.b, ix->params.delta,
                ix->N, ix->avg_len, (unsigned long long)ix->total_len, (unsigned long long)ix->nnz, tok.c_str(), ix->V,
                ix->N_global, ix->doc_base, (unsigned long long)ix->total_len);
  std::string m(meta);
  if (tm && tm->stopwords) {  // extension: the list itself, so load_index restores the set (SPEC keeps the hash)
    m += ",\n \"stopwords\": [";
    for (size_t i = 0; i < tm->stopwords->size(); ++i) {
      if (i) m += ", ";
      json::escape_into(m, (*tm->stopwords)[i]);
    }
    m += "]";
  }
  m += "\n}\n";
  SL_TRY(write_file(join(dir, "meta.json"), m.data(), m.size()));
  std::string vocab = "{";
  vocab.reserve((size_t)ix->V * 20);
  for (uint32_t t = 0; t < ix->V; ++t) {
    if (t) vocab += ", ";
    if (tm && tm->tokens) json::escape_into(vocab, (*tm->tokens)[t]);
    else vocab += "\"" + std::to_string(t) + "\"";
    vocab += ": " + std::to_string(t);
  }
  vocab += "}\n";
  SL_TRY(write_file(join(dir, "vocab.json"), vocab.data(), vocab.size()));
  std::string docs = "[";
  docs.reserve((size_t)ix->N * 12);
  for (uint32_t d = 0; d < ix->N; ++d) {
    if (d) docs += ", ";
    if (tm && tm->ext_ids) json::escape_into(docs, (*tm->ext_ids)[d]);
    else docs += "\"" + std::to_string((uint64_t)ix->doc_base + d) + "\"";
  }
  docs += "]\n";
  SL_TRY(write_file(join(dir, "docs.json"), docs.data(), docs.size()));
  SL_TRY(write_file(join(dir, "df.bin"), df.data(), df.size() * 4));
  SL_TRY(write_file(join(dir, "theta.bin"), theta.data(), theta.size() * 4));
  SL_TRY(write_file(join(dir, "indptr.bin"), indptr.data(), indptr.size() * 8));
  SL_TRY(write_file(join(dir, "docids.bin"), docids.data(), docids.size() * 4));
  SL_TRY(write_file(join(dir, "values.bin"), values.data(), values.size() * 4));
  SL_TRY(write_file(join(dir, "doclens.bin"), doclens.data(), doclens.size() * 4));
  return SL_OK;
}

int32_t load_index_impl(const std::string& dir, int32_t device, float dense_min_density, sl_index** out,
                        LoadedText* text) {
  *out = nullptr;
  std::string meta, err;
  SL_TRY(read_file(join(dir, "meta.json"), meta));
  json::Value mv;
  if (!json::Parser(meta).parse(mv, err) || mv.kind != json::Value::kObject)
    SL_FAIL(SL_ECORRUPT, "load_index: corrupt meta.json (" + err + ")");
  const json::Value* fv = mv.get("format_version");
  if (!fv || fv->kind != json::Value::kNumber || fv->num() != kFormatVersion)
    SL_FAIL(SL_EUNSUPPORTED, "load_index: format version mismatch (expected " + std::to_string(kFormatVersion) +
                                 ", found " + (fv ? fv->text : std::string("none")) + ")");
  auto num = [&](const char* k, double& v) -> bool {
    const json::Value* x = mv.get(k);
    if (!x || x->kind != json::Value::kNumber) return false;
    v = x->num();
    return true;
  };
  HostIndex h;
  double k1, b, delta, nd, nnzd, avg, ntok;
  const json::Value* vn = mv.get("variant");
  if (!vn || vn->kind != json::Value::kString || !num("k1", k1) || !num("b", b) || !num("delta", delta) ||
      !num("num_docs", nd) || !num("avg_len", avg) || !num("num_nonzeros", nnzd) || !num("num_tokens", ntok))
    SL_FAIL(SL_ECORRUPT, "load_index: corrupt meta.json (missing fields)");
  h.params = sl_params{variant_from_name(vn->text), k1, b, delta};
  if (h.params.variant < 0) SL_FAIL(SL_ECORRUPT, "load_index: corrupt meta.json (unknown variant " + vn->text + ")");
  h.N = (uint32_t)nd;
  h.avg_len = avg;
  h.total_len = (uint64_t)ntok;
  double x;
  h.N_global = num("num_docs_global", x) ? (uint32_t)x : h.N;
  h.doc_base = num("doc_base", x) ? (uint32_t)x : 0u;
  if (num("total_len_global", x)) h.total_len = (uint64_t)x;
  // V from indptr.bin; vocab.json must agree (SPEC: structural error otherwise)
  std::string raw;
  SL_TRY(read_file(join(dir, "indptr.bin"), raw));
  if (raw.size() < 8 || raw.size() % 8) SL_FAIL(SL_ECORRUPT, "load_index: corrupt matrix (indptr.bin length)");
  h.V = (uint32_t)(raw.size() / 8 - 1);
  h.indptr.resize((size_t)h.V + 1);
  std::memcpy(h.indptr.data(), raw.data(), raw.size());
  std::string vocab;
  SL_TRY(read_file(join(dir, "vocab.json"), vocab));
  std::vector<std::pair<std::string, uint64_t>> ventries;
  if (!json::Parser(vocab).string_u64_object(ventries, err))
    SL_FAIL(SL_ECORRUPT, "load_index: structural error (vocab.json: " + err + ")");
  if (ventries.size() != h.V)
    SL_FAIL(SL_ECORRUPT, "load_index: structural error (vocab.json has " + std::to_string(ventries.size()) +
                             " tokens, indptr.bin describes " + std::to_string(h.V) + ")");
  if (text) {  // tokens in id order: the ids must be a permutation of 0..V-1
    text->tokens.assign(h.V, std::string());
    std::vector<uint8_t> seen(h.V, 0);
    for (auto& e : ventries) {
      if (e.second >= h.V || seen[e.second])
        SL_FAIL(SL_ECORRUPT, "load_index: structural error (vocab.json ids are not 0..V-1)");
      seen[e.second] = 1;
      text->tokens[e.second] = std::move(e.first);
    }
  }
  ventries.clear();
  ventries.shrink_to_fit();
  const uint64_t nnz = h.indptr.back();
  if (nnz != (uint64_t)nnzd) SL_FAIL(SL_ECORRUPT, "load_index: corrupt matrix (num_nonzeros != indptr[V])");
  SL_TRY(read_array(join(dir, "docids.bin"), h.docids, nnz, "docids.bin"));
  SL_TRY(read_array(join(dir, "values.bin"), h.values, nnz, "values.bin"));
  SL_TRY(read_array(join(dir, "df.bin"), h.df, h.V, "df.bin"));
  SL_TRY(read_array(join(dir, "theta.bin"), h.theta, h.V, "theta.bin"));
  SL_TRY(read_array(join(dir, "doclens.bin"), h.doclens, h.N, "doclens.bin"));
  std::string docs;
  SL_TRY(read_file(join(dir, "docs.json"), docs));
  std::vector<std::string> ids;
  if (!json::Parser(docs).string_array(ids, err))
    SL_FAIL(SL_ECORRUPT, "load_index: structural error (docs.json: " + err + ")");
  if (ids.size() != h.N) SL_FAIL(SL_ECORRUPT, "load_index: structural error (docs.json does not list num_docs ids)");
  if (text) {
    text->ext_ids = std::move(ids);
    const json::Value* tk = mv.get("tokenizer");
    text->lowercase = false;
    text->stemmer = SL_STEMMER_NONE;
    text->has_hash = false;
    text->stopwords.clear();
    if (tk && tk->kind == json::Value::kObject) {
      const json::Value* lc = tk->get("lowercase");
      text->lowercase = lc && lc->kind == json::Value::kBool && lc->b;
      const json::Value* st = tk->get("stemmer");
      if (st && st->kind == json::Value::kString) {
        if (st->text == "snowball-english" || st->text == "snowball_english") text->stemmer = SL_STEMMER_SNOWBALL_ENGLISH;
        else if (st->text != "none") SL_FAIL(SL_ECORRUPT, "load_index: corrupt meta.json (unknown stemmer " + st->text + ")");
      }
      const json::Value* hv = tk->get("stopwords_hash");
      if (hv && hv->kind == json::Value::kNumber) {
        text->has_hash = true;
        text->stopwords_hash = hv->u64();
      }
    }
    const json::Value* sw = mv.get("stopwords");
    if (sw && sw->kind == json::Value::kArray)
      for (const auto& w : sw->arr)
        if (w.kind == json::Value::kString) text->stopwords.push_back(w.text);
  }
  return load_index_from_host(h, device, dense_min_density, out);
}

}  // namespace sl

extern "C" {

int32_t sl_index_save(const sl_index* ix, const char* directory) {
  if (!ix || !directory) SL_FAIL(SL_EINVAL, "save_index: null argument");
  return save_index_impl(ix, directory, nullptr);
}

int32_t sl_index_load(const char* directory, int32_t device, float dense_min_density, sl_index** out) {
  if (!directory || !out) SL_FAIL(SL_EINVAL, "load_index: null argument");
  return load_index_impl(directory, device, dense_min_density, out, nullptr);
}

}  // extern "C"
