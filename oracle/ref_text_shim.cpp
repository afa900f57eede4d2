// ref_text_shim.cpp — extern "C" entry points over the REFERENCE's own text pipeline.
//
// Compiled by oracle/Makefile together with /root/reference/proj/src/{tokenizer,stemmer,
// unicode_tables}.cpp (read in place, never copied) into oracle/_ref/libref_text.so. Test
// infrastructure only: it pins the oracle's restated tokenizer / stemmer and generates the
// golden fixtures under tests/golden/ (tests/golden/make_text_golden.py).
//
// The reference declares english_stopwords() (proj/include/sparselex/stopwords.hpp:11) and
// calls it from TokenizerConfig::english() (proj/src/tokenizer.cpp:133-135) but never defines
// it; this shim defines it over the list the caller installs (ref_set_stopwords), which the
// tests fill from paper_2407_03618_b200/data/stopwords_en.txt.
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include "sparselex/stemmer.hpp"
#include "sparselex/stopwords.hpp"
#include "sparselex/tokenizer.hpp"
#include "sparselex/vocabulary.hpp"

namespace {
std::unordered_set<std::string> g_stop;

std::vector<std::string> split_lines(const char* s, size_t n) {
  std::vector<std::string> out;
  std::string cur;
  for (size_t i = 0; i < n; ++i) {
    if (s[i] == '\n') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(s[i]);
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

sparselex::TokenizerConfig make_cfg(int lowercase, int stop, int stem) {
  sparselex::TokenizerConfig c;
  c.lowercase = lowercase != 0;
  if (stop) c.stopwords = g_stop;
  c.stemmer = stem ? sparselex::StemmerKind::snowball_english : sparselex::StemmerKind::none;
  return c;
}

// joins strings with '\n' into out (cap bytes); returns the needed size
size_t join(const std::vector<std::string>& v, char* out, size_t cap) {
  size_t need = 0;
  for (const auto& s : v) need += s.size() + 1;
  if (out && need <= cap) {
    size_t o = 0;
    for (const auto& s : v) {
      std::memcpy(out + o, s.data(), s.size());
      o += s.size();
      out[o++] = '\n';
    }
  }
  return need;
}
}  // namespace

namespace sparselex {
const std::unordered_set<std::string>& english_stopwords() { return g_stop; }
}  // namespace sparselex

extern "C" {
// newline-separated list (the data file's non-comment lines)
void ref_set_stopwords(const char* words, size_t n) {
  g_stop.clear();
  for (auto& w : split_lines(words, n)) g_stop.insert(w);
}

// split_text (tokenizer.hpp:34): tokens joined with '\n'; returns the needed size
size_t ref_split_text(const char* text, size_t n, int lowercase, char* out, size_t cap) {
  return join(sparselex::split_text(std::string_view(text, n), lowercase != 0), out, cap);
}

// stem_english (stemmer.hpp:18): returns the stem's byte length (written when it fits)
size_t ref_stem(const char* word, size_t n, char* out, size_t cap) {
  const std::string s = sparselex::stem_english(std::string_view(word, n));
  if (out && s.size() <= cap) std::memcpy(out, s.data(), s.size());
  return s.size();
}

void* ref_vocab_new(void) { return new sparselex::Vocabulary(); }
void ref_vocab_free(void* v) { delete static_cast<sparselex::Vocabulary*>(v); }
uint32_t ref_vocab_size(void* v) { return static_cast<sparselex::Vocabulary*>(v)->size(); }
// all tokens in id order, joined with '\n'
size_t ref_vocab_tokens(void* v, char* out, size_t cap) {
  return join(static_cast<sparselex::Vocabulary*>(v)->tokens(), out, cap);
}

// tokenize_build / tokenize_query (tokenizer.hpp:38-47) over one document or query text.
// Writes up to cap ids; returns the id count.
size_t ref_tokenize(void* vocab, int build, int lowercase, int stop, int stem, const char* text, size_t n,
                    uint32_t* ids, size_t cap) {
  auto* v = static_cast<sparselex::Vocabulary*>(vocab);
  const auto cfg = make_cfg(lowercase, stop, stem);
  const std::string_view t(text, n);
  const std::vector<uint32_t> r = build ? sparselex::tokenize_build(t, cfg, *v) : sparselex::tokenize_query(t, cfg, *v);
  if (ids && r.size() <= cap) std::memcpy(ids, r.data(), r.size() * 4);
  return r.size();
}

// A whole corpus (doc byte offsets[n_docs+1]) through tokenize_build with one vocabulary:
// ids[] and per-doc id offsets (tok_off[n_docs+1]); returns the total id count (ids written
// only when it fits cap).
uint64_t ref_tokenize_corpus(void* vocab, int lowercase, int stop, int stem, const char* text,
                             const uint64_t* doc_off, uint32_t n_docs, uint32_t* ids, uint64_t cap,
                             uint64_t* tok_off) {
  auto* v = static_cast<sparselex::Vocabulary*>(vocab);
  const auto cfg = make_cfg(lowercase, stop, stem);
  uint64_t total = 0;
  if (tok_off) tok_off[0] = 0;
  for (uint32_t d = 0; d < n_docs; ++d) {
    const std::vector<uint32_t> r =
        sparselex::tokenize_build(std::string_view(text + doc_off[d], doc_off[d + 1] - doc_off[d]), cfg, *v);
    if (ids && total + r.size() <= cap) std::memcpy(ids + total, r.data(), r.size() * 4);
    total += r.size();
    if (tok_off) tok_off[d + 1] = total;
  }
  return total;
}
}
