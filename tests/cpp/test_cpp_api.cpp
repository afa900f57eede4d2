// C++ SPEC-API smoke test through include/sparselex/b200.hpp (run by tests/test_gpu_cpp_api.py).
// Toy corpus of SPEC.md [MODULE] index: ["cat sat", "dog ran", "cat cat cat"], ids cat=0 sat=1
// dog=2 ran=3; expected values verified against the reference's scoring.cpp.
#include <cmath>
#include <cstdio>
#include <string>
#include <unistd.h>
#include <stdexcept>
#include <vector>

#include "sparselex/b200.hpp"

using namespace sparselex::b200;

#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                     \
    }                                                               \
  } while (0)

int main() {
  const std::vector<uint64_t> off = {0, 2, 4, 7};
  const std::vector<uint32_t> tok = {0, 1, 2, 3, 0, 0, 0};
  TokenCorpus corpus{off, tok, 4};
  SearchIndex ix = build_index(corpus, BM25Params{});
  EXPECT(ix.num_docs() == 3);
  EXPECT(std::fabs(ix.avg_len() - 7.0 / 3.0) < 1e-15);
  auto a = ix.export_arrays();
  EXPECT(a.indptr == (std::vector<uint64_t>{0, 2, 3, 4, 5}));
  EXPECT(a.docids == (std::vector<uint32_t>{0, 2, 0, 1, 1}));
  EXPECT(a.values[0] == 0.200917587f && a.values[1] == 0.292446703f);

  const std::vector<uint32_t> q = {0};
  auto s = score_query(ix, q);
  EXPECT(s.size() == 3 && s[1] == 0.f && s[2] == 0.292446703f);
  auto r = retrieve(ix, q, 2);
  EXPECT(r.doc_indices == (std::vector<uint32_t>{2, 0}));
  auto all = retrieve_batch(ix, {{0}, {}, {3, 1}}, 5, true, 4);
  EXPECT(all.size() == 3 && all[0].doc_indices.size() == 3);
  EXPECT(all[1].doc_indices == (std::vector<uint32_t>{0, 1, 2}));  // empty query: ties -> smaller id
  auto t = top_k(std::vector<float>{0.1f, 0.9f, 0.3f, 0.7f}, 2);
  EXPECT(t.doc_indices == (std::vector<uint32_t>{1, 3}));  // SPEC top_k example

  bool threw = false;
  try {
    build_index(corpus, BM25Params{Variant::tfldp, 1.5, 0.75, 0.2});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    retrieve(ix, std::vector<uint32_t>{7}, 1);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  auto bp = BM25Params::for_variant(Variant::bm25plus);
  EXPECT(bp.delta == 1.0);
  SearchIndex ixp = build_index(corpus, bp);
  auto ap = ixp.export_arrays();
  EXPECT(ap.theta[0] == 0.693147181f && ap.values[0] == 0.740767956f);
  // text side: SPEC.md:65-67 and the SPEC toy corpus built from text
  {
    TokenizerConfig tc{true, {"the", "is"}, StemmerKind::snowball_english};
    Vocabulary v;
    auto tk = tokenize_build({"the cat is running", "cat cat"}, tc, v);
    auto toks = v.tokens();
    EXPECT(toks == (std::vector<std::string>{"cat", "run"}));
    EXPECT(tk.doc(0) == (std::vector<uint32_t>{0, 1}) && tk.doc(1) == (std::vector<uint32_t>{0, 0}));
    EXPECT(tokenize_query({"zebra running"}, tc, v).doc(0) == (std::vector<uint32_t>{1}));
    {  // the streaming entry point on a pre-concatenated corpus gives the per-call result
      Vocabulary v2;
      const std::string all = "the cat is runningcat cat";
      auto ts = tokenize_stream(all, {0, 18, 25}, tc, v2, true, 8);
      EXPECT(v2.tokens() == toks && ts.doc(0) == tk.doc(0) && ts.doc(1) == tk.doc(1));
    }
    EXPECT(stem_english({"running", "skies", "generously"}) ==
           (std::vector<std::string>{"run", "sky", "generous"}));
    TextIndex ti = build_text_index({"cat sat", "dog ran", "cat cat cat"}, BM25Params{}, TokenizerConfig{});
    EXPECT(ti.vocab_tokens() == (std::vector<std::string>{"cat", "sat", "dog", "ran"}));
    auto rt = retrieve(ti, "Cat!", 2);
    EXPECT(rt.doc_indices == (std::vector<uint32_t>{2, 0}) && rt.scores[0] == 0.292446703f);
    EXPECT(rt.external_ids == (std::vector<std::string>{"2", "0"}));
  }
  // SPEC build_index over (external_id, text) pairs -> save -> load -> retrieve with external ids
  {
    const std::vector<std::pair<std::string, std::string>> corpus = {
        {"doc-a", "The cats sat on the mat"}, {"doc \"b\"", "Dogs ran; a dog runs."}, {"c/\u00e9", "cat cat cat"}};
    TokenizerConfig tc{true, {"the", "on", "a"}, StemmerKind::snowball_english};
    TextIndex t = build_text_index(corpus, BM25Params::for_variant(Variant::bm25plus), tc);
    EXPECT(t.num_docs() == 3 && t.doc_external_ids()[1] == "doc \"b\"");
    auto r1 = retrieve_batch(t, {"cat", "dogs running", "zebra"}, 2);
    EXPECT(r1.size() == 3 && r1[0].external_ids == (std::vector<std::string>{"c/\u00e9", "doc-a"}));
    EXPECT(r1[1].external_ids[0] == "doc \"b\"");
    const std::string dir = "/tmp/sl_cpp_text_index_" + std::to_string(::getpid());
    save_index(t, dir);
    TextIndex u = load_text_index(dir);
    EXPECT(u.doc_external_ids() == t.doc_external_ids() && u.vocab_tokens() == t.vocab_tokens());
    auto tcu = u.tokenizer_config();
    EXPECT(tcu.lowercase && tcu.stemmer == StemmerKind::snowball_english && tcu.stopwords.size() == 3);
    auto r2 = retrieve_batch(u, {"cat", "dogs running", "zebra"}, 2);
    for (size_t i = 0; i < r1.size(); ++i)
      EXPECT(r2[i].doc_indices == r1[i].doc_indices && r2[i].scores == r1[i].scores &&
             r2[i].external_ids == r1[i].external_ids);
    bool dup = false;
    try {
      build_text_index(std::vector<std::pair<std::string, std::string>>{{"x", "cat"}, {"x", "dog"}}, BM25Params{}, tc);
    } catch (const std::invalid_argument& e) {
      dup = std::string(e.what()).find("duplicate external ids") != std::string::npos;
    }
    EXPECT(dup);
    bool degenerate = false;
    try {
      build_text_index(std::vector<std::pair<std::string, std::string>>{{"x", "the"}, {"y", "! ?"}}, BM25Params{}, tc);
    } catch (const std::invalid_argument& e) {
      degenerate = std::string(e.what()).find("degenerate corpus") != std::string::npos;
    }
    EXPECT(degenerate);
  }
  // the reference's scoring functions are this library's too (bm25.hpp)
  {
    EXPECT(sparselex::variant_from_string("bm25l") == Variant::bm25l && sparselex::to_string(Variant::atire) == "atire");
    sparselex::CorpusStats st;
    st.num_docs = 3;
    st.avg_len = 7.0 / 3.0;
    EXPECT(static_cast<float>(sparselex::score(3.0, 2, 3.0, st, BM25Params{})) == 0.292446703f);
  }
  std::printf("cpp api ok\n");
  return 0;
}
