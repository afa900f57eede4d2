// bm25_caller.cpp — a caller of the reference's scoring interface (<sparselex/bm25.hpp>), written
// the way reference code uses it, exposed as extern "C" for tests/test_bm25_abi.py. The test
// compiles this ONE source twice against the SAME header — once linked with the reference's own
// proj/src/scoring.cpp, once linked with libsparselex_b200.so — and requires bit-identical
// results and identical error messages: reference code links against this library unchanged.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "sparselex/bm25.hpp"

using namespace sparselex;

namespace {
thread_local std::string g_msg;
BM25Params mk(int v, double k1, double b, double d) { return BM25Params{static_cast<Variant>(v), k1, b, d}; }
template <class F>
int run(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_msg = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {
const char* caller_msg() { return g_msg.c_str(); }
int caller_from_string(const char* name, int* out) {
  return run([&] { *out = static_cast<int>(variant_from_string(name)); });
}
int caller_to_string(int v, char* buf, int cap) {
  return run([&] {
    const std::string_view s = to_string(static_cast<Variant>(v));
    std::snprintf(buf, cap, "%.*s", (int)s.size(), s.data());
  });
}
int caller_is_sparse(int v) { return is_sparse_variant(static_cast<Variant>(v)) ? 1 : 0; }
double caller_default_delta(int v) { return BM25Params::default_delta(static_cast<Variant>(v)); }
int caller_for_variant(int v, double k1, double b, double* out4) {
  return run([&] {
    const BM25Params p = BM25Params::for_variant(static_cast<Variant>(v), k1, b);
    out4[0] = static_cast<double>(static_cast<int>(p.variant));
    out4[1] = p.k1;
    out4[2] = p.b;
    out4[3] = p.delta;
  });
}
int caller_validate(int v, double k1, double b, double d) { return run([&] { mk(v, k1, b, d).validate(); }); }
int caller_idf(int v, unsigned df, unsigned n, double* out) {
  return run([&] { *out = idf(static_cast<Variant>(v), df, n); });
}
int caller_tf_component(double tf, double dl, double avg, int v, double k1, double b, double d, double* out) {
  return run([&] {
    CorpusStats st;
    st.avg_len = avg;
    *out = tf_component(tf, dl, st, mk(v, k1, b, d));
  });
}
int caller_score(double tf, unsigned df, double dl, unsigned n, double avg, int v, double k1, double b, double d,
                 double* out) {
  return run([&] {
    CorpusStats st;
    st.num_docs = n;
    st.avg_len = avg;
    st.doc_lengths = {1u, 2u, 3u};  // the struct's vector member crosses the boundary too
    *out = score(tf, df, dl, st, mk(v, k1, b, d));
  });
}
int caller_nonoccurrence(unsigned df, unsigned n, int v, double k1, double b, double d, double* out) {
  return run([&] { *out = nonoccurrence_score(df, n, mk(v, k1, b, d)); });
}
}
