// ref_shim.cpp — extern "C" entry points over the REFERENCE's own scoring code.
//
// Compiled by oracle/Makefile together with /root/reference/proj/src/scoring.cpp
// (read in place, never copied) into oracle/_ref/libref_scoring.so. Test
// infrastructure only: tests/test_oracle.py::test_restatement_pinned_to_reference_scoring calls these to pin the oracle's
// restated formulas against the reference implementation itself.
// Declarations come from the reference header proj/include/sparselex/bm25.hpp:25-72.
#include <cmath>
#include <stdexcept>
#include <string>

#include "sparselex/bm25.hpp"

using sparselex::BM25Params;
using sparselex::CorpusStats;
using sparselex::Variant;

namespace {
thread_local std::string g_err;
BM25Params mk(int v, double k1, double b, double delta) {
  return BM25Params{static_cast<Variant>(v), k1, b, delta};
}
template <class F>
double guard(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return NAN;
  }
}
}  // namespace

extern "C" {
const char* ref_last_error(void) { return g_err.c_str(); }

double ref_idf(int v, unsigned df, unsigned n) {
  return guard([&] { return sparselex::idf(static_cast<Variant>(v), df, n); });
}
double ref_tf_component(double tf, double dl, double avg, int v, double k1, double b, double delta) {
  return guard([&] {
    CorpusStats st;
    st.avg_len = avg;
    return sparselex::tf_component(tf, dl, st, mk(v, k1, b, delta));
  });
}
double ref_score(double tf, unsigned df, double dl, unsigned n, double avg, int v, double k1, double b,
                 double delta) {
  return guard([&] {
    CorpusStats st;
    st.num_docs = n;
    st.avg_len = avg;
    return sparselex::score(tf, df, dl, st, mk(v, k1, b, delta));
  });
}
double ref_nonoccurrence(unsigned df, unsigned n, int v, double k1, double b, double delta) {
  return guard([&] { return sparselex::nonoccurrence_score(df, n, mk(v, k1, b, delta)); });
}
int ref_validate(int v, double k1, double b, double delta) {
  try {
    mk(v, k1, b, delta).validate();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
double ref_default_delta(int v) { return BM25Params::default_delta(static_cast<Variant>(v)); }
int ref_is_sparse(int v) { return sparselex::is_sparse_variant(static_cast<Variant>(v)) ? 1 : 0; }
}
