// sl_bm25.cpp — host side of the scoring boundary: the functions declared by
// include/sparselex/bm25.hpp (the reference's proj/include/sparselex/bm25.hpp:25-72, same
// signatures and exported C++ symbols) and their C-ABI twins in include/sparselex_b200.h.
// Behaviour follows proj/src/scoring.cpp:8-145 (argument checks and std::invalid_argument
// messages); the arithmetic is sl_bm25_math.h with HostOps, i.e. the expression trees the GPU
// build evaluates per nonzero. Compiled by g++ with -ffp-contract=off (no FMA contraction).
#include <cmath>
#include <stdexcept>
#include <string>

#include "sl_bm25_math.h"
#include "sl_internal_host.h"
#include "sparselex/bm25.hpp"
#include "sparselex_b200.h"

namespace sparselex {
namespace {
constexpr const char* kNames[] = {"robertson", "atire", "lucene", "bm25l", "bm25plus", "tfldp"};

int vi(Variant v) {
  const int i = static_cast<int>(v);
  if (i < 0 || i > 5) throw std::invalid_argument("invalid Variant value");
  return i;
}
}  // namespace

Variant variant_from_string(std::string_view name) {
  for (int i = 0; i < 6; ++i)
    if (name == kNames[i]) return static_cast<Variant>(i);
  throw std::invalid_argument("unknown BM25 variant: " + std::string(name));
}

std::string_view to_string(Variant v) { return kNames[vi(v)]; }

bool is_sparse_variant(Variant v) { return sl::bm25::sparse(static_cast<int>(v)); }

double BM25Params::default_delta(Variant v) {
  switch (v) {
    case Variant::bm25l: return 0.5;
    case Variant::bm25plus: return 1.0;
    case Variant::tfldp: return 0.5;
    default: return 0.0;
  }
}

BM25Params BM25Params::for_variant(Variant v, double k1, double b) { return BM25Params{v, k1, b, default_delta(v)}; }

void BM25Params::validate() const {
  if (!(k1 > 0.0)) throw std::invalid_argument("BM25Params: k1 must be > 0");
  if (!(b >= 0.0 && b <= 1.0)) throw std::invalid_argument("BM25Params: b must be in [0, 1]");
  if (!(delta >= 0.0)) throw std::invalid_argument("BM25Params: delta must be >= 0");
  if (variant == Variant::tfldp && !(delta > std::exp(-1.0)))
    throw std::invalid_argument("BM25Params: tfldp requires delta > exp(-1)");
}

double idf(Variant v, uint32_t df, uint32_t num_docs) {
  if (df == 0 || df > num_docs) throw std::invalid_argument("idf: df must satisfy 1 <= df <= num_docs");
  return sl::bm25::idf<sl::bm25::HostOps>(vi(v), static_cast<double>(num_docs), static_cast<double>(df));
}

double tf_component(double tf, double doc_len, const CorpusStats& stats, const BM25Params& params) {
  if (tf < 0.0) throw std::invalid_argument("tf_component: tf must be >= 0");
  if (!(stats.avg_len > 0.0)) throw std::invalid_argument("tf_component: avg_len must be > 0");
  using O = sl::bm25::HostOps;
  const int v = vi(params.variant);
  const double nrm = sl::bm25::norm<O>(doc_len, stats.avg_len, params.b);
  if (v == sl::bm25::kTfldp) {  // the two logarithms' domains (scoring.cpp:104-110)
    const double c = tf / nrm;
    if (c + params.delta <= 0.0) throw std::invalid_argument("tf_component: tfldp needs c + delta > 0");
    if (1.0 + std::log(c + params.delta) <= 0.0)
      throw std::invalid_argument("tf_component: tfldp needs 1 + ln(c + delta) > 0");
  }
  return sl::bm25::tf_component<O>(v, tf, nrm, params.k1, params.delta);
}

double score(double tf, uint32_t df, double doc_len, const CorpusStats& stats, const BM25Params& params) {
  if (tf == 0.0 && is_sparse_variant(params.variant)) return 0.0;
  return idf(params.variant, df, stats.num_docs) * tf_component(tf, doc_len, stats, params);
}

double nonoccurrence_score(uint32_t df, uint32_t num_docs, const BM25Params& params) {
  if (is_sparse_variant(params.variant)) return 0.0;
  const double i = idf(params.variant, df, num_docs);
  if (params.variant == Variant::tfldp && 1.0 + std::log(params.delta) <= 0.0)
    throw std::invalid_argument("nonoccurrence_score: tfldp needs delta > exp(-1)");
  return sl::bm25::nonoccurrence<sl::bm25::HostOps>(vi(params.variant), i, params.k1, params.delta);
}

}  // namespace sparselex

// ---------------------------------------------------------------- C-ABI twins
namespace {
template <class F>
int32_t guarded(F&& f) {
  try {
    f();
    return SL_OK;
  } catch (const std::invalid_argument& e) {
    sl::set_error(e.what());
    return SL_EINVAL;
  } catch (const std::exception& e) {
    sl::set_error(e.what());
    return SL_EUNSUPPORTED;
  }
}

sparselex::BM25Params cxx(const sl_params* p) {
  if (!p) throw std::invalid_argument("null params");
  if (p->variant < 0 || p->variant > 5) throw std::invalid_argument("invalid Variant value");
  return sparselex::BM25Params{static_cast<sparselex::Variant>(p->variant), p->k1, p->b, p->delta};
}
}  // namespace

extern "C" {

int32_t sl_params_validate(const sl_params* p) {
  return guarded([&] { cxx(p).validate(); });
}

double sl_default_delta(int32_t variant) {
  if (variant < 0 || variant > 5) return 0.0;
  return sparselex::BM25Params::default_delta(static_cast<sparselex::Variant>(variant));
}

int32_t sl_variant_from_string(const char* name, int32_t* out) {
  return guarded([&] {
    if (!name || !out) throw std::invalid_argument("sl_variant_from_string: null argument");
    *out = static_cast<int32_t>(sparselex::variant_from_string(name));
  });
}

const char* sl_variant_to_string(int32_t variant) {
  if (variant < 0 || variant > 5) {
    sl::set_error("invalid Variant value");
    return nullptr;
  }
  return sparselex::to_string(static_cast<sparselex::Variant>(variant)).data();
}

int32_t sl_is_sparse_variant(int32_t variant) { return sl::bm25::sparse(variant) ? 1 : 0; }

int32_t sl_idf(int32_t variant, uint32_t df, uint32_t num_docs, double* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("sl_idf: null output");
    if (variant < 0 || variant > 5) throw std::invalid_argument("invalid Variant value");
    *out = sparselex::idf(static_cast<sparselex::Variant>(variant), df, num_docs);
  });
}

int32_t sl_tf_component(double tf, double doc_len, uint32_t num_docs, double avg_len, const sl_params* p,
                        double* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("sl_tf_component: null output");
    sparselex::CorpusStats st;
    st.num_docs = num_docs;
    st.avg_len = avg_len;
    *out = sparselex::tf_component(tf, doc_len, st, cxx(p));
  });
}

int32_t sl_score(double tf, uint32_t df, double doc_len, uint32_t num_docs, double avg_len, const sl_params* p,
                 double* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("sl_score: null output");
    sparselex::CorpusStats st;
    st.num_docs = num_docs;
    st.avg_len = avg_len;
    *out = sparselex::score(tf, df, doc_len, st, cxx(p));
  });
}

int32_t sl_nonoccurrence_score(uint32_t df, uint32_t num_docs, const sl_params* p, double* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("sl_nonoccurrence_score: null output");
    *out = sparselex::nonoccurrence_score(df, num_docs, cxx(p));
  });
}

}  // extern "C"
