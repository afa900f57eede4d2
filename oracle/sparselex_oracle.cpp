// sparselex_oracle.cpp — CPU ORACLE (test infrastructure only; never on the product path).
//
// A plain C++ restatement of the reference's eager sparse-scoring path for
// token-id input, used by tests/ as the parity checker and by bench.py's
// cpu_baseline / --impl reference legs as the timed CPU implementation.
// Only tests/, __graft_entry__.smoke() and bench.py may load it.
//
// What it follows (paths relative to the reference root):
//   scoring   proj/src/scoring.cpp:60-145  (idf, tf_component, score,
//             nonoccurrence_score) — restated below expression-for-expression
//             and pinned against the reference's own scoring.cpp, compiled by
//             oracle/Makefile into oracle/_ref/libref_scoring.so
//             (tests/test_oracle.py::test_restatement_pinned_to_reference_scoring);
//   counting  proj/src/tokenizer.cpp:162-168 (count_terms: tf per id,
//             length = #ids) and proj/include/sparselex/vocabulary.hpp:37-42 (DF);
//   index     SPEC.md [MODULE] index: two-pass build_index (pass 1 DF + lengths,
//             L_avg = sum|D|/N, pass 2 S^Δ = S - S^θ in f64 narrowed to f32 into
//             preallocated token-major slices with strictly increasing doc ids;
//             theta = S^θ as f32; structural zeros kept; empty docs kept);
//   retrieval SPEC.md [MODULE] retrieval: score_query (f64 dense accumulator,
//             repeated tokens count per repetition, + Σ S^θ constant), top_k
//             (introselect via std::nth_element, then sort; ties -> smaller doc
//             index), retrieve_batch (worker pool, identical results for any
//             worker count).
// Pinned decisions: tokens with df = 0 (never occur in the
// synthetic corpus) get an empty row and theta = 0 and are dropped at query time,
// the SPEC's OOV rule (SPEC.md tokenizer DESIGN DECISIONS).
// Parity against the upstream Python BM25S package is unpinned (not present);
// parity against SPEC.md + scoring.cpp is pinned by tests/golden + the _ref build.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

enum Variant { ROBERTSON = 0, ATIRE = 1, LUCENE = 2, BM25L = 3, BM25PLUS = 4, TFLDP = 5 };

thread_local std::string g_err;

struct Params {
  int variant;
  double k1, b, delta;
};

bool is_sparse(int v) { return v == ROBERTSON || v == ATIRE || v == LUCENE; }  // scoring.cpp:30-32

// scoring.cpp:47-58
void validate(const Params& p) {
  if (p.variant < 0 || p.variant > 5) throw std::invalid_argument("invalid Variant value");
  if (!(p.k1 > 0.0)) throw std::invalid_argument("BM25Params: k1 must be > 0");
  if (!(p.b >= 0.0 && p.b <= 1.0)) throw std::invalid_argument("BM25Params: b must be in [0, 1]");
  if (!(p.delta >= 0.0)) throw std::invalid_argument("BM25Params: delta must be >= 0");
  if (p.variant == TFLDP && !(p.delta > std::exp(-1.0)))
    throw std::invalid_argument("BM25Params: tfldp requires delta > exp(-1)");
}

// scoring.cpp:60-79
double idf(int v, uint32_t df, uint32_t num_docs) {
  if (df == 0 || df > num_docs) throw std::invalid_argument("idf: df must satisfy 1 <= df <= num_docs");
  const double n = (double)num_docs;
  const double d = (double)df;
  switch (v) {
    case LUCENE: return std::log(1.0 + (n - d + 0.5) / (d + 0.5));
    case ROBERTSON: return std::log((n - d + 0.5) / (d + 0.5));
    case ATIRE: return std::log(n / d);
    case BM25L: return std::log((n + 1.0) / (d + 0.5));
    case BM25PLUS:
    case TFLDP: return std::log((n + 1.0) / d);
  }
  throw std::invalid_argument("invalid Variant value");
}

// scoring.cpp:81-114
double tf_component(double tf, double doc_len, double avg_len, const Params& p) {
  if (tf < 0.0) throw std::invalid_argument("tf_component: tf must be >= 0");
  if (!(avg_len > 0.0)) throw std::invalid_argument("tf_component: avg_len must be > 0");
  const double norm = 1.0 - p.b + p.b * doc_len / avg_len;
  switch (p.variant) {
    case LUCENE: return tf / (tf + p.k1 * norm);
    case ROBERTSON:
    case ATIRE: return ((p.k1 + 1.0) * tf) / (tf + p.k1 * norm);
    case BM25L: {
      const double c = tf / norm;
      return ((p.k1 + 1.0) * (c + p.delta)) / (p.k1 + c + p.delta);
    }
    case BM25PLUS: {
      const double c = tf / norm;
      return ((p.k1 + 1.0) * c) / (p.k1 + c) + p.delta;
    }
    case TFLDP: {
      const double c = tf / norm;
      if (c + p.delta <= 0.0) throw std::invalid_argument("tf_component: tfldp needs c + delta > 0");
      const double inner = 1.0 + std::log(c + p.delta);
      if (inner <= 0.0) throw std::invalid_argument("tf_component: tfldp needs 1 + ln(c + delta) > 0");
      return 1.0 + std::log(inner);
    }
  }
  throw std::invalid_argument("invalid Variant value");
}

// scoring.cpp:116-123
double score(double tf, uint32_t df, double doc_len, uint32_t num_docs, double avg_len, const Params& p) {
  if (tf == 0.0 && is_sparse(p.variant)) return 0.0;
  return idf(p.variant, df, num_docs) * tf_component(tf, doc_len, avg_len, p);
}

// scoring.cpp:125-145
double nonoccurrence(uint32_t df, uint32_t num_docs, const Params& p) {
  if (is_sparse(p.variant)) return 0.0;
  const double i = idf(p.variant, df, num_docs);
  switch (p.variant) {
    case BM25L: return i * ((p.k1 + 1.0) * p.delta) / (p.k1 + p.delta);
    case BM25PLUS: return i * p.delta;
    case TFLDP: {
      const double inner = 1.0 + std::log(p.delta);
      if (inner <= 0.0) throw std::invalid_argument("nonoccurrence_score: tfldp needs delta > exp(-1)");
      return i * (1.0 + std::log(inner));
    }
    default: return 0.0;
  }
}

struct OracleIndex {
  Params p;
  uint32_t N = 0, V = 0;
  double avg_len = 0.0;
  uint64_t total_len = 0;
  std::vector<uint64_t> indptr;   // u64[V+1]   (SPEC index External Interfaces: indptr.bin)
  std::vector<uint32_t> docids;   // u32[nnz]
  std::vector<float> values;      // f32[nnz]  S^Δ
  std::vector<uint32_t> tf;       // u32[nnz]  (debug export for the bit-exact TF check)
  std::vector<uint32_t> df;       // u32[V]
  std::vector<float> theta;       // f32[V]
  std::vector<uint32_t> doclens;  // u32[N]
};

// count_terms (tokenizer.cpp:162-168) restated as sort + run-length: same
// multiset semantics, distinct ids emitted ascending.
void count_terms(const uint32_t* ids, uint64_t n, std::vector<uint32_t>& scratch,
                 std::vector<std::pair<uint32_t, uint32_t>>& out) {
  scratch.assign(ids, ids + n);
  std::sort(scratch.begin(), scratch.end());
  out.clear();
  for (uint64_t i = 0; i < n;) {
    uint64_t j = i + 1;
    while (j < n && scratch[j] == scratch[i]) ++j;
    out.emplace_back(scratch[i], (uint32_t)(j - i));
    i = j;
  }
}

// gdf/gN/gtotal: optional global statistics of a document-sharded corpus;
// with them, idf, S^θ and L_avg are those of the whole corpus while rows hold this shard's docs.
OracleIndex* build(const uint64_t* offsets, const uint32_t* tokens, uint32_t N, uint32_t V, const Params& p,
                   const uint32_t* gdf = nullptr, uint32_t gN = 0, uint64_t gtotal = 0) {
  validate(p);
  if (N == 0) throw std::invalid_argument("build_index: empty corpus");
  if (V == 0) throw std::invalid_argument("build_index: empty vocabulary");
  auto* ix = new OracleIndex();
  ix->p = p;
  ix->N = N;
  ix->V = V;
  ix->df.assign(V, 0);
  ix->doclens.assign(N, 0);
  std::vector<uint32_t> scratch;
  std::vector<std::pair<uint32_t, uint32_t>> counts;
  // pass 1: DF + lengths (SPEC index DESIGN DECISIONS "Build is two-pass")
  uint64_t total = 0;
  for (uint32_t d = 0; d < N; ++d) {
    const uint64_t b = offsets[d], e = offsets[d + 1];
    if (e < b) { delete ix; throw std::invalid_argument("build_index: doc offsets must be non-decreasing"); }
    for (uint64_t i = b; i < e; ++i)
      if (tokens[i] >= V) { delete ix; throw std::invalid_argument("build_index: token id >= vocab size"); }
    count_terms(tokens + b, e - b, scratch, counts);
    for (auto& c : counts) ++ix->df[c.first];  // vocabulary.hpp:38 bump_doc_frequency
    ix->doclens[d] = (uint32_t)(e - b);         // tokenizer.cpp:166 length = ids.size()
    total += e - b;
  }
  if (total == 0) { delete ix; throw std::invalid_argument("build_index: degenerate corpus (all documents empty)"); }
  std::vector<uint32_t> local_df = ix->df;
  uint32_t Ns = N;
  if (gdf) {
    for (uint32_t t = 0; t < V; ++t) ix->df[t] = gdf[t];
    total = gtotal;
    Ns = gN;
  }
  ix->total_len = total;
  ix->avg_len = (double)total / (double)Ns;  // SPEC scoring CorpusStats: L_avg
  ix->indptr.assign((size_t)V + 1, 0);
  for (uint32_t t = 0; t < V; ++t) ix->indptr[t + 1] = ix->indptr[t] + local_df[t];
  const uint64_t nnz = ix->indptr[V];
  ix->docids.resize(nnz);
  ix->values.resize(nnz);
  ix->tf.resize(nnz);
  ix->theta.assign(V, 0.0f);
  std::vector<double> theta64(V, 0.0);
  for (uint32_t t = 0; t < V; ++t)
    if (ix->df[t] > 0) {
      theta64[t] = nonoccurrence(ix->df[t], Ns, p);
      ix->theta[t] = (float)theta64[t];
    }
  // pass 2: S^Δ = S - S^θ in f64, stored f32, docs ascending => strictly increasing per row
  std::vector<uint64_t> cursor(ix->indptr.begin(), ix->indptr.end() - 1);
  for (uint32_t d = 0; d < N; ++d) {
    const uint64_t b = offsets[d], e = offsets[d + 1];
    count_terms(tokens + b, e - b, scratch, counts);
    const double dl = (double)ix->doclens[d];
    for (auto& c : counts) {
      const uint32_t t = c.first;
      const uint64_t pos = cursor[t]++;
      ix->docids[pos] = d;
      ix->tf[pos] = c.second;
      const double s = score((double)c.second, ix->df[t], dl, Ns, ix->avg_len, p);
      ix->values[pos] = (float)(s - theta64[t]);
    }
  }
  return ix;
}

// SPEC retrieval score_query: result[D] = Σ S^Δ(q_i,D) + Σ S^θ(q_i), f64 accumulator.
void score_query(const OracleIndex& ix, const uint32_t* q, uint32_t qlen, double* acc) {
  std::fill(acc, acc + ix.N, 0.0);
  double constant = 0.0;
  for (uint32_t j = 0; j < qlen; ++j) {
    const uint32_t t = q[j];
    if (t >= ix.V) throw std::invalid_argument("score_query: token id >= vocab size");
    if (ix.df[t] == 0) continue;  // OOV drop
    for (uint64_t i = ix.indptr[t]; i < ix.indptr[t + 1]; ++i) acc[ix.docids[i]] += (double)ix.values[i];
    constant += (double)ix.theta[t];
  }
  if (constant != 0.0)
    for (uint32_t d = 0; d < ix.N; ++d) acc[d] += constant;
}

// SPEC retrieval top_k: introselect (std::nth_element) + O(k log k) sort,
// ties broken by smaller document index.
uint32_t top_k(const double* s, uint32_t n, uint32_t k, int ordered, std::vector<uint32_t>& idx,
               uint32_t* out_ids, double* out_scores) {
  if (k == 0) throw std::invalid_argument("top_k: k must be >= 1");
  idx.resize(n);
  for (uint32_t i = 0; i < n; ++i) idx[i] = i;
  auto better = [s](uint32_t a, uint32_t b) { return s[a] > s[b] || (s[a] == s[b] && a < b); };
  const uint32_t m = k < n ? k : n;
  if (m < n) std::nth_element(idx.begin(), idx.begin() + m, idx.end(), better);
  if (ordered) std::sort(idx.begin(), idx.begin() + m, better);
  for (uint32_t i = 0; i < m; ++i) {
    out_ids[i] = idx[i];
    if (out_scores) out_scores[i] = s[idx[i]];
  }
  return m;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

template <class F>
void for_doc_ranges(uint32_t N, int threads, F&& f) {
  threads = std::max(1, threads);
  std::vector<std::thread> th;
  for (int t = 0; t < threads; ++t) {
    const uint32_t a = (uint32_t)((uint64_t)N * t / threads), b = (uint32_t)((uint64_t)N * (t + 1) / threads);
    th.emplace_back([&f, t, a, b] { f(t, a, b); });
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

typedef struct OracleIndex orc_index;

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_build(const uint64_t* offsets, const uint32_t* tokens, uint32_t N, uint32_t V, int variant,
              double k1, double b, double delta, orc_index** out) {
  return guarded([&] { *out = build(offsets, tokens, N, V, Params{variant, k1, b, delta}); });
}

// One shard of a document-sharded corpus built with the corpus-wide df / N / Σ|D|.
int orc_build_shard(const uint64_t* offsets, const uint32_t* tokens, uint32_t N, uint32_t V, int variant, double k1,
                    double b, double delta, const uint32_t* global_df, uint32_t global_n, uint64_t global_total,
                    orc_index** out) {
  return guarded([&] {
    *out = build(offsets, tokens, N, V, Params{variant, k1, b, delta}, global_df, global_n, global_total);
  });
}

void orc_free(orc_index* ix) { delete ix; }

uint64_t orc_nnz(const orc_index* ix) { return ix->indptr.back(); }
double orc_avg_len(const orc_index* ix) { return ix->avg_len; }
uint64_t orc_total_len(const orc_index* ix) { return ix->total_len; }

void orc_export(const orc_index* ix, uint64_t* indptr, uint32_t* docids, float* values, uint32_t* df,
                float* theta, uint32_t* doclens, uint32_t* tf) {
  const size_t nnz = ix->docids.size();
  if (indptr) std::memcpy(indptr, ix->indptr.data(), ix->indptr.size() * 8);
  if (docids) std::memcpy(docids, ix->docids.data(), nnz * 4);
  if (values) std::memcpy(values, ix->values.data(), nnz * 4);
  if (tf) std::memcpy(tf, ix->tf.data(), nnz * 4);
  if (df) std::memcpy(df, ix->df.data(), (size_t)ix->V * 4);
  if (theta) std::memcpy(theta, ix->theta.data(), (size_t)ix->V * 4);
  if (doclens) std::memcpy(doclens, ix->doclens.data(), (size_t)ix->N * 4);
}

int orc_score_query(const orc_index* ix, const uint32_t* q, uint32_t qlen, double* out) {
  return guarded([&] { score_query(*ix, q, qlen, out); });
}

// returns the number of results (min(k, n)) or -1 on error
int64_t orc_top_k(const double* scores, uint32_t n, uint32_t k, int ordered, uint32_t* ids, double* out) {
  int64_t m = -1;
  std::vector<uint32_t> idx;
  if (guarded([&] { m = top_k(scores, n, k, ordered, idx, ids, out); })) return -1;
  return m;
}

// SPEC retrieve_batch over token-id queries. Output B*k, padded with
// id 0xFFFFFFFF / score -inf where k > N.
int orc_retrieve_batch(const orc_index* ix, const uint64_t* q_offsets, const uint32_t* q_tokens, uint32_t B,
                       uint32_t k, int ordered, int workers, uint32_t* out_ids, double* out_scores) {
  return guarded([&] {
    if (k == 0) throw std::invalid_argument("top_k: k must be >= 1");
    if (workers < 1) throw std::invalid_argument("retrieve_batch: workers must be >= 1");
    std::atomic<uint32_t> next{0};
    std::vector<std::string> errs(workers);
    auto work = [&](int w) {
      std::vector<double> acc(ix->N);  // per-worker accumulator (SPEC retrieval DESIGN DECISIONS)
      std::vector<uint32_t> idx;
      try {
        for (uint32_t q; (q = next.fetch_add(1)) < B;) {
          const uint64_t b = q_offsets[q], e = q_offsets[q + 1];
          score_query(*ix, q_tokens + b, (uint32_t)(e - b), acc.data());
          uint32_t* ids = out_ids + (uint64_t)q * k;
          double* sc = out_scores + (uint64_t)q * k;
          const uint32_t m = top_k(acc.data(), ix->N, k, ordered, idx, ids, sc);
          for (uint32_t i = m; i < k; ++i) {
            ids[i] = 0xFFFFFFFFu;
            sc[i] = -INFINITY;
          }
        }
      } catch (const std::exception& ex) {
        errs[w] = ex.what();
        next.store(B);
      }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < workers; ++w) pool.emplace_back(work, w);
    work(0);
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::invalid_argument(e);
  });
}

// Naive dense scorer (SPEC ACCEPTANCE CRITERIA 1/6): B(Q,D) = Σ_i S(q_i, D) computed
// directly from raw tf/df/lengths per document, no shifting, no index.
int orc_dense_score(const uint64_t* offsets, const uint32_t* tokens, uint32_t N, uint32_t V, int variant,
                    double k1, double b, double delta, const uint32_t* q, uint32_t qlen, double* out) {
  return guarded([&] {
    const Params p{variant, k1, b, delta};
    validate(p);
    std::vector<uint32_t> df(V, 0), scratch;
    std::vector<std::pair<uint32_t, uint32_t>> counts;
    uint64_t total = 0;
    for (uint32_t d = 0; d < N; ++d) {
      count_terms(tokens + offsets[d], offsets[d + 1] - offsets[d], scratch, counts);
      for (auto& c : counts) ++df[c.first];
      total += offsets[d + 1] - offsets[d];
    }
    const double avg = (double)total / (double)N;
    for (uint32_t d = 0; d < N; ++d) {
      const uint64_t bo = offsets[d], eo = offsets[d + 1];
      double s = 0.0;
      for (uint32_t j = 0; j < qlen; ++j) {
        const uint32_t t = q[j];
        if (t >= V || df[t] == 0) continue;  // OOV drop
        uint32_t tf = 0;
        for (uint64_t i = bo; i < eo; ++i) tf += tokens[i] == t;
        s += score((double)tf, df[t], (double)(eo - bo), N, avg, p);
      }
      out[d] = s;
    }
  });
}

// Restated scoring primitives, exported for the pin against the reference's own
// scoring.cpp (oracle/_ref) and the SPEC golden values. NaN + error on contract violation.
double orc_idf(int v, uint32_t df, uint32_t N) {
  double r = NAN;
  guarded([&] { r = idf(v, df, N); });
  return r;
}
double orc_tf_component(double tf, double dl, double avg, int v, double k1, double b, double delta) {
  double r = NAN;
  guarded([&] { r = tf_component(tf, dl, avg, Params{v, k1, b, delta}); });
  return r;
}
double orc_score(double tf, uint32_t df, double dl, uint32_t N, double avg, int v, double k1, double b,
                 double delta) {
  double r = NAN;
  guarded([&] { r = score(tf, df, dl, N, avg, Params{v, k1, b, delta}); });
  return r;
}
double orc_nonoccurrence(uint32_t df, uint32_t N, int v, double k1, double b, double delta) {
  double r = NAN;
  guarded([&] { r = nonoccurrence(df, N, Params{v, k1, b, delta}); });
  return r;
}
int orc_validate(int v, double k1, double b, double delta) {
  return guarded([&] { validate(Params{v, k1, b, delta}); });
}


// ---- streaming checks for corpora too large to index on the CPU (c5: 1.65e10 tokens) ----
// Each runs over one shard's tokens in `threads` contiguous document ranges and keeps only
// what the check needs, so host memory stays at one shard's tokens.


// DF by streaming count (vocabulary.hpp:37-42 semantics: one bump per distinct id per
// document), ADDED into df_out[V]; *total_len_out += Σ|D|.
int orc_stream_df(const uint64_t* offsets, const uint32_t* tokens, uint32_t N, uint32_t V, int threads,
                  uint64_t* df_out, uint64_t* total_len_out) {
  return guarded([&] {
    threads = std::max(1, threads);
    std::vector<std::vector<uint32_t>> local(threads);
    std::vector<uint64_t> tot(threads, 0);
    std::atomic<int> bad{0};
    for_doc_ranges(N, threads, [&](int t, uint32_t a, uint32_t b) {
      auto& df = local[t];
      df.assign(V, 0);
      std::vector<uint32_t> scratch;
      std::vector<std::pair<uint32_t, uint32_t>> counts;
      for (uint32_t d = a; d < b; ++d) {
        const uint64_t o = offsets[d], e = offsets[d + 1];
        for (uint64_t i = o; i < e; ++i)
          if (tokens[i] >= V) bad = 1;
        if (bad) return;
        count_terms(tokens + o, e - o, scratch, counts);
        for (auto& c : counts) ++df[c.first];
        tot[t] += e - o;
      }
    });
    if (bad) throw std::invalid_argument("stream_df: token id >= vocab size");
    for (int t = 0; t < threads; ++t) {
      for (uint32_t v = 0; v < V; ++v) df_out[v] += local[t][v];
      *total_len_out += tot[t];
    }
  });
}

// Selected rows of a shard's score matrix by streaming: for the nsel tokens in sel, the
// documents containing them (ascending, local ids), their tf and the stored value
// f32(S - S^θ) computed with the GLOBAL statistics (gdf, gN, avg) exactly as pass 2 of
// build() does. row_off[nsel+1] is always written; docs/tfs/values (may be null) are
// filled in row order when given (sized row_off[nsel]).
int orc_stream_rows(const uint64_t* offsets, const uint32_t* tokens, uint32_t N, uint32_t V, const uint32_t* sel,
                    uint32_t nsel, const uint32_t* gdf, uint32_t gN, double avg, int variant, double k1, double b,
                    double delta, int threads, uint64_t* row_off, uint32_t* docs, uint32_t* tfs, float* values) {
  return guarded([&] {
    const Params p{variant, k1, b, delta};
    validate(p);
    threads = std::max(1, threads);
    std::vector<int32_t> slot(V, -1);
    for (uint32_t i = 0; i < nsel; ++i) {
      if (sel[i] >= V) throw std::invalid_argument("stream_rows: selected token >= vocab size");
      slot[sel[i]] = (int32_t)i;
    }
    auto doc_counts = [&](uint32_t d, std::vector<uint32_t>& scratch, std::vector<std::pair<uint32_t, uint32_t>>& out) {
      scratch.clear();
      for (uint64_t i = offsets[d]; i < offsets[d + 1]; ++i)
        if (slot[tokens[i]] >= 0) scratch.push_back(tokens[i]);
      std::sort(scratch.begin(), scratch.end());
      out.clear();
      for (size_t i = 0; i < scratch.size();) {
        size_t j = i + 1;
        while (j < scratch.size() && scratch[j] == scratch[i]) ++j;
        out.emplace_back(scratch[i], (uint32_t)(j - i));
        i = j;
      }
    };
    std::vector<std::vector<uint64_t>> cnt(threads, std::vector<uint64_t>(nsel, 0));
    for_doc_ranges(N, threads, [&](int t, uint32_t a, uint32_t bb) {
      std::vector<uint32_t> scratch;
      std::vector<std::pair<uint32_t, uint32_t>> c;
      for (uint32_t d = a; d < bb; ++d) {
        doc_counts(d, scratch, c);
        for (auto& x : c) ++cnt[t][slot[x.first]];
      }
    });
    row_off[0] = 0;
    for (uint32_t i = 0; i < nsel; ++i) {
      uint64_t s = 0;
      for (int t = 0; t < threads; ++t) s += cnt[t][i];
      row_off[i + 1] = row_off[i] + s;
    }
    if (!docs) return;
    // per-thread write cursors: rows in doc order = thread order
    std::vector<std::vector<uint64_t>> cur(threads, std::vector<uint64_t>(nsel));
    for (uint32_t i = 0; i < nsel; ++i) {
      uint64_t c = row_off[i];
      for (int t = 0; t < threads; ++t) {
        cur[t][i] = c;
        c += cnt[t][i];
      }
    }
    std::vector<double> theta64(nsel, 0.0);
    for (uint32_t i = 0; i < nsel; ++i)
      if (gdf[sel[i]]) theta64[i] = nonoccurrence(gdf[sel[i]], gN, p);
    for_doc_ranges(N, threads, [&](int t, uint32_t a, uint32_t bb) {
      std::vector<uint32_t> scratch;
      std::vector<std::pair<uint32_t, uint32_t>> c;
      for (uint32_t d = a; d < bb; ++d) {
        doc_counts(d, scratch, c);
        const double dl = (double)(offsets[d + 1] - offsets[d]);
        for (auto& x : c) {
          const int32_t i = slot[x.first];
          const uint64_t pos = cur[t][i]++;
          docs[pos] = d;
          if (tfs) tfs[pos] = x.second;
          if (values) {
            const double sc = score((double)x.second, gdf[x.first], dl, gN, avg, p);
            values[pos] = (float)(sc - theta64[i]);
          }
        }
      }
    });
  });
}

// Streaming naive dense scorer (SPEC.md [MODULE] retrieval property "naive dense scorer",
// AC1/AC6): for each query, B(Q,D) = Σ_i S(q_i, D) from raw tf / global df / |D| for every
// document of the shard (query tokens in query order, repeats counted), and the best k by
// (score desc, doc asc) over the shard. Documents containing none of a query's tokens all
// score Σ_i S(q_i, tf=0) (length-independent); of those only the k smallest ids can place.
// Outputs [B x k]: global doc ids (doc_base + local), f64 scores; unused slots id 0xFFFFFFFF.
int orc_stream_topk(const uint64_t* offsets, const uint32_t* tokens, uint32_t N, uint32_t doc_base, uint32_t V,
                    const uint64_t* q_off, const uint32_t* q_tok, uint32_t B, const uint32_t* gdf, uint32_t gN,
                    double avg, int variant, double k1, double b, double delta, uint32_t k, int threads,
                    uint32_t* out_ids, double* out_scores) {
  return guarded([&] {
    const Params p{variant, k1, b, delta};
    validate(p);
    if (k == 0) throw std::invalid_argument("top_k: k must be >= 1");
    threads = std::max(1, threads);
    // compact ids of the distinct query tokens with df > 0 (OOV drop)
    std::vector<int32_t> cid(V, -1);
    std::vector<uint32_t> utok;
    std::vector<std::vector<int32_t>> qc(B);
    for (uint32_t q = 0; q < B; ++q)
      for (uint64_t j = q_off[q]; j < q_off[q + 1]; ++j) {
        const uint32_t t = q_tok[j];
        if (t >= V) throw std::invalid_argument("score_query: token id >= vocab size");
        if (gdf[t] == 0) continue;
        if (cid[t] < 0) {
          cid[t] = (int32_t)utok.size();
          utok.push_back(t);
        }
        qc[q].push_back(cid[t]);
      }
    const uint32_t U = (uint32_t)utok.size();
    std::vector<double> s0(U);
    for (uint32_t u = 0; u < U; ++u) s0[u] = score(0.0, gdf[utok[u]], 1.0, gN, avg, p);
    std::vector<double> base(B, 0.0);
    for (uint32_t q = 0; q < B; ++q)
      for (int32_t c : qc[q]) base[q] += s0[c];
    using Cand = std::pair<double, uint32_t>;  // (score, global doc)
    auto better = [](const Cand& x, const Cand& y) { return x.first > y.first || (x.first == y.first && x.second < y.second); };
    std::vector<std::vector<std::vector<Cand>>> heaps(threads, std::vector<std::vector<Cand>>(B));
    std::vector<std::vector<std::vector<uint32_t>>> untouched(threads, std::vector<std::vector<uint32_t>>(B));
    for_doc_ranges(N, threads, [&](int t, uint32_t a, uint32_t bb) {
      std::vector<uint32_t> tfc(U, 0), touched;
      std::vector<double> val(U);
      for (uint32_t d = a; d < bb; ++d) {
        touched.clear();
        for (uint64_t i = offsets[d]; i < offsets[d + 1]; ++i) {
          const int32_t c = cid[tokens[i]];
          if (c >= 0 && tfc[c]++ == 0) touched.push_back((uint32_t)c);
        }
        const double dl = (double)(offsets[d + 1] - offsets[d]);
        for (uint32_t c : touched) val[c] = score((double)tfc[c], gdf[utok[c]], dl, gN, avg, p);
        const uint32_t g = doc_base + d;
        for (uint32_t q = 0; q < B; ++q) {
          bool hit = false;
          double s = 0.0;
          for (int32_t c : qc[q]) {
            if (tfc[c]) {
              hit = true;
              s += val[c];
            } else {
              s += s0[c];
            }
          }
          if (!hit) {
            if (untouched[t][q].size() < k) untouched[t][q].push_back(g);
            continue;
          }
          auto& h = heaps[t][q];  // min-heap on `better` of the best k
          const Cand cd{s, g};
          if (h.size() < k) {
            h.push_back(cd);
            std::push_heap(h.begin(), h.end(), better);
          } else if (better(cd, h.front())) {
            std::pop_heap(h.begin(), h.end(), better);
            h.back() = cd;
            std::push_heap(h.begin(), h.end(), better);
          }
        }
        for (uint32_t c : touched) tfc[c] = 0;
      }
    });
    for (uint32_t q = 0; q < B; ++q) {
      std::vector<Cand> all;
      std::vector<uint32_t> un;
      for (int t = 0; t < threads; ++t) {
        all.insert(all.end(), heaps[t][q].begin(), heaps[t][q].end());
        un.insert(un.end(), untouched[t][q].begin(), untouched[t][q].end());  // thread order = doc order
      }
      for (uint32_t i = 0; i < un.size() && i < k; ++i) all.emplace_back(base[q], un[i]);
      std::sort(all.begin(), all.end(), better);
      for (uint32_t i = 0; i < k; ++i) {
        out_ids[(uint64_t)q * k + i] = i < all.size() ? all[i].second : 0xFFFFFFFFu;
        out_scores[(uint64_t)q * k + i] = i < all.size() ? all[i].first : -INFINITY;
      }
    }
  });
}

}  // extern "C"
