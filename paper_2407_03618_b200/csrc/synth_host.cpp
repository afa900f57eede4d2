// synth_host.cpp — host side of the seeded synthetic workload generator (libsl_synth.so).
//
// Restates BASELINE.json's five configs as generators (SURVEY.md §8d "Generator
// decisions"): Zipf rank r -> token id r-1, Philox4x32-10 uniforms keyed by
// (seed, stream, index), doc lengths on the host only (Poisson by inversion,
// lognormal by Box-Muller with libm), queries of distinct tokens, and the c5
// "5% head tail" (all tokens uniform over the top-64 ranks). Corpus seed 1000+i,
// query seed 2000+i for config ci.
//
// Pure C++/libm, no CUDA: tests and the CPU oracle use it on machines without a GPU;
// the device generator (sl_synth_dev.cu) reproduces sl_synth_tokens bit-exactly.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "sl_synth.h"

extern "C" {

typedef struct {
  uint32_t num_docs;
  uint32_t vocab;
  double zipf_s;
  int len_kind;      // 0 = Poisson(len_a), 1 = lognormal(median len_a, sigma len_b)
  double len_a, len_b;
  uint32_t len_min, len_max;
  uint32_t n_queries, qlen_min, qlen_max;
  double head_frac;  // fraction of head-heavy queries (c5)
  uint32_t head_ranks;
  uint32_t corpus_seed, query_seed;
} sl_synth_config;

// BASELINE.json "configs" (1-based: c1..c5). c3 reuses c2's shapes.
int sl_synth_config_get(int i, sl_synth_config* c) {
  if (!c) return 1;
  std::memset(c, 0, sizeof(*c));
  c->corpus_seed = 1000u + (uint32_t)i;
  c->query_seed = 2000u + (uint32_t)i;
  c->head_ranks = 64;
  switch (i) {
    case 1:
      c->num_docs = 10000; c->vocab = 5000; c->zipf_s = 1.1;
      c->len_kind = 0; c->len_a = 50.0; c->len_min = 1; c->len_max = 0xFFFFFFFFu;
      c->n_queries = 1000; c->qlen_min = 3; c->qlen_max = 8;
      return 0;
    case 2:
    case 3:
      c->num_docs = 1000000; c->vocab = 200000; c->zipf_s = 1.07;
      c->len_kind = 1; c->len_a = 60.0; c->len_b = 0.8; c->len_min = 1; c->len_max = 2000;
      c->n_queries = 10000; c->qlen_min = 2; c->qlen_max = 12;
      return 0;
    case 4:
      c->num_docs = 8800000; c->vocab = 1000000; c->zipf_s = 1.05;
      c->len_kind = 0; c->len_a = 56.0; c->len_min = 0; c->len_max = 0xFFFFFFFFu;
      c->n_queries = 8192; c->qlen_min = 3; c->qlen_max = 10;
      return 0;
    case 5:
      c->num_docs = 50000000; c->vocab = 4000000; c->zipf_s = 1.0;
      c->len_kind = 1; c->len_a = 200.0; c->len_b = 1.0; c->len_min = 1; c->len_max = 20000;
      c->n_queries = 65536; c->qlen_min = 2; c->qlen_max = 32;
      c->head_frac = 0.05;
      return 0;
    default:
      return 1;
  }
}

// cdf[r] = sum_{j<=r} (j+1)^-s / sum_{j<V} (j+1)^-s, serial f64 prefix sum; cdf[V-1] = 1.
int sl_synth_zipf_cdf(uint32_t V, double s, double* cdf) {
  if (V == 0 || !cdf) return 1;
  double acc = 0.0;
  for (uint32_t r = 0; r < V; ++r) {
    acc += std::pow((double)(r + 1), -s);
    cdf[r] = acc;
  }
  const double total = acc;
  for (uint32_t r = 0; r < V; ++r) cdf[r] /= total;
  cdf[V - 1] = 1.0;
  return 0;
}

static uint32_t doc_len(const sl_synth_config* c, uint32_t d) {
  double len;
  if (c->len_kind == 0) {
    // Poisson by inversion (sequential search of the CDF).
    const double u = sl_uniform(c->corpus_seed, SL_STREAM_DOCLEN, d);
    const double lam = c->len_a;
    double p = std::exp(-lam), F = p;
    uint32_t k = 0;
    const uint32_t kmax = (uint32_t)(10.0 * lam + 1000.0);
    while (u > F && k < kmax) {
      ++k;
      p *= lam / (double)k;
      F += p;
    }
    len = (double)k;
  } else {
    double u1, u2;
    sl_uniform2(c->corpus_seed, SL_STREAM_DOCLEN, d, &u1, &u2);
    const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
    len = std::floor(std::exp(std::log(c->len_a) + c->len_b * z) + 0.5);
  }
  if (len < (double)c->len_min) len = (double)c->len_min;
  if (len > (double)c->len_max) len = (double)c->len_max;
  return (uint32_t)len;
}

// Doc offsets for docs [d_begin, d_begin+n): offsets[0] = base, offsets[j+1] = offsets[j] + len.
int sl_synth_doc_offsets(const sl_synth_config* c, uint32_t d_begin, uint32_t n, uint64_t base,
                         uint64_t* offsets) {
  if (!c || !offsets) return 1;
  offsets[0] = base;
  for (uint32_t j = 0; j < n; ++j) offsets[j + 1] = offsets[j] + doc_len(c, d_begin + j);
  return 0;
}

// Tokens at global positions [begin, begin+count).
int sl_synth_tokens(const double* cdf, uint32_t V, uint32_t seed, uint64_t begin, uint64_t count,
                    uint32_t* out, int threads) {
  if (!cdf || !out || V == 0) return 1;
  if (threads < 1) threads = 1;
  if (count < 65536) threads = 1;
  std::vector<std::thread> pool;
  const uint64_t chunk = (count + (uint64_t)threads - 1) / (uint64_t)threads;
  for (int t = 0; t < threads; ++t) {
    const uint64_t lo = (uint64_t)t * chunk;
    const uint64_t hi = lo + chunk < count ? lo + chunk : count;
    if (lo >= hi) break;
    pool.emplace_back([=] {
      for (uint64_t i = lo; i < hi; ++i) out[i] = sl_corpus_token(cdf, V, seed, begin + i);
    });
  }
  for (auto& th : pool) th.join();
  return 0;
}

// Queries [q_begin, q_begin+nq): distinct tokens, length U{qlen_min..qlen_max}.
// q_offsets[0] = 0 (relative); q_tokens needs room for nq*qlen_max ids.
int sl_synth_queries(const sl_synth_config* c, const double* cdf, uint32_t q_begin, uint32_t nq,
                     uint64_t* q_offsets, uint32_t* q_tokens) {
  if (!c || !cdf || !q_offsets || !q_tokens) return 1;
  uint64_t pos = 0;
  q_offsets[0] = 0;
  const uint32_t span = c->qlen_max - c->qlen_min + 1;
  for (uint32_t j = 0; j < nq; ++j) {
    const uint32_t q = q_begin + j;
    uint32_t len = c->qlen_min +
                   (uint32_t)(sl_uniform(c->query_seed, SL_STREAM_QLEN, q) * (double)span);
    if (len > c->qlen_max) len = c->qlen_max;
    if (len > c->vocab) len = c->vocab;
    const bool head = c->head_frac > 0.0 &&
                      sl_uniform(c->query_seed, SL_STREAM_QHEAD, q) < c->head_frac;
    const uint32_t hr = c->head_ranks < c->vocab ? c->head_ranks : c->vocab;
    if (head && len > hr) len = hr;
    uint32_t got = 0;
    for (uint64_t a = 0; got < len && a < 65536; ++a) {
      const double u = sl_uniform(c->query_seed, SL_STREAM_QTOK, (uint64_t)q * 65536u + a);
      const uint32_t tok = head ? (uint32_t)(u * (double)hr) : sl_zipf_lookup(cdf, c->vocab, u);
      bool dup = false;
      for (uint32_t x = 0; x < got; ++x) dup |= (q_tokens[pos + x] == tok);
      if (!dup) q_tokens[pos + got++] = tok;
    }
    pos += got;
    q_offsets[j + 1] = pos;
  }
  return 0;
}

// Renders token-id documents as text (the text-pipeline workload): token t -> words[t]
// (word_off[n_words+1] into `words`), each followed by a separator drawn with Philox
// (seed, SL_STREAM_TEXT, global token position); 10% of words start with a capital.
// out == NULL: only out_doc_off[N+1] (byte offsets) is filled; call again with a buffer of
// out_doc_off[N] bytes.
static const char* kSeps[] = {" ", ", ", ". ", "\n", "; ", " (", ") ", " - ", "! "};
static const double kSepCdf[] = {0.80, 0.86, 0.90, 0.93, 0.95, 0.97, 0.98, 0.99, 1.01};

static inline int pick_sep(double u) {
  int k = 0;
  while (u >= kSepCdf[k]) ++k;
  return k;
}

int sl_synth_render_text(const uint32_t* tokens, const uint64_t* doc_off, uint32_t N, const char* words,
                         const uint64_t* word_off, uint32_t n_words, uint32_t seed, char* out,
                         uint64_t* out_doc_off, int threads) {
  if (!tokens || !doc_off || !words || !word_off || !out_doc_off) return 1;
  if (threads < 1) threads = 1;
  std::vector<uint64_t> sz(N, 0);
  auto run = [&](auto&& body) {
    std::vector<std::thread> pool;
    const uint32_t chunk = (N + (uint32_t)threads - 1) / (uint32_t)threads;
    for (int t = 0; t < threads; ++t) {
      const uint32_t lo = (uint32_t)t * chunk, hi = lo + chunk < N ? lo + chunk : N;
      if (lo >= hi) break;
      pool.emplace_back([=, &body] {
        for (uint32_t d = lo; d < hi; ++d) body(d);
      });
    }
    for (auto& th : pool) th.join();
  };
  if (!out) {
    int bad = 0;
    run([&](uint32_t d) {
      uint64_t n = 0;
      for (uint64_t i = doc_off[d]; i < doc_off[d + 1]; ++i) {
        const uint32_t t = tokens[i];
        if (t >= n_words) {
          bad = 1;
          continue;
        }
        double u0, u1;
        sl_uniform2(seed, SL_STREAM_TEXT, i, &u0, &u1);
        n += (word_off[t + 1] - word_off[t]) + std::strlen(kSeps[pick_sep(u0)]);
      }
      sz[d] = n;
    });
    out_doc_off[0] = 0;
    for (uint32_t d = 0; d < N; ++d) out_doc_off[d + 1] = out_doc_off[d] + sz[d];
    return bad;
  }
  run([&](uint32_t d) {
    char* o = out + out_doc_off[d];
    for (uint64_t i = doc_off[d]; i < doc_off[d + 1]; ++i) {
      const uint32_t t = tokens[i];
      if (t >= n_words) continue;
      double u0, u1;
      sl_uniform2(seed, SL_STREAM_TEXT, i, &u0, &u1);
      const uint64_t wl = word_off[t + 1] - word_off[t];
      std::memcpy(o, words + word_off[t], wl);
      if (u1 < 0.1 && o[0] >= 'a' && o[0] <= 'z') o[0] = (char)(o[0] - 32);
      o += wl;
      const char* s = kSeps[pick_sep(u0)];
      const size_t sl = std::strlen(s);
      std::memcpy(o, s, sl);
      o += sl;
    }
  });
  return 0;
}

}  // extern "C"
