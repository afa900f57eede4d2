/* sl_synth.h — seeded synthetic-corpus primitives shared bit-exactly by host and device.
 *
 * BASELINE.json configs name no dataset files (the paper's BEIR sets are not in the
 * container), so every corpus and query set is generated from these
 * primitives with the seeds pinned in BASELINE.md §5:
 *   - Philox4x32-10 keyed by (seed, stream) with a 64-bit counter = element index;
 *   - u64 -> double in [0,1) by taking the top 53 bits (exact on host and device);
 *   - Zipf(s) over ranks 1..V by inverse CDF: the token id is the smallest r with
 *     u < cdf[r], cdf built on the host in f64 (serial prefix sum of (r+1)^-s) and
 *     shipped to the device unchanged, so the comparison chain is identical.
 * Doc lengths use libm (Poisson inversion, lognormal Box-Muller) and are host-only.
 *
 * Not on the product hot path: this is input generation for bench.py and tests.
 */
#ifndef SL_SYNTH_H
#define SL_SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SL_HD __host__ __device__ __forceinline__
#else
#define SL_HD static inline
#endif

/* stream ids (pinned) */
#define SL_STREAM_DOCLEN 1u
#define SL_STREAM_TOKEN 2u
#define SL_STREAM_QLEN 3u
#define SL_STREAM_QTOK 4u
#define SL_STREAM_QHEAD 5u
#define SL_STREAM_TEXT 6u

SL_HD void sl_mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  *lo = (uint32_t)p;
}

/* Philox4x32-10 (Salmon et al. 2011). out[0..3] for counter (idx_lo, idx_hi, 0, 0). */
SL_HD void sl_philox4x32(uint32_t seed, uint32_t stream, uint64_t idx, uint32_t out[4]) {
  uint32_t c0 = (uint32_t)idx, c1 = (uint32_t)(idx >> 32), c2 = 0u, c3 = 0u;
  uint32_t k0 = seed, k1 = stream;
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    sl_mulhilo32(0xD2511F53u, c0, &hi0, &lo0);
    sl_mulhilo32(0xCD9E8D57u, c2, &hi1, &lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

SL_HD double sl_u01_from_u64(uint64_t x) {
  return (double)(x >> 11) * (1.0 / 9007199254740992.0); /* 2^-53 */
}

/* Two independent uniforms in [0,1) from one Philox draw. */
SL_HD void sl_uniform2(uint32_t seed, uint32_t stream, uint64_t idx, double* u0, double* u1) {
  uint32_t o[4];
  sl_philox4x32(seed, stream, idx, o);
  *u0 = sl_u01_from_u64(((uint64_t)o[1] << 32) | o[0]);
  *u1 = sl_u01_from_u64(((uint64_t)o[3] << 32) | o[2]);
}

SL_HD double sl_uniform(uint32_t seed, uint32_t stream, uint64_t idx) {
  double a, b;
  sl_uniform2(seed, stream, idx, &a, &b);
  return a;
}

/* smallest r in [0, V) with u < cdf[r]; cdf[V-1] == 1.0 and u < 1 so it exists. */
SL_HD uint32_t sl_zipf_lookup(const double* cdf, uint32_t V, double u) {
  uint32_t lo = 0, hi = V - 1;
  while (lo < hi) {
    uint32_t mid = lo + ((hi - lo) >> 1);
    if (u < cdf[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

/* token at global corpus position i */
SL_HD uint32_t sl_corpus_token(const double* cdf, uint32_t V, uint32_t seed, uint64_t i) {
  return sl_zipf_lookup(cdf, V, sl_uniform(seed, SL_STREAM_TOKEN, i));
}

#endif /* SL_SYNTH_H */
