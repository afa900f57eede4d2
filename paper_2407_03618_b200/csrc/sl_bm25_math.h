// sl_bm25_math.h — the BM25 scoring math of proj/src/scoring.cpp:60-145, written ONCE for both
// sides of the library:
//   * the device (index build, sl_build.cu k_token_stats / k_values) instantiates it with
//     DevOps: every operation explicitly rounded (__dadd_rn, ...), so nvcc cannot contract a
//     multiply-add into an FMA the reference's C++ never performs;
//   * the host boundary functions of include/sparselex/bm25.hpp (sl_bm25.cpp, g++ with
//     -ffp-contract=off) instantiate it with HostOps and glibc's log — bit-identical to the
//     reference's compiled scoring.cpp (tests/test_bm25_abi.py).
// The expression trees follow the reference's C++ operator precedence exactly; preconditions
// (df range, tf >= 0, tfldp domains) are checked by the callers.
#pragma once

#include <cmath>

#if defined(__CUDACC__)
#define SL_MATH_HD __host__ __device__ __forceinline__
#else
#define SL_MATH_HD inline
#endif

namespace sl {
namespace bm25 {

// variant numbering of bm25.hpp:16-23 / sl_variant
enum : int { kRobertson = 0, kAtire = 1, kLucene = 2, kBm25l = 3, kBm25plus = 4, kTfldp = 5 };

struct HostOps {
  static inline double add(double a, double b) { return a + b; }
  static inline double sub(double a, double b) { return a - b; }
  static inline double mul(double a, double b) { return a * b; }
  static inline double div(double a, double b) { return a / b; }
  static inline double ln(double a) { return std::log(a); }
};

#if defined(__CUDACC__)
struct DevOps {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double ln(double a) { return ::log(a); }
};
#endif

SL_MATH_HD bool sparse(int v) { return v == kRobertson || v == kAtire || v == kLucene; }

// scoring.cpp:60-79 for 1 <= df <= N (n = N, d = df as doubles)
template <class O>
SL_MATH_HD double idf(int v, double n, double d) {
  switch (v) {
    case kLucene:  // ln(1 + (n - d + 0.5) / (d + 0.5))
      return O::ln(O::add(1.0, O::div(O::add(O::sub(n, d), 0.5), O::add(d, 0.5))));
    case kRobertson:  // ln((n - d + 0.5) / (d + 0.5))
      return O::ln(O::div(O::add(O::sub(n, d), 0.5), O::add(d, 0.5)));
    case kAtire:  // ln(n / d)
      return O::ln(O::div(n, d));
    case kBm25l:  // ln((n + 1) / (d + 0.5))
      return O::ln(O::div(O::add(n, 1.0), O::add(d, 0.5)));
    default:  // bm25plus, tfldp: ln((n + 1) / d)
      return O::ln(O::div(O::add(n, 1.0), d));
  }
}

// the length normalisation of scoring.cpp:86: (1 - b) + ((b * dl) / avg)
template <class O>
SL_MATH_HD double norm(double dl, double avg, double b) {
  return O::add(O::sub(1.0, b), O::div(O::mul(b, dl), avg));
}

// scoring.cpp:81-114 given norm (tfldp's domain is checked by the caller)
template <class O>
SL_MATH_HD double tf_component(int v, double tf, double nrm, double k1, double delta) {
  switch (v) {
    case kLucene:  // tf / (tf + k1 * norm)
      return O::div(tf, O::add(tf, O::mul(k1, nrm)));
    case kRobertson:
    case kAtire:  // ((k1 + 1) * tf) / (tf + k1 * norm)
      return O::div(O::mul(O::add(k1, 1.0), tf), O::add(tf, O::mul(k1, nrm)));
    case kBm25l: {  // c = tf / norm; ((k1 + 1) * (c + delta)) / ((k1 + c) + delta)
      const double c = O::div(tf, nrm);
      return O::div(O::mul(O::add(k1, 1.0), O::add(c, delta)), O::add(O::add(k1, c), delta));
    }
    case kBm25plus: {  // ((k1 + 1) * c) / (k1 + c) + delta
      const double c = O::div(tf, nrm);
      return O::add(O::div(O::mul(O::add(k1, 1.0), c), O::add(k1, c)), delta);
    }
    default: {  // tfldp: 1 + ln(1 + ln(c + delta))
      const double c = O::div(tf, nrm);
      return O::add(1.0, O::ln(O::add(1.0, O::ln(O::add(c, delta)))));
    }
  }
}

// scoring.cpp:125-145 given the idf (0 for the sparse variants)
template <class O>
SL_MATH_HD double nonoccurrence(int v, double i, double k1, double delta) {
  switch (v) {
    case kBm25l:  // (i * ((k1 + 1) * delta)) / (k1 + delta)
      return O::div(O::mul(i, O::mul(O::add(k1, 1.0), delta)), O::add(k1, delta));
    case kBm25plus:  // i * delta
      return O::mul(i, delta);
    case kTfldp:  // i * (1 + ln(1 + ln(delta)))
      return O::mul(i, O::add(1.0, O::ln(O::add(1.0, O::ln(delta)))));
    default:
      return 0.0;
  }
}

}  // namespace bm25
}  // namespace sl
