// sl_text.cu — the text side of the path on the device:
// UTF-8 split -> lowercase -> stopword filter -> Snowball English stem -> vocabulary ids.
//
// Reference semantics (paths relative to /root/reference):
//   split_text / for_each_token   proj/src/tokenizer.cpp:52-113  maximal runs of >= 2 word
//                                 codepoints; malformed UTF-8 byte -> U+FFFD (a separator)
//                                 consuming one byte; a sequence never crosses its document
//   word class / lowercase        proj/src/tokenizer.cpp:12-33  (tables: sl_unicode.inc)
//   run_pipeline                  proj/src/tokenizer.cpp:115-129 stopwords compared on the
//                                 lowercased, pre-stem token; stem; id
//   stem_english                  proj/src/stemmer.cpp:29-411    (the reference's variant)
//   Vocabulary                    proj/include/sparselex/vocabulary.hpp:13-48 ids in first-
//                                 encounter order (document order, then position)
//
// Device design (byte-parallel, HBM-streaming):
//   k_doc_marks     bitmap of document start bytes
//   k_classify      one thread per byte: decode start / covering sequence (looks at <= 3
//                   bytes either side), word class -> two bitmaps (word byte, word
//                   codepoint start) written by warp ballots (1/4 of the text in bytes)
//   k_tok_count/emit one thread per 32-byte bitmap word: token begins = word bytes whose
//                   predecessor is not a word byte (or a document start); end and codepoint
//                   count by bit scans; tokens of >= 2 codepoints kept, in byte order
//   k_norm          one thread per token: lowercase, stopword probe, stem (on a one-byte-
//                   per-codepoint shadow of the word: ASCII as itself, others as 0x80, so the
//                   rules see exactly what the reference's codepoint loop sees), two 64-bit
//                   hashes, vocabulary probe; normalised bytes to an arena (2x text)
//   build mode      new tokens sorted by hash (the build's radix sort), grouped, groups
//                   ordered by first occurrence -> ids appended to the vocabulary in the
//                   reference's first-encounter order; open-addressing device hash table
//   query mode      tokens absent from the frozen vocabulary are dropped (SPEC OOV rule)
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <string>
#include <vector>

#include "sl_index.cuh"

#define SL_UNI_QUAL __device__
#ifndef SL_TAIL_INLINE
#define SL_TAIL_INLINE __noinline__
#endif
namespace sl {
namespace uni {
#include "sl_unicode.inc"
}
}  // namespace sl

struct sl_vocab {
  int device = 0;
  uint32_t V = 0;
  uint32_t vcap = 0;         // capacity of offs (vcap + 1) / h2 / lens
  uint64_t* offs = nullptr;  // [V+1] byte offsets into bytes
  uint64_t* h2 = nullptr;    // [V] second hash (identity check)
  uint8_t* bytes = nullptr;
  uint64_t bcap = 0;
  uint64_t bused = 0;
  uint64_t* tkey = nullptr;  // [tcap] first hash (0 = empty)
  uint32_t* tval = nullptr;  // [tcap] id
  uint32_t tcap = 0;         // power of two
  int32_t weak = 0;          // test hook (SL_TEXT_WEAK_HASH=1): degenerate hashes exercise the collision paths
};

struct sl_token_batch {
  int device = 0;
  uint32_t N = 0;
  uint64_t T = 0;
  uint64_t* offs = nullptr;  // [N+1] token offsets per document
  uint32_t* ids = nullptr;   // [T]
};

namespace sl {
namespace {

constexpr uint32_t kNew = 0xFFFFFFFFu;
constexpr int kFastBytes = 64;  // tokens up to this many raw bytes normalise in registers/local memory

// ------------------------------------------------------------------ unicode
__device__ __forceinline__ bool is_word_cp(uint32_t c) {
  if (c < 0x80) return (c >= '0' && c <= '9') || (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_';
  int lo = 0, hi = uni::kSlWordRangeCount;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (uni::kSlWordRanges[2 * mid] <= c) lo = mid + 1; else hi = mid;
  }
  return lo > 0 && c <= uni::kSlWordRanges[2 * (lo - 1) + 1];
}

__device__ __forceinline__ uint32_t lower_cp(uint32_t c) {
  if (c < 0x80) return (c >= 'A' && c <= 'Z') ? c + 32 : c;
  int lo = 0, hi = uni::kSlLowerCount;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (uni::kSlLowerFrom[mid] < c) lo = mid + 1; else hi = mid;
  }
  return (lo < uni::kSlLowerCount && uni::kSlLowerFrom[lo] == c) ? uni::kSlLowerTo[lo] : c;
}

__device__ __forceinline__ int put_utf8(uint8_t* o, uint32_t c) {
  if (c < 0x80) {
    o[0] = (uint8_t)c;
    return 1;
  }
  if (c < 0x800) {
    o[0] = (uint8_t)(0xC0 | (c >> 6));
    o[1] = (uint8_t)(0x80 | (c & 0x3F));
    return 2;
  }
  if (c < 0x10000) {
    o[0] = (uint8_t)(0xE0 | (c >> 12));
    o[1] = (uint8_t)(0x80 | ((c >> 6) & 0x3F));
    o[2] = (uint8_t)(0x80 | (c & 0x3F));
    return 3;
  }
  o[0] = (uint8_t)(0xF0 | (c >> 18));
  o[1] = (uint8_t)(0x80 | ((c >> 12) & 0x3F));
  o[2] = (uint8_t)(0x80 | ((c >> 6) & 0x3F));
  o[3] = (uint8_t)(0x80 | (c & 0x3F));
  return 4;
}

__device__ __forceinline__ int lead_len(uint32_t b) {
  return (b >= 0xC0 && b <= 0xDF) ? 2 : (b >= 0xE0 && b <= 0xEF) ? 3 : (b >= 0xF0 && b <= 0xF7) ? 4 : 0;
}

// decode one codepoint of a known-good (or leniently accepted) sequence at p; returns length
__device__ __forceinline__ int decode_at(const uint8_t* s, uint32_t* cp) {
  const uint32_t b = s[0];
  if (b < 0x80) {
    *cp = b;
    return 1;
  }
  const int L = lead_len(b);
  uint32_t c = b & (L == 2 ? 0x1F : L == 3 ? 0x0F : 0x07);
  for (int i = 1; i < L; ++i) c = (c << 6) | (s[i] & 0x3F);
  *cp = c;
  return L;
}

// ------------------------------------------------------------------ hashing
__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}
__host__ __device__ inline uint64_t fnv1a64(const uint8_t* s, uint32_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint32_t i = 0; i < n; ++i) h = (h ^ s[i]) * 0x100000001b3ull;
  return h;
}
struct H2 {
  uint64_t a, b;
};
// two independent 64-bit hashes of one byte string; a is never 0 (0 = empty table slot)
__device__ __forceinline__ H2 hash2(const uint8_t* s, uint32_t n) {
  uint64_t a = 0xcbf29ce484222325ull, b = 0x9e3779b97f4a7c15ull ^ n;
  for (uint32_t i = 0; i < n; ++i) {
    a = (a ^ s[i]) * 0x100000001b3ull;
    b = (b + s[i] + 1) * 0xd6e8feb86659fd93ull;
    b ^= b >> 29;
  }
  a = fmix64(a ^ n);
  b = fmix64(b);
  return H2{a ? a : 1ull, b};
}

__device__ __forceinline__ ulonglong2 cas128(ulonglong2* p, ulonglong2 cmp, ulonglong2 val) {
  ulonglong2 old;
  asm volatile(
      "{\n\t.reg .b128 c, v, o;\n\t"
      "mov.b128 c, {%2, %3};\n\tmov.b128 v, {%4, %5};\n\t"
      "atom.global.cas.b128 o, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(old.x), "=l"(old.y)
      : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(p)
      : "memory");
  return old;
}

// ------------------------------------------------------------------ segmentation
struct TextView {
  const uint8_t* text;
  uint64_t n;
  const uint32_t* dstart;  // bitmap: document start bytes
};

__device__ __forceinline__ uint32_t byte_at(const TextView& t, int64_t p) {
  return (p >= 0 && (uint64_t)p < t.n) ? (uint32_t)__ldg(t.text + p) : 0u;
}
__device__ __forceinline__ bool dstart_at(const TextView& t, uint64_t p) {
  return p < t.n && ((__ldg(t.dstart + (p >> 5)) >> (p & 31)) & 1u);
}

// a valid UTF-8 sequence (tokenizer.cpp:52-94 rules) starts at q and stays in its document
__device__ bool valid_at(const TextView& t, uint64_t q, uint32_t* cp, int* len) {
  const uint32_t b = byte_at(t, (int64_t)q);
  const int L = lead_len(b);
  if (!L || q + L > t.n) return false;
  uint32_t c = b & (L == 2 ? 0x1F : L == 3 ? 0x0F : 0x07);
  for (int i = 1; i < L; ++i) {
    if (dstart_at(t, q + i)) return false;
    const uint32_t x = byte_at(t, (int64_t)(q + i));
    if ((x & 0xC0) != 0x80) return false;
    c = (c << 6) | (x & 0x3F);
  }
  const uint32_t lo = L == 2 ? 0x80u : L == 3 ? 0x800u : 0x10000u;
  if (c < lo || c > 0x10FFFF || (c >= 0xD800 && c <= 0xDFFF)) return false;
  *cp = c;
  *len = L;
  return true;
}

__global__ void k_doc_marks(const uint64_t* __restrict__ off, uint32_t N, uint64_t n, uint32_t* __restrict__ bits) {
  for (uint32_t d = blockIdx.x * blockDim.x + threadIdx.x; d < N; d += gridDim.x * blockDim.x) {
    const uint64_t b = off[d];
    if (b < off[d + 1] && b < n) atomicOr(bits + (b >> 5), 1u << (b & 31));
  }
}

// per byte: word-byte bit and word-codepoint-start bit
__global__ void k_classify(TextView t, uint32_t* __restrict__ wbits, uint32_t* __restrict__ sbits) {
  const uint64_t nw = (t.n + 31) >> 5;
  for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint64_t b = (w << 5) + (threadIdx.x & 31);
    bool word = false, start = false;
    if (b < t.n) {
      const uint32_t x = byte_at(t, (int64_t)b);
      uint32_t cp = 0;
      int L = 0;
      bool covered = false;
      if ((x & 0xC0) == 0x80) {  // continuation byte: inside the nearest preceding valid sequence?
        for (int back = 1; back <= 3 && (int64_t)b - back >= 0; ++back) {
          const uint64_t q = b - back;
          if (dstart_at(t, q + 1)) break;  // q is in an earlier document
          const uint32_t y = byte_at(t, (int64_t)q);
          if ((y & 0xC0) == 0x80) continue;
          if (valid_at(t, q, &cp, &L) && q + L > b) covered = true;
          break;
        }
      }
      if (!covered) {
        start = true;
        if (x < 0x80) cp = x;
        else if (!valid_at(t, b, &cp, &L)) cp = 0xFFFD;
      }
      word = is_word_cp(cp);
    }
    const uint32_t wm = __ballot_sync(0xffffffffu, word);
    const uint32_t sm = __ballot_sync(0xffffffffu, word && start);
    if ((threadIdx.x & 31) == 0) {
      wbits[w] = wm;
      sbits[w] = sm;
    }
  }
}

// byte b's (word, codepoint-start) flags, the general path of k_classify
__device__ __forceinline__ void classify_byte(const TextView& t, uint64_t b, bool& word, bool& start) {
  const uint32_t x = byte_at(t, (int64_t)b);
  uint32_t cp = 0;
  int L = 0;
  bool covered = false;
  if ((x & 0xC0) == 0x80) {  // continuation byte: inside the nearest preceding valid sequence?
    for (int back = 1; back <= 3 && (int64_t)b - back >= 0; ++back) {
      const uint64_t q = b - back;
      if (dstart_at(t, q + 1)) break;  // q is in an earlier document
      const uint32_t y = byte_at(t, (int64_t)q);
      if ((y & 0xC0) == 0x80) continue;
      if (valid_at(t, q, &cp, &L) && q + L > b) covered = true;
      break;
    }
  }
  start = !covered;
  if (!covered) {
    if (x < 0x80) cp = x;
    else if (!valid_at(t, b, &cp, &L)) cp = 0xFFFD;
  }
  word = is_word_cp(cp);
}

// Four bytes per thread from one aligned 32-bit load: an all-ASCII group (the common case)
// classifies in registers; any other group takes classify_byte. Eight lanes' nibbles OR
// into one bitmap word. Requires a 4-byte-aligned text pointer.
__global__ void k_classify4(TextView t, uint32_t* __restrict__ wbits, uint32_t* __restrict__ sbits) {
  const uint64_t nq = (t.n + 3) >> 2;                 // 4-byte groups
  const uint64_t nq_pad = ((nq + 31) >> 5) << 5;      // whole warps iterate together
  const int lane = threadIdx.x & 31;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nq_pad; g += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t wn = 0, sn = 0;  // nibbles
    const uint64_t b0 = g << 2;
    if (b0 + 4 <= t.n) {
      const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(t.text) + g);
      if (!(v & 0x80808080u)) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t c = (v >> (8 * j)) & 0xFFu;
          const bool w = (c - '0' < 10u) || ((c | 0x20u) - 'a' < 26u) || c == '_';
          wn |= (uint32_t)w << j;
        }
        sn = wn;  // ASCII bytes are codepoint starts
      } else {
        for (int j = 0; j < 4; ++j) {
          bool w, st;
          classify_byte(t, b0 + j, w, st);
          wn |= (uint32_t)w << j;
          sn |= (uint32_t)(w && st) << j;
        }
      }
    } else if (b0 < t.n) {
      for (int j = 0; j < 4 && b0 + j < t.n; ++j) {
        bool w, st;
        classify_byte(t, b0 + j, w, st);
        wn |= (uint32_t)w << j;
        sn |= (uint32_t)(w && st) << j;
      }
    }
    uint32_t wv = wn << (4 * (lane & 7)), sv = sn << (4 * (lane & 7));
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      wv |= __shfl_xor_sync(0xffffffffu, wv, o);
      sv |= __shfl_xor_sync(0xffffffffu, sv, o);
    }
    const uint64_t word_idx = g >> 3;
    if ((lane & 7) == 0 && (word_idx << 5) < t.n) {
      wbits[word_idx] = wv;
      sbits[word_idx] = sv;
    }
  }
}

// word-byte mask of four ASCII bytes (SWAR: [0-9], letters after | 0x20, '_'); bit j = byte j
__device__ __forceinline__ uint32_t ascii_word_mask4(uint32_t v) {
  const uint32_t dg = (v + 0x50505050u) & ~(v + 0x46464646u);  // >= '0' and < ':'
  const uint32_t u = v | 0x20202020u;
  const uint32_t al = (u + 0x1F1F1F1Fu) & ~(u + 0x05050505u);  // >= 'a' and < '{'
  const uint32_t x = v ^ 0x5F5F5F5Fu;
  const uint32_t nz = ((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x;    // bit 7: byte != '_'
  const uint32_t w = (dg | al | ~nz) & 0x80808080u;
  return ((w >> 7) & 1u) | ((w >> 14) & 2u) | ((w >> 21) & 4u) | ((w >> 28) & 8u);
}

// 16 bytes per thread from one 16-byte load (text 16-byte aligned): all-ASCII groups classify
// with SWAR arithmetic; any other group takes classify_byte per byte. Two lanes form one
// 32-byte bitmap word (one shuffle each for the word and start bitmaps).
__global__ void k_classify16(TextView t, uint32_t* __restrict__ wbits, uint32_t* __restrict__ sbits) {
  const uint64_t ng = (t.n + 15) >> 4;
  const uint64_t ng_pad = ((ng + 31) >> 5) << 5;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ng_pad; g += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t wm = 0, sm = 0;
    const uint64_t b0 = g << 4;
    if (b0 + 16 <= t.n) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(t.text) + g);
      if (!((v.x | v.y | v.z | v.w) & 0x80808080u)) {
        wm = ascii_word_mask4(v.x) | (ascii_word_mask4(v.y) << 4) | (ascii_word_mask4(v.z) << 8) |
             (ascii_word_mask4(v.w) << 12);
        sm = wm;  // ASCII bytes are codepoint starts
      } else {
        for (int j = 0; j < 16; ++j) {
          bool w, st;
          classify_byte(t, b0 + j, w, st);
          wm |= (uint32_t)w << j;
          sm |= (uint32_t)(w && st) << j;
        }
      }
    } else if (b0 < t.n) {
      for (int j = 0; j < 16 && b0 + j < t.n; ++j) {
        bool w, st;
        classify_byte(t, b0 + j, w, st);
        wm |= (uint32_t)w << j;
        sm |= (uint32_t)(w && st) << j;
      }
    }
    const int sh = 16 * (int)(g & 1);
    uint32_t wv = wm << sh, sv = sm << sh;
    wv |= __shfl_xor_sync(0xffffffffu, wv, 1);
    sv |= __shfl_xor_sync(0xffffffffu, sv, 1);
    const uint64_t word_idx = g >> 1;
    if (!(g & 1) && (word_idx << 5) < t.n) {
      wbits[word_idx] = wv;
      sbits[word_idx] = sv;
    }
  }
}

// 32 bytes (one bitmap word) per thread from two 16-byte loads in flight together (text 16-byte
// aligned); all-ASCII halves classify with SWAR arithmetic, others per byte (classify_byte).
__device__ __forceinline__ void classify_half(const TextView& t, uint64_t b0, const uint4& v, uint32_t& wm,
                                              uint32_t& sm) {
  if (!((v.x | v.y | v.z | v.w) & 0x80808080u)) {
    wm = ascii_word_mask4(v.x) | (ascii_word_mask4(v.y) << 4) | (ascii_word_mask4(v.z) << 8) |
         (ascii_word_mask4(v.w) << 12);
    sm = wm;  // ASCII bytes are codepoint starts
  } else {
    wm = sm = 0;
    for (int j = 0; j < 16; ++j) {
      bool w, st;
      classify_byte(t, b0 + j, w, st);
      wm |= (uint32_t)w << j;
      sm |= (uint32_t)(w && st) << j;
    }
  }
}

__global__ void k_classify32(TextView t, uint32_t* __restrict__ wbits, uint32_t* __restrict__ sbits) {
  const uint64_t nw = (t.n + 31) >> 5;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b0 = w << 5;
    uint32_t wm0 = 0, sm0 = 0, wm1 = 0, sm1 = 0;
    if (b0 + 32 <= t.n) {
      const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(t.text) + 2 * w);
      const uint4 v1 = __ldg(reinterpret_cast<const uint4*>(t.text) + 2 * w + 1);
      classify_half(t, b0, v0, wm0, sm0);
      classify_half(t, b0 + 16, v1, wm1, sm1);
    } else {
      for (int j = 0; j < 32 && b0 + j < t.n; ++j) {
        bool wd, st;
        classify_byte(t, b0 + j, wd, st);
        (j < 16 ? wm0 : wm1) |= (uint32_t)wd << (j & 15);
        (j < 16 ? sm0 : sm1) |= (uint32_t)(wd && st) << (j & 15);
      }
    }
    wbits[w] = wm0 | (wm1 << 16);
    sbits[w] = sm0 | (sm1 << 16);
  }
}

// Does the token starting at bit j of word k have >= 2 codepoints (word-codepoint starts,
// sbits, inside it)? The same count as a walk to the token's end, from words k and k + 1 only:
// a token running through all of word k + 1 spans more than 32 bytes, hence >= 8 codepoints
// (a codepoint is at most 4 bytes).
__device__ __forceinline__ bool token_two_cp(uint32_t W0, uint32_t S0, uint32_t D0, uint32_t W1, uint32_t S1,
                                             uint32_t D1, bool has1, uint32_t j) {
  const uint32_t from = 0xFFFFFFFFu << j;
  const uint32_t stop0 = (~W0 | D0) & (j == 31 ? 0u : (0xFFFFFFFFu << (j + 1)));
  if (stop0) return __popc(S0 & from & ((stop0 & (0u - stop0)) - 1u)) >= 2;
  const uint32_t n = __popc(S0 & from);
  if (n >= 2) return true;
  if (!has1) return false;
  const uint32_t stop1 = ~W1 | D1;
  if (!stop1) return true;
  return n + __popc(S1 & ((stop1 & (0u - stop1)) - 1u)) >= 2;
}

// end (exclusive byte position) of the token starting at bit j of word k: the first stop after j
__device__ __forceinline__ uint64_t token_end(const uint32_t* wbits, const uint32_t* dbits, uint64_t nw, uint64_t k,
                                              uint32_t j, uint32_t W0, uint32_t D0, uint32_t W1, uint32_t D1) {
  uint32_t stop = (~W0 | D0) & (j == 31 ? 0u : (0xFFFFFFFFu << (j + 1)));
  if (stop) return (k << 5) + (__ffs(stop) - 1);
  if (++k >= nw) return nw << 5;
  stop = ~W1 | D1;
  while (!stop) {
    if (++k >= nw) return nw << 5;
    stop = ~wbits[k] | dbits[k];
  }
  return (k << 5) + (__ffs(stop) - 1);
}

// Token starts with >= 2 codepoints, one thread per 32-byte bitmap word, tiles of 256 words.
// Count pass: per-word counts (u8: at most 16 starts per word) and per-tile totals; the tile
// totals are scanned; emit pass: a block scan of the word counts gives every word's first
// output slot (no word-sized scan). Both read words i - 1 .. i + 1 only (token_two_cp); the
// emit pass walks on to a token's end when it runs past word i + 1.
constexpr int kTokThreads = 256;
#ifndef SL_CLASSIFY32
#define SL_CLASSIFY32 1  // one 32-byte bitmap word per thread (two 16-byte loads in flight)
#endif

template <bool EMIT>
__global__ void __launch_bounds__(kTokThreads) k_tokens(const uint32_t* __restrict__ wbits,
                                                        const uint32_t* __restrict__ sbits,
                                                        const uint32_t* __restrict__ dbits, uint64_t nw,
                                                        uint8_t* __restrict__ wcnt, uint32_t* __restrict__ tile,
                                                        uint64_t* __restrict__ tbeg, uint32_t* __restrict__ tlen) {
  __shared__ uint32_t sw[kTokThreads / 32 + 1];
  const uint64_t i = (uint64_t)blockIdx.x * kTokThreads + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t W = 0, S = 0, D = 0, W1 = 0, S1 = 0, D1 = 0, B = 0;
  const bool has1 = i + 1 < nw;
  if (i < nw) {
    W = wbits[i];
    S = sbits[i];
    D = dbits[i];
    if (has1) {
      W1 = wbits[i + 1];
      S1 = sbits[i + 1];
      D1 = dbits[i + 1];
    }
    const uint32_t prev = i ? (wbits[i - 1] >> 31) : 0u;
    B = W & (D | ~((W << 1) | prev));
  }
  uint32_t c = 0;
  if (!EMIT) {
    if (i < nw) {
      for (uint32_t b = B; b; b &= b - 1) c += token_two_cp(W, S, D, W1, S1, D1, has1, __ffs(b) - 1);
      wcnt[i] = (uint8_t)c;
    }
  } else {
    c = i < nw ? wcnt[i] : 0u;
  }
  // block exclusive scan of c (EMIT) / block total (count)
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sw[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int k = 0; k < kTokThreads / 32; ++k) {
      const uint32_t t = sw[k];
      sw[k] = run;
      run += t;
    }
    sw[kTokThreads / 32] = run;
  }
  __syncthreads();
  if (!EMIT) {
    if (threadIdx.x == 0) tile[blockIdx.x] = sw[kTokThreads / 32];
    return;
  }
  if (!c) return;
  uint32_t o = tile[blockIdx.x] + sw[w] + x - c;
  while (B) {
    const uint32_t j = __ffs(B) - 1;
    B &= B - 1;
    if (token_two_cp(W, S, D, W1, S1, D1, has1, j)) {
      const uint64_t p = (i << 5) + j;
      tbeg[o] = p;
      tlen[o] = (uint32_t)(token_end(wbits, dbits, nw, i, j, W, D, W1, D1) - p);
      ++o;
    }
  }
}

// ------------------------------------------------------------------ stemmer (shadow form)
// w: one byte per codepoint (ASCII as itself, anything else 0x80). Restates the
// reference's stemmer.cpp:125-391 step by step; returns the new length. Suffix tests run on
// a register copy of the last 8 symbols (byte k = w[n-1-k]) against compile-time packed
// constants, so each test is one AND + one compare.
__device__ __forceinline__ bool sv(uint32_t c) {  // a e i o u y
  const uint32_t d = c - 'a';
  return d < 26u && ((0x1104111u >> d) & 1u);
}

template <int M>
__host__ __device__ constexpr uint64_t pk(const char (&s)[M]) {
  uint64_t v = 0;
  for (int k = 0; k < M - 1; ++k) v |= (uint64_t)(uint8_t)s[M - 2 - k] << (8 * k);
  return v;
}
__host__ __device__ constexpr uint64_t lenmask(int m) { return m >= 8 ? ~0ull : ((1ull << (8 * m)) - 1ull); }

__device__ SL_TAIL_INLINE uint64_t tail8(const uint8_t* w, int n) {
  uint64_t t = 0;
  const int m = n < 8 ? n : 8;
  for (int k = 0; k < m; ++k) t |= (uint64_t)w[n - 1 - k] << (8 * k);
  return t;
}

// compile-time constants for a literal suffix
#define SL_PK(S) (std::integral_constant<uint64_t, pk(S)>::value)
#define SL_MK(S) (std::integral_constant<uint64_t, lenmask((int)sizeof(S) - 1)>::value)
#define ENDS(S) (n >= (int)sizeof(S) - 1 && (t & SL_MK(S)) == SL_PK(S))
#define SAME(S) (n == (int)sizeof(S) - 1 && (t & SL_MK(S)) == SL_PK(S))
#define SYNC() (t = tail8(w, n))
#define REPL(S, R)                                                    \
  do {                                                                \
    n -= (int)sizeof(S) - 1;                                          \
    for (int i_ = 0; i_ < (int)sizeof(R) - 1; ++i_) w[n + i_] = (uint8_t)(R)[i_]; \
    n += (int)sizeof(R) - 1;                                          \
    SYNC();                                                           \
  } while (0)
#define CUT(M)  \
  do {          \
    n -= (M);   \
    SYNC();     \
  } while (0)
#define PUSH(C)                        \
  do {                                 \
    w[n++] = (uint8_t)(C);             \
    t = (t << 8) | (uint64_t)(uint8_t)(C); \
  } while (0)
#define LAST(K) ((uint8_t)(t >> (8 * (K))))

__device__ __forceinline__ bool vowel_before(const uint8_t* w, int end) {
  for (int i = 0; i < end; ++i)
    if (sv(w[i])) return true;
  return false;
}
__device__ __forceinline__ bool short_syl(const uint8_t* w, int end) {
  if (end >= 3) {
    const uint8_t a = w[end - 3], b = w[end - 2], c = w[end - 1];
    if (!sv(c) && c != 'w' && c != 'x' && c != 'Y' && sv(b) && !sv(a)) return true;
  }
  return end == 2 && sv(w[0]) && !sv(w[1]);
}
__device__ __forceinline__ bool is_dbl(uint32_t c) {  // b d f g m n p r t
  const uint32_t d = c - 'a';
  return d < 26u && ((0xAB06Au >> d) & 1u);
}
__device__ __forceinline__ bool li_end(uint32_t c) {  // c d e g h k m n r t
  const uint32_t d = c - 'a';
  return d < 26u && ((0xA34DCu >> d) & 1u);
}

// Stems the shadow in place. Returns the final length; *shift = leading apostrophe removed;
// *ymark = some y was marked (postlude turns every 'Y' into 'y').
__device__ int stem_shadow(uint8_t* w, int n, int* shift, bool* ymark) {
  *shift = 0;
  *ymark = false;
  uint64_t t;
  SYNC();
  // irregular forms (stemmer.cpp:162-186), checked on the whole word before the prelude
#define SL_IRR(F, T)                                                        \
  if (SAME(F)) {                                                            \
    for (int i_ = 0; i_ < (int)sizeof(T) - 1; ++i_) w[i_] = (uint8_t)(T)[i_]; \
    return (int)sizeof(T) - 1;                                              \
  }
  SL_IRR("skis", "ski") SL_IRR("skies", "sky") SL_IRR("dying", "die") SL_IRR("lying", "lie")
  SL_IRR("tying", "tie") SL_IRR("idly", "idl") SL_IRR("gently", "gentl") SL_IRR("ugly", "ugli")
  SL_IRR("early", "earli") SL_IRR("only", "onli") SL_IRR("singly", "singl")
#undef SL_IRR
  if (SAME("sky") || SAME("news") || SAME("howe") || SAME("atlas") || SAME("cosmos") || SAME("bias") ||
      SAME("andes"))
    return n;
  // prelude
  if (n > 0 && w[0] == '\'') {
    for (int i = 1; i < n; ++i) w[i - 1] = w[i];
    --n;
    *shift = 1;
  }
  bool ym = false;
  if (n > 0 && w[0] == 'y') {
    w[0] = 'Y';
    ym = true;
  }
  for (int i = 1; i < n; ++i)
    if (w[i] == 'y' && sv(w[i - 1])) {
      w[i] = 'Y';
      ym = true;
    }
  *ymark = ym;
  SYNC();
  // regions (stemmer.cpp:204-226; R1 starts AT the first non-vowel after a vowel)
  int r1 = n, r2 = n;
  {
    int i = 0;
    if (n >= 5 && w[0] == 'g' && w[1] == 'e' && w[2] == 'n' && w[3] == 'e' && w[4] == 'r') i = 5;
    else if (n >= 6 && w[0] == 'c' && w[1] == 'o' && w[2] == 'm' && w[3] == 'm' && w[4] == 'u' && w[5] == 'n') i = 6;
    else if (n >= 5 && w[0] == 'a' && w[1] == 'r' && w[2] == 's' && w[3] == 'e' && w[4] == 'n') i = 5;
    bool done = false;
    if (i == 0) {
      while (i < n && !sv(w[i])) ++i;
      while (i < n && sv(w[i])) ++i;
      if (i == n) done = true;
    }
    if (!done) {
      r1 = i;
      while (i < n && !sv(w[i])) ++i;
      while (i < n && sv(w[i])) ++i;
      if (i != n) r2 = i;
    }
  }
  // step 0
  if (ENDS("'s'")) CUT(3);
  else if (ENDS("'s")) CUT(2);
  else if (ENDS("'")) CUT(1);
  // step 1a
  if (ENDS("sses")) {
    REPL("sses", "ss");
  } else if (ENDS("ied") || ENDS("ies")) {
    if (n >= 5) REPL("ies", "i");
    else REPL("ies", "ie");
  } else if (ENDS("us") || ENDS("ss")) {
  } else if (ENDS("s")) {
    if (n >= 3 && vowel_before(w, n - 2)) CUT(1);
  }
  if (SAME("inning") || SAME("outing") || SAME("canning") || SAME("herring") || SAME("earring") ||
      SAME("proceed") || SAME("exceed") || SAME("succeed"))
    return n;
  // step 1b
  if (ENDS("eedly") || ENDS("eed")) {
    const int m = ENDS("eedly") ? 5 : 3;
    if (n - m >= r1) {
      CUT(m);
      PUSH('e');
      PUSH('e');
    }
  } else {
    int m = 0;
    if (ENDS("ingly")) m = 5;
    else if (ENDS("edly")) m = 4;
    else if (ENDS("ing")) m = 3;
    else if (ENDS("ed")) m = 2;
    if (m && vowel_before(w, n - m)) {
      CUT(m);
      if (ENDS("at") || ENDS("bl") || ENDS("iz")) {
        PUSH('e');
      } else if (n >= 2 && LAST(0) == LAST(1) && is_dbl(LAST(0))) {
        CUT(1);
      } else if (n == r1 && short_syl(w, n)) {
        PUSH('e');
      }
    }
  }
  // step 1c
  if (n >= 3 && (LAST(0) == 'y' || LAST(0) == 'Y') && !sv(LAST(1))) {
    w[n - 1] = 'i';
    t = (t & ~0xFFull) | 'i';
  }
  // steps 2 and 3 (R1): the first listed suffix that matches decides
#define SL_RULE(S, R, DONE)                        \
  if (ENDS(S)) {                                   \
    if (n - (int)(sizeof(S) - 1) >= r1) REPL(S, R); \
    goto DONE;                                     \
  }
  SL_RULE("ization", "ize", done_step2) SL_RULE("ational", "ate", done_step2)
  SL_RULE("fulness", "ful", done_step2) SL_RULE("ousness", "ous", done_step2)
  SL_RULE("iveness", "ive", done_step2) SL_RULE("tional", "tion", done_step2)
  SL_RULE("biliti", "ble", done_step2) SL_RULE("lessli", "less", done_step2)
  SL_RULE("entli", "ent", done_step2) SL_RULE("fulli", "ful", done_step2) SL_RULE("ation", "ate", done_step2)
  SL_RULE("alism", "al", done_step2) SL_RULE("aliti", "al", done_step2) SL_RULE("ousli", "ous", done_step2)
  SL_RULE("iviti", "ive", done_step2) SL_RULE("enci", "ence", done_step2) SL_RULE("anci", "ance", done_step2)
  SL_RULE("abli", "able", done_step2) SL_RULE("izer", "ize", done_step2) SL_RULE("ator", "ate", done_step2)
  SL_RULE("alli", "al", done_step2) SL_RULE("bli", "ble", done_step2)
  if (ENDS("ogi")) {
    const int s = n - 3;
    if (s >= r1 && s >= 1 && LAST(3) == 'l') REPL("ogi", "og");
  } else if (ENDS("li")) {
    const int s = n - 2;
    if (s >= r1 && s >= 1 && li_end(LAST(2))) CUT(2);
  }
done_step2:
  // step 3
  if (ENDS("ative")) {
    const int s = n - 5;
    if (s >= r1 && s >= r2) CUT(5);
  } else {
    SL_RULE("ational", "ate", done_step3) SL_RULE("tional", "tion", done_step3)
    SL_RULE("alize", "al", done_step3) SL_RULE("icate", "ic", done_step3) SL_RULE("iciti", "ic", done_step3)
    SL_RULE("ical", "ic", done_step3) SL_RULE("ness", "", done_step3) SL_RULE("ful", "", done_step3)
  }
#undef SL_RULE
done_step3:
  // step 4 (R2)
  if (ENDS("ement")) {
    if (n - 5 >= r2) CUT(5);
  } else if (ENDS("ion")) {
    const int s = n - 3;
    if (s >= r2 && s >= 1 && (LAST(3) == 's' || LAST(3) == 't')) CUT(3);
  } else {
#define SL_DEL4(S)                                        \
  if (ENDS(S)) {                                          \
    if (n - (int)(sizeof(S) - 1) >= r2) CUT((int)sizeof(S) - 1); \
    goto done_step4;                                      \
  }
    SL_DEL4("ance") SL_DEL4("ence") SL_DEL4("able") SL_DEL4("ible") SL_DEL4("ment") SL_DEL4("ant")
    SL_DEL4("ent") SL_DEL4("ism") SL_DEL4("ate") SL_DEL4("iti") SL_DEL4("ous") SL_DEL4("ive") SL_DEL4("ize")
    SL_DEL4("al") SL_DEL4("er") SL_DEL4("ic")
#undef SL_DEL4
  }
done_step4:
  // step 5
  if (n >= 1 && LAST(0) == 'e') {
    if (n - 1 >= r2 || (n - 1 >= r1 && !short_syl(w, n - 1))) --n;
  } else if (n >= 2 && LAST(0) == 'l' && LAST(1) == 'l' && n - 1 >= r2) {
    --n;
  }
  return n;
}
#undef ENDS
#undef SAME
#undef SYNC
#undef REPL
#undef CUT
#undef PUSH
#undef LAST

// stem_english over UTF-8 bytes `in` (length len) into `out` (capacity >= len); `sh` is a
// shadow buffer of >= len bytes. Lenient decode like stemmer.cpp:33-62 (malformed ->
// unchanged). Returns the output length.
__device__ uint32_t stem_utf8(const uint8_t* in, uint32_t len, uint8_t* sh, uint8_t* out) {
  int n = 0;
  bool ok = true;
  for (uint32_t p = 0; p < len;) {
    const uint32_t b = in[p];
    if (b < 0x80) {
      sh[n++] = (uint8_t)b;
      ++p;
      continue;
    }
    const int L = lead_len(b);
    if (!L || p + L > len) {
      ok = false;
      break;
    }
    for (int i = 1; i < L; ++i)
      if ((in[p + i] & 0xC0) != 0x80) ok = false;
    if (!ok) break;
    sh[n++] = 0x80;
    p += L;
  }
  if (!ok || n <= 2) {
    for (uint32_t i = 0; i < len; ++i) out[i] = in[i];
    return len;
  }
  int shift;
  bool ym;
  const int m = stem_shadow(sh, n, &shift, &ym);
  // rebuild: placeholders are the original codepoints at the same position (+ shift)
  uint32_t o = 0, p = 0;
  for (int i = 0; i < shift; ++i) p += (in[p] < 0x80) ? 1 : lead_len(in[p]);
  for (int i = 0; i < m; ++i) {
    const uint32_t L = in[p] < 0x80 ? 1u : (uint32_t)lead_len(in[p]);
    if (sh[i] == 0x80) {
      for (uint32_t k = 0; k < L; ++k) out[o++] = in[p + k];
    } else {
      out[o++] = (ym && sh[i] == 'Y') ? (uint8_t)'y' : sh[i];
    }
    p += L;  // positions past the original length only occur for ASCII replacements
    if (p > len) p = len;
  }
  return o;
}

// ------------------------------------------------------------------ normalisation
struct StopView {
  const uint64_t* key;   // [cap] fnv1a64 of the word (0 = empty)
  const uint32_t* off;   // [cap] byte offset into bytes
  const uint32_t* len;   // [cap]
  const uint8_t* bytes;
  uint32_t cap;          // power of two (0 = no stopwords)
  uint32_t max_len;      // longest stopword (bytes): longer tokens skip the probe
};
struct VocabView {
  const uint64_t* tkey;
  const uint32_t* tval;
  uint32_t tcap;  // 0 = empty vocabulary
  const uint64_t* offs;
  const uint64_t* h2;
  const uint8_t* bytes;
};
struct NormArgs {
  TextView t;
  const uint64_t* tbeg;
  const uint32_t* tlen;
  uint64_t n_tok;
  int32_t lowercase, stem;
  StopView stop;
  VocabView voc;
  uint8_t* arena;            // normalised bytes at 2 * tbeg (build mode), or nullptr
  uint32_t* keep;            // 1 = not a stopword
  uint32_t* id;              // vocabulary id or kNew
  uint32_t* flen;            // normalised length
  uint64_t* h1;
  uint64_t* h2;
  uint32_t* long_flag;       // token deferred to the global-scratch pass
  uint32_t* err;
  int32_t weak;              // test hook: degenerate first hashes (collision paths)
};

__device__ bool is_stopword(const StopView& s, const uint8_t* w, uint32_t n) {
  if (!s.cap || n > s.max_len) return false;
  const uint64_t k = fnv1a64(w, n) | 1ull;
  for (uint32_t slot = (uint32_t)k & (s.cap - 1);; slot = (slot + 1) & (s.cap - 1)) {
    const uint64_t e = s.key[slot];
    if (!e) return false;
    if (e == k && s.len[slot] == n) {
      bool eq = true;
      for (uint32_t i = 0; i < n && eq; ++i) eq = s.bytes[s.off[slot] + i] == w[i];
      if (eq) return true;
    }
  }
}

__device__ uint32_t vocab_find(const VocabView& v, const uint8_t* w, uint32_t n, H2 h) {
  if (!v.tcap) return kNew;
  for (uint32_t slot = (uint32_t)h.a & (v.tcap - 1);; slot = (slot + 1) & (v.tcap - 1)) {
    const uint64_t e = v.tkey[slot];
    if (!e) return kNew;
    if (e == h.a) {  // identity = bytes: a string sharing the first hash keeps probing
      const uint32_t id = v.tval[slot];
      const uint64_t o = v.offs[id];
      bool eq = v.h2[id] == h.b && v.offs[id + 1] - o == n;
      for (uint32_t i = 0; i < n && eq; ++i) eq = v.bytes[o + i] == w[i];
      if (eq) return id;
    }
  }
}

// normalise token i with caller-provided buffers (nb: 2*len, sh: len+1, fb: 2*len)
__device__ void norm_one(const NormArgs& a, uint64_t i, uint8_t* nb, uint8_t* sh, uint8_t* fb) {
  const uint64_t b = a.tbeg[i];
  const uint32_t len = a.tlen[i];
  const uint8_t* src = a.t.text + b;
  uint32_t nl = 0;
  if (a.lowercase) {
    for (uint32_t p = 0; p < len;) {
      const uint32_t c0 = src[p];
      if (c0 < 0x80) {  // ASCII fast path
        nb[nl++] = (uint8_t)((c0 >= 'A' && c0 <= 'Z') ? c0 + 32 : c0);
        ++p;
        continue;
      }
      uint32_t cp;
      p += decode_at(src + p, &cp);
      nl += put_utf8(nb + nl, lower_cp(cp));
    }
  } else {
    for (uint32_t p = 0; p < len; ++p) nb[p] = src[p];
    nl = len;
  }
  if (is_stopword(a.stop, nb, nl)) {
    a.keep[i] = 0;
    a.id[i] = kNew;
    a.flen[i] = 0;
    return;
  }
  a.keep[i] = 1;
  const uint8_t* fin = nb;
  uint32_t fl = nl;
  if (a.stem) {
    fl = stem_utf8(nb, nl, sh, fb);
    fin = fb;
  }
  H2 h = hash2(fin, fl);
  if (a.weak) h.a = (h.a & 7ull) | 1ull;  // test hook (SL_TEXT_WEAK_HASH): first-hash collisions everywhere
  a.flen[i] = fl;
  a.h1[i] = h.a;
  a.h2[i] = h.b;
  a.id[i] = vocab_find(a.voc, fin, fl, h);
  if (a.arena)
    for (uint32_t k = 0; k < fl; ++k) a.arena[2 * b + k] = fin[k];
}

__global__ void k_norm_fast(NormArgs a) {
  uint8_t nb[2 * kFastBytes], sh[kFastBytes + 1], fb[2 * kFastBytes];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_tok;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (a.tlen[i] > kFastBytes) {
      a.long_flag[i] = 1;
      continue;
    }
    a.long_flag[i] = 0;
    norm_one(a, i, nb, sh, fb);
  }
}

// long tokens: scratch slot of 5 * len bytes each (nb 2len | sh len | fb 2len)
__global__ void k_norm_long(NormArgs a, const uint32_t* __restrict__ list, uint32_t n_list,
                            const uint64_t* __restrict__ soff, uint8_t* __restrict__ scratch) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n_list; j += gridDim.x * blockDim.x) {
    const uint64_t i = list[j];
    uint8_t* base = scratch + soff[j];
    const uint32_t len = a.tlen[i];
    norm_one(a, i, base, base + 2 * (uint64_t)len, base + 3 * (uint64_t)len + 1);
  }
}

// ------------------------------------------------------------------ small helpers
__global__ void k_flag_to_u32(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t n,
                              uint32_t* __restrict__ out, int mode) {
  // mode 0: out = a (copy); mode 1: out = a && b == kNew (new kept token); mode 2: a && b != kNew
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = mode == 0 ? a[i] : mode == 1 ? (a[i] && b[i] == kNew) : (a[i] && b[i] != kNew);
}

__global__ void k_compact_idx(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, uint64_t n,
                              uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[pos[i]] = (uint32_t)i;
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx, uint32_t n,
                             uint32_t* __restrict__ out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) out[j] = src[idx[j]];
}

// batch-local distinct-string table of the NEW normalised strings: 128-bit key per string
// (kx, ky: the two 64-bit hashes, or a reseeded pair after a verified collision), first =
// smallest raw-entry index. A plain read comes first, so repeated strings stay read-only.
__global__ void k_dedup_insert(const uint32_t* __restrict__ ntok, uint32_t M, const uint64_t* __restrict__ kx,
                               const uint64_t* __restrict__ ky, ulonglong2* __restrict__ key,
                               uint32_t* __restrict__ first, uint32_t cap, uint32_t* __restrict__ cnt) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < M; j += gridDim.x * blockDim.x) {
    const uint32_t i = ntok[j];
    ulonglong2 k = make_ulonglong2(kx[j], ky[j]);
    if ((k.x | k.y) == 0ull) k.y = 1ull;  // (0, 0) marks an empty slot
    uint32_t slot = (uint32_t)k.x & (cap - 1);
    for (uint32_t probes = 0;; ++probes) {
      if (probes == cap) {
        atomicOr(cnt + 1, 1u);
        break;
      }
      ulonglong2 cur = key[slot];
      if ((cur.x | cur.y) == 0ull) {
        cur = cas128(key + slot, make_ulonglong2(0ull, 0ull), k);
        if ((cur.x | cur.y) == 0ull) {
          atomicAdd(cnt, 1u);
          cur = k;
        }
      }
      if (cur.x == k.x && cur.y == k.y) {
        if (first[slot] > i) atomicMin(first + slot, i);
        break;
      }
      slot = (slot + 1) & (cap - 1);
    }
  }
}

// 128-bit dedup keys of the new strings: seed 0 = the normalisation's own (h1, h2); a reseeded
// pair from the normalised bytes (arena) after a verified collision
__global__ void k_new_keys(const uint32_t* __restrict__ ntok, uint32_t M, const uint64_t* __restrict__ h1,
                           const uint64_t* __restrict__ h2, const uint8_t* __restrict__ arena,
                           const uint64_t* __restrict__ tbeg, const uint32_t* __restrict__ flen, uint32_t seed,
                           int32_t weak, uint64_t* __restrict__ kx, uint64_t* __restrict__ ky) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < M; j += gridDim.x * blockDim.x) {
    const uint32_t i = ntok[j];
    if (seed == 0) {
      kx[j] = weak ? (uint64_t)flen[i] : h1[i];  // weak: test hook, every equal-length string collides
      ky[j] = weak ? 1ull : h2[i];
      continue;
    }
    const uint8_t* w = arena + 2 * tbeg[i];
    uint64_t a = 0x8ebc6af09c88c6e3ull * seed, b = 0x589965cc75374cc3ull + seed;
    for (uint32_t k = 0; k < flen[i]; ++k) {
      a = (a ^ w[k]) * 0x100000001b3ull;
      b = (b + w[k] + 1) * 0xd6e8feb86659fd93ull;
      b ^= b >> 29;
    }
    kx[j] = fmix64(a ^ flen[i]);
    ky[j] = fmix64(b);
  }
}

__global__ void k_slot_flags(const uint64_t* __restrict__ key, uint32_t cap, uint32_t* __restrict__ flag) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < cap; s += gridDim.x * blockDim.x)
    flag[s] = key[s] != 0ull;
}

__global__ void k_slot_list(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                            const uint32_t* __restrict__ first, uint32_t cap, uint32_t* __restrict__ slots,
                            uint32_t* __restrict__ fk) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < cap; s += gridDim.x * blockDim.x)
    if (flag[s]) {
      slots[pos[s]] = s;
      fk[pos[s]] = first[s];
    }
}

// id of every new token; its normalised bytes must equal its group's first occurrence's
// (a mismatch is a verified 128-bit collision: err bit 2, the host redoes the dedup reseeded)
__global__ void k_dedup_assign(const uint32_t* __restrict__ ntok, uint32_t M, const uint64_t* __restrict__ kx,
                               const uint64_t* __restrict__ ky, const uint32_t* __restrict__ flen,
                               const uint8_t* __restrict__ arena, const uint64_t* __restrict__ tbeg,
                               const ulonglong2* __restrict__ key, const uint32_t* __restrict__ first,
                               const uint32_t* __restrict__ rank, uint32_t cap, uint32_t V0, uint32_t* __restrict__ id,
                               uint32_t* __restrict__ err) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < M; j += gridDim.x * blockDim.x) {
    const uint32_t i = ntok[j];
    ulonglong2 k = make_ulonglong2(kx[j], ky[j]);
    if ((k.x | k.y) == 0ull) k.y = 1ull;
    uint32_t slot = (uint32_t)k.x & (cap - 1);
    while (key[slot].x != k.x || key[slot].y != k.y) slot = (slot + 1) & (cap - 1);
    const uint32_t f = first[slot];
    if (f != i) {
      bool eq = flen[f] == flen[i];
      const uint8_t* a = arena + 2 * tbeg[i];
      const uint8_t* b = arena + 2 * tbeg[f];
      for (uint32_t c = 0; c < flen[i] && eq; ++c) eq = a[c] == b[c];
      if (!eq) atomicOr(err, 4u);
    }
    id[i] = V0 + rank[slot];
  }
}

// groups sorted by first occurrence: rank -> id = V0 + rank
__global__ void k_group_rank(const uint32_t* __restrict__ gsorted, uint32_t G, uint32_t* __restrict__ grank) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < G; r += gridDim.x * blockDim.x) grank[gsorted[r]] = r;
}

// new vocabulary entries in id order: representative token, length
__global__ void k_new_entries(const uint32_t* __restrict__ gsorted_first, uint32_t G, const uint32_t* __restrict__ flen,
                              uint32_t* __restrict__ elen) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < G; r += gridDim.x * blockDim.x)
    elen[r] = flen[gsorted_first[r]];
}

__global__ void k_copy_entries(const uint32_t* __restrict__ first, uint32_t G, const uint64_t* __restrict__ tbeg,
                               const uint32_t* __restrict__ flen, const uint8_t* __restrict__ arena,
                               const uint32_t* __restrict__ epos, uint64_t base, uint32_t V0,
                               const uint64_t* __restrict__ h2tok, uint8_t* __restrict__ bytes,
                               uint64_t* __restrict__ offs, uint64_t* __restrict__ h2v) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < G; r += gridDim.x * blockDim.x) {
    const uint32_t t = first[r];
    const uint64_t o = base + epos[r];
    const uint32_t n = flen[t];
    for (uint32_t k = 0; k < n; ++k) bytes[o + k] = arena[2 * tbeg[t] + k];
    offs[V0 + r + 1] = o + n;
    h2v[V0 + r] = h2tok[t];
  }
}

__global__ void k_table_insert(const uint64_t* __restrict__ h1tok, const uint32_t* __restrict__ first, uint32_t G,
                               uint32_t V0, uint64_t* __restrict__ tkey, uint32_t* __restrict__ tval, uint32_t tcap,
                               uint32_t* __restrict__ err) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < G; r += gridDim.x * blockDim.x) {
    const uint64_t k = h1tok[first[r]];
    for (uint32_t slot = (uint32_t)k & (tcap - 1);; slot = (slot + 1) & (tcap - 1)) {
      const unsigned long long prev = atomicCAS((unsigned long long*)tkey + slot, 0ull, (unsigned long long)k);
      if (prev == 0ull) {
        tval[slot] = V0 + r;
        break;
      }
      // prev == k: another string with the same first hash (vocab_find compares bytes): probe on
    }
  }
}

// re-insert an existing vocabulary into a larger table: hash recomputed from the bytes
__global__ void k_table_rehash(const uint64_t* __restrict__ offs, const uint8_t* __restrict__ bytes, uint32_t V,
                               uint64_t* __restrict__ tkey, uint32_t* __restrict__ tval, uint32_t tcap,
                               uint64_t* __restrict__ h2v, int32_t weak) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < V; id += gridDim.x * blockDim.x) {
    H2 h = hash2(bytes + offs[id], (uint32_t)(offs[id + 1] - offs[id]));
    if (weak) h.a = (h.a & 7ull) | 1ull;  // the same degenerate first hash as norm_one
    h2v[id] = h.b;
    for (uint32_t slot = (uint32_t)h.a & (tcap - 1);; slot = (slot + 1) & (tcap - 1)) {
      if (atomicCAS((unsigned long long*)tkey + slot, 0ull, (unsigned long long)h.a) == 0ull) {
        tval[slot] = id;
        break;
      }
    }
  }
}

// token offsets per document: lower_bound of the document's first byte among kept tokens
__global__ void k_doc_token_offsets(const uint64_t* __restrict__ doc_off, uint32_t N,
                                    const uint64_t* __restrict__ kbeg, uint64_t T, uint64_t* __restrict__ out) {
  for (uint32_t d = blockIdx.x * blockDim.x + threadIdx.x; d <= N; d += gridDim.x * blockDim.x) {
    if (d == N) {
      out[d] = T;
      continue;
    }
    const uint64_t x = doc_off[d];
    uint64_t lo = 0, hi = T;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (kbeg[mid] < x) lo = mid + 1; else hi = mid;
    }
    out[d] = lo;
  }
}

__global__ void k_stem_batch(const uint8_t* __restrict__ in, const uint64_t* __restrict__ off, uint32_t n,
                             uint8_t* __restrict__ scratch, uint8_t* __restrict__ out, uint32_t* __restrict__ olen) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t b = off[i];
    const uint32_t len = (uint32_t)(off[i + 1] - b);
    olen[i] = stem_utf8(in + b, len, scratch + b, out + b);
  }
}

// ------------------------------------------------------------------ raw-string dedup
// Normalisation (lowercase, stopwords, stemming) is a function of the token's raw bytes, and a
// Zipf corpus repeats a few hundred thousand surface forms tens of millions of times: the raw
// strings are deduplicated first (two 64-bit hashes per token, an L2-resident table) and only
// the distinct ones are normalised.
// table of distinct raw strings: key = a 128-bit hash of the bytes (two 64-bit lanes, the
// second mixed with the length), inserted with one 128-bit CAS, so strings that share one lane
// simply occupy different slots; first = smallest token index; tslot[i] = token i's slot.
struct RawMix {
  uint64_t a, b;
  // seed > 0 only after a verified collision (k_raw_verify): the table is rebuilt with new hashes
  __device__ __forceinline__ RawMix(uint32_t n, uint32_t seed)
      : a((0x243f6a8885a308d3ull ^ n) + 0xa0761d6478bd642full * seed),
        b(0x13198a2e03707344ull + 0x9e3779b97f4a7c15ull * n + 0xe7037ed1a0b428dbull * seed) {}
  __device__ __forceinline__ void add(uint64_t w) {  // the next (up to) 8 bytes, little-endian
    a = (a ^ w) * 0x100000001b3ull;
    a ^= a >> 29;
    b = (b + w) * 0xd6e8feb86659fd93ull;
    b ^= b >> 32;
  }
  __device__ __forceinline__ ulonglong2 key() const {
    ulonglong2 k;
    k.x = fmix64(a);
    k.y = fmix64(b ^ (a >> 7));
    if ((k.x | k.y) == 0ull) k.y = 1ull;  // (0, 0) marks an empty slot
    return k;
  }
};

// 8 bytes per mixing round on two independent lanes (batch-local: never compared with hashes
// from elsewhere). ALIGNED (text 4-byte aligned): the rounds' bytes come from aligned 32-bit
// words joined by funnel shifts (never a word past the one holding the token's last byte);
// otherwise byte loads. Both feed identical 8-byte words.
// the (up to) 8 bytes [p, p + m) of text as a little-endian word, zero-padded. ALIGNED (text
// 4-byte aligned): from aligned 32-bit words joined by funnel shifts (never a word past the one
// holding the last byte); otherwise byte loads.
template <bool ALIGNED>
__device__ __forceinline__ uint64_t load_word8(const uint8_t* __restrict__ text, uint64_t p, uint32_t m) {
  if (ALIGNED) {
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(text);
    const uint32_t sh = (uint32_t)(p & 3) * 8;
    const uint64_t wi = p >> 2, wl = (p + m - 1) >> 2;  // words holding the first / last byte
    const uint32_t w0 = __ldg(w32 + wi);
    const uint32_t w1 = wl > wi ? __ldg(w32 + wi + 1) : 0u;
    const uint32_t w2 = wl > wi + 1 ? __ldg(w32 + wi + 2) : 0u;
    uint64_t w = ((uint64_t)__funnelshift_r(w1, w2, sh) << 32) | __funnelshift_r(w0, w1, sh);
    if (m < 8) w &= (1ull << (8 * m)) - 1ull;
    return w;
  }
  uint64_t w = 0;
  for (uint32_t j = 0; j < m; ++j) w |= (uint64_t)__ldg(text + p + j) << (8 * j);
  return w;
}

template <bool ALIGNED>
__device__ __forceinline__ ulonglong2 raw_key(const uint8_t* __restrict__ text, uint64_t beg, uint32_t n,
                                              uint32_t seed) {
  RawMix h(n, seed);
  for (uint32_t i = 0; i < n; i += 8) h.add(load_word8<ALIGNED>(text, beg + i, min(8u, n - i)));
  return h.key();
}

// byte equality of text[a, a + n) and text[b, b + n), 8 bytes per step
template <bool ALIGNED>
__device__ __forceinline__ bool bytes_equal(const uint8_t* __restrict__ text, uint64_t a, uint64_t b, uint32_t n) {
  for (uint32_t i = 0; i < n; i += 8) {
    const uint32_t m = min(8u, n - i);
    if (load_word8<ALIGNED>(text, a + i, m) != load_word8<ALIGNED>(text, b + i, m)) return false;
  }
  return true;
}

// Identity of raw strings is BYTE equality (the reference's string map, vocabulary.hpp:26-33).
// A token of at most 15 bytes IS its key: (bytes 0-7, bytes 8-14 | length << 56), so equal keys
// mean equal strings by construction. Longer tokens key on a 128-bit hash (top byte 0xFF, which
// no short key has); the claimant of such a slot records its (position << 24 | length) in
// wrep[slot], and k_raw_verify_long then checks every long token byte by byte against its
// slot's claimant. A mismatch (a verified 128-bit collision) makes the host rebuild the table
// with another seed.
#ifndef SL_EXACT_KEY_BYTES
#define SL_EXACT_KEY_BYTES 15
#endif
constexpr uint32_t kExactKeyBytes = SL_EXACT_KEY_BYTES;

template <bool ALIGNED>
__global__ void k_raw_insert(const uint8_t* __restrict__ text, const uint64_t* __restrict__ tbeg,
                             const uint32_t* __restrict__ tlen, uint64_t n, ulonglong2* __restrict__ key,
                             uint32_t* __restrict__ first, uint64_t* __restrict__ wrep, uint32_t cap,
                             uint32_t* __restrict__ cnt, uint32_t* __restrict__ tslot, uint32_t seed, int32_t weak) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t beg = tbeg[i];
    const uint32_t len = tlen[i];
    const bool exact = len <= kExactKeyBytes;
    ulonglong2 k;
    if (exact) {
      k.x = load_word8<ALIGNED>(text, beg, min(8u, len));
      k.y = (len > 8 ? load_word8<ALIGNED>(text, beg + 8, len - 8) : 0ull) | ((uint64_t)len << 56);
    } else if (len >= 0xFFFFFFu) {  // (position, length) packs the length in 24 bits
      atomicOr(cnt + 2, 2u);
      continue;
    } else if (weak && seed == 0) {  // test hook: every long string of one length collides
      k = make_ulonglong2((uint64_t)len, 0xFFull << 56);
    } else {
      k = raw_key<ALIGNED>(text, beg, len, seed);
      k.y |= 0xFFull << 56;
    }
    // probe start: mixed key (a short key's raw bytes are a poor hash); weak: length only
    uint32_t slot = (uint32_t)(weak ? len * 0x9E3779B1u : fmix64(k.x ^ (k.y * 0x9e3779b97f4a7c15ull))) & (cap - 1);
    for (uint32_t probes = 0;; ++probes) {
      if (probes == cap) {
        atomicOr(cnt + 1, 1u);
        break;
      }
      ulonglong2 cur = key[slot];  // plain read first: repeated strings skip the atomics
      if ((cur.x | cur.y) == 0ull) {
        cur = cas128(key + slot, make_ulonglong2(0ull, 0ull), k);
        if ((cur.x | cur.y) == 0ull) {
          atomicAdd(cnt, 1u);
          cur = k;
          if (!exact) wrep[slot] = (beg << 24) | len;  // read by k_raw_verify_long (after this kernel)
        }
      }
      if (cur.x == k.x && cur.y == k.y) {
        // a stale (larger) cached value only costs an atomicMin that changes nothing
        if (first[slot] > (uint32_t)i) atomicMin(first + slot, (uint32_t)i);
        tslot[i] = slot;
        break;
      }
      slot = (slot + 1) & (cap - 1);
    }
  }
}

// Every hashed (long) token against its slot's claimant, byte by byte (cnt[2] on a mismatch).
// A block takes 2048 tokens, queues its long ones in shared memory and verifies the queue with
// all threads busy (long tokens are a minority: a per-token loop would idle most lanes).
constexpr int kVerTile = 2048;
template <bool ALIGNED>
__global__ void __launch_bounds__(256) k_raw_verify_long(const uint8_t* __restrict__ text,
                                                         const uint64_t* __restrict__ tbeg,
                                                         const uint32_t* __restrict__ tlen, uint64_t n,
                                                         const uint32_t* __restrict__ tslot,
                                                         const uint64_t* __restrict__ wrep, uint32_t* __restrict__ cnt) {
  __shared__ uint32_t q[kVerTile];
  __shared__ uint32_t qn;
  if (*(volatile uint32_t*)(cnt + 1)) return;  // the insert overflowed: the table is rebuilt anyway
  for (uint64_t t0 = (uint64_t)blockIdx.x * kVerTile; t0 < n; t0 += (uint64_t)gridDim.x * kVerTile) {
    if (threadIdx.x == 0) qn = 0;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < kVerTile; j += blockDim.x) {
      const uint64_t i = t0 + j;
      if (i < n && tlen[i] > kExactKeyBytes) q[atomicAdd(&qn, 1u)] = j;
    }
    __syncthreads();
    const uint32_t m = qn;
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
      const uint64_t i = t0 + q[j];
      const uint32_t len = tlen[i];
      const uint64_t beg = tbeg[i];
      const uint64_t rp = wrep[tslot[i]];
      if ((rp >> 24) != beg && ((uint32_t)(rp & 0xFFFFFFu) != len || !bytes_equal<ALIGNED>(text, beg, rp >> 24, len)))
        atomicOr(cnt + 2, 1u);
    }
    __syncthreads();
  }
}

__global__ void k_slot_flags128(const ulonglong2* __restrict__ key, uint32_t cap, uint32_t* __restrict__ flag) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < cap; s += gridDim.x * blockDim.x) {
    const ulonglong2 k = key[s];
    flag[s] = (k.x | k.y) != 0ull;
  }
}

// per occupied slot of the raw table: its entry's id (31 bits: ids < 2^31 or kNew) and the
// kept flag (build: not a stopword; query: also in the vocabulary) in one word
__global__ void k_raw_slots(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ rank, uint32_t cap,
                            const uint32_t* __restrict__ rkeep, const uint32_t* __restrict__ rid, int build,
                            uint32_t* __restrict__ rs) {
  for (uint32_t sl = blockIdx.x * blockDim.x + threadIdx.x; sl < cap; sl += gridDim.x * blockDim.x) {
    if (!flag[sl]) continue;
    const uint32_t r = rank[sl];
    const uint32_t t = rid[r];
    const bool kept = rkeep[r] && (build || t != kNew);
    rs[sl] = (t & 0x7FFFFFFFu) | (kept ? 0x80000000u : 0u);
  }
}

// Kept tokens in order, in two passes over tiles of kKeepTile tokens: round j of a tile is
// tokens [j*256, j*256 + 256) (thread tid takes token j*256 + tid: coalesced loads). The kept
// flag is the token's raw entry's flag, read through its slot. k_keep_count counts each tile's
// kept tokens, one scan of the tile counts, then k_keep_emit ranks every kept token by the
// ballots of its (round, warp) and writes its id and first byte (coalesced runs).
constexpr int kKeepThreads = 256, kKeepRounds = 16, kKeepTile = kKeepThreads * kKeepRounds;
constexpr int kKeepWarps = kKeepThreads / 32;

__global__ void __launch_bounds__(kKeepThreads) k_keep_count(const uint32_t* __restrict__ tslot, uint64_t n,
                                                             const uint32_t* __restrict__ rs,
                                                             uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t s_c[kKeepWarps];
  const uint64_t t0 = (uint64_t)blockIdx.x * kKeepTile + threadIdx.x;
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kKeepRounds; ++j) {
    const uint64_t i = t0 + (uint64_t)j * kKeepThreads;
    const bool kept = i < n && (__ldg(rs + __ldg(tslot + i)) >> 31);
    c += __popc(__ballot_sync(0xffffffffu, kept));
  }
  if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < kKeepWarps; ++w) tot += s_c[w];
    tile_cnt[blockIdx.x] = tot;
  }
}

__global__ void __launch_bounds__(kKeepThreads) k_keep_emit(const uint32_t* __restrict__ tslot, uint64_t n,
                                                            const uint32_t* __restrict__ rs,
                                                            const uint64_t* __restrict__ tbeg,
                                                            const uint32_t* __restrict__ tile_off,
                                                            uint32_t* __restrict__ ids, uint64_t* __restrict__ kbeg) {
  __shared__ uint32_t s_off[kKeepRounds * kKeepWarps];  // (round, warp) -> first output index in the tile
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t t0 = (uint64_t)blockIdx.x * kKeepTile + threadIdx.x;
  uint32_t ik[kKeepRounds], bal[kKeepRounds];
#pragma unroll
  for (int j = 0; j < kKeepRounds; ++j) {
    const uint64_t i = t0 + (uint64_t)j * kKeepThreads;
    ik[j] = i < n ? __ldg(rs + __ldg(tslot + i)) : 0u;
    bal[j] = __ballot_sync(0xffffffffu, ik[j] >> 31);
    if (lane == 0) s_off[j * kKeepWarps + w] = __popc(bal[j]);
  }
  __syncthreads();
  if (w == 0) {  // exclusive scan of the 128 (round, warp) counts, 4 per lane
    uint32_t v[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[q] = s_off[lane * 4 + q];
      sum += v[q];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t run = x - sum;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      s_off[lane * 4 + q] = run;
      run += v[q];
    }
  }
  __syncthreads();
  const uint32_t o = tile_off[blockIdx.x];
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kKeepRounds; ++j) {
    if (ik[j] >> 31) {
      const uint64_t i = t0 + (uint64_t)j * kKeepThreads;
      const uint32_t pos = o + s_off[j * kKeepWarps + w] + __popc(bal[j] & lt);
      const uint32_t t = ik[j] & 0x7FFFFFFFu;
      ids[pos] = t == 0x7FFFFFFFu ? kNew : t;
      kbeg[pos] = __ldg(tbeg + i);
    }
  }
}

__global__ void k_gather_u64(const uint64_t* __restrict__ src, const uint32_t* __restrict__ idx, uint32_t n,
                             uint64_t* __restrict__ out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) out[j] = src[idx[j]];
}

__global__ void k_add_u64(const uint64_t* __restrict__ in, uint64_t n, uint64_t add, uint64_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i] + add;
}

// ------------------------------------------------------------------ host side
inline int text_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
  return cache[dev] > 0 ? cache[dev] : 1;
}

inline unsigned grid_for(uint64_t n, int per = 256) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + per - 1) / per, 64ull * text_sms()));
}

struct TScratch {
  cudaStream_t st;
  std::vector<void*> ps;
  explicit TScratch(cudaStream_t s) : st(s) {}
  template <class T>
  int32_t alloc(T** p, uint64_t n) {
    if (n == 0) n = 1;
    if (cudaMallocAsync((void**)p, n * sizeof(T), st) != cudaSuccess) {
      *p = nullptr;
      SL_FAIL(SL_ENOMEM, "tokenizer: device allocation of " + std::to_string(n * sizeof(T)) + " bytes failed");
    }
    ps.push_back(*p);
    return SL_OK;
  }
  ~TScratch() {
    for (void* p : ps) cudaFreeAsync(p, st);
  }
};

struct TextStream {
  int device = -1;
  cudaStream_t st = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // sl_tokenize_stream's copy streams (created once)
};
thread_local TextStream t_text_stream[16];

int32_t text_stream(int device, cudaStream_t* out) {
  if (device < 0 || device >= 16) SL_FAIL(SL_EINVAL, "device ordinal out of range");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    SL_FAIL(SL_ECUDA, "tokenizer: no CUDA device available (there is no CPU fallback)");
  SL_CUDA_TRY(cudaSetDevice(device));
  TextStream& s = t_text_stream[device];
  if (!s.st) {
    SL_CUDA_TRY(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
    s.device = device;
    cudaMemPool_t pool;  // keep freed scratch mapped between calls (no page re-mapping per batch)
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  *out = s.st;
  return SL_OK;
}

uint32_t pow2_at_least(uint64_t x) {
  uint64_t c = 16;
  while (c < x) c <<= 1;
  return (uint32_t)std::min<uint64_t>(c, 1ull << 31);
}

// host-built stopword table
struct StopTable {
  std::vector<uint64_t> key;
  std::vector<uint32_t> off, len;
  std::vector<uint8_t> bytes;
  uint32_t cap = 0;
  uint32_t max_len = 0;
};

std::vector<std::string> parse_stopwords(const char* s, uint64_t n) {
  std::vector<std::string> out;
  std::string cur;
  auto flush = [&] {
    // trim trailing '\r' and surrounding spaces; '#' lines are comments (stopwords.hpp:13-15)
    while (!cur.empty() && (cur.back() == '\r' || cur.back() == ' ' || cur.back() == '\t')) cur.pop_back();
    size_t a = 0;
    while (a < cur.size() && (cur[a] == ' ' || cur[a] == '\t')) ++a;
    cur = cur.substr(a);
    if (!cur.empty() && cur[0] != '#') out.push_back(cur);
    cur.clear();
  };
  for (uint64_t i = 0; i < n; ++i) {
    if (s[i] == '\n') flush();
    else cur += s[i];
  }
  flush();
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

StopTable make_stop_table(const std::vector<std::string>& words) {
  StopTable t;
  if (words.empty()) return t;
  t.cap = pow2_at_least(words.size() * 2);
  t.key.assign(t.cap, 0);
  t.off.assign(t.cap, 0);
  t.len.assign(t.cap, 0);
  for (const auto& w : words) {
    const uint64_t k = fnv1a64(reinterpret_cast<const uint8_t*>(w.data()), (uint32_t)w.size()) | 1ull;
    uint32_t slot = (uint32_t)k & (t.cap - 1);
    while (t.key[slot]) slot = (slot + 1) & (t.cap - 1);
    t.key[slot] = k;
    t.off[slot] = (uint32_t)t.bytes.size();
    t.len[slot] = (uint32_t)w.size();
    t.max_len = std::max<uint32_t>(t.max_len, (uint32_t)w.size());
    t.bytes.insert(t.bytes.end(), w.begin(), w.end());
  }
  return t;
}

// grow a device array (stream-ordered), keeping `keep` elements
template <class T>
int32_t grow(T** p, uint64_t keep, uint64_t newcap, cudaStream_t st) {
  T* q = nullptr;
  if (cudaMallocAsync((void**)&q, std::max<uint64_t>(newcap, 1) * sizeof(T), st) != cudaSuccess)
    SL_FAIL(SL_ENOMEM, "vocabulary: device allocation failed");
  if (*p && keep) SL_CUDA_TRY(cudaMemcpyAsync(q, *p, keep * sizeof(T), cudaMemcpyDeviceToDevice, st));
  if (*p) cudaFreeAsync(*p, st);
  *p = q;
  return SL_OK;
}

int32_t vocab_reserve(sl_vocab* v, uint64_t n_entries, uint64_t n_bytes, cudaStream_t st) {
  if (n_entries > v->vcap) {
    const uint64_t cap = std::max<uint64_t>(n_entries, (uint64_t)v->vcap * 2);
    if (n_entries > 0x7FFFFFF0ull) SL_FAIL(SL_EUNSUPPORTED, "vocabulary larger than 2^31 entries");
    SL_TRY(grow(&v->offs, v->V + 1ull, cap + 1, st));
    SL_TRY(grow(&v->h2, v->V, cap, st));
    if (v->vcap == 0) SL_CUDA_TRY(cudaMemsetAsync(v->offs, 0, 8, st));
    v->vcap = (uint32_t)cap;
  }
  if (n_bytes > v->bcap) {
    const uint64_t cap = std::max<uint64_t>(n_bytes, v->bcap * 2);
    SL_TRY(grow(&v->bytes, v->bused, cap, st));
    v->bcap = cap;
  }
  const uint64_t want = pow2_at_least(n_entries * 2);
  if (want > v->tcap) {  // rebuild the hash table
    if (v->tkey) cudaFreeAsync(v->tkey, st);
    if (v->tval) cudaFreeAsync(v->tval, st);
    if (cudaMallocAsync((void**)&v->tkey, want * 8, st) != cudaSuccess ||
        cudaMallocAsync((void**)&v->tval, want * 4, st) != cudaSuccess)
      SL_FAIL(SL_ENOMEM, "vocabulary: hash table allocation failed");
    SL_CUDA_TRY(cudaMemsetAsync(v->tkey, 0, want * 8, st));
    v->tcap = (uint32_t)want;
    if (v->V) {
      k_table_rehash<<<grid_for(v->V), 256, 0, st>>>(v->offs, v->bytes, v->V, v->tkey, v->tval, v->tcap, v->h2,
                                                         v->weak);
      ++t_launches;
    }
  }
  SL_CUDA_TRY(cudaGetLastError());
  return SL_OK;
}

int32_t tokenize_impl(sl_vocab* v, const sl_tokenizer_config* cfg, int32_t build, const char* text_in,
                      const uint64_t* doc_off_in, uint32_t N, int32_t mem, sl_token_batch** out) {
  if (!v || !cfg || !out) SL_FAIL(SL_EINVAL, "tokenize: null argument");
  if (mem != SL_MEM_HOST && mem != SL_MEM_DEVICE) SL_FAIL(SL_EINVAL, "tokenize: bad mem kind");
  if (cfg->stemmer != SL_STEMMER_NONE && cfg->stemmer != SL_STEMMER_SNOWBALL_ENGLISH)
    SL_FAIL(SL_EINVAL, "unknown stemmer");
  if (N && !doc_off_in) SL_FAIL(SL_EINVAL, "tokenize: null document offsets");
  cudaStream_t st;
  SL_TRY(text_stream(v->device, &st));
  TScratch scr(st);
  // ---- inputs on the device
  uint64_t first = 0, last = 0;
  const uint64_t* doc_off = doc_off_in;
  if (N) {
    if (mem == SL_MEM_HOST) {
      first = doc_off_in[0];
      last = doc_off_in[N];
      for (uint32_t d = 0; d < N; ++d)
        if (doc_off_in[d + 1] < doc_off_in[d]) SL_FAIL(SL_EINVAL, "tokenize: document offsets must be non-decreasing");
    } else {
      SL_CUDA_TRY(cudaMemcpyAsync(&first, doc_off_in, 8, cudaMemcpyDeviceToHost, st));
      SL_CUDA_TRY(cudaMemcpyAsync(&last, doc_off_in + N, 8, cudaMemcpyDeviceToHost, st));
      SL_CUDA_TRY(cudaStreamSynchronize(st));
      if (last < first) SL_FAIL(SL_EINVAL, "tokenize: document offsets must be non-decreasing");
    }
    if (first != 0) SL_FAIL(SL_EINVAL, "tokenize: doc_offsets[0] must be 0");
  }
  const uint64_t nb = last;
  if (nb && !text_in) SL_FAIL(SL_EINVAL, "tokenize: null text");
  const uint8_t* text = reinterpret_cast<const uint8_t*>(text_in);
  if (mem == SL_MEM_HOST || N == 0) {
    uint8_t* dt;
    uint64_t* doff;
    SL_TRY(scr.alloc(&dt, nb));
    SL_TRY(scr.alloc(&doff, (uint64_t)N + 1));
    if (nb) SL_CUDA_TRY(cudaMemcpyAsync(dt, text_in, nb, cudaMemcpyHostToDevice, st));
    if (N) SL_CUDA_TRY(cudaMemcpyAsync(doff, doc_off_in, ((uint64_t)N + 1) * 8, cudaMemcpyHostToDevice, st));
    else SL_CUDA_TRY(cudaMemsetAsync(doff, 0, 8, st));
    text = dt;
    doc_off = doff;
  }
  auto* tb = new sl_token_batch();
  tb->device = v->device;
  tb->N = N;
  auto fail = [&](int32_t rc) {
    if (tb->offs) cudaFreeAsync(tb->offs, st);
    if (tb->ids) cudaFreeAsync(tb->ids, st);
    cudaStreamSynchronize(st);
    delete tb;
    return rc;
  };
#define SL_TTRY(x)                      \
  do {                                  \
    const int32_t rc_ = (x);            \
    if (rc_ != SL_OK) return fail(rc_); \
  } while (0)
  if (cudaMallocAsync((void**)&tb->offs, ((uint64_t)N + 1) * 8, st) != cudaSuccess)
    return fail((set_error("tokenize: allocation failed"), SL_ENOMEM));
  // ---- segmentation
  const uint64_t nw = (nb + 31) / 32;
  uint32_t *dbits, *wbits, *sbits;
  SL_TTRY(scr.alloc(&dbits, nw));
  SL_TTRY(scr.alloc(&wbits, nw));
  SL_TTRY(scr.alloc(&sbits, nw));
  uint64_t n_tok = 0;
  uint64_t *tbeg = nullptr;
  uint32_t* tlen = nullptr;
  if (nb) {
    if (cudaMemsetAsync(dbits, 0, nw * 4, st) != cudaSuccess) return fail((set_error("memset"), SL_ECUDA));
    k_doc_marks<<<grid_for(N), 256, 0, st>>>(doc_off, N, nb, dbits); ++t_launches;
    const TextView tv{text, nb, dbits};
    if ((reinterpret_cast<uintptr_t>(text) & 15u) == 0) {
#if SL_CLASSIFY32
      k_classify32<<<grid_for(nw), 256, 0, st>>>(tv, wbits, sbits); ++t_launches;
#else
      k_classify16<<<grid_for((nb + 15) / 16), 256, 0, st>>>(tv, wbits, sbits); ++t_launches;
#endif
    } else if ((reinterpret_cast<uintptr_t>(text) & 3u) == 0) {
      k_classify4<<<grid_for((nb + 3) / 4), 256, 0, st>>>(tv, wbits, sbits); ++t_launches;
    } else {
      k_classify<<<grid_for(nw * 32), 256, 0, st>>>(tv, wbits, sbits); ++t_launches;
    }
    const uint64_t tok_tiles = (nw + kTokThreads - 1) / kTokThreads;
    uint8_t* wcnt;
    uint32_t* tok_tile;
    SL_TTRY(scr.alloc(&wcnt, nw));
    SL_TTRY(scr.alloc(&tok_tile, tok_tiles));
    k_tokens<false><<<(unsigned)tok_tiles, kTokThreads, 0, st>>>(wbits, sbits, dbits, nw, wcnt, tok_tile, nullptr,
                                                                  nullptr);
    ++t_launches;
    uint32_t tot = 0;
    SL_TTRY(exclusive_scan_u32(tok_tile, tok_tile, tok_tiles, st, &tot));
    n_tok = tot;
    SL_TTRY(scr.alloc(&tbeg, n_tok));
    SL_TTRY(scr.alloc(&tlen, n_tok));
    k_tokens<true><<<(unsigned)tok_tiles, kTokThreads, 0, st>>>(wbits, sbits, dbits, nw, wcnt, tok_tile, tbeg, tlen);
    ++t_launches;
  }
  // ---- normalisation + vocabulary probe
  std::vector<std::string> sw;
  if (cfg->stopwords && cfg->stopwords_bytes) sw = parse_stopwords(cfg->stopwords, cfg->stopwords_bytes);
  const StopTable stab = make_stop_table(sw);
  StopView sv{};
  if (stab.cap) {
    uint64_t* k;
    uint32_t *o, *l;
    uint8_t* by;
    SL_TTRY(scr.alloc(&k, stab.cap));
    SL_TTRY(scr.alloc(&o, stab.cap));
    SL_TTRY(scr.alloc(&l, stab.cap));
    SL_TTRY(scr.alloc(&by, stab.bytes.size()));
    cudaMemcpyAsync(k, stab.key.data(), stab.cap * 8ull, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(o, stab.off.data(), stab.cap * 4ull, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(l, stab.len.data(), stab.cap * 4ull, cudaMemcpyHostToDevice, st);
    if (!stab.bytes.empty()) cudaMemcpyAsync(by, stab.bytes.data(), stab.bytes.size(), cudaMemcpyHostToDevice, st);
    sv = StopView{k, o, l, by, stab.cap, stab.max_len};
  }
  uint32_t* err;
  SL_TTRY(scr.alloc(&err, 1));
  if (cudaMemsetAsync(err, 0, 4, st) != cudaSuccess) return fail((set_error("memset"), SL_ECUDA));
  // ---- distinct raw strings: entry r in first-occurrence order, tr[i] = entry of token i
  uint32_t R = 0;
  uint64_t* rbeg = nullptr;
  uint32_t* rlen = nullptr;
  uint32_t *r_flag = nullptr, *r_rank = nullptr, *r_tslot = nullptr;
  uint64_t r_cap = 0;
  if (n_tok) {
    SL_TTRY(scr.alloc(&r_tslot, n_tok));
    // sized for a Zipf vocabulary (grows 4x and retries when more than half full)
    uint64_t cap = pow2_at_least(2ull * std::min<uint64_t>(n_tok, 1ull << 19));
    uint32_t *first = nullptr, *cntr = nullptr;
    ulonglong2* key = nullptr;
    uint64_t* wrep = nullptr;
    SL_TTRY(scr.alloc(&cntr, 3));
    const bool al = (reinterpret_cast<uintptr_t>(text) & 3u) == 0;
    if (nb >> 40) return fail((set_error("tokenize: batch text beyond 2^40 bytes"), SL_EUNSUPPORTED));
    for (uint32_t seed = 0;;) {
      SL_TTRY(scr.alloc(&key, cap));
      SL_TTRY(scr.alloc(&first, cap));
      SL_TTRY(scr.alloc(&wrep, cap));
      if (cudaMemsetAsync(key, 0, cap * 16, st) != cudaSuccess || cudaMemsetAsync(first, 0xFF, cap * 4, st) != cudaSuccess ||
          cudaMemsetAsync(cntr, 0, 12, st) != cudaSuccess)
        return fail((set_error("memset"), SL_ECUDA));
      const unsigned vg = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_tok + kVerTile - 1) / kVerTile,
                                                                           8ull * text_sms()));
      if (al) {
        k_raw_insert<true><<<grid_for(n_tok), 256, 0, st>>>(text, tbeg, tlen, n_tok, key, first, wrep, (uint32_t)cap,
                                                            cntr, r_tslot, seed, v->weak);
        k_raw_verify_long<true><<<vg, 256, 0, st>>>(text, tbeg, tlen, n_tok, r_tslot, wrep, cntr);
      } else {
        k_raw_insert<false><<<grid_for(n_tok), 256, 0, st>>>(text, tbeg, tlen, n_tok, key, first, wrep, (uint32_t)cap,
                                                             cntr, r_tslot, seed, v->weak);
        k_raw_verify_long<false><<<vg, 256, 0, st>>>(text, tbeg, tlen, n_tok, r_tslot, wrep, cntr);
      }
      t_launches += 2;
      uint32_t h[3];
      SL_CUDA_TRY(cudaMemcpyAsync(h, cntr, 12, cudaMemcpyDeviceToHost, st));
      SL_CUDA_TRY(cudaStreamSynchronize(st));
      if (!h[1] && (uint64_t)h[0] * 2 <= cap && !h[2]) break;
      if (h[2] & 2u) return fail((set_error("tokenize: a token longer than 16 MiB"), SL_EUNSUPPORTED));
      if (h[2]) {  // verified collision of distinct raw strings: new hashes, same table size
        if (++seed > 8) return fail((set_error("tokenize: raw-string hash collisions persist across seeds"), SL_ECUDA));
        continue;
      }
      if (cap >= (1ull << 31)) return fail((set_error("tokenize: too many distinct tokens in one batch"), SL_EUNSUPPORTED));
      cap = std::min<uint64_t>(cap * 4, 1ull << 31);
    }
    uint32_t *sflag, *spos, *slots, *fk, *k0, *k1, *v0, *v1, *rank, *repf;
    SL_TTRY(scr.alloc(&sflag, cap));
    SL_TTRY(scr.alloc(&spos, cap));
    SL_TTRY(scr.alloc(&rank, cap));
    k_slot_flags128<<<grid_for(cap), 256, 0, st>>>(key, (uint32_t)cap, sflag); ++t_launches;
    SL_TTRY(exclusive_scan_u32(sflag, spos, cap, st, &R));
    SL_TTRY(scr.alloc(&slots, R));
    SL_TTRY(scr.alloc(&fk, R));
    SL_TTRY(scr.alloc(&k0, R));
    SL_TTRY(scr.alloc(&k1, R));
    SL_TTRY(scr.alloc(&v0, R));
    SL_TTRY(scr.alloc(&v1, R));
    SL_TTRY(scr.alloc(&repf, R));
    k_slot_list<<<grid_for(cap), 256, 0, st>>>(sflag, spos, first, (uint32_t)cap, slots, fk); ++t_launches;
    const uint32_t *fs, *ss;
    SL_TTRY(radix_sort_pairs(fk, slots, R, 32, k0, k1, v0, v1, st, &fs, &ss, 0, nullptr));
    SL_CUDA_TRY(cudaMemcpyAsync(repf, fs, R * 4ull, cudaMemcpyDeviceToDevice, st));  // first token of entry r
    k_group_rank<<<grid_for(R), 256, 0, st>>>(ss, R, rank); ++t_launches;            // slot -> r
    r_flag = sflag;
    r_rank = rank;
    r_cap = cap;
    SL_TTRY(scr.alloc(&rbeg, R));
    SL_TTRY(scr.alloc(&rlen, R));
    k_gather_u64<<<grid_for(R), 256, 0, st>>>(tbeg, repf, R, rbeg); ++t_launches;
    k_gather_u32<<<grid_for(R), 256, 0, st>>>(tlen, repf, R, rlen); ++t_launches;
  }
  // normalisation works on the R distinct raw strings ("tokens" below are raw entries)
  const uint64_t n_all = n_tok;
  NormArgs na{};
  na.t = TextView{text, nb, dbits};
  na.tbeg = rbeg;
  na.tlen = rlen;
  na.n_tok = R;
  na.lowercase = cfg->lowercase ? 1 : 0;
  na.stem = cfg->stemmer == SL_STEMMER_SNOWBALL_ENGLISH ? 1 : 0;
  na.stop = sv;
  na.voc = VocabView{v->tkey, v->tval, v->V ? v->tcap : 0u, v->offs, v->h2, v->bytes};
  na.err = err;
  na.weak = v->weak;
  const uint64_t nR = R;
  SL_TTRY(scr.alloc(&na.keep, nR));
  SL_TTRY(scr.alloc(&na.id, nR));
  SL_TTRY(scr.alloc(&na.flen, nR));
  SL_TTRY(scr.alloc(&na.h1, nR));
  SL_TTRY(scr.alloc(&na.h2, nR));
  SL_TTRY(scr.alloc(&na.long_flag, nR));
  if (build) SL_TTRY(scr.alloc(&na.arena, 2 * nb));
  if (nR) {
    k_norm_fast<<<grid_for(nR, 128), 128, 0, st>>>(na); ++t_launches;
    // deferred long tokens
    uint32_t* lpos;
    SL_TTRY(scr.alloc(&lpos, nR));
    uint32_t n_long = 0;
    SL_TTRY(exclusive_scan_u32(na.long_flag, lpos, nR, st, &n_long));
    if (n_long) {
      uint32_t* list;
      SL_TTRY(scr.alloc(&list, n_long));
      k_compact_idx<<<grid_for(nR), 256, 0, st>>>(na.long_flag, lpos, nR, list); ++t_launches;
      // per long token scratch: 5 * len + 1 bytes
      std::vector<uint64_t> so(n_long + 1, 0);
      {
        std::vector<uint32_t> lens(n_long);
        uint32_t* dl;
        SL_TTRY(scr.alloc(&dl, n_long));
        k_gather_u32<<<grid_for(n_long), 256, 0, st>>>(tlen, list, n_long, dl); ++t_launches;
        SL_CUDA_TRY(cudaMemcpyAsync(lens.data(), dl, n_long * 4ull, cudaMemcpyDeviceToHost, st));
        SL_CUDA_TRY(cudaStreamSynchronize(st));
        for (uint32_t j = 0; j < n_long; ++j) so[j + 1] = so[j] + 5ull * lens[j] + 1;
      }
      uint64_t* dso;
      uint8_t* scratch;
      SL_TTRY(scr.alloc(&dso, n_long + 1ull));
      SL_TTRY(scr.alloc(&scratch, so[n_long]));
      SL_CUDA_TRY(cudaMemcpyAsync(dso, so.data(), (n_long + 1ull) * 8, cudaMemcpyHostToDevice, st));
      k_norm_long<<<grid_for(n_long, 64), 64, 0, st>>>(na, list, n_long, dso, scratch); ++t_launches;
    }
  }
  // ---- new vocabulary entries (build mode)
  if (build && R) {
    uint32_t *nflag, *npos;
    SL_TTRY(scr.alloc(&nflag, nR));
    SL_TTRY(scr.alloc(&npos, nR));
    k_flag_to_u32<<<grid_for(nR), 256, 0, st>>>(na.keep, na.id, nR, nflag, 1); ++t_launches;
    uint32_t M = 0;
    SL_TTRY(exclusive_scan_u32(nflag, npos, nR, st, &M));
    if (M) {
      uint32_t *ntok, *slots, *fk, *k0, *k1, *v0, *v1, *elen, *epos, *cnt2;
      SL_TTRY(scr.alloc(&ntok, M));
      k_compact_idx<<<grid_for(nR), 256, 0, st>>>(nflag, npos, nR, ntok); ++t_launches;
      // distinct new strings: batch-local table keyed by 128-bit hashes, value = the smallest
      // raw-entry index (first occurrence); grows and retries on overflow; identity verified by
      // bytes (k_dedup_assign), a verified collision redoes the dedup with reseeded keys
      uint64_t cap = pow2_at_least(2ull * std::min<uint64_t>(M, 1ull << 22));
      ulonglong2* key = nullptr;
      uint32_t *first = nullptr, *rank = nullptr, *sflag = nullptr, *spos = nullptr, *gs_k = nullptr;
      uint64_t *kx, *ky;
      SL_TTRY(scr.alloc(&cnt2, 2));
      SL_TTRY(scr.alloc(&kx, M));
      SL_TTRY(scr.alloc(&ky, M));
      uint32_t G = 0;
      const uint32_t V0 = v->V;
      for (uint32_t seed = 0;; ++seed) {
        k_new_keys<<<grid_for(M), 256, 0, st>>>(ntok, M, na.h1, na.h2, na.arena, na.tbeg, na.flen, seed, na.weak, kx,
                                                ky);
        ++t_launches;
        for (;;) {
          SL_TTRY(scr.alloc(&key, cap));
          SL_TTRY(scr.alloc(&first, cap));
          if (cudaMemsetAsync(key, 0, cap * 16, st) != cudaSuccess ||
              cudaMemsetAsync(first, 0xFF, cap * 4, st) != cudaSuccess || cudaMemsetAsync(cnt2, 0, 8, st) != cudaSuccess)
            return fail((set_error("memset"), SL_ECUDA));
          k_dedup_insert<<<grid_for(M), 256, 0, st>>>(ntok, M, kx, ky, key, first, (uint32_t)cap, cnt2); ++t_launches;
          uint32_t h[2];
          SL_CUDA_TRY(cudaMemcpyAsync(h, cnt2, 8, cudaMemcpyDeviceToHost, st));
          SL_CUDA_TRY(cudaStreamSynchronize(st));
          if (!h[1] && (uint64_t)h[0] * 2 <= cap) break;
          if (cap >= (1ull << 31))
            return fail((set_error("tokenize: too many distinct tokens in one batch"), SL_EUNSUPPORTED));
          cap = std::min<uint64_t>(cap * 4, 1ull << 31);
        }
        SL_TTRY(scr.alloc(&sflag, cap));
        SL_TTRY(scr.alloc(&spos, cap));
        SL_TTRY(scr.alloc(&rank, cap));
        k_slot_flags128<<<grid_for(cap), 256, 0, st>>>(key, (uint32_t)cap, sflag); ++t_launches;
        SL_TTRY(exclusive_scan_u32(sflag, spos, cap, st, &G));
        SL_TTRY(scr.alloc(&slots, G));
        SL_TTRY(scr.alloc(&fk, G));
        SL_TTRY(scr.alloc(&k0, G));
        SL_TTRY(scr.alloc(&k1, G));
        SL_TTRY(scr.alloc(&v0, G));
        SL_TTRY(scr.alloc(&v1, G));
        SL_TTRY(scr.alloc(&elen, G));
        SL_TTRY(scr.alloc(&epos, G));
        k_slot_list<<<grid_for(cap), 256, 0, st>>>(sflag, spos, first, (uint32_t)cap, slots, fk); ++t_launches;
        // groups in first-occurrence order (document order, then position)
        const uint32_t *fs, *ss;
        SL_TTRY(radix_sort_pairs(fk, slots, G, 32, k0, k1, v0, v1, st, &fs, &ss, 0, nullptr));
        uint32_t* gs_slot;
        SL_TTRY(scr.alloc(&gs_k, G));
        SL_TTRY(scr.alloc(&gs_slot, G));
        SL_CUDA_TRY(cudaMemcpyAsync(gs_k, fs, G * 4ull, cudaMemcpyDeviceToDevice, st));     // first token per rank
        SL_CUDA_TRY(cudaMemcpyAsync(gs_slot, ss, G * 4ull, cudaMemcpyDeviceToDevice, st));  // slot per rank
        k_group_rank<<<grid_for(G), 256, 0, st>>>(gs_slot, G, rank); ++t_launches;
        if (cudaMemsetAsync(err, 0, 4, st) != cudaSuccess) return fail((set_error("memset"), SL_ECUDA));
        k_dedup_assign<<<grid_for(M), 256, 0, st>>>(ntok, M, kx, ky, na.flen, na.arena, na.tbeg, key, first, rank,
                                                    (uint32_t)cap, V0, na.id, err);
        ++t_launches;
        uint32_t h_err = 0;
        SL_CUDA_TRY(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, st));
        SL_CUDA_TRY(cudaStreamSynchronize(st));
        if (!(h_err & 4u)) break;
        if (seed >= 8) return fail((set_error("tokenize: normalised-string hash collisions persist across seeds"), SL_ECUDA));
      }
      // append strings
      k_new_entries<<<grid_for(G), 256, 0, st>>>(gs_k, G, na.flen, elen); ++t_launches;
      uint32_t ebytes = 0;
      SL_TTRY(exclusive_scan_u32(elen, epos, G, st, &ebytes));
      SL_TTRY(vocab_reserve(v, (uint64_t)V0 + G, v->bused + ebytes, st));
      k_copy_entries<<<grid_for(G), 256, 0, st>>>(gs_k, G, na.tbeg, na.flen, na.arena, epos, v->bused, V0, na.h2,
                                                  v->bytes, v->offs, v->h2); ++t_launches;
      k_table_insert<<<grid_for(G), 256, 0, st>>>(na.h1, gs_k, G, V0, v->tkey, v->tval, v->tcap, err); ++t_launches;
      v->V = V0 + G;
      v->bused += ebytes;
    }
  }
  // ---- every token takes its raw entry's id; kept flags
  uint32_t T = 0;
  uint32_t* rslot = nullptr;
  uint32_t* tile_off = nullptr;
  const uint64_t keep_tiles = (n_all + kKeepTile - 1) / kKeepTile;
  if (n_all) {
    SL_TTRY(scr.alloc(&rslot, r_cap));
    k_raw_slots<<<grid_for(r_cap), 256, 0, st>>>(r_flag, r_rank, (uint32_t)r_cap, na.keep, na.id, build ? 1 : 0, rslot);
    ++t_launches;
    SL_TTRY(scr.alloc(&tile_off, keep_tiles));
    k_keep_count<<<(unsigned)keep_tiles, kKeepThreads, 0, st>>>(r_tslot, n_all, rslot, tile_off); ++t_launches;
    SL_TTRY(exclusive_scan_u32(tile_off, tile_off, keep_tiles, st, &T));
  }
  // ---- outputs
  tb->T = T;
  if (cudaMallocAsync((void**)&tb->ids, std::max<uint64_t>(T, 1) * 4, st) != cudaSuccess)
    return fail((set_error("tokenize: allocation failed"), SL_ENOMEM));
  uint64_t* kbeg;
  SL_TTRY(scr.alloc(&kbeg, T));
  if (T) {
    k_keep_emit<<<(unsigned)keep_tiles, kKeepThreads, 0, st>>>(r_tslot, n_all, rslot, tbeg, tile_off, tb->ids, kbeg);
    ++t_launches;
  }
  k_doc_token_offsets<<<grid_for((uint64_t)N + 1), 256, 0, st>>>(doc_off, N, kbeg, T, tb->offs); ++t_launches;
  uint32_t h_err = 0;
  SL_CUDA_TRY(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, st));
  if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return fail((set_error(std::string("tokenize: CUDA failure: ") + cudaGetErrorString(cudaGetLastError())),
                 SL_ECUDA));
  if (h_err) {
    set_error("tokenize: internal table error");
    return fail(SL_ECUDA);
  }
#undef SL_TTRY
  *out = tb;
  return SL_OK;
}

}  // namespace
}  // namespace sl

using namespace sl;

extern "C" {

int32_t sl_vocab_create(int32_t device, sl_vocab** out) {
  if (!out) SL_FAIL(SL_EINVAL, "sl_vocab_create: null output");
  cudaStream_t st;
  SL_TRY(text_stream(device, &st));
  auto* v = new sl_vocab();
  v->device = device;
  if (const char* e = std::getenv("SL_TEXT_WEAK_HASH")) v->weak = *e && *e != '0';
  const int32_t rc = vocab_reserve(v, 16, 256, st);
  cudaStreamSynchronize(st);
  if (rc != SL_OK) {
    delete v;
    return rc;
  }
  *out = v;
  return SL_OK;
}

int32_t sl_vocab_destroy(sl_vocab* v) {
  if (!v) return SL_OK;
  cudaSetDevice(v->device);
  void* ps[] = {v->offs, v->h2, v->bytes, v->tkey, v->tval};
  for (void* p : ps)
    if (p) cudaFree(p);
  delete v;
  return SL_OK;
}

int32_t sl_vocab_size(const sl_vocab* v, uint32_t* size) {
  if (!v || !size) SL_FAIL(SL_EINVAL, "sl_vocab_size: null argument");
  *size = v->V;
  return SL_OK;
}

int32_t sl_vocab_export(const sl_vocab* v, uint64_t* offsets, char* bytes, uint64_t* total_bytes) {
  if (!v) SL_FAIL(SL_EINVAL, "sl_vocab_export: null vocabulary");
  SL_CUDA_TRY(cudaSetDevice(v->device));
  if (total_bytes) *total_bytes = v->bused;
  if (offsets) SL_CUDA_TRY(cudaMemcpy(offsets, v->offs, (v->V + 1ull) * 8, cudaMemcpyDeviceToHost));
  if (bytes && v->bused) SL_CUDA_TRY(cudaMemcpy(bytes, v->bytes, v->bused, cudaMemcpyDeviceToHost));
  return SL_OK;
}

int32_t sl_vocab_import(sl_vocab* v, const uint64_t* offsets, const char* bytes, uint32_t n) {
  if (!v || (n && (!offsets || !bytes))) SL_FAIL(SL_EINVAL, "sl_vocab_import: null argument");
  if (v->V) SL_FAIL(SL_EINVAL, "sl_vocab_import: vocabulary is not empty");
  if (n && offsets[0] != 0) SL_FAIL(SL_EINVAL, "sl_vocab_import: offsets[0] must be 0");
  for (uint32_t i = 0; i < n; ++i)
    if (offsets[i + 1] < offsets[i]) SL_FAIL(SL_EINVAL, "sl_vocab_import: offsets must be non-decreasing");
  cudaStream_t st;
  SL_TRY(text_stream(v->device, &st));
  const uint64_t nbytes = n ? offsets[n] : 0;
  // duplicates would make ids ambiguous (vocabulary.hpp: one id per token)
  {
    std::vector<std::string_view> s(n);
    for (uint32_t i = 0; i < n; ++i) s[i] = std::string_view(bytes + offsets[i], offsets[i + 1] - offsets[i]);
    std::sort(s.begin(), s.end());
    for (uint32_t i = 1; i < n; ++i)
      if (s[i] == s[i - 1]) SL_FAIL(SL_ECORRUPT, "sl_vocab_import: duplicate token '" + std::string(s[i]) + "'");
  }
  SL_TRY(vocab_reserve(v, std::max<uint64_t>(n, 16), std::max<uint64_t>(nbytes, 256), st));
  if (n) {
    SL_CUDA_TRY(cudaMemcpyAsync(v->offs, offsets, (n + 1ull) * 8, cudaMemcpyHostToDevice, st));
    if (nbytes) SL_CUDA_TRY(cudaMemcpyAsync(v->bytes, bytes, nbytes, cudaMemcpyHostToDevice, st));
    // h2 + table from the bytes (k_table_rehash writes the table; h2 via the same hash)
    SL_CUDA_TRY(cudaMemsetAsync(v->tkey, 0, v->tcap * 8ull, st));
    v->V = n;
    v->bused = nbytes;
    k_table_rehash<<<grid_for(n), 256, 0, st>>>(v->offs, v->bytes, n, v->tkey, v->tval, v->tcap, v->h2, v->weak);
    ++t_launches;
  }
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  SL_CUDA_TRY(cudaGetLastError());
  return SL_OK;
}

int32_t sl_tokenize(sl_vocab* vocab, const sl_tokenizer_config* cfg, int32_t build, const char* text,
                    const uint64_t* doc_offsets, uint32_t num_docs, int32_t mem, sl_token_batch** out) {
  return tokenize_impl(vocab, cfg, build, text, doc_offsets, num_docs, mem, out);
}

int32_t sl_tokenize_stream(sl_vocab* v, const sl_tokenizer_config* cfg, int32_t build, const char* text,
                           const uint64_t* off, uint32_t N, uint64_t chunk_bytes, uint64_t* out_off,
                           uint32_t* out_ids, uint64_t cap, uint64_t* num_tokens) {
  if (!v || !cfg || !num_tokens || !out_off || (N && !off)) SL_FAIL(SL_EINVAL, "tokenize_stream: null argument");
  *num_tokens = 0;
  out_off[0] = 0;
  if (N == 0) return SL_OK;
  if (off[0] != 0) SL_FAIL(SL_EINVAL, "tokenize: doc_offsets[0] must be 0");
  for (uint32_t d = 0; d < N; ++d)
    if (off[d + 1] < off[d]) SL_FAIL(SL_EINVAL, "tokenize: document offsets must be non-decreasing");
  if (off[N] && !text) SL_FAIL(SL_EINVAL, "tokenize: null text");
  if (!chunk_bytes) chunk_bytes = 256ull << 20;  // 16-64 MiB chunks: per-call overhead (~1.7 ms) dominates
  // document-aligned chunks [d_a, d_b) of about chunk_bytes
  std::vector<uint32_t> cut{0};
  while (cut.back() < N) {
    const uint32_t a = cut.back();
    const uint64_t target = off[a] + chunk_bytes;
    uint32_t b = (uint32_t)(std::upper_bound(off + a + 1, off + N + 1, target) - off) - 1;
    if (b <= a) b = a + 1;  // a document longer than a chunk travels alone
    cut.push_back(b);
  }
  const size_t K = cut.size() - 1;
  uint64_t max_bytes = 0, max_docs = 0;
  for (size_t i = 0; i < K; ++i) {
    max_bytes = std::max<uint64_t>(max_bytes, off[cut[i + 1]] - off[cut[i]]);
    max_docs = std::max<uint64_t>(max_docs, cut[i + 1] - cut[i]);
  }
  cudaStream_t st;
  SL_TRY(text_stream(v->device, &st));
  TextStream& ts = t_text_stream[v->device];
  if (!ts.h2d) SL_CUDA_TRY(cudaStreamCreateWithFlags(&ts.h2d, cudaStreamNonBlocking));
  if (!ts.d2h) SL_CUDA_TRY(cudaStreamCreateWithFlags(&ts.d2h, cudaStreamNonBlocking));
  cudaStream_t h2d = ts.h2d, d2h = ts.d2h;
  cudaEvent_t in_ready[2], out_done[2];
  for (int i = 0; i < 2; ++i) {
    SL_CUDA_TRY(cudaEventCreateWithFlags(&in_ready[i], cudaEventDisableTiming));
    SL_CUDA_TRY(cudaEventCreateWithFlags(&out_done[i], cudaEventDisableTiming));
  }
  uint8_t* dtext[2] = {nullptr, nullptr};
  uint64_t *draw[2] = {nullptr, nullptr}, *doff[2] = {nullptr, nullptr}, *dout[2] = {nullptr, nullptr};
  sl_token_batch* pending[2] = {nullptr, nullptr};
  int32_t rc = SL_OK;
  // staging buffers come from the device's stream-ordered pool (kept mapped between calls)
  auto cleanup = [&]() {
    cudaStreamSynchronize(h2d);
    cudaStreamSynchronize(d2h);
    for (int i = 0; i < 2; ++i) {
      if (pending[i]) sl_token_batch_destroy(pending[i]);
      if (dtext[i]) cudaFreeAsync(dtext[i], st);
      if (draw[i]) cudaFreeAsync(draw[i], st);
      if (doff[i]) cudaFreeAsync(doff[i], st);
      if (dout[i]) cudaFreeAsync(dout[i], st);
      cudaEventDestroy(in_ready[i]);
      cudaEventDestroy(out_done[i]);
    }
    cudaStreamSynchronize(st);
  };
  auto cuda_ok = [&](cudaError_t e, const char* what) {
    if (e == cudaSuccess) return true;
    set_error(std::string("tokenize_stream: ") + what + ": " + cudaGetErrorString(e));
    rc = e == cudaErrorMemoryAllocation ? SL_ENOMEM : SL_ECUDA;
    return false;
  };
  for (int i = 0; i < 2 && rc == SL_OK; ++i) {
    if (!cuda_ok(cudaMallocAsync(&dtext[i], std::max<uint64_t>(max_bytes, 1), st), "allocation") ||
        !cuda_ok(cudaMallocAsync(&draw[i], (max_docs + 1) * 8, st), "allocation") ||
        !cuda_ok(cudaMallocAsync(&doff[i], (max_docs + 1) * 8, st), "allocation") ||
        !cuda_ok(cudaMallocAsync(&dout[i], (max_docs + 1) * 8, st), "allocation"))
      break;
  }
  // the copy streams use the buffers only after the allocations are ordered before them
  if (rc == SL_OK) cuda_ok(cudaStreamSynchronize(st), "sync");
  // chunk i -> buffer i % 2: text bytes and the chunk's offsets rebased to its first byte
  auto issue_h2d = [&](size_t i) {
    const int bsel = (int)(i & 1);
    const uint32_t a = cut[i], b = cut[i + 1];
    const uint64_t bytes = off[b] - off[a];
    if (bytes && !cuda_ok(cudaMemcpyAsync(dtext[bsel], text + off[a], bytes, cudaMemcpyHostToDevice, h2d), "copy"))
      return;
    if (!cuda_ok(cudaMemcpyAsync(draw[bsel], off + a, (b - a + 1ull) * 8, cudaMemcpyHostToDevice, h2d), "copy"))
      return;
    k_add_u64<<<grid_for(b - a + 1ull), 256, 0, h2d>>>(draw[bsel], b - a + 1ull, 0ull - off[a], doff[bsel]);
    ++t_launches;
    cuda_ok(cudaEventRecord(in_ready[bsel], h2d), "event");
  };
  uint64_t tok_base = 0;
  const char* tenv = std::getenv("SL_STREAM_TRACE");
  const bool trace = tenv && std::atoi(tenv);
  if (rc == SL_OK) issue_h2d(0);
  for (size_t i = 0; i < K && rc == SL_OK; ++i) {
    const int bsel = (int)(i & 1);
    const uint32_t a = cut[i], b = cut[i + 1];
    // buffer (i+1)%2 was last read by chunk i-1's tokenize (finished: the call is synchronous)
    if (i + 1 < K) issue_h2d(i + 1);
    const auto tw0 = std::chrono::steady_clock::now();
    if (rc != SL_OK || !cuda_ok(cudaEventSynchronize(in_ready[bsel]), "event")) break;
    const auto tw1 = std::chrono::steady_clock::now();
    sl_token_batch* tb = nullptr;
    rc = tokenize_impl(v, cfg, build, reinterpret_cast<const char*>(dtext[bsel]), doff[bsel], b - a, SL_MEM_DEVICE,
                       &tb);
    if (rc != SL_OK) break;
    if (trace) {
      const auto tw2 = std::chrono::steady_clock::now();
      fprintf(stderr, "[stream] chunk %zu: %llu bytes, wait %.3f ms, tokenize %.3f ms\n", i,
              (unsigned long long)(off[b] - off[a]), std::chrono::duration<double, std::milli>(tw1 - tw0).count(),
              std::chrono::duration<double, std::milli>(tw2 - tw1).count());
    }
    // the batch that used this output slot two chunks ago must have been copied out
    if (pending[bsel]) {
      if (!cuda_ok(cudaEventSynchronize(out_done[bsel]), "event")) break;
      sl_token_batch_destroy(pending[bsel]);
    }
    pending[bsel] = tb;
    if (tok_base + tb->T > cap) {
      set_error("tokenize_stream: ids_capacity too small for the corpus's tokens");
      rc = SL_EINVAL;
      break;
    }
    k_add_u64<<<grid_for(b - a + 1ull), 256, 0, d2h>>>(tb->offs, b - a + 1ull, tok_base, dout[bsel]);
    ++t_launches;
    if (tb->T && !cuda_ok(cudaMemcpyAsync(out_ids + tok_base, tb->ids, tb->T * 4, cudaMemcpyDeviceToHost, d2h), "copy"))
      break;
    if (!cuda_ok(cudaMemcpyAsync(out_off + a, dout[bsel], (b - a + 1ull) * 8, cudaMemcpyDeviceToHost, d2h), "copy"))
      break;
    if (!cuda_ok(cudaEventRecord(out_done[bsel], d2h), "event")) break;
    tok_base += tb->T;
  }
  if (rc == SL_OK) cuda_ok(cudaStreamSynchronize(d2h), "sync");
  cleanup();
  if (rc == SL_OK) *num_tokens = tok_base;
  return rc;
}

int32_t sl_token_batch_info(const sl_token_batch* b, uint32_t* num_docs, uint64_t* num_tokens,
                            const uint64_t** d_offsets, const uint32_t** d_ids) {
  if (!b) SL_FAIL(SL_EINVAL, "sl_token_batch_info: null batch");
  if (num_docs) *num_docs = b->N;
  if (num_tokens) *num_tokens = b->T;
  if (d_offsets) *d_offsets = b->offs;
  if (d_ids) *d_ids = b->ids;
  return SL_OK;
}

int32_t sl_token_batch_copy(const sl_token_batch* b, uint64_t* offsets, uint32_t* ids) {
  if (!b) SL_FAIL(SL_EINVAL, "sl_token_batch_copy: null batch");
  SL_CUDA_TRY(cudaSetDevice(b->device));
  if (offsets) SL_CUDA_TRY(cudaMemcpy(offsets, b->offs, (b->N + 1ull) * 8, cudaMemcpyDeviceToHost));
  if (ids && b->T) SL_CUDA_TRY(cudaMemcpy(ids, b->ids, b->T * 4, cudaMemcpyDeviceToHost));
  return SL_OK;
}

int32_t sl_token_batch_destroy(sl_token_batch* b) {
  if (!b) return SL_OK;
  cudaSetDevice(b->device);
  if (b->offs) cudaFree(b->offs);
  if (b->ids) cudaFree(b->ids);
  delete b;
  return SL_OK;
}

int32_t sl_stem_batch(const char* words, const uint64_t* offsets, uint32_t n, int32_t device, char* out,
                      uint32_t* out_len) {
  if (n && (!words || !offsets || !out || !out_len)) SL_FAIL(SL_EINVAL, "sl_stem_batch: null argument");
  if (!n) return SL_OK;
  cudaStream_t st;
  SL_TRY(text_stream(device, &st));
  TScratch scr(st);
  const uint64_t nb = offsets[n];
  uint8_t *din, *dout, *dsh;
  uint64_t* doff;
  uint32_t* dlen;
  SL_TRY(scr.alloc(&din, nb));
  SL_TRY(scr.alloc(&dout, nb));
  SL_TRY(scr.alloc(&dsh, nb));
  SL_TRY(scr.alloc(&doff, n + 1ull));
  SL_TRY(scr.alloc(&dlen, n));
  if (nb) SL_CUDA_TRY(cudaMemcpyAsync(din, words, nb, cudaMemcpyHostToDevice, st));
  SL_CUDA_TRY(cudaMemcpyAsync(doff, offsets, (n + 1ull) * 8, cudaMemcpyHostToDevice, st));
  k_stem_batch<<<grid_for(n, 128), 128, 0, st>>>(din, doff, n, dsh, dout, dlen); ++t_launches;
  if (nb) SL_CUDA_TRY(cudaMemcpyAsync(out, dout, nb, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaMemcpyAsync(out_len, dlen, n * 4ull, cudaMemcpyDeviceToHost, st));
  SL_CUDA_TRY(cudaStreamSynchronize(st));
  SL_CUDA_TRY(cudaGetLastError());
  return SL_OK;
}

}  // extern "C"
