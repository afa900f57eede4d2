// text_oracle.cpp — CPU restatement of the reference's text pipeline (TEST INFRASTRUCTURE:
// only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load it; the product path
// never does).
//
// Restates, function by function:
//   decode_utf8          proj/src/tokenizer.cpp:52-94  (malformed byte -> U+FFFD, 1 byte)
//   is_word / to_lower   proj/src/tokenizer.cpp:12-33  (tables: csrc/sl_unicode.inc, generated
//                        by tools/gen_unicode_tables.py and pinned to the reference over every
//                        codepoint in tests/test_text_oracle.py)
//   split                proj/src/tokenizer.cpp:96-113 (maximal word runs of >= 2 codepoints)
//   pipeline             proj/src/tokenizer.cpp:115-129 (split -> stopword -> stem -> id)
//   stem                 proj/src/stemmer.cpp:29-411   (the reference's Snowball English
//                        variant, including its region rule p1 = first non-vowel after a vowel)
//   vocabulary           proj/include/sparselex/vocabulary.hpp:13-48 (first-encounter ids)
// Pinned against oracle/_ref/libref_text.so (the reference compiled in place) and the golden
// fixtures in tests/golden/text_golden.json.
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace {
#include "../paper_2407_03618_b200/csrc/sl_unicode.inc"

bool is_word(char32_t cp) {
  int lo = 0, hi = kSlWordRangeCount;  // first range with first > cp
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (kSlWordRanges[2 * mid] <= cp) lo = mid + 1; else hi = mid;
  }
  return lo > 0 && cp <= kSlWordRanges[2 * (lo - 1) + 1];
}

char32_t to_lower(char32_t cp) {
  if (cp < 0x80) return (cp >= 'A' && cp <= 'Z') ? cp + 32 : cp;
  int lo = 0, hi = kSlLowerCount;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (kSlLowerFrom[mid] < cp) lo = mid + 1; else hi = mid;
  }
  return (lo < kSlLowerCount && kSlLowerFrom[lo] == cp) ? kSlLowerTo[lo] : cp;
}

void put_utf8(std::string& o, char32_t c) {
  if (c < 0x80) {
    o += char(c);
  } else if (c < 0x800) {
    o += char(0xC0 | (c >> 6));
    o += char(0x80 | (c & 0x3F));
  } else if (c < 0x10000) {
    o += char(0xE0 | (c >> 12));
    o += char(0x80 | ((c >> 6) & 0x3F));
    o += char(0x80 | (c & 0x3F));
  } else {
    o += char(0xF0 | (c >> 18));
    o += char(0x80 | ((c >> 12) & 0x3F));
    o += char(0x80 | ((c >> 6) & 0x3F));
    o += char(0x80 | (c & 0x3F));
  }
}

// One codepoint at p (advances p); malformed -> U+FFFD consuming one byte.
char32_t next_cp(const unsigned char* s, size_t n, size_t& p) {
  const unsigned b = s[p];
  if (b < 0x80) {
    ++p;
    return b;
  }
  int len;
  char32_t c;
  if (b >= 0xC0 && b <= 0xDF) {
    len = 2;
    c = b & 0x1F;
  } else if (b >= 0xE0 && b <= 0xEF) {
    len = 3;
    c = b & 0x0F;
  } else if (b >= 0xF0 && b <= 0xF7) {
    len = 4;
    c = b & 0x07;
  } else {
    ++p;
    return 0xFFFD;
  }
  if (p + len > n) {
    ++p;
    return 0xFFFD;
  }
  for (int i = 1; i < len; ++i) {
    if ((s[p + i] & 0xC0) != 0x80) {
      ++p;
      return 0xFFFD;
    }
    c = (c << 6) | (s[p + i] & 0x3F);
  }
  const char32_t lo = len == 2 ? 0x80 : len == 3 ? 0x800 : 0x10000;
  if (c < lo || c > 0x10FFFF || (c >= 0xD800 && c <= 0xDFFF)) {
    ++p;
    return 0xFFFD;
  }
  p += len;
  return c;
}

template <class F>
void split(std::string_view text, bool lowercase, F&& emit) {
  const auto* s = reinterpret_cast<const unsigned char*>(text.data());
  std::string cur;
  size_t ncp = 0, p = 0;
  while (p < text.size()) {
    const char32_t c = next_cp(s, text.size(), p);
    if (is_word(c)) {
      put_utf8(cur, lowercase ? to_lower(c) : c);
      ++ncp;
    } else {
      if (ncp >= 2) emit(cur);
      cur.clear();
      ncp = 0;
    }
  }
  if (ncp >= 2) emit(cur);
}

// ---------------------------------------------------------------- stemmer
using U = std::u32string;

bool vowel(char32_t c) { return c == 'a' || c == 'e' || c == 'i' || c == 'o' || c == 'u' || c == 'y'; }

bool ends_with(const U& w, const char* suf) {
  const size_t m = std::strlen(suf);
  if (w.size() < m) return false;
  for (size_t i = 0; i < m; ++i)
    if (w[w.size() - m + i] != (char32_t)(unsigned char)suf[i]) return false;
  return true;
}

bool equals(const U& w, const char* s) { return w.size() == std::strlen(s) && ends_with(w, s); }

void set_tail(U& w, size_t cut, const char* rep) {  // drop `cut` codepoints, append rep
  w.resize(w.size() - cut);
  for (const char* r = rep; *r; ++r) w.push_back((char32_t)(unsigned char)*r);
}

struct Word {
  U w;
  size_t r1 = 0, r2 = 0;
  bool ymark = false;

  bool vowel_in_prefix(size_t end) const {
    for (size_t i = 0; i < end; ++i)
      if (vowel(w[i])) return true;
    return false;
  }
  bool short_syl(size_t end) const {
    if (end >= 3) {
      const char32_t a = w[end - 3], b = w[end - 2], c = w[end - 1];
      if (!vowel(c) && c != 'w' && c != 'x' && c != 'Y' && vowel(b) && !vowel(a)) return true;
    }
    return end == 2 && vowel(w[0]) && !vowel(w[1]);
  }
};

const char* kIrregular[][2] = {{"skis", "ski"},     {"skies", "sky"}, {"dying", "die"},   {"lying", "lie"},
                               {"tying", "tie"},    {"idly", "idl"},  {"gently", "gentl"}, {"ugly", "ugli"},
                               {"early", "earli"},  {"only", "onli"}, {"singly", "singl"}};
const char* kKeep[] = {"sky", "news", "howe", "atlas", "cosmos", "bias", "andes"};
const char* kStop1a[] = {"inning", "outing", "canning", "herring", "earring", "proceed", "exceed", "succeed"};

void regions(Word& x) {
  const U& w = x.w;
  const size_t n = w.size();
  x.r1 = x.r2 = n;
  size_t i = 0;
  for (const char* pre : {"gener", "commun", "arsen"}) {
    const size_t m = std::strlen(pre);
    bool ok = n >= m;
    for (size_t j = 0; ok && j < m; ++j) ok = w[j] == (char32_t)pre[j];
    if (ok) {
      i = m;
      break;
    }
  }
  if (i == 0) {
    while (i < n && !vowel(w[i])) ++i;
    while (i < n && vowel(w[i])) ++i;
    if (i == n) return;
  }
  x.r1 = i;
  while (i < n && !vowel(w[i])) ++i;
  while (i < n && vowel(w[i])) ++i;
  if (i == n) return;
  x.r2 = i;
}

// suffix rules "first listed match decides" (stemmer.cpp step_2/step_3 semantics)
struct Rule {
  const char* suf;
  const char* rep;
};

bool apply_r1_rules(Word& x, const Rule* rules, size_t n_rules) {
  for (size_t i = 0; i < n_rules; ++i) {
    if (!ends_with(x.w, rules[i].suf)) continue;
    const size_t m = std::strlen(rules[i].suf);
    if (x.w.size() - m >= x.r1) set_tail(x.w, m, rules[i].rep);
    return true;
  }
  return false;
}

void stem_u(Word& x) {
  U& w = x.w;
  // prelude
  if (!w.empty() && w[0] == '\'') w.erase(0, 1);
  if (!w.empty() && w[0] == 'y') {
    w[0] = 'Y';
    x.ymark = true;
  }
  for (size_t i = 1; i < w.size(); ++i)
    if (w[i] == 'y' && vowel(w[i - 1])) {
      w[i] = 'Y';
      x.ymark = true;
    }
  regions(x);
  // step 0
  for (const char* s : {"'s'", "'s", "'"})
    if (ends_with(w, s)) {
      w.resize(w.size() - std::strlen(s));
      break;
    }
  // step 1a
  if (ends_with(w, "sses")) {
    set_tail(w, 4, "ss");
  } else if (ends_with(w, "ied") || ends_with(w, "ies")) {
    set_tail(w, 3, w.size() >= 5 ? "i" : "ie");
  } else if (ends_with(w, "us") || ends_with(w, "ss")) {
  } else if (ends_with(w, "s")) {
    if (w.size() >= 3 && x.vowel_in_prefix(w.size() - 2)) w.pop_back();
  }
  for (const char* f : kStop1a)
    if (equals(w, f)) return;
  // step 1b
  if (ends_with(w, "eedly") || ends_with(w, "eed")) {
    const size_t m = ends_with(w, "eedly") ? 5 : 3;
    if (w.size() - m >= x.r1) set_tail(w, m, "ee");
  } else {
    size_t m = 0;
    if (ends_with(w, "ingly")) m = 5;
    else if (ends_with(w, "edly")) m = 4;
    else if (ends_with(w, "ing")) m = 3;
    else if (ends_with(w, "ed")) m = 2;
    if (m && x.vowel_in_prefix(w.size() - m)) {
      w.resize(w.size() - m);
      const size_t n = w.size();
      if (ends_with(w, "at") || ends_with(w, "bl") || ends_with(w, "iz")) {
        w.push_back('e');
      } else if (n >= 2 && w[n - 1] == w[n - 2] &&
                 std::u32string_view(U"bdfgmnprt").find(w[n - 1]) != std::u32string_view::npos) {
        w.pop_back();
      } else if (n == x.r1 && x.short_syl(n)) {
        w.push_back('e');
      }
    }
  }
  // step 1c
  if (w.size() >= 3 && (w.back() == 'y' || w.back() == 'Y') && !vowel(w[w.size() - 2])) w.back() = 'i';
  // step 2
  static const Rule k2[] = {{"ization", "ize"}, {"ational", "ate"}, {"fulness", "ful"}, {"ousness", "ous"},
                            {"iveness", "ive"}, {"tional", "tion"}, {"biliti", "ble"},  {"lessli", "less"},
                            {"entli", "ent"},   {"fulli", "ful"},   {"ation", "ate"},   {"alism", "al"},
                            {"aliti", "al"},    {"ousli", "ous"},   {"iviti", "ive"},   {"enci", "ence"},
                            {"anci", "ance"},   {"abli", "able"},   {"izer", "ize"},    {"ator", "ate"},
                            {"alli", "al"},     {"bli", "ble"}};
  if (!apply_r1_rules(x, k2, sizeof(k2) / sizeof(k2[0]))) {
    if (ends_with(w, "ogi")) {
      const size_t s = w.size() - 3;
      if (s >= x.r1 && s >= 1 && w[s - 1] == 'l') set_tail(w, 3, "og");
    } else if (ends_with(w, "li")) {
      const size_t s = w.size() - 2;
      if (s >= x.r1 && s >= 1 && std::u32string_view(U"cdeghkmnrt").find(w[s - 1]) != std::u32string_view::npos)
        w.resize(s);
    }
  }
  // step 3
  static const Rule k3[] = {{"ational", "ate"}, {"tional", "tion"}, {"alize", "al"}, {"icate", "ic"},
                            {"iciti", "ic"},    {"ical", "ic"},     {"ness", ""},    {"ful", ""}};
  if (ends_with(w, "ative")) {
    const size_t s = w.size() - 5;
    if (s >= x.r1 && s >= x.r2) w.resize(s);
  } else {
    apply_r1_rules(x, k3, sizeof(k3) / sizeof(k3[0]));
  }
  // step 4
  static const char* k4[] = {"ement", "ance", "ence", "able", "ible", "ment", "ant", "ent", "ism",
                             "ate",   "iti",  "ous",  "ive",  "ize",  "al",   "er",  "ic"};
  if (ends_with(w, "ement")) {
    if (w.size() - 5 >= x.r2) w.resize(w.size() - 5);
  } else if (ends_with(w, "ion")) {
    const size_t s = w.size() - 3;
    if (s >= x.r2 && s >= 1 && (w[s - 1] == 's' || w[s - 1] == 't')) w.resize(s);
  } else {
    for (const char* suf : k4) {
      if (!ends_with(w, suf)) continue;
      const size_t m = std::strlen(suf);
      if (w.size() - m >= x.r2) w.resize(w.size() - m);
      break;
    }
  }
  // step 5
  const size_t n = w.size();
  if (n >= 1 && w[n - 1] == 'e') {
    if (n - 1 >= x.r2 || (n - 1 >= x.r1 && !x.short_syl(n - 1))) w.pop_back();
  } else if (n >= 2 && w[n - 1] == 'l' && w[n - 2] == 'l' && n - 1 >= x.r2) {
    w.pop_back();
  }
}

// The stemmer's own decoder (stemmer.cpp:33-62) is lenient: any lead byte with the right
// number of continuation bytes is accepted (no overlong / surrogate / range check); anything
// else makes stem() return its input unchanged.
bool decode_lenient(std::string_view in, U& w) {
  const auto* s = reinterpret_cast<const unsigned char*>(in.data());
  for (size_t p = 0; p < in.size();) {
    const unsigned b = s[p];
    if (b < 0x80) {
      w.push_back(b);
      ++p;
      continue;
    }
    const int len = b >= 0xC0 && b <= 0xDF ? 2 : b >= 0xE0 && b <= 0xEF ? 3 : b >= 0xF0 && b <= 0xF7 ? 4 : 0;
    if (!len || p + len > in.size()) return false;
    char32_t v = b & (len == 2 ? 0x1F : len == 3 ? 0x0F : 0x07);
    for (int i = 1; i < len; ++i) {
      if ((s[p + i] & 0xC0) != 0x80) return false;
      v = (v << 6) | (s[p + i] & 0x3F);
    }
    w.push_back(v);
    p += len;
  }
  return true;
}

std::string stem(std::string_view word) {
  U w;
  if (!decode_lenient(word, w)) return std::string(word);
  if (w.size() <= 2) return std::string(word);
  std::string out;
  for (const auto& ir : kIrregular)
    if (equals(w, ir[0])) return ir[1];
  for (const char* k : kKeep)
    if (equals(w, k)) return k;
  Word x{w};
  stem_u(x);
  for (char32_t c : x.w) put_utf8(out, (x.ymark && c == 'Y') ? U'y' : c);
  return out;
}

// ---------------------------------------------------------------- vocabulary + pipeline
struct Vocab {
  std::unordered_map<std::string, uint32_t> ids;
  std::vector<std::string> tokens;
};

std::unordered_set<std::string> g_stop;

template <class F>
void pipeline(std::string_view text, bool lowercase, bool stop, bool stm, F&& sink) {
  split(text, lowercase, [&](const std::string& t) {
    if (stop && g_stop.count(t)) return;
    sink(stm ? stem(t) : t);
  });
}

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

extern "C" {
void orc_set_stopwords(const char* words, size_t n) {
  g_stop.clear();
  std::string cur;
  for (size_t i = 0; i <= n; ++i) {
    if (i == n || words[i] == '\n') {
      if (!cur.empty()) g_stop.insert(cur);
      cur.clear();
    } else {
      cur += words[i];
    }
  }
}

size_t orc_split_text(const char* text, size_t n, int lowercase, char* out, size_t cap) {
  std::vector<std::string> v;
  split(std::string_view(text, n), lowercase != 0, [&](const std::string& t) { v.push_back(t); });
  return join(v, out, cap);
}

size_t orc_stem(const char* word, size_t n, char* out, size_t cap) {
  const std::string s = stem(std::string_view(word, n));
  if (out && s.size() <= cap) std::memcpy(out, s.data(), s.size());
  return s.size();
}

int orc_is_word(uint32_t cp) { return is_word(cp) ? 1 : 0; }
uint32_t orc_to_lower(uint32_t cp) { return to_lower(cp); }

void* orc_vocab_new(void) { return new Vocab(); }
void orc_vocab_free(void* v) { delete static_cast<Vocab*>(v); }
uint32_t orc_vocab_size(void* v) { return (uint32_t) static_cast<Vocab*>(v)->tokens.size(); }
size_t orc_vocab_tokens(void* v, char* out, size_t cap) { return join(static_cast<Vocab*>(v)->tokens, out, cap); }

size_t orc_tokenize(void* vocab, int build, int lowercase, int stop, int stm, const char* text, size_t n,
                    uint32_t* ids, size_t cap) {
  auto* V = static_cast<Vocab*>(vocab);
  std::vector<uint32_t> r;
  pipeline(std::string_view(text, n), lowercase, stop, stm, [&](const std::string& t) {
    auto it = V->ids.find(t);
    if (it != V->ids.end()) {
      r.push_back(it->second);
    } else if (build) {
      const uint32_t id = (uint32_t)V->tokens.size();
      V->ids.emplace(t, id);
      V->tokens.push_back(t);
      r.push_back(id);
    }
  });
  if (ids && r.size() <= cap) std::memcpy(ids, r.data(), r.size() * 4);
  return r.size();
}

uint64_t orc_tokenize_corpus(void* vocab, int build, int lowercase, int stop, int stm, const char* text,
                             const uint64_t* doc_off, uint32_t n_docs, uint32_t* ids, uint64_t cap,
                             uint64_t* tok_off) {
  uint64_t total = 0;
  if (tok_off) tok_off[0] = 0;
  std::vector<uint32_t> tmp;
  for (uint32_t d = 0; d < n_docs; ++d) {
    const size_t len = doc_off[d + 1] - doc_off[d];
    tmp.resize(len / 2 + 1);  // a token spans >= 2 bytes
    const size_t m = orc_tokenize(vocab, build, lowercase, stop, stm, text + doc_off[d], len, tmp.data(), tmp.size());
    if (ids && total + m <= cap) std::memcpy(ids + total, tmp.data(), m * 4);
    total += m;
    if (tok_off) tok_off[d + 1] = total;
  }
  return total;
}
}
