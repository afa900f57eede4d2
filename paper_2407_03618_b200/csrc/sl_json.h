// sl_json.h — the small JSON reader/writer the SPEC index layout needs (SPEC.md [MODULE] index,
// "External Interfaces": meta.json, vocab.json {token: id}, docs.json [external ids]).
// Host-only. Strings are UTF-8 byte strings; the writer escapes '"', '\\' and control bytes and
// passes every other byte through (like json.dump(..., ensure_ascii=False)); the reader decodes
// every escape (\uXXXX incl. surrogate pairs -> UTF-8). Numbers keep their source text, so a
// u64 (stopwords_hash) round-trips exactly.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace sl {
namespace json {

inline void escape_into(std::string& out, std::string_view s) {
  static const char* hex = "0123456789abcdef";
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      default:
        if (c < 0x20) {
          out += "\\u00";
          out += hex[c >> 4];
          out += hex[c & 15];
        } else {
          out += (char)c;
        }
    }
  }
  out += '"';
}

struct Value {
  enum Kind { kNull, kBool, kNumber, kString, kArray, kObject } kind = kNull;
  bool b = false;
  std::string text;  // number source text or decoded string
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  const Value* get(std::string_view key) const {
    if (kind != kObject) return nullptr;
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  double num() const { return std::strtod(text.c_str(), nullptr); }
  uint64_t u64() const { return std::strtoull(text.c_str(), nullptr, 10); }
};

class Parser {
 public:
  explicit Parser(std::string_view s) : s_(s) {}
  // false on any syntax error; `err` says where
  bool parse(Value& out, std::string& err) {
    ws();
    if (!value(out, 0)) {
      err = "JSON syntax error at byte " + std::to_string(p_);
      return false;
    }
    ws();
    if (p_ != s_.size()) {
      err = "trailing bytes after JSON value at byte " + std::to_string(p_);
      return false;
    }
    return true;
  }

  // top-level [string, ...] (docs.json) without building a tree
  bool string_array(std::vector<std::string>& out, std::string& err) {
    ws();
    bool ok = p_ < s_.size() && s_[p_] == '[';
    if (ok) {
      ++p_;
      ws();
      if (p_ < s_.size() && s_[p_] == ']') {
        ++p_;
      } else {
        while (ok) {
          ws();
          out.emplace_back();
          ok = str(out.back());
          ws();
          if (!ok || p_ >= s_.size()) {
            ok = false;
          } else if (s_[p_] == ',') {
            ++p_;
          } else if (s_[p_] == ']') {
            ++p_;
            break;
          } else {
            ok = false;
          }
        }
      }
    }
    ws();
    if (!ok || p_ != s_.size()) {
      err = "expected a JSON array of strings (byte " + std::to_string(p_) + ")";
      return false;
    }
    return true;
  }
  // top-level {string: unsigned integer, ...} (vocab.json) without building a tree
  bool string_u64_object(std::vector<std::pair<std::string, uint64_t>>& out, std::string& err) {
    ws();
    bool ok = p_ < s_.size() && s_[p_] == '{';
    if (ok) {
      ++p_;
      ws();
      if (p_ < s_.size() && s_[p_] == '}') {
        ++p_;
      } else {
        while (ok) {
          ws();
          out.emplace_back();
          ok = str(out.back().first);
          ws();
          ok = ok && p_ < s_.size() && s_[p_] == ':';
          if (!ok) break;
          ++p_;
          ws();
          const size_t b = p_;
          while (p_ < s_.size() && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
          ok = p_ > b && p_ - b <= 19;
          if (!ok) break;
          out.back().second = std::strtoull(std::string(s_.substr(b, p_ - b)).c_str(), nullptr, 10);
          ws();
          if (p_ >= s_.size()) {
            ok = false;
          } else if (s_[p_] == ',') {
            ++p_;
          } else if (s_[p_] == '}') {
            ++p_;
            break;
          } else {
            ok = false;
          }
        }
      }
    }
    ws();
    if (!ok || p_ != s_.size()) {
      err = "expected a JSON object of string -> id (byte " + std::to_string(p_) + ")";
      return false;
    }
    return true;
  }

 private:
  std::string_view s_;
  size_t p_ = 0;

  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\r' || s_[p_] == '\t')) ++p_;
  }
  bool lit(std::string_view w) {
    if (s_.substr(p_, w.size()) != w) return false;
    p_ += w.size();
    return true;
  }
  static void utf8(std::string& o, uint32_t cp) {
    if (cp < 0x80) {
      o += (char)cp;
    } else if (cp < 0x800) {
      o += (char)(0xC0 | (cp >> 6));
      o += (char)(0x80 | (cp & 63));
    } else if (cp < 0x10000) {
      o += (char)(0xE0 | (cp >> 12));
      o += (char)(0x80 | ((cp >> 6) & 63));
      o += (char)(0x80 | (cp & 63));
    } else {
      o += (char)(0xF0 | (cp >> 18));
      o += (char)(0x80 | ((cp >> 12) & 63));
      o += (char)(0x80 | ((cp >> 6) & 63));
      o += (char)(0x80 | (cp & 63));
    }
  }
  bool hex4(uint32_t& v) {
    if (p_ + 4 > s_.size()) return false;
    v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = s_[p_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
      else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
      else return false;
    }
    return true;
  }
  bool str(std::string& o) {
    if (p_ >= s_.size() || s_[p_] != '"') return false;
    ++p_;
    o.clear();
    while (p_ < s_.size()) {
      const char c = s_[p_++];
      if (c == '"') return true;
      if (c != '\\') {
        o += c;
        continue;
      }
      if (p_ >= s_.size()) return false;
      const char e = s_[p_++];
      switch (e) {
        case '"': o += '"'; break;
        case '\\': o += '\\'; break;
        case '/': o += '/'; break;
        case 'b': o += '\b'; break;
        case 'f': o += '\f'; break;
        case 'n': o += '\n'; break;
        case 'r': o += '\r'; break;
        case 't': o += '\t'; break;
        case 'u': {
          uint32_t cp;
          if (!hex4(cp)) return false;
          if (cp >= 0xD800 && cp < 0xDC00 && p_ + 6 <= s_.size() && s_[p_] == '\\' && s_[p_ + 1] == 'u') {
            const size_t save = p_;
            p_ += 2;
            uint32_t lo;
            if (hex4(lo) && lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            else p_ = save;
          }
          utf8(o, cp);
          break;
        }
        default: return false;
      }
    }
    return false;
  }
  bool value(Value& v, int depth) {
    if (depth > 64 || p_ >= s_.size()) return false;
    const char c = s_[p_];
    if (c == '"') {
      v.kind = Value::kString;
      return str(v.text);
    }
    if (c == '{') {
      v.kind = Value::kObject;
      ++p_;
      ws();
      if (p_ < s_.size() && s_[p_] == '}') return ++p_, true;
      while (true) {
        ws();
        std::pair<std::string, Value> kv;
        if (!str(kv.first)) return false;
        ws();
        if (p_ >= s_.size() || s_[p_] != ':') return false;
        ++p_;
        ws();
        if (!value(kv.second, depth + 1)) return false;
        v.obj.push_back(std::move(kv));
        ws();
        if (p_ < s_.size() && s_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < s_.size() && s_[p_] == '}') return ++p_, true;
        return false;
      }
    }
    if (c == '[') {
      v.kind = Value::kArray;
      ++p_;
      ws();
      if (p_ < s_.size() && s_[p_] == ']') return ++p_, true;
      while (true) {
        ws();
        v.arr.emplace_back();
        if (!value(v.arr.back(), depth + 1)) return false;
        ws();
        if (p_ < s_.size() && s_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < s_.size() && s_[p_] == ']') return ++p_, true;
        return false;
      }
    }
    if (lit("true")) return v.kind = Value::kBool, v.b = true, true;
    if (lit("false")) return v.kind = Value::kBool, v.b = false, true;
    if (lit("null")) return v.kind = Value::kNull, true;
    const size_t b = p_;
    if (p_ < s_.size() && (s_[p_] == '-' || s_[p_] == '+')) ++p_;
    while (p_ < s_.size() && ((s_[p_] >= '0' && s_[p_] <= '9') || s_[p_] == '.' || s_[p_] == 'e' || s_[p_] == 'E' ||
                              s_[p_] == '-' || s_[p_] == '+'))
      ++p_;
    if (p_ == b) return false;
    v.kind = Value::kNumber;
    v.text.assign(s_.substr(b, p_ - b));
    return true;
  }
};

}  // namespace json
}  // namespace sl
