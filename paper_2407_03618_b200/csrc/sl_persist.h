// sl_persist.h — the SPEC index directory layout (sl_persist.cu) for the token-id index and the
// text index (sl_textindex.cpp): the text index adds its vocabulary, external document ids and
// tokenizer configuration to the same nine files.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "sparselex_b200.h"

namespace sl {
struct TextMeta {
  const std::vector<std::string>* tokens = nullptr;     // vocab.json keys in id order (null: decimal ids)
  const std::vector<std::string>* ext_ids = nullptr;    // docs.json (null: global doc ids)
  const std::vector<std::string>* stopwords = nullptr;  // meta.json "stopwords" extension
  bool lowercase = false;
  int32_t stemmer = SL_STEMMER_NONE;
  uint64_t stopwords_hash = 0;  // stopwords.hpp:17-19
};
struct LoadedText {
  std::vector<std::string> tokens, ext_ids, stopwords;
  bool lowercase = false, has_hash = false;
  int32_t stemmer = SL_STEMMER_NONE;
  uint64_t stopwords_hash = 0;
};
int32_t save_index_impl(const sl_index* ix, const std::string& dir, const TextMeta* tm);
int32_t load_index_impl(const std::string& dir, int32_t device, float dense_min_density, sl_index** out,
                        LoadedText* text);
}  // namespace sl
