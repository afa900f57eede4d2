"""Generates tests/golden/text_golden.json from the REFERENCE's own text pipeline
(oracle/_ref/libref_text.so: proj/src/tokenizer.cpp + stemmer.cpp + unicode_tables.cpp
compiled in place by oracle/Makefile). Run in the build container (needs /root/reference):

    make -C oracle && python tests/golden/make_text_golden.py

Contents:
  * "ac4": SPEC AC4 tokenizer-conformance fixture — the strings below (punctuation, Unicode
    words, 1-character words, stopwords, inflected forms, malformed UTF-8) x the four Table 2
    configurations (stopwords on/off x stemmer on/off, lowercase on) plus lowercase off;
    expected token strings per string (each string tokenized alone).
  * "stems": reference stems of 3,000 seeded synthetic words (tests/text_words.py).
  * "word_class_sha256" / "lower_sha256": digests of the reference's word-codepoint set and
    lowercase map over every codepoint (probed through split_text), so the tables can be
    checked where the reference is absent.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.text import TextOracle  # noqa: E402
from tests.text_words import make_words  # noqa: E402

AC4 = [
    "The cat is running",
    "cats, dogs; and mice!",
    "I a x y z b c",
    "Running runners ran quickly",
    "généralement les élèves étudient",
    "Straße groß ÄÖÜ",
    "naïve café résumé",
    "ΑΘΗΝΑ Ελληνικά",
    "Москва столица России",
    "中文 分词 测试",
    "hello_world foo_bar _x_",
    "123 4567 3.14159 1e10",
    "it's John's book",
    "e-mail co-operate re-enter",
    "The quick brown fox jumps over the lazy dog",
    "generously generate generation",
    "communication community communal",
    "arsenal arsenic",
    "skies dying lying tying idly gently ugly early only singly",
    "sky news howe atlas cosmos bias andes",
    "inning outing canning herring earring proceed exceed succeed",
    "happily happiness hopefully hopelessness",
    "nationalization rationalizing conditional",
    "electricity electrical electrician",
    "agreed agreement disagreeing",
    "controlling controlled controller",
    "ℌello ǅungla ﬁnance",
    "tab\tseparated\nnew line\r\nwindows",
    "emoji 😀 between words 👍ok",
    "İstanbul İZMİR",
    "ALL CAPS SHOUTING WORDS",
    "mixedCase camelCaseWord PascalCase",
    "",
    "   ",
    "a an the of and or",
    "yes yellow yielding saying buyers",
    "the THE The tHe",
    b"caf\xc3 \xffbad\xe2\x82ok \xed\xa0\x80surrogate \xc0\xafoverlong \xf4\x90\x80\x80big",
    "½ ² ª º ٣٤ ߀",
    "abcdefghijklmnopqrstuvwxyzabcdefghijklmnopqrstuvwxyzabcdefghijklmnopqrstuvwxyzabcdefghijklmnopqrstuvwxyz",
]
CONFIGS = [  # (lowercase, stopwords, stemmer)
    (True, False, False), (True, True, False), (True, False, True), (True, True, True), (False, False, False),
    (False, True, True),
]


def main():
    ref = TextOracle("ref")
    out = {"source": "oracle/_ref/libref_text.so (reference tokenizer.cpp/stemmer.cpp/unicode_tables.cpp)",
           "configs": CONFIGS, "ac4": [], "stems": []}
    for s in AC4:
        b = s if isinstance(s, bytes) else s.encode("utf-8")
        row = {"text_hex": b.hex(), "tokens": []}
        for lc, stop, stem in CONFIGS:
            v = ref.vocab_new()
            ids = ref.tokenize(v, b, True, lc, stop, stem)
            toks = ref.vocab_tokens(v)
            ref.vocab_free(v)
            row["tokens"].append([toks[i] for i in ids])
        out["ac4"].append(row)
    for w in make_words(3000, seed=3):
        out["stems"].append([w, ref.stem(w).decode("utf-8")])
    # word class + lowercase digests over every codepoint
    wc, lo = hashlib.sha256(), hashlib.sha256()
    for cp in range(0x110000):
        if 0xD800 <= cp <= 0xDFFF:
            continue
        t = ref.split_text("a" + chr(cp), True)
        if t:
            wc.update(cp.to_bytes(4, "little"))
            lo.update(cp.to_bytes(4, "little") + ord(t[0][1]).to_bytes(4, "little"))
    out["word_class_sha256"] = wc.hexdigest()
    out["lower_sha256"] = lo.hexdigest()
    with open(os.path.join(HERE, "text_golden.json"), "w", encoding="utf-8") as f:
        json.dump(out, f, ensure_ascii=False, indent=0)
    print("wrote", os.path.join(HERE, "text_golden.json"))


if __name__ == "__main__":
    main()
