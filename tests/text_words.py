"""Seeded synthetic word / text generators for the tokenizer and stemmer parity tests and the
text bench. Words are built from syllables plus the suffixes every stemmer rule looks at, so
each step of the stemmer is exercised; no dictionary or dataset is involved."""
import numpy as np

ONSETS = ["", "b", "c", "d", "f", "g", "h", "j", "k", "l", "m", "n", "p", "r", "s", "t", "v", "w", "y", "z",
          "bl", "br", "ch", "cl", "cr", "dr", "fl", "fr", "gl", "gr", "pl", "pr", "sc", "sh", "sk", "sl", "sp",
          "st", "str", "th", "tr", "wh", "x", "qu"]
NUCLEI = ["a", "e", "i", "o", "u", "y", "ai", "ea", "ee", "ie", "oa", "oo", "ou", "ay", "oy", "ey"]
CODAS = ["", "b", "d", "g", "l", "m", "n", "p", "r", "s", "t", "x", "w", "ck", "ll", "ng", "nt", "rd", "rt",
         "ss", "st", "bb", "dd", "ff", "gg", "mm", "nn", "pp", "rr", "tt", "y"]
SUFFIXES = ["", "", "", "s", "es", "ies", "ied", "ing", "ingly", "ed", "edly", "eed", "eedly", "ly", "sses",
            "us", "ss", "ization", "ational", "fulness", "ousness", "iveness", "tional", "biliti", "lessli",
            "entli", "fulli", "ation", "alism", "aliti", "ousli", "iviti", "enci", "anci", "abli", "izer",
            "ator", "alli", "bli", "ogi", "li", "alize", "icate", "iciti", "ical", "ness", "ful", "ative",
            "ement", "ance", "ence", "able", "ible", "ment", "ant", "ent", "ism", "ate", "iti", "ous", "ive",
            "ize", "al", "er", "ic", "ion", "sion", "tion", "e", "le", "ll", "at", "bl", "iz", "y"]
PREFIXES = ["", "", "", "", "gener", "commun", "arsen", "re", "un", "y"]
SPECIAL = ["skis", "skies", "dying", "lying", "tying", "idly", "gently", "ugly", "early", "only", "singly",
           "sky", "news", "howe", "atlas", "cosmos", "bias", "andes", "inning", "outing", "canning",
           "herring", "earring", "proceed", "exceed", "succeed", "innings", "outings", "proceeds", "yes",
           "yy", "y", "ay", "eye", "sayyid", "yelling", "mayday"]
UNICODE_BITS = ["é", "ü", "ß", "ñ", "ø", "ł", "İ", "Ω", "ж", "Д", "中", "文", "ǅ", "ﬁ", "𝔘", "٣", "½", "ª"]


def make_words(n, seed=7, unicode_frac=0.05):
    rng = np.random.default_rng(seed)
    out = list(SPECIAL)
    while len(out) < n:
        w = PREFIXES[rng.integers(len(PREFIXES))]
        for _ in range(int(rng.integers(1, 4))):
            w += ONSETS[rng.integers(len(ONSETS))] + NUCLEI[rng.integers(len(NUCLEI))] + CODAS[rng.integers(len(CODAS))]
        w += SUFFIXES[rng.integers(len(SUFFIXES))]
        if rng.random() < unicode_frac:
            i = int(rng.integers(len(w) + 1))
            w = w[:i] + UNICODE_BITS[rng.integers(len(UNICODE_BITS))] + w[i:]
        out.append(w)
    return out[:n]


SEPARATORS = [" ", " ", " ", " ", ", ", ". ", "; ", " - ", "\n", "\t", "(", ")", " \"", "\" ", "'", "’", " / ",
              "!", "?", " & ", "…", " ", " 1 ", " a ", " I "]


def make_corpus(n_docs, vocab_words, mean_words=60, seed=11, zipf_s=1.1, malformed_frac=0.0, case_frac=0.1):
    """Seeded text corpus: words drawn Zipf(s) from vocab_words, random separators and
    capitalisation, optional malformed UTF-8 bytes. Returns (bytes, u64 doc byte offsets)."""
    rng = np.random.default_rng(seed)
    V = len(vocab_words)
    p = 1.0 / np.arange(1, V + 1) ** zipf_s
    p /= p.sum()
    enc = [w.encode("utf-8") for w in vocab_words]
    enc_cap = [w.capitalize().encode("utf-8") for w in vocab_words]
    seps = [s.encode("utf-8") for s in SEPARATORS]
    lens = np.maximum(0, rng.poisson(mean_words, n_docs))
    total = int(lens.sum())
    picks = rng.choice(V, size=total, p=p)
    sep_pick = rng.integers(len(seps), size=total)
    caps = rng.random(total) < case_frac
    bad = rng.random(total) < malformed_frac
    bad_bytes = [b"\xff", b"\xc3", b"\xe2\x82", b"\xed\xa0\x80", b"\xc0\xaf", b"\x80", b"\xf4\x90\x80\x80"]
    parts, off, pos, j = [], [0], 0, 0
    for d in range(n_docs):
        for _ in range(int(lens[d])):
            w = enc_cap[picks[j]] if caps[j] else enc[picks[j]]
            piece = w + seps[sep_pick[j]]
            if bad[j]:
                piece = bad_bytes[j % len(bad_bytes)] + piece
            parts.append(piece)
            pos += len(piece)
            j += 1
        off.append(pos)
    return b"".join(parts), np.array(off, dtype=np.uint64)
