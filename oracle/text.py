"""CPU ORACLE for the text pipeline — test infrastructure only (tests/, __graft_entry__.smoke(),
bench.py's CPU legs). Never imported by the product package.

Two implementations behind one interface:
  TextOracle("port")  liboracle_text.so  — our restatement (oracle/text_oracle.cpp)
  TextOracle("ref")   _ref/libref_text.so — the reference's tokenizer.cpp / stemmer.cpp /
                      unicode_tables.cpp compiled in place (pins the restatement; present
                      where /root/reference was at build time)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(_HERE, "liboracle_text.so")
REF_PATH = os.path.join(_HERE, "_ref", "libref_text.so")
STOPWORDS_EN = os.path.join(os.path.dirname(_HERE), "paper_2407_03618_b200", "data", "stopwords_en.txt")

_sz, _vp, _u32, _u64, _i = C.c_size_t, C.c_void_p, C.c_uint32, C.c_uint64, C.c_int


def _sig(prefix):
    return {
        f"{prefix}_set_stopwords": (None, [C.c_char_p, _sz]),
        f"{prefix}_split_text": (_sz, [C.c_char_p, _sz, _i, _vp, _sz]),
        f"{prefix}_stem": (_sz, [C.c_char_p, _sz, _vp, _sz]),
        f"{prefix}_vocab_new": (_vp, []),
        f"{prefix}_vocab_free": (None, [_vp]),
        f"{prefix}_vocab_size": (_u32, [_vp]),
        f"{prefix}_vocab_tokens": (_sz, [_vp, _vp, _sz]),
    }


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def bundled_stopwords() -> list:
    out = []
    with open(STOPWORDS_EN, encoding="utf-8") as f:
        for line in f:
            w = line.strip()
            if w and not w.startswith("#"):
                out.append(w)
    return out


class TextOracle:
    _cache = {}

    def __init__(self, kind: str = "port"):
        self.kind = kind
        self.p = "orc" if kind == "port" else "ref"
        if kind not in TextOracle._cache:
            path = PORT_PATH if kind == "port" else REF_PATH
            if not os.path.exists(path):
                raise RuntimeError(f"{path} missing: run `make -C oracle`")
            L = C.CDLL(path)
            for n, (r, a) in _sig(self.p).items():
                getattr(L, n).restype = r
                getattr(L, n).argtypes = a
            tok = getattr(L, f"{self.p}_tokenize")
            tok.restype = _sz
            tok.argtypes = [_vp, _i, _i, _i, _i, C.c_char_p, _sz, _vp, _sz]
            if kind == "port":
                L.orc_tokenize_corpus.restype = _u64
                L.orc_tokenize_corpus.argtypes = [_vp, _i, _i, _i, _i, C.c_char_p, _vp, _u32, _vp, _u64, _vp]
                L.orc_is_word.restype = _i
                L.orc_is_word.argtypes = [_u32]
                L.orc_to_lower.restype = _u32
                L.orc_to_lower.argtypes = [_u32]
            else:
                L.ref_tokenize_corpus.restype = _u64
                L.ref_tokenize_corpus.argtypes = [_vp, _i, _i, _i, C.c_char_p, _vp, _u32, _vp, _u64, _vp]
            blob = "\n".join(bundled_stopwords()).encode()
            getattr(L, f"{self.p}_set_stopwords")(blob, len(blob))
            TextOracle._cache[kind] = L
        self.L = TextOracle._cache[kind]

    def _f(self, name):
        return getattr(self.L, f"{self.p}_{name}")

    def split_text(self, text, lowercase=True) -> list:
        b = text.encode("utf-8") if isinstance(text, str) else bytes(text)
        n = self._f("split_text")(b, len(b), int(lowercase), None, 0)
        buf = C.create_string_buffer(n + 1)
        self._f("split_text")(b, len(b), int(lowercase), buf, n + 1)
        return [t.decode("utf-8") for t in buf.raw[:n].split(b"\n")[:-1]] if n else []

    def stem(self, word) -> bytes:
        b = word.encode("utf-8") if isinstance(word, str) else bytes(word)
        buf = C.create_string_buffer(len(b) + 8)
        n = self._f("stem")(b, len(b), buf, len(b) + 8)
        return buf.raw[:n]

    def tokenize_corpus(self, text: bytes, doc_off, lowercase=True, stop=False, stem=False, vocab=None):
        """tokenize_build over every document with one vocabulary -> (token offsets, ids, vocab tokens)."""
        off = np.ascontiguousarray(doc_off, np.uint64)
        N = len(off) - 1
        own = vocab is None
        v = self._f("vocab_new")() if own else vocab
        cap = max(1, len(text) // 2 + N)
        ids = np.empty(cap, np.uint32)
        toff = np.empty(N + 1, np.uint64)
        f = self._f("tokenize_corpus")
        if self.kind == "port":
            T = f(v, 1, int(lowercase), int(stop), int(stem), text, off.ctypes.data, N, ids.ctypes.data, cap,
                  toff.ctypes.data)
        else:
            T = f(v, int(lowercase), int(stop), int(stem), text, off.ctypes.data, N, ids.ctypes.data, cap,
                  toff.ctypes.data)
        toks = self.vocab_tokens(v)
        if own:
            self._f("vocab_free")(v)
        return toff, ids[:T].copy(), toks

    def tokenize(self, vocab, text, build, lowercase=True, stop=False, stem=False) -> list:
        b = text.encode("utf-8") if isinstance(text, str) else bytes(text)
        cap = len(b) // 2 + 1
        ids = np.empty(cap, np.uint32)
        n = self._f("tokenize")(vocab, int(build), int(lowercase), int(stop), int(stem), b, len(b), ids.ctypes.data,
                                cap)
        return ids[:n].tolist()

    def vocab_new(self):
        return self._f("vocab_new")()

    def vocab_free(self, v):
        self._f("vocab_free")(v)

    def vocab_tokens(self, v) -> list:
        n = self._f("vocab_tokens")(v, None, 0)
        buf = C.create_string_buffer(n + 1)
        self._f("vocab_tokens")(v, buf, n + 1)
        return [t.decode("utf-8") for t in buf.raw[:n].split(b"\n")[:-1]] if n else []
