"""Seeded synthetic workloads for BASELINE.json's configs c1..c5 (libsl_synth + device generator).

Generator decisions are pinned in SURVEY.md §8d / BASELINE.md §5. The paper's BEIR
datasets are absent, so these stand in for them with the configs' shapes, sizes and
distributions. Input generation only — not part of the measured path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


class SynthConfig(C.Structure):
    _fields_ = [
        ("num_docs", C.c_uint32),
        ("vocab", C.c_uint32),
        ("zipf_s", C.c_double),
        ("len_kind", C.c_int),
        ("len_a", C.c_double),
        ("len_b", C.c_double),
        ("len_min", C.c_uint32),
        ("len_max", C.c_uint32),
        ("n_queries", C.c_uint32),
        ("qlen_min", C.c_uint32),
        ("qlen_max", C.c_uint32),
        ("head_frac", C.c_double),
        ("head_ranks", C.c_uint32),
        ("corpus_seed", C.c_uint32),
        ("query_seed", C.c_uint32),
    ]


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def config(i: int, **overrides) -> SynthConfig:
    c = SynthConfig()
    if _lib.synth_lib().sl_synth_config_get(C.c_int(i), C.byref(c)) != 0:
        raise ValueError(f"unknown config c{i}")
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


def custom(num_docs, vocab, zipf_s, len_kind, len_a, len_b=0.0, len_min=1, len_max=2**32 - 1,
           n_queries=100, qlen_min=1, qlen_max=8, head_frac=0.0, corpus_seed=7, query_seed=8) -> SynthConfig:
    c = SynthConfig()
    c.num_docs, c.vocab, c.zipf_s = num_docs, vocab, zipf_s
    c.len_kind, c.len_a, c.len_b, c.len_min, c.len_max = len_kind, len_a, len_b, len_min, len_max
    c.n_queries, c.qlen_min, c.qlen_max = n_queries, qlen_min, qlen_max
    c.head_frac, c.head_ranks = head_frac, 64
    c.corpus_seed, c.query_seed = corpus_seed, query_seed
    return c


def zipf_cdf(cfg: SynthConfig) -> np.ndarray:
    cdf = np.empty(cfg.vocab, dtype=np.float64)
    L = _lib.synth_lib()
    L.sl_synth_zipf_cdf.argtypes = [C.c_uint32, C.c_double, C.c_void_p]
    if L.sl_synth_zipf_cdf(cfg.vocab, cfg.zipf_s, _ptr(cdf)) != 0:
        raise ValueError("zipf cdf")
    return cdf


def doc_offsets(cfg: SynthConfig, d_begin: int = 0, n: int | None = None, base: int = 0) -> np.ndarray:
    n = cfg.num_docs - d_begin if n is None else n
    off = np.empty(n + 1, dtype=np.uint64)
    L = _lib.synth_lib()
    L.sl_synth_doc_offsets.argtypes = [C.POINTER(SynthConfig), C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p]
    if L.sl_synth_doc_offsets(C.byref(cfg), d_begin, n, base, _ptr(off)) != 0:
        raise ValueError("doc offsets")
    return off


def tokens_host(cfg: SynthConfig, cdf: np.ndarray, begin: int, count: int, threads: int = 8) -> np.ndarray:
    out = np.empty(count, dtype=np.uint32)
    L = _lib.synth_lib()
    L.sl_synth_tokens.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int]
    if L.sl_synth_tokens(_ptr(cdf), cfg.vocab, cfg.corpus_seed, begin, count, _ptr(out), threads) != 0:
        raise ValueError("tokens")
    return out


def tokens_device(cfg: SynthConfig, cdf: np.ndarray, begin: int, count: int, out_ptr: int) -> None:
    """Corpus tokens [begin, begin+count) generated on the current CUDA device into out_ptr
    (bit-identical to tokens_host; libsl_synth's device generator, not the product library)."""
    e = _lib.synth_lib().sl_synth_tokens_device(_ptr(cdf), cfg.vocab, cfg.corpus_seed, int(begin), int(count), 0,
                                                out_ptr)
    if e != 0:
        raise RuntimeError(f"sl_synth_tokens_device failed (cudaError {e})")


def queries(cfg: SynthConfig, cdf: np.ndarray, q_begin: int = 0, nq: int | None = None):
    nq = cfg.n_queries - q_begin if nq is None else nq
    off = np.empty(nq + 1, dtype=np.uint64)
    tok = np.empty(max(1, nq * cfg.qlen_max), dtype=np.uint32)
    L = _lib.synth_lib()
    L.sl_synth_queries.argtypes = [C.POINTER(SynthConfig), C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                   C.c_void_p]
    if L.sl_synth_queries(C.byref(cfg), _ptr(cdf), q_begin, nq, _ptr(off), _ptr(tok)) != 0:
        raise ValueError("queries")
    return off, tok[: int(off[-1])].copy()


@dataclass
class Corpus:
    cfg: SynthConfig
    cdf: np.ndarray
    offsets: np.ndarray  # u64[N+1]
    tokens: np.ndarray | None  # u32[T] (host) or None when generated on device only


def corpus_host(cfg: SynthConfig, threads: int = 8) -> Corpus:
    cdf = zipf_cdf(cfg)
    off = doc_offsets(cfg)
    tok = tokens_host(cfg, cdf, 0, int(off[-1]), threads)
    return Corpus(cfg, cdf, off, tok)


# ---------------------------------------------------------------- text workload (t<i>)
_ON = ["", "b", "c", "d", "f", "g", "h", "j", "k", "l", "m", "n", "p", "r", "s", "t", "v", "w", "z", "bl", "br",
       "ch", "cl", "cr", "dr", "fl", "fr", "gl", "gr", "pl", "pr", "sc", "sh", "sk", "sl", "sp", "st", "str", "th",
       "tr", "wh", "qu"]
_NU = ["a", "e", "i", "o", "u", "y", "ai", "ea", "ee", "ie", "oa", "oo", "ou", "ay", "oy"]
_CO = ["", "b", "d", "g", "l", "m", "n", "p", "r", "s", "t", "x", "ck", "ll", "ng", "nt", "rd", "rt", "ss", "st"]
_SUF = ["", "", "", "", "", "s", "es", "ing", "ed", "ly", "er", "ation", "ness", "ment", "ful", "ity", "ize",
        "able", "ous", "ive", "al", "ism", "ist", "ence", "ance"]


def word_list(n: int, seed: int = 17) -> list:
    """n distinct lowercase ASCII pseudo-words (syllables + suffixes), rank order = Zipf
    rank order; none is a bundled stopword or shorter than 2 letters."""
    rng = np.random.default_rng(seed)
    stop = set()
    try:
        import os
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "stopwords_en.txt")) as f:
            stop = {w.strip() for w in f if w.strip() and not w.startswith("#")}
    except OSError:
        pass
    out, seen = [], set()
    while len(out) < n:
        m = max(1024, (n - len(out)) * 2)
        ns = rng.integers(1, 4, m)
        o = rng.integers(len(_ON), size=(m, 3))
        u = rng.integers(len(_NU), size=(m, 3))
        c = rng.integers(len(_CO), size=(m, 3))
        sfx = rng.integers(len(_SUF), size=m)
        for i in range(m):
            w = "".join(_ON[o[i, j]] + _NU[u[i, j]] + _CO[c[i, j]] for j in range(ns[i])) + _SUF[sfx[i]]
            if len(w) >= 2 and w not in seen and w not in stop:
                seen.add(w)
                out.append(w)
                if len(out) == n:
                    break
    return out


def render_text(tokens: np.ndarray, doc_off: np.ndarray, words: list, seed: int, threads: int = 16):
    """Token-id documents -> UTF-8 text: token t -> words[t] + a Philox-drawn separator, 10%
    capitalised (libsl_synth sl_synth_render_text). Returns (bytes ndarray u8, u64 offsets)."""
    enc = [w.encode("utf-8") for w in words]
    wo = np.zeros(len(enc) + 1, np.uint64)
    wo[1:] = np.cumsum([len(e) for e in enc])
    wb = np.frombuffer(b"".join(enc), np.uint8)
    tok = np.ascontiguousarray(tokens, np.uint32)
    off = np.ascontiguousarray(doc_off, np.uint64)
    N = len(off) - 1
    L = _lib.synth_lib()
    L.sl_synth_render_text.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32,
                                       C.c_uint32, C.c_void_p, C.c_void_p, C.c_int]
    toff = np.empty(N + 1, np.uint64)
    if L.sl_synth_render_text(_ptr(tok), _ptr(off), N, _ptr(wb), _ptr(wo), len(enc), seed, None, _ptr(toff),
                              threads) != 0:
        raise ValueError("render_text: token id outside the word list")
    text = np.empty(max(1, int(toff[-1])), np.uint8)
    L.sl_synth_render_text(_ptr(tok), _ptr(off), N, _ptr(wb), _ptr(wo), len(enc), seed, _ptr(text), _ptr(toff),
                           threads)
    return text[:int(toff[-1])], toff
