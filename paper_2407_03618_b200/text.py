"""Text side of the SPEC API on the device (SPEC.md [MODULE] tokenizer).

Mirrors the reference's tokenizer interface (proj/include/sparselex/tokenizer.hpp,
stemmer.hpp, stopwords.hpp, vocabulary.hpp) over the C-ABI (sl_tokenize / sl_vocab_* /
sl_stem_batch in include/sparselex_b200.h):

  TokenizerConfig(lowercase, stopwords, stemmer), TokenizerConfig.english()
  split_text(text, lowercase)            tokenizer.hpp:31-34
  tokenize_build(texts, config, vocab)   tokenizer.hpp:36-39 (vocabulary grows, first-encounter ids)
  tokenize_query(texts, config, vocab)   tokenizer.hpp:41-45 (frozen vocabulary, OOV dropped)
  stem_english(word) / stem_batch(words) stemmer.hpp:16-18
  english_stopwords(), load_stopwords(path), stopwords_hash(words)   stopwords.hpp:10-19
  Vocabulary                             vocabulary.hpp:13-48
  build_text_index(corpus, params, config) / retrieve_text(...)      SPEC build_index / retrieve

All compute runs on the GPU; the only host work is argument marshalling.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import SL_MEM_DEVICE, SL_MEM_HOST, check, lib
from .api import BM25Params, QueryResult, SearchIndex

_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")
STOPWORDS_EN = os.path.join(_DATA, "stopwords_en.txt")


class StemmerKind(enum.IntEnum):
    """stemmer.hpp:8-11."""
    none = 0
    snowball_english = 1

    @staticmethod
    def from_string(name: str) -> "StemmerKind":  # stemmer.cpp:11-16
        if name == "none":
            return StemmerKind.none
        if name in ("snowball-english", "snowball_english"):
            return StemmerKind.snowball_english
        raise ValueError(f"unknown stemmer: {name}")

    def to_string(self) -> str:
        return "none" if self == StemmerKind.none else "snowball-english"


def load_stopwords(path: str) -> frozenset:
    """stopwords.hpp:13-15: one lowercase token per line, UTF-8; blank and '#' lines ignored."""
    out = set()
    with open(path, encoding="utf-8") as f:
        for line in f:
            w = line.strip()
            if w and not w.startswith("#"):
                out.add(w)
    return frozenset(out)


def english_stopwords() -> frozenset:
    """The bundled English list (env SPARSELEX_STOPWORDS overrides the path, SPEC cmd flags)."""
    return load_stopwords(os.environ.get("SPARSELEX_STOPWORDS") or STOPWORDS_EN)


def stopwords_hash(words) -> int:
    """Order-independent hash of the set (stopwords.hpp:17-19): sum mod 2^64 of the FNV-1a-64
    of each word's UTF-8 bytes."""
    tot = 0
    for w in words:
        h = 0xCBF29CE484222325
        for b in w.encode("utf-8"):
            h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
        tot = (tot + h) & 0xFFFFFFFFFFFFFFFF
    return tot


@dataclass
class TokenizerConfig:
    """tokenizer.hpp:16-23."""
    lowercase: bool = True
    stopwords: frozenset = field(default_factory=frozenset)
    stemmer: StemmerKind = StemmerKind.none

    @staticmethod
    def english() -> "TokenizerConfig":
        return TokenizerConfig(True, english_stopwords(), StemmerKind.snowball_english)

    def to_c(self):
        blob = "\n".join(sorted(self.stopwords)).encode("utf-8")
        c = _lib.TokenizerConfig(int(bool(self.lowercase)), int(StemmerKind(self.stemmer)), blob or None, len(blob))
        return c, blob

    def to_json(self) -> dict:  # SPEC meta.json "tokenizer"
        return {"lowercase": bool(self.lowercase), "stopwords_hash": stopwords_hash(self.stopwords),
                "stemmer": StemmerKind(self.stemmer).to_string()}


def _texts_to_csr(texts):
    """list[str | bytes] -> (utf-8 bytes, u64 offsets[n+1])."""
    if isinstance(texts, tuple) and len(texts) == 2:
        return texts[0], np.ascontiguousarray(texts[1], np.uint64)
    enc = [t.encode("utf-8") if isinstance(t, str) else bytes(t) for t in texts]
    off = np.zeros(len(enc) + 1, np.uint64)
    if enc:
        off[1:] = np.cumsum([len(e) for e in enc])
    return b"".join(enc), off


class Vocabulary:
    """Device-resident token <-> id map (vocabulary.hpp:13-48); ids in first-encounter order."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().sl_vocab_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self._cache = None
        self._index = None

    @property
    def handle(self):
        if not self._h:
            raise ValueError("Vocabulary is closed")
        return self._h

    def size(self) -> int:
        n = C.c_uint32()
        check(lib().sl_vocab_size(self.handle, C.byref(n)))
        return n.value

    __len__ = size

    def tokens(self) -> list:
        n = self.size()
        if self._cache is not None and len(self._cache) == n:
            return self._cache
        off = np.empty(n + 1, np.uint64)
        tot = C.c_uint64()
        check(lib().sl_vocab_export(self.handle, None, None, C.byref(tot)))
        buf = C.create_string_buffer(max(1, tot.value))
        check(lib().sl_vocab_export(self.handle, off.ctypes.data, buf, C.byref(tot)))
        raw = buf.raw
        self._cache = [raw[off[i]:off[i + 1]].decode("utf-8") for i in range(n)]
        return self._cache

    def token(self, i: int) -> str:
        return self.tokens()[i]

    def lookup(self, token: str):
        """vocabulary.hpp:20-24: the id of a (normalised) token, or None."""
        toks = self.tokens()
        if getattr(self, "_index", None) is None or len(self._index) != len(toks):
            self._index = {t: i for i, t in enumerate(toks)}
        return self._index.get(token)

    @staticmethod
    def from_tokens(tokens, device: int = 0) -> "Vocabulary":
        v = Vocabulary(device)
        enc = [t.encode("utf-8") for t in tokens]
        off = np.zeros(len(enc) + 1, np.uint64)
        if enc:
            off[1:] = np.cumsum([len(e) for e in enc])
        blob = b"".join(enc)
        check(lib().sl_vocab_import(v.handle, off.ctypes.data, blob or b"\0", len(enc)))
        return v

    @staticmethod
    def borrowed(handle, device: int = 0) -> "Vocabulary":
        """A view of a vocabulary owned by someone else (a TextIndex): never destroyed here."""
        v = Vocabulary.__new__(Vocabulary)
        v._h, v.device, v._cache, v._index, v._owned = C.c_void_p(handle), device, None, None, False
        return v

    def close(self):
        if self._h and getattr(self, "_owned", True):
            lib().sl_vocab_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TokenBatch:
    """Tokenizer output on the device: document d's ids are ids[offsets[d]:offsets[d+1]]."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        n, t = C.c_uint32(), C.c_uint64()
        po, pi = C.c_void_p(), C.c_void_p()
        check(lib().sl_token_batch_info(self._h, C.byref(n), C.byref(t), C.byref(po), C.byref(pi)))
        self.num_docs, self.num_tokens = n.value, t.value
        self.d_offsets, self.d_ids = po.value, pi.value

    def to_numpy(self):
        off = np.empty(self.num_docs + 1, np.uint64)
        ids = np.empty(max(1, self.num_tokens), np.uint32)
        check(lib().sl_token_batch_copy(self._h, off.ctypes.data, ids.ctypes.data))
        return off, ids[:self.num_tokens]

    def lists(self):
        off, ids = self.to_numpy()
        return [ids[off[d]:off[d + 1]].tolist() for d in range(self.num_docs)]

    def close(self):
        if self._h:
            lib().sl_token_batch_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _tokenize_raw(text_ptr: int, off_ptr: int, n_docs: int, config: TokenizerConfig, vocab: Vocabulary, build: bool,
                  mem: int) -> TokenBatch:
    """sl_tokenize on raw pointers (host or device per mem): bench / zero-copy callers."""
    cfg, blob = config.to_c()
    h = C.c_void_p()
    check(lib().sl_tokenize(vocab.handle, C.byref(cfg), int(build), text_ptr, off_ptr, n_docs, mem, C.byref(h)))
    return TokenBatch(h.value)


def _tokenize(texts, config: TokenizerConfig, vocab: Vocabulary, build: bool, mem=None) -> TokenBatch:
    text, off = texts if mem == SL_MEM_DEVICE else _texts_to_csr(texts)
    cfg, blob = config.to_c()
    if mem == SL_MEM_DEVICE:  # (torch uint8 tensor, torch uint64 tensor) already on the device
        tp, op = text.data_ptr(), off.data_ptr()
        n = off.numel() - 1
    else:
        tb = np.frombuffer(text, np.uint8) if len(text) else np.zeros(1, np.uint8)
        tp, op, n = tb.ctypes.data, off.ctypes.data, len(off) - 1
        mem = SL_MEM_HOST
    h = C.c_void_p()
    check(lib().sl_tokenize(vocab.handle, C.byref(cfg), int(build), tp, op, n, mem, C.byref(h)))
    return TokenBatch(h.value)


def tokenize_build(texts, config: TokenizerConfig, vocab: Vocabulary, mem=None) -> TokenBatch:
    """tokenize_build for every text in order (the vocabulary grows in first-encounter order)."""
    return _tokenize(texts, config, vocab, True, mem)


def tokenize_query(texts, config: TokenizerConfig, vocab: Vocabulary, mem=None) -> TokenBatch:
    """tokenize_query for every text (frozen vocabulary; out-of-vocabulary tokens dropped)."""
    return _tokenize(texts, config, vocab, False, mem)


def _tokenize_stream(text, offsets, config: TokenizerConfig, vocab: Vocabulary, build: bool, chunk_bytes: int,
                     out_ids=None, out_offsets=None):
    """sl_tokenize_stream: host corpus in, host (offsets, ids) out, chunked with the copies in
    both directions overlapping the device work. text: bytes / uint8 array / pinned uint8
    torch tensor; out_* (optional, e.g. pinned): preallocated output arrays."""
    if hasattr(text, "data_ptr"):  # torch tensor in host memory
        tp, nb = text.data_ptr(), text.numel()
    else:
        tb = np.frombuffer(text, np.uint8) if not isinstance(text, np.ndarray) else text
        tp, nb = (tb.ctypes.data if tb.size else 0), tb.size
    if hasattr(offsets, "data_ptr"):  # 64-bit torch tensor in host memory (e.g. pinned)
        off_ptr, n = offsets.data_ptr(), offsets.numel() - 1
    else:
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        off_ptr, n = off.ctypes.data, len(off) - 1
    if out_offsets is None:
        out_offsets = np.empty(n + 1, np.uint64)
    if out_ids is None:
        out_ids = np.empty(max(1, nb // 2 + 1), np.uint32)  # >= 2 bytes per token
    op = out_offsets.data_ptr() if hasattr(out_offsets, "data_ptr") else out_offsets.ctypes.data
    ip = out_ids.data_ptr() if hasattr(out_ids, "data_ptr") else out_ids.ctypes.data
    cap = out_ids.numel() if hasattr(out_ids, "numel") else out_ids.size
    cfg, blob = config.to_c()
    nt = C.c_uint64()
    check(lib().sl_tokenize_stream(vocab.handle, C.byref(cfg), int(build), tp, off_ptr, n, int(chunk_bytes), op, ip,
                                   cap, C.byref(nt)))
    return out_offsets, out_ids[:nt.value]


def tokenize_build_stream(text, offsets, config: TokenizerConfig, vocab: Vocabulary, chunk_bytes: int = 256 << 20,
                          out_ids=None, out_offsets=None):
    """tokenize_build over a host corpus (text bytes + u64 doc offsets), pipelined in
    document-aligned chunks; returns host (token offsets u64[N+1], ids u32[T])."""
    return _tokenize_stream(text, offsets, config, vocab, True, chunk_bytes, out_ids, out_offsets)


def tokenize_query_stream(text, offsets, config: TokenizerConfig, vocab: Vocabulary, chunk_bytes: int = 256 << 20,
                          out_ids=None, out_offsets=None):
    """tokenize_query counterpart of tokenize_build_stream (frozen vocabulary)."""
    return _tokenize_stream(text, offsets, config, vocab, False, chunk_bytes, out_ids, out_offsets)


def split_text(text: str | bytes, lowercase: bool = True) -> list:
    """split_text (tokenizer.hpp:31-34): maximal runs of >= 2 word codepoints, in order."""
    v = Vocabulary()
    b = tokenize_build([text], TokenizerConfig(lowercase), v)
    toks = v.tokens()
    out = [toks[i] for i in b.lists()[0]]
    b.close()
    v.close()
    return out


def stem_batch(words, device: int = 0) -> list:
    """stem_english for each word (stemmer.hpp:16-18), on the device."""
    enc = [w.encode("utf-8") if isinstance(w, str) else bytes(w) for w in words]
    if not enc:
        return []
    off = np.zeros(len(enc) + 1, np.uint64)
    off[1:] = np.cumsum([len(e) for e in enc])
    blob = b"".join(enc) or b"\0"
    out = C.create_string_buffer(max(1, len(blob)))
    ln = np.empty(len(enc), np.uint32)
    check(lib().sl_stem_batch(blob, off.ctypes.data, len(enc), device, out, ln.ctypes.data))
    raw = out.raw
    res = [raw[int(off[i]):int(off[i]) + int(ln[i])] for i in range(len(enc))]
    return [r.decode("utf-8", errors="surrogateescape") if isinstance(w, str) else r for r, w in zip(res, words)]


def stem_english(word: str) -> str:
    return stem_batch([word])[0]


# ---------------------------------------------------------------- text-level index (SPEC build_index)
class TextIndex:
    """SPEC SearchIndex with its vocabulary, tokenizer config and external document ids — the
    library's sl_text_index (C++), this class only holds the handle."""

    def __init__(self, handle, device: int = 0, params: BM25Params | None = None):
        self._h = C.c_void_p(handle)
        self.device = device
        self.params = params
        L = lib()
        self.index = SearchIndex(L.sl_text_index_index(self._h), device, owned=False)
        self.vocab = Vocabulary.borrowed(L.sl_text_index_vocab(self._h), device)
        c = _lib.TokenizerConfig()
        check(L.sl_text_index_config(self._h, C.byref(c)))
        sw = C.string_at(c.stopwords, c.stopwords_bytes).decode("utf-8") if c.stopwords_bytes else ""
        self.config = TokenizerConfig(bool(c.lowercase), frozenset(w for w in sw.split("\n") if w),
                                      StemmerKind(c.stemmer))
        self._ids = None

    @property
    def handle(self):
        if not self._h:
            raise ValueError("TextIndex is closed")
        return self._h

    @property
    def num_docs(self) -> int:
        n = C.c_uint32()
        check(lib().sl_text_index_num_docs(self.handle, C.byref(n)))
        return n.value

    @property
    def doc_ids(self) -> list:
        """SearchIndex.doc_external_ids."""
        if self._ids is None:
            p, n = C.c_void_p(), C.c_uint64()
            out = []
            for d in range(self.num_docs):
                check(lib().sl_text_index_external_id(self.handle, d, C.byref(p), C.byref(n)))
                out.append(C.string_at(p, n.value).decode("utf-8", errors="surrogateescape"))
            self._ids = out
        return self._ids

    def external_ids(self, doc_indices) -> list:
        ids = self.doc_ids
        return [ids[int(d)] for d in doc_indices]

    def save(self, directory: str) -> None:
        """SPEC save_index: the 9 files with the real vocab.json, docs.json and tokenizer metadata."""
        check(lib().sl_text_index_save(self.handle, str(directory).encode()))

    def close(self) -> None:
        if self._h:
            lib().sl_text_index_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _blob(items):
    enc = [x.encode("utf-8") if isinstance(x, str) else bytes(x) for x in items]
    off = np.zeros(len(enc) + 1, np.uint64)
    if enc:
        off[1:] = np.cumsum([len(e) for e in enc])
    return b"".join(enc) or b"\0", off


def build_text_index(corpus, params: BM25Params | None = None, config: TokenizerConfig | None = None, *,
                     device: int = 0, dense_min_density: float = 0.0) -> TextIndex:
    """SPEC build_index(corpus: sequence of (external_id, text), params, tokenizer_config), in the
    library (sl_text_index_build). Errors as the SPEC: empty corpus; every document tokenizing to
    nothing ("degenerate corpus"); duplicate external ids."""
    params = params or BM25Params()
    config = config or TokenizerConfig.english()
    corpus = list(corpus)
    ids, ioff = _blob([str(c[0]) for c in corpus])
    text, toff = _blob([c[1] for c in corpus])
    cfg, keep = config.to_c()
    p = params.to_c()
    h = C.c_void_p()
    check(lib().sl_text_index_build(ids, ioff.ctypes.data, text, toff.ctypes.data, len(corpus), C.byref(p),
                                    C.byref(cfg), device, float(dense_min_density), C.byref(h)))
    return TextIndex(h.value, device, params)


def load_text_index(directory: str, *, device: int = 0, dense_min_density: float = 0.0) -> TextIndex:
    """SPEC load_index for a text index (sl_text_index_load): the stopword list is checked against
    meta.json's stopwords_hash."""
    h = C.c_void_p()
    check(lib().sl_text_index_load(str(directory).encode(), device, float(dense_min_density), C.byref(h)))
    return TextIndex(h.value, device)


def retrieve_text_batch(tindex: TextIndex, queries, k: int, ordered: bool = True, workers: int = 1):
    """SPEC retrieve_batch over query texts (sl_text_index_retrieve: tokenize_query with the index's
    config and frozen vocabulary on the device, score + top-k); each QueryResult carries the
    external ids of its documents."""
    if workers < 1:
        raise ValueError("retrieve_batch: workers must be >= 1")
    if k <= 0:
        raise ValueError("top_k: k must be >= 1")
    text, off = _blob(list(queries))
    B = len(off) - 1
    ids = np.empty((max(B, 1), k), np.uint32)
    sc = np.empty((max(B, 1), k), np.float32)
    check(lib().sl_text_index_retrieve(tindex.handle, text, off.ctypes.data, B, k, int(ordered), ids.ctypes.data,
                                       sc.ctypes.data))
    m = min(k, tindex.num_docs)
    ext = tindex.doc_ids
    return [QueryResult(ids[b, :m].copy(), sc[b, :m].copy(), [ext[int(d)] for d in ids[b, :m]]) for b in range(B)]


def retrieve_text(tindex: TextIndex, text: str, k: int, ordered: bool = True) -> QueryResult:
    """SPEC retrieve(index, text, k, ordered)."""
    return retrieve_text_batch(tindex, [text], k, ordered)[0]
