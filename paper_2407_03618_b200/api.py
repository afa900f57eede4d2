"""Host-side mirror of the reference's index/retrieval interface, over the C-ABI.

Names, argument meaning and error behaviour follow the SPEC operations:
  build_index  (SPEC [MODULE] index)       -> SearchIndex (device-resident shard)
  score_query  (SPEC [MODULE] retrieval)   -> dense |C| score vector
  top_k        (SPEC [MODULE] retrieval)   -> (doc indices, scores), ties -> smaller index
  retrieve / retrieve_batch                -> QueryResult(s)
plus BM25Params / Variant as in proj/include/sparselex/bm25.hpp:16-47.
Contract violations raise ValueError (the reference throws std::invalid_argument);
CUDA / NCCL failures raise RuntimeError. Inputs are token ids (the configs bypass text).
Arrays may be numpy (host) or torch CUDA tensors (device-resident, zero-copy).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import SL_MEM_DEVICE, SL_MEM_HOST, check, lib


class Variant(enum.IntEnum):
    """bm25.hpp:16-23 (same order)."""
    robertson = 0
    atire = 1
    lucene = 2
    bm25l = 3
    bm25plus = 4
    tfldp = 5

    @staticmethod
    def from_string(name: str) -> "Variant":  # scoring.cpp:8-16
        try:
            return Variant[name]
        except KeyError:
            raise ValueError(f"unknown BM25 variant: {name}") from None


def is_sparse_variant(v: Variant) -> bool:  # scoring.cpp:30-32
    return Variant(v) in (Variant.robertson, Variant.atire, Variant.lucene)


@dataclass
class BM25Params:
    """bm25.hpp:31-47."""
    variant: Variant = Variant.lucene
    k1: float = 1.5
    b: float = 0.75
    delta: float = 0.0

    @staticmethod
    def default_delta(v: Variant) -> float:
        return float(lib().sl_default_delta(int(v)))

    @staticmethod
    def for_variant(v: Variant, k1: float = 1.5, b: float = 0.75) -> "BM25Params":
        return BM25Params(Variant(v), k1, b, BM25Params.default_delta(v))

    def to_c(self) -> _lib.Params:
        return _lib.Params(int(self.variant), float(self.k1), float(self.b), float(self.delta))

    def validate(self) -> None:
        p = self.to_c()
        check(lib().sl_params_validate(C.byref(p)))


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _as_arg(x, dtype):
    """(pointer, mem kind, keepalive) for a numpy array or torch tensor."""
    if _is_torch(x):
        import torch
        tdt = {np.uint32: torch.uint32, np.uint64: torch.uint64, np.float32: torch.float32}[dtype]
        if x.dtype != tdt:
            raise ValueError(f"expected tensor of {tdt}, got {x.dtype}")
        if not x.is_contiguous():
            x = x.contiguous()
        return x.data_ptr(), (SL_MEM_DEVICE if x.is_cuda else SL_MEM_HOST), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data, SL_MEM_HOST, a


@dataclass
class QueryResult:
    """SPEC retrieval QueryResult: doc indices (global), exact B(Q,D) scores (descending) and, for
    a text index, the matching external ids."""
    doc_indices: np.ndarray
    scores: np.ndarray
    external_ids: list | None = None


class SearchIndex:
    """A device-resident index shard (SPEC SearchIndex minus vocabulary / external ids)."""

    def __init__(self, handle: int, device: int, comm=None, owned: bool = True):
        self._h = C.c_void_p(handle)
        self.device = device
        self.comm = comm
        self._owned = owned  # False: a view of the index inside a TextIndex

    @property
    def handle(self):
        if not self._h:
            raise ValueError("SearchIndex is closed")
        return self._h

    def info(self) -> _lib.IndexInfo:
        inf = _lib.IndexInfo()
        check(lib().sl_index_get_info(self.handle, C.byref(inf)))
        return inf

    @property
    def num_docs(self) -> int:
        return self.info().num_docs_global

    @property
    def vocab_size(self) -> int:
        return self.info().vocab_size

    @property
    def nnz(self) -> int:
        return self.info().nnz_local

    @property
    def avg_len(self) -> float:
        return self.info().avg_len

    def export(self, tf: bool = False, fields=None) -> dict:
        """Host copies of the ScoreMatrix + SearchIndex arrays (SPEC index External Interfaces);
        `fields` limits the copy to some of indptr / docids / values / df / theta / doclens."""
        inf = self.info()
        V, nnz, N = inf.vocab_size, inf.nnz_local, inf.num_docs_local
        shapes = {"indptr": (V + 1, np.uint64), "docids": (nnz, np.uint32), "values": (nnz, np.float32),
                  "df": (V, np.uint32), "theta": (V, np.float32), "doclens": (N, np.uint32)}
        want = set(shapes) if fields is None else set(fields)
        out = {key: np.empty(n, dt) for key, (n, dt) in shapes.items() if key in want}
        tfa = np.empty(nnz, np.uint32) if tf else None
        p = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        g = out.get
        check(lib().sl_index_export(self.handle, SL_MEM_HOST, p(g("indptr")), p(g("docids")), p(g("values")),
                                    p(g("df")), p(g("theta")), p(g("doclens")), p(tfa)))
        if tf:
            out["tf"] = tfa
        out["avg_len"] = inf.avg_len
        out["doc_base"] = inf.doc_base
        return out

    def save(self, directory: str) -> None:
        """SPEC save_index: the 9-file layout (meta.json, vocab.json, df/theta/indptr/docids/
        values/doclens .bin, docs.json)."""
        check(lib().sl_index_save(self.handle, str(directory).encode()))

    def close(self) -> None:
        if self._h and self._owned:
            lib().sl_index_destroy(self._h)
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


def build_index(doc_offsets, token_ids, vocab_size: int, params: BM25Params | None = None, *, device: int = 0,
                keep_tf: bool = False, dense_min_density: float = 0.0, doc_base: int = 0, num_docs: int | None = None,
                comm=None, global_stats: tuple | None = None) -> SearchIndex:
    """SPEC build_index over token ids: doc d holds token_ids[doc_offsets[d]:doc_offsets[d+1]]."""
    params = params or BM25Params()
    off_p, m1, keep1 = _as_arg(doc_offsets, np.uint64)
    tok_p, m2, keep2 = _as_arg(token_ids, np.uint32)
    if m1 != m2:
        raise ValueError("doc_offsets and token_ids must live in the same memory space")
    n = (len(keep1) - 1) if num_docs is None else num_docs
    if n < 0 or n + 1 > len(keep1):
        raise ValueError("build_index: doc_offsets must have num_docs + 1 entries")
    if m1 == SL_MEM_HOST and n >= 0 and len(keep1):
        # the library copies tokens [offsets[0], offsets[n]) from the host pointer: keep it in bounds
        o0, on = int(keep1[0]), int(keep1[n])
        if on > len(keep2) or o0 > on:
            raise ValueError("build_index: doc offsets exceed the token array (offsets[num_docs] > len(token_ids))")
    d = _lib.BuildDesc()
    d.doc_offsets, d.token_ids = off_p, tok_p
    d.num_docs, d.vocab_size, d.doc_base, d.mem = n, vocab_size, doc_base, m1
    d.params = params.to_c()
    d.device, d.keep_tf, d.dense_min_density = device, int(keep_tf), float(dense_min_density)
    d.comm = comm.handle if comm is not None else None
    if global_stats is not None:  # (df[V] summed over shards, N_global, sum_len_global)
        gdf = np.ascontiguousarray(global_stats[0], np.uint32)
        if len(gdf) != vocab_size:
            raise ValueError("global_stats df must have vocab_size entries")
        d.global_df, d.global_num_docs, d.global_total_len = gdf.ctypes.data, int(global_stats[1]), int(global_stats[2])
    h = C.c_void_p()
    check(lib().sl_index_build(C.byref(d), C.byref(h)))
    return SearchIndex(h.value, device, comm)


def load_index(directory: str, *, device: int = 0, dense_min_density: float = 0.0) -> SearchIndex:
    """SPEC load_index: validates every ScoreMatrix invariant, uploads, rebuilds query structures."""
    h = C.c_void_p()
    check(lib().sl_index_load(str(directory).encode(), device, float(dense_min_density), C.byref(h)))
    return SearchIndex(h.value, device)


def _queries_to_csr(queries):
    if isinstance(queries, tuple) and len(queries) == 2:
        return queries
    lens = [len(q) for q in queries]
    off = np.zeros(len(queries) + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    tok = np.concatenate([np.asarray(q, np.uint32) for q in queries]) if queries else np.zeros(0, np.uint32)
    return off, tok


def retrieve_batch(index: SearchIndex, queries, k: int, ordered: bool = True, workers: int = 1, *,
                   as_arrays: bool = False):
    """SPEC retrieve_batch. `queries` is a list of token-id lists or a CSR pair (offsets, tokens).

    Results are identical for any `workers` (accepted for API parity; the batch is one GPU
    launch). Returns a list of QueryResult, or (ids[B,k], scores[B,k]) with as_arrays=True
    (padded with id 0xFFFFFFFF / -inf where k exceeds the corpus).
    """
    if workers < 1:
        raise ValueError("retrieve_batch: workers must be >= 1")
    if k <= 0:
        raise ValueError("top_k: k must be >= 1")
    off, tok = _queries_to_csr(queries)
    off_p, m1, k1 = _as_arg(off, np.uint64)
    tok_p, m2, k2 = _as_arg(tok if len(tok) else np.zeros(1, np.uint32), np.uint32)
    if m1 != m2:
        raise ValueError("query offsets and tokens must live in the same memory space")
    B = len(k1) - 1
    if m1 == SL_MEM_HOST and B >= 0 and int(k1[B]) > (len(tok) if len(tok) else 0):
        raise ValueError("retrieve_batch: query offsets exceed the token array")
    if m1 == SL_MEM_DEVICE:
        import torch
        ids = torch.empty((B, k), dtype=torch.uint32, device=k1.device)
        sc = torch.empty((B, k), dtype=torch.float32, device=k1.device)
        check(lib().sl_retrieve_batch(index.handle, off_p, tok_p, B, k, int(ordered), m1, ids.data_ptr(),
                                      sc.data_ptr()))
        return ids, sc
    ids = np.empty((B, k), np.uint32)
    sc = np.empty((B, k), np.float32)
    check(lib().sl_retrieve_batch(index.handle, off_p, tok_p, B, k, int(ordered), SL_MEM_HOST, ids.ctypes.data,
                                  sc.ctypes.data))
    if as_arrays:
        return ids, sc
    m = min(k, index.num_docs)
    return [QueryResult(ids[b, :m].copy(), sc[b, :m].copy()) for b in range(B)]


def retrieve_local(index: SearchIndex, queries, k: int):
    """Per-shard half of retrieve_batch (sl_retrieve_local): this shard's best k candidate keys
    per query, u64[B, k] (0 = empty slot), and the per-query constant Σ S^θ, f64[B]. Feed the
    keys of every shard to merge_candidates (any transport in between)."""
    if k <= 0:
        raise ValueError("top_k: k must be >= 1")
    off, tok = _queries_to_csr(queries)
    off = np.ascontiguousarray(off, np.uint64)
    tok = np.ascontiguousarray(tok if len(tok) else np.zeros(1, np.uint32), np.uint32)
    B = len(off) - 1
    if B >= 0 and int(off[B]) > len(tok):
        raise ValueError("retrieve_batch: query offsets exceed the token array")
    keys = np.zeros((max(B, 0), k), np.uint64)
    qc = np.zeros(max(B, 0), np.float64)
    check(lib().sl_retrieve_local(index.handle, off.ctypes.data, tok.ctypes.data, B, k, SL_MEM_HOST,
                                  keys.ctypes.data, qc.ctypes.data))
    return keys, qc


def merge_candidates(keys, qconst, device: int = 0):
    """Rank-0 merge (sl_merge_candidates): keys u64[G, B, k] of G shards + the query constants
    -> (ids u32[B, k], scores f32[B, k]), exactly what retrieve_batch on the unsharded index returns."""
    keys = np.ascontiguousarray(keys, np.uint64)
    if keys.ndim != 3:
        raise ValueError("merge_candidates: keys must be [shards, queries, k]")
    G, B, k = keys.shape
    qc = np.ascontiguousarray(qconst, np.float64)
    if len(qc) != B:
        raise ValueError("merge_candidates: one query constant per query")
    ids = np.empty((B, k), np.uint32)
    sc = np.empty((B, k), np.float32)
    check(lib().sl_merge_candidates(keys.ctypes.data, G, B, k, qc.ctypes.data, SL_MEM_HOST, device, ids.ctypes.data,
                                    sc.ctypes.data))
    return ids, sc


def retrieve(index: SearchIndex, query_tokens, k: int, ordered: bool = True) -> QueryResult:
    """SPEC retrieve for an already tokenised query (token ids; OOV ids have df = 0 and drop)."""
    return retrieve_batch(index, [list(query_tokens)], k, ordered)[0]


def score_query(index: SearchIndex, query_tokens) -> np.ndarray:
    """SPEC score_query over the local shard: f32 |C_r| vector including Σ S^θ."""
    q = np.ascontiguousarray(np.asarray(query_tokens, np.uint32))
    out = np.empty(index.info().num_docs_local, np.float32)
    check(lib().sl_score_query(index.handle, q.ctypes.data if len(q) else None, len(q), SL_MEM_HOST,
                               out.ctypes.data))
    return out


def top_k(scores, k: int, ordered: bool = True, device: int = 0):
    """SPEC top_k on the GPU: min(k, n) best indices, score desc, ties -> smaller index."""
    if k <= 0:
        raise ValueError("top_k: k must be >= 1")
    s = np.ascontiguousarray(np.asarray(scores, np.float32))
    ids = np.empty(k, np.uint32)
    out = np.empty(k, np.float32)
    check(lib().sl_top_k(s.ctypes.data if len(s) else None, len(s), k, int(ordered), SL_MEM_HOST, device,
                         ids.ctypes.data, out.ctypes.data))
    m = min(k, len(s))
    return ids[:m], out[:m]


class Comm:
    """NCCL communicator owned by the library (one process per GPU)."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib().sl_comm_init(buf, nranks, rank, device, C.byref(h)))
        self.handle = h
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().sl_comm_unique_id(buf))
        return bytes(buf)

    def close(self):
        if self.handle:
            lib().sl_comm_destroy(self.handle)
            self.handle = None


def shard_ranges(doc_offsets: np.ndarray, nranks: int) -> list[tuple[int, int]]:
    """Contiguous document ranges balanced by token count."""
    off = np.asarray(doc_offsets, np.uint64)
    n = len(off) - 1
    total = int(off[-1] - off[0])
    bounds = [0]
    for r in range(1, nranks):
        target = int(off[0]) + (total * r) // nranks
        d = int(np.searchsorted(off, np.uint64(target), side="left"))
        bounds.append(min(max(d, bounds[-1]), n))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(nranks)]
