"""CPU ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's CPU legs).

ctypes wrappers over:
  liboracle.so            our C++ restatement of the reference path (sparselex_oracle.cpp)
  _ref/libref_scoring.so  the reference's own proj/src/scoring.cpp (pins the restatement)
Never imported by the product package paper_2407_03618_b200.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(_HERE, "liboracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libref_scoring.so")

_d, _u32, _i32, _vp, _u64 = C.c_double, C.c_uint32, C.c_int32, C.c_void_p, C.c_uint64

_SIG = {
    "orc_last_error": (C.c_char_p, []),
    "orc_build": (_i32, [_vp, _vp, _u32, _u32, _i32, _d, _d, _d, C.POINTER(_vp)]),
    "orc_build_shard": (_i32, [_vp, _vp, _u32, _u32, _i32, _d, _d, _d, _vp, _u32, _u64, C.POINTER(_vp)]),
    "orc_free": (None, [_vp]),
    "orc_nnz": (_u64, [_vp]),
    "orc_avg_len": (_d, [_vp]),
    "orc_total_len": (_u64, [_vp]),
    "orc_export": (None, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "orc_score_query": (_i32, [_vp, _vp, _u32, _vp]),
    "orc_top_k": (C.c_int64, [_vp, _u32, _u32, _i32, _vp, _vp]),
    "orc_retrieve_batch": (_i32, [_vp, _vp, _vp, _u32, _u32, _i32, _i32, _vp, _vp]),
    "orc_dense_score": (_i32, [_vp, _vp, _u32, _u32, _i32, _d, _d, _d, _vp, _u32, _vp]),
    "orc_idf": (_d, [_i32, _u32, _u32]),
    "orc_tf_component": (_d, [_d, _d, _d, _i32, _d, _d, _d]),
    "orc_score": (_d, [_d, _u32, _d, _u32, _d, _i32, _d, _d, _d]),
    "orc_nonoccurrence": (_d, [_u32, _u32, _i32, _d, _d, _d]),
    "orc_validate": (_i32, [_i32, _d, _d, _d]),
    "orc_stream_df": (_i32, [_vp, _vp, _u32, _u32, _i32, _vp, _vp]),
    "orc_stream_rows": (_i32, [_vp, _vp, _u32, _u32, _vp, _u32, _vp, _u32, _d, _i32, _d, _d, _d, _i32, _vp, _vp, _vp,
                               _vp]),
    "orc_stream_topk": (_i32, [_vp, _vp, _u32, _u32, _u32, _vp, _vp, _u32, _vp, _u32, _d, _i32, _d, _d, _d, _u32,
                               _i32, _vp, _vp]),
}
_REF_SIG = {
    "ref_last_error": (C.c_char_p, []),
    "ref_idf": (_d, [_i32, _u32, _u32]),
    "ref_tf_component": (_d, [_d, _d, _d, _i32, _d, _d, _d]),
    "ref_score": (_d, [_d, _u32, _d, _u32, _d, _i32, _d, _d, _d]),
    "ref_nonoccurrence": (_d, [_u32, _u32, _i32, _d, _d, _d]),
    "ref_validate": (_i32, [_i32, _d, _d, _d]),
    "ref_default_delta": (_d, [_i32]),
    "ref_is_sparse": (_i32, [_i32]),
}

_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_PATH):
            raise RuntimeError(f"{ORACLE_PATH} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_PATH)
        for n, (r, a) in _SIG.items():
            getattr(L, n).restype = r
            getattr(L, n).argtypes = a
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        L = C.CDLL(REF_PATH)
        for n, (r, a) in _REF_SIG.items():
            getattr(L, n).restype = r
            getattr(L, n).argtypes = a
        _ref = L
    return _ref


def _err() -> str:
    return lib().orc_last_error().decode()


def _p(a):
    return None if a is None else a.ctypes.data


class OracleIndex:
    """SPEC build_index restated on the CPU (two-pass, f64 math, f32 storage)."""

    def __init__(self, offsets, tokens, vocab_size, variant=2, k1=1.5, b=0.75, delta=0.0, global_stats=None):
        self.offsets = np.ascontiguousarray(offsets, np.uint64)
        self.tokens = np.ascontiguousarray(tokens, np.uint32)
        self.N = len(self.offsets) - 1
        self.V = vocab_size
        self.params = (int(variant), float(k1), float(b), float(delta))
        h = _vp()
        tok = self.tokens if len(self.tokens) else np.zeros(1, np.uint32)
        if global_stats is None:
            rc = lib().orc_build(_p(self.offsets), _p(tok), self.N, vocab_size, *self.params, C.byref(h))
        else:  # shard of a document-sharded corpus: (global df[V], N_global, sum_len_global)
            self._gdf = np.ascontiguousarray(global_stats[0], np.uint32)
            rc = lib().orc_build_shard(_p(self.offsets), _p(tok), self.N, vocab_size, *self.params, _p(self._gdf),
                                       int(global_stats[1]), int(global_stats[2]), C.byref(h))
        if rc:
            raise ValueError(_err())
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_free(self._h)
            self._h = None

    @property
    def nnz(self) -> int:
        return lib().orc_nnz(self._h)

    @property
    def avg_len(self) -> float:
        return lib().orc_avg_len(self._h)

    def export(self) -> dict:
        nnz, V, N = self.nnz, self.V, self.N
        out = {"indptr": np.empty(V + 1, np.uint64), "docids": np.empty(nnz, np.uint32),
               "values": np.empty(nnz, np.float32), "df": np.empty(V, np.uint32), "theta": np.empty(V, np.float32),
               "doclens": np.empty(N, np.uint32), "tf": np.empty(nnz, np.uint32)}
        lib().orc_export(self._h, _p(out["indptr"]), _p(out["docids"]), _p(out["values"]), _p(out["df"]),
                         _p(out["theta"]), _p(out["doclens"]), _p(out["tf"]))
        out["avg_len"] = self.avg_len
        return out

    def score_query(self, q) -> np.ndarray:
        q = np.ascontiguousarray(q, np.uint32)
        out = np.empty(self.N, np.float64)
        if lib().orc_score_query(self._h, _p(q) if len(q) else None, len(q), _p(out)):
            raise ValueError(_err())
        return out

    def retrieve_batch(self, q_offsets, q_tokens, k, ordered=True, workers=1):
        off = np.ascontiguousarray(q_offsets, np.uint64)
        tok = np.ascontiguousarray(q_tokens, np.uint32)
        if len(tok) == 0:
            tok = np.zeros(1, np.uint32)
        B = len(off) - 1
        ids = np.empty((B, k), np.uint32)
        sc = np.empty((B, k), np.float64)
        if lib().orc_retrieve_batch(self._h, _p(off), _p(tok), B, k, int(ordered), workers, _p(ids), _p(sc)):
            raise ValueError(_err())
        return ids, sc


def top_k(scores, k, ordered=True):
    s = np.ascontiguousarray(scores, np.float64)
    ids = np.empty(max(k, 1), np.uint32)
    out = np.empty(max(k, 1), np.float64)
    m = lib().orc_top_k(_p(s) if len(s) else None, len(s), k, int(ordered), _p(ids), _p(out))
    if m < 0:
        raise ValueError(_err())
    return ids[:m], out[:m]


def dense_score(offsets, tokens, vocab_size, q, variant=2, k1=1.5, b=0.75, delta=0.0) -> np.ndarray:
    off = np.ascontiguousarray(offsets, np.uint64)
    tok = np.ascontiguousarray(tokens, np.uint32)
    q = np.ascontiguousarray(q, np.uint32)
    N = len(off) - 1
    out = np.empty(N, np.float64)
    rc = lib().orc_dense_score(_p(off), _p(tok) if len(tok) else None, N, vocab_size, variant, k1, b, delta,
                               _p(q) if len(q) else None, len(q), _p(out))
    if rc:
        raise ValueError(_err())
    return out


def idf(v, df, n):
    return lib().orc_idf(v, df, n)


def tf_component(tf, dl, avg, v, k1=1.5, b=0.75, delta=0.0):
    return lib().orc_tf_component(tf, dl, avg, v, k1, b, delta)


def score(tf, df, dl, n, avg, v, k1=1.5, b=0.75, delta=0.0):
    return lib().orc_score(tf, df, dl, n, avg, v, k1, b, delta)


def nonoccurrence(df, n, v, k1=1.5, b=0.75, delta=0.0):
    return lib().orc_nonoccurrence(df, n, v, k1, b, delta)


# ---- streaming checks (corpora too large for OracleIndex: c5) ----
def stream_df(offsets, tokens, V, threads=16, df=None):
    """DF by streaming count over one shard (added into `df`, u64[V]); returns (df, Σ|D|)."""
    off = np.ascontiguousarray(offsets, np.uint64)
    tok = np.ascontiguousarray(tokens, np.uint32)
    df = np.zeros(V, np.uint64) if df is None else df
    tot = C.c_uint64(0)
    if lib().orc_stream_df(_p(off), _p(tok) if len(tok) else None, len(off) - 1, V, threads, _p(df), C.byref(tot)):
        raise ValueError(_err())
    return df, tot.value


def stream_rows(offsets, tokens, V, sel, global_stats, variant=2, k1=1.5, b=0.75, delta=0.0, threads=16):
    """Rows `sel` of a shard's score matrix from its tokens with global statistics
    (gdf[V], N_global, avg_len): dict token -> (docs u32, tf u32, values f32)."""
    off = np.ascontiguousarray(offsets, np.uint64)
    tok = np.ascontiguousarray(tokens, np.uint32)
    sel = np.ascontiguousarray(sel, np.uint32)
    gdf = np.ascontiguousarray(global_stats[0], np.uint32)
    args = (_p(off), _p(tok), len(off) - 1, V, _p(sel), len(sel), _p(gdf), int(global_stats[1]),
            float(global_stats[2]), variant, k1, b, delta, threads)
    ro = np.zeros(len(sel) + 1, np.uint64)
    if lib().orc_stream_rows(*args, _p(ro), None, None, None):
        raise ValueError(_err())
    n = int(ro[-1])
    docs, tfs, vals = np.empty(max(n, 1), np.uint32), np.empty(max(n, 1), np.uint32), np.empty(max(n, 1), np.float32)
    if lib().orc_stream_rows(*args, _p(ro), _p(docs), _p(tfs), _p(vals)):
        raise ValueError(_err())
    return {int(t): (docs[ro[i]:ro[i + 1]], tfs[ro[i]:ro[i + 1]], vals[ro[i]:ro[i + 1]]) for i, t in enumerate(sel)}


def stream_topk(offsets, tokens, V, doc_base, q_offsets, q_tokens, global_stats, k, variant=2, k1=1.5, b=0.75,
                delta=0.0, threads=16):
    """Streaming naive dense scorer over one shard: best k (global ids, f64 B(Q,D)) per query,
    global statistics (gdf[V], N_global, avg_len)."""
    off = np.ascontiguousarray(offsets, np.uint64)
    tok = np.ascontiguousarray(tokens, np.uint32)
    qo = np.ascontiguousarray(q_offsets, np.uint64)
    qt = np.ascontiguousarray(q_tokens if len(q_tokens) else np.zeros(1), np.uint32)
    gdf = np.ascontiguousarray(global_stats[0], np.uint32)
    B = len(qo) - 1
    ids = np.empty((B, k), np.uint32)
    sc = np.empty((B, k), np.float64)
    if lib().orc_stream_topk(_p(off), _p(tok), len(off) - 1, doc_base, V, _p(qo), _p(qt), B, _p(gdf),
                             int(global_stats[1]), float(global_stats[2]), variant, k1, b, delta, k, threads, _p(ids),
                             _p(sc)):
        raise ValueError(_err())
    return ids, sc
