"""Parity helpers shared by the GPU tests (oracle = checker only)."""
from __future__ import annotations

import numpy as np

import oracle

TOL = 1e-5  # north_star: scores within 1e-5 relative


def csr(queries):
    off = np.zeros(len(queries) + 1, np.uint64)
    off[1:] = np.cumsum([len(q) for q in queries])
    tok = np.concatenate([np.asarray(q, np.uint32) for q in queries]) if queries else np.zeros(0, np.uint32)
    return off, tok


def query_scale(exp: dict, q) -> float:
    """Upper bound of Σ|terms| for the query: absolute floor for cancellation (Robertson)."""
    s = 0.0
    for t in q:
        t = int(t)
        if t >= len(exp["df"]) or exp["df"][t] == 0:
            continue
        b, e = int(exp["indptr"][t]), int(exp["indptr"][t + 1])
        if e > b:
            s += float(np.abs(exp["values"][b:e]).max())
        s += abs(float(exp["theta"][t]))
    return s


def assert_topk_match(gpu_ids, gpu_sc, ref_ids, ref_sc, k, n_docs, full_scores_fn, scale_fn, what=""):
    """Top-k parity: ids identical except where scores tie within tolerance.

    gpu_ids/gpu_sc: [B,k] (padded 0xFFFFFFFF/-inf); ref_*: oracle [B,k] (f64).
    full_scores_fn(b) -> oracle f64 score vector of query b (only called on mismatch).
    """
    m = min(k, n_docs)
    B = gpu_ids.shape[0]
    mism = 0
    for b in range(B):
        gi, gs = gpu_ids[b, :m].astype(np.int64), gpu_sc[b, :m].astype(np.float64)
        ri, rs = ref_ids[b, :m].astype(np.int64), ref_sc[b, :m]
        tol = TOL * np.maximum(np.abs(rs), scale_fn(b)) + 1e-30
        assert np.all(np.abs(gs - rs) <= tol), f"{what} q{b}: scores differ {np.max(np.abs(gs - rs))}"
        assert np.all(gpu_ids[b, m:] == 0xFFFFFFFF) and np.all(np.isneginf(gpu_sc[b, m:])), f"{what} q{b}: padding"
        assert np.all(np.diff(gs) <= 0), f"{what} q{b}: not descending"
        if np.array_equal(gi, ri):
            continue
        mism += 1
        S = full_scores_fn(b)
        assert len(set(gi.tolist())) == m, f"{what} q{b}: duplicate ids"
        # every returned doc's true score matches the reported one
        t2 = TOL * np.maximum(np.abs(S[gi]), scale_fn(b)) + 1e-30
        assert np.all(np.abs(S[gi] - gs) <= t2), f"{what} q{b}: reported score != true score"
        # the set differs from the oracle's only inside the tie band at the k-th score
        kth = rs[-1]
        band = TOL * max(abs(kth), scale_fn(b)) + 1e-30
        assert np.all(S[gi] >= kth - band), f"{what} q{b}: returned doc below the k-th score"
        must = np.nonzero(S > kth + band)[0]
        assert set(must.tolist()) <= set(gi.tolist()), f"{what} q{b}: missed a doc above the tie band"
    return mism
