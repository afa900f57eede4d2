"""BASELINE.json configs c2 / c3 / c4 at full size against the oracle, plus a c5-distribution shard
(c5 itself, with corpus-wide statistics, is tests/test_gpu_c5.py).

c2: full CSC structure bit-exact (indptr, docids, df, doclens, tf); values within 1e-5 (and counted
    for bit-identity); ALL 10,000 queries at top-10 and top-100 against the oracle's retrieve_batch.
c3: variant sweep (Robertson, ATIRE, BM25L d=.5, BM25+ d=.5) on c2's corpus — full CSC compare and
    ALL 10,000 queries at top-10, exercising the non-sparse S^θ shift path.
c4: full 1-GPU CSC and ALL 8,192 queries of batch 0 at top-1000.
Parity = ids identical except where scores tie within 1e-5 at the k-th place (tests/helpers.py).
Beyond the oracle: every query returns k distinct ids in non-increasing score order, and for every
97th query the reported scores equal the GPU's own dense score_query at those documents.
"""
import numpy as np
import pytest

import oracle
from paper_2407_03618_b200 import BM25Params, Variant, build_index, retrieve_batch, score_query, synth
from tests.helpers import TOL, assert_topk_match, query_scale

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def c2():
    cfg = synth.config(2)
    corp = synth.corpus_host(cfg, threads=16)
    qoff, qtok = synth.queries(cfg, corp.cdf)
    return cfg, corp, qoff, qtok


def _check_build(gx, ox, what):
    for key in ("indptr", "docids", "df", "doclens", "tf"):
        assert np.array_equal(gx[key], ox[key]), f"{what}: {key}"
    assert gx["avg_len"] == ox["avg_len"]
    v_o = ox["values"].astype(np.float64)
    rel = np.abs(gx["values"] - v_o) / np.maximum(np.abs(v_o), 1e-30)
    assert rel.max() <= TOL, f"{what}: values rel {rel.max()}"
    n_diff = int(np.count_nonzero(gx["values"] != ox["values"]))
    assert n_diff <= len(v_o) // 100000, f"{what}: {n_diff} values not bit-identical"
    assert np.array_equal(gx["theta"], ox["theta"]) or np.max(
        np.abs(gx["theta"] - ox["theta"]) / np.maximum(np.abs(ox["theta"]), 1e-30)) <= TOL


def _sample(qoff, qtok, n, seed):
    if n is None:  # the whole batch
        n = len(qoff) - 1
        idx = np.arange(n)
    else:
        idx = np.sort(np.random.default_rng(seed).choice(len(qoff) - 1, n, replace=False))
    qs = [qtok[int(qoff[i]):int(qoff[i + 1])] for i in idx]
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(q) for q in qs])
    return qs, off, np.concatenate(qs).astype(np.uint32)


def _run(cfg, corp, qoff, qtok, p, ks, nsample, seed):
    ox = oracle.OracleIndex(corp.offsets, corp.tokens, cfg.vocab, int(p.variant), p.k1, p.b, p.delta)
    exp = ox.export()
    qs, so, st = _sample(qoff, qtok, nsample, seed)
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p, keep_tf=True) as gi:
        _check_build(gi.export(tf=True), exp, p.variant.name)
        for k in ks:
            rid, rsc = ox.retrieve_batch(so, st, k, True, 16)
            gid, gsc = retrieve_batch(gi, (so, st), k, as_arrays=True)
            assert_topk_match(gid, gsc, rid, rsc, k, cfg.num_docs, lambda b: ox.score_query(qs[b]),
                              lambda b: query_scale(exp, qs[b]), f"{p.variant.name} k={k}")
        # full batch: structural properties + score recomputation on the device
        gid, gsc = retrieve_batch(gi, (qoff, qtok), ks[0], as_arrays=True)
        assert np.all(np.diff(gsc.astype(np.float64), axis=1) <= 0)
        srt = np.sort(gid.astype(np.int64), axis=1)
        assert np.all(np.diff(srt, axis=1) > 0)  # k distinct ids per query
        for b in range(0, len(qoff) - 1, 97):
            q = qtok[int(qoff[b]):int(qoff[b + 1])]
            s = score_query(gi, q)
            np.testing.assert_array_equal(s[gid[b].astype(np.int64)], gsc[b])


def test_c2_lucene(cuda_ok, c2):
    cfg, corp, qoff, qtok = c2
    _run(cfg, corp, qoff, qtok, BM25Params(Variant.lucene, 1.5, 0.75), (10, 100), None, 2)


@pytest.mark.parametrize("p", [BM25Params(Variant.robertson), BM25Params(Variant.atire),
                               BM25Params(Variant.bm25l, 1.5, 0.75, 0.5), BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5)],
                         ids=lambda p: p.variant.name)
def test_c3_variant_sweep(cuda_ok, c2, p):
    cfg, corp, qoff, qtok = c2  # c3 = c2's corpus shapes with the variant sweep
    _run(cfg, corp, qoff, qtok, p, (10,), None, 3)


def test_c4_csc_and_top1000(cuda_ok):
    """c4 (8.8M passages, V=1M, ~4.9e8 tokens): full 1-GPU CSC vs the oracle and top-1000 parity
    on all 8,192 queries of the first batch (SURVEY.md §8d asks for >= 512)."""
    cfg = synth.config(4)
    corp = synth.corpus_host(cfg, threads=32)
    qoff, qtok = synth.queries(cfg, corp.cdf, 0, 8192)
    _run(cfg, corp, qoff, qtok, BM25Params(Variant.lucene, 1.5, 0.75), (1000,), None, 4)


def test_c5_shard_csc_and_top100(cuda_ok):
    """c5's distribution (50M long docs, V=4M, Zipf(1.0), queries of 2-32 tokens with a 5% head
    tail) on one shard: shard 0 of a 64-way token-balanced sharding (~780k docs, ~2.6e8 tokens)
    built with shard-local statistics, full CSC vs the oracle and top-100 parity on 96 queries of
    the first batch (head-heavy queries included) — SURVEY.md §8d c5 parity plan, shard-sized."""
    cfg = synth.config(5)
    cdf = synth.zipf_cdf(cfg)
    off = synth.doc_offsets(cfg, 0, 781_250)  # the first 1/64 of the documents
    tok = synth.tokens_host(cfg, cdf, 0, int(off[-1]), threads=32)
    corp = synth.Corpus(cfg, cdf, off, tok)
    qoff, qtok = synth.queries(cfg, cdf, 0, 4096)
    n_head = sum(1 for q in range(len(qoff) - 1) if int(qoff[q + 1] - qoff[q]) and
                 int(qtok[int(qoff[q]):int(qoff[q + 1])].max()) < cfg.head_ranks)
    assert n_head > 100  # the 5% head tail is present in the batch
    sub = synth.config(5, num_docs=781_250)
    _run(sub, corp, qoff, qtok, BM25Params(Variant.lucene, 1.5, 0.75), (100,), 96, 5)
