"""GPU parity: CUDA path (through the C-ABI) vs the CPU oracle on the same seeded inputs.

Bar (north_star): TF/DF counts, CSC structure and doc ids bit-exact; values and scores
within 1e-5 relative; top-k ids identical except where scores tie within 1e-5.
"""
import numpy as np
import pytest

import oracle
from paper_2407_03618_b200 import BM25Params, Variant, build_index, retrieve_batch, score_query, synth, top_k
from tests.helpers import TOL, assert_topk_match, csr, query_scale

pytestmark = pytest.mark.gpu

VARIANTS = [
    BM25Params(Variant.lucene, 1.5, 0.75, 0.0),
    BM25Params(Variant.robertson, 1.5, 0.75, 0.0),
    BM25Params(Variant.atire, 1.5, 0.75, 0.0),
    BM25Params(Variant.bm25l, 1.5, 0.75, 0.5),
    BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5),
    BM25Params(Variant.bm25plus, 1.5, 0.75, 1.0),
    BM25Params(Variant.tfldp, 1.5, 0.75, 0.5),
]


@pytest.fixture(scope="module")
def c1():
    cfg = synth.config(1)
    corp = synth.corpus_host(cfg)
    qoff, qtok = synth.queries(cfg, corp.cdf)
    return cfg, corp, qoff, qtok


def _oracle(corp, V, p):
    return oracle.OracleIndex(corp.offsets, corp.tokens, V, int(p.variant), p.k1, p.b, p.delta)


def assert_index_equal(gx, ox, what=""):
    for key in ("indptr", "docids", "df", "doclens", "tf"):
        assert np.array_equal(gx[key], ox[key]), f"{what}: {key} differs"
    assert gx["avg_len"] == ox["avg_len"], what
    rel = np.abs(gx["values"].astype(np.float64) - ox["values"]) / np.maximum(np.abs(ox["values"]), 1e-30)
    assert rel.max(initial=0) <= TOL, f"{what}: values rel err {rel.max()}"
    relt = np.abs(gx["theta"].astype(np.float64) - ox["theta"]) / np.maximum(np.abs(ox["theta"]), 1e-30)
    assert relt.max(initial=0) <= TOL, f"{what}: theta rel err {relt.max()}"
    return int(np.count_nonzero(gx["values"] != ox["values"]))


def test_device_generator_matches_host(cuda_ok, c1):
    import torch
    cfg, corp, _, _ = c1
    T = int(corp.offsets[-1])
    out = torch.empty(T, dtype=torch.uint32, device="cuda")
    synth.tokens_device(cfg, corp.cdf, 0, T, out.data_ptr())
    assert np.array_equal(out.cpu().numpy(), corp.tokens)
    # c5's generator (V = 4M, Zipf 1.0) at positions beyond 2^32 (the last shard of 1.65e10 tokens)
    c5 = synth.config(5)
    cdf5 = synth.zipf_cdf(c5)
    n, begin = 4_000_000, 16_000_000_000
    out = torch.empty(n, dtype=torch.uint32, device="cuda")
    synth.tokens_device(c5, cdf5, begin, n, out.data_ptr())
    assert np.array_equal(out.cpu().numpy(), synth.tokens_host(c5, cdf5, begin, n, threads=8))


@pytest.mark.parametrize("p", VARIANTS, ids=lambda p: f"{p.variant.name}-d{p.delta}")
def test_build_c1_bitexact(cuda_ok, c1, p):
    cfg, corp, _, _ = c1
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p, keep_tf=True) as gi:
        gx = gi.export(tf=True)
    ox = _oracle(corp, cfg.vocab, p).export()
    n_diff = assert_index_equal(gx, ox, p.variant.name)
    # f64 log may differ from glibc by an ulp; after f32 narrowing almost always identical
    assert n_diff <= max(3, len(ox["values"]) // 100000), f"{n_diff} values not bit-identical"


@pytest.mark.parametrize("k", [10, 100, 1000])
def test_retrieve_c1_lucene(cuda_ok, c1, k):
    cfg, corp, qoff, qtok = c1
    p = BM25Params(Variant.lucene, 1.5, 0.75)
    ox = _oracle(corp, cfg.vocab, p)
    exp = ox.export()
    rid, rsc = ox.retrieve_batch(qoff, qtok, k, True, 8)
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
        gid, gsc = retrieve_batch(gi, (qoff, qtok), k, as_arrays=True)
    q = lambda b: qtok[int(qoff[b]):int(qoff[b + 1])]  # noqa: E731
    assert_topk_match(gid, gsc, rid, rsc, k, cfg.num_docs, lambda b: ox.score_query(q(b)),
                      lambda b: query_scale(exp, q(b)), f"c1 k={k}")


@pytest.mark.parametrize("p", VARIANTS, ids=lambda p: f"{p.variant.name}-d{p.delta}")
def test_retrieve_c1_variants(cuda_ok, c1, p):
    cfg, corp, qoff, qtok = c1
    ox = _oracle(corp, cfg.vocab, p)
    exp = ox.export()
    rid, rsc = ox.retrieve_batch(qoff, qtok, 10, True, 8)
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
        gid, gsc = retrieve_batch(gi, (qoff, qtok), 10, as_arrays=True)
    q = lambda b: qtok[int(qoff[b]):int(qoff[b + 1])]  # noqa: E731
    assert_topk_match(gid, gsc, rid, rsc, 10, cfg.num_docs, lambda b: ox.score_query(q(b)),
                      lambda b: query_scale(exp, q(b)), p.variant.name)


@pytest.mark.parametrize("density", [0.0001, 0.01, 0.25, 2.0])
def test_dense_threshold_variants_match_oracle(cuda_ok, c1, density):
    """Dense query-side row copies are an access path: any threshold (all rows dense ..
    none dense) must reproduce the oracle's top-k."""
    cfg, corp, qoff, qtok = c1
    p = BM25Params(Variant.bm25l, 1.5, 0.75, 0.5)
    ox = _oracle(corp, cfg.vocab, p)
    exp = ox.export()
    rid, rsc = ox.retrieve_batch(qoff, qtok, 100, True, 8)
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p, dense_min_density=density) as b:
        assert (b.info().dense_rows > 0) == (density <= 1.0)
        gid, gsc = retrieve_batch(b, (qoff, qtok), 100, as_arrays=True)
    q = lambda i: qtok[int(qoff[i]):int(qoff[i + 1])]  # noqa: E731
    assert_topk_match(gid, gsc, rid, rsc, 100, cfg.num_docs, lambda i: ox.score_query(q(i)),
                      lambda i: query_scale(exp, q(i)), f"density={density}")


@pytest.mark.parametrize("k", [10, 50])
def test_group_and_split_invariance(cuda_ok, c1, monkeypatch, k):
    """Per-document summation order is fixed: any run size (queries of one dense signature per
    warp item, the undo-log path for R > 1), doc split, work order or dense-chunk kernel gives
    identical bits."""
    cfg, corp, qoff, qtok = c1
    p = BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5)
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
        ref = retrieve_batch(gi, (qoff, qtok), k, as_arrays=True)
        for r, s, order, narrow in [(1, 1, 1, 4), (2, 3, 0, 4), (4, 1, 1, 0), (3, 7, 1, 1000), (2, 10, 1, 0)]:
            monkeypatch.setenv("SL_RUN", str(r))
            monkeypatch.setenv("SL_SPLITS", str(s))
            monkeypatch.setenv("SL_RUN_ORDER", str(order))
            monkeypatch.setenv("SL_NARROW_ITEMS", str(narrow))
            out = retrieve_batch(gi, (qoff, qtok), k, as_arrays=True)
            np.testing.assert_array_equal(out[0], ref[0])
            np.testing.assert_array_equal(out[1], ref[1])


def test_score_query_dense_vector(cuda_ok, c1):
    cfg, corp, qoff, qtok = c1
    for p in VARIANTS:
        ox = _oracle(corp, cfg.vocab, p)
        exp = ox.export()
        with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
            for b in range(0, 1000, 97):
                q = qtok[int(qoff[b]):int(qoff[b + 1])]
                g = score_query(gi, q).astype(np.float64)
                r = ox.score_query(q)
                tol = TOL * np.maximum(np.abs(r), query_scale(exp, q)) + 1e-30
                assert np.all(np.abs(g - r) <= tol), (p.variant.name, b)


def test_edge_queries(cuda_ok):
    # toy corpus of SPEC index examples: ["cat sat", "dog ran", "cat cat cat"], ids cat=0 sat=1 dog=2 ran=3, 4=unused
    off = np.array([0, 2, 4, 7], np.uint64)
    tok = np.array([0, 1, 2, 3, 0, 0, 0], np.uint32)
    for p in VARIANTS:
        ox = oracle.OracleIndex(off, tok, 5, int(p.variant), p.k1, p.b, p.delta)
        exp = ox.export()
        queries = [[], [0], [0, 0], [4], [4, 1], [0, 1, 2, 3], [3, 3, 1]]
        qo, qt = csr(queries)
        for k in (1, 2, 3, 5):
            rid, rsc = ox.retrieve_batch(qo, qt, k, True, 1)
            with build_index(off, tok, 5, p) as gi:
                gid, gsc = retrieve_batch(gi, (qo, qt), k, as_arrays=True)
            assert_topk_match(gid, gsc, rid, rsc, k, 3, lambda b: ox.score_query(queries[b]),
                              lambda b: query_scale(exp, queries[b]), f"toy {p.variant.name} k={k}")


def test_toy_corpus_golden(cuda_ok):
    """SURVEY.md §4 values verified with the reference's own scoring.cpp."""
    off = np.array([0, 2, 4, 7], np.uint64)
    tok = np.array([0, 1, 2, 3, 0, 0, 0], np.uint32)
    with build_index(off, tok, 4, BM25Params(Variant.lucene)) as gi:
        e = gi.export()
    assert e["indptr"].tolist() == [0, 2, 3, 4, 5]  # 5 nonzeros (SPEC.md:207 says 6: erratum)
    assert e["docids"].tolist() == [0, 2, 0, 1, 1]
    np.testing.assert_array_equal(e["values"], np.array([0.200917587, 0.292446703, 0.419285774, 0.419285774,
                                                         0.419285774], np.float32))
    assert e["avg_len"] == 7 / 3
    with build_index(off, tok, 4, BM25Params(Variant.bm25plus, 1.5, 0.75, 1.0)) as gi:
        e = gi.export()
    assert np.float32(e["theta"][0]) == np.float32(0.693147181)
    np.testing.assert_array_equal(e["values"][:2], np.array([0.740767956, 1.07822895], np.float32))


def test_errors(cuda_ok):
    off = np.array([0, 2, 4, 7], np.uint64)
    tok = np.array([0, 1, 2, 3, 0, 0, 0], np.uint32)
    with pytest.raises(ValueError, match="token id >= vocab size"):
        build_index(off, tok, 3)
    with pytest.raises(ValueError, match="degenerate corpus"):
        build_index(np.zeros(3, np.uint64), np.zeros(0, np.uint32), 4)
    with pytest.raises(ValueError, match="empty corpus"):
        build_index(np.zeros(1, np.uint64), np.zeros(0, np.uint32), 4)
    with pytest.raises(ValueError, match="k1 must be > 0"):
        build_index(off, tok, 4, BM25Params(Variant.lucene, 0.0))
    with pytest.raises(ValueError, match="tfldp requires"):
        build_index(off, tok, 4, BM25Params(Variant.tfldp, 1.5, 0.75, 0.3))
    with build_index(off, tok, 4) as gi:
        with pytest.raises(ValueError, match="token id >= vocab size"):
            retrieve_batch(gi, [[9]], 2)
        with pytest.raises(ValueError, match="k must be >= 1"):
            retrieve_batch(gi, [[0]], 0)


def test_empty_docs_and_unused_tokens(cuda_ok):
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 6, 300)
    lens[:7] = 0
    off = np.zeros(301, np.uint64)
    off[1:] = np.cumsum(lens)
    tok = rng.integers(0, 40, int(off[-1])).astype(np.uint32) * 3  # ids ≡ 0 mod 3: most of V=150 unused
    queries = [list(rng.integers(0, 150, rng.integers(0, 6))) for _ in range(200)]
    qo, qt = csr(queries)
    for p in VARIANTS:
        ox = oracle.OracleIndex(off, tok, 150, int(p.variant), p.k1, p.b, p.delta)
        exp = ox.export()
        with build_index(off, tok, 150, p, keep_tf=True) as gi:
            assert_index_equal(gi.export(tf=True), exp, p.variant.name)
            for k in (1, 7, 300, 400):
                gid, gsc = retrieve_batch(gi, (qo, qt), k, as_arrays=True)
                rid, rsc = ox.retrieve_batch(qo, qt, k, True, 2)
                assert_topk_match(gid, gsc, rid, rsc, k, 300, lambda b: ox.score_query(queries[b]),
                                  lambda b: query_scale(exp, queries[b]), f"ragged {p.variant.name} k={k}")


def test_random_corpora_ac1_ac2(cuda_ok):
    """SPEC acceptance criteria 1 and 2 on the GPU path, at their stated sizes:
    50 random corpora (10-200 docs, vocab <= 300, doc length 1-50) x all 6 variants x 20 random
    queries. AC1: score_query equals the naive dense scorer (B(Q,D) from raw tf/df/lengths)
    within 1e-5 element-wise. AC2: for the shifted variants (bm25l, bm25plus, tfldp) the ranking
    of the whole corpus from retrieve_batch (k = |C|) equals the dense oracle's ranking up to
    ties within the tolerance, and the reported scores include the query constant."""
    rng = np.random.default_rng(11)
    shifted = {Variant.bm25l, Variant.bm25plus, Variant.tfldp}
    for trial in range(50):
        N = int(rng.integers(10, 201))
        V = int(rng.integers(5, 301))
        lens = rng.integers(1, 51, N)
        off = np.zeros(N + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        tok = rng.integers(0, V, int(off[-1])).astype(np.uint32)
        queries = [list(rng.integers(0, V, rng.integers(1, 6))) for _ in range(20)]
        qo, qt = csr(queries)
        for p in VARIANTS:
            with build_index(off, tok, V, p) as gi:
                dense = [oracle.dense_score(off, tok, V, q, int(p.variant), p.k1, p.b, p.delta) for q in queries]
                for q, d in zip(queries, dense):
                    g = score_query(gi, q).astype(np.float64)
                    scale = np.abs(d).max() + 1e-12
                    assert np.all(np.abs(g - d) <= TOL * np.maximum(np.abs(d), scale)), (trial, p)
                if p.variant not in shifted:
                    continue
                gid, gsc = retrieve_batch(gi, (qo, qt), N, as_arrays=True)
                for b, d in enumerate(dense):
                    scale = np.abs(d).max() + 1e-12
                    tol = TOL * scale
                    order = np.lexsort((np.arange(N), -d))  # dense oracle's ranking (ties -> smaller doc)
                    ids = gid[b].astype(np.int64)
                    assert sorted(ids.tolist()) == list(range(N)), (trial, p, b)
                    # same ranking up to ties: position by position the oracle scores agree
                    assert np.all(np.abs(d[ids] - d[order]) <= tol), (trial, p, b)
                    # reported scores are B(Q,D) including the constant Σ S^θ
                    assert np.all(np.abs(gsc[b].astype(np.float64) - d[ids]) <= tol), (trial, p, b)


def test_top_k_random_vectors_ac3(cuda_ok):
    """SPEC acceptance criterion 3 at its stated size: 1,000 random vectors of
    length 1-10,000 (every third duplicate-heavy): the selected set and order equal a full-sort
    oracle's, ordered output globally descending, ties -> smaller index."""
    rng = np.random.default_rng(3)
    for i in range(1000):
        n = int(rng.integers(1, 10001))
        if i % 3 == 0:
            s = rng.integers(0, 4, n).astype(np.float32)  # duplicate-heavy
        else:
            s = rng.standard_normal(n).astype(np.float32)
        k = int(rng.integers(1, 300))
        gi, gs = top_k(s, k)
        ri, rs = oracle.top_k(s.astype(np.float64), k)
        assert np.array_equal(gi.astype(np.int64), ri.astype(np.int64)), i
        assert np.array_equal(gs, rs.astype(np.float32)), i


@pytest.mark.parametrize("p", [BM25Params(Variant.lucene), BM25Params(Variant.robertson),
                               BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5)], ids=lambda p: p.variant.name)
@pytest.mark.parametrize("k", [10, 1000])
def test_blockmax_pruning_is_exact(cuda_ok, c1, monkeypatch, p, k):
    """Opt-in block-max pruning (SL_BLOCKMAX=1 build, SL_PRUNE=1 query) skips (query, tile)
    pairs whose bound cannot beat the threshold: the top-k must be bit-identical."""
    cfg, corp, qoff, qtok = c1
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as a:
        ref = retrieve_batch(a, (qoff, qtok), k, as_arrays=True)
    monkeypatch.setenv("SL_BLOCKMAX", "1")
    monkeypatch.setenv("SL_PRUNE", "1")
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as b:
        out = retrieve_batch(b, (qoff, qtok), k, as_arrays=True)
    np.testing.assert_array_equal(out[0], ref[0])
    np.testing.assert_array_equal(out[1], ref[1])


@pytest.mark.parametrize("p", [BM25Params(Variant.lucene), BM25Params(Variant.bm25l, 1.5, 0.75, 0.5)],
                         ids=lambda p: p.variant.name)
def test_long_queries_mixed_batch(cuda_ok, c1, p):
    """Queries with > 32 gathered rows (e.g. passage-length BEIR queries) run on the CTA kernel;
    a batch mixing them with short queries must match the oracle query by query."""
    cfg, corp, qoff, qtok = c1
    rng = np.random.default_rng(9)
    queries = []
    for i in range(120):
        if i % 3 == 0:  # long: 40..300 tokens, mostly distinct mid/low-frequency ids (+ some repeats)
            n = int(rng.integers(40, 301))
            q = list(rng.integers(30, cfg.vocab, n)) + list(rng.integers(0, 30, 5))
        else:
            q = list(qtok[int(qoff[i]):int(qoff[i + 1])])
        queries.append(q)
    qo, qt = csr(queries)
    ox = _oracle(corp, cfg.vocab, p)
    exp = ox.export()
    for k in (10, 100):
        rid, rsc = ox.retrieve_batch(qo, qt, k, True, 8)
        with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
            gid, gsc = retrieve_batch(gi, (qo, qt), k, as_arrays=True)
            for b in range(0, 120, 7):
                s = score_query(gi, queries[b])  # the CTA kernel: same bits as the top-k path
                np.testing.assert_array_equal(s[gid[b, :k].astype(np.int64)], gsc[b, :k])
        assert_topk_match(gid, gsc, rid, rsc, k, cfg.num_docs, lambda b: ox.score_query(queries[b]),
                          lambda b: query_scale(exp, queries[b]), f"long {p.variant.name} k={k}")


def test_large_k_full_ranking(cuda_ok, c1):
    """k > 4096 (SPEC top_k: up to |C|, 'k >= n returns all documents'): stable full ranking."""
    cfg, corp, qoff, qtok = c1
    p = BM25Params(Variant.robertson)
    ox = _oracle(corp, cfg.vocab, p)
    exp = ox.export()
    sel = [0, 5, 77, 500, 999]
    qs = [qtok[int(qoff[b]):int(qoff[b + 1])] for b in sel]
    qo, qt = csr(qs)
    for k in (5000, cfg.num_docs, cfg.num_docs + 7):
        rid, rsc = ox.retrieve_batch(qo, qt, k, True, 4)
        with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
            gid, gsc = retrieve_batch(gi, (qo, qt), k, as_arrays=True)
            small = retrieve_batch(gi, (qo, qt), 100, as_arrays=True)
        np.testing.assert_array_equal(gid[:, :100], small[0])  # same ranking as the fused path
        np.testing.assert_array_equal(gsc[:, :100], small[1])
        assert_topk_match(gid, gsc, rid, rsc, k, cfg.num_docs, lambda b: ox.score_query(qs[b]),
                          lambda b: query_scale(exp, qs[b]), f"large k={k}")
    s = np.random.default_rng(1).integers(0, 50, 20000).astype(np.float32)
    gi_, gs_ = top_k(s, 20000)
    ri_, rs_ = oracle.top_k(s.astype(np.float64), 20000)
    np.testing.assert_array_equal(gi_.astype(np.int64), ri_.astype(np.int64))


@pytest.mark.parametrize("cap", ["0", "3"])
def test_dense_cap_planning_path(cuda_ok, c1, monkeypatch, cap):
    """SL_DENSE_MAX_ROWS binds the dense-copy cap: the build plans its access structures on the
    host (capped path) instead of the device fast path; the highest-df rows stay dense and the
    top-k still matches the oracle."""
    cfg, corp, qoff, qtok = c1
    p = BM25Params(Variant.lucene)
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
        assert gi.info().dense_rows > 3
    ox = _oracle(corp, cfg.vocab, p)
    exp = ox.export()
    rid, rsc = ox.retrieve_batch(qoff, qtok, 20, True, 8)
    monkeypatch.setenv("SL_DENSE_MAX_ROWS", cap)
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
        assert gi.info().dense_rows <= int(cap)  # ties at the cap boundary stay sparse
        gid, gsc = retrieve_batch(gi, (qoff, qtok), 20, as_arrays=True)
    q = lambda i: qtok[int(qoff[i]):int(qoff[i + 1])]  # noqa: E731
    assert_topk_match(gid, gsc, rid, rsc, 20, cfg.num_docs, lambda i: ox.score_query(q(i)),
                      lambda i: query_scale(exp, q(i)), f"dense cap {cap}")


def test_dense_pair_rows_exact(cuda_ok, c1, monkeypatch):
    """Pair rows (r_a + r_b) and triple rows ((r_a + r_b) + r_c) of the leading dense slots are
    access paths: queries whose dense signature starts with them — including repeated dense
    tokens, which have none — give bit-identical top-k with them on and off."""
    cfg, corp, _, _ = c1
    p = BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5)
    rng = np.random.default_rng(41)
    queries = [list(rng.integers(0, 12, rng.integers(2, 6))) + list(rng.integers(0, cfg.vocab, 2)) for _ in range(300)]
    queries += [[0, 0], [1, 0, 1], [0, 1], [2, 2, 2, 3], [0, 1, 2, 3, 4, 5]]
    qo, qt = csr(queries)
    out = []
    for pairs, triples in (("0", "0"), ("16", "0"), ("16", "8")):  # none, pair rows, pair + triple rows
        monkeypatch.setenv("SL_DENSE_PAIRS", pairs)
        monkeypatch.setenv("SL_DENSE_TRIPLES", triples)
        with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
            out.append(retrieve_batch(gi, (qo, qt), 20, as_arrays=True))
    for o in out[1:]:
        np.testing.assert_array_equal(out[0][0], o[0])
        np.testing.assert_array_equal(out[0][1], o[1])


def test_zero_score_ties_across_splits(cuda_ok, c1, monkeypatch):
    """Robertson head-token queries: documents containing them score below 0, the rest exactly 0,
    so the top-k is score-0 ties resolved by the smallest doc ids. Splits publish their k-th key
    one score ordinal lower as a shared threshold; one ordinal below 0 is not a float of its own
    (-0 and +0 share it) and must still let exact zeros through — in every split, whatever the
    order the splits run in."""
    cfg, corp, _, _ = c1
    p = BM25Params(Variant.robertson, 1.5, 0.75)
    ox = _oracle(corp, cfg.vocab, p)
    exp = ox.export()
    heads = [t for t in range(50) if exp["df"][t] > cfg.num_docs // 2][:6]
    assert heads, "c1 has tokens in more than half of the documents"
    queries = [[t] for t in heads] * 20 + [heads[:2]] * 20
    qo, qt = csr(queries)
    rid, rsc = ox.retrieve_batch(qo, qt, 64, True, 4)
    monkeypatch.setenv("SL_SPLITS", "8")
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
        for _ in range(5):
            gid, gsc = retrieve_batch(gi, (qo, qt), 64, as_arrays=True)
            np.testing.assert_array_equal(gid, rid.astype(np.uint32))


def test_zero_ties_after_split_threshold_published(cuda_ok, monkeypatch):
    """The one-ordinal-below-zero split threshold: token 0 sits in more than half of the
    documents (Robertson idf < 0, so they score below 0) except 5 documents at 10235..10239 and
    the tail from 12240. Later splits meet their exact zeros early and publish their k-th key;
    the split holding 10235..10239 reaches them after reading that threshold, and they are the
    best documents (smallest ids among the ties). With the threshold mapped to -0.0 the 5-split
    plan lost them (+0 > -0 is false)."""
    N, T = 20480, 1024
    in0 = np.zeros(N, bool)
    in0[:10235] = True
    in0[10240:12240] = True
    docs = [[0, 1] if in0[d] else [2, 1] for d in range(N)]
    off = np.zeros(N + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in docs])
    tok = np.concatenate([np.asarray(x, np.uint32) for x in docs])
    p = BM25Params(Variant.robertson, 1.5, 0.75)
    ox = oracle.OracleIndex(off, tok, 3, int(p.variant), p.k1, p.b, p.delta)
    qo, qt = csr([[0]])
    rid, rsc = ox.retrieve_batch(qo, qt, 10, True, 1)
    assert list(rid[0]) == [10235, 10236, 10237, 10238, 10239, 12240, 12241, 12242, 12243, 12244]
    for splits in ("2", "5", "20"):
        monkeypatch.setenv("SL_SPLITS", splits)
        with build_index(off, tok, 3, p) as gi:
            for _ in range(3):
                gid, gsc = retrieve_batch(gi, (qo, qt), 10, as_arrays=True)
                np.testing.assert_array_equal(gid[0], rid[0].astype(np.uint32), err_msg=f"splits {splits}")


@pytest.mark.parametrize("p", [BM25Params(Variant.lucene), BM25Params(Variant.robertson),
                               BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5)], ids=lambda p: p.variant.name)
def test_long_queries_vs_f64_oracle(cuda_ok, c1, p):
    """Queries with more than 32 gathered rows (k_score_long) and up to 200 tokens, repeats
    included: the f32 accumulation (north_star) stays within 1e-5 of the SPEC's f64 accumulator,
    and the top-k order equals the f64 oracle's except inside that tie band (INTEGRATION.md,
    "Accumulation precision")."""
    cfg, corp, _, _ = c1
    rng = np.random.default_rng(21)
    queries = [list(rng.integers(0, cfg.vocab, int(rng.integers(33, 201)))) for _ in range(60)]
    queries += [list(rng.integers(0, 50, 120)) for _ in range(10)]  # head tokens, many repeats
    qo, qt = csr(queries)
    ox = _oracle(corp, cfg.vocab, p)
    exp = ox.export()
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
        for k in (10, 100):
            gid, gsc = retrieve_batch(gi, (qo, qt), k, as_arrays=True)
            rid, rsc = ox.retrieve_batch(qo, qt, k, True, 4)
            assert_topk_match(gid, gsc, rid, rsc, k, cfg.num_docs, lambda b: ox.score_query(queries[b]),
                              lambda b: query_scale(exp, queries[b]), f"long {p.variant.name} k={k}")


@pytest.mark.parametrize("k", [10, 1000])
def test_query_chunking_bit_identical(cuda_ok, c1, monkeypatch, k):
    """A batch whose candidate scratch exceeds SL_CAND_MB is scored in chunks of queries; the
    results are bit-identical to one chunk (1 MB forces dozens of chunks at c1)."""
    cfg, corp, qoff, qtok = c1
    with build_index(corp.offsets, corp.tokens, cfg.vocab, BM25Params()) as gi:
        ids1, sc1 = retrieve_batch(gi, (qoff, qtok), k, as_arrays=True)
        monkeypatch.setenv("SL_CAND_MB", "1")
        ids2, sc2 = retrieve_batch(gi, (qoff, qtok), k, as_arrays=True)
    np.testing.assert_array_equal(sc1, sc2)
    np.testing.assert_array_equal(ids1, ids2)


@pytest.mark.parametrize("V", [2, 100, 5_000, 300_000, 1 << 22, (1 << 22) + 5])
def test_build_sort_tiles_and_digit_widths(cuda_ok, V):
    """The build's stable (token, doc) sort across digit widths (1 .. 23-bit keys: 1 to 4 radix
    passes) and tile shapes: documents longer than a sort tile, empty documents, one hot token,
    a tail that is not a whole tile, token ids up to V - 1 — CSC equal to the oracle's."""
    rng = np.random.default_rng(V)
    lens = rng.integers(0, 40, 3000)
    lens[::97] = 0
    lens[5], lens[1700] = 9000, 13000  # longer than a sort tile
    off = np.zeros(len(lens) + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    T = int(off[-1])
    tok = np.minimum(rng.zipf(1.1, T) - 1, V - 1).astype(np.uint32)
    tok[rng.random(T) < 0.05] = V - 1
    tok[int(off[5]):int(off[6])] = 0  # one document of a single hot token
    p = BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5)
    ox = oracle.OracleIndex(off, tok, V, int(p.variant), p.k1, p.b, p.delta).export()
    with build_index(off, tok, V, p, keep_tf=True) as gi:
        assert_index_equal(gi.export(tf=True), ox, f"V={V}")


@pytest.mark.parametrize("k", [10, 100])
def test_signature_grouping_extremes(cuda_ok, c1, k):
    """Query grouping (hash table of dense signatures) and run packing at their extremes: one
    signature shared by thousands of queries (one group packed by a warp), thousands of empty /
    OOV-only queries, every query distinct, and long queries (> 32 gathered rows) mixed in at
    random positions — the results equal the oracle's whatever the grouping."""
    cfg, corp, qoff, qtok = c1
    p = BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5)
    ox = _oracle(corp, cfg.vocab, p)
    exp = ox.export()
    rng = np.random.default_rng(11)
    base = [list(qtok[int(qoff[b]):int(qoff[b + 1])]) for b in range(len(qoff) - 1)]
    heavy = [list(rng.integers(0, cfg.vocab, 60)) for _ in range(20)]  # > 32 gathered rows
    batches = {
        "one signature x3000": [base[0]] * 3000,
        "empty and one-rare-token x2000": [[] for _ in range(1000)] + [[cfg.vocab - 1] * 3 for _ in range(1000)],
        "distinct + long mixed": base + heavy + base[::-1],
    }
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as gi:
        for what, queries in batches.items():
            order = rng.permutation(len(queries))
            queries = [queries[i] for i in order]
            qo, qt = csr(queries)
            gid, gsc = retrieve_batch(gi, (qo, qt), k, as_arrays=True)
            rid, rsc = ox.retrieve_batch(qo, qt, k, True, 8)
            assert_topk_match(gid, gsc, rid, rsc, k, cfg.num_docs, lambda b: ox.score_query(queries[b]),
                              lambda b: query_scale(exp, queries[b]), f"{what} k={k}")
