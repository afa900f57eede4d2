"""Document sharding on one GPU (SURVEY.md §4 tier 2 "virtual shards") and the NCCL path.

* virtual shards: G shard indexes on the same GPU built with the corpus-wide df / N / Σ|D|
  (sl_build_desc.global_df); per-shard top-k merged by (score desc, global doc asc) must be
  BIT-IDENTICAL to the unsharded index — the per-document summation order does not depend on
  the shard layout.
* NCCL: a 1-rank communicator drives the real ncclAllReduce (build) and ncclSend/Recv +
  rank-0 merge (retrieve) code path; results must equal the communicator-free path.
"""
import numpy as np
import pytest

from paper_2407_03618_b200 import BM25Params, Comm, Variant, build_index, retrieve_batch, shard_ranges, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def corpus():
    cfg = synth.config(1)
    corp = synth.corpus_host(cfg)
    qoff, qtok = synth.queries(cfg, corp.cdf)
    return cfg, corp, qoff, qtok


def merge(cands, k):
    """rank-0 merge semantics of K7: (score desc, global doc asc), padding dropped."""
    B = cands[0][0].shape[0]
    ids = np.full((B, k), 0xFFFFFFFF, np.uint32)
    sc = np.full((B, k), -np.inf, np.float32)
    for b in range(B):
        allc = [(float(s), int(i)) for ci, cs in cands for i, s in zip(ci[b], cs[b]) if i != 0xFFFFFFFF]
        allc.sort(key=lambda x: (-x[0], x[1]))
        for j, (s, i) in enumerate(allc[:k]):
            ids[b, j], sc[b, j] = i, s
    return ids, sc


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("p", [BM25Params(Variant.lucene), BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5)],
                         ids=lambda p: p.variant.name)
def test_virtual_shards_bit_identical(cuda_ok, corpus, G, p):
    cfg, corp, qoff, qtok = corpus
    k = 20
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as full:
        ref_ids, ref_sc = retrieve_batch(full, (qoff, qtok), k, as_arrays=True)
    ranges = shard_ranges(corp.offsets, G)
    shards = []
    for d0, d1 in ranges:
        o0 = int(corp.offsets[d0])
        off = (corp.offsets[d0:d1 + 1] - np.uint64(o0)).astype(np.uint64)
        tok = corp.tokens[o0:int(corp.offsets[d1])]
        shards.append((d0, off, tok))
    # corpus-wide statistics from the shards' own counts (what the NCCL all-reduce computes)
    gdf = np.zeros(cfg.vocab, np.uint64)
    for d0, off, tok in shards:
        with build_index(off, tok, cfg.vocab, p) as local:
            gdf += local.export()["df"]
    stats = (gdf.astype(np.uint32), cfg.num_docs, int(corp.offsets[-1]))
    cands = []
    for d0, off, tok in shards:
        with build_index(off, tok, cfg.vocab, p, doc_base=d0, global_stats=stats) as sh:
            assert sh.num_docs == cfg.num_docs
            cands.append(retrieve_batch(sh, (qoff, qtok), k, as_arrays=True))
    ids, sc = merge(cands, k)
    np.testing.assert_array_equal(sc, ref_sc)
    np.testing.assert_array_equal(ids, ref_ids)


def test_nccl_single_rank_path(cuda_ok, corpus):
    cfg, corp, qoff, qtok = corpus
    p = BM25Params(Variant.bm25l, 1.5, 0.75, 0.5)
    comm = Comm(Comm.unique_id(), 1, 0, 0)
    try:
        with build_index(corp.offsets, corp.tokens, cfg.vocab, p, comm=comm, keep_tf=True) as a, \
                build_index(corp.offsets, corp.tokens, cfg.vocab, p, keep_tf=True) as b:
            ea, eb = a.export(tf=True), b.export(tf=True)
            for key in ("indptr", "docids", "values", "df", "theta", "doclens", "tf"):
                np.testing.assert_array_equal(ea[key], eb[key])
            ia, sa = retrieve_batch(a, (qoff, qtok), 100, as_arrays=True)
            ib, sb = retrieve_batch(b, (qoff, qtok), 100, as_arrays=True)
            np.testing.assert_array_equal(ia, ib)
            np.testing.assert_array_equal(sa, sb)
    finally:
        comm.close()
