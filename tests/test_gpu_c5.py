"""c5 as configured (BASELINE.json configs[4]): 50,000,000 long documents, V = 4,000,000,
Zipf(1.0), ~1.65e10 tokens, with CORPUS-WIDE statistics (SURVEY.md §8d c5 parity plan).

The corpus is document-sharded 8 ways by tokens (the 8-GPU layout). One GPU builds the 8
shards one after another:
  pass 1  each shard is built with its local statistics; its df and doclens are exported and
          checked against a CPU streaming count of the same tokens (oracle.stream_df), and
          summed into the corpus-wide df, N and Σ|D| (what the NCCL all-reduce computes);
  pass 2  each shard is rebuilt with those global statistics (sl_build_desc.global_df) and
          * shard 0: every row with global df > N/32 plus 1,000 random rows are compared with
            the oracle's rows built from the same tokens and global statistics
            (oracle.stream_rows: doc ids / tf bit-exact, values within 1e-5);
          * 64 queries (56 of the batch + 8 head-heavy ones) take their per-shard top-100 keys
            (sl_retrieve_local), merged across the 8 shards by sl_merge_candidates, and are
            compared with the streaming naive dense scorer over all 50M documents
            (oracle.stream_topk, SPEC.md [MODULE] retrieval "naive dense scorer").
Tokens are generated on the device (libsl_synth, bit-identical to the host generator:
test_gpu_parity.py::test_device_generator_matches_host) and copied to the host for the CPU checks.
"""
import numpy as np
import pytest

import oracle
from paper_2407_03618_b200 import (BM25Params, Variant, build_index, merge_candidates, retrieve_local, shard_ranges,
                                   synth)
from tests.helpers import TOL

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
G = 8
K = 100


def _queries(cfg, cdf):
    qoff, qtok = synth.queries(cfg, cdf, 0, 4096)
    qs = [qtok[int(qoff[i]):int(qoff[i + 1])] for i in range(len(qoff) - 1)]
    head = [q for q in qs if len(q) and int(q.max()) < cfg.head_ranks][:8]
    assert len(head) == 8
    pick = qs[:56] + head
    off = np.zeros(len(pick) + 1, np.uint64)
    off[1:] = np.cumsum([len(q) for q in pick])
    return pick, off, np.concatenate(pick).astype(np.uint32)


def _merge_cpu(parts, k):
    """(score desc, global id asc) over the shards' CPU top-k lists."""
    ids = np.concatenate([p[0] for p in parts], axis=1)
    sc = np.concatenate([p[1] for p in parts], axis=1)
    out_i = np.full((ids.shape[0], k), 0xFFFFFFFF, np.uint32)
    out_s = np.full((ids.shape[0], k), -np.inf)
    for b in range(ids.shape[0]):
        c = sorted((-s, int(i)) for i, s in zip(ids[b], sc[b]) if i != 0xFFFFFFFF)[:k]
        out_i[b, :len(c)] = [i for _, i in c]
        out_s[b, :len(c)] = [-s for s, _ in c]
    return out_i, out_s


def test_c5_corpus_wide(cuda_ok):
    import torch
    cfg = synth.config(5)
    cdf = synth.zipf_cdf(cfg)
    offsets = synth.doc_offsets(cfg)
    N, V, T = cfg.num_docs, cfg.vocab, int(offsets[-1])
    assert N == 50_000_000 and V == 4_000_000 and T > 1.5e10
    ranges = shard_ranges(offsets, G)
    p = BM25Params(Variant.lucene, 1.5, 0.75)

    def shard(s):
        d0, d1 = ranges[s]
        o0, o1 = int(offsets[d0]), int(offsets[d1])
        tok = torch.empty(o1 - o0, dtype=torch.uint32, device="cuda")
        synth.tokens_device(cfg, cdf, o0, o1 - o0, tok.data_ptr())
        loff = (offsets[d0:d1 + 1] - np.uint64(o0)).astype(np.uint64)
        return d0, d1, loff, tok

    # ---- pass 1: shard-local builds, df / doclens vs the CPU streaming count
    gdf_gpu = np.zeros(V, np.uint64)
    gdf_cpu = np.zeros(V, np.uint64)
    total = 0
    for s in range(G):
        d0, d1, loff, tok = shard(s)
        with build_index(torch.from_numpy(loff).cuda(), tok, V, p, doc_base=d0) as ix:
            ex = ix.export(fields=("df", "doclens"))
        np.testing.assert_array_equal(ex["doclens"], np.diff(loff).astype(np.uint32), err_msg=f"shard {s} doclens")
        gdf_gpu += ex["df"]
        h = tok.cpu().numpy()
        del tok
        _, tl = oracle.stream_df(loff, h, V, threads=16, df=gdf_cpu)
        total += tl
        del h
    np.testing.assert_array_equal(gdf_gpu, gdf_cpu)
    assert total == T
    assert int(gdf_gpu.max()) <= N
    gstats = (gdf_gpu.astype(np.uint32), N, T)
    avg = T / N

    # ---- pass 2: global-statistics shards, rows of shard 0, 64-query top-100 over all shards
    pick, qoff, qtok = _queries(cfg, cdf)
    keys, ref_parts, qconst = [], [], None
    rng = np.random.default_rng(55)
    for s in range(G):
        d0, d1, loff, tok = shard(s)
        with build_index(torch.from_numpy(loff).cuda(), tok, V, p, doc_base=d0, global_stats=gstats) as ix:
            inf = ix.info()
            assert inf.num_docs_global == N and inf.total_len_global == T and inf.avg_len == avg
            kk, qc = retrieve_local(ix, (qoff, qtok), K)
            keys.append(kk)
            if qconst is None:
                qconst = qc
            np.testing.assert_array_equal(qc, qconst)
            if s == 0:
                ex = ix.export(fields=("indptr", "docids", "values", "df"))
                np.testing.assert_array_equal(ex["df"], gstats[0])
        h = tok.cpu().numpy()
        del tok
        if s == 0:
            rl = np.diff(ex["indptr"].astype(np.int64))
            heavy = np.nonzero(gstats[0] > N // 32)[0]
            assert len(heavy) > 10
            present = np.nonzero(rl > 0)[0]
            sel = np.union1d(heavy, rng.choice(present, 1000, replace=False)).astype(np.uint32)
            rows = oracle.stream_rows(loff, h, V, sel, (gstats[0], N, avg), int(p.variant), p.k1, p.b, p.delta,
                                      threads=16)
            ndiff = 0
            for t in sel:
                b, e = int(ex["indptr"][t]), int(ex["indptr"][t + 1])
                docs, _, vals = rows[int(t)]
                np.testing.assert_array_equal(ex["docids"][b:e], docs, err_msg=f"row {t} doc ids")
                g = ex["values"][b:e].astype(np.float64)
                r = vals.astype(np.float64)
                assert np.all(np.abs(g - r) <= TOL * np.abs(r)), f"row {t} values"
                ndiff += int(np.count_nonzero(ex["values"][b:e] != vals))
            nsel = int(sum(len(rows[int(t)][0]) for t in sel))
            assert ndiff <= nsel // 100000 + 1, (ndiff, nsel)
            del ex
        ref_parts.append(oracle.stream_topk(loff, h, V, d0, qoff, qtok, (gstats[0], N, avg), K, int(p.variant),
                                            p.k1, p.b, p.delta, threads=16))
        del h
    gid, gsc = merge_candidates(np.stack(keys), qconst)
    rid, rsc = _merge_cpu(ref_parts, K)
    mism = 0
    for b in range(len(pick)):
        gs, rs = gsc[b].astype(np.float64), rsc[b]
        tol = TOL * np.abs(rs) + 1e-30
        assert np.all(np.abs(gs - rs) <= tol), f"q{b}: scores differ by {np.max(np.abs(gs - rs) / np.abs(rs))}"
        if np.array_equal(gid[b], rid[b]):
            continue
        mism += 1
        # ids may differ only among documents tied (within tolerance) at the k-th score
        band = TOL * abs(rs[-1])
        diff = set(gid[b].tolist()) ^ set(rid[b].tolist())
        gmap = dict(zip(gid[b].tolist(), gs.tolist()))
        rmap = dict(zip(rid[b].tolist(), rs.tolist()))
        for d in diff:
            sd = gmap.get(d, rmap.get(d))
            assert abs(sd - rs[-1]) <= band, f"q{b}: doc {d} outside the tie band of the k-th score"
    assert mism <= 8, mism
