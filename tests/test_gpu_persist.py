"""SPEC save_index / load_index (SPEC.md [MODULE] index, External Interfaces).

* roundtrip: load(save(idx)) has identical arrays and answers every query bit-identically
  (SPEC acceptance criterion 5: byte-identical run files);
* the files are the SPEC layout, readable by any conformant reader (numpy here) and equal to
  the oracle's CSC; an oracle-written directory loads on the GPU;
* errors: missing file (I/O error naming the path), truncated values.bin ("corrupt matrix"),
  version mismatch, vocabulary/indptr mismatch ("structural error"), broken row order,
  unwritable target.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2407_03618_b200 import BM25Params, Variant, build_index, load_index, retrieve_batch, synth
from paper_2407_03618_b200._lib import SparselexError, SparselexIOError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    cfg = synth.config(1)
    corp = synth.corpus_host(cfg)
    qoff, qtok = synth.queries(cfg, corp.cdf)
    return cfg, corp, qoff, qtok


def _run_file(ids, sc):
    """TREC-style run lines, as SPEC AC5 compares them."""
    return "\n".join(f"{q} Q0 {int(i)} {r + 1} {float(s):.9g} sl" for q in range(ids.shape[0])
                     for r, (i, s) in enumerate(zip(ids[q], sc[q])) if i != 0xFFFFFFFF)


@pytest.mark.parametrize("p", [BM25Params(Variant.lucene), BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5),
                               BM25Params(Variant.robertson)], ids=lambda p: p.variant.name)
def test_roundtrip_bit_identical(cuda_ok, c1, tmp_path, p):
    cfg, corp, qoff, qtok = c1
    d = tmp_path / "idx"
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as a:
        a.save(str(d))
        ea = a.export()
        ra = retrieve_batch(a, (qoff, qtok), 100, as_arrays=True)
    assert sorted(os.listdir(d)) == sorted(["meta.json", "vocab.json", "df.bin", "theta.bin", "indptr.bin",
                                            "docids.bin", "values.bin", "doclens.bin", "docs.json"])
    with load_index(str(d)) as b:
        eb = b.export()
        rb = retrieve_batch(b, (qoff, qtok), 100, as_arrays=True)
        assert b.avg_len == ea["avg_len"]
    for k in ("indptr", "docids", "values", "df", "theta", "doclens"):
        np.testing.assert_array_equal(ea[k], eb[k])
    assert _run_file(*ra) == _run_file(*rb)


def test_layout_matches_oracle_and_meta(cuda_ok, c1, tmp_path):
    cfg, corp, _, _ = c1
    p = BM25Params(Variant.bm25l, 1.5, 0.75, 0.5)
    with build_index(corp.offsets, corp.tokens, cfg.vocab, p) as g:
        g.save(str(tmp_path))
    ox = oracle.OracleIndex(corp.offsets, corp.tokens, cfg.vocab, int(p.variant), p.k1, p.b, p.delta).export()
    rd = lambda f, t: np.fromfile(tmp_path / f, dtype=t)  # noqa: E731
    np.testing.assert_array_equal(rd("indptr.bin", "<u8"), ox["indptr"])
    np.testing.assert_array_equal(rd("docids.bin", "<u4"), ox["docids"])
    np.testing.assert_array_equal(rd("df.bin", "<u4"), ox["df"])
    np.testing.assert_array_equal(rd("doclens.bin", "<u4"), ox["doclens"])
    v = rd("values.bin", "<f4").astype(np.float64)
    assert np.max(np.abs(v - ox["values"]) / np.maximum(np.abs(ox["values"]), 1e-30)) <= 1e-5
    meta = json.load(open(tmp_path / "meta.json"))
    assert meta["format_version"] == 1 and meta["variant"] == "bm25l"
    assert (meta["k1"], meta["b"], meta["delta"]) == (1.5, 0.75, 0.5)
    assert meta["num_docs"] == cfg.num_docs and meta["avg_len"] == ox["avg_len"]
    assert meta["num_nonzeros"] == len(ox["docids"]) and meta["num_tokens"] == int(corp.offsets[-1])
    assert set(meta["tokenizer"]) >= {"lowercase", "stopwords_hash", "stemmer"}
    assert len(json.load(open(tmp_path / "vocab.json"))) == cfg.vocab
    assert json.load(open(tmp_path / "docs.json"))[:3] == ["0", "1", "2"]


def _write_oracle_layout(d, ox, cfg, corp, p):
    os.makedirs(d, exist_ok=True)
    meta = {"format_version": 1, "variant": p.variant.name, "k1": p.k1, "b": p.b, "delta": p.delta,
            "num_docs": cfg.num_docs, "avg_len": ox["avg_len"], "num_tokens": int(corp.offsets[-1]),
            "num_nonzeros": len(ox["docids"]),
            "tokenizer": {"lowercase": True, "stopwords_hash": "", "stemmer": "none"}}
    json.dump(meta, open(os.path.join(d, "meta.json"), "w"))
    json.dump({f"tok{t}": t for t in range(cfg.vocab)}, open(os.path.join(d, "vocab.json"), "w"))
    json.dump([f"doc-{i}" for i in range(cfg.num_docs)], open(os.path.join(d, "docs.json"), "w"))
    for name, key, dt in [("indptr.bin", "indptr", "<u8"), ("docids.bin", "docids", "<u4"),
                          ("values.bin", "values", "<f4"), ("df.bin", "df", "<u4"), ("theta.bin", "theta", "<f4"),
                          ("doclens.bin", "doclens", "<u4")]:
        ox[key].astype(dt).tofile(os.path.join(d, name))


def test_oracle_written_layout_loads(cuda_ok, c1, tmp_path):
    cfg, corp, qoff, qtok = c1
    p = BM25Params(Variant.bm25plus, 1.5, 0.75, 1.0)
    o = oracle.OracleIndex(corp.offsets, corp.tokens, cfg.vocab, int(p.variant), p.k1, p.b, p.delta)
    _write_oracle_layout(str(tmp_path), o.export(), cfg, corp, p)
    rid, rsc = o.retrieve_batch(qoff, qtok, 10, True, 8)
    with load_index(str(tmp_path)) as g:
        gid, gsc = retrieve_batch(g, (qoff, qtok), 10, as_arrays=True)
    assert np.allclose(gsc, rsc, rtol=1e-5, atol=1e-5)
    assert np.mean(gid == rid) > 0.999


def test_load_errors(cuda_ok, c1, tmp_path):
    cfg, corp, _, _ = c1
    d = str(tmp_path / "idx")
    with build_index(corp.offsets, corp.tokens, cfg.vocab) as g:
        g.save(d)
    with pytest.raises(SparselexIOError, match="missing file .*nope"):
        load_index(str(tmp_path / "nope"))
    vals = open(os.path.join(d, "values.bin"), "rb").read()
    open(os.path.join(d, "values.bin"), "wb").write(vals[:-8])
    with pytest.raises(SparselexError, match="corrupt matrix"):
        load_index(d)
    open(os.path.join(d, "values.bin"), "wb").write(vals)
    meta = open(os.path.join(d, "meta.json")).read()
    open(os.path.join(d, "meta.json"), "w").write(meta.replace('"format_version": 1', '"format_version": 9'))
    with pytest.raises(SparselexError, match="version mismatch"):
        load_index(d)
    open(os.path.join(d, "meta.json"), "w").write(meta)
    voc = json.load(open(os.path.join(d, "vocab.json")))
    voc.pop("7")
    json.dump(voc, open(os.path.join(d, "vocab.json"), "w"))
    with pytest.raises(SparselexError, match="structural error"):
        load_index(d)
    json.dump({str(i): i for i in range(cfg.vocab)}, open(os.path.join(d, "vocab.json"), "w"))
    ids = np.fromfile(os.path.join(d, "docids.bin"), "<u4")
    bad = ids.copy()
    bad[1], bad[2] = ids[2], ids[1]  # break strict ordering inside row 0
    bad.tofile(os.path.join(d, "docids.bin"))
    with pytest.raises(SparselexError, match="corrupt matrix"):
        load_index(d)
    ids.tofile(os.path.join(d, "docids.bin"))
    os.remove(os.path.join(d, "docids.bin"))
    with pytest.raises(SparselexIOError, match="docids.bin"):
        load_index(d)
    blocker = tmp_path / "file"
    blocker.write_text("x")
    with build_index(corp.offsets, corp.tokens, cfg.vocab) as g:
        with pytest.raises(SparselexIOError, match="cannot create directory"):
            g.save(str(blocker / "sub"))
