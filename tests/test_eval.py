"""SPEC [MODULE] eval (AC7: hand-computed NDCG examples, permutation invariance below rank k)
on the CPU, and AC8 (BEIR-format triple -> index -> search -> TREC run -> NDCG@10) on the GPU."""
import json
import math

import numpy as np
import pytest

from paper_2407_03618_b200 import evalh


def test_ndcg_hand_examples():
    qrels = {"q": {"d1": 1}}
    assert evalh.ndcg_at_k({"q": ["d1", "x", "y"]}, qrels)[1] == 1.0
    v = evalh.ndcg_at_k({"q": ["x", "d1", "y"]}, qrels)[1]
    assert abs(v - 1 / math.log2(3)) < 1e-12 and abs(v - 0.63093) < 1e-5
    assert evalh.ndcg_at_k({"q": [f"x{i}" for i in range(10)] + ["d1"]}, qrels)[1] == 0.0


def test_ndcg_properties():
    rng = np.random.default_rng(0)
    for _ in range(50):
        docs = [f"d{i}" for i in range(30)]
        qrels = {"q": {d: int(rng.integers(0, 4)) for d in rng.choice(docs, 8, replace=False)}}
        run = list(rng.permutation(docs))
        per, mean, _ = evalh.ndcg_at_k({"q": run}, qrels, 10)
        if not per:
            continue
        assert 0.0 <= mean <= 1.0
        tail = run[10:]
        rng.shuffle(tail)
        assert evalh.ndcg_at_k({"q": run[:10] + tail}, qrels, 10)[1] == mean
        ideal = sorted(docs, key=lambda d: -qrels["q"].get(d, 0))
        assert abs(evalh.ndcg_at_k({"q": ideal}, qrels, 10)[1] - 1.0) < 1e-12


def test_ndcg_skips_and_errors():
    per, mean, skipped = evalh.ndcg_at_k({"a": ["d"], "b": ["d"], "c": ["d"]}, {"a": {"d": 1}, "b": {"e": 0}})
    assert skipped == 1 and per == {"a": 1.0} and mean == 1.0  # b has no relevant docs: excluded
    with pytest.raises(ValueError, match="no query ids"):
        evalh.ndcg_at_k({"a": ["d"]}, {"b": {"d": 1}})


def test_io_roundtrip(tmp_path):
    (tmp_path / "qrels.tsv").write_text("query-id\tcorpus-id\tscore\nq1\td1\t2\nq1\td2\t0\n")
    assert evalh.read_qrels_tsv(str(tmp_path / "qrels.tsv")) == {"q1": {"d1": 2, "d2": 0}}
    (tmp_path / "c.jsonl").write_text(json.dumps({"_id": "d1", "title": "T", "text": "body"}) + "\n")
    assert evalh.read_corpus_jsonl(str(tmp_path / "c.jsonl")) == [("d1", "T body")]

    class R:
        def __init__(self, i, s):
            self.doc_indices, self.scores = np.array(i), np.array(s, np.float32)
    evalh.write_trec_run(str(tmp_path / "run.txt"), ["q1"], [R([1, 0], [2.5, 1.0])], ["d1", "d2"])
    assert evalh.read_trec_run(str(tmp_path / "run.txt")) == {"q1": ["d2", "d1"]}


@pytest.mark.gpu
def test_beir_triple_end_to_end(cuda_ok, tmp_path):
    """AC8: a 100-doc synthetic BEIR triple goes index -> search -> eval."""
    from paper_2407_03618_b200 import BM25Params, text as T
    from tests.text_words import make_corpus, make_words
    words = make_words(400, seed=3)
    text, off = make_corpus(100, words, seed=1, mean_words=30)
    docs = [(f"doc{d}", text[off[d]:off[d + 1]].decode()) for d in range(100)]
    with open(tmp_path / "corpus.jsonl", "w") as f:
        for i, t in docs:
            f.write(json.dumps({"_id": i, "title": "", "text": t}) + "\n")
    # each query = 3 words of one document; that document is relevant
    rng = np.random.default_rng(5)
    queries, qrels = [], {}
    for q in range(20):
        d = int(rng.integers(100))
        ws = docs[d][1].split()[:3]
        queries.append((f"q{q}", " ".join(ws)))
        qrels[f"q{q}"] = {docs[d][0]: 1}
    with open(tmp_path / "queries.jsonl", "w") as f:
        for i, t in queries:
            f.write(json.dumps({"_id": i, "text": t}) + "\n")
    with open(tmp_path / "qrels.tsv", "w") as f:
        f.write("query-id\tcorpus-id\tscore\n")
        for q, r in qrels.items():
            for d, g in r.items():
                f.write(f"{q}\t{d}\t{g}\n")
    corpus = evalh.read_corpus_jsonl(str(tmp_path / "corpus.jsonl"))
    ti = T.build_text_index(corpus, BM25Params(), T.TokenizerConfig.english())
    qs = evalh.read_queries_jsonl(str(tmp_path / "queries.jsonl"))
    res = T.retrieve_text_batch(ti, [t for _, t in qs], 10)
    evalh.write_trec_run(str(tmp_path / "run.txt"), [q for q, _ in qs], res, ti.doc_ids)
    per, mean, skipped = evalh.ndcg_at_k(evalh.read_trec_run(str(tmp_path / "run.txt")),
                                         evalh.read_qrels_tsv(str(tmp_path / "qrels.tsv")))
    assert skipped == 0 and len(per) == 20 and 0.5 < mean <= 1.0
    b = evalh.bench(ti, [t for _, t in qs], 10, 3)
    assert set(b) >= {"qps_retrieve", "qps_end_to_end", "qps_naive", "speedup"} and b["qps_retrieve"] > 0
