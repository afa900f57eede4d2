"""Evaluation / benchmark harness of the SPEC (SPEC.md [MODULE] eval and cmd_bench; SURVEY §8f
row 4): BEIR-format readers, TREC run files, NDCG@k, and the cmd_bench QPS fields.

  read_corpus_jsonl / read_queries_jsonl / read_qrels_tsv   BEIR formats (SPEC External Interfaces)
  write_trec_run / read_trec_run                            "qid Q0 docid rank score tag"
  ndcg_at_k(run, qrels, k=10)                               gain 2^rel - 1, log2(rank+1) discount;
                                                            queries without relevant docs excluded
  bench(tindex, queries, k, repetitions)                    {qps_retrieve, qps_end_to_end, qps_naive,
                                                             speedup} (median of repetitions)
Host plumbing around the device path; retrieval itself runs through text.py / api.py.
"""
from __future__ import annotations

import json
import math
import statistics
import time

import numpy as np


def read_corpus_jsonl(path: str):
    """[(external_id, text)], title prepended with one space when present (SPEC: BEIR convention)."""
    out = []
    with open(path, encoding="utf-8") as f:
        for line in f:
            line = line.strip()
            if not line:
                continue
            o = json.loads(line)
            text = o.get("text", "")
            if o.get("title"):
                text = o["title"] + " " + text
            out.append((str(o["_id"]), text))
    return out


def read_queries_jsonl(path: str):
    return [(str(o["_id"]), o.get("text", "")) for o in
            (json.loads(x) for x in open(path, encoding="utf-8") if x.strip())]


def read_qrels_tsv(path: str) -> dict:
    """qid<TAB>docid<TAB>relevance (header optional) -> {qid: {docid: grade}}; grades >= 0."""
    q: dict = {}
    with open(path, encoding="utf-8") as f:
        for i, line in enumerate(f):
            parts = line.rstrip("\n").split("\t")
            if len(parts) < 3:
                continue
            try:
                rel = int(parts[2])
            except ValueError:
                if i == 0:
                    continue  # header
                raise ValueError(f"qrels line {i + 1}: bad relevance {parts[2]!r}") from None
            if rel < 0:
                raise ValueError(f"qrels line {i + 1}: negative relevance")
            q.setdefault(parts[0], {})[parts[1]] = rel
    return q


def write_trec_run(path: str, qids, results, doc_ids, tag: str = "sparselex-b200") -> None:
    """One line per retrieved doc: qid Q0 external_docid rank score tag (rank from 1)."""
    with open(path, "w", encoding="utf-8") as f:
        for qid, r in zip(qids, results):
            for rank, (d, s) in enumerate(zip(r.doc_indices, r.scores)):
                f.write(f"{qid} Q0 {doc_ids[int(d)]} {rank + 1} {float(s):.9g} {tag}\n")


def read_trec_run(path: str) -> dict:
    """{qid: [docid in rank order]}."""
    runs: dict = {}
    with open(path, encoding="utf-8") as f:
        for line in f:
            p = line.split()
            if len(p) >= 6:
                runs.setdefault(p[0], []).append((int(p[3]), p[2]))
    return {q: [d for _, d in sorted(v)] for q, v in runs.items()}


def ndcg_at_k(run: dict, qrels: dict, k: int = 10):
    """SPEC eval ndcg_at_k -> (per-query dict, mean, skipped). Run queries absent from qrels are
    skipped (counted); queries with no relevant document are excluded from the mean."""
    common = [q for q in run if q in qrels]
    if not common:
        raise ValueError("ndcg_at_k: run and qrels share no query ids")
    per = {}
    for q in common:
        rel = qrels[q]
        dcg = sum((2 ** rel.get(d, 0) - 1) / math.log2(i + 2) for i, d in enumerate(run[q][:k]))
        ideal = sorted((g for g in rel.values() if g > 0), reverse=True)[:k]
        idcg = sum((2 ** g - 1) / math.log2(i + 2) for i, g in enumerate(ideal))
        if idcg > 0:
            per[q] = dcg / idcg
    mean = float(np.mean(list(per.values()))) if per else 0.0
    return per, mean, len(run) - len(common)


def bench(tindex, queries, k: int = 10, repetitions: int = 3) -> dict:
    """cmd_bench fields: qps_retrieve (pre-tokenised, device-resident ids),
    qps_end_to_end (tokenize + retrieve from host text), qps_naive (dense per-query scoring:
    score_query over every document + top_k), speedup = qps_retrieve / qps_naive; median of
    `repetitions`."""
    import ctypes as C

    import torch

    from . import text as T
    from ._lib import SL_MEM_DEVICE, check, lib
    from .api import score_query, top_k
    texts = [q if isinstance(q, str) else q[1] for q in queries]
    B = len(texts)
    qb = T.tokenize_query(texts, tindex.config, tindex.vocab)
    dev = f"cuda:{tindex.index.device}"
    ids = torch.empty((B, k), dtype=torch.uint32, device=dev)
    sc = torch.empty((B, k), dtype=torch.float32, device=dev)

    def retrieve_only():
        check(lib().sl_retrieve_batch(tindex.index.handle, qb.d_offsets, qb.d_ids or qb.d_offsets, B, k, 1,
                                      SL_MEM_DEVICE, ids.data_ptr(), sc.data_ptr()))

    def timed(fn):
        ts = []
        for _ in range(repetitions):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts)

    retrieve_only()
    t_ret = timed(retrieve_only)
    t_e2e = timed(lambda: T.retrieve_text_batch(tindex, texts, k))
    lists = qb.lists()
    n_naive = min(B, 64)

    def naive():
        for q in lists[:n_naive]:
            top_k(score_query(tindex.index, q), k)

    t_naive = timed(naive) * B / n_naive
    qb.close()
    return {"qps_retrieve": B / t_ret, "qps_end_to_end": B / t_e2e, "qps_naive": B / t_naive,
            "speedup": t_naive / t_ret, "repetitions": repetitions, "statistic": "median",
            "naive_sample_queries": n_naive}
