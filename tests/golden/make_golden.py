"""Generate golden fixtures from the REFERENCE's own scoring code (oracle/_ref/libref_scoring.so,
compiled from /root/reference/proj/src/scoring.cpp by oracle/Makefile). Run in the build
container: `python tests/golden/make_golden.py`. The fixtures are committed; the GPU box
never needs /root/reference.

scoring_golden.json : idf / score / nonoccurrence_score at seeded random arguments plus the
                      SPEC.md scoring examples.
toy_corpus.json     : the SPEC.md index example corpus ["cat sat","dog ran","cat cat cat"]
                      (ids cat=0 sat=1 dog=2 ran=3) — CSC layout derived by hand from the
                      SPEC rules, values = f32(ref_score - ref_nonoccurrence) per nonzero.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import oracle  # noqa: E402

R = oracle.ref()
HERE = os.path.dirname(os.path.abspath(__file__))
DELTA = {3: 0.5, 4: 1.0, 5: 0.5}


def scoring():
    rng = np.random.default_rng(20240703)
    g = {"idf": [], "score": [], "nonoccurrence": []}
    spec = [(2, 1, 3), (0, 3, 3), (2, 3, 3)]
    for v, df, n in spec:
        g["idf"].append({"v": v, "df": df, "n": n, "out": R.ref_idf(v, df, n)})
    g["score"].append(dict(tf=3.0, df=2, dl=3.0, n=3, avg=3.0, v=2, k1=1.5, b=0.75, delta=0.0,
                           out=R.ref_score(3.0, 2, 3.0, 3, 3.0, 2, 1.5, 0.75, 0.0)))
    g["score"].append(dict(tf=0.0, df=1, dl=3.0, n=2, avg=3.0, v=3, k1=1.2, b=0.75, delta=0.5,
                           out=R.ref_score(0.0, 1, 3.0, 2, 3.0, 3, 1.2, 0.75, 0.5)))
    g["nonoccurrence"].append(dict(df=1, n=2, v=4, k1=1.5, b=0.75, delta=1.0,
                                   out=R.ref_nonoccurrence(1, 2, 4, 1.5, 0.75, 1.0)))
    for _ in range(300):
        v = int(rng.integers(0, 6))
        n = int(rng.integers(1, 10**8))
        df = int(rng.integers(1, n + 1))
        tf = float(rng.integers(0, 40))
        dl = float(rng.integers(0, 5000))
        avg = float(rng.uniform(1, 400))
        k1, b = float(rng.uniform(0.5, 2.5)), float(rng.uniform(0, 1))
        delta = DELTA.get(v, float(rng.uniform(0.4, 1.5)))
        g["idf"].append({"v": v, "df": df, "n": n, "out": R.ref_idf(v, df, n)})
        g["score"].append(dict(tf=tf, df=df, dl=dl, n=n, avg=avg, v=v, k1=k1, b=b, delta=delta,
                               out=R.ref_score(tf, df, dl, n, avg, v, k1, b, delta)))
        g["nonoccurrence"].append(dict(df=df, n=n, v=v, k1=k1, b=b, delta=delta,
                                       out=R.ref_nonoccurrence(df, n, v, k1, b, delta)))
    return g


def toy():
    # docs: 0 "cat sat" (cat:1 sat:1, |D|=2), 1 "dog ran" (dog:1 ran:1, |D|=2), 2 "cat cat cat" (cat:3, |D|=3)
    rows = {0: [(0, 1, 2), (2, 3, 3)], 1: [(0, 1, 2)], 2: [(1, 1, 2)], 3: [(1, 1, 2)]}  # t -> [(doc, tf, |D|)]
    N, avg = 3, 7 / 3
    cases = []
    for v, delta in [(2, 0.0), (0, 0.0), (1, 0.0), (3, 0.5), (4, 1.0), (5, 0.5)]:
        indptr, docids, values, theta = [0], [], [], []
        for t in range(4):
            df = len(rows[t])
            th = R.ref_nonoccurrence(df, N, v, 1.5, 0.75, delta)
            theta.append(float(np.float32(th)))
            for d, tf, dl in rows[t]:
                docids.append(d)
                values.append(float(np.float32(R.ref_score(tf, df, dl, N, avg, v, 1.5, 0.75, delta) - th)))
            indptr.append(len(docids))
        # score_query([cat]) = slice accumulation (f64) + theta(cat)
        acc = [0.0] * N
        for j in range(indptr[0], indptr[1]):
            acc[docids[j]] += float(np.float32(values[j]))
        score_cat = [a + theta[0] for a in acc]
        cases.append(dict(v=v, delta=delta, indptr=indptr, docids=docids, values=values, theta=theta,
                          score_cat=score_cat))
    return {"corpus": ["cat sat", "dog ran", "cat cat cat"], "ids": {"cat": 0, "sat": 1, "dog": 2, "ran": 3},
            "k1": 1.5, "b": 0.75, "cases": cases}


if __name__ == "__main__":
    json.dump(scoring(), open(os.path.join(HERE, "scoring_golden.json"), "w"), indent=0)
    json.dump(toy(), open(os.path.join(HERE, "toy_corpus.json"), "w"), indent=1)
    print("wrote", HERE)
