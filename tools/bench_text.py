"""Text-pipeline timing: render config c<i>'s token corpus as text (synth.render_text), then
time sl_tokenize(build) on the device (text resident in HBM) and the reference tokenizer
(oracle/_ref, else the oracle port) on a bounded CPU sample.

  python tools/bench_text.py --config 2 [--reps 3] [--cpu-docs 20000] [--config-name english]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-docs", type=int, default=20000)
    ap.add_argument("--tok", default="english", choices=["english", "plain"])
    a = ap.parse_args()
    import torch
    from paper_2407_03618_b200 import synth, text as T
    from paper_2407_03618_b200._lib import SL_MEM_DEVICE, check, lib
    cfg = synth.config(a.config)
    corp = synth.corpus_host(cfg, threads=16)
    words = synth.word_list(cfg.vocab)
    t0 = time.time()
    text, off = synth.render_text(corp.tokens, corp.offsets, words, cfg.corpus_seed)
    gen_s = time.time() - t0
    nb, N = len(text), len(off) - 1
    tc = T.TokenizerConfig.english() if a.tok == "english" else T.TokenizerConfig()
    dtext = torch.from_numpy(text).cuda()
    doff = torch.from_numpy(off.view(np.int64)).cuda()
    ts, T_out, V = [], 0, 0
    for r in range(a.reps + 1):
        v = T.Vocabulary()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b = T.tokenize_build((dtext, doff), tc, v, mem=SL_MEM_DEVICE)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if r:
            ts.append(dt)
        T_out, V = b.num_tokens, v.size()
        b.close()
        v.close()
    best = min(ts)
    res = {"workload": f"t{a.config}: c{a.config} corpus rendered as text", "docs": N, "bytes": nb,
           "tokens": T_out, "vocab": V, "tokenizer": a.tok, "ms": best * 1e3, "GBps": nb / best / 1e9,
           "tokens_per_s": T_out / best, "gen_s": gen_s}
    # CPU: the reference's tokenize_build (oracle/_ref) on the first cpu-docs documents, 1 thread
    from oracle.text import TextOracle, ref_available
    kind = "ref" if ref_available() else "port"
    o = TextOracle(kind)
    n = min(N, a.cpu_docs)
    sample = bytes(text[:int(off[n])])
    t0 = time.perf_counter()
    toff, ids, toks = o.tokenize_corpus(sample, off[:n + 1], 1, int(a.tok == "english"), int(a.tok == "english"))
    cs = time.perf_counter() - t0
    res["cpu_baseline"] = {"kind": "reference" if kind == "ref" else "port", "cores": 1, "docs": n,
                           "bytes": len(sample), "GBps": len(sample) / cs / 1e9, "tokens_per_s": len(ids) / cs}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
