"""Profiling driver: build config c<i> on the device, run `--reps` retrieve_batch steps.
Used under ncu (one GPU) for the launch list and the --set full capture of k_score_topk."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--queries", type=int, default=0)
    ap.add_argument("--dense-density", type=float, default=0.0)
    a = ap.parse_args()
    import torch
    from paper_2407_03618_b200 import BM25Params, build_index, retrieve_batch, synth
    from paper_2407_03618_b200._lib import SL_MEM_HOST, check, lib
    cfg = synth.config(a.config)
    cdf = synth.zipf_cdf(cfg)
    off = synth.doc_offsets(cfg)
    T = int(off[-1])
    tok = torch.empty(T, dtype=torch.uint32, device="cuda")
    synth.tokens_device(cfg, cdf, 0, T, tok.data_ptr())
    idx = build_index(torch.from_numpy(off).cuda(), tok, cfg.vocab, BM25Params(), dense_min_density=a.dense_density)
    del tok
    qoff, qtok = synth.queries(cfg, cdf, 0, a.queries or None)
    d_off = torch.from_numpy(qoff).cuda()
    d_tok = torch.from_numpy(qtok).cuda()
    for _ in range(a.reps):
        ids, sc = retrieve_batch(idx, (d_off, d_tok), a.k)
    torch.cuda.synchronize()
    print("ok", ids.shape, float(sc[0, 0]))


if __name__ == "__main__":
    main()
