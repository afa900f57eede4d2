"""Tuning sweep: build config c<i> once, time retrieve_batch under plan overrides
(SL_RUN / SL_SPLITS / SL_GTAU / SL_DEBUG_SKIP env vars read by the library at each call)."""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--sweep", default='[{}]')
    ap.add_argument("--dense-density", type=float, default=0.0)
    ap.add_argument("--shard-of", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2407_03618_b200 import BM25Params, build_index, synth, _lib
    from paper_2407_03618_b200._lib import SL_MEM_DEVICE, SL_MEM_HOST, check, lib
    cfg = synth.config(a.config)
    cdf = synth.zipf_cdf(cfg)
    off = synth.doc_offsets(cfg)
    if a.shard_of > 1:  # one shard of a document-sharded corpus (c5 on one GPU)
        from paper_2407_03618_b200 import shard_ranges
        d0, d1 = shard_ranges(off, a.shard_of)[0]
        os.environ.setdefault("SL_DENSE_MAX_ROWS", str((12 << 30) // (4 * cfg.num_docs)))  # the full corpus's cap
        off = (off[d0:d1 + 1] - off[d0]).astype(np.uint64)
        base = int(synth.doc_offsets(cfg, 0, d0)[-1]) if d0 else 0
    else:
        base = 0
    T = int(off[-1])
    tok = torch.empty(T, dtype=torch.uint32, device="cuda")
    synth.tokens_device(cfg, cdf, base, T, tok.data_ptr())
    idx = build_index(torch.from_numpy(off).cuda(), tok, cfg.vocab, BM25Params(), dense_min_density=a.dense_density)
    inf = idx.info()
    print(json.dumps({"build_ms": inf.build_ms, "dense_rows": inf.dense_rows, "skip_rows": inf.skip_rows,
                      "tiles": inf.num_tiles}), flush=True)
    del tok
    qoff, qtok = synth.queries(cfg, cdf)
    d_off = torch.from_numpy(qoff).cuda()
    d_tok = torch.from_numpy(qtok).cuda()
    B = len(qoff) - 1
    ids = torch.empty((B, a.k), dtype=torch.uint32, device="cuda")
    sc = torch.empty((B, a.k), dtype=torch.float32, device="cuda")
    st = _lib.RetrieveStats()
    for env in json.loads(a.sweep):
        for key in ("SL_RUN", "SL_SPLITS", "SL_GTAU", "SL_DEBUG_SKIP", "SL_RUN_ORDER", "SL_MERGE_WARP", "SL_MIN_TILES", "SL_SPLIT_GAMMA", "SL_MERGE_BIG"):
            os.environ.pop(key, None)
        os.environ.update({k: str(v) for k, v in env.items()})
        ts = []
        for i in range(5):
            check(lib().sl_retrieve_batch_timed(idx.handle, d_off.data_ptr(), d_tok.data_ptr(), B, a.k, SL_MEM_DEVICE,
                                                ids.data_ptr(), sc.data_ptr(), C.byref(st)))
            if i >= 2:
                ts.append((st.total_ms, st.score_kernel_ms, st.merge_ms))
        tot = min(t[0] for t in ts)
        print(json.dumps({"env": env, "total_ms": tot, "kernel_ms": min(t[1] for t in ts),
                          "merge_ms": min(t[2] for t in ts), "qps": B / tot * 1e3}), flush=True)


if __name__ == "__main__":
    main()
