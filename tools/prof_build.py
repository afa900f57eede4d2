"""Profiling driver for the index build: synthesize config c<i> on the device, build twice."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    import torch
    from paper_2407_03618_b200 import BM25Params, build_index, synth
    from paper_2407_03618_b200._lib import SL_MEM_HOST, check, lib
    cfg = synth.config(a.config)
    cdf = synth.zipf_cdf(cfg)
    off = synth.doc_offsets(cfg)
    tok = torch.empty(int(off[-1]), dtype=torch.uint32, device="cuda")
    synth.tokens_device(cfg, cdf, 0, int(off[-1]), tok.data_ptr())
    doff = torch.from_numpy(off).cuda()
    for _ in range(2):
        idx = build_index(doff, tok, cfg.vocab, BM25Params())
        print("build_ms", idx.info().build_ms)
        idx.close()


if __name__ == "__main__":
    main()
