"""Text e2e sweep: sl_tokenize_stream chunk sizes on the t2 corpus (pinned in/out), plus the
plain H2D copy time of the text for reference."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2407_03618_b200 import synth, text as T
    cfg = synth.config(2)
    corp = synth.corpus_host(cfg, threads=os.cpu_count() or 8)
    text, off = synth.render_text(corp.tokens, corp.offsets, synth.word_list(cfg.vocab), cfg.corpus_seed)
    tc = T.TokenizerConfig.english()
    htext = torch.from_numpy(text).pin_memory()
    hoff = torch.from_numpy(off.view(np.int64)).pin_memory()
    d = torch.empty(len(text), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(htext, non_blocking=True)
        torch.cuda.synchronize()
        h2d = time.perf_counter() - t0
    print(f"h2d {len(text) / h2d / 1e9:.1f} GB/s ({h2d * 1e3:.1f} ms)")
    h_off = torch.empty(len(off), dtype=torch.int64).pin_memory()
    h_ids = torch.empty(len(text) // 8, dtype=torch.int32).pin_memory()
    for mb in (16, 32, 64, 128, 256, 1024):
        best = 1e9
        for _ in range(3):
            v = T.Vocabulary()
            t0 = time.perf_counter()
            T.tokenize_build_stream(htext, hoff, tc, v, chunk_bytes=mb << 20, out_ids=h_ids, out_offsets=h_off)
            best = min(best, time.perf_counter() - t0)
            v.close()
        print(f"chunk {mb} MiB: {best * 1e3:.1f} ms")


if __name__ == "__main__":
    main()
