"""Text-pipeline driver for ncu launch lists: c<i> corpus rendered as text, `--reps`
tokenize_build calls (english config) on the device, device times printed."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2407_03618_b200 import synth, text as T
    from paper_2407_03618_b200._lib import SL_MEM_DEVICE
    cfg = synth.config(int(os.environ.get("CFG", "2")))
    corp = synth.corpus_host(cfg, threads=16)
    words = synth.word_list(cfg.vocab)
    text, off = synth.render_text(corp.tokens, corp.offsets, words, cfg.corpus_seed)
    dtext = torch.from_numpy(text).cuda()
    doff = torch.from_numpy(off.view(np.int64)).cuda()
    tc = T.TokenizerConfig.english()
    ms = []
    for _ in range(int(os.environ.get("REPS", "4"))):
        v = T.Vocabulary()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        b = T.tokenize_build((dtext, doff), tc, v, mem=SL_MEM_DEVICE)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        b.close()
        v.close()
    print("text ms", ms)


if __name__ == "__main__":
    main()
