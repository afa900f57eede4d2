#!/bin/bash
# text pipeline timing of several library builds (SPARSELEX_LIB), device-resident c2 text
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cat > /tmp/tb.py <<'PY'
import sys, os; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2407_03618_b200 import synth, text as T
from paper_2407_03618_b200._lib import SL_MEM_DEVICE
cfg = synth.config(2)
corp = synth.corpus_host(cfg, threads=16)
words = synth.word_list(cfg.vocab)
text, off = synth.render_text(corp.tokens, corp.offsets, words, cfg.corpus_seed)
dtext = torch.from_numpy(text).cuda(); doff = torch.from_numpy(off.view(np.int64)).cuda()
tc = T.TokenizerConfig.english()
ms = []
for r in range(5):
    v = T.Vocabulary()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    b = T.tokenize_build((dtext, doff), tc, v, mem=SL_MEM_DEVICE)
    e1.record(); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1)); b.close(); v.close()
print(os.environ.get("SPARSELEX_LIB", "cur"), min(ms[1:]), ms)
PY
for L in $LIBS; do SPARSELEX_LIB=$L timeout 300 python /tmp/tb.py >> gpurun_out/textvar.log 2>&1; done
