#!/bin/bash
# A/B of the text pipeline: round-1 library (build/old) vs the current one, launch lists under ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cat > /tmp/tb.py <<'PY'
import sys, json, os; sys.path.insert(0, '.')
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
for r in range(int(os.environ.get("REPS", "4"))):
    v = T.Vocabulary()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    b = T.tokenize_build((dtext, doff), tc, v, mem=SL_MEM_DEVICE)
    e1.record(); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1)); b.close(); v.close()
print(os.environ.get("SPARSELEX_LIB", "cur"), ms)
PY
for L in paper_2407_03618_b200/csrc/build/old/libsparselex_b200.so paper_2407_03618_b200/libsparselex_b200.so; do
  SPARSELEX_LIB=$L python /tmp/tb.py >> gpurun_out/textab.log 2>&1
  n=$(basename $(dirname $L))
  SPARSELEX_LIB=$L REPS=2 timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv python /tmp/tb.py > gpurun_out/textab_ncu_$n.csv 2>/dev/null
done
