"""Small repro for sanitizer runs: c1 build + one retrieve_batch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_03618_b200 import BM25Params, Variant, build_index, retrieve_batch, synth  # noqa: E402

cfg = synth.config(1)
corp = synth.corpus_host(cfg)
qoff, qtok = synth.queries(cfg, corp.cdf, 0, int(sys.argv[1]) if len(sys.argv) > 1 else 100)
with build_index(corp.offsets, corp.tokens, cfg.vocab, BM25Params(Variant.lucene)) as ix:
    ids, sc = retrieve_batch(ix, (qoff, qtok), 10, as_arrays=True)
print("ok", ids[0][:5])
