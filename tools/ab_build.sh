#!/bin/bash
# A/B of the index build (bench.py index_build block) for library builds: bash tools/ab_build.sh tags...
cd "$(dirname "$0")/.."
for L in "$@"; do
  if [ "$L" = main ]; then unset SPARSELEX_LIB; else export SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/$L/libsparselex_b200.so; fi
  for c in ${AB_CONFIGS:-2}; do
    python bench.py --config $c --steps 2 --warmup 3 --no-text --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json; d = json.loads(sys.stdin.read()); b = d['index_build']
print('$L', 'c$c', 'build_ms %.3f' % b['ms'], 'tokens/s %.3g' % d['index_tokens_per_s'], 'qps %.0f' % d['value'])"
  done
done
