#!/bin/bash
# score-kernel variants (SPARSELEX_LIB builds): c2 top-10 / top-100 and c4 top-1000 retrieve times
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for L in $LIBS; do
  for ck in "2 10" "2 100" "4 1000"; do
    set -- $ck
    echo "== $L c$1 k$2" >> gpurun_out/varbench.log
    SPARSELEX_LIB=$L timeout 300 python tools/tune.py --config $1 --k $2 --sweep '[{}]' >> gpurun_out/varbench.log 2>&1
  done
done
