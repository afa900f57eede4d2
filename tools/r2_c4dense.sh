#!/bin/bash
# c4 dense-copy budget sweep (build-time env): pairs / triples / density vs top-1000 and top-10
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for e in "" "SL_DENSE_TRIPLES=0" "SL_DENSE_PAIRS=0 SL_DENSE_TRIPLES=0" "SL_DENSE_PAIRS=8 SL_DENSE_TRIPLES=0"; do
  echo "== $e" >> gpurun_out/c4dense.log
  env $e timeout 300 python tools/tune.py --config 4 --k 1000 --sweep '[{}]' >> gpurun_out/c4dense.log 2>&1
  env $e timeout 300 python tools/tune.py --config 4 --k 10 --sweep '[{}]' >> gpurun_out/c4dense.log 2>&1
done
for dd in 0.25 0.0625; do
  echo "== density $dd" >> gpurun_out/c4dense.log
  timeout 300 python tools/tune.py --config 4 --k 1000 --dense-density $dd --sweep '[{}]' >> gpurun_out/c4dense.log 2>&1
done
