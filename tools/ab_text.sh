#!/bin/bash
# A/B of text-pipeline builds inside one gpurun call: bash tools/ab_text.sh [tags...] (main = in-tree)
cd "$(dirname "$0")/.."
for L in "${@:-main}"; do
  if [ "$L" = main ]; then unset SPARSELEX_LIB; else export SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/$L/libsparselex_b200.so; fi
  echo "$L $(python tools/bench_text.py --config ${AB_CONFIG:-2} --cpu-docs 200 ${AB_ARGS:-} 2>&1 | tail -1 | cut -c1-260)"
done
