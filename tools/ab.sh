#!/bin/bash
# A/B timing of library builds inside ONE gpurun call (box-to-box variance is ~15%).
# usage: bash tools/ab.sh [tags...]   tag "main" = in-tree lib, else csrc/build/<tag>/
# Cases: env AB_CASES, default "2:10 2:100 4:1000" (config:k).
cd "$(dirname "$0")/.."
CASES=${AB_CASES:-"2:10 2:100 4:1000"}
for L in "${@:-main}"; do
  if [ "$L" = main ]; then unset SPARSELEX_LIB; else export SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/$L/libsparselex_b200.so; fi
  for c in $CASES; do
    echo "$L c${c%%:*} k${c##*:} $(python tools/tune.py --config ${c%%:*} --k ${c##*:} ${AB_ARGS:-} 2>&1 | grep "\"env\"" | tr "\n" " ")"
  done
done
