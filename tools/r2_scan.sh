#!/bin/bash
# single-pass scan: fast GPU suite, then build (c2, c4) and text timings of build/head vs in-tree
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-scan}
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for i in 1 2; do
  AB_CONFIGS="2 4" bash tools/ab_build.sh head main >> gpurun_out/${T}_build.log 2>&1
  for L in head main; do
    if [ "$L" = main ]; then unset SPARSELEX_LIB; else export SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/$L/libsparselex_b200.so; fi
    echo "$L $(REPS=5 python tools/text_step.py 2>&1 | tail -1)" >> gpurun_out/${T}_text.log
  done
done
