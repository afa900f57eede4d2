#!/bin/bash
# scoring-kernel A/B of library builds in one session: c2 top-10 / top-100, c4 top-1000
# (tools/ab.sh, twice, alternating) and optionally the c5 shard 0 of 8 (C5=1)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-ab}
for i in 1 2; do bash tools/ab.sh ${LIBS:-main} >> gpurun_out/${T}.log 2>&1; done
if [ -n "$C5" ]; then
  for L in ${LIBS:-main}; do
    if [ "$L" = main ]; then unset SPARSELEX_LIB; else export SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/$L/libsparselex_b200.so; fi
    echo "$L c5s k100 $(python tools/tune.py --config 5 --k 100 --shard-of 8 2>&1 | grep '"env"' | tr '\n' ' ')" >> gpurun_out/${T}.log
  done
fi
