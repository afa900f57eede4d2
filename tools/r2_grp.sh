#!/bin/bash
# signature grouping / plan: fast GPU suite, A/B vs build/head, shard sweeps (c2 1/2, 1/4, 1/8)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-grp}
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
LIBS="head main" C5=1 TAG=${T}_ab bash tools/r2_ab.sh
for f in 2 4 8; do
  for L in head main; do
    if [ "$L" = main ]; then unset SPARSELEX_LIB; else export SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/$L/libsparselex_b200.so; fi
    echo "$L c2/$f $(python tools/tune.py --config 2 --k 10 --shard-of $f --sweep '[{}, {}]' 2>&1 | grep '"env"' | tail -1)" >> gpurun_out/${T}_shards.log
    echo "$L c4/$f $(python tools/tune.py --config 4 --k 1000 --shard-of $f --sweep '[{}, {}]' 2>&1 | grep '"env"' | tail -1)" >> gpurun_out/${T}_shards.log
  done
  unset SPARSELEX_LIB
  python tools/tune.py --config 2 --k 10 --shard-of $f --sweep '[{"SL_SPLITS": 1}, {"SL_SPLITS": 2}, {"SL_SPLITS": 4}, {"SL_SPLITS": 8}]' 2>&1 | grep '"env"' | sed "s|^|c2/$f |" >> gpurun_out/${T}_shards.log
done
