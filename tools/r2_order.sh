#!/bin/bash
# run-order A/B (SL_RUN_ORDER=0/1, alternating in one process per workload) + fast GPU suite
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-ord}
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
SW='[{"SL_RUN_ORDER":0},{"SL_RUN_ORDER":1},{"SL_RUN_ORDER":0},{"SL_RUN_ORDER":1}]'
for c in "2 10 1" "2 100 1" "4 1000 1" "2 10 2" "2 10 4" "2 10 8" "4 1000 8" "5 100 8"; do
  set -- $c
  python tools/tune.py --config $1 --k $2 --shard-of $3 --sweep "$SW" 2>&1 | grep '"env"' | sed "s|^|c$1 k$2 /$3 |" >> gpurun_out/${T}.log
done
