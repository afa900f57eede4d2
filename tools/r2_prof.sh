#!/bin/bash
# build phase traces (c2, c4) + one ncu --set full capture of k_score_runs at c4 top-1000
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 2 4; do SL_BUILD_TRACE=1 timeout 300 python tools/prof_build.py --config $c; done > gpurun_out/r2_buildtrace.log 2>&1
NAME=r2_c4k1000 timeout 900 bash tools/ncu_kernel.sh k_score_runs python tools/prof_step.py --config 4 --k 1000 --reps 1
