#!/bin/bash
# Quick GPU cycle: full GPU test suite, build phase trace (c2, c4), default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 2 4; do SL_BUILD_TRACE=1 python tools/prof_build.py --config $c; done > gpurun_out/trace.log 2>&1
if [ -n "$BENCH" ]; then timeout 600 python bench.py $BENCH > gpurun_out/bench.log 2>&1; fi
