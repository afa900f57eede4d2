#!/bin/bash
# Round-2 GPU cycle: fast GPU tests, smoke, then the full-scale parity tests (c2/c3/c4, c5).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/r2_pytest_fast.log 2>&1
echo "fast rc=$?" >> gpurun_out/r2_pytest_fast.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
if [ -z "$NO_SLOW" ]; then
timeout 2400 python -m pytest tests -m "gpu and slow" -q --durations=0 ${SLOW_K:+-k "$SLOW_K"} > gpurun_out/r2_pytest_slow.log 2>&1
echo "slow rc=$?" >> gpurun_out/r2_pytest_slow.log
fi
