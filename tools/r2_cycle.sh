#!/bin/bash
# Round-2 quick cycle: fast GPU tests, smoke, default bench line, reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-cyc}
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${T}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${T}_bench.log
if [ -n "$REF" ]; then
timeout 900 python bench.py --impl reference $REF > gpurun_out/${T}_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/${T}_ref.log
fi
