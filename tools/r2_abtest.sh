#!/bin/bash
# parity subset on the in-tree library, then tools/r2_ab.sh (LIBS, TAG, C5, AB_CASES as there)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-ab}
timeout 1500 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_sharding.py tests/test_gpu_multirank.py} -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
bash tools/r2_ab.sh
