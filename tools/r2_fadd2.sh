#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-fa}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for i in 1 2; do bash tools/ab.sh main nofadd2 >> gpurun_out/${T}.log 2>&1; done
export SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/nofadd2/libsparselex_b200.so
for c in 2:10 2:100 4:1000; do
python tools/tune.py --config ${c%%:*} --k ${c##*:} --sweep '[{}, {"SL_RUN":1}, {"SL_RUN":2}, {"SL_RUN":3}, {"SL_RUN":4}, {}]' 2>&1 | grep '"env"' > gpurun_out/${T}_run_c${c%%:*}k${c##*:}.log
done
