#!/bin/bash
# Multisplit radix sort: GPU correctness (fast GPU tests + the full c2 CSC), build A/B of
# variants (in-tree main, SL_SORT_NARROW=1 = the previous 7-bit passes, build/<tag> libs), the
# c2 build launch list with DRAM bytes, then the plan sweeps (tools/r2_sweep.sh).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-srt}
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python -m pytest tests/test_gpu_large.py -x -q -k "c2_lucene" > gpurun_out/${T}_c2csc.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_c2csc.log
for i in 1 2; do
AB_CONFIGS="2 4" bash tools/ab_build.sh main ${VARIANTS:-} >> gpurun_out/${T}_ab.log 2>&1
SL_SORT_NARROW=1 AB_CONFIGS="2 4" bash tools/ab_build.sh main | sed 's/^main/narrow/' >> gpurun_out/${T}_ab.log 2>&1
done
SL_BUILD_TRACE=1 timeout 300 python tools/prof_build.py --config 2 > gpurun_out/${T}_trace.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_build_launches_c2.csv python tools/prof_build.py --config 2 > /dev/null 2>&1
[ -n "$SWEEP" ] && TAG=${T}sw bash tools/r2_sweep.sh
