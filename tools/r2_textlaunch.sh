#!/bin/bash
# text pipeline evidence: launch list (time + DRAM bytes, cold-cache serialised) of two tokenize_build
# calls on the c2 text, live device times, and --set full captures of the two heaviest kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r2}
REPS=4 timeout 600 python tools/text_step.py > gpurun_out/${T}_text_live.log 2>&1
REPS=2 timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_text_launches.csv python tools/text_step.py > /dev/null 2>&1
for k in k_raw_insert k_tokens; do
  NAME=${T}_$k SKIP=${SKIP:-1} REPS=2 timeout 900 bash tools/ncu_kernel.sh $k python tools/text_step.py
done
