#!/bin/bash
# ncu --set full captures (source-level) of the text pipeline's heaviest kernels at t2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-tp}
for k in k_raw_insert k_tokens k_keep_emit k_raw_verify_long; do
  NAME=${T}_$k SKIP=${SKIP:-1} REPS=2 timeout 900 bash tools/ncu_kernel.sh $k python tools/text_step.py
done
