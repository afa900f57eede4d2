#!/bin/bash
# Time breakdown of the scoring kernel by phase (SL_DEBUG_SKIP: 1 gather, 2 filter, 4 dense)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/tune.py --config 2 --k 10 --sweep '[{}, {"SL_DEBUG_SKIP": 1}, {"SL_DEBUG_SKIP": 2}, {"SL_DEBUG_SKIP": 3}, {"SL_DEBUG_SKIP": 6}, {"SL_DEBUG_SKIP": 7}, {"SL_DEBUG_SKIP": 5}]' 2>&1 | tee gpurun_out/skip.log
