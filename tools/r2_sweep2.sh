#!/bin/bash
# plan re-sweep after the heaviest-first work order
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${TAG:-sw2}
python tools/tune.py --config 2 --k 10 --sweep '[{}, {"SL_SPLITS": 8}, {"SL_SPLITS": 10}, {"SL_SPLITS": 14}, {"SL_SPLITS": 16}, {}]' 2>&1 | grep env > ${O}_c2k10.log
python tools/tune.py --config 2 --k 100 --sweep '[{}, {"SL_SPLITS": 6}, {"SL_SPLITS": 10}, {"SL_SPLITS": 12}, {}]' 2>&1 | grep env > ${O}_c2k100.log
python tools/tune.py --config 4 --k 1000 --sweep '[{}, {"SL_SPLITS": 12}, {"SL_SPLITS": 24}, {}]' 2>&1 | grep env > ${O}_c4k1000.log
python tools/tune.py --config 2 --k 10 --shard-of 8 --sweep '[{}, {"SL_SPLITS": 1}, {"SL_SPLITS": 3}, {"SL_SPLITS": 4}, {}]' 2>&1 | grep env > ${O}_c2s8.log
python tools/tune.py --config 2 --k 10 --shard-of 4 --sweep '[{}, {"SL_SPLITS": 3}, {"SL_SPLITS": 6}, {}]' 2>&1 | grep env > ${O}_c2s4.log
python tools/tune.py --config 5 --k 100 --shard-of 8 --sweep '[{}, {"SL_SPLITS": 64}, {"SL_SPLITS": 128}, {}]' 2>&1 | grep env > ${O}_c5.log
