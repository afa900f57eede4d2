#!/bin/bash
# Round-2 plan sweeps (one box): doc splits at c2 top-10 / top-100 and c4 top-1000, and
# the scoring kernel's DRAM bytes per launch at a few split counts (ncu counters only).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/${TAG:-sw}
python tools/tune.py --config 2 --k 10 --sweep '[{}, {"SL_SPLITS": 8}, {"SL_SPLITS": 24}, {"SL_SPLITS": 48}, {"SL_SPLITS": 96}, {}]' > ${O}_c2k10.log 2>&1
python tools/tune.py --config 2 --k 100 --sweep '[{}, {"SL_SPLITS": 16}, {"SL_SPLITS": 32}, {"SL_SPLITS": 64}, {}]' > ${O}_c2k100.log 2>&1
python tools/tune.py --config 4 --k 1000 --sweep '[{}, {"SL_SPLITS": 64}, {"SL_SPLITS": 128}, {}]' > ${O}_c4k1000.log 2>&1
for s in 12 24 48 96; do
  SL_SPLITS=$s timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum \
    --clock-control none -k regex:k_score_runs -c 1 --csv python tools/prof_step.py --config 2 --k 10 --reps 1 > ${O}_ncu_s$s.csv 2>&1
done
REPS=2 timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python tools/text_step.py > ${O}_text_launches.csv 2>&1
python tools/text_step.py > ${O}_text_ms.log 2>&1
