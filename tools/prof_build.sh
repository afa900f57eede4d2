#!/bin/bash
# Launch lists of the index build (c2, c4) under ncu: per-kernel time shares of one build.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${PB_CONFIGS:-2 4}; do
  python tools/prof_build.py --config $c > gpurun_out/prof_build_c$c.log 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/build_launches_c$c.csv python tools/prof_build.py --config $c > /dev/null 2>&1
done
