#!/bin/bash
# Round-end evidence: default bench line (c2 top-10, cpu baseline, text block), the reference
# arm, other config bench lines, the bench launch list, build launch lists -> gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=${R:-r03}
timeout 900 python bench.py > gpurun_out/${R}_bench_c2.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_reference.log 2>&1
timeout 600 python bench.py --k 100 --no-cpu-baseline --no-text > gpurun_out/${R}_bench_c2_k100.log 2>&1
timeout 900 python bench.py --config 4 --k 1000 --steps 3 --warmup 3 --no-cpu-baseline --no-text > gpurun_out/${R}_bench_c4_k1000.log 2>&1
timeout 300 python bench.py --config 1 --no-text > gpurun_out/${R}_bench_c1.log 2>&1
timeout 900 python bench.py --config 4 --k 10 --steps 3 --warmup 3 --no-cpu-baseline --no-text > gpurun_out/${R}_bench_c4_k10.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_c2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-text > /dev/null 2>&1
for c in 2 4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_build_launches_c$c.csv python tools/prof_build.py --config $c > /dev/null 2>&1
done
