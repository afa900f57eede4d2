#!/bin/bash
# Round-2 evidence: full GPU suite (fast + slow), smoke, default bench line, the reference arm
# (driver's steps / warmup), bench launch list, --set full capture of k_score_runs (c2), build
# launch lists (c2, c4) -> gpurun_out/${R}_*
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=${R:-r2f}
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${R}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${R}_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${R}_bench.log
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${R}_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/${R}_ref.log
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_c2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-text --no-extra --no-ncu > /dev/null 2>&1
NAME=${R}_c2 timeout 900 bash tools/ncu_kernel.sh k_score_runs python tools/prof_step.py --config 2 --k 10 --reps 2
for c in 2 4; do
  timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_build_launches_c$c.csv python tools/prof_build.py --config $c > /dev/null 2>&1
done
