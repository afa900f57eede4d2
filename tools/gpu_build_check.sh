#!/bin/bash
# Build-path check: new build tests, memcheck on small corpora, full GPU suite, build timings.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_build_paths.py -x -q > gpurun_out/t_build_paths.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_build_paths.py -x -q \
  -k "window_edges and packed or single_token or invalid" > gpurun_out/memcheck_build.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_build.log
for c in 2 4; do python tools/prof_build.py --config $c; done > gpurun_out/prof_build_new.log 2>&1
SL_BUILD_PAIRS=1 python tools/prof_build.py --config 2 >> gpurun_out/prof_build_new.log 2>&1
if [ -n "$FULL" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_full.log 2>&1; fi
if [ -n "$NCU" ]; then
  for c in 2 4; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/build_launches_new_c$c.csv python tools/prof_build.py --config $c > /dev/null 2>&1
  done
fi
tail -n 3 gpurun_out/t_build_paths.log gpurun_out/memcheck_build.log gpurun_out/prof_build_new.log
