#!/bin/bash
# text pipeline A/B: GPU text tests on the in-tree lib, then tokenize_build timings of
# build/<tag> libs vs the in-tree one (alternating), and the in-tree launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-tab}
timeout 900 python -m pytest tests/test_gpu_text.py -x -q > gpurun_out/${T}_text_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_text_tests.log
for i in 1 2; do
  for L in ${LIBS:-head} main; do
    if [ "$L" = main ]; then unset SPARSELEX_LIB; else export SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/$L/libsparselex_b200.so; fi
    echo "$L $(REPS=5 python tools/text_step.py 2>&1 | tail -1)" >> gpurun_out/${T}_ab.log
  done
done
unset SPARSELEX_LIB
REPS=2 timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python tools/text_step.py > gpurun_out/${T}_launches.csv 2>&1
