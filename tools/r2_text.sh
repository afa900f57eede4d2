#!/bin/bash
# text pipeline: GPU text tests + c2 text timing (device-resident and e2e)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_text.py -x -q > gpurun_out/${TAG:-t}_text.log 2>&1; echo rc=$? >> gpurun_out/${TAG:-t}_text.log
timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import bench
for i in range(2):
    b = bench.text_pipeline_block(2, 6465.8)
    print(json.dumps({k: b[k] for k in ('ms','tokens_per_s')}), b['e2e']['ms'])
" > gpurun_out/${TAG:-t}_textbench.log 2>&1
