cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_text.py tests/test_gpu_cpp_api.py -x -q > gpurun_out/c4_text.log 2>&1; echo "rc=$?" >> gpurun_out/c4_text.log
timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import bench
b = bench.text_pipeline_block(2, 6465.8)
print(json.dumps({k: b[k] for k in ('ms','tokens_per_s')}), b['e2e']['ms'])
" > gpurun_out/c4_textbench.log 2>&1
timeout 600 python tools/tune.py --config 4 --k 1000 --sweep '[{}, {"SL_SPLITS": 34}, {"SL_SPLITS": 68}, {"SL_SPLITS": 9}, {"SL_SPLITS": 136}]' > gpurun_out/c4_tune_k1000.log 2>&1
timeout 600 python tools/tune.py --config 4 --k 10 --sweep '[{}, {"SL_SPLITS": 64}, {"SL_SPLITS": 128}, {"SL_SPLITS": 32}]' > gpurun_out/c4_tune_k10.log 2>&1
