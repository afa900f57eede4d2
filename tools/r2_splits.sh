#!/bin/bash
# doc-split re-sweep after the run-descriptor setup (per-item cost ~10x lower): c2 top-10 / top-100, c4 top-1000
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-sp}
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py tests/test_gpu_multirank.py tests/test_gpu_large.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
python tools/tune.py --config 2 --k 10 --sweep '[{}, {"SL_SPLITS":8}, {"SL_SPLITS":12}, {"SL_SPLITS":16}, {"SL_SPLITS":20}, {"SL_SPLITS":24}, {"SL_SPLITS":32}, {}]' 2>&1 | grep '"env"' > gpurun_out/${T}_c2k10.log
python tools/tune.py --config 2 --k 100 --sweep '[{}, {"SL_SPLITS":6}, {"SL_SPLITS":8}, {"SL_SPLITS":12}, {"SL_SPLITS":16}, {"SL_SPLITS":24}, {}]' 2>&1 | grep '"env"' > gpurun_out/${T}_c2k100.log
python tools/tune.py --config 4 --k 1000 --sweep '[{}, {"SL_SPLITS":12}, {"SL_SPLITS":17}, {"SL_SPLITS":24}, {"SL_SPLITS":34}, {"SL_SPLITS":48}, {}]' 2>&1 | grep '"env"' > gpurun_out/${T}_c4k1000.log
python tools/tune.py --config 2 --k 10 --shard-of 8 --sweep '[{}, {"SL_SPLITS":2}, {"SL_SPLITS":3}, {"SL_SPLITS":4}, {"SL_SPLITS":6}, {}]' 2>&1 | grep '"env"' > gpurun_out/${T}_c2s8.log
