#!/bin/bash
# c5 on one GPU, one shard at a time: each of the 8 document shards (balanced by tokens) is
# built with shard-local statistics and queried with the full 65,536-query batch (top-100).
# An 8-GPU run is as fast as its slowest shard plus the rank-0 merge, so the spread of these
# per-shard rates bounds the strong-scaling efficiency. Output: one JSON line per shard.
cd "$(dirname "$0")/.."
for s in 0 1 2 3 4 5 6 7; do
  python bench.py --config 5 --k 100 --shard-of 8 --shard-index $s --steps 3 --warmup 2 --no-text --no-cpu-baseline \
    2>/dev/null | tail -1 | python -c "
import sys, json; d = json.loads(sys.stdin.read())
print(json.dumps({'shard': $s, 'qps': d['value'], 'ms_per_step': d['ms_per_step'], 'build_ms': d['index_build']['ms'],
                  'nnz': d['config']['nnz_local'], 'dense_rows': d['config']['dense_rows'],
                  'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons']}))"
done
