cd /root/repo
SW='[{}, {"SL_SPLIT_GAMMA": 1.3}, {"SL_SPLIT_GAMMA": 1.6}, {"SL_SPLIT_GAMMA": 2.0}, {}]'
for c in "2 10 1" "2 100 1" "4 1000 1" "2 10 8"; do set -- $c
  python tools/tune.py --config $1 --k $2 --shard-of $3 --sweep "$SW" 2>&1 | grep env | sed "s|^|main c$1 k$2 /$3 |" >> gpurun_out/gam.log
  SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/head/libsparselex_b200.so python tools/tune.py --config $1 --k $2 --shard-of $3 --sweep '[{}, {}]' 2>&1 | grep env | sed "s|^|head c$1 k$2 /$3 |" >> gpurun_out/gam.log
done
