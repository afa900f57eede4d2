cd /root/repo
for i in 1 2; do for L in ${LIBS:-old} main; do
  if [ $L = main ]; then unset SPARSELEX_LIB; else export SPARSELEX_LIB=$PWD/paper_2407_03618_b200/csrc/build/$L/libsparselex_b200.so; fi
  echo "$L $(python -c "
import sys, json; sys.path.insert(0,'.')
import bench
b = bench.text_pipeline_block(2, 6465.8)
print(json.dumps({'ms': b['ms'], 'e2e_ms': b['e2e']['ms']}))
" 2>&1 | tail -1)" >> gpurun_out/te2e.log
done; done
