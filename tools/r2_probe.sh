mkdir -p gpurun_out
(lscpu; free -g; nproc; nvidia-smi) > gpurun_out/r2_box.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_base_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_base_bench.log
t0=$(date +%s)
timeout 600 /usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,gpu__time_duration.sum,lts__t_bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_score_runs -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-text > gpurun_out/r2_ncu_probe.csv 2> gpurun_out/r2_ncu_probe.err
echo "ncu rc=$? secs=$(( $(date +%s) - t0 ))" >> gpurun_out/r2_ncu_probe.err
