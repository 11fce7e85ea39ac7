set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_v47.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launches_v47.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__issue_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_tc_mma -s 300 -c 40 --log-file $OUT/ncu_mma_v47.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_mma_v47.log 2>&1
