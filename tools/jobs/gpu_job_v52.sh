set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python bench.py > $OUT/v52_bench_default.jsonl 2> $OUT/v52_bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum --clock-control none --csv -k regex:k_jacobi_db -s 3 -c 1 --log-file $OUT/v52_ncu_jdb.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/v52_ncu_jdb.log 2>&1
