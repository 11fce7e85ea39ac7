set -u
OUT=gpurun_out; mkdir -p $OUT
MPS_JACOBI_TRACE=128 timeout 600 python tools/trace_sweeps.py 128 280 128 > $OUT/v45_trace128.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_v45.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launches_v45.log 2>&1
