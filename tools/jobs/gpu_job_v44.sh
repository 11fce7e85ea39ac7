set -u
OUT=gpurun_out; mkdir -p $OUT
MPS_JACOBI_TRACE=3 timeout 300 python tools/trace_sweeps.py 128 280 3 > $OUT/v44_trace.log 2>&1
timeout 900 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py tests/test_gpu_mp.py tests/test_gpu_graded.py tests/test_gpu_config1_full.py > $OUT/v44_tests.log 2>&1; echo "rc=$?" >> $OUT/v44_tests.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/v44_bench.jsonl 2> $OUT/v44_bench.err
MPS_FO=0 timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/v44_bench_nofo.jsonl 2> $OUT/v44_bench_nofo.err
