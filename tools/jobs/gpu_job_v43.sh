set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py tests/test_gpu_cert.py tests/test_gpu_mp.py > $OUT/v43_tests.log 2>&1; echo "rc=$?" >> $OUT/v43_tests.log
MPS_JACOBI_PHASES=1 timeout 600 python tools/trace_sweeps.py 128 280 296 > $OUT/v43_phases.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/v43_bench.jsonl 2> $OUT/v43_bench.err
