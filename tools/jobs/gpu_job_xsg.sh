#!/bin/bash
# GEMM form of the refinement sweeps (R26): parity tests, sweep trace, A/B bench against MPS_XS_GEMM=0.
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT
MPS_JACOBI_TRACE=4 timeout 300 python tools/trace_sweeps.py 128 280 8 > $OUT/trace_${TAG}_chi128_p280.log 2>&1
MPS_JACOBI_TRACE=2 timeout 300 python tools/trace_sweeps.py 64 512 4 > $OUT/trace_${TAG}_chi64_p512.log 2>&1
timeout 1500 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py tests/test_gpu_fo.py tests/test_gpu_graded.py tests/test_gpu_variants.py tests/test_gpu_mps.py tests/test_gpu_configs.py > $OUT/ab_tests_$TAG.log 2>&1
rc=$?; echo "tests rc=$rc" >> $OUT/ab_tests_$TAG.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_default.jsonl 2> $OUT/ab_bench_${TAG}_default.err
MPS_XS_GEMM=0 timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_alt.jsonl 2> $OUT/ab_bench_${TAG}_alt.err
echo done
