#!/bin/bash
# binary32 first phase of the block Jacobi (R27): sweep trace, phase cycles, parity tests, A/B bench (MPS_JD_SP=0).
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT
MPS_JACOBI_TRACE=1001 timeout 300 python tools/trace_sweeps.py 128 280 8 > $OUT/trace_${TAG}_chi128_p280.log 2>&1
MPS_JD_PROF=1 timeout 300 python tools/trace_sweeps.py 128 280 148 > $OUT/jdprof_${TAG}.log 2>&1
MPS_JD_SP=0 MPS_JD_PROF=1 timeout 300 python tools/trace_sweeps.py 128 280 148 > $OUT/jdprof_${TAG}_nosp.log 2>&1
timeout 1500 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py tests/test_gpu_fo.py tests/test_gpu_xsgemm.py > $OUT/ab_tests_$TAG.log 2>&1
rc=$?; echo "tests rc=$rc" >> $OUT/ab_tests_$TAG.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_default.jsonl 2> $OUT/ab_bench_${TAG}_default.err
MPS_JD_SP=0 timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_alt.jsonl 2> $OUT/ab_bench_${TAG}_alt.err
echo done
