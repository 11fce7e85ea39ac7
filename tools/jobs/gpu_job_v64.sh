#!/bin/bash
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT
MPS_JACOBI_TRACE=1001 timeout 300 python tools/trace_sweeps.py 128 280 8 2>&1 | grep "block Jacobi\|sweeps {\|first-order" > $OUT/trace_${TAG}.log
timeout 1500 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py tests/test_gpu_fo.py tests/test_gpu_graded.py tests/test_gpu_configs.py tests/test_gpu_xsgemm.py > $OUT/tests_$TAG.log 2>&1
echo "tests rc=$?" >> $OUT/tests_$TAG.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_${TAG}_nocpu.jsonl 2> $OUT/bench_${TAG}_nocpu.err
echo done
