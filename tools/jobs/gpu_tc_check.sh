#!/bin/bash
# First GPU run of the tensor-core GEMM path: small parity tests under a short timeout, then
# the full-size ones and the A/B bench (MPS_TC=1 default vs MPS_TC=0).
set -u
TAG=$1
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python -m pytest -x -q -rA tests/test_gpu_update2.py > $OUT/tc_small_$TAG.log 2>&1
rc=$?; echo "small rc=$rc" >> $OUT/tc_small_$TAG.log
if [ $rc -ne 0 ]; then echo "small tests failed rc=$rc"; exit 1; fi
timeout 1500 python -m pytest -q -rA tests/test_gpu_mp.py tests/test_gpu_mps.py tests/test_gpu_cfg1_golden.py tests/test_gpu_config1_full.py tests/test_gpu_configs.py "tests/test_gpu_variants.py::test_path_parity[MPS_TC]" > $OUT/tc_tests_$TAG.log 2>&1
echo "tests rc=$?" >> $OUT/tc_tests_$TAG.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_tc_$TAG.jsonl 2> $OUT/bench_tc_$TAG.err
MPS_TC=0 timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_notc_$TAG.jsonl 2> $OUT/bench_notc_$TAG.err
echo done
