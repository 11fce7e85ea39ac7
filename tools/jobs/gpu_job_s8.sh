#!/bin/bash
# A/B of a development build of the library (MPS_B200_SO) against the default one on one box:
# parity tests with the alternative build, then bench lines of both.
#   bash tools/jobs/gpu_job_s8.sh <tag> <alt .so> [pytest targets...]
set -u
TAG=$1; ALT=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
T=${@:-tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py tests/test_gpu_fo.py tests/test_gpu_graded.py}
MPS_B200_SO=$ALT timeout 1200 python -m pytest -x -q $T > $OUT/ab_tests_$TAG.log 2>&1
rc=$?; echo "tests rc=$rc" >> $OUT/ab_tests_$TAG.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_default.jsonl 2> $OUT/ab_bench_${TAG}_default.err
MPS_B200_SO=$ALT timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_alt.jsonl 2> $OUT/ab_bench_${TAG}_alt.err
echo done
