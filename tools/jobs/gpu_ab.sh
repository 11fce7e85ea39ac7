#!/bin/bash
# One gpurun call of the build -> measure loop for a switchable path: a short parity check,
# then bench lines of the default library and with the switch set (A/B on one box).
#   bash tools/jobs/gpu_ab.sh <tag> <ENV=VALUE> [pytest targets...]
set -u
TAG=$1; AB=$2; shift 2
OUT=gpurun_out
mkdir -p $OUT
T=${@:-tests/test_gpu_update2.py}
timeout 900 python -m pytest -x -q $T > $OUT/ab_tests_$TAG.log 2>&1
rc=$?; echo "tests rc=$rc" >> $OUT/ab_tests_$TAG.log
if [ $rc -ne 0 ]; then echo "tests failed"; exit 1; fi
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_$TAG.jsonl 2> $OUT/ab_bench_$TAG.err
env $AB timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_alt.jsonl 2> $OUT/ab_bench_${TAG}_alt.err
echo done
