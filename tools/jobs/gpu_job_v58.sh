#!/bin/bash
# v58: A/B of development builds (tests + bench each), then launch list of the default build.
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for v in "$@"; do
  name=${v%%=*}; so=${v#*=}
  MPS_B200_SO=$so timeout 900 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py tests/test_gpu_fo.py > $OUT/ab_tests_${TAG}_$name.log 2>&1
  echo "tests rc=$?" >> $OUT/ab_tests_${TAG}_$name.log
  MPS_B200_SO=$so timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_$name.jsonl 2> $OUT/ab_bench_${TAG}_$name.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/launches_$TAG.log 2>&1
echo done
