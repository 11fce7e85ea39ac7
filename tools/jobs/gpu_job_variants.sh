#!/bin/bash
# A/B of development builds (MPS_B200_SO) on one box: for each library a short parity run and a
# bench line.   bash tools/jobs/gpu_job_variants.sh <tag> <name=path.so> ...
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
MPS_JACOBI_TRACE=4 timeout 300 python tools/trace_sweeps.py 128 280 8 > $OUT/trace_${TAG}_chi128_p280.log 2>&1
for v in "$@"; do
  name=${v%%=*}; so=${v#*=}
  MPS_B200_SO=$so timeout 900 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py > $OUT/ab_tests_${TAG}_$name.log 2>&1
  echo "tests rc=$?" >> $OUT/ab_tests_${TAG}_$name.log
  MPS_B200_SO=$so timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_$name.jsonl 2> $OUT/ab_bench_${TAG}_$name.err
done
echo done
