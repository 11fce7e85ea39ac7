#!/bin/bash
# v59: A/B of development builds (short parity run + bench each), then the default bench line
# (e2e and cpu_baseline included) and the e2e-only A/B of the chunked copies.
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for v in "$@"; do
  name=${v%%=*}; so=${v#*=}
  MPS_B200_SO=$so timeout 900 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py > $OUT/ab_tests_${TAG}_$name.log 2>&1
  echo "tests rc=$?" >> $OUT/ab_tests_${TAG}_$name.log
  MPS_B200_SO=$so timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_$name.jsonl 2> $OUT/ab_bench_${TAG}_$name.err
done
timeout 1200 python bench.py > $OUT/bench_${TAG}_default.jsonl 2> $OUT/bench_${TAG}_default.err
MPS_E2E_CHUNK=0 timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/bench_${TAG}_e2e_onechunk.jsonl 2> $OUT/bench_${TAG}_e2e_onechunk.err
echo done
