#!/bin/bash
# v60: norm-window variants of the binary32 phase, e2e chunking A/B.
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for c in 0 296 512; do MPS_E2E_CHUNK=$c timeout 300 python tools/time_e2e.py 128 280 1024 3 >> $OUT/e2e_${TAG}.log 2>&1; done
for v in "$@"; do
  name=${v%%=*}; so=${v#*=}
  MPS_B200_SO=$so MPS_JACOBI_TRACE=4 timeout 300 python tools/trace_sweeps.py 128 280 8 2>&1 | grep "block Jacobi\|sweeps {" > $OUT/trace_${TAG}_$name.log
  MPS_B200_SO=$so timeout 900 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py > $OUT/ab_tests_${TAG}_$name.log 2>&1
  echo "tests rc=$?" >> $OUT/ab_tests_${TAG}_$name.log
  MPS_B200_SO=$so timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_$name.jsonl 2> $OUT/ab_bench_${TAG}_$name.err
done
echo done
