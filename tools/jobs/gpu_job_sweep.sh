#!/bin/bash
# configs[1] sweep and whole-circuit timings at the end of the round, then the path-variant tests
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/sweep_$TAG.jsonl
for cfg in "64 280 1024" "256 280 296" "32 280 1024" "64 512 1024" "256 512 148"; do
  set -- $cfg
  timeout 900 python bench.py --chi $1 --prec $2 --batch $3 --steps 2 --warmup 3 --no-e2e --no-cpu >> $OUT/sweep_$TAG.jsonl 2>> $OUT/sweep_$TAG.err
done
: > $OUT/config_times_$TAG.jsonl
timeout 600 python tools/time_configs.py --config 2 >> $OUT/config_times_$TAG.jsonl 2>> $OUT/config_times_$TAG.err
timeout 600 python tools/time_configs.py --config 3 --depth 9 >> $OUT/config_times_$TAG.jsonl 2>> $OUT/config_times_$TAG.err
timeout 600 python tools/time_configs.py --config 3 --depth 16 >> $OUT/config_times_$TAG.jsonl 2>> $OUT/config_times_$TAG.err
timeout 1500 python -m pytest -q tests/test_gpu_variants.py tests/test_gpu_xsgemm.py tests/test_gpu_fo.py > $OUT/tests_variants_$TAG.log 2>&1
echo "tests rc=$?" >> $OUT/tests_variants_$TAG.log
echo done
