#!/bin/bash
# One gpurun call of the build -> measure loop: GPU test suite, bench lines of the default
# library and of an A/B library (optional), whole-circuit timings.  Usage on the GPU box:
#   bash tools/jobs/gpu_check.sh <tag> [ab_library.so] [extra pytest args]
set -u
TAG=$1
AB=${2:-}
OUT=gpurun_out
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q ${3:-} > $OUT/gputests_$TAG.log 2>&1
echo "pytest rc=$?" >> $OUT/gputests_$TAG.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_$TAG.jsonl 2> $OUT/bench_$TAG.err
if [ -n "$AB" ]; then
  MPS_B200_SO=$PWD/$AB timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_${TAG}_ab.jsonl 2> $OUT/bench_${TAG}_ab.err
fi
timeout 600 python tools/time_configs.py > $OUT/config_times_$TAG.jsonl 2> $OUT/config_times_$TAG.err
timeout 600 python tools/time_configs.py --config 3 --depth 16 >> $OUT/config_times_$TAG.jsonl 2>> $OUT/config_times_$TAG.err
echo done
