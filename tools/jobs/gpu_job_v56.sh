#!/bin/bash
# v56: full GPU suite + smoke on the default build, launch list of one bench step, bench lines of
# development builds.   bash tools/jobs/gpu_job_v56.sh <tag> [name=path.so ...]
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_${TAG}_nocpu.jsonl 2> $OUT/bench_${TAG}_nocpu.err
for v in "$@"; do
  name=${v%%=*}; so=${v#*=}
  MPS_B200_SO=$so timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ab_bench_${TAG}_$name.jsonl 2> $OUT/ab_bench_${TAG}_$name.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/launches_$TAG.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $OUT/gputests_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
echo done
