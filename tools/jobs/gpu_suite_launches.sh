#!/bin/bash
# One gpurun call: the full GPU test suite, smoke(), and the launch list of one bench step.
#   bash tools/jobs/gpu_suite_launches.sh <tag>
set -u
TAG=${1:-cur}
OUT=gpurun_out
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q > $OUT/gputests_$TAG.log 2>&1
echo "pytest rc=$?" >> $OUT/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launches_$TAG.log 2>&1
echo done
