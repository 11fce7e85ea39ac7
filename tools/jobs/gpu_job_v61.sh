#!/bin/bash
# v61: packed drain (TC_PACKED): sweep trace, full GPU suite, bench, launch list.
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT
MPS_JACOBI_TRACE=1001 timeout 300 python tools/trace_sweeps.py 128 280 8 2>&1 | grep "block Jacobi\|sweep \|sweeps {" > $OUT/trace_${TAG}.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_${TAG}_nocpu.jsonl 2> $OUT/bench_${TAG}_nocpu.err
timeout 1800 python -m pytest tests -m gpu -q > $OUT/gputests_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/launches_$TAG.log 2>&1
echo done
