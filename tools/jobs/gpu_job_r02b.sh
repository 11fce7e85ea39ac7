#!/bin/bash
# Round-2 re-entry job: GPU suite + smoke, compute-sanitizer on small cases, configs[4] depth-40 timing.
set -u
OUT=gpurun_out; mkdir -p $OUT
TAG=${1:-r02b}
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gputests_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_case.py cfg0 cfg1 > $OUT/sanitizer_memcheck_$TAG.log 2>&1; echo "rc=$?" >> $OUT/sanitizer_memcheck_$TAG.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_case.py cfg0 cfg1 > $OUT/sanitizer_synccheck_$TAG.log 2>&1; echo "rc=$?" >> $OUT/sanitizer_synccheck_$TAG.log
timeout 600 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_case.py cfg0 > $OUT/sanitizer_racecheck_$TAG.log 2>&1; echo "rc=$?" >> $OUT/sanitizer_racecheck_$TAG.log
timeout 2400 python tools/time_configs.py --config 4 --depth 40 > $OUT/cfg4_depth40_$TAG.jsonl 2> $OUT/cfg4_depth40_$TAG.err
echo "cfg4 rc=$?" >> $OUT/cfg4_depth40_$TAG.err
