#!/bin/bash
# v62: R27 with the scaled binary32 copy and the unitarity fallback: hand-over checks on configs[3],
# full GPU suite, bench, launch list.
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT
T="tests/test_gpu_configs.py::test_config_vs_cached_oracle[cfg3_oracle_d9.json]"
MPS_JACOBI_TRACE=2001 timeout 600 python -m pytest -x -q -s "$T" 2>&1 | grep "hand-over check\|passed\|failed" > $OUT/handover_${TAG}.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_${TAG}_nocpu.jsonl 2> $OUT/bench_${TAG}_nocpu.err
timeout 1800 python -m pytest tests -m gpu -q > $OUT/gputests_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
MPS_E2E_TRACE=1 timeout 300 python tools/time_e2e.py 128 280 1024 2 > $OUT/e2e_${TAG}.log 2>&1
echo done
