#!/bin/bash
# tensor-core GEMMs at 512 bits: parity tests, A/B bench at chi = 64 / 512 bits (MPS_TC=0), configs[4] depth-12 timing
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py tests/test_gpu_graded.py tests/test_gpu_cfg5_pins.py tests/test_gpu_configs.py tests/test_gpu_mp.py tests/test_gpu_cert.py > $OUT/tests_$TAG.log 2>&1
echo "tests rc=$?" >> $OUT/tests_$TAG.log
timeout 900 python bench.py --chi 64 --prec 512 --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_${TAG}_p512.jsonl 2> $OUT/bench_${TAG}_p512.err
MPS_TC=0 timeout 900 python bench.py --chi 64 --prec 512 --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/bench_${TAG}_p512_notc.jsonl 2> $OUT/bench_${TAG}_p512_notc.err
timeout 900 python tools/time_configs.py --config 4 --depth 14 > $OUT/cfg4_d14_$TAG.jsonl 2> $OUT/cfg4_d14_$TAG.err
echo done
