set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 180 python -m pytest -x -q tests/test_gpu_update2.py > $OUT/tc2_small.log 2>&1; rc=$?; echo "rc=$rc" >> $OUT/tc2_small.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest -x -q tests/test_gpu_cfg1_golden.py tests/test_gpu_mp.py tests/test_gpu_graded.py tests/test_gpu_config1_full.py tests/test_gpu_mps.py > $OUT/tc2_tests.log 2>&1; echo "rc=$?" >> $OUT/tc2_tests.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/tc2_bench.jsonl 2> $OUT/tc2_bench.err
