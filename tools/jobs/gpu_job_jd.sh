set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest -x -q tests/test_gpu_update2.py tests/test_gpu_cfg1_golden.py tests/test_gpu_graded.py > $OUT/jd_tests.log 2>&1; echo "rc=$?" >> $OUT/jd_tests.log
MPS_JD_PROF=1 timeout 300 python tools/trace_sweeps.py 128 280 296 > $OUT/jd_prof.log 2>&1
MPS_B200_SO=$PWD/paper_1111_3124_b200/libmps_b200_nocross.so MPS_JD_PROF=1 timeout 300 python tools/trace_sweeps.py 128 280 296 > $OUT/jd_prof_nocross.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/jd_bench.jsonl 2> $OUT/jd_bench.err
MPS_B200_SO=$PWD/paper_1111_3124_b200/libmps_b200_nocross.so timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/jd_bench_nocross.jsonl 2> $OUT/jd_bench_nocross.err
