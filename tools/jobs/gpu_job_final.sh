#!/bin/bash
# End-of-round job: full GPU suite + smoke, default bench line, reference arm, 512-bit line, launch
# list of one bench step and ncu --set full captures of the two dominant kernels.
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/gputests_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 1200 python bench.py > $OUT/bench_${TAG}_default.jsonl 2> $OUT/bench_${TAG}_default.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_${TAG}_reference.jsonl 2> $OUT/bench_${TAG}_reference.err
timeout 900 python bench.py --chi 128 --prec 512 --steps 2 --warmup 3 --no-cpu > $OUT/bench_${TAG}_chi128_p512.jsonl 2> $OUT/bench_${TAG}_chi128_p512.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/launches_$TAG.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_jacobi_blk<float>' -s 3 -c 1 \
  -o $OUT/ncu_${TAG}_jsp python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_${TAG}_jsp.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_tc_mma<.*10, .*0, .*10, .*36>' -s 10 -c 1 \
  -o $OUT/ncu_${TAG}_tcmma python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_${TAG}_tcmma.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_jacobi_blk<double>' -s 3 -c 1 \
  -o $OUT/ncu_${TAG}_jdb python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_${TAG}_jdb.log 2>&1
echo done
