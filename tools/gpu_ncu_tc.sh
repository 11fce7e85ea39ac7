#!/bin/bash
# ncu --set full of one k_tc_mma launch of the P = Theta' X_2 GEMM (LG = 10) of a bench step, for
# the default library and (optionally) a development build.
#   bash tools/gpu_ncu_tc.sh <tag> [alt.so]
set -u
TAG=$1; ALT=${2:-}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncutc_plain_$TAG.log 2>&1 || { echo "plain bench failed"; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_tc_mma<.*10, .*0, .*10, .*36>' -s 14 -c 1 \
  -o $OUT/ncutc_${TAG}_default python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncutc_${TAG}_default.log 2>&1
if [ -n "$ALT" ]; then
  MPS_B200_SO=$ALT timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_tc_mma<.*10, .*0, .*10, .*36>' -s 14 -c 1 \
    -o $OUT/ncutc_${TAG}_alt python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncutc_${TAG}_alt.log 2>&1
fi
echo done
