#!/bin/bash
# ncu --set full captures of selected kernels of one bench launch (after the bench ran clean).
#   bash tools/gpu_ncu_full.sh <tag> <kernel-regex> <skip> [<kernel-regex> <skip> ...]
set -u
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncufull_plain_$TAG.log 2>&1 || { echo "plain bench failed"; exit 1; }
i=0
while [ $# -ge 2 ]; do
  K=$1; S=$2; shift 2
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 \
      -o $OUT/ncufull_${TAG}_$i python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncufull_${TAG}_$i.log 2>&1
  i=$((i+1))
done
echo done
