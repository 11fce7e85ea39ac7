#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python tools/dbg_layers.py 3 9 $OUT/layers_sp.json > $OUT/bisect3.log 2>&1
MPS_JD_SP=0 timeout 600 python tools/dbg_layers.py 3 9 $OUT/layers_nosp.json >> $OUT/bisect3.log 2>&1
timeout 600 python tools/dbg_layers_cmp.py $OUT/layers_sp.json $OUT/layers_nosp.json >> $OUT/bisect3.log 2>&1
echo done
