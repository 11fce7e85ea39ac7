#!/bin/bash
# ncu --set full with source correlation of ONE k_jacobi launch (296 items = one wave at C = 1,
# chi = 128, 280 bits) and the per-opcode instruction mix of the bench launch (1024 items), after
# the same command has exited 0 without ncu.  Usage: bash tools/gpu_ncu_source.sh <tag>
set -u
TAG=$1
OUT=gpurun_out
mkdir -p $OUT
python bench.py --steps 1 --warmup 1 --batch 296 --no-e2e --no-cpu > $OUT/plain296_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:'^k_jacobi$' -s 1 -c 1 -o $OUT/jac_$TAG \
    python bench.py --steps 1 --warmup 1 --batch 296 --no-e2e --no-cpu > $OUT/ncu_full_$TAG.log 2>&1
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/plain1024_$TAG.log 2>&1 || { echo "plain 1024 failed"; exit 1; }
ncu --metrics sass__inst_executed_per_opcode,smsp__inst_executed.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_alu.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --print-metric-instances details --clock-control none -k regex:'^k_jacobi$' -s 3 -c 1 --csv \
    --log-file $OUT/ncu_opcodes_$TAG.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_opc_$TAG.log 2>&1
echo done
