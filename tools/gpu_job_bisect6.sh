#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
T="tests/test_gpu_configs.py::test_config_vs_cached_oracle[cfg3_oracle_d9.json]"
MPS_JACOBI_TRACE=2001 timeout 600 python -m pytest -x -q -s "$T" 2>&1 | grep "hand-over check\|block Jacobi (binary.*sweeps$" > $OUT/bisect6.log
echo done
