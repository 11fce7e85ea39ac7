#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
T="tests/test_gpu_configs.py::test_config_vs_cached_oracle[cfg3_oracle_d9.json]"
MPS_JACOBI_TRACE=1 timeout 600 python -m pytest -x -q -s "$T" > $OUT/bisect2_sp.log 2>&1
MPS_JD_SP=0 MPS_JACOBI_TRACE=1 timeout 600 python -m pytest -x -q -s "$T" > $OUT/bisect2_nosp.log 2>&1
echo done
