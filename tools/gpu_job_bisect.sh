#!/bin/bash
# bisect a failing parity test over the path switches
set -u
OUT=gpurun_out; mkdir -p $OUT
T="tests/test_gpu_configs.py::test_config_vs_cached_oracle[cfg3_oracle_d9.json]"
: > $OUT/bisect.log
for sw in "X=1" "MPS_JD_SP=0" "MPS_XS_GEMM=0" "MPS_TC=0" "MPS_XSWEEP=0" "MPS_E2E_CHUNK=0"; do
  echo "== $sw" >> $OUT/bisect.log
  env $sw timeout 600 python -m pytest -x -q "$T" 2>&1 | grep -E "passed|failed|AssertionError: |assert mpf" | cut -c1-100 >> $OUT/bisect.log
done
echo done
