#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
T="tests/test_gpu_configs.py::test_config_vs_cached_oracle[cfg3_oracle_d9.json]"
: > $OUT/bisect4.log
for sw in "MPS_JD_SP_SWEEPS=0" "MPS_JD_SP_SWEEPS=1" "MPS_JD_SP_SWEEPS=3" "MPS_JD_SP_SWEEPS=6" "MPS_JD_SP_SWEEPS=40"; do
  echo "== $sw" >> $OUT/bisect4.log
  env $sw timeout 600 python -m pytest -x -q "$T" 2>&1 | grep -E "passed|failed|AssertionError: |assert mpf" | cut -c1-100 >> $OUT/bisect4.log
done
echo done
