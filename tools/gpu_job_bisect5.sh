#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
T="tests/test_gpu_configs.py::test_config_vs_cached_oracle[cfg3_oracle_d9.json]"
: > $OUT/bisect5.log
for sw in "MPS_ACCUMULATE_V=1" "MPS_NO_CERT=1" "MPS_JD_SP=0 MPS_B200_SO=paper_1111_3124_b200/libmps_b200_tol.so" "MPS_JD_SP=0 MPS_ACCUMULATE_V=1 MPS_B200_SO=paper_1111_3124_b200/libmps_b200_tol.so"; do
  echo "== $sw" >> $OUT/bisect5.log
  env $sw timeout 600 python -m pytest -x -q "$T" 2>&1 | grep -E "passed|failed|AssertionError: |assert mpf" | cut -c1-100 >> $OUT/bisect5.log
done
echo done
