set -u
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/tc_bisect.log
for b in 0 1 2 4 8 3 6; do
  echo "== bisect $b" >> $OUT/tc_bisect.log
  MPS_TC_BISECT=$b MPS_TC_DEBUG=1 timeout 120 python -m pytest -x -q "tests/test_gpu_update2.py::test_theta_contraction_parity" 2>&1 | grep "tc L\|passed\|failed" | head -8 >> $OUT/tc_bisect.log
done
