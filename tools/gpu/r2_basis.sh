#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2j_*
SKEL_BASIS=1 timeout 900 python -m pytest tests -q -m gpu -k "residual or estimate or cur" --deselect tests/test_gpu_c5.py > gpurun_out/r2j_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2j_pytest.log
for v in 0 1; do
for c in "C2 col_id" "C3 cur" "C4 col_id" "C4 row_id"; do
  set -- $c
  SKEL_BASIS=$v SKEL_DEBUG_NS=1 timeout 300 python tools/probe_residual.py --config $1 --kind $2 --reps 9 >> gpurun_out/r2j_plain.log 2>&1
done
done
echo done
