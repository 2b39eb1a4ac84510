#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2h_*
timeout 900 python -m pytest tests -x -q -m gpu -k "residual or estimate or dist or cholqr or deim" --deselect tests/test_gpu_c5.py > gpurun_out/r2h_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2h_pytest.log
for v in "" 1; do
for c in "C2 col_id" "C3 cur" "C4 col_id" "C4 row_id"; do
  set -- $c
  SKEL_NO_NS=$v timeout 300 python tools/probe_residual.py --config $1 --kind $2 --reps 9 >> gpurun_out/r2h_plain.log 2>&1
done
done
echo done
