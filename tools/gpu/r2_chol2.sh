#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2d_*
timeout 900 python -m pytest tests -x -q -m gpu -k "residual or estimate or dist or cholqr or deim" --deselect tests/test_gpu_c5.py > gpurun_out/r2d_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
for v in "" 1; do
  for c in "C2 col_id" "C4 col_id"; do
    set -- $c
    SKEL_CHOL_DREG=$v timeout 300 python tools/probe_residual.py --config $1 --kind $2 >> gpurun_out/r2d_plain.log 2>&1
  done
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2d_launch_c2.csv python tools/probe_residual.py --config C2 --kind col_id --reps 1 --profile > gpurun_out/r2d_ncu.log 2>&1
echo done
