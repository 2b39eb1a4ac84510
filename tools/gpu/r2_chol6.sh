#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2g_*
timeout 900 python -m pytest tests -x -q -m gpu -k "residual or estimate or dist or cholqr or deim" --deselect tests/test_gpu_c5.py > gpurun_out/r2g_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2g_pytest.log
for c in "C2 col_id" "C3 cur" "C4 col_id" "C4 row_id"; do
  set -- $c
  timeout 300 python tools/probe_residual.py --config $1 --kind $2 --reps 9 >> gpurun_out/r2g_plain.log 2>&1
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2g_launch_c2.csv python tools/probe_residual.py --config C2 --kind col_id --reps 1 --profile > gpurun_out/r2g_ncu.log 2>&1
echo done
