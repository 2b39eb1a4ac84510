#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2o_*
timeout 1500 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_c5.py > gpurun_out/r2o_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2o_pytest.log
for c in "C2 col_id" "C3 cur" "C4 col_id" "C4 row_id"; do
  set -- $c
  timeout 300 python tools/probe_residual.py --config $1 --kind $2 --reps 9 >> gpurun_out/r2o_plain.log 2>&1
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2o_launch_c4.csv python tools/probe_residual.py --config C4 --kind col_id --reps 1 --profile > gpurun_out/r2o_ncu.log 2>&1
echo done
