#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2m_*
timeout 1500 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_c5.py > gpurun_out/r2m_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2m_pytest.log
for v in "" 1; do
for c in "C2 col_id" "C3 cur" "C4 col_id" "C4 row_id"; do
  set -- $c
  if [ -z "$v" ]; then timeout 300 python tools/probe_residual.py --config $1 --kind $2 --reps 9 >> gpurun_out/r2m_plain.log 2>&1;
  else SKEL_CHOL_L2=1 timeout 300 python tools/probe_residual.py --config $1 --kind $2 --reps 9 >> gpurun_out/r2m_plain.log 2>&1; fi
done
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2m_launch_c2.csv python tools/probe_residual.py --config C2 --kind col_id --reps 1 --profile > gpurun_out/r2m_ncu.log 2>&1
echo done
