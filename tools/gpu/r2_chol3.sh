#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2e_*
for v in "" 1; do
for m in 7 1 0; do
  echo "dreg=$v mask $m" >> gpurun_out/r2e_plain.log
  SKEL_CHOL_DREG=$v SKEL_CHOL_MASK=$m timeout 300 python tools/probe_residual.py --config C2 --kind col_id --reps 9 >> gpurun_out/r2e_plain.log 2>&1
done
done
echo blocked >> gpurun_out/r2e_plain.log
SKEL_BLOCKED_CHOL=1 timeout 300 python tools/probe_residual.py --config C2 --kind col_id --reps 9 >> gpurun_out/r2e_plain.log 2>&1
echo done
