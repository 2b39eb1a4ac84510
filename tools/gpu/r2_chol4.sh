#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2f_*
SKEL_CHOL_MASK=15 timeout 300 python tools/probe_residual.py --config C2 --kind col_id --reps 3 > gpurun_out/r2f_plain.log 2>&1
SKEL_CHOL_DREG=1 SKEL_CHOL_MASK=15 timeout 300 python tools/probe_residual.py --config C2 --kind col_id --reps 3 >> gpurun_out/r2f_plain.log 2>&1
echo done
