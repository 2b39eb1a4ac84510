#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_potrf_cluster|k_trsm_rows" -c 2 \
  -o gpurun_out/r2c_full -f python tools/probe_residual.py --config C2 --kind col_id --reps 1 --profile > gpurun_out/r2c_ncu_full.log 2>&1
echo done
