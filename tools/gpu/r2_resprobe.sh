#!/bin/bash
# residual chain probes: plain timings, then an ncu launch list of one residual call per config
mkdir -p gpurun_out
for c in "C2 col_id" "C3 cur" "C4 col_id" "C4 row_id"; do
  set -- $c
  timeout 300 python tools/probe_residual.py --config $1 --kind $2 >> gpurun_out/r2r_plain.log 2>&1
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2r_launch_c2.csv python tools/probe_residual.py --config C2 --kind col_id --reps 1 --profile > gpurun_out/r2r_ncu.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2r_launch_c4.csv python tools/probe_residual.py --config C4 --kind row_id --reps 1 --profile >> gpurun_out/r2r_ncu.log 2>&1
echo done
