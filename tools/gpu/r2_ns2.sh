#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2i_*
for c in "C2 col_id" "C3 cur" "C4 col_id"; do
  set -- $c
  SKEL_DEBUG_NS=1 timeout 300 python tools/probe_residual.py --config $1 --kind $2 --reps 2 >> gpurun_out/r2i_plain.log 2>&1
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2i_launch_c2.csv python tools/probe_residual.py --config C2 --kind col_id --reps 1 --profile > gpurun_out/r2i_ncu.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2i_launch_c4.csv python tools/probe_residual.py --config C4 --kind col_id --reps 1 --profile >> gpurun_out/r2i_ncu.log 2>&1
echo done
