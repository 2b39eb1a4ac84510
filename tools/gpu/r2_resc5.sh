#!/bin/bash
mkdir -p gpurun_out
python tools/probe_residual_c5.py > gpurun_out/rc5_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/rc5_launches.csv python tools/probe_residual_c5.py --profile --reps 1 > gpurun_out/rc5_ncu.log 2>&1
echo done
