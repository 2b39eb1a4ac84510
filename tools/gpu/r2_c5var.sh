#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/c5var_$i.log 2>&1; done
timeout 900 python tools/probe_residual_c5.py --m 131072 --noise 0 --reps 2 > gpurun_out/c5var_probe.log 2>&1
echo done
