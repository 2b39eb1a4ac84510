#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"k_omega_image|k_sketch_pre|k_sketch_splitk" -s 9 -c 3 -o /tmp/prof_pre python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_pre.log 2>&1
python tools/ncu_summary.py /tmp/prof_pre.ncu-rep > gpurun_out/ncu_sketch_pre.txt 2>&1
echo done
