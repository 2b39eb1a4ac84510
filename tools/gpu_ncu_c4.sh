#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/bench_sketch.py --only "C4 k=200" --reps 2 > gpurun_out/c4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"k_sketch_pre|k_omega_image|k_sketch_splitk" -s 3 -c 3 -o /tmp/prof_c4 python tools/bench_sketch.py --only "C4 k=200" --reps 1 > gpurun_out/ncu_c4.log 2>&1
python tools/ncu_summary.py /tmp/prof_c4.ncu-rep > gpurun_out/ncu_c4_summary.txt 2>&1
ncu -i /tmp/prof_c4.ncu-rep --page raw --csv > gpurun_out/ncu_c4_raw.csv 2>/dev/null
echo done
