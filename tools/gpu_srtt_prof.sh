#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/bench_sketch.py --only "C3 srtt" --reps 2 > gpurun_out/b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_srtt" -s 1 -c 1 -o gpurun_out/prof_srtt python tools/bench_sketch.py --only "C3 srtt" --reps 1 > gpurun_out/ncu_srtt.log 2>&1
echo done
