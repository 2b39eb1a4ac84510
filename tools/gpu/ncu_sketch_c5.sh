#!/bin/bash
# ncu --set full of one C5-block chunk GEMM of the dense sketch (k_sketch_pre<48,8,0>), source-level.
mkdir -p gpurun_out
python tools/bench_sketch.py --only "C5 block" --reps 1 > gpurun_out/ncu_c5_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_sketch_pre -s 2 -c 1 \
    -o gpurun_out/prof_c5pre python tools/bench_sketch.py --only "C5 block" --reps 1 > gpurun_out/ncu_c5.log 2>&1
echo done
