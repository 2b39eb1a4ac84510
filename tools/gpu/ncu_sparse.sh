#!/bin/bash
# ncu --set full of the C3 sparse-sign sketch kernel (k_sketch_sparse4)
mkdir -p gpurun_out
python tools/bench_sketch.py --only "C3 sparse" --reps 1 > gpurun_out/ncu_sp_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_sketch_sparse4 -s 2 -c 1 \
    -o gpurun_out/prof_sparse4 python tools/bench_sketch.py --only "C3 sparse" --reps 1 > gpurun_out/ncu_sp.log 2>&1
echo done
