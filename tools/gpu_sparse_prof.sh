#!/bin/bash
# ncu of the sparse-sign sketch at C3 (16384^2, l=510): full set + source page.
mkdir -p gpurun_out
timeout 300 python tools/bench_sketch.py --only "C3 sparse" --reps 3 > gpurun_out/sparse_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_sparse" -s 1 -c 1 -o gpurun_out/prof_sparse python tools/bench_sketch.py --only "C3 sparse" --reps 1 > gpurun_out/ncu_sparse.log 2>&1
echo done
