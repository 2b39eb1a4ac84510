#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "sparse or c3" > gpurun_out/pytest_sparse.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sparse.log
timeout 300 python tools/bench_sketch.py --only sparse --reps 5 > gpurun_out/bench_sparse.log 2>&1
SKEL_SPARSE_V2=1 timeout 300 python tools/bench_sketch.py --only sparse --reps 3 >> gpurun_out/bench_sparse.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_sparse" -s 1 -c 1 -o gpurun_out/prof_sparse python tools/bench_sketch.py --only sparse --reps 1 > gpurun_out/ncu_sparse.log 2>&1
echo done
