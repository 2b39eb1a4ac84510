#!/bin/bash
# sparse sketch: parity tests + C3 timing (+ ncu if $1 == prof)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sparse" > gpurun_out/pytest_sparse.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sparse.log
timeout 300 python tools/bench_sketch.py --only "sparse" --reps 5 > gpurun_out/sparse_plain.log 2>&1
SKEL_SPARSE_NW=16 timeout 300 python tools/bench_sketch.py --only "sparse" --reps 5 >> gpurun_out/sparse_plain.log 2>&1
if [ "$1" == "prof" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_sparse|k_sparse_csr" -s 2 -c 2 -o gpurun_out/prof_sparse4 python tools/bench_sketch.py --only "C3 sparse" --reps 1 > gpurun_out/ncu_sparse.log 2>&1
fi
echo done
