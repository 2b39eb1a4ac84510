#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sketch or c2_full or c4 or rand_lupp or power or deim" > gpurun_out/pytest_dense.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dense.log
timeout 300 python tools/bench_sketch.py --only "k=" > gpurun_out/dense_plain.log 2>&1
echo "--- no cluster reduce" >> gpurun_out/dense_plain.log
SKEL_PRE_NO_CLUSTER=1 timeout 300 python tools/bench_sketch.py --only "k=" >> gpurun_out/dense_plain.log 2>&1
timeout 1000 python tools/sweep_pre.py > gpurun_out/sweep_pre2.txt 2>&1
