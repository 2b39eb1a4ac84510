#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "sketch_dense_plans or c4_full" > gpurun_out/r2h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_pytest.log
timeout 900 python tools/sweep_pre.py C4 > gpurun_out/r2h_sweep_c4.log 2>&1
timeout 300 python tools/bench_sketch.py --only C > gpurun_out/r2h_sketch.log 2>&1
echo done
