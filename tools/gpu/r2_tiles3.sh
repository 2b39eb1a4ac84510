#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/sweep_pre.py > gpurun_out/t3_sweep.txt 2>&1
timeout 600 python tools/bench_sketch.py --only "C" --reps 5 > gpurun_out/t3_sketch.txt 2>&1
echo done
