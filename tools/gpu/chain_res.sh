#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/probe_residual_c5.py --m 131072 --noise 0 --reps 2 > gpurun_out/chain_res_c5.log 2>&1
timeout 600 python tools/sweep_pre.py > gpurun_out/chain_sweep.txt 2>&1
timeout 600 python tools/bench_sketch.py --only "C" > gpurun_out/chain_sketch_all.txt 2>&1
echo done
