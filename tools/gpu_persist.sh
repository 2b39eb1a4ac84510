#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/bench_sketch.py --only "k=" > gpurun_out/persist_off.log 2>&1
SKEL_PRE_PERSIST=1 timeout 300 python tools/bench_sketch.py --only "k=" > gpurun_out/persist_on.log 2>&1
SKEL_PRE_PERSIST=1 timeout 600 python -m pytest tests -m gpu -x -q -k "sketch or c2_full or c4 or c5 or residual" > gpurun_out/pt_persist.log 2>&1; echo rc=$? >> gpurun_out/pt_persist.log
