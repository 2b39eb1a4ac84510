#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sketch or c5_full or c2_full or c4_full or dist_lib" > gpurun_out/r2e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_pytest.log
for ch in 2048 4096 8192 0; do echo "chunk $ch" >> gpurun_out/r2e_chunks.log; timeout 300 python tools/bench_sketch.py --only "C5 block" --tune 0,0,0,$ch >> gpurun_out/r2e_chunks.log 2>&1; done
timeout 300 python tools/bench_sketch.py >> gpurun_out/r2e_sketch_all.log 2>&1
echo done
