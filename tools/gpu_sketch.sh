#!/bin/bash
# Sketch-only GPU cycle: sketch parity tests, per-shape timing, ncu of the C2 k=512 launch.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "sketch or c2_full or rng" > gpurun_out/pytest_sketch.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sketch.log
timeout 300 python tools/bench_sketch.py > gpurun_out/bench_sketch.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sketch.log
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_tma" -s 1 -c 1 -o gpurun_out/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
echo done
