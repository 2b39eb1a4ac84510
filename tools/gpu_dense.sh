#!/bin/bash
# dense sketch: parity + per-shape timings (pre-generated Omega) + bench C2 / C5 / C4
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sketch or c2_full or c4 or rand_lupp or power or deim or c5" > gpurun_out/pytest_dense.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dense.log
timeout 300 python tools/bench_sketch.py --only "k=" > gpurun_out/dense_plain.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2k512.log 2>&1
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/bench_c5.log 2>&1
