#!/bin/bash
# round 2: chunked-Omega sketch -- parity, per-shape timing, C5 bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sketch or c2_full or c4_full" > gpurun_out/r2s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_pytest.log
timeout 600 python tools/bench_sketch.py > gpurun_out/r2s_bench_sketch.log 2>&1
for t in "0,40,0,0" "0,48,0,0" "0,64,0,0" "0,48,0,65536"; do echo "tune $t" >> gpurun_out/r2s_bench_sketch_c4.log; timeout 300 python tools/bench_sketch.py --only C4 --tune $t >> gpurun_out/r2s_bench_sketch_c4.log 2>&1; done
timeout 1200 python bench.py --steps 3 --warmup 2 > gpurun_out/r2s_bench_c5.log 2>&1
echo done
