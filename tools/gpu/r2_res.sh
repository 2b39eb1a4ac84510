#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "residual or c2_full or c4_full or c3_full or dist_lib or sketch or smoke or estimates or c5_full or power" > gpurun_out/r2i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_pytest.log
timeout 900 python tools/sweep_pre.py C4 > gpurun_out/r2i_sweep_c4.log 2>&1
timeout 300 python tools/bench_sketch.py --only C > gpurun_out/r2i_sketch.log 2>&1
timeout 600 python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/r2i_bench_c2.log 2>&1
timeout 600 python bench.py --config C4 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r2i_bench_c4.log 2>&1
timeout 1500 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/r2i_bench_c5.log 2>&1
echo done
