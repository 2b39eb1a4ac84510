#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "dual or estimates or power or sketch_cols or stream_select or abi" > gpurun_out/r2c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_pytest.log
timeout 600 python bench.py --config C2 --piter 1 --steps 5 --warmup 3 > gpurun_out/r2c_bench_c2_piter.log 2>&1
timeout 300 python tools/bench_dual.py > gpurun_out/r2c_dual.log 2>&1
echo done
