#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2l_*
timeout 900 python -m pytest tests -q -m gpu -k "host or dual or pipelined or chunk or e2e" --deselect tests/test_gpu_c5.py > gpurun_out/r2l_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2l_pytest.log
timeout 1500 python bench.py --steps 2 --warmup 1 > gpurun_out/r2l_bench_c5.log 2>&1
timeout 600 python bench.py --config C2 --steps 3 > gpurun_out/r2l_bench_c2.log 2>&1
echo done
