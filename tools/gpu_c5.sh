#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c5.py -x -q > gpurun_out/pytest_c5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c5.log
timeout 900 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 600 python bench.py --config C3 --steps 3 --warmup 1 > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> gpurun_out/bench_c5.log
echo done
