#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "rand_lupp" > gpurun_out/pytest_e2e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_e2e.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e.log 2>&1; echo "rc=$?" >> gpurun_out/bench_e2e.log
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_e2e_c3.log
