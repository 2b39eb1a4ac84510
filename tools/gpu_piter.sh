#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "power or piter or sketch" > gpurun_out/pytest_piter.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_piter.log
timeout 300 python bench.py --piter 1 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_piter.log 2>&1
echo done
