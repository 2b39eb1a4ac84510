#!/bin/bash
# Per-step-exchange LUPP on one B200: GPU parity tests + per-step timings.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist_step.py -x -q > gpurun_out/pytest_dist_step.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dist_step.log
timeout 600 python tools/bench_lupp_dist.py > gpurun_out/bench_lupp_dist.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_lupp_dist.log
