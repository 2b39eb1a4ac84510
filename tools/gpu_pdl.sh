#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_lupp.py > gpurun_out/bench_lupp.log 2>&1
SKEL_NO_PDL=1 timeout 300 python tools/bench_lupp.py > gpurun_out/bench_lupp_nopdl.log 2>&1
