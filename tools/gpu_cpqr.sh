#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cpqr" > gpurun_out/pytest_cpqr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cpqr.log
timeout 300 python tools/bench_lupp.py > gpurun_out/bench_lupp.log 2>&1
