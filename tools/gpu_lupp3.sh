#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "select or lupp or full or residual or id_coeffs or edges or dist" > gpurun_out/pytest_lupp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lupp.log
timeout 300 python tools/bench_lupp.py > gpurun_out/bench_lupp.log 2>&1
SKEL_LUPP_PROBE=1 timeout 300 python tools/bench_lupp.py --reps 1 > gpurun_out/probe.log 2>&1
