#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "srtt" > gpurun_out/pytest_srtt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_srtt.log
timeout 300 python tools/bench_sketch.py --only "srtt" > gpurun_out/srtt_plain.log 2>&1
