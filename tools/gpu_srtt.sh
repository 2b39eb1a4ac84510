#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "srtt or sketch_dense or sparse" > gpurun_out/pytest_srtt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_srtt.log
timeout 300 python tools/bench_sketch.py --only srtt --reps 5 > gpurun_out/bench_srtt.log 2>&1
echo done
