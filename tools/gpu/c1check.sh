#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/probe_c1_sketch.py > gpurun_out/c1probe.txt 2>&1
timeout 600 python bench.py --config C1 > gpurun_out/c1bench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_plans or chained or sketch" > gpurun_out/c1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c1_pytest.log
bash tools/gpu/ab_libs.sh "C5 half" chain3 tileord
echo done
