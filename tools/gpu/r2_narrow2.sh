#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "dense_plans" > gpurun_out/nw2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/nw2_pytest.log
timeout 1500 python tools/sweep_pre.py > gpurun_out/nw2_sweep.txt 2>&1
echo done
