#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_plans or sketch" > gpurun_out/chain_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/chain_pytest.log
bash tools/gpu/ab_libs.sh "C5 half" nochain chain3 nochain chain3
echo done
