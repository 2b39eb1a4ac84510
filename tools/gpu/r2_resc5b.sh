#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/probe_residual_c5.py > gpurun_out/rc5b_plain.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "dense_plans or residual" > gpurun_out/rc5b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rc5b_pytest.log
timeout 600 python tools/sweep_pre.py C5 > gpurun_out/rc5b_sweep.txt 2>&1
echo done
