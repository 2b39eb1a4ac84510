#!/bin/bash
mkdir -p gpurun_out
T=tests/test_gpu_parity.py::test_sketch_dense_plans
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest -q -x "$T[plan19]" > gpurun_out/n40c_pytest.txt 2>&1
timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import tests.test_gpu_parity as t
t.test_sketch_dense_plans((0,40,1,0,2)); print('direct ok')" > gpurun_out/n40c_direct.txt 2>&1
timeout 120 python tools/probe_n40.py 1000 700 61 > gpurun_out/n40c_probe.txt 2>&1
echo done
