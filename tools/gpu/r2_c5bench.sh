#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/c5b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c5b_pytest.log
timeout 1500 python bench.py > gpurun_out/c5b_bench.log 2>&1
timeout 600 python bench.py --config C2 > gpurun_out/c5b_bench_c2.log 2>&1
echo done
