#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_c5.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py -q -x > gpurun_out/chain_c5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/chain_c5_pytest.log
timeout 1500 python bench.py > gpurun_out/chain_bench_c5.log 2>&1
echo done
