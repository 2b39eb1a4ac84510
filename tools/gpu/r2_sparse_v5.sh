#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu/r2_sparse_ab.sh eg2 v6 eg2 v6
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py -q -k "sparse or c3" > gpurun_out/sp6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sp6_pytest.log
echo done
