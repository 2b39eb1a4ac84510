#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/nw3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/nw3_pytest.log
timeout 900 python bench.py --config C4 --steps 5 > gpurun_out/nw3_bench_c4.log 2>&1
timeout 900 python tools/bench_sketch.py --only "C4" > gpurun_out/nw3_sketch.txt 2>&1
echo done
