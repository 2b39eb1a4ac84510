#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py tests/test_gpu_dist_lib.py -q -x > gpurun_out/ra_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ra_pytest.log
for cfg in "C2 col_id" "C3 cur" "C4 col_id" "C4 row_id"; do set -- $cfg; timeout 300 python tools/probe_residual.py --config $1 --kind $2 >> gpurun_out/ra_probe.txt 2>&1; done
timeout 900 python bench.py --config C4 --steps 5 > gpurun_out/ra_bench_c4.log 2>&1
timeout 900 python bench.py --config C3 --steps 5 > gpurun_out/ra_bench_c3.log 2>&1
echo done
