#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "residual or c2_full or c4_full or c3_full or dist_lib or estimates or id_coeffs or c1 or smoke or stream" > gpurun_out/r2m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_pytest.log
timeout 900 python bench.py --config C3 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r2m_bench_c3.log 2>&1
timeout 900 python bench.py --config C4 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r2m_bench_c4.log 2>&1
timeout 900 python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/r2m_bench_c2.log 2>&1
echo done
