#!/bin/bash
# Re-entry check of HEAD: full GPU suite, smoke, C2/C3/C4/C5 bench lines.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/h_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/h_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/h_smoke.log
timeout 600 python bench.py --config C2 > gpurun_out/h_bench_c2.log 2>&1
timeout 900 python bench.py --config C3 --steps 5 > gpurun_out/h_bench_c3.log 2>&1
timeout 900 python bench.py --config C4 --steps 5 > gpurun_out/h_bench_c4.log 2>&1
timeout 1500 python bench.py > gpurun_out/h_bench_c5.log 2>&1
echo done
