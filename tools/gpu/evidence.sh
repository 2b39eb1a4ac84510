#!/bin/bash
# Full evidence pass: tests, smoke, bench lines for every config, per-kernel benches.
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/ev_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
timeout 1500 python bench.py > gpurun_out/ev_bench_c5.log 2>&1
timeout 600 python bench.py --config C1 > gpurun_out/ev_bench_c1.log 2>&1
timeout 600 python bench.py --config C2 > gpurun_out/ev_bench_c2.log 2>&1
timeout 900 python bench.py --config C3 --steps 5 > gpurun_out/ev_bench_c3.log 2>&1
timeout 900 python bench.py --config C4 --steps 5 > gpurun_out/ev_bench_c4.log 2>&1
timeout 600 python bench.py --config C2 --piter 1 --steps 5 > gpurun_out/ev_bench_c2_1piter.log 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ev_bench_ref_c5.log 2>&1
timeout 300 python tools/bench_lupp.py > gpurun_out/ev_bench_lupp.log 2>&1
echo done
