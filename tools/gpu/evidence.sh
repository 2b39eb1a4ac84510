#!/bin/bash
# Full evidence pass: tests, smoke, bench lines for every config, per-kernel benches, launch list.
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2k512.log 2>&1
timeout 600 python bench.py --config C1 > gpurun_out/bench_c1.log 2>&1
timeout 900 python bench.py --config C3 --steps 5 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --config C4 --steps 5 > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --piter 1 --steps 5 > gpurun_out/bench_c2_1piter.log 2>&1
timeout 300 python tools/bench_sketch.py > gpurun_out/bench_sketch.log 2>&1
timeout 300 python tools/bench_lupp.py > gpurun_out/bench_lupp.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo done
