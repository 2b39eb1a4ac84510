#!/bin/bash
# One GPU verification cycle: gpu tests, smoke, bench, then ncu of the kernels matching $1.
# usage (under gpurun): bash tools/gpu_cycle.sh '<kernel regex>' [extra bench args]
KRE=${1:-k_sketch_tma}
shift
EXTRA="$@"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py $EXTRA > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $EXTRA > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 1 -c 2 -o gpurun_out/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $EXTRA > gpurun_out/ncu_full.log 2>&1
echo cycle done
