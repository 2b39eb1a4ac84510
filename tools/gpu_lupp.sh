#!/bin/bash
# LUPP cycle: LUPP/CPQR parity tests, per-shape timing, launch list + ncu of the panel kernel.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "select or lupp or cpqr or id_coeffs or residual or full" > gpurun_out/pytest_lupp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lupp.log
timeout 300 python tools/bench_lupp.py > gpurun_out/bench_lupp.log 2>&1; echo "rc=$?" >> gpurun_out/bench_lupp.log
SKEL_LUPP_NO_LOOKAHEAD=1 timeout 300 python tools/bench_lupp.py > gpurun_out/bench_lupp_nola.log 2>&1
timeout 300 python tools/bench_sketch.py --reps 5 > gpurun_out/bench_sketch.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lupp_panel" -s 2 -c 1 -o gpurun_out/prof_lupp python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_lupp.log 2>&1
echo done
