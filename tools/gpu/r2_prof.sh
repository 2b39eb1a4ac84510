#!/bin/bash
# round 2 evidence: C5 bench line, sketch chunk sweep, ncu launch list of one C5 step, ncu --set full of the sketch kernels
mkdir -p gpurun_out
for ch in 8192 16384 0; do echo "chunk $ch" >> gpurun_out/r2f_chunks.log; timeout 300 python tools/bench_sketch.py --only "C5 block" --tune 0,0,0,$ch >> gpurun_out/r2f_chunks.log 2>&1; done
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2f_bench_c5.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 $CMD > gpurun_out/r2f_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemm" -c 3000 --csv --log-file gpurun_out/r2f_launches_c5.csv $CMD > gpurun_out/r2f_ncu_launch.log 2>&1
timeout 900 $CMD > gpurun_out/r2f_plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_pre|k_omega_image" -c 3 -o gpurun_out/r2f_prof_c5 $CMD > gpurun_out/r2f_ncu_full.log 2>&1
echo done
