#!/bin/bash
# ncu --set full captures of the hot kernels of one C2 k=512 bench step; reports stay in /tmp on
# the box, only the text summaries come back
mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_all.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none \
  -k regex:"k_lupp_panel_v2|k_cpqr|k_lupp_u12|k_diag_inv|k_right_tri_mul|k_gemm|k_lupp_init" --launch-skip 0 --launch-count 24 \
  -o /tmp/prof_all python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_all.log 2>&1
python tools/ncu_summary.py /tmp/prof_all.ncu-rep > gpurun_out/ncu_all_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_sketch_srtt" -c 1 \
  -o /tmp/prof_srtt python tools/bench_sketch.py --only "C3 srtt" --reps 1 > gpurun_out/ncu_srtt.log 2>&1
python tools/ncu_summary.py /tmp/prof_srtt.ncu-rep > gpurun_out/ncu_srtt_summary.txt 2>&1
echo done
