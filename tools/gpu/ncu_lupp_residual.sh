#!/bin/bash
# ncu --set full of the LUPP and residual kernels on the round-2 head: one C2 k=512 step (single-cluster
# panel, U12, the Cholesky pair, the row solves, the Gram / sum-of-squares GEMMs) and the tall panels
# (C4 rows, C5 columns / rows: 4 and 32 co-resident clusters).  Summaries -> profiles/round2/ncu_lupp_residual/.
O=gpurun_out/ncu7; R=/tmp/ncu7; mkdir -p $O $R   # reports stay on the box (gpurun_out is capped at 64 MiB); summaries come back
KR='regex:k_lupp_panel_v2|k_lupp_u12|k_potrf_cluster|k_trsm_rows|k_sketch_pre|k_gemm|k_newton'
timeout 600 python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/plain_c2.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on -k "$KR" -c 60 -f -o $R/prof_c2 \
    python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_c2.log 2>&1
python tools/ncu_summary.py $R/prof_c2.ncu-rep > $O/ncu_c2_summary.txt 2>&1
timeout 600 python tools/bench_lupp_tall.py > $O/plain_tall.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_lupp_panel_v2 -c 8 -f -o $R/prof_tall \
    python tools/bench_lupp_tall.py > $O/ncu_tall.log 2>&1
python tools/ncu_summary.py $R/prof_tall.ncu-rep > $O/ncu_tall_summary.txt 2>&1
ls -la $O $R
echo done
