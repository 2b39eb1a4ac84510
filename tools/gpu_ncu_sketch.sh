#!/bin/bash
# ncu --set full of the sketch kernels at the bench configurations (C2 k=512 Gaussian, C3 sparse)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_omega_image|k_sketch_pre|k_sketch_splitk" -s 6 -c 3 -o gpurun_out/prof_pre python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_pre.log 2>&1
timeout 300 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sparse_csr|k_sketch_sparse4" -s 4 -c 2 -o gpurun_out/prof_sparse_c3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sparse_c3.log 2>&1
echo done
