#!/bin/bash
# compute-sanitizer memcheck (one tool) over the small GPU parity cases of the round-2 code paths
mkdir -p gpurun_out
K="sketch_dense_plans or (sketch_dual and 1000) or alg3_sketch_only or (sketch_power_ortho and 256) or id_coeffs_parity or id_coeffs_spec or select_cols_ties or select_cols_rank or (select_cols_parity and 256-40) or (select_rows_parity and 500) or gather_cols_bitwise or (cpqr_parity and 26)"
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" > gpurun_out/r2n_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_memcheck.log
echo done
