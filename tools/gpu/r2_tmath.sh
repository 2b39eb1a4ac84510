#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r2k_*
for t in 512 256 128; do
for c in "C3 cur" "C4 col_id" "C4 row_id" "C3 col_id"; do
  set -- $c
  echo "kmin $t" >> gpurun_out/r2k_plain.log
  SKEL_TMA_SUMSQ_MIN=$t timeout 300 python tools/probe_residual.py --config $1 --kind $2 --reps 7 >> gpurun_out/r2k_plain.log 2>&1
done
done
echo done
