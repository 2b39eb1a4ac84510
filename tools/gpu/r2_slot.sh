#!/bin/bash
mkdir -p gpurun_out
for ch in 4096 6144 8192; do
  echo "chunk $ch" >> gpurun_out/r2q_slot.log
  timeout 300 python tools/bench_sketch.py --only "C5" --tune 0,0,0,$ch >> gpurun_out/r2q_slot.log 2>&1
  CMD="python tools/bench_sketch.py --only C5 --reps 1 --tune 0,0,0,$ch"
  timeout 300 $CMD > gpurun_out/r2q_plain_$ch.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sketch_pre|k_omega_image" -s 40 -c 20 --csv --log-file gpurun_out/r2q_dram_$ch.csv $CMD > gpurun_out/r2q_ncu_$ch.log 2>&1
done
echo done
