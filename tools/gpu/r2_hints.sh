#!/bin/bash
# A/B: L2 cache hints on the sketch GEMM's TMA loads (A evict_first, Omega slot evict_last)
mkdir -p gpurun_out
cp paper_2104_05877_b200/libskel.so /tmp/libskel_cur.so
for v in nohints hints; do
  cp tools/ab/libskel_$v.so paper_2104_05877_b200/libskel.so
  echo "== $v" >> gpurun_out/r2g_ab.log
  timeout 300 python tools/bench_sketch.py --only "C" >> gpurun_out/r2g_ab.log 2>&1
  CMD="python tools/bench_sketch.py --only C5 --reps 1"
  timeout 300 $CMD > gpurun_out/r2g_plain_$v.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sketch_pre|k_omega_image" -c 8 --csv --log-file gpurun_out/r2g_dram_$v.csv $CMD > gpurun_out/r2g_ncu_$v.log 2>&1
done
cp /tmp/libskel_cur.so paper_2104_05877_b200/libskel.so
echo done
