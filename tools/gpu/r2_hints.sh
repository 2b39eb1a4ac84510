#!/bin/bash
# A/B of the sketch GEMM's L2 hints at C5 width with 12-warp tiles: time and DRAM bytes per chunk GEMM
mkdir -p gpurun_out
cp paper_2104_05877_b200/libskel.so /tmp/libskel_orig.so
for v in anorm hints1; do
  cp ab/libskel_$v.so paper_2104_05877_b200/libskel.so
  echo "== $v" >> gpurun_out/hints_ab.txt
  timeout 300 python tools/bench_sketch.py --only "C5 rows" --reps 5 >> gpurun_out/hints_ab.txt 2>&1
  timeout 300 python tools/bench_sketch.py --only "C5 block" --reps 3 >> gpurun_out/hints_ab.txt 2>&1
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_sketch_pre -s 2 -c 1 --csv \
      python tools/bench_sketch.py --only "C5 rows" --reps 1 2>/dev/null | grep -E 'dram__|gpu__time' >> gpurun_out/hints_ab.txt
done
cp /tmp/libskel_orig.so paper_2104_05877_b200/libskel.so
echo done
