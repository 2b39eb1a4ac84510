#!/bin/bash
# A/B of sparse-sketch variants (ab/libskel_<v>.so swapped into place); args: variant names
mkdir -p gpurun_out
cp paper_2104_05877_b200/libskel.so /tmp/libskel_orig.so
for v in "$@"; do
  cp ab/libskel_$v.so paper_2104_05877_b200/libskel.so
  echo "== $v" >> gpurun_out/sp_ab.txt
  timeout 300 python tools/bench_sketch.py --only "C3 sparse" --reps 20 >> gpurun_out/sp_ab.txt 2>&1
done
cp /tmp/libskel_orig.so paper_2104_05877_b200/libskel.so
echo done
