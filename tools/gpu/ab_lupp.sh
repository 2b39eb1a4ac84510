#!/bin/bash
mkdir -p gpurun_out
cp paper_2104_05877_b200/libskel.so /tmp/libskel_orig.so
for v in base norest; do
  cp ab/libskel_$v.so paper_2104_05877_b200/libskel.so
  echo "== $v" >> gpurun_out/lupp_ab.txt
  timeout 300 python tools/bench_lupp_tall.py >> gpurun_out/lupp_ab.txt 2>&1
  timeout 300 python tools/bench_lupp.py >> gpurun_out/lupp_ab.txt 2>&1
done
cp /tmp/libskel_orig.so paper_2104_05877_b200/libskel.so
