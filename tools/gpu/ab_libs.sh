#!/bin/bash
# A/B of compile-time variants of libskel.so: ab/libskel_<name>.so (built here by tools/mkab.sh <name> "<-D flags>")
# swapped into place one after another; args: the shape filter of tools/bench_sketch.py, then variant names.
# e.g.  bash tools/gpu/ab_libs.sh "C3 sparse" eg2 v6
mkdir -p gpurun_out
only="$1"; shift
cp paper_2104_05877_b200/libskel.so /tmp/libskel_orig.so
for v in "$@"; do
  cp ab/libskel_$v.so paper_2104_05877_b200/libskel.so
  echo "== $v" >> gpurun_out/ab_libs.txt
  timeout 300 python tools/bench_sketch.py --only "$only" --reps 10 >> gpurun_out/ab_libs.txt 2>&1
done
cp /tmp/libskel_orig.so paper_2104_05877_b200/libskel.so
