#!/bin/bash
mkdir -p gpurun_out
for t in "" "0,0,0,32768" "0,0,0,65536" "0,80,8,65536,4" "0,80,16,65536,4" "0,40,16,65536,2"; do
  echo "tune '$t'" >> gpurun_out/c4chunk.txt
  timeout 300 python tools/bench_sketch.py --only "C4 k" --reps 10 ${t:+--tune $t} >> gpurun_out/c4chunk.txt 2>&1
done
