#!/bin/bash
mkdir -p gpurun_out
for t in "" "0,40,1,0,16" "0,32,1,0,16" "0,40,2,0,16"; do
  echo "tune $t" >> gpurun_out/t4_sketch.txt
  if [ -z "$t" ]; then timeout 300 python tools/bench_sketch.py --only "C5" --reps 5 >> gpurun_out/t4_sketch.txt 2>&1
  else timeout 300 python tools/bench_sketch.py --only "C5" --reps 5 --tune $t >> gpurun_out/t4_sketch.txt 2>&1; fi
done
for t in "0,40,0,0,16" "0,32,0,0,16"; do
  echo "tune $t" >> gpurun_out/t4_sketch.txt
  timeout 300 python tools/bench_sketch.py --only "C2 k" --reps 10 --tune $t >> gpurun_out/t4_sketch.txt 2>&1
done
echo done
