#!/bin/bash
mkdir -p gpurun_out
for t in "" "0,80,1,0,12" "0,48,1,0,12" "0,96,1,0,8" "0,64,1,0,8"; do
  echo "tune $t" >> gpurun_out/t2_sketch.txt
  if [ -z "$t" ]; then timeout 300 python tools/bench_sketch.py --only "C5 rows" --reps 5 >> gpurun_out/t2_sketch.txt 2>&1
  else timeout 300 python tools/bench_sketch.py --only "C5 rows" --reps 5 --tune $t >> gpurun_out/t2_sketch.txt 2>&1; fi
done
echo done
