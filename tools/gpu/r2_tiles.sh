#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "dense_plans" > gpurun_out/t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t_pytest.log
for t in "" "0,48,1,0,8" "0,80,1,0,12" "0,48,1,0,12" "0,96,1,0,8" "0,80,2,0,12"; do
  echo "tune $t" >> gpurun_out/t_sketch.txt
  if [ -z "$t" ]; then timeout 300 python tools/bench_sketch.py --only "C5 block" --reps 5 >> gpurun_out/t_sketch.txt 2>&1
  else timeout 300 python tools/bench_sketch.py --only "C5 block" --reps 5 --tune $t >> gpurun_out/t_sketch.txt 2>&1; fi
done
for t in "0,80,0,0,12" "0,48,0,0,12" "0,96,0,0,8"; do
  echo "tune $t" >> gpurun_out/t_sketch.txt
  timeout 300 python tools/bench_sketch.py --only "C2 k=512" --reps 10 --tune $t >> gpurun_out/t_sketch.txt 2>&1
done
echo done
