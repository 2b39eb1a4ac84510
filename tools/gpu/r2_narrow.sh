#!/bin/bash
# 112-column (narrow-n) sketch tiles: plan parity, C4 full-size parity, sketch timings, C4 bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "dense_plans" > gpurun_out/nw_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/nw_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "c4" > gpurun_out/nw_pytest_c4.log 2>&1; echo "rc=$?" >> gpurun_out/nw_pytest_c4.log
timeout 600 python tools/bench_sketch.py --only "C4 k" > gpurun_out/nw_sketch_auto.txt 2>&1
for t in "0,80,0,0,4" "3,80,8,0,4" "2,80,8,0,4" "0,80,16,0,4" "0,40,0,0,2" "0,40,0,0,7"; do
  echo "tune $t" >> gpurun_out/nw_sketch_tune.txt
  timeout 300 python tools/bench_sketch.py --only "C4 k" --tune $t >> gpurun_out/nw_sketch_tune.txt 2>&1
done
timeout 600 python tools/bench_sketch.py --only "C2 k" > gpurun_out/nw_sketch_c2.txt 2>&1
timeout 900 python bench.py --config C4 --steps 5 > gpurun_out/nw_bench_c4.log 2>&1
echo done
