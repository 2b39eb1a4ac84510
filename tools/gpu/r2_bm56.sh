#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "sketch_dense" > gpurun_out/r2l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_pytest.log
for t in "0,48,0,0" "0,56,0,0" "0,64,0,0" "0,56,0,16384" "0,48,0,16384"; do echo "tune $t" >> gpurun_out/r2l_bm.log; timeout 300 python tools/bench_sketch.py --only "C5" --tune $t >> gpurun_out/r2l_bm.log 2>&1; done
for t in "0,48,0,0" "0,56,0,0"; do echo "tune $t" >> gpurun_out/r2l_bm.log; timeout 300 python tools/bench_sketch.py --only "C2 k=512" --tune $t >> gpurun_out/r2l_bm.log 2>&1; done
echo done
