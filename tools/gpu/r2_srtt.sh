#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k srtt > gpurun_out/r2t_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2t_pytest.log
timeout 300 python tools/bench_sketch.py --only srtt > gpurun_out/r2t_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_srtt_big -s 2 -c 1 -o gpurun_out/r2t_srtt_big -f python tools/bench_sketch.py --only "C5 block srtt" --reps 1 > gpurun_out/r2t_ncu.log 2>&1
echo done
