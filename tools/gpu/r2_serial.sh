#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sketch or c2_full or c4_full or power or dual" > gpurun_out/r2j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_pytest.log
timeout 300 python tools/bench_sketch.py --only C > gpurun_out/r2j_sketch.log 2>&1
timeout 600 python tools/sweep_pre.py "C2 k=512" > gpurun_out/r2j_sweep.log 2>&1
CMD="python tools/bench_sketch.py --only C5 --reps 1"
timeout 300 $CMD > gpurun_out/r2j_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sketch_pre|k_omega_image" -c 6 --csv --log-file gpurun_out/r2j_dram_c5.csv $CMD > gpurun_out/r2j_ncu.log 2>&1
CMD2="python tools/bench_sketch.py --only C2 --reps 1"
timeout 300 $CMD2 > gpurun_out/r2j_plain2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sketch|k_omega" --csv --log-file gpurun_out/r2j_dram_c2.csv $CMD2 > gpurun_out/r2j_ncu2.log 2>&1
echo done
