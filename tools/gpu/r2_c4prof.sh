#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/bench_sketch.py --only C > gpurun_out/r2k_sketch.log 2>&1
CMD="python tools/bench_sketch.py --only C4 --reps 2"
timeout 300 $CMD > gpurun_out/r2k_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_" --csv --log-file gpurun_out/r2k_c4.csv $CMD > gpurun_out/r2k_ncu.log 2>&1
echo done
