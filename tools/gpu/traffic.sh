#!/bin/bash
# DRAM bytes of one sk_sketch call per bench configuration (the bench line's roofline "traffic")
mkdir -p gpurun_out
for cfg in C2_k512 C3_k500 C4_k200 C5_k1000; do
  python tools/sketch_traffic.py $cfg > gpurun_out/traffic_plain_$cfg.log 2>&1 &&
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/traffic_$cfg.csv python tools/sketch_traffic.py $cfg > gpurun_out/traffic_ncu_$cfg.log 2>&1
done
echo done
