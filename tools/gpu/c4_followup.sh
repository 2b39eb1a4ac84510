#!/bin/bash
# C4 after dropping the one-whole-image rule: bench line, sketch traffic, sketch plan parity
mkdir -p gpurun_out/ev4b
timeout 900 python bench.py --config C4 --steps 5 > gpurun_out/ev4b/bench_c4.log 2>&1
python tools/sketch_traffic.py C4_k200 > gpurun_out/ev4b/traffic_plain_C4_k200.log 2>&1 &&
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ev4b/traffic_C4_k200.csv python tools/sketch_traffic.py C4_k200 > gpurun_out/ev4b/traffic_ncu_C4_k200.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "dense or c4 or chained" > gpurun_out/ev4b/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ev4b/pytest.log
echo done
