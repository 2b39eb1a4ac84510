#!/bin/bash
# Round-2 closing checks: the driver's exact bench command timed by the wall clock (it must fit the
# driver's run), the column-sharded path at world size 1 with both exchanges after the chained-chunk
# change, and the raw pinned H2D bandwidth the C5 e2e figure is bounded by.
mkdir -p gpurun_out/ev5
nvidia-smi -L > gpurun_out/ev5/gpu.txt
python tools/h2d_probe.py > gpurun_out/ev5/h2d_probe.txt 2>&1
( time timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/ev5/bench_driver_cmd.log 2>&1
export SKEL_BENCH_DIST=1
for ex in replicate step; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --steps 3 --warmup 3 --no-e2e --dist-exchange $ex > gpurun_out/ev5/bench_dist_world1_$ex.log 2>&1
done
echo done
