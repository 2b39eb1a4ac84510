#!/bin/bash
# The N>1 bench path at world size 1 (SKEL_BENCH_DIST=1 under torchrun), both LUPP exchanges.
mkdir -p gpurun_out
for ex in replicate step p2p; do
SKEL_BENCH_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 --dist-exchange $ex > gpurun_out/bench_dist_$ex.log 2>&1; echo "rc=$?" >> gpurun_out/bench_dist_$ex.log
done
