#!/bin/bash
# The column-sharded bench path on the library's distributed context at world size 1 (torchrun, NCCL);
# args: extra bench.py flags (e.g. --dist-exchange step, --sketch-tuning 2,0,0,0)
mkdir -p gpurun_out
export SKEL_BENCH_DIST=1
tag=${TAG:-w1}
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --steps 2 --warmup 1 --no-e2e "$@" > gpurun_out/dist_$tag.log 2>&1
