#!/bin/bash
# round 2: library-owned distributed context -- full GPU suite, world-1 torchrun bench, chunk sweep
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_pytest.log
for ch in 2048 4096 8192 16384 131072; do echo "chunk $ch" >> gpurun_out/r2d_chunks.log; timeout 300 python tools/bench_sketch.py --only "C5 block" --tune 0,0,0,$ch >> gpurun_out/r2d_chunks.log 2>&1; done
SKEL_BENCH_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --steps 2 --warmup 1 > gpurun_out/r2d_bench_dist1.log 2>&1
SKEL_BENCH_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --steps 2 --warmup 1 --dist-exchange step --no-e2e > gpurun_out/r2d_bench_dist1_step.log 2>&1
echo done
