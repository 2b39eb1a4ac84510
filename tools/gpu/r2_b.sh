#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 --deselect tests/test_gpu_c5.py::test_c5_oracle_streamed > gpurun_out/r2b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_smoke.log
timeout 600 python tools/bench_sketch.py --only "C5 block" > gpurun_out/r2b_sketch.log 2>&1
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_c2.log 2>&1
timeout 600 python bench.py --config C2 --piter 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_c2_piter.log 2>&1
echo done
