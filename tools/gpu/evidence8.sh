#!/bin/bash
# Closing check after the right-looking U12 substitution: full GPU suite, smoke, every bench line.
# C2/C3/C4 bench lines with the per-LUPP 8(d) figures.
O=gpurun_out/ev8; mkdir -p $O
nvidia-smi -L > $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
( time timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 ) > $O/bench_c5.log 2>&1
( time timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > $O/bench_c5_reference.log 2>&1
timeout 600 python bench.py --config C2 > $O/bench_c2.log 2>&1
timeout 900 python bench.py --config C3 --steps 5 > $O/bench_c3.log 2>&1
timeout 900 python bench.py --config C4 --steps 5 > $O/bench_c4.log 2>&1
echo done
