#!/bin/bash
# Evidence pass 4 (round 2 final: tile-ordered chained chunks): full GPU suite, smoke, every bench line,
# reference arm, the C5 launch list and an ncu --set full capture of the C5 sketch GEMM.
mkdir -p gpurun_out/ev4
nvidia-smi -L > gpurun_out/ev4/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/ev4/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev4/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev4/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev4/smoke.log
timeout 1500 python bench.py > gpurun_out/ev4/bench_c5.log 2>&1
timeout 600 python bench.py --config C1 > gpurun_out/ev4/bench_c1.log 2>&1
timeout 600 python bench.py --config C2 > gpurun_out/ev4/bench_c2.log 2>&1
timeout 900 python bench.py --config C3 --steps 5 > gpurun_out/ev4/bench_c3.log 2>&1
timeout 900 python bench.py --config C4 --steps 5 > gpurun_out/ev4/bench_c4.log 2>&1
timeout 600 python bench.py --config C2 --piter 1 --steps 5 > gpurun_out/ev4/bench_c2_1piter.log 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ev4/bench_ref_c5.log 2>&1
timeout 300 python tools/bench_lupp.py > gpurun_out/ev4/bench_lupp.log 2>&1
timeout 600 python tools/bench_sketch.py --only "C" > gpurun_out/ev4/bench_sketch.log 2>&1
python tools/bench_sketch.py --only "C5 half" --reps 1 > gpurun_out/ev4/ncu_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_sketch_pre -s 2 -c 1 \
    -o gpurun_out/ev4/prof_c5pre_t48 python tools/bench_sketch.py --only "C5 half" --reps 1 > gpurun_out/ev4/ncu.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 $CMD > gpurun_out/ev4/launch_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemm" -c 3000 --csv --log-file gpurun_out/ev4/launches_c5.csv $CMD > gpurun_out/ev4/ncu_launch.log 2>&1
echo done
for cfg in C2_k512 C3_k500 C4_k200 C5_k1000; do
  python tools/sketch_traffic.py $cfg > gpurun_out/ev4/traffic_plain_$cfg.log 2>&1 &&
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/ev4/traffic_$cfg.csv python tools/sketch_traffic.py $cfg > gpurun_out/ev4/traffic_ncu_$cfg.log 2>&1
done
echo done3
