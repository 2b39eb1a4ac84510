#!/bin/bash
# Exploration cycle: sketch timing under planner overrides and debug modes
# (SKEL_SKETCH_DBG: 1 = producers skip Box-Muller, 2 = consumers skip DMMA).
mkdir -p gpurun_out
for dbg in 0 1 2; do
  for plan in "32,2,1" "32,1,1" "64,2,1" "64,1,1"; do
    echo "== SKEL_SKETCH_DBG=$dbg SKEL_TMA_PLAN=$plan" >> gpurun_out/explore.log
    SKEL_SKETCH_DBG=$dbg SKEL_TMA_PLAN=$plan timeout 300 python tools/bench_sketch.py --reps 5 2>&1 | sed -n 3,4p >> gpurun_out/explore.log
  done
done
echo done
