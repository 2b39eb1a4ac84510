#!/bin/bash
mkdir -p gpurun_out
for co in "" 100 0; do
echo "--- carveout '$co'" >> gpurun_out/carve.log
env ${co:+SKEL_CARVEOUT=$co} timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms'])" >> gpurun_out/carve.log
done
