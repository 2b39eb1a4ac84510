#!/bin/bash
# A/B at C2 k=512: the planner's tile choice against pinned row-tile heights (the pin applies to the
# sketch, the residual's Q^T A and its fused sum-of-squares GEMM alike).
O=gpurun_out/ab_c2; mkdir -p $O
for t in "" "0,48,0,0,8" "0,64,0,0,8" "0,56,0,0,8" "0,40,0,0,8" "0,32,0,0,8"; do
  nm=${t//,/_}; [ -z "$nm" ] && nm=auto
  timeout 300 python bench.py --config C2 --steps 10 --no-cpu-baseline --no-e2e ${t:+--sketch-tuning $t} > $O/c2_$nm.log 2>&1
  python - "$O/c2_$nm.log" "$nm" <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); s = d["stages_ms"]
        print(sys.argv[2], "sketch %.3f residual %.3f value %.3f" % (s["sketch"], s["residual"], d["value"]))
PY
done
