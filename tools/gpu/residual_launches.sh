#!/bin/bash
# Per-kernel launch list of one sk_residual call (tools/probe_residual.py) under ncu; args: config kind
# e.g.  bash tools/gpu/residual_launches.sh C4 row_id ; then python tools/launch_table.py gpurun_out/res_<cfg>_<kind>.csv
mkdir -p gpurun_out
cfg=${1:-C2}; kind=${2:-col_id}
python tools/probe_residual.py --config $cfg --kind $kind > gpurun_out/res_plain_${cfg}_$kind.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/res_${cfg}_$kind.csv python tools/probe_residual.py --config $cfg --kind $kind --profile --reps 1 \
    > gpurun_out/res_ncu_${cfg}_$kind.log 2>&1
