#!/bin/bash
mkdir -p gpurun_out
SKEL_CHOL_DBG=1 timeout 300 python tools/probe_residual.py --config C2 --kind col_id --reps 1 > gpurun_out/r2n_dbg.log 2>&1
echo done
