#!/bin/bash
# ncu --set full of the multi-cluster LUPP panel (C4 rows shape: 4 clusters of 16) and its block transition
mkdir -p gpurun_out
cat > /tmp/tall_once.py <<'P'
import torch, paper_2104_05877_b200 as sk
g = torch.Generator(device="cuda").manual_seed(5)
C = torch.randn((200, 65536), dtype=torch.float64, device="cuda", generator=g).t()
sk.select_rows(C, 200, want_factors=False); torch.cuda.synchronize()
P
timeout 120 python /tmp/tall_once.py > gpurun_out/tall_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lupp_panel_v2|k_lupp_u12|k_gemm" -s 4 -c 3 -o /tmp/prof_tall python /tmp/tall_once.py > gpurun_out/ncu_tall.log 2>&1
python tools/ncu_summary.py /tmp/prof_tall.ncu-rep > gpurun_out/ncu_tall_summary.txt 2>&1
echo done
