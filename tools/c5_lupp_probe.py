"""One tall select_cols / select_rows with SKEL_LUPP_PROBE=1 (per-step phase cycles to stderr)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(5)
for n, k in [(65536, 1000), (65536, 200), (16384, 500), (4096, 512)]:
    X = torch.randn((k + 10, n), dtype=torch.float64, device="cuda", generator=g)
    sk.select_cols(X, k, want_factors=False)
    torch.cuda.synchronize()
