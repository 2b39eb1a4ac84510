"""Tall-panel LUPP (several clusters, DESIGN.md 7.3'): C4 rows, C5 columns, C5 rows (131072 rows)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


g = torch.Generator(device="cuda").manual_seed(5)
for name, n, k, rows in [("C4 rows", 65536, 200, True), ("C5 cols", 65536, 1000, False),
                         ("C5 rows", 131072, 1000, True), ("tall 32768", 32768, 500, True)]:
    if rows:
        C = torch.randn((k, n), dtype=torch.float64, device="cuda", generator=g).t()   # n x k column-major
        f = lambda: sk.select_rows(C, k, want_factors=False)  # noqa: E731
    else:
        X = torch.randn((k + 100, n), dtype=torch.float64, device="cuda", generator=g)
        f = lambda: sk.select_cols(X, k, want_factors=False)  # noqa: E731
    ms = timed(f)
    print(f"{name:12s} n={n:7d} k={k:5d} {ms:9.3f} ms {1e3 * ms / k:7.2f} us/step", flush=True)
