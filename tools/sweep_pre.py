"""Sweep the dense sketch's plans (sk_set_sketch_tuning: row-tile height, K-splits, HBM partials vs
cluster DSMEM reduction) for the BASELINE shapes.  usage: python tools/sweep_pre.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402

SHAPES = [("C2 k=16", 4096, 4096, 26), ("C2 k=64", 4096, 4096, 74), ("C2 k=256", 4096, 4096, 266),
          ("C2 k=512", 4096, 4096, 522), ("C4 k=50", 65536, 784, 100), ("C4 k=100", 65536, 784, 200),
          ("C4 k=200", 65536, 784, 400), ("C5 block", 131072, 8192, 1100), ("C5 rows", 16384, 65536, 1100)]
PLANS = [(64, 8), (56, 8), (96, 8), (48, 8), (40, 8), (32, 8), (40, 7), (48, 7), (80, 4), (40, 2), (48, 12), (80, 12)]   # (bm, warps); 4 / 2 = 112-column tiles, 12 = 384 / 192


def timed(fn, reps=5):
    flush = torch.empty(512 << 18, dtype=torch.int32, device="cuda")
    fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


only = sys.argv[1] if len(sys.argv) > 1 else ""
for name, m, n, l in SHAPES:
    if only and only not in name:
        continue
    A = sk.fortran(torch.randn(m, n, dtype=torch.float64, device="cuda"))
    X = torch.empty((l, n), dtype=torch.float64, device="cuda")
    sk.set_sketch_tuning()
    ms = timed(lambda: sk.sketch(A, l, "gaussian", 7, out=X))
    ref = X.clone()
    print(f"{name:10s} default plan {ms:8.4f} ms {2 * l * m * n / ms / 1e9 / 37.13:6.1%}", flush=True)
    res = []
    for bm, nw in PLANS:
        for sp in (1, 2, 4, 8, 16, 32, 64):
            if sp > 1 and m // sp < 1024:
                break
            for cl in ((0, 1) if sp > 1 and sp <= 8 and bm % sp == 0 and nw > 4 else (0,)):
                sk.set_sketch_tuning(path=3 if cl else 2, bm=bm, splits=sp, warps=nw)
                ms = timed(lambda: sk.sketch(A, l, "gaussian", 7, out=X))
                err = float((X - ref).norm() / ref.norm())
                res.append((ms, bm, nw, sp, cl, err))
    res.sort()
    for ms, bm, nw, sp, cl, err in res[:8]:
        print(f"    {bm:3d} {nw:3d} {sp:3d} cl{cl}  {ms:8.4f} ms {2 * l * m * n / ms / 1e9 / 37.13:6.1%}  rel {err:.1e}",
              flush=True)
    del A, X
    sk.set_sketch_tuning()
