"""Time sk_residual alone on C2 / C3 / C4 (device-resident A, CUDA events), optionally bracketed by
cudaProfilerStart/Stop so `ncu --profile-from-start off` captures only the residual calls.
usage: python tools/probe_residual.py [--config C2] [--kind col_id] [--reps 5] [--profile]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402
from inputs import make_c2, make_c3, make_c4  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--kind", default="col_id")
ap.add_argument("--k", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
A, _ = {"C2": make_c2, "C3": make_c3, "C4": make_c4}[a.config]()
k = a.k or {"C2": 512, "C3": 500, "C4": 200}[a.config]
Ad = sk.fortran(torch.from_numpy(A).to(dev))
X = sk.sketch(Ad, k + 10, "gaussian", 5)
Js, _, _, _ = sk.select_cols(X, k)
Is = None
if a.kind in ("row_id", "cur"):
    Is, _, _, _ = sk.select_rows(sk.gather_cols(Ad, Js), k)
for _ in range(2):
    sk.residual(Ad, Js, Is, a.kind)
torch.cuda.synchronize()
if a.profile:
    torch.cuda.profiler.start()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r, nA = sk.residual(Ad, Js, Is, a.kind)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
if a.profile:
    torch.cuda.profiler.stop()
print(f"{a.config} {a.kind} k={k}: residual {sorted(ts)[len(ts) // 2]:.3f} ms (median of {a.reps}), r={r:.6e} |A|={nA:.6e} r^2/|A|^2={(r / nA) ** 2:.3e}")
