"""Column-ID residual at C5's width with a shorter A: m x 65536, k = 1000, A of exact rank 1000 plus a
tiny perturbation (so the explicit sum-of-squares path runs, r^2 << 1e-3 ||A||^2), J_s = the first k
columns.  CUDA-event time of sk_residual; with --profile the timed calls are bracketed by
cudaProfilerStart/Stop for an ncu launch list.  usage: python tools/probe_residual_c5.py [--m 32768]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=32768)
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--k", type=int, default=1000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--noise", type=float, default=1e-9, help="perturbation size (0: exact rank k)")
ap.add_argument("--tune", default="", help="path,bm,splits,chunk[,warps] for sk_set_sketch_tuning")
a = ap.parse_args()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
B = torch.randn(a.m, a.k, dtype=torch.float64, device=dev, generator=g)
Cf = torch.randn(a.k, a.n, dtype=torch.float64, device=dev, generator=g)
Cf *= torch.arange(1, a.k + 1, dtype=torch.float64, device=dev).pow(-1.5)[:, None]
A = sk.fortran(B @ Cf)
del B, Cf
if a.noise > 0:
    A.add_(torch.randn(A.shape, dtype=torch.float64, device=dev, generator=g).t().contiguous().t(), alpha=a.noise)
if a.tune:
    t = [int(x) for x in a.tune.split(",")]
    sk.set_sketch_tuning(*t[:4], warps=t[4] if len(t) > 4 else 0)
Js = torch.arange(a.k, dtype=torch.int64, device=dev)
r, nA = sk.residual(A, Js, None, "col_id")
torch.cuda.synchronize()
if a.profile:
    torch.cuda.profiler.start()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r, nA = sk.residual(A, Js, None, "col_id")
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
if a.profile:
    torch.cuda.profiler.stop()
ms = sorted(ts)[len(ts) // 2]
fl = 4.0 * a.k * a.m * a.n
print(f"m={a.m} n={a.n} k={a.k}: residual {ms:.2f} ms, {fl / ms / 1e9:.2f} TF/s = {fl / ms / 1e9 / 37.13:.1%} of the "
      f"4kmn bound; r={r:.3e} |A|={nA:.3e} r^2/|A|^2={(r / nA) ** 2:.2e}")
