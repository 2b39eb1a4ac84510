"""Feasibility: does the 16-CTA-cluster LUPP panel get SMs while sketch kernels occupy the GPU?
Runs LUPP alone, sketches alone, then both (LUPP on a high-priority stream launched after the
sketches are queued) and reports when each finishes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402

dev = "cuda"
m = n = 4096
k, l = 512, 522
A = sk.fortran(torch.randn(m, n, dtype=torch.float64, device=dev))
X = sk.sketch(A, l, "gaussian", 3)
Xs = [torch.empty_like(X) for _ in range(4)]
lo = torch.cuda.Stream(priority=0)
hi = torch.cuda.Stream(priority=-5)


def ev():
    return torch.cuda.Event(enable_timing=True)


for rep in range(3):
    torch.cuda.synchronize()
    e0 = ev(); e0.record()
    with torch.cuda.stream(hi):
        hi.wait_event(e0)
        sk.select_cols(X, k, want_factors=False)
        e_l = ev(); e_l.record(hi)
    torch.cuda.synchronize()
    t_lupp = e0.elapsed_time(e_l)
    e0 = ev(); e0.record()
    with torch.cuda.stream(lo):
        lo.wait_event(e0)
        for q in range(4):
            sk.sketch(A, l, "gaussian", 3, out=Xs[q])
        e_s = ev(); e_s.record(lo)
    torch.cuda.synchronize()
    t_sk = e0.elapsed_time(e_s)
    e0 = ev(); e0.record()
    with torch.cuda.stream(lo):
        lo.wait_event(e0)
        for q in range(4):
            sk.sketch(A, l, "gaussian", 3, out=Xs[q])
        e_s = ev(); e_s.record(lo)
    with torch.cuda.stream(hi):
        hi.wait_event(e0)
        sk.select_cols(X, k, want_factors=False)
        e_l = ev(); e_l.record(hi)
    torch.cuda.synchronize()
    print(f"alone: LUPP {t_lupp:.3f} ms, 4 sketches {t_sk:.3f} ms | together: LUPP done at {e0.elapsed_time(e_l):.3f} ms,"
          f" sketches done at {e0.elapsed_time(e_s):.3f} ms", flush=True)
