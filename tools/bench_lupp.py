"""Time sk_select_cols / sk_select_rows / sk_select_cols_cpqr alone on the BASELINE panel shapes.

usage: python tools/bench_lupp.py [--reps 10]
Per shape: ms per call and us per pivot step (the k-step argmax chain is the bound).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402

SHAPES = [  # (name, kind, panel rows n, l, k)
    ("C1 cols", "cols", 256, 40, 20),
    ("C2 k=16", "cols", 4096, 26, 16),
    ("C2 k=64", "cols", 4096, 74, 64),
    ("C2 k=256", "cols", 4096, 266, 256),
    ("C2 k=512", "cols", 4096, 522, 512),
    ("C2 k=512 cpqr", "cpqr", 4096, 522, 512),
    ("C3 cols", "cols", 16384, 510, 500),
    ("C3 rows", "rows", 16384, 500, 500),
    ("C4 k=200 rows", "rows", 65536, 200, 200),
]


def timeit(fn, reps):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    for name, kind, n, l, k in SHAPES:
        if kind == "rows":
            C = sk.fortran(torch.randn(n, k, dtype=torch.float64, device=dev, generator=g))
            fn = lambda: sk.select_rows(C, k, check=False)  # noqa: E731
        else:
            X = torch.randn(l, n, dtype=torch.float64, device=dev, generator=g)
            if kind == "cols":
                fn = lambda: sk.select_cols(X, k, check=False)  # noqa: E731
            else:
                fn = lambda: sk.select_cols_cpqr(X, k, check=False)  # noqa: E731
        ms = timeit(fn, a.reps)
        print(f"{name:16s} n={n:6d} k={k:4d}  {ms:8.4f} ms  {1e3 * ms / k:7.2f} us/step")


if __name__ == "__main__":
    main()
