"""Time sk_sketch alone on the BASELINE shapes (device-resident A, CUDA events, L2 flushed).

usage: python tools/bench_sketch.py [--reps 10]
Prints one line per shape: ms, TFLOP/s (2 l m n), fraction of the measured 37.13 TF/s DMMA ceiling
(dense) or achieved GB/s of (8mn + 8ln) bytes against MEASURED_PEAKS hbm_gbs (sparse).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402

PEAK = 37.13
SHAPES = [  # (name, m, n, l, embedding)
    ("C2 k=16", 4096, 4096, 26, "gaussian"),
    ("C2 k=64", 4096, 4096, 74, "gaussian"),
    ("C2 k=256", 4096, 4096, 266, "gaussian"),
    ("C2 k=512", 4096, 4096, 522, "gaussian"),
    ("C4 k=50", 65536, 784, 100, "gaussian"),
    ("C4 k=100", 65536, 784, 200, "gaussian"),
    ("C4 k=200", 65536, 784, 400, "gaussian"),
    ("C5 block", 131072, 8192, 1100, "gaussian"),
    ("C5 rows", 16384, 65536, 1100, "gaussian"),     # two of C5's 16 K-chunks at its full width (the N = 1 tile grid)
    ("C5 half", 65536, 65536, 1100, "gaussian"),     # eight of C5's 16 K-chunks at its full width
    ("C3 sparse", 16384, 16384, 510, "sparse_sign"),
    ("C2 srtt k=512", 4096, 4096, 522, "srtt"),
    ("C3 srtt", 16384, 16384, 510, "srtt"),
    ("C4 srtt k=200", 65536, 784, 400, "srtt"),
    ("C5 block srtt", 131072, 8192, 1100, "srtt"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="", help="substring filter on the shape name")
    ap.add_argument("--tune", default="", help="path,bm,splits,chunk[,warps] for sk_set_sketch_tuning")
    a = ap.parse_args()
    if a.tune:
        t = [int(x) for x in a.tune.split(",")]
        sk.set_sketch_tuning(*t[:4], warps=t[4] if len(t) > 4 else 0)
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 18, dtype=torch.int32, device=dev)
    for name, m, n, l, emb in SHAPES:
        if a.only and a.only not in name:
            continue
        A = sk.fortran(torch.randn(m, n, dtype=torch.float64, device=dev))
        X = torch.empty((l, n), dtype=torch.float64, device=dev)
        for _ in range(3):
            sk.sketch(A, l, emb, 7, out=X)
        ts = []
        for _ in range(a.reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sk.sketch(A, l, emb, 7, out=X)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        if emb == "gaussian":
            tf = 2.0 * l * m * n / (ms * 1e-3) / 1e12
            print(f"{name:12s} m={m:6d} n={n:6d} l={l:4d}  {ms:8.4f} ms  {tf:6.2f} TF/s  {tf / PEAK:5.1%} of DMMA peak")
        else:   # sparse sign / SRTT: HBM bound (A once + X)
            gbs = 8.0 * (m * n + l * n) / (ms * 1e-3) / 1e9
            print(f"{name:12s} m={m:6d} n={n:6d} l={l:4d}  {ms:8.4f} ms  {gbs:7.1f} GB/s  {gbs / 6439.8:5.1%} of HBM")
        del A, X


if __name__ == "__main__":
    main()
