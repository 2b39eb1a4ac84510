"""Time sk_sketch_dual (Algorithm 3's one-pass X = Gamma A, Y = A Omega^T) against the two separate
sketches (sk_sketch + sk_sketch_cols), device-resident A, L2 flushed, CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402

SHAPES = [("C2 k=256", 4096, 4096, 266), ("C2 k=512", 4096, 4096, 522), ("C3-size", 16384, 16384, 510),
          ("C4 k=200", 65536, 784, 400)]


def timeit(fn, flush, reps=5):
    for _ in range(2):
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


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 18, dtype=torch.int32, device=dev)
    for name, m, n, l in SHAPES:
        A = sk.fortran(torch.randn(m, n, dtype=torch.float64, device=dev))
        ly = min(l, n)
        t_dev = timeit(lambda: sk.sketch_dual(A, l, ly, 1, 2), flush)
        Ah = A.t().cpu().pin_memory().t()                     # column-major, page-locked host copy
        t_host = timeit(lambda: sk.sketch_dual(Ah, l, ly, 1, 2), flush, reps=3)
        t_h2d = timeit(lambda: A.copy_(Ah, non_blocking=True), flush, reps=3)
        tf = 2.0 * (l + ly) * m * n / (t_dev * 1e-3) / 1e12
        print(f"{name:10s} m={m:6d} n={n:6d} lx={l:4d} ly={ly:4d}  device A {t_dev:8.3f} ms ({tf:5.2f} TF/s, "
              f"{tf / 37.13:5.1%} of DMMA)  host A one pass {t_host:8.3f} ms  (H2D of A alone {t_h2d:8.3f} ms)")
        del Ah
        del A


if __name__ == "__main__":
    main()
