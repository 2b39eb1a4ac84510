"""C2 end-to-end probe: pinned H2D bandwidth alone, sk_rand_lupp from host A, and from device A."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402
from inputs import make_c2  # noqa: E402


def tm(fn, reps=8):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return np.median(ts), min(ts)


A_np, _ = make_c2(seed=1002)
A_host = torch.from_numpy(np.ascontiguousarray(A_np.T)).pin_memory().t()
A_dev = torch.empty((4096, 4096), dtype=torch.float64, device="cuda").t()
print("h2d 134MB pinned", tm(lambda: A_dev.copy_(A_host, non_blocking=True)))
A_dev.copy_(A_host)
print("rand_lupp host", tm(lambda: sk.rand_lupp(A_host, 512, 522, seed=2514)))
print("rand_lupp dev ", tm(lambda: sk.rand_lupp(A_dev, 512, 522, seed=2514)))
t0 = time.perf_counter()
for _ in range(10):
    sk.rand_lupp(A_host, 512, 522, seed=2514)
print("rand_lupp host wall", (time.perf_counter() - t0) / 10 * 1e3)
