"""cuBLAS DGEMM reference (torch.matmul on float64) — the measured FP64 tensor denominator.

Best-of-10 burst and a ~3 s sustained loop, CUDA events. Context for DESIGN.md's roofline.
"""
import json
import time

import torch


def main():
    dev = torch.device("cuda:0")
    out = {}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"dgemm_{n}_burst_tflops"] = 2 * n**3 / best / 1e9
        t0 = time.time()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cnt = 0
        while time.time() - t0 < 3.0:
            torch.matmul(a, b)
            cnt += 1
        e1.record()
        torch.cuda.synchronize()
        out[f"dgemm_{n}_sustained_tflops"] = 2 * n**3 * cnt / e0.elapsed_time(e1) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
