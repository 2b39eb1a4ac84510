"""Raw page-locked host -> device copy bandwidth on this box (context for the e2e numbers, which are
PCIe-bound at C5): 8 GiB in 1 GiB copies, CUDA events."""
import torch

dev = torch.device("cuda", 0)
n = 1 << 27                                        # 1 GiB of float64
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device=dev)
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(8):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"pinned H2D: {8 * 8 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
