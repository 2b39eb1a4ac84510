import torch
dev = "cuda"
for (M, K, N) in [(522, 4096, 4096), (528, 4096, 4096), (512, 4096, 4096), (1100, 131072, 8192), (400, 65536, 784), (8192, 8192, 8192)]:
    O = torch.randn(M, K, dtype=torch.float64, device=dev)
    A = torch.randn(K, N, dtype=torch.float64, device=dev).t().contiguous().t()   # column-major like ours
    for _ in range(3): X = O @ A
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); X = O @ A; e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[5]
    print(f"cuBLAS DGEMM {M}x{K}x{N}: {ms:.4f} ms  {2*M*K*N/ms/1e9:.2f} TF/s  ({2*M*K*N/ms/1e9/37.13:.1%} of 37.13)", flush=True)
