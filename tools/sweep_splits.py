import os, sys, torch
sys.path.insert(0, '/root/repo')
import paper_2104_05877_b200 as sk
m = n = 4096; l = 522
A = sk.fortran(torch.randn(m, n, dtype=torch.float64, device="cuda"))
X = torch.empty((l, n), dtype=torch.float64, device="cuda")
flush = torch.empty(512 << 18, dtype=torch.int32, device="cuda")
def timed(reps=7):
    sk.sketch(A, l, "gaussian", 7, out=X); ts = []
    for _ in range(reps):
        flush.fill_(1); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sk.sketch(A, l, "gaussian", 7, out=X); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts)//2]
for plan in ["48,8,4,0", "48,8,3,0", "48,8,5,0", "48,8,6,0", "48,8,7,0", "48,8,8,0", "64,8,3,0", "64,8,5,0", "32,8,5,0", "32,8,6,0"]:
    os.environ["SKEL_PRE_PLAN"] = plan
    ms = timed()
    print(plan, f"{ms:.4f} ms {2*l*m*n/ms/1e9/37.13:.1%}", flush=True)
