"""C1 sketch timing alone and right after a residual call (checks that no helper-stream work leaks into
the next sketch).  usage: python tools/probe_c1_sketch.py"""
import sys, torch
sys.path.insert(0, '.')
import paper_2104_05877_b200 as sk
from inputs import make_c1
A, _ = make_c1(seed=1001)
Ad = sk.fortran(torch.from_numpy(A).cuda())
X = torch.empty((40, 256), dtype=torch.float64, device='cuda')
for _ in range(3): sk.sketch(Ad, 40, 'gaussian', 2001, out=X)
torch.cuda.synchronize()
def t(f, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
print('sketch only', t(lambda: sk.sketch(Ad, 40, 'gaussian', 2001, out=X)))
Js, Lf, _, _ = sk.select_cols(X, 20)
print('residual (col ID)', t(lambda: sk.residual(Ad, Js, None, 'col_id'), 5))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
sk.residual(Ad, Js, None, 'col_id')
e0.record(); sk.sketch(Ad, 40, 'gaussian', 2001, out=X); e1.record(); torch.cuda.synchronize()
print('sketch right after a residual', e0.elapsed_time(e1))
