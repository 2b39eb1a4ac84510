import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2104_05877_b200 as sk
from oracle import sketch as o_sketch
m, n, l = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A = np.random.default_rng(1).standard_normal((m, n))
Ad = sk.fortran(torch.from_numpy(A).cuda())
sk.set_sketch_tuning(0, 40, 1, 0, warps=2)
X = sk.sketch(Ad, l, "gaussian", 77).cpu().numpy()
Xo = o_sketch.sketch(A, l, "gaussian", 77)
print(m, n, l, np.linalg.norm(X - Xo) / np.linalg.norm(Xo))
