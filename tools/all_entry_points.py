"""Small calls of every entry point in one process (compute-sanitizer is closed on this pool, so this
is the whole-library smoke: any CUDA fault surfaces as an exception here)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402

dev = "cuda"
rng = np.random.default_rng(1)
m, n, k, l = 600, 300, 24, 34
A = sk.fortran(torch.from_numpy(rng.standard_normal((m, n))).to(dev))
X = sk.sketch(A, l, "gaussian", 3)
Xs = sk.sketch(A, l, "sparse_sign", 3)
Xp = sk.sketch_power(A, l, "gaussian", 3, q=1)
A2 = sk.fortran(torch.from_numpy(rng.standard_normal((512, 200))).to(dev))
Xt = sk.sketch(A2, l, "srtt", 3)
Js, Lf, U, _ = sk.select_cols(X, k)
Jc, _ = sk.select_cols_cpqr(X, k)[:2]
Z, eta = sk.id_coeffs(Lf, Js, want_eta=True)
C = sk.gather_cols(A, Js)
Is, _, _, _ = sk.select_rows(C, k)
for kind in ("col_id", "row_id", "cur"):
    sk.residual(A, Js, Is, kind)
sk.residual(A, Js, None, "id_coeffs", Z)
Jd = sk.select_cols_deim(A, X, k)
sk.rand_lupp(A.cpu().t().contiguous().t(), k, l)
# per-step distributed LUPP, both exchanges (3 ranks emulated)
from paper_2104_05877_b200.dist import shard  # noqa: E402
world = 3
sels = []
for r in range(world):
    c0, nc = shard(n, world, r)
    sels.append((sk.LuppDist(nc, k, c0, world, 0), X[:, c0:c0 + nc].contiguous()))
for s_, b in sels:
    s_.begin(b)
for t in range(1, k + 1):
    g = torch.cat([s_.cand for s_, _ in sels])
    for s_, _ in sels:
        s_.gathered.copy_(g)
        s_.step(t)
boxes = [sk.ipc_alloc(sk.mailbox_bytes(k, world), 0) for _ in range(world)]
peers = torch.tensor(boxes, dtype=torch.int64, device=dev)
ps = []
for r in range(world):
    c0, nc = shard(n, world, r)
    ps.append((sk.LuppDistP2P(nc, k, c0, world, r, peers, boxes[r], 0), X[:, c0:c0 + nc].contiguous()))
for s_, b in ps:
    s_.begin(b)
for t in range(1, k + 1):
    for s_, _ in ps:
        s_.step(t)
torch.cuda.synchronize()
for b in boxes:
    sk.ipc_free(b, 0)
print("all entry points done")
