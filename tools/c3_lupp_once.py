import torch, sys
sys.path.insert(0, '/root/repo')
import paper_2104_05877_b200 as sk
X = torch.randn(510, 16384, dtype=torch.float64, device="cuda")
for _ in range(3): sk.select_cols(X, 500, want_factors=False)
torch.cuda.synchronize()
sk.select_cols(X, 500, want_factors=False)
torch.cuda.synchronize()
