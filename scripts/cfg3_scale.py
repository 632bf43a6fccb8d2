"""Developer: spectral scale of config 3's minibatch estimates (largest
eigenvalues of B_t = blockdiag(X2^T X2, Y2^T Y2)/h and of the cross block),
to pick a stable step size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import CONFIGS, cca_views
cfg = CONFIGS[3]
b = cfg.batch; h = b // 2
X, Y = cca_views(cfg, b, seed=11, device="cuda:0", dtype=torch.float32)
x2, y2 = X[h:].double(), Y[h:].double()
x1, y1 = X[:h].double(), Y[:h].double()
sx = torch.linalg.svdvals(x2)[:4] ** 2 / h
sy = torch.linalg.svdvals(y2)[:4] ** 2 / h
sxy = torch.linalg.svdvals(x1.T @ y1 / h)[:4]
print("lambda_max(Bxx) top:", sx.tolist())
print("lambda_max(Byy) top:", sy.tolist())
print("sigma_max(Cxy) top:", sxy.tolist())
print("mean |X|", X.abs().mean().item(), "row norm^2 mean", (X.double() ** 2).sum(1).mean().item())
