"""Run a few fused CCA steps at config 3 (developer: target for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
math = sys.argv[2] if len(sys.argv) > 2 else "bf16x2"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev = "cuda:0"
b = cfg.batch
X, Y = cca_views(cfg, b, seed=5, device=dev, dtype=torch.bfloat16)
s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math=math, data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho, max_rows=b)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
for it in range(n):
    geig.geig_step_cca(s.h, X, Y, b, cfg.eta, cfg.gamma)
torch.cuda.synchronize()
print("ok")
