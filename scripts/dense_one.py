"""One config-4 dense products launch (tf32) after two warm-up launches
(developer: target for ncu captures of the products kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, dense_gep_large, gaussian_init
cfg = CONFIGS[4]
dev = "cuda:0"
a, b = dense_gep_large(cfg.d, seed=0, device=dev)
s = geig.Solver(geig.GEIG_DENSE, cfg.d, 0, cfg.k, math="tf32", rho=cfg.rho)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
AV = torch.empty(cfg.k, cfg.d, device=dev); BV = torch.empty_like(AV)
for _ in range(3):
    geig.geig_products_dense(s.h, a, b, 0, cfg.d, AV, BV)
torch.cuda.synchronize()
print("ok")
