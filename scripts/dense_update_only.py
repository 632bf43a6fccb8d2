"""Developer: config-4 update launches only (target of ncu captures of the
k > 64 update: the tensor-core Gram launch and update_kernel<2>)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, dense_gep_large, gaussian_init
cfg = CONFIGS[4]
dev = "cuda:0"
a, b = dense_gep_large(cfg.d, seed=0, device=dev)
s = geig.Solver(geig.GEIG_DENSE, cfg.d, 0, cfg.k, math=sys.argv[1] if len(sys.argv) > 1 else "tf32", rho=cfg.rho)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
AV = torch.empty(cfg.k, cfg.d, device=dev); BV = torch.empty_like(AV)
geig.geig_products_dense(s.h, a, b, 0, cfg.d, AV, BV)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    geig.geig_update(s.h, AV, BV, cfg.eta, cfg.gamma)
torch.cuda.synchronize()
e[0].record()
for _ in range(n):
    geig.geig_update(s.h, AV, BV, cfg.eta, cfg.gamma)
e[1].record()
torch.cuda.synchronize()
print(f"update {e[0].elapsed_time(e[1]) / n * 1e3:.1f} us; phases (us):",
      [x / 1e3 for x in geig.geig_update_phase_ns(s.h)[:4]])
