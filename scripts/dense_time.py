"""Developer: config 4 (dense GEP d=16384, k=128, fp32 A/B) step time on the
staged tf32 / 3xTF32 path: products (A V^T, B V^T reading 2 GiB) + update."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, dense_gep_large, gaussian_init
cfg = CONFIGS[4]
dev = "cuda:0"
a, b = dense_gep_large(cfg.d, seed=0, device=dev)
for math in sys.argv[1:] or ["tf32", "3xtf32"]:
    s = geig.Solver(geig.GEIG_DENSE, cfg.d, 0, cfg.k, math=math, rho=cfg.rho)
    s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
    AV = torch.empty(cfg.k, cfg.d, device=dev); BV = torch.empty_like(AV)
    for _ in range(3):
        geig.geig_step_dense(s.h, a, b, cfg.eta, cfg.gamma)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    n = 20
    e[0].record()
    for _ in range(n):
        geig.geig_products_dense(s.h, a, b, 0, cfg.d, AV, BV)
    e[1].record()
    for _ in range(n):
        geig.geig_update(s.h, AV, BV, cfg.eta, cfg.gamma)
    e[2].record()
    torch.cuda.synchronize()
    tp = e[0].elapsed_time(e[1]) / n
    tu = e[1].elapsed_time(e[2]) / n
    byts = 2 * cfg.d * cfg.d * 4
    print(f"{math}: products {tp*1e3:.1f} us ({byts / (tp*1e-3) / 1e12:.2f} TB/s of A,B), update {tu*1e3:.1f} us, "
          f"tensor {4 * cfg.k * cfg.d * cfg.d / (tp*1e-3) / 1e12:.1f} TFLOP/s")
    s.close()
# phase split of the last update (CTA 0 %globaltimer): gram, reduce, coef+update
s = geig.Solver(geig.GEIG_DENSE, cfg.d, 0, cfg.k, math="tf32", rho=cfg.rho)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
AV = torch.empty(cfg.k, cfg.d, device=dev); BV = torch.empty_like(AV)
geig.geig_products_dense(s.h, a, b, 0, cfg.d, AV, BV)
for _ in range(3):
    geig.geig_update(s.h, AV, BV, cfg.eta, cfg.gamma)
torch.cuda.synchronize()
print("update phases (us):", [x / 1e3 for x in geig.geig_update_phase_ns(s.h)[:3]])
