"""Full-pool (b = n) convergence probe (developer): Alg. 2 on the GPU with
the whole pool as the batch every step (the paper's b = n setting,
PAPER.md:1096), eta constant; per-vector and principal angles vs the pool's
exact GEP (oracle).  usage: conv_full.py CFG MATH STEPS ETA GAMMA [DX K N]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_04993_b200 import geig
from oracle import estimators, linalg, metrics
from synth import CONFIGS, cca_views, gaussian_init

cfg = CONFIGS[int(sys.argv[1])]
math = sys.argv[2]
steps, eta, gam = int(sys.argv[3]), float(sys.argv[4]), float(sys.argv[5])
dx = int(sys.argv[6]) if len(sys.argv) > 6 else cfg.dx
k = int(sys.argv[7]) if len(sys.argv) > 7 else cfg.k
n = int(sys.argv[8]) if len(sys.argv) > 8 else min(cfg.n, 100_000)
dev = "cuda:0"
dt = torch.bfloat16 if math in ("bf16", "bf16x2") else torch.float32
x, y = cca_views(cfg, n, seed=3)
x, y = x[:, :dx].to(dt).contiguous(), y[:, :dx].to(dt).contiguous()
t0 = time.time()
a_t, b_t = estimators.cca_minibatch_matrices(x.double().numpy(), y.double().numpy())
w, Vt = linalg.generalized_eigh(a_t, b_t, k + 1)
print(f"n={n} d={2*dx} k={k} top-k {np.round(w[:k], 4)} lambda_k+1 {w[k]:.4f} min gap {np.min(-np.diff(w[:k+1])):.2e} "
      f"({time.time()-t0:.1f}s)", flush=True)
w, Vt = w[:k], Vt[:k]
xd, yd = x.to(dev), y.to(dev)
s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math=math, data_dtype=1 if dt == torch.bfloat16 else 0, rho=cfg.rho, max_rows=n)
s.init_state(torch.tensor(gaussian_init(k, 2 * dx, 0), dtype=torch.float32, device=dev))
done, t0 = 0, time.time()
CH = max(1, steps // 10)
while done < steps:
    m = min(CH, steps - done)
    if math in ("bf16", "bf16x2"):
        geig.geig_run_cca(s.h, [xd] * m, [yd] * m, n, eta, gam)
    else:
        for _ in range(m):
            geig.geig_step_cca(s.h, xd, yd, n, eta, gam)
    done += m
    V, _ = s.state()
    Vg = V.double().cpu().numpy()
    ang = metrics.per_vector_angles(Vg, Vt)
    Q1, _ = np.linalg.qr(Vg.T); Q2, _ = np.linalg.qr(Vt.T)
    pa = np.arccos(np.clip(np.linalg.svd(Q1.T @ Q2, compute_uv=False), -1, 1))
    print(f"step {done:7d} ({time.time()-t0:5.1f}s) per-vector mean {ang.mean():.2e} max {ang.max():.2e} | principal mean {pa.mean():.2e} max {pa.max():.2e}", flush=True)
s.close()
