"""Streamed-minibatch convergence probe (developer): Alg. 2 on the GPU over
minibatches drawn with replacement from a seeded pool of a BASELINE recipe,
eta_t = eta0 / (1 + t / tau) (square-summable, not summable: Theorem 1),
gamma_t = gamma0 / (1 + t / tau_g); prints per-vector angles and principal
angles vs the pool's exact GEP (oracle, fp64) at checkpoints.
usage: conv_streamed.py CFG MATH STEPS ETA0 TAU GAMMA0 TAUG [DX K POOL]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_04993_b200 import geig
from oracle import estimators, linalg, metrics
from synth import CONFIGS, cca_views, gaussian_init

cfg = CONFIGS[int(sys.argv[1])]
math = sys.argv[2]
steps, eta0, tau, g0, taug = int(sys.argv[3]), float(sys.argv[4]), float(sys.argv[5]), float(sys.argv[6]), float(sys.argv[7])
dx = int(sys.argv[8]) if len(sys.argv) > 8 else cfg.dx
k = int(sys.argv[9]) if len(sys.argv) > 9 else cfg.k
n = int(sys.argv[10]) if len(sys.argv) > 10 else min(cfg.n, 200_000)
b = cfg.batch
dev = "cuda:0"
dt = torch.bfloat16 if math in ("bf16", "bf16x2") else torch.float32
x, y = cca_views(cfg, n, seed=3)
x, y = x[:, :dx].to(dt).contiguous(), y[:, :dx].to(dt).contiguous()
t0 = time.time()
a, bm = estimators.cca_matrices(x.double().numpy(), y.double().numpy())
w, Vt = linalg.generalized_eigh(a, bm, k + 1)
print("lambda_{k+1} =", round(float(w[k]), 4))
w, Vt = w[:k], Vt[:k]
print(f"pool {n} rows, d={2*dx}, k={k}; exact top-k correlations {np.round(w, 4)}; gaps {np.round(-np.diff(w), 4)} "
      f"(solve {time.time()-t0:.1f}s)", flush=True)
xd, yd = x.to(dev), y.to(dev)
s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math=math, data_dtype=1 if dt == torch.bfloat16 else 0, rho=cfg.rho, max_rows=b)
s.init_state(torch.tensor(gaussian_init(k, 2 * dx, 0), dtype=torch.float32, device=dev))
g = torch.Generator(device=dev)
g.manual_seed(11)
CH = 500
done = 0
t0 = time.time()
while done < steps:
    nch = min(CH, steps - done)
    idx = torch.randint(0, n, (nch, b), generator=g, device=dev)
    XB = xd[idx]
    YB = yd[idx]
    for i in range(nch):
        t = done + i
        eta = eta0 / (1 + t / tau)
        gam = g0 / (1 + t / taug)
        geig.geig_step_cca(s.h, XB[i], YB[i], b, eta, gam)
    done += nch
    if done % (steps // 10) < CH or done == steps:
        V, _ = s.state()
        Vg = V.double().cpu().numpy()
        ang = metrics.per_vector_angles(Vg, Vt)
        Q1, _ = np.linalg.qr(Vg.T); Q2, _ = np.linalg.qr(Vt.T)
        pa = np.arccos(np.clip(np.linalg.svd(Q1.T @ Q2, compute_uv=False), -1, 1))
        print(f"step {done:7d} ({time.time()-t0:5.1f}s) mean angle {ang.mean():.2e} max {ang.max():.2e} "
              f"| principal angles mean {pa.mean():.2e} max {pa.max():.2e}", flush=True)
s.close()
