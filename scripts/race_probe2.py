"""Developer: single-step launches (geig_step_cca) at a large batch, the
state checked after every step; on the first non-finite state, report the
step's Gram tables (finite or not) and which players / columns are hit.
usage: race_probe2.py CFG ROWS DX K STEPS R ETA [MATH]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[int(sys.argv[1])]
n, dx, k, steps, R, eta = (int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]),
                           int(sys.argv[6]), float(sys.argv[7]))
math = sys.argv[8] if len(sys.argv) > 8 else "bf16x2"
x, y = cca_views(cfg, n, seed=3)
x, y = x[:, :dx].to(torch.bfloat16).contiguous().cuda(), y[:, :dx].to(torch.bfloat16).contiguous().cuda()
for r in range(R):
    s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math=math, data_dtype=1, rho=cfg.rho, max_rows=n)
    s.init_state(torch.tensor(gaussian_init(k, 2 * dx, 0), dtype=torch.float32, device="cuda:0"))
    bad = None
    for t in range(steps):
        geig.geig_step_cca(s.h, x, y, n, eta, 1.0)
        if t % 10 == 9:
            V, A = s.state()
            if not (torch.isfinite(V).all() and torch.isfinite(A).all()):
                ga, gb, gc = s.gram()
                bad = t
                print(f"repeat {r}: non-finite at step <= {t}; gram finite A {bool(torch.isfinite(ga).all())} "
                      f"B {bool(torch.isfinite(gb).all())} C {bool(torch.isfinite(gc).all())}; "
                      f"nonfinite V rows {torch.nonzero(~torch.isfinite(V).all(1)).flatten().tolist()} "
                      f"cols {torch.nonzero(~torch.isfinite(V).all(0)).flatten().tolist()[:20]}", flush=True)
                print("ga diag", torch.diagonal(ga).tolist(), "\ngb diag", torch.diagonal(gb).tolist(), flush=True)
                break
    if bad is None:
        print(f"repeat {r}: ok", flush=True)
    s.close()
