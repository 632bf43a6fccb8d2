"""Developer: localise the first non-finite state of the multi-step fused
launch: chunks of C steps; at the first bad chunk print which players /
columns of V and [Bv] are non-finite and whether the step's Gram tables
are finite.  usage: race_probe3.py ROWS STEPS C R"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[1]
n, steps, C, R = (int(a) for a in sys.argv[1:5])
dx, k, eta = 64, 8, 0.0086
x, y = cca_views(cfg, n, seed=3)
x, y = x[:, :dx].to(torch.bfloat16).contiguous().cuda(), y[:, :dx].to(torch.bfloat16).contiguous().cuda()
for r in range(R):
    s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math="bf16x2", data_dtype=1, rho=cfg.rho, max_rows=n)
    s.init_state(torch.tensor(gaussian_init(k, 2 * dx, 0), dtype=torch.float32, device="cuda:0"))
    for c in range(steps // C):
        geig.geig_run_cca(s.h, [x] * C, [y] * C, n, eta, 1.0)
        V, A = s.state()
        Vr = torch.empty_like(V)
        geig.geig_get(s.h, None, None)
        if not (torch.isfinite(V).all() and torch.isfinite(A).all()):
            ga, gb, gc = s.gram()
            badV = ~torch.isfinite(V)
            badA = ~torch.isfinite(A)
            print(f"repeat {r} chunk {c}: V bad rows {torch.nonzero(badV.any(1)).flatten().tolist()} "
                  f"cols {torch.nonzero(badV.any(0)).flatten().tolist()[:40]} | AUX bad rows "
                  f"{torch.nonzero(badA.any(1)).flatten().tolist()} cols {torch.nonzero(badA.any(0)).flatten().tolist()[:40]} "
                  f"| gram finite A {bool(torch.isfinite(ga).all())} B {bool(torch.isfinite(gb).all())} "
                  f"C {bool(torch.isfinite(gc).all())}", flush=True)
            print("  V finite-part max", float(V[torch.isfinite(V)].abs().max()), "gb diag", torch.diagonal(gb).tolist())
            break
    else:
        print(f"repeat {r}: ok", flush=True)
    s.close()
