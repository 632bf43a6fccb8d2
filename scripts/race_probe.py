"""Developer: determinism probe of the fused step at a large batch.  Runs the
same seeded sequence R times (fresh solver each), chunks of C steps per
geig_run_cca launch, and reports the first chunk where the states of the
repeats differ bitwise or turn NaN.  usage: race_probe.py CFG ROWS DX K STEPS C R ETA"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[int(sys.argv[1])]
n, dx, k, steps, C, R, eta = (int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]),
                              int(sys.argv[6]), int(sys.argv[7]), float(sys.argv[8]))
math = sys.argv[9] if len(sys.argv) > 9 else "bf16x2"
x, y = cca_views(cfg, n, seed=3)
x, y = x[:, :dx].to(torch.bfloat16).contiguous().cuda(), y[:, :dx].to(torch.bfloat16).contiguous().cuda()
hist = []
for r in range(R):
    s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math=math, data_dtype=1, rho=cfg.rho, max_rows=n)
    s.init_state(torch.tensor(gaussian_init(k, 2 * dx, 0), dtype=torch.float32, device="cuda:0"))
    states = []
    for c in range(steps // C):
        if os.environ.get("SINGLE"):
            for _ in range(C):
                geig.geig_step_cca(s.h, x, y, n, eta, 1.0)
        else:
            geig.geig_run_cca(s.h, [x] * C, [y] * C, n, eta, 1.0)
        V, A = s.state()
        states.append(torch.cat([V.flatten(), A.flatten()]).cpu())
    s.close()
    hist.append(states)
    bad = [i for i, st in enumerate(states) if not torch.isfinite(st).all()]
    print(f"repeat {r}: first non-finite chunk {bad[0] if bad else None}", flush=True)
for r in range(1, R):
    diff = [i for i in range(len(hist[0])) if not torch.equal(hist[0][i], hist[r][i])]
    print(f"repeat {r} vs 0: first differing chunk {diff[0] if diff else None} (of {len(hist[0])})", flush=True)
