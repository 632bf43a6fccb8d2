"""Same-box A/B of GEIG_OPT_FUSED_M_TILES (0 = auto, 1, 2: 128-row M tiles
per fused work item) on geig_run_cca, interleaved: median us/step over 200
distinct-batch steps (a ring of batches larger than L2 where it fits)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = "cuda:0"
# optional shape override: DX K B (views sliced from the config's recipe)
dx = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.dx
k = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.k
b = int(sys.argv[5]) if len(sys.argv) > 5 else cfg.batch
P = max(4, min(64, int(4 * 126e6 // (b * 2 * dx * 2)) + 1))
X, Y = cca_views(cfg, P * b, seed=5, device=dev, dtype=torch.bfloat16)
X, Y = X[:, :dx].contiguous(), Y[:, :dx].contiguous()
Xs = [X[i * b:(i + 1) * b].contiguous() for i in range(P)]
Ys = [Y[i * b:(i + 1) * b].contiguous() for i in range(P)]
T = 200
opts = (0, 1, 2)
solvers = {}
for o in opts:
    s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho,
                    max_rows=b)
    geig.geig_set_option(s.h, geig.GEIG_OPT_FUSED_M_TILES, o)
    s.init_state(torch.tensor(gaussian_init(k, 2 * dx, 0), dtype=torch.float32, device=dev))
    solvers[o] = s
args = geig.cca_batches([Xs[i % P] for i in range(T)], [Ys[i % P] for i in range(T)])
res = {o: [] for o in opts}
for r in range(rounds):
    for o in opts:
        s = solvers[o]
        geig.geig_run_cca(s.h, None, None, b, cfg.eta, cfg.gamma, batches=args)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        geig.geig_run_cca(s.h, None, None, b, cfg.eta, cfg.gamma, batches=args)
        e1.record()
        torch.cuda.synchronize()
        res[o].append(e0.elapsed_time(e1) * 1e3 / T)
print(f"dx=dy={dx} k={k} b={b}")
for o in opts:
    print(f"m_tiles={o}: median {statistics.median(res[o]):.2f} us/step  all {[round(x, 2) for x in res[o]]}")
