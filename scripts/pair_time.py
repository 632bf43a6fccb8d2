"""Same-box A/B of the fused config-3 step with and without CTA pairs
(GEIG_OPT_FUSED_PAIRS), interleaved: median us/step of geig_run_cca over
200 distinct-batch steps (a ring of 4 batches)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = "cuda:0"
b = cfg.batch
P = 4
X, Y = cca_views(cfg, P * b, seed=5, device=dev, dtype=torch.bfloat16)
Xs = [X[i * b:(i + 1) * b].contiguous() for i in range(P)]
Ys = [Y[i * b:(i + 1) * b].contiguous() for i in range(P)]
T = 200
solvers = {}
for pairs in (0, 1, 2):
    s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho,
                    max_rows=b)
    geig.geig_set_option(s.h, geig.GEIG_OPT_FUSED_PAIRS, pairs)
    s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
    solvers[pairs] = s
args = geig.cca_batches([Xs[i % P] for i in range(T)], [Ys[i % P] for i in range(T)])
res = {0: [], 1: [], 2: []}
for r in range(rounds):
    for pairs in (0, 1, 2):
        s = solvers[pairs]
        geig.geig_run_cca(s.h, None, None, b, cfg.eta, cfg.gamma, batches=args)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        geig.geig_run_cca(s.h, None, None, b, cfg.eta, cfg.gamma, batches=args)
        e1.record()
        torch.cuda.synchronize()
        res[pairs].append(e0.elapsed_time(e1) * 1e3 / T)
for pairs in (0, 1, 2):
    print(f"pairs={pairs}: median {statistics.median(res[pairs]):.2f} us/step  all {[round(x, 2) for x in res[pairs]]}")
