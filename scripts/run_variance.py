"""Developer: time geig_run_cca over repeated windows of K steps (config 3) to
expose run-to-run variance (clocks, power capping, L2 policy)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[3]
dev = "cuda:0"
b = cfg.batch
P = 4
X, Y = cca_views(cfg, P * b, seed=1, device=dev, dtype=torch.bfloat16)
Xs = [X[i * b:(i + 1) * b] for i in range(P)]
Ys = [Y[i * b:(i + 1) * b] for i in range(P)]
st = torch.cuda.Stream()
s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math=sys.argv[1] if len(sys.argv) > 1 else "bf16x2",
                data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho, max_rows=b, stream=st.cuda_stream)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
K = 100
with torch.cuda.stream(st):
    out = []
    for rep in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        geig.geig_run_cca(s.h, [Xs[i % P] for i in range(K)], [Ys[i % P] for i in range(K)], b, cfg.eta, cfg.gamma)
        e1.record(st)
        e1.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / K)
print("us/step per window of %d:" % K, " ".join(f"{v:.1f}" for v in out))
