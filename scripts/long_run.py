"""Developer: sustained run of the fused step (config 3, bf16x2): N steps in
persistent launches over a ring of distinct batches; checks the state stays
finite and on the sphere, reports the sustained step time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[3]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
eta = float(sys.argv[2]) if len(sys.argv) > 2 else cfg.eta
gamma = float(sys.argv[3]) if len(sys.argv) > 3 else cfg.gamma
dev = "cuda:0"
b = cfg.batch
P = 4
X, Y = cca_views(cfg, P * b, seed=11, device=dev, dtype=torch.bfloat16)
Xs = [X[i * b:(i + 1) * b] for i in range(P)]
Ys = [Y[i * b:(i + 1) * b] for i in range(P)]
s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho,
                max_rows=b)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
chunk = 2000
args = geig.cca_batches([Xs[i % P] for i in range(chunk)], [Ys[i % P] for i in range(chunk)])
torch.cuda.synchronize()
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N // chunk):
    geig.geig_run_cca(s.h, None, None, b, eta, gamma, batches=args)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
V, Bv = s.state()
n = V.norm(dim=1)
print(f"{N} steps: {ms * 1e3 / N:.2f} us/step, {N * b / (ms / 1e3) / 1e6:.1f} M samples/s; "
      f"finite V {bool(torch.isfinite(V).all())}, [Bv] {bool(torch.isfinite(Bv).all())}, "
      f"|v_i| in [{n.min().item():.6f}, {n.max().item():.6f}]")
ga, gb, gc = s.gram()
print(f"eta {eta} gamma {gamma}: diag <v_i, [Bv]_i> (first 8):", [round(x, 3) for x in torch.diagonal(gc)[:8].tolist()])
print("  lambda_i estimates <v_i, A_t v_i> / <v_i, [Bv]_i> (first 8):",
      [round(x, 3) for x in (torch.diagonal(ga) / torch.diagonal(gc))[:8].tolist()])
s.close()
