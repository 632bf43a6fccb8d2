"""Per-phase timing of the hot path on one workload (developer tool):
CUDA-event time of the products stage and %globaltimer phase stamps of the
cooperative update kernel."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import build
build.build()
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
math = sys.argv[2] if len(sys.argv) > 2 else "bf16"
dev = "cuda:0"
dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
X, Y = cca_views(cfg, 4 * cfg.batch, seed=5, device=dev, dtype=dt)
b = cfg.batch
s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math=math,
                data_dtype=geig.GEIG_DATA_BF16 if dt == torch.bfloat16 else geig.GEIG_DATA_F32,
                rho=cfg.rho, max_rows=b)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
AV = torch.empty(cfg.k, cfg.d, device=dev); BV = torch.empty_like(AV)
st = torch.cuda.current_stream()
prod, upd, phases = [], [], []
for it in range(30):
    i = it % 4
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(st)
    geig.geig_products_cca(s.h, X[i*b:(i+1)*b], Y[i*b:(i+1)*b], b, 1.0/(b//2), AV, BV)
    e1.record(st)
    geig.geig_update(s.h, AV, BV, cfg.eta, cfg.gamma)
    e2.record(st)
    torch.cuda.synchronize()
    if it >= 5:
        prod.append(e0.elapsed_time(e1) * 1e3); upd.append(e1.elapsed_time(e2) * 1e3)
        phases.append(geig.geig_update_phase_ns(s.h))
print(f"config {cfg.index} {math}: products {statistics.median(prod):.1f} us, update {statistics.median(upd):.1f} us")
steps = []
for it in range(30):
    i = it % 4
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    e0.record(st)
    geig.geig_step_cca(s.h, X[i*b:(i+1)*b], Y[i*b:(i+1)*b], b, cfg.eta, cfg.gamma)
    e1.record(st)
    torch.cuda.synchronize()
    if it >= 5:
        steps.append((e0.elapsed_time(e1) * 1e3, geig.geig_update_phase_ns(s.h)))
print(f"  geig_step_cca: {statistics.median(t for t, _ in steps):.1f} us/step; fused phases: "
      f"forward {statistics.median(p[3] for _, p in steps)/1e3:.1f} reshuffle+backward {statistics.median(p[4] for _, p in steps)/1e3:.1f} "
      f"gram {statistics.median(p[0] for _, p in steps)/1e3:.1f} reduce {statistics.median(p[1] for _, p in steps)/1e3:.1f} "
      f"coef+update {statistics.median(p[2] for _, p in steps)/1e3:.1f} us")
names = ["gram", "reduce", "coef+update"]
for j, n in enumerate(names):
    print(f"  phase {n:8s} {statistics.median(p[j] for p in phases)/1e3:8.2f} us")
