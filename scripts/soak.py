"""Soak test (developer tool): repeats multi-step fused launches against
single-step launches on the same batches and requires BIT-IDENTICAL states
every time — a race in the persistent kernel's phase hand-offs (counters,
mbarriers, CTA-pair exchange, cluster reductions) shows up as a rare
mismatch or a NaN.  Usage: soak.py SECONDS_PER_CASE"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import build
build.build()
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
dev = "cuda:0"
# (config recipe, dx, k, batch, math, data dtype, steps per launch)
CASES = [(3, 8192, 64, 4096, "bf16x2", torch.bfloat16, 6),     # CTA pairs, the benched configuration
         (3, 1024, 64, 1024, "bf16x2", torch.bfloat16, 12),    # pairs on a small grid
         (2, 784, 16, 1024, "bf16x2", torch.bfloat16, 12),     # config 2: one CTA per item, widened grid
         (2, 784, 16, 1024, "bf16", torch.bfloat16, 12),
         (1, 64, 8, 256, "f32", torch.float32, 40)]            # small-problem cluster step
bad = 0
for ci, dx, k, b, math, dt, T in CASES:
    cfg = CONFIGS[ci]
    X, Y = cca_views(cfg, T * b, seed=11, device=dev, dtype=dt)
    X, Y = X[:, :dx].contiguous(), Y[:, :dx].contiguous()
    xs = [X[i * b:(i + 1) * b] for i in range(T)]
    ys = [Y[i * b:(i + 1) * b] for i in range(T)]
    G = torch.tensor(gaussian_init(k, 2 * dx, 0), dtype=torch.float32, device=dev)
    dd = geig.GEIG_DATA_BF16 if dt == torch.bfloat16 else geig.GEIG_DATA_F32

    def fresh():
        s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math=math, data_dtype=dd, rho=cfg.rho, max_rows=b)
        s.init_state(G)
        return s
    s = fresh()
    for i in range(T):
        geig.geig_step_cca(s.h, xs[i], ys[i], b, cfg.eta, cfg.gamma)
    Vr, Ar = s.state()
    s.close()
    assert torch.isfinite(Vr).all() and torch.isfinite(Ar).all(), "reference steps are not finite"
    t0, n, miss = time.time(), 0, 0
    s = fresh()
    while time.time() - t0 < budget:
        s.init_state(G)
        if n % 2 == 0:
            geig.geig_run_cca(s.h, xs, ys, b, cfg.eta, cfg.gamma)
        else:
            for i in range(T):
                geig.geig_step_cca(s.h, xs[i], ys[i], b, cfg.eta, cfg.gamma)
        V, A = s.state()
        if not (torch.equal(V, Vr) and torch.equal(A, Ar)):
            miss += 1
            print(f"  MISMATCH rep {n}: max |dV| {(V - Vr).abs().max().item():.3e} finite {bool(torch.isfinite(V).all())}",
                  flush=True)
        n += 1
    s.close()
    bad += miss
    print(f"config-{ci} recipe dx={dx} k={k} b={b} {math}: {n} repeats x {T} steps, {miss} mismatches", flush=True)
print("SOAK", "FAILED" if bad else "ok")
sys.exit(1 if bad else 0)
