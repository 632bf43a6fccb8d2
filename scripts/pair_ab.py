"""Developer A/B: one fused config-3 step with and without CTA pairs from the
same state (plain bf16 and bf16x2), repeated; prints the relative
differences of V and [Bv]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views
from tests.gpu_harness import random_state, rel_err
cfg = CONFIGS[3]
dev = "cuda:0"
b = cfg.batch
X, Y = cca_views(cfg, b, seed=5, device=dev, dtype=torch.bfloat16)
V, aux = random_state(cfg.k, cfg.d, 3)
for math in ("bf16", "bf16x2"):
    for rep in range(3):
        out = []
        for pairs in (1, 0):
            s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math=math, data_dtype=geig.GEIG_DATA_BF16,
                            rho=cfg.rho, max_rows=b)
            geig.geig_set_option(s.h, geig.GEIG_OPT_FUSED_PAIRS, pairs)
            s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
            geig.geig_step_cca(s.h, X, Y, b, 0.02, cfg.gamma)
            out.append([t.double().cpu().numpy() for t in s.state()])
            s.close()
        (Vp, ap), (Vs, as_) = out
        d = np.linalg.norm(Vp - Vs, axis=1) / np.linalg.norm(Vs - V, axis=1)
        print(math, rep, "step", rel_err(Vp - V, Vs - V), "aux", rel_err(ap, as_), "worst rows", np.argsort(d)[-6:], d[np.argsort(d)[-3:]])
