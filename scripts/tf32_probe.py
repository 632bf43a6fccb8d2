"""Developer probe: tf32 CCA products (staged path) vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
from paper_2206_04993_b200 import geig
import tests.gpu_harness as gh
_cv = gh.cca_views
gh.cca_views = lambda *a, **kw: tuple(t.float() for t in _cv(*a, **kw))
for args in [(1, 256, None, None, None), (2, 300, 24, 200, 136), (2, 1024, 16, 784, 784)]:
    errs, got = gh.check_cca_step(geig, args[0], args[1], k=args[2], dx=args[3], dy=args[4], math="tf32")
    print(args, {k: float(f"{v:.3g}") for k, v in errs.items()}, "av max", float(abs(got["av"]).max()))
