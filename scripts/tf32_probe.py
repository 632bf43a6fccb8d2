"""Developer probe: tf32 / 3xTF32 CCA products (staged path) vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
import tests.gpu_harness as gh
_cv = gh.cca_views
gh.cca_views = lambda *a, **kw: tuple(t.float() for t in _cv(*a, **kw))
for math in sys.argv[1:] or ["tf32", "3xtf32"]:
    for args in [(1, 256, None, None, None), (2, 300, 24, 200, 136), (2, 1024, 16, 784, 784), (3, 2048, 64, 1024, 512)]:
        errs, got = gh.check_cca_step(geig, args[0], args[1], k=args[2], dx=args[3], dy=args[4], math=math)
        print(math, args, {k: float(f"{v:.3g}") for k, v in errs.items()}, flush=True)
