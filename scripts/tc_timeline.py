"""Per-CTA timeline of the tensor-core product kernels (developer tool)."""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import build
build.build()
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[3]
dev = "cuda:0"
X, Y = cca_views(cfg, 2 * cfg.batch, seed=5, device=dev, dtype=torch.bfloat16)
b = cfg.batch
s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math="bf16", data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho, max_rows=b)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
AV = torch.empty(cfg.k, cfg.d, device=dev); BV = torch.empty_like(AV)
lib = geig._lib
lib.geig_debug_set_tc_stamps.argtypes = [ctypes.c_void_p]
for it in range(3):
    geig.geig_products_cca(s.h, X[:b], Y[:b], b, 1.0 / (b // 2), AV, BV)
torch.cuda.synchronize()
buf = torch.zeros(4 * 8192, dtype=torch.int64, device=dev)
lib.geig_debug_set_tc_stamps(ctypes.c_void_p(buf.data_ptr()))
geig.geig_products_cca(s.h, X[b:2*b], Y[b:2*b], b, 1.0 / (b // 2), AV, BV)
torch.cuda.synchronize()
lib.geig_debug_set_tc_stamps(None)
t = buf.view(-1, 4).cpu()
t0 = t[t[:, 0] > 0][:, 0].min().item()
off = 0
for name, n in (("forward", 128), ("backward", 128)):
    tt = t[off:off + n]
    off += n
    st = ((tt - t0).double() / 1e3)
    print(f"{name} ({n} CTAs): start [{st[:,0].min():.1f},{st[:,0].max():.1f}] "
          f"first-data med {statistics.median(st[:,1].tolist()):.1f} "
          f"accum-ready med {statistics.median(st[:,2].tolist()):.1f} max {st[:,2].max():.1f} "
          f"end med {statistics.median(st[:,3].tolist()):.1f} max {st[:,3].max():.1f} us")
