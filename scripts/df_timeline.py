"""Per-CTA timeline of the dataflow step kernel (developer tool)."""
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
lib = geig._lib
lib.geig_debug_set_tc_stamps.argtypes = [ctypes.c_void_p]
for it in range(3):
    geig.geig_step_cca(s.h, X[:b], Y[:b], b, cfg.eta, cfg.gamma)
torch.cuda.synchronize()
buf = torch.zeros(8 * 256, dtype=torch.int64, device=dev)
lib.geig_debug_set_tc_stamps(ctypes.c_void_p(buf.data_ptr()))
geig.geig_step_cca(s.h, X[b:2*b], Y[b:2*b], b, cfg.eta, cfg.gamma)
torch.cuda.synchronize()
lib.geig_debug_set_tc_stamps(None)
t = buf.view(-1, 8).cpu()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min().item()
st = (t - t0).double() / 1e3
names = ["start", "producer done", "MMA done", "epilogue done", "F issued", "F drained"]
for j, n in enumerate(names):
    col = st[:, j]
    col = col[t[:, j] > 0]
    if len(col):
        print(f"{n:14s} min {col.min():7.1f} med {statistics.median(col.tolist()):7.1f} max {col.max():7.1f} us (n={len(col)})")
order = sorted(range(len(t)), key=lambda i: -st[i, 5].item())
print("slowest F-drained CTAs:", [(i, round(st[i, 5].item(), 1), round(st[i, 4].item(), 1)) for i in order[:12]])
print("fastest:", [(i, round(st[i, 5].item(), 1)) for i in order[-5:]])

red = t[:, 6].double() / 1e3
fix = t[:, 7].double() / 1e3
print(f"epilogue red-phase total per CTA: med {statistics.median(red.tolist()):.1f} max {red.max():.1f} us; fix-up total: med {statistics.median(fix.tolist()):.1f} max {fix.max():.1f} us")
