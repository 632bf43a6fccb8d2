"""Developer check of the CTA-pair exchange (needs a GEIG_DEV_KNOBS build):
one fused step at config 3 with pairs (GEIG_DBG_MODE=16384 dumps the
exchanged AV / BV tiles to the solver's AV, BV) vs the products-only launch."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[3]
MATH = sys.argv[1] if len(sys.argv) > 1 else "bf16x2"
dev = "cuda:0"
b = cfg.batch
X, Y = cca_views(cfg, b, seed=5, device=dev, dtype=torch.bfloat16)
G = torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev)
s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math=MATH, data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho, max_rows=b)
s.init_state(G)
AV = torch.zeros(cfg.k, cfg.d, device=dev); BV = torch.zeros_like(AV)
geig.geig_products_cca(s.h, X, Y, b, 1.0 / (b // 2), AV, BV)
torch.cuda.synchronize()
# the solver's internal AV / BV: the arena after V, AUX
kd = cfg.k * cfg.d
s.init_state(G)
os.environ["GEIG_DBG_MODE"] = "16384"
geig.geig_step_cca(s.h, X, Y, b, cfg.eta, cfg.gamma)
torch.cuda.synchronize()
lib = geig._lib
lib.geig_debug_products.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]
pa, pb = ctypes.c_void_p(), ctypes.c_void_p()
lib.geig_debug_products(s.h, ctypes.byref(pa), ctypes.byref(pb))
nb = kd * 4
ha = torch.empty(kd, dtype=torch.float32)
hb = torch.empty(kd, dtype=torch.float32)
torch.cuda.synchronize()
lib_rt = ctypes.CDLL("libcudart.so.12")


def d2h(ptr, out):   # cudaMemcpy device -> host of the raw pointer
    lib_rt.cudaMemcpy(ctypes.c_void_p(out.data_ptr()), ptr, ctypes.c_size_t(nb), 2)
d2h(pa, ha); d2h(pb, hb)
ga = ha.view(cfg.k, cfg.d).numpy(); gb = hb.view(cfg.k, cfg.d).numpy()
ra = AV.cpu().numpy(); rb = BV.cpu().numpy()
for name, g_, r_ in (("AV", ga, ra), ("BV", gb, rb)):
    err = np.linalg.norm(g_ - r_) / np.linalg.norm(r_)
    colerr = np.linalg.norm(g_ - r_, axis=0) / (np.linalg.norm(r_, axis=0) + 1e-30)
    bad = np.nonzero(colerr > 1e-3)[0]
    print(name, "rel err", err, "bad columns", len(bad), bad[:20], "zero cols", int(np.sum(np.all(g_ == 0, axis=0))))
    if len(bad):
        c = bad[0]
        print("  col", c, "got", g_[:4, c], "ref", r_[:4, c])
        # is the column a shifted copy of another reference column?
        m = np.argmin(np.linalg.norm(r_ - g_[:, c:c + 1], axis=0))
        print("  closest ref column", m, np.linalg.norm(r_[:, m] - g_[:, c]) / np.linalg.norm(r_[:, m]))

