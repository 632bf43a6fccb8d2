"""Per-CTA timeline of the fused CCA step kernel (developer tool): per CTA,
%globaltimer (cross-CTA) and clock64 (intra-CTA intervals) stamps written
through geig_debug_set_tc_stamps (64 slots per CTA)."""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import build
build.build()
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
math = sys.argv[2] if len(sys.argv) > 2 else "bf16x2"
MHZ = float(os.environ.get("SM_MHZ", "1965"))
dev = "cuda:0"
b = cfg.batch
X, Y = cca_views(cfg, 2 * b, seed=5, device=dev, dtype=torch.bfloat16)
s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math=math, data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho, max_rows=b)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
lib = geig._lib
lib.geig_debug_set_tc_stamps.argtypes = [ctypes.c_void_p]
names = {0: "launch", 1: "setup", 2: "F done", 3: "F sync", 4: "S done", 5: "S sync", 6: "B done", 7: "B sync",
         8: "U staged", 9: "F accf", 10: "B coef end", 11: "B accf", 12: "B red all", 13: "U coef", 14: "U update",
         15: "B fence0", 16: "B epi fence", 17: "B epi end", 18: "pair drained", 19: "coef raw", 20: "coef N", 21: "U tiles", 22: "U penalty", 23: "S zinit", 24: "S zsum", 25: "S gram", 26: "S tri", 27: "B red own", 28: "Uc pst", 29: "F mma end", 30: "F epi end", 31: "F side end"}
for it in range(50):
    geig.geig_step_cca(s.h, X[:b], Y[:b], b, cfg.eta, cfg.gamma)
torch.cuda.synchronize()
buf = torch.zeros(64 * 1024, dtype=torch.int64, device=dev)
buf.zero_()
lib.geig_debug_set_tc_stamps(ctypes.c_void_p(buf.data_ptr()))
geig.geig_step_cca(s.h, X[b:], Y[b:], b, cfg.eta, cfg.gamma)
lib.geig_debug_set_tc_stamps(None)
geig.geig_step_cca(s.h, X[:b], Y[:b], b, cfg.eta, cfg.gamma)
torch.cuda.synchronize()
t = buf.view(-1, 64).cpu()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min().item()
print(f"{t.shape[0]} CTAs; globaltimer us from first CTA start (min / median / max) | clock64 us since slot 0 (median)")
for j, nm in names.items():
    col = ((t[:, j] - t0).double() / 1e3).tolist()
    ck = ((t[:, 32 + j] - t[:, 32]).double() / MHZ).tolist() if j != 15 else [0]
    print(f"  {j:2d} {nm:12s} {min(col):7.2f} {statistics.median(col):7.2f} {max(col):7.2f} | {statistics.median(ck):7.2f}")
order = [0, 1, 2, 3, 23, 24, 25, 26, 4, 5, 17, 6, 7, 8, 27, 28, 9, 10, 11, 12, 13, 21, 22, 14]
prev = None
out = []
for j in order:
    col = t[:, 32 + j]
    if (col == 0).all():
        continue
    med = statistics.median(((col - t[:, 32]).double() / MHZ).tolist())
    if prev is not None:
        out.append(f"{names.get(j, j)}:{med - prev:.2f}")
    prev = med
print("phase durations (clock64 us, medians):", " ".join(out), f"| total {prev:.2f}")
dg = (t[:, 14] - t[:, 0]).double()
dc = (t[:, 46] - t[:, 32]).double()
print("effective SM clock over the kernel (clock64 / globaltimer): median %.0f MHz" % statistics.median((dc / dg * 1e3).tolist()))
# stragglers: the CTAs that reach a stamp last (CTA id: us after the median)
ids = torch.nonzero(buf.view(-1, 64)[:, 0].cpu() > 0).flatten().tolist()
for j in (2, 30, 3, 24, 25, 4, 5, 17, 18, 7, 8, 21, 22, 14):
    col = ((t[:, j] - t0).double() / 1e3)
    med = col.median().item()
    top = torch.argsort(col, descending=True)[:8].tolist()
    print(f"late at {names[j]:12s} (median {med:6.2f}):", " ".join(f"{ids[i]}:+{col[i].item() - med:.2f}" for i in top))
