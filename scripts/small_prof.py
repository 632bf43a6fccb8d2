"""Per-phase cycles of the one-CTA small step kernel (developer tool):
python scripts/small_prof.py [CFG] [STEPS] — config 1 by default, one
geig_run_cca launch of STEPS distinct batches, clock64 cycles per step of
each phase (stage wait, forward, backward, combine, Gram, coefficients,
update) and the CUDA-event time per step."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import build
build.build()
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
CL = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # GEIG_OPT_SMALL_CLUSTER (0 auto)
dev = "cuda:0"
b = cfg.batch
P = 16
X, Y = cca_views(cfg, P * b, seed=5, device=dev)
Xs = [X[i * b:(i + 1) * b].contiguous() for i in range(P)]
Ys = [Y[i * b:(i + 1) * b].contiguous() for i in range(P)]
s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math="f32", rho=cfg.rho, max_rows=b)
geig.geig_set_option(s.h, geig.GEIG_OPT_SMALL_CLUSTER, CL)
s.init_state(torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev))
args = geig.cca_batches([Xs[i % P] for i in range(T)], [Ys[i % P] for i in range(T)])
for _ in range(3):
    geig.geig_run_cca(s.h, None, None, b, cfg.eta, cfg.gamma, batches=args)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
geig.geig_run_cca(s.h, None, None, b, cfg.eta, cfg.gamma, batches=args)
e1.record()
torch.cuda.synchronize()
print(f"config {cfg.name} cluster option {CL}: {e0.elapsed_time(e1) * 1e3 / T:.2f} us/step (events, {T} steps, one launch)")
buf = torch.zeros(64, dtype=torch.int64, device=dev)
geig._lib.geig_debug_set_tc_stamps.argtypes = [ctypes.c_void_p]
geig._lib.geig_debug_set_tc_stamps(ctypes.c_void_p(buf.data_ptr()))
geig.geig_run_cca(s.h, None, None, b, cfg.eta, cfg.gamma, batches=args)
torch.cuda.synchronize()
geig._lib.geig_debug_set_tc_stamps(None)
c = buf[:8].tolist()
names = ["stage wait", "forward", "backward", "combine", "gram", "coef", "update", "tail"]
print("cycles per step:", {n: round(v / T) for n, v in zip(names, c)}, "total", round(sum(c) / T))
