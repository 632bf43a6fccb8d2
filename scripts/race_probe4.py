"""Developer (dev-knob build): NaN tracing of the multi-step fused launch.
Stamp buffer set: after the G x 64 stamp slots, 8 per CTA record (step + 1)
of the first non-finite value: 0 backward epilogue (AV/BV), 1 forward
epilogue (z partials), 2 phase S (summed z), 3 phase U v'', 4 phase U
direction, 5 phase U BV / V tiles (7: current step)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import geig
from synth import CONFIGS, cca_views, gaussian_init
cfg = CONFIGS[1]
n, steps, C, R = (int(a) for a in sys.argv[1:5])
dx, k, eta = 64, 8, 0.0086
x, y = cca_views(cfg, n, seed=3)
x, y = x[:, :dx].to(torch.bfloat16).contiguous().cuda(), y[:, :dx].to(torch.bfloat16).contiguous().cuda()
lib = geig._lib
lib.geig_debug_set_tc_stamps.argtypes = [ctypes.c_void_p]
buf = torch.zeros(64 * 1024, dtype=torch.int64, device="cuda:0")
names = {56: "B epi AV/BV", 57: "F epi z", 58: "S z", 59: "U v''", 60: "U AV tile", 61: "U BV/V tile"}
for r in range(R):
    s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math="bf16x2", data_dtype=1, rho=cfg.rho, max_rows=n)
    s.init_state(torch.tensor(gaussian_init(k, 2 * dx, 0), dtype=torch.float32, device="cuda:0"))
    for c in range(steps // C):
        buf.zero_()
        lib.geig_debug_set_tc_stamps(ctypes.c_void_p(buf.data_ptr()))
        geig.geig_run_cca(s.h, [x] * C, [y] * C, n, eta, 1.0)
        lib.geig_debug_set_tc_stamps(None)
        V, A = s.state()
        G = 4
        t = buf[G * 64:G * 64 + G * 8].view(G, 8)[:, 0:6].cpu()
        if t.any() or not torch.isfinite(V).all():
            rec = {names[56 + j]: sorted(set(int(v) for v in t[:, j].tolist() if v)) for j in range(6)}
            ctas = {names[56 + j]: torch.nonzero(t[:, j]).flatten().tolist()[:8] for j in range(6)}
            print(f"repeat {r} chunk {c}: V finite {bool(torch.isfinite(V).all())}; first-bad step (+1) per site {rec}; "
                  f"CTAs {ctas}", flush=True)
            break
    else:
        print(f"repeat {r}: ok", flush=True)
    s.close()
