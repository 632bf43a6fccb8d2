"""Quick numerical probe of the tcgen05 products against a float64 torch
reference (developer tool; the graded parity tests are tests/test_gpu_parity.py)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_04993_b200 import build
build.build()
from paper_2206_04993_b200 import geig

def ref_cca(X, Y, V, dx):
    X, Y, V = X.double(), Y.double(), V.double()
    h = X.shape[0] // 2
    vx, vy = V[:, :dx].T, V[:, dx:].T
    x1, y1, x2, y2 = X[:h], Y[:h], X[h:2*h], Y[h:2*h]
    av = torch.cat([x1.T @ (y1 @ vy), y1.T @ (x1 @ vx)], 0) / h
    bv = torch.cat([x2.T @ (x2 @ vx), y2.T @ (y2 @ vy)], 0) / h
    return av.T, bv.T

def rel(a, b):
    return ((a.double() - b.double()).norm() / b.double().norm()).item()

def probe_cca(dx, dy, b, k, math, dt):
    torch.manual_seed(0)
    X = torch.randn(b, dx, device="cuda").to(dt)
    Y = torch.randn(b, dy, device="cuda").to(dt)
    s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math=math,
                    data_dtype=geig.GEIG_DATA_BF16 if dt == torch.bfloat16 else geig.GEIG_DATA_F32,
                    rho=0.01, max_rows=b)
    G = torch.randn(k, dx + dy, device="cuda")
    s.init_state(G)
    V, _ = s.state()
    AV = torch.empty(k, dx + dy, device="cuda"); BV = torch.empty_like(AV)
    geig.geig_products_cca(s.h, X, Y, b, 1.0 / (b // 2), AV, BV)
    torch.cuda.synchronize()
    Vq = V.to(dt).float() if dt == torch.bfloat16 else V
    ra, rb = ref_cca(X, Y, Vq, dx)
    print(f"cca {math} dx={dx} dy={dy} b={b} k={k}: AV rel {rel(AV, ra):.3e} BV rel {rel(BV, rb):.3e}", flush=True)
    s.close()

def probe_dense(d, k, math):
    torch.manual_seed(1)
    A = torch.randn(d, d, device="cuda"); A = (A + A.T) / 2
    B = torch.randn(d, d, device="cuda"); B = B @ B.T / d + torch.eye(d, device="cuda")
    s = geig.Solver(geig.GEIG_DENSE, d, 0, k, math=math, rho=0.01)
    s.init_state(torch.randn(k, d, device="cuda"))
    V, _ = s.state()
    AV = torch.empty(k, d, device="cuda"); BV = torch.empty_like(AV)
    geig.geig_products_dense(s.h, A, B, 0, d, AV, BV)
    torch.cuda.synchronize()
    print(f"dense {math} d={d} k={k}: AV rel {rel(AV, (A.double() @ V.double().T).T):.3e} "
          f"BV rel {rel(BV, (B.double() @ V.double().T).T):.3e}", flush=True)
    s.close()

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "cca"):
    probe_cca(64, 64, 256, 16, "bf16", torch.bfloat16)
    probe_cca(256, 192, 512, 16, "bf16", torch.bfloat16)
    probe_cca(784, 784, 1024, 16, "bf16", torch.bfloat16)
    probe_cca(64, 64, 256, 8, "tf32", torch.float32)
    probe_cca(8192, 8192, 4096, 64, "bf16", torch.bfloat16)
if which == "tf32":
    probe_cca(64, 64, 256, 8, "bf16", torch.bfloat16)
    probe_cca(64, 64, 256, 16, "tf32", torch.float32)
    probe_cca(256, 128, 512, 32, "tf32", torch.float32)
    probe_cca(8192, 8192, 4096, 64, "tf32", torch.float32)
if which in ("all", "dense"):
    probe_dense(256, 16, "tf32")
    probe_dense(2048, 128, "tf32")
