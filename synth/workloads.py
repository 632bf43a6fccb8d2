"""Workload recipes of BASELINE.json `configs` (seeded, synthetic).

Every function here only DRAWS inputs: problem matrices (configs 0 and 4),
paired CCA views (configs 1-3) and the raw Gaussian draws of Alg. 1/2 line 2
("v_i ~ N(0_d, I_d)"; the division by the norm belongs to the method and is
done by each implementation itself).  Torch is used so that the large
configs can be synthesised directly in HBM; with device="cpu" the same code
feeds the fp64 oracle.

Centering: PAPER.md §1 ("we typically assume the data has mean zero") — the
views are centred with the column mean of the generated pool before they are
cast to their storage dtype.  That is data preparation, not part of the
update rule.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass(frozen=True)
class WorkloadConfig:
    index: int
    name: str
    problem: str            # "dense" | "cca"
    dx: int                 # dense: d ; cca: view-x dim
    dy: int                 # dense: 0 ; cca: view-y dim
    k: int
    batch: int              # rows per step (cca) ; 0 for full-batch dense
    n: int                  # dataset size quoted by BASELINE.json (cca)
    dtype: str              # storage dtype of the data: "f64" | "f32" | "bf16"
    rho: float
    eta: float
    gamma: float
    steps: int = 0
    latent: int = 0
    view_kind: str = ""     # "gauss" | "image" | "activation"
    recipe: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def d(self) -> int:
        return self.dx + self.dy


# The five BASELINE.json configs.  eta/gamma/rho where BASELINE.json is silent
# are our choices (DESIGN.md §"Readings"): rho lower-bounds sigma_min(B) per
# Alg. 2's "scalar rho lower bounding sigma_min(B)".
CONFIGS = {
    0: WorkloadConfig(0, "dense_d16_k4", "dense", 16, 0, 4, 0, 0, "f64",
                      rho=0.05, eta=0.05, gamma=1.0, steps=2000,
                      recipe="A=Q diag(lam) Q^T, lam~U[-5,5]; B=R diag(mu) R^T, "
                             "mu log-uniform [0.1,10]; Q,R Haar"),
    1: WorkloadConfig(1, "cca_gauss_d64_k8", "cca", 64, 64, 8, 256, 100_000, "f32",
                      rho=0.1, eta=0.1, gamma=1.0, latent=8, view_kind="gauss",
                      recipe="z~N(0,I_8); X=zW_x+0.5N(0,I); Y=zW_y+0.5N(0,I); W~N(0,1/8)"),
    2: WorkloadConfig(2, "cca_image_d784_k16", "cca", 784, 784, 16, 1024, 1_000_000, "bf16",
                      rho=1e-3, eta=0.1, gamma=1.0, latent=32, view_kind="image",
                      recipe="clip(sigmoid(zW+0.3 noise),0,1), latent 32"),
    3: WorkloadConfig(3, "cca_activation_d8192_k64", "cca", 8192, 8192, 64, 4096, 10_000_000, "bf16",
                      rho=1e-2, eta=1e-4, gamma=0.5, latent=256, view_kind="activation",
                      recipe="ReLU(zW + t_3 noise), latent 256"),
    4: WorkloadConfig(4, "dense_d16384_k128", "dense", 16384, 0, 128, 0, 0, "f32",
                      rho=5e-4, eta=0.05, gamma=1.0,
                      recipe="A=Q diag(lam) Q^T, lam_i = i^-1; B=R diag(mu) R^T, cond 1e3"),
}


def _np_rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(seed))


def haar_orthogonal(n: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-distributed orthogonal matrix (QR of a Gaussian with the sign of
    R's diagonal folded into Q)."""
    g = rng.standard_normal((n, n))
    q, r = np.linalg.qr(g)
    return q * np.sign(np.diag(r))[None, :]


def dense_gep_small(seed: int = 0, d: int = 16):
    """Config 0: A = Q diag(lam) Q^T (lam ~ U[-5,5]), B = R diag(mu) R^T
    (mu log-uniform in [0.1, 10]); float64 numpy."""
    rng = _np_rng(seed)
    lam = rng.uniform(-5.0, 5.0, size=d)
    mu = np.exp(rng.uniform(math.log(0.1), math.log(10.0), size=d))
    q = haar_orthogonal(d, rng)
    r = haar_orthogonal(d, rng)
    a = (q * lam[None, :]) @ q.T
    b = (r * mu[None, :]) @ r.T
    a = 0.5 * (a + a.T)
    b = 0.5 * (b + b.T)
    return a, b


def dense_gep_large(d: int, seed: int = 0, device="cpu", cond: float = 1e3,
                    dtype=torch.float32):
    """Config 4 recipe at any size: A = Q diag(i^-1) Q^T, B = R diag(mu) R^T
    with mu geometrically spaced so that cond(B) = `cond`.  Returns torch
    tensors (d x d, row-major) on `device`."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def orth():
        m = torch.randn(d, d, generator=g, device=device, dtype=torch.float32)
        q, r = torch.linalg.qr(m)
        return q * torch.sign(torch.diagonal(r))[None, :]

    lam = 1.0 / torch.arange(1, d + 1, device=device, dtype=torch.float32)
    u = torch.linspace(0.0, 1.0, d, device=device, dtype=torch.float32)
    mu = torch.pow(torch.tensor(cond, device=device), -u)      # in [1/cond, 1]
    q = orth()
    a = (q * lam[None, :]) @ q.T
    r = orth()
    b = (r * mu[None, :]) @ r.T
    a = 0.5 * (a + a.T)
    b = 0.5 * (b + b.T)
    return a.to(dtype).contiguous(), b.to(dtype).contiguous()


def _student_t3(shape, g, device):
    # t_nu = N / sqrt(chi2_nu / nu), nu = 3
    n = torch.randn(shape, generator=g, device=device)
    c = torch.randn((3,) + tuple(shape), generator=g, device=device).pow(2).sum(0)
    return n / torch.sqrt(c / 3.0)


def cca_views(cfg: WorkloadConfig, rows: int, seed: int = 0, device="cpu",
              dtype: torch.dtype | None = None, center: bool = True,
              row_block: int = 8192):
    """Paired views (X, Y), each `rows` x d_view, row-major, drawn from the
    latent model of `cfg` (configs 1-3).  The mixing matrices W_x, W_y are a
    function of `seed` only, so pools drawn with different `rows` share the
    same population.  Returns torch tensors of `dtype` (default: the config's
    storage dtype) on `device`."""
    assert cfg.problem == "cca"
    if dtype is None:
        dtype = {"f32": torch.float32, "bf16": torch.bfloat16, "f64": torch.float64}[cfg.dtype]
    gw = torch.Generator(device=device)
    gw.manual_seed(1_000_003 * seed + 17)
    lat = cfg.latent
    wx = torch.randn(lat, cfg.dx, generator=gw, device=device) / math.sqrt(lat)
    wy = torch.randn(lat, cfg.dy, generator=gw, device=device) / math.sqrt(lat)
    g = torch.Generator(device=device)
    g.manual_seed(7_919 * seed + 101)
    xs, ys = [], []
    for r0 in range(0, rows, row_block):
        r = min(row_block, rows - r0)
        z = torch.randn(r, lat, generator=g, device=device)
        if cfg.view_kind == "gauss":
            x = z @ wx + 0.5 * torch.randn(r, cfg.dx, generator=g, device=device)
            y = z @ wy + 0.5 * torch.randn(r, cfg.dy, generator=g, device=device)
        elif cfg.view_kind == "image":
            x = torch.sigmoid(z @ wx + 0.3 * torch.randn(r, cfg.dx, generator=g, device=device)).clamp(0, 1)
            y = torch.sigmoid(z @ wy + 0.3 * torch.randn(r, cfg.dy, generator=g, device=device)).clamp(0, 1)
        elif cfg.view_kind == "activation":
            x = torch.relu(z @ wx + _student_t3((r, cfg.dx), g, device))
            y = torch.relu(z @ wy + _student_t3((r, cfg.dy), g, device))
        else:
            raise ValueError(cfg.view_kind)
        xs.append(x)
        ys.append(y)
    x = torch.cat(xs, 0)
    y = torch.cat(ys, 0)
    if center:
        x = x - x.mean(0, keepdim=True)
        y = y - y.mean(0, keepdim=True)
    return x.to(dtype).contiguous(), y.to(dtype).contiguous()


def gaussian_init(k: int, d: int, seed: int = 0) -> np.ndarray:
    """Raw draws v_i ~ N(0_d, I_d) (Alg. 1/2 line 2), shape k x d (player-major),
    float64.  The normalisation v_i / ||v_i|| is done by the consumer."""
    return _np_rng(10_007 * seed + 3).standard_normal((k, d))


def appendix_b_example():
    """The 2x2 (A, B) pair printed in PAPER.md Appendix B ("As an example
    consider setting"), used for the Fig. 1 utility illustration."""
    a = np.array([[0.77759061, 0.26842584], [0.26842584, 0.87788983]])
    b = np.array([[0.2325605, 0.06042127], [0.06042127, 0.03241424]])
    return a, b


def planted_cca_views(n: int, dx: int, dy: int, corrs, seed: int = 0, device="cpu",
                      dtype: torch.dtype = torch.float32):
    """Paired views with planted canonical correlations `corrs` and identity
    population covariances: coordinates i < r of x are z_i, of y are
    c_i z_i + sqrt(1-c_i^2) e_i, the rest independent N(0,1); each view is then
    rotated by a seeded Haar matrix.  Population generalized eigenvalues of
    the CCA GEP are +-c_i (and 0).  Used by convergence tests."""
    r = len(corrs)
    rng = _np_rng(31 * seed + 5)
    qx = torch.tensor(haar_orthogonal(dx, rng), dtype=torch.float32, device=device)
    qy = torch.tensor(haar_orthogonal(dy, rng), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(97 * seed + 13)
    z = torch.randn(n, r, generator=g, device=device)
    x = torch.randn(n, dx, generator=g, device=device)
    y = torch.randn(n, dy, generator=g, device=device)
    c = torch.tensor(list(corrs), dtype=torch.float32, device=device)
    x[:, :r] = z
    y[:, :r] = c * z + torch.sqrt(1 - c * c) * y[:, :r]
    return (x @ qx).to(dtype).contiguous(), (y @ qy).to(dtype).contiguous()
