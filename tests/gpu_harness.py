"""Shared helpers for the GPU parity tests: run one gamma-EigenGame step
through the C ABI and the same step through the fp64 oracle on identical
seeded inputs."""
import numpy as np
import torch

from oracle import estimators, game
from synth import CONFIGS, cca_views, gaussian_init


def rel_err(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def random_state(k, d, seed, aux_noise=0.3):
    """A non-converged state: v from the Gaussian init, [Bv] = v + noise (so the
    aux path and the rho floor are exercised)."""
    V, _ = game.init_state(gaussian_init(k, d, seed))
    rng = np.random.default_rng(seed + 99)
    aux = V + aux_noise * rng.standard_normal(V.shape) / np.sqrt(d)
    return V, aux


def oracle_cca_step(x64, y64, V, aux, eta, gamma, rho):
    av, bv = estimators.cca_products(x64, y64, V)
    V2, aux2 = game.step_alg2(V, aux, [(av, bv)], eta, gamma, rho)
    return av, bv, V2, aux2


def gram_ref(V, aux, av, bv):
    ga = np.tril(V @ av.T)
    gc = np.tril(V @ aux.T)
    gb = np.diag(np.sum(V * bv, 1))
    return ga, gb, gc


def run_gpu_cca_step(geig, x, y, V, aux, k, dx, dy, math, eta, gamma, rho, dtype_flag, use_step=False):
    dev = "cuda:0"
    b = x.shape[0]
    s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math=math, data_dtype=dtype_flag, rho=rho, max_rows=b)
    try:
        Vd = torch.tensor(V, dtype=torch.float32, device=dev)
        Ad = torch.tensor(aux, dtype=torch.float32, device=dev)
        s.set_state(Vd, Ad)
        xd, yd = x.to(dev).contiguous(), y.to(dev).contiguous()
        AV = torch.full((k, dx + dy), float("nan"), device=dev)
        BV = torch.full_like(AV, float("nan"))
        if use_step:
            # geig_step_cca: the fused single-launch kernel on the bf16 path
            geig.geig_step_cca(s.h, xd, yd, b, eta, gamma)
        else:
            geig.geig_products_cca(s.h, xd, yd, b, 1.0 / (b // 2), AV, BV)
            geig.geig_update(s.h, AV, BV, eta, gamma)
        V2, aux2 = s.state()
        ga, gb, gc = s.gram()
        out = dict(av=AV.double().cpu().numpy(), bv=BV.double().cpu().numpy(),
                   V=V2.double().cpu().numpy(), aux=aux2.double().cpu().numpy(),
                   ga=ga.double().cpu().numpy(), gb=gb.double().cpu().numpy(),
                   gc=gc.double().cpu().numpy(), launches=s.launches())
    finally:
        s.close()
    return out


def check_cca_step(geig, cfg_idx, rows, k=None, dx=None, dy=None, math="f32", tol=1e-4, seed=0,
                   eta=None, gamma=None, use_step=False):
    cfg = CONFIGS[cfg_idx]
    x, y = cca_views(cfg, rows, seed=seed)
    dx = dx or cfg.dx
    dy = dy or cfg.dy
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    k = k or cfg.k
    eta = cfg.eta if eta is None else eta
    gamma = cfg.gamma if gamma is None else gamma
    d = dx + dy
    V, aux = random_state(k, d, seed)
    V32 = V.astype(np.float32).astype(np.float64)
    aux32 = aux.astype(np.float32).astype(np.float64)
    dtype_flag = 1 if x.dtype == torch.bfloat16 else 0
    got = run_gpu_cca_step(geig, x, y, V32, aux32, k, dx, dy, math, eta, gamma, cfg.rho, dtype_flag,
                           use_step=use_step)
    x64, y64 = x.double().numpy(), y.double().numpy()
    av, bv, V2, aux2 = oracle_cca_step(x64, y64, V32, aux32, eta, gamma, cfg.rho)
    ga, gb, gc = gram_ref(V32, aux32, av, bv)
    errs = dict(ga=rel_err(got["ga"], ga), gb=rel_err(got["gb"], gb), gc=rel_err(got["gc"], gc),
                step=rel_err(got["V"] - V32, V2 - V32), aux=rel_err(got["aux"], aux2),
                sphere=float(np.max(np.abs(np.linalg.norm(got["V"], axis=1) - 1))))
    if not use_step:
        errs["av"] = rel_err(got["av"], av)
        errs["bv"] = rel_err(got["bv"], bv)
    return errs, got
