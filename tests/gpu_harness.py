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


def row_rel_err(got, ref, base=None):
    """Per-player (row) relative error max_i ||got_i - ref_i|| / ||ref_i - base_i||
    (base = None: relative to ||ref_i||).  One player's error is not diluted
    by the other k - 1 rows as in the normwise rel_err."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = ref if base is None else ref - np.asarray(base, np.float64)
    num = np.linalg.norm(got - ref, axis=1)
    dn = np.linalg.norm(den, axis=1)
    return float(np.max(num / np.maximum(dn, 1e-300)))


def tri_row_rel_err(got, ref):
    """Per-row relative error of a lower-triangular k x k table (row i holds
    the entries j <= i; row norms over those entries)."""
    got, ref = np.tril(np.asarray(got, np.float64)), np.tril(np.asarray(ref, np.float64))
    return row_rel_err(got, ref)


def random_state(k, d, seed, aux_noise=0.3):
    """A non-converged state: v from the Gaussian init, [Bv] = v + noise
    (<v_j,[Bv]_j> ~ 1: the rho floor of Alg. 2 l.8 is NOT active; see
    floor_state for states that clip)."""
    V, _ = game.init_state(gaussian_init(k, d, seed))
    rng = np.random.default_rng(seed + 99)
    aux = V + aux_noise * rng.standard_normal(V.shape) / np.sqrt(d)
    return V, aux


def floor_state(k, d, seed, rho, aux_noise=1.0):
    """A state with the rho floor of Alg. 2 line 8 ("may
    not be positive definite, therefore, we manually clip the result to be
    greater than or equal to rho") active for several parents: player j gets
    <v_j,[Bv]_j> = t_j exactly (in fp64; far from the clip boundary in fp32)
    with t_j cycling through 1 (no clip), -0.5 (negative), 0.5 rho, 2 rho
    (just above), -0.05, 0.25 rho, 4 rho, 0 — [Bv]_j = t_j v_j plus noise
    orthogonal to v_j, so [Bv]_j != B_t v_j and the penalty's [By]_j term
    carries a component the clip does not touch."""
    V, _ = game.init_state(gaussian_init(k, d, seed))
    rng = np.random.default_rng(seed + 199)
    targets = np.array([1.0, -0.5, 0.5 * rho, 2.0 * rho, -0.05, 0.25 * rho, 4.0 * rho, 0.0])
    t = targets[np.arange(k) % len(targets)]
    n = rng.standard_normal(V.shape)
    n -= np.sum(n * V, 1, keepdims=True) * V
    n *= aux_noise / np.linalg.norm(n, axis=1, keepdims=True)       # ||noise_j|| = aux_noise
    aux = t[:, None] * V + n
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


def run_gpu_cca_step(geig, x, y, V, aux, k, dx, dy, math, eta, gamma, rho, dtype_flag, use_step=False,
                     options=None):
    dev = "cuda:0"
    b = x.shape[0]
    s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math=math, data_dtype=dtype_flag, rho=rho, max_rows=b)
    try:
        for key, val in (options or {}).items():
            geig.geig_set_option(s.h, key, val)
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
                   eta=None, gamma=None, use_step=False, state="random", rows_err=False, options=None):
    cfg = CONFIGS[cfg_idx]
    x, y = cca_views(cfg, rows, seed=seed)
    dx = dx or cfg.dx
    dy = dy or cfg.dy
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    k = k or cfg.k
    eta = cfg.eta if eta is None else eta
    gamma = cfg.gamma if gamma is None else gamma
    d = dx + dy
    V, aux = random_state(k, d, seed) if state == "random" else floor_state(k, d, seed, cfg.rho)
    V32 = V.astype(np.float32).astype(np.float64)
    aux32 = aux.astype(np.float32).astype(np.float64)
    dtype_flag = 1 if x.dtype == torch.bfloat16 else 0
    got = run_gpu_cca_step(geig, x, y, V32, aux32, k, dx, dy, math, eta, gamma, cfg.rho, dtype_flag,
                           use_step=use_step, options=options)
    x64, y64 = x.double().numpy(), y.double().numpy()
    av, bv, V2, aux2 = oracle_cca_step(x64, y64, V32, aux32, eta, gamma, cfg.rho)
    ga, gb, gc = gram_ref(V32, aux32, av, bv)
    errs = dict(ga=rel_err(got["ga"], ga), gb=rel_err(got["gb"], gb), gc=rel_err(got["gc"], gc),
                step=rel_err(got["V"] - V32, V2 - V32), aux=rel_err(got["aux"], aux2),
                sphere=float(np.max(np.abs(np.linalg.norm(got["V"], axis=1) - 1))))
    if not use_step:
        errs["av"] = rel_err(got["av"], av)
        errs["bv"] = rel_err(got["bv"], bv)
    if rows_err:
        errs.update(row_step=row_rel_err(got["V"], V2, V32), row_aux=row_rel_err(got["aux"], aux2),
                    row_ga=tri_row_rel_err(got["ga"], ga), row_gc=tri_row_rel_err(got["gc"], gc),
                    row_gb=float(np.max(np.abs(np.diag(got["gb"]) - np.diag(gb)) / np.abs(np.diag(gb)))))
        if not use_step:
            errs.update(row_av=row_rel_err(got["av"], av), row_bv=row_rel_err(got["bv"], bv))
    got["clipped"] = [j for j in range(k - 1) if float(V32[j] @ aux32[j]) < cfg.rho]
    return errs, got
