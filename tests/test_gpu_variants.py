"""GPU parity of the update variants (next rows of the scope table):
Alg. 3, "Smooth Stochastic gamma-EigenGame", and Adam
ascent on v_i (Appendix H), against the fp64 oracle over
several steps on identical seeded inputs — through the staged path (fp32),
the fused single-step kernel and the persistent multi-step launch."""
import numpy as np
import pytest
import torch

from oracle import estimators, game
from synth import CONFIGS, cca_views
from tests.gpu_harness import rel_err, random_state

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def geig():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2206_04993_b200 import build
    build.build()
    from paper_2206_04993_b200 import geig as g
    return g

CASES = [("f32", 1, 256, None, None, None),
         ("bf16x2", 3, 4096, None, None, None),
         ("bf16x2", 2, 1000, 24, 200, 136)]


def _batches(cfg_idx, rows, dx, dy, T, seed):
    cfg = CONFIGS[cfg_idx]
    x, y = cca_views(cfg, T * rows, seed=seed)
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    return [(x[t * rows:(t + 1) * rows], y[t * rows:(t + 1) * rows]) for t in range(T)]


def _run_gpu(geig, cfg, math, batches, k, dx, dy, V, aux, eta, gamma, setup, multi):
    dev = "cuda:0"
    rows = batches[0][0].shape[0]
    flag = 1 if batches[0][0].dtype == torch.bfloat16 else 0
    s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math=math, data_dtype=flag, rho=cfg.rho, max_rows=rows)
    try:
        s.set_state(torch.tensor(V, dtype=torch.float32, device=dev),
                    torch.tensor(aux, dtype=torch.float32, device=dev))
        setup(s)
        Xd = [b_[0].to(dev).contiguous() for b_ in batches]
        Yd = [b_[1].to(dev).contiguous() for b_ in batches]
        if multi:
            geig.geig_run_cca(s.h, Xd, Yd, rows, eta, gamma)
        else:
            for xd, yd in zip(Xd, Yd):
                geig.geig_step_cca(s.h, xd, yd, rows, eta, gamma)
        Vg, Ag = s.state()
        out = {"V": Vg.double().cpu().numpy(), "aux": Ag.double().cpu().numpy()}
        if getattr(s, "_smooth", False):
            z = torch.empty(k, device=dev)
            geig.geig_smooth_state(s.h, None, z)
            geig.geig_sync(s.h)
            out["z"] = z.double().cpu().numpy()
    finally:
        s.close()
    return out


def _setup_case(cfg_idx, k, dx, dy, seed):
    cfg = CONFIGS[cfg_idx]
    k = k or cfg.k
    dx, dy = dx or cfg.dx, dy or cfg.dy
    V, aux = random_state(k, dx + dy, seed)
    return cfg, k, dx, dy, V.astype(np.float32).astype(np.float64), aux.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("math,cfg_idx,rows,k,dx,dy", CASES)
def test_smooth_alg3_matches_oracle(geig, math, cfg_idx, rows, k, dx, dy):
    """T steps of Alg. 3 (sigmoid-parameterised denominators, z ascent) from
    a random non-converged state and random z: V, [Bv] and z match the
    oracle's step_alg3."""
    T = 3
    cfg, k, dx, dy, V, aux = _setup_case(cfg_idx, k, dx, dy, 5)
    nu = 20.0
    z0 = np.random.default_rng(6).standard_normal(k).astype(np.float32).astype(np.float64)
    batches = _batches(cfg_idx, rows, dx, dy, T, 7)

    def setup(s):
        geig.geig_set_smooth(s.h, nu)
        geig.geig_smooth_state(s.h, torch.tensor(z0, dtype=torch.float32, device="cuda:0"), None)
        s._smooth = True

    got = _run_gpu(geig, cfg, math, batches, k, dx, dy, V, aux, cfg.eta, cfg.gamma, setup, multi=math != "f32")
    Vo, Ao, Zo = V, aux, z0
    for xb, yb in batches:
        av, bv = estimators.cca_products(xb.double().numpy(), yb.double().numpy(), Vo)
        Vo, Ao, Zo = game.step_alg3(Vo, Ao, Zo, [(av, bv)], cfg.eta, cfg.gamma, cfg.rho, nu)
    tol = 1e-3
    assert rel_err(got["V"] - V, Vo - V) < tol
    assert rel_err(got["aux"], Ao) < tol
    assert rel_err(got["z"] - z0, Zo - z0) < tol


@pytest.mark.parametrize("math,cfg_idx,rows,k,dx,dy", CASES)
def test_adam_matches_oracle(geig, math, cfg_idx, rows, k, dx, dy):
    """T steps with Adam ascent on v_i (fresh moments, bias corrections of
    steps 1..T): V and [Bv] match the oracle's step_alg2_adam.  eps = 1e-3
    keeps Adam's per-coordinate normalisation away from the sign flips of
    near-zero gradient coordinates, which would amplify rounding."""
    T = 3
    cfg, k, dx, dy, V, aux = _setup_case(cfg_idx, k, dx, dy, 8)
    b1, b2, eps, lr = 0.9, 0.999, 1e-3, 1e-3
    batches = _batches(cfg_idx, rows, dx, dy, T, 9)

    def setup(s):
        geig.geig_set_adam(s.h, b1, b2, eps)

    got = _run_gpu(geig, cfg, math, batches, k, dx, dy, V, aux, lr, cfg.gamma, setup, multi=math != "f32")
    Vo, Ao = V, aux
    Mo, So = np.zeros_like(V), np.zeros_like(V)
    for t, (xb, yb) in enumerate(batches, start=1):
        av, bv = estimators.cca_products(xb.double().numpy(), yb.double().numpy(), Vo)
        Vo, Ao, Mo, So = game.step_alg2_adam(Vo, Ao, Mo, So, t, [(av, bv)], lr, cfg.gamma, cfg.rho, b1, b2, eps)
    tol = 1e-3
    assert rel_err(got["V"] - V, Vo - V) < tol
    assert rel_err(got["aux"], Ao) < tol


def test_variants_single_and_multi_step_launches_agree(geig):
    """Alg. 3 + Adam together: T geig_step_cca launches and one geig_run_cca
    launch of T steps (z double buffer and Adam step count advanced inside the
    kernel) leave bit-identical states."""
    T = 4
    cfg, k, dx, dy, V, aux = _setup_case(3, None, 2048, 1024, 10)
    batches = _batches(3, 1024, dx, dy, T, 11)

    def setup(s):
        geig.geig_set_smooth(s.h, 20.0)
        geig.geig_set_adam(s.h, 0.9, 0.999, 1e-3)
        s._smooth = True

    a = _run_gpu(geig, cfg, "bf16x2", batches, k, dx, dy, V, aux, 1e-3, cfg.gamma, setup, multi=True)
    b = _run_gpu(geig, cfg, "bf16x2", batches, k, dx, dy, V, aux, 1e-3, cfg.gamma, setup, multi=False)
    for key in ("V", "aux", "z"):
        assert np.array_equal(a[key], b[key]), key


def test_variant_errors_are_loud(geig):
    s = geig.Solver(geig.GEIG_CCA, 64, 64, 8, math="f32", rho=0.1, max_rows=64)
    try:
        with pytest.raises(geig.GeigError):
            geig.geig_set_smooth(s.h, 0.05)          # nu <= rho
        with pytest.raises(geig.GeigError):
            geig.geig_smooth_state(s.h, None, torch.empty(8, device="cuda:0"))   # Alg. 3 off
        with pytest.raises(geig.GeigError):
            geig.geig_set_adam(s.h, 1.5, 0.999, 1e-8)
    finally:
        s.close()
