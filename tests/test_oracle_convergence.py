"""Theorem-level pins: the oracle's iteration converges to the exact
generalized eigenvectors (Theorem 1) and its stochastic update
is unbiased (Appendix C)."""
import numpy as np

from oracle import estimators, game, linalg, metrics
from synth import CONFIGS, cca_views, dense_gep_small, gaussian_init


def test_config0_converges_to_exact_solution():
    """Config 0 (d=16, k=4, rho=0.05, 2000 steps, fp64): Alg. 2 with exact
    A, B reaches every generalized eigenvector within 1e-3 rad and the
    Appendix A subspace error is ~0; also Alg. 1."""
    cfg = CONFIGS[0]
    a, b = dense_gep_small(0)
    w, Vt = linalg.generalized_eigh(a, b, cfg.k)
    assert np.all(w > 0) and np.all(np.diff(w) < 0)
    V, aux = game.init_state(gaussian_init(cfg.k, cfg.d, 0))
    V1 = V.copy()
    for _ in range(cfg.steps):
        av, bv = estimators.dense_products(a, b, V)
        V, aux = game.step_alg2(V, aux, [(av, bv)], cfg.eta, cfg.gamma, cfg.rho)
    assert np.all(metrics.per_vector_angles(V, Vt) < 1e-3)
    assert metrics.subspace_error(V, a, b) < 1e-6
    # B-orthonormality of the converged y_hat = v / sqrt(<v,[Bv]>)
    y = V / np.sqrt(np.sum(V * aux, 1))[:, None]
    g = y @ b @ y.T
    assert np.allclose(g, np.eye(cfg.k), atol=1e-4)
    for _ in range(cfg.steps):
        V1 = game.step_alg1(V1, a, b, cfg.eta)
    assert np.all(metrics.per_vector_angles(V1, Vt) < 1e-3)


def _direction_minibatch_parent(i, V, AUX, AV, BV, rho):
    """NEGATIVE CONTROL (not the paper's rule): Alg. 2's direction with the
    parents' minibatch products B_t v_j in place of the auxiliary variable
    [Bv]_j in [By]_j — the biased estimator that PAPER.md:991 introduces the
    auxiliary variable to avoid ("This effectively replaces B y_j with a
    non-random variable, avoiding the bias dilemma")."""
    vi = V[i]
    avi, bvi = AV[i], BV[i]
    out = (vi @ bvi) * avi - (vi @ avi) * bvi
    for j in range(i):
        den = game.clip_denominator(V[j], AUX[j], rho)
        a_yj, byj = AV[j] / den, BV[j] / den
        out = out - (vi @ a_yj) * ((vi @ bvi) * byj - (vi @ byj) * bvi)
    return out


def test_stochastic_update_unbiased_monte_carlo():
    """Appendix C and PAPER.md:989-991: freeze a state with a
    non-random aux [Bv]_j = B v_j; the mean of Alg. 2's stochastic direction
    over independent minibatches equals the full-batch direction (within 4.5
    standard errors componentwise).  Positive control of the test's power:
    the same draws through the estimator that uses the minibatch B_t v_j in
    place of [Bv]_j (the bias the auxiliary variable exists to avoid) must
    sit more than 8 standard errors away.  Minibatches of 4 rows (h = 2: A_t
    and B_t from independent pairs of rows) make that bias large."""
    cfg = CONFIGS[1]
    x, y = cca_views(cfg, 4096, seed=1)
    x, y = x.double().numpy()[:, :6], y.double().numpy()[:, :6]
    a, b = estimators.cca_matrices(x, y)
    rng = np.random.default_rng(2)
    V, _ = game.init_state(rng.standard_normal((3, 12)))
    aux = (b @ V.T).T
    av, bv = estimators.dense_products(a, b, V)
    full = np.array([game.direction_alg2(i, V, aux, av, bv, 1e-3) for i in range(3)])
    paper, biased = [], []
    for _ in range(40000):
        idx = rng.choice(4096, size=4, replace=False)
        sav, sbv = estimators.cca_products(x[idx], y[idx], V)
        paper.append([game.direction_alg2(i, V, aux, sav, sbv, 1e-3) for i in range(3)])
        biased.append([_direction_minibatch_parent(i, V, aux, sav, sbv, 1e-3) for i in range(3)])
    z = {}
    for name, d in (("paper", np.array(paper)), ("biased", np.array(biased))):
        se = d.std(0) / np.sqrt(len(d))
        z[name] = np.abs(d.mean(0) - full) / (se + 1e-300)
    assert np.all(z["paper"] <= 4.5), z["paper"].max()
    # player 0 has no parents (both forms agree); the bias shows on the children
    assert z["biased"][1:].max() > 8.0, z["biased"].max()


def test_stochastic_cca_converges_small():
    """Alg. 2 on minibatches of a config-1-shaped problem (reduced d) reaches
    the exact top-k CCA subspace of the pool (Appendix A subspace error) and
    captures the top-k correlations (the top eigengap here is only 0.035, so
    per-vector angles are checked in the deterministic test instead)."""
    cfg = CONFIGS[1]
    n, dv, k = 20000, 8, 3
    x, y = cca_views(cfg, n, seed=4)
    x, y = x.double().numpy()[:, :dv], y.double().numpy()[:, :dv]
    a, b = estimators.cca_matrices(x, y)
    w, Vt = linalg.generalized_eigh(a, b, k)
    V, aux = game.init_state(gaussian_init(k, 2 * dv, 4))
    rng = np.random.default_rng(5)
    for t in range(3000):
        idx = rng.choice(n, size=256, replace=False)
        av, bv = estimators.cca_products(x[idx], y[idx], V)
        eta = 1.0 / (1 + t / 300)
        V, aux = game.step_alg2(V, aux, [(av, bv)], eta, 0.5, cfg.rho)
    assert metrics.subspace_error(V, a, b) < 2e-2
    # Fig. comparison metric: proportion of correlations captured
    lam_hat = [game.rayleigh(v, a, b) for v in V]
    assert np.sum(lam_hat) / np.sum(w) > 0.98
