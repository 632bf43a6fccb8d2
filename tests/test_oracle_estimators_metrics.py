"""Pins for oracle/estimators.py and oracle/metrics.py."""
import numpy as np
import pytest

from oracle import estimators, linalg, metrics
from synth import CONFIGS, cca_views, dense_gep_small


def test_cca_block_structure_and_product_form():
    """A has zero diagonal blocks, B zero off-diagonal blocks;
    the product form of A_t v / B_t v equals the explicit matrices of the
    halves (reading R1: rows [0,h) -> A, [h,b) -> B)."""
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal((30, 4)), rng.standard_normal((30, 5))
    a, b = estimators.cca_matrices(x, y)
    assert np.all(a[:4, :4] == 0) and np.all(a[4:, 4:] == 0)
    assert np.all(b[:4, 4:] == 0) and np.all(b[4:, :4] == 0)
    assert np.allclose(a, a.T) and np.allclose(b, b.T)
    V = rng.standard_normal((3, 9))
    a_t, b_t = estimators.cca_minibatch_matrices(x, y)
    av, bv = estimators.cca_products(x, y, V)
    assert np.allclose(av, V @ a_t, atol=1e-12)
    assert np.allclose(bv, V @ b_t, atol=1e-12)
    a1, _ = estimators.cca_matrices(x[:15], y[:15])
    _, b2 = estimators.cca_matrices(x[15:], y[15:])
    assert np.allclose(a_t, a1) and np.allclose(b_t, b2)


def test_cca_1d_closed_form_correlation():
    """d_x = d_y = 1 with unit variances and correlation r: the generalized
    eigenvalues of the CCA GEP are +-r (closed form)."""
    r = 0.6
    rng = np.random.default_rng(1)
    n = 400_000
    z = rng.standard_normal(n)
    x = z
    y = r * z + np.sqrt(1 - r * r) * rng.standard_normal(n)
    a, b = estimators.cca_matrices(x[:, None], y[:, None])
    w, _ = linalg.generalized_eigh(a, b)
    emp_r = np.corrcoef(x, y)[0, 1]
    assert np.allclose(w, [emp_r, -emp_r], atol=1e-12)
    assert abs(emp_r - r) < 5e-3


def test_cca_identical_views_top_eigenvalue_one():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((500, 3))
    a, b = estimators.cca_matrices(x, x.copy())
    w, _ = linalg.generalized_eigh(a, b)
    assert np.isclose(w[0], 1.0, atol=1e-10)


def test_minibatch_estimates_unbiased():
    """E[A_t] = A and E[B_t] = B over random minibatches of a finite
    dataset (Appendix C unbiasedness of the estimates), 4-SE entrywise."""
    cfg = CONFIGS[1]
    x, y = cca_views(cfg, 2048, seed=3)
    x, y = x.double().numpy()[:, :6], y.double().numpy()[:, :5]
    a, b = estimators.cca_matrices(x, y)
    rng = np.random.default_rng(3)
    draws_a, draws_b = [], []
    for _ in range(3000):
        idx = rng.choice(2048, size=32, replace=False)
        at, bt = estimators.cca_minibatch_matrices(x[idx], y[idx])
        draws_a.append(at)
        draws_b.append(bt)
    for draws, ref in ((np.array(draws_a), a), (np.array(draws_b), b)):
        mean = draws.mean(0)
        se = draws.std(0) / np.sqrt(len(draws)) + 1e-15
        assert np.all(np.abs(mean - ref) <= 4.5 * se + 1e-12)


def test_subspace_error_properties():
    a, b = dense_gep_small(0)
    w, Vt = linalg.generalized_eigh(a, b, 4)
    assert abs(metrics.subspace_error(Vt, a, b)) < 1e-10
    rng = np.random.default_rng(4)
    q, _ = np.linalg.qr(rng.standard_normal((4, 4)))
    rot = q @ Vt
    rot = rot * np.sign(rng.standard_normal(4))[:, None]
    assert abs(metrics.subspace_error(rot, a, b)) < 1e-8
    # orthogonal complement in a diagonal B=I problem: error 1
    d = 8
    ad = np.diag(np.arange(d, 0, -1.0))
    bot = np.eye(d)[4:]
    assert np.isclose(metrics.subspace_error(bot, ad, np.eye(d), 4), 1.0, atol=1e-10)


def test_orth_angle_lower_bound_lemma():
    """Lemma orth_angle_change: orthonormal u, v measured in
    an SPD C with condition kappa are more than (1/8)(1+kappa)^(-5/4) apart."""
    rng = np.random.default_rng(5)
    for trial in range(300):
        d = int(rng.integers(2, 9))
        q, _ = np.linalg.qr(rng.standard_normal((d, d)))
        kappa = 10 ** rng.uniform(0, 4)
        mu = np.geomspace(1, 1 / kappa, d)
        r, _ = np.linalg.qr(rng.standard_normal((d, d)))
        c = (r * mu) @ r.T
        th = metrics.angle_under_metric(q[:, 0], q[:, 1], c)
        assert th > 0.125 * (1 + kappa) ** (-1.25)


def test_angle_blowup_upper_bound_lemma():
    """Lemma angle_blowup: eps-close vectors are at most
    4 sqrt((1+kappa) sqrt(kappa) eps + (kappa^2/4+1) eps^2) apart in the C metric."""
    rng = np.random.default_rng(6)
    for trial in range(300):
        kappa = 10 ** rng.uniform(0, 2)
        r, _ = np.linalg.qr(rng.standard_normal((2, 2)))
        c = (r * np.array([1.0, 1.0 / kappa])) @ r.T
        eps = rng.uniform(0, min(1 / kappa, 0.5))
        u = np.array([1.0, 0.0])
        v = np.array([np.sqrt(1 - eps * eps), eps])
        th = metrics.angle_under_metric(u, v, c)
        assert th <= 4 * np.sqrt((1 + kappa) * np.sqrt(kappa) * eps + (kappa ** 2 / 4 + 1) * eps ** 2) + 1e-12
