"""Pins for oracle/linalg.py (exact generalized eigensolve) against library
routines, closed forms, brute force and the paper's Appendix B example."""
import os

import numpy as np
import pytest
import scipy.linalg as sl

from oracle import linalg, metrics
from synth import appendix_b_example, dense_gep_small

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "appendix_b_2x2.txt")


def _golden():
    out = {}
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        key, *vals = line.split()
        out[key] = np.array([float(v) for v in vals])
    return out


def _rand_spd(n, rng, cond=10.0):
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    mu = np.geomspace(1.0, 1.0 / cond, n)
    return (q * mu) @ q.T


def test_cholesky_matches_definition_and_library():
    rng = np.random.default_rng(1)
    b = _rand_spd(9, rng, 100.0)
    l = linalg.cholesky(b)
    assert np.allclose(np.triu(l, 1), 0.0)
    assert np.allclose(l @ l.T, b, atol=1e-13)
    assert np.allclose(l, np.linalg.cholesky(b), atol=1e-12)
    with pytest.raises(ValueError):
        linalg.cholesky(-b)


def test_triangular_solves_match_library():
    rng = np.random.default_rng(2)
    l = np.tril(rng.standard_normal((7, 7))) + 5 * np.eye(7)
    r = rng.standard_normal((7, 3))
    assert np.allclose(linalg.solve_lower(l, r), sl.solve_triangular(l, r, lower=True))
    assert np.allclose(linalg.solve_upper(l.T, r), sl.solve_triangular(l.T, r, lower=False))


@pytest.mark.parametrize("n", [1, 2, 5, 16, 33])
def test_jacobi_matches_numpy_eigh(n):
    rng = np.random.default_rng(n)
    s = rng.standard_normal((n, n))
    s = s + s.T
    w, v = linalg.sym_eigh(s, "jacobi")
    w_ref = np.sort(np.linalg.eigvalsh(s))[::-1]
    assert np.allclose(w, w_ref, atol=1e-11 * max(1, np.abs(w_ref).max()))
    assert np.allclose(v.T @ v, np.eye(n), atol=1e-12)
    assert np.allclose(s @ v, v * w[None, :], atol=1e-10)


def test_generalized_eigh_residual_borth_and_scipy():
    a, b = dense_gep_small(0)
    w, V = linalg.generalized_eigh(a, b)
    ref = sl.eigh(a, b, eigvals_only=True)[::-1]
    assert np.allclose(w, ref, atol=1e-10)
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    for lam, v in zip(w, V):
        assert np.linalg.norm(a @ v - lam * b @ v) <= 1e-9 * (na + abs(lam) * nb)
        assert abs(np.linalg.norm(v) - 1) < 1e-12
    assert metrics.b_orthogonality_defect(V, b) < 1e-10


def test_generalized_eigh_matches_eigh_path_large():
    rng = np.random.default_rng(3)
    n = 300
    a = rng.standard_normal((n, n))
    a = a + a.T
    b = _rand_spd(n, rng, 50.0)
    w, V = linalg.generalized_eigh(a, b, 5)
    ref_w, ref_v = sl.eigh(a, b)
    assert np.allclose(w, ref_w[::-1][:5], atol=1e-8)
    ref_v = ref_v[:, ::-1][:, :5].T
    ref_v /= np.linalg.norm(ref_v, axis=1, keepdims=True)
    assert np.all(metrics.per_vector_angles(V, ref_v) < 1e-8)


def test_appendix_b_example_against_paper_and_closed_form():
    """PAPER.md:1246 matrices; Fig. 1 caption: eigenvectors 71 deg apart in the
    Euclidean metric, 90 deg in the B metric.  Eigenvalues pinned by the
    closed-form roots of det(A - lam B) = 0 (2x2 quadratic)."""
    g = _golden()
    a, b = appendix_b_example()
    assert np.allclose(a.ravel(), g["A"]) and np.allclose(b.ravel(), g["B"])
    w, V = linalg.generalized_eigh(a, b)
    # det(A - lam B) = c2 lam^2 + c1 lam + c0
    c2 = b[0, 0] * b[1, 1] - b[0, 1] ** 2
    c1 = -(a[0, 0] * b[1, 1] + a[1, 1] * b[0, 0] - 2 * a[0, 1] * b[0, 1])
    c0 = a[0, 0] * a[1, 1] - a[0, 1] ** 2
    disc = np.sqrt(c1 * c1 - 4 * c2 * c0)
    roots = sorted([(-c1 + disc) / (2 * c2), (-c1 - disc) / (2 * c2)], reverse=True)
    assert np.allclose(w, roots, rtol=1e-10)
    ang = np.degrees(np.arccos(abs(V[0] @ V[1])))
    assert abs(ang - g["euclid_angle_deg"][0]) <= g["angle_tol_deg"][0]
    assert abs(np.degrees(metrics.angle_under_metric(V[0], V[1], b)) - g["b_angle_deg"][0]) < 1e-6


def test_brute_force_top_eigenpair_2d():
    """Brute force: maximise the generalized Rayleigh quotient over a fine
    grid of the unit circle (d = 2)."""
    a, b = appendix_b_example()
    th = np.linspace(0, np.pi, 200001)
    vs = np.stack([np.cos(th), np.sin(th)], 1)
    rq = np.einsum("ni,ij,nj->n", vs, a, vs) / np.einsum("ni,ij,nj->n", vs, b, vs)
    w, V = linalg.generalized_eigh(a, b)
    assert abs(rq.max() - w[0]) < 1e-6 * w[0]
    best = vs[np.argmax(rq)]
    assert np.degrees(metrics.per_vector_angles(best[None], V[:1])[0]) < 0.01


def test_power_iteration_top_pair_d16():
    """Independent second path (brute force at d <= 16): power iteration on
    B^{-1}(A + sI) with a shift making it positive, for config 0."""
    a, b = dense_gep_small(0)
    w, V = linalg.generalized_eigh(a, b, 1)
    shift = 10.0 * np.max(np.abs(np.linalg.eigvals(np.linalg.solve(b, a))))
    m = np.linalg.solve(b, a + shift * b)
    x = np.ones(16)
    for _ in range(20000):
        x = m @ x
        x /= np.linalg.norm(x)
    lam = (x @ a @ x) / (x @ b @ x)
    assert abs(lam - w[0]) < 1e-8 * abs(w[0])
    assert metrics.per_vector_angles(x[None], V)[0] < 1e-6


def test_sqrtm_spd():
    rng = np.random.default_rng(5)
    b = _rand_spd(8, rng, 1e3)
    h = linalg.sqrtm_spd(b)
    assert np.allclose(h @ h, b, atol=1e-12)
    assert np.allclose(linalg.sqrtm_spd(b, inverse=True) @ h, np.eye(8), atol=1e-9)
