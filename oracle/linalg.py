"""ORACLE (test infrastructure only) — dense linear algebra for the exact
generalized eigensolve used as ground truth.

North star: "a direct generalized eigensolve (Cholesky of B plus Jacobi)".
PAPER.md:1163 (Lemma b_orth) / PAPER.md:1169 (Prop. sim_mat): the GEP
Av = lambda Bv is similar to a symmetric eigenproblem; with B = L L^T the
matrix C = L^{-1} A L^{-T} is symmetric, has the same eigenvalues, and its
eigenvectors w map back by v = L^{-T} w.  (Prop. sim_mat states the same with
B^{1/2}; any factor F with F F^T = B gives the same eigenpairs.)
"""
from __future__ import annotations

import numpy as np


def cholesky(b: np.ndarray) -> np.ndarray:
    """Textbook Cholesky–Banachiewicz: lower-triangular L with L L^T = B.
    Raises ValueError if B is not (numerically) positive definite."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    l = np.zeros_like(b)
    for i in range(n):
        for j in range(i + 1):
            s = b[i, j] - np.dot(l[i, :j], l[j, :j])
            if i == j:
                if s <= 0.0:
                    raise ValueError("matrix is not positive definite")
                l[i, i] = np.sqrt(s)
            else:
                l[i, j] = s / l[j, j]
    return l


def solve_lower(l: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """Forward substitution L X = RHS (L lower-triangular)."""
    rhs = np.array(rhs, dtype=np.float64)
    squeeze = rhs.ndim == 1
    if squeeze:
        rhs = rhs[:, None]
    n = l.shape[0]
    x = np.zeros_like(rhs)
    for i in range(n):
        x[i] = (rhs[i] - l[i, :i] @ x[:i]) / l[i, i]
    return x[:, 0] if squeeze else x


def solve_upper(u: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """Back substitution U X = RHS (U upper-triangular)."""
    rhs = np.array(rhs, dtype=np.float64)
    squeeze = rhs.ndim == 1
    if squeeze:
        rhs = rhs[:, None]
    n = u.shape[0]
    x = np.zeros_like(rhs)
    for i in range(n - 1, -1, -1):
        x[i] = (rhs[i] - u[i, i + 1:] @ x[i + 1:]) / u[i, i]
    return x[:, 0] if squeeze else x


def jacobi_eigh(s: np.ndarray, tol: float = 1e-15, max_sweeps: int = 60):
    """Cyclic Jacobi rotations for a symmetric matrix (Golub & Van Loan
    Alg. 8.5.3).  Returns (eigenvalues, eigenvectors as columns), unsorted.
    Sweeps until the off-diagonal Frobenius norm is below tol * ||S||_F."""
    a = np.array(s, dtype=np.float64)
    n = a.shape[0]
    v = np.eye(n)
    scale = max(np.linalg.norm(a), 1e-300)
    for _ in range(max_sweeps):
        off = np.sqrt(max(np.sum(a * a) - np.sum(np.diag(a) ** 2), 0.0))
        if off <= tol * scale:
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = a[p, q]
                if abs(apq) <= 1e-300:
                    continue
                tau = (a[q, q] - a[p, p]) / (2.0 * apq)
                if abs(tau) > 1e150:
                    t = 0.5 / tau
                else:
                    t = (1.0 if tau >= 0 else -1.0) / (abs(tau) + np.sqrt(1.0 + tau * tau))
                c = 1.0 / np.sqrt(1.0 + t * t)
                sn = t * c
                ap = a[:, p].copy()
                aq = a[:, q].copy()
                a[:, p] = c * ap - sn * aq
                a[:, q] = sn * ap + c * aq
                ap = a[p, :].copy()
                aq = a[q, :].copy()
                a[p, :] = c * ap - sn * aq
                a[q, :] = sn * ap + c * aq
                a[p, q] = 0.0
                a[q, p] = 0.0
                vp = v[:, p].copy()
                vq = v[:, q].copy()
                v[:, p] = c * vp - sn * vq
                v[:, q] = sn * vp + c * vq
    return np.diag(a).copy(), v


def sym_eigh(s: np.ndarray, method: str = "auto"):
    """Symmetric eigendecomposition, eigenvalues DESCENDING.  method="jacobi"
    (in-repo, d <= ~256), "eigh" (numpy.linalg.eigh library primitive, for
    the large configs), "auto" picks by size."""
    s = 0.5 * (np.asarray(s, dtype=np.float64) + np.asarray(s, dtype=np.float64).T)
    if method == "auto":
        method = "jacobi" if s.shape[0] <= 96 else "eigh"
    if method == "jacobi":
        w, v = jacobi_eigh(s)
    elif method == "eigh":
        w, v = np.linalg.eigh(s)
    else:
        raise ValueError(method)
    order = np.argsort(-w, kind="stable")
    return w[order], v[:, order]


def canonical_sign(v: np.ndarray) -> np.ndarray:
    """Flip each row so its largest-|.| entry is positive (+-v are both
    solutions, PAPER.md:885 Lemma well_posed_utils "up to sign")."""
    v = np.array(v, dtype=np.float64)
    idx = np.argmax(np.abs(v), axis=1)
    sgn = np.sign(v[np.arange(v.shape[0]), idx])
    sgn[sgn == 0] = 1.0
    return v * sgn[:, None]


def generalized_eigh(a: np.ndarray, b: np.ndarray, k: int | None = None,
                     method: str = "auto"):
    """Exact top-k generalized eigenpairs of A v = lambda B v.

    Cholesky B = L L^T, C = L^{-1} A L^{-T} (symmetric, similar to B^{-1}A —
    PAPER.md:1169 Prop. sim_mat), Jacobi on C, v = L^{-T} w.  Returns
    (lambda descending [k], V [k x d] with unit Euclidean-norm rows,
    canonical sign) — the unit-sphere normalisation of the game's strategy
    space."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = a.shape[0]
    k = n if k is None else k
    if n <= 256:
        l = cholesky(b)
        c = solve_lower(l, solve_lower(l, a).T).T          # L^{-1} A L^{-T}
    else:
        l = np.linalg.cholesky(b)
        c = np.linalg.solve(l, np.linalg.solve(l, a).T).T
    w, wv = sym_eigh(c, method)
    if n <= 256:
        vv = solve_upper(l.T, wv[:, :k])                    # L^{-T} w
    else:
        vv = np.linalg.solve(l.T, wv[:, :k])
    vv = vv.T
    vv /= np.linalg.norm(vv, axis=1, keepdims=True)
    return w[:k], canonical_sign(vv)


def sqrtm_spd(b: np.ndarray, inverse: bool = False, method: str = "auto") -> np.ndarray:
    """B^{1/2} (or B^{-1/2}) of an SPD matrix via its eigendecomposition
    (needed by the Appendix A subspace error)."""
    w, v = sym_eigh(b, method)
    if np.min(w) <= 0:
        raise ValueError("matrix is not positive definite")
    p = -0.5 if inverse else 0.5
    return (v * (w ** p)[None, :]) @ v.T
