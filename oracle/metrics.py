"""ORACLE (test infrastructure only) — evaluation metrics."""
from __future__ import annotations

import numpy as np

from .linalg import sqrtm_spd, sym_eigh


def subspace_error(Vhat: np.ndarray, a: np.ndarray, b: np.ndarray, k: int | None = None,
                   method: str = "auto") -> float:
    """Normalised subspace error of Appendix A:
    W = top-k eigenvectors of B^{-1/2} A B^{-1/2}, W_hat = B^{1/2} V_hat,
    U* = W W^+, P = W_hat W_hat^+, error = 1 - tr(U* P)/k in [0, 1].
    Vhat rows are the k approximations."""
    Vhat = np.atleast_2d(np.asarray(Vhat, dtype=np.float64))
    k = Vhat.shape[0] if k is None else k
    bmh = sqrtm_spd(b, inverse=True, method=method)
    bh = sqrtm_spd(b, method=method)
    _, w = sym_eigh(bmh @ a @ bmh, method)
    w = w[:, :k]
    what = bh @ Vhat[:k].T
    u_star = w @ np.linalg.pinv(w)
    p = what @ np.linalg.pinv(what)
    return float(1.0 - np.trace(u_star @ p) / k)


def angle_under_metric(u: np.ndarray, v: np.ndarray, c: np.ndarray) -> float:
    """arccos(|<C^{1/2}u, C^{1/2}v>| / (||C^{1/2}u|| ||C^{1/2}v||)) — Lemma
    orth_angle_change; equals the angle in the C inner product."""
    num = abs(float(u @ c @ v))
    den = np.sqrt(float(u @ c @ u) * float(v @ c @ v))
    return float(np.arccos(np.clip(num / den, 0.0, 1.0)))


def per_vector_angles(Vhat: np.ndarray, Vtrue: np.ndarray) -> np.ndarray:
    """Euclidean angle (radians, sign-folded) between each v_hat_i and the
    exact generalized eigenvector v_i (both unit-sphere)."""
    num = np.abs(np.sum(Vhat * Vtrue, axis=1))
    den = np.linalg.norm(Vhat, axis=1) * np.linalg.norm(Vtrue, axis=1)
    return np.arccos(np.clip(num / den, 0.0, 1.0))


def b_orthogonality_defect(V: np.ndarray, b: np.ndarray) -> float:
    """max_{i != j} |v_i^T B v_j| / ||B||_F (Lemma b_orth)."""
    g = V @ b @ V.T
    np.fill_diagonal(g, 0.0)
    return float(np.max(np.abs(g)) / np.linalg.norm(b)) if V.shape[0] > 1 else 0.0
