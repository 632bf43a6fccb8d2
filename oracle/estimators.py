"""ORACLE (test infrastructure only) — the matrices A, B of the GEP and their
unbiased minibatch estimates.

CCA (§1): A = [[0, E xy^T],[E yx^T, 0]], B = [[E xx^T, 0],[0, E yy^T]],
with expectations replaced by sample means ("means over a finite
sample dataset (e.g. 1/n X^T X)").

Minibatch estimates (§3, Alg. 2 line 7 "unbiased estimates
using independent data batches"): DESIGN.md reading R1 — the b paired rows of
step t are split into two disjoint halves; rows [0, h) estimate A, rows
[h, b) estimate B, h = b/2.
"""
from __future__ import annotations

import numpy as np


def cca_matrices(x: np.ndarray, y: np.ndarray):
    """Sample CCA matrices from paired rows x (n x dx),
    y (n x dy): A has zero diagonal blocks, B zero off-diagonal blocks."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n, dx = x.shape
    dy = y.shape[1]
    cxy = x.T @ y / n
    a = np.zeros((dx + dy, dx + dy))
    a[:dx, dx:] = cxy
    a[dx:, :dx] = cxy.T
    b = np.zeros((dx + dy, dx + dy))
    b[:dx, :dx] = x.T @ x / n
    b[dx:, dx:] = y.T @ y / n
    return a, b


def cca_minibatch_matrices(x: np.ndarray, y: np.ndarray):
    """(A_t, B_t) of one step: A_t from rows [0,h), B_t from rows [h,b)
    (reading R1)."""
    b = x.shape[0]
    h = b // 2
    a_t, _ = cca_matrices(x[:h], y[:h])
    _, b_t = cca_matrices(x[h:2 * h], y[h:2 * h])
    return a_t, b_t


def cca_products(x: np.ndarray, y: np.ndarray, V: np.ndarray):
    """A_t v_j and B_t v_j for every row v_j of V (k x (dx+dy)) without
    forming the (dx+dy)^2 matrices: by the block structure of PAPER.md:831,
      A_t v = 1/h [X1^T (Y1 v_y) ; Y1^T (X1 v_x)],
      B_t v = 1/h [X2^T (X2 v_x) ; Y2^T (Y2 v_y)].
    Returns (AV, BV), each k x (dx+dy), float64."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    dx = x.shape[1]
    h = x.shape[0] // 2
    x1, y1, x2, y2 = x[:h], y[:h], x[h:2 * h], y[h:2 * h]
    vx, vy = V[:, :dx].T, V[:, dx:].T              # d_view x k
    av = np.concatenate([x1.T @ (y1 @ vy), y1.T @ (x1 @ vx)], axis=0) / h
    bv = np.concatenate([x2.T @ (x2 @ vx), y2.T @ (y2 @ vy)], axis=0) / h
    return av.T.copy(), bv.T.copy()


def dense_products(a: np.ndarray, b: np.ndarray, V: np.ndarray):
    """Full-batch products A v_j, B v_j for every row v_j of V (configs 0, 4)."""
    return (np.asarray(a, np.float64) @ V.T).T.copy(), (np.asarray(b, np.float64) @ V.T).T.copy()
