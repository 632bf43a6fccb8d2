"""ORACLE (test infrastructure only) — the gamma-EigenGame utilities and
update rules, written out per player in the paper's order and notation.

Notation (§2-3): players i = 0..k-1 (the paper's 1..k), strategies
v_i on the unit sphere stored as the ROWS of V (k x d); auxiliary variables
[Bv]_i as the rows of AUX (k x d).  "A v" for the stochastic algorithm means
the minibatch product A_t v (Alg. 2 line 10 "A_tm"); the
products for every player are passed in as AV[j] = A_t v_j, BV[j] = B_t v_j
(Appendix F, "we parallelized the estimation of the
matrix-vector products Av_i and Bv_i for all i").  Where the paper writes a
product with a normalised parent (A y_j, B y_j) it is formed by linearity
from these products, exactly as the paper itself forms
[By]_j = [Bv]_j / sqrt(.) (Alg. 2 line 9).
"""
from __future__ import annotations

import numpy as np


# ---------------------------------------------------------------------------
# Utilities (§2)
# ---------------------------------------------------------------------------

def rayleigh(v: np.ndarray, a: np.ndarray, b: np.ndarray) -> float:
    """Generalized Rayleigh quotient <v,Av>/<v,Bv>."""
    return float(v @ a @ v) / float(v @ b @ v)


def utility(i: int, V: np.ndarray, a: np.ndarray, b: np.ndarray) -> float:
    """u_i(v_i | v_{j<i}), first form of Eq. util_new:
    <v_i,Av_i>/<v_i,Bv_i> - sum_{j<i} <v_j,Av_j><v_i,Bv_j>^2 /
    (<v_j,Bv_j>^2 <v_i,Bv_i>)."""
    vi = V[i]
    bii = vi @ b @ vi
    u = (vi @ a @ vi) / bii
    for j in range(i):
        vj = V[j]
        u -= (vj @ a @ vj) * (vi @ b @ vj) ** 2 / ((vj @ b @ vj) ** 2 * bii)
    return float(u)


def utility_y_form(i: int, V: np.ndarray, a: np.ndarray, b: np.ndarray) -> float:
    """Second form of Eq. util_new: lambda_i -
    sum_{j<i} lambda_j <y_i, B y_j>^2 with y = v / ||v||_B."""
    def y(v):
        return v / np.sqrt(v @ b @ v)
    lam = [rayleigh(V[j], a, b) for j in range(i + 1)]
    u = lam[i]
    yi = y(V[i])
    for j in range(i):
        u -= lam[j] * (yi @ b @ y(V[j])) ** 2
    return float(u)


def utility_gradient(i: int, V: np.ndarray, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Eq. eq:util_grad, 'up to scaling factors' the gradient of
    u_i w.r.t. v_i (it equals exactly half of it):
    [(v_i^T B v_i) A v_i - (v_i^T A v_i) B v_i]/<v_i,Bv_i>^2
    - sum_{j<i} lambda_j/<v_j,Bv_j> (v_i^T B v_j)
      [<v_i,Bv_i> B v_j - <v_i,B v_j> B v_i]/<v_i,Bv_i>^2."""
    vi = V[i]
    avi, bvi = a @ vi, b @ vi
    bii = vi @ bvi
    g = (bii * avi - (vi @ avi) * bvi) / bii ** 2
    for j in range(i):
        vj = V[j]
        bvj = b @ vj
        lam_j = (vj @ a @ vj) / (vj @ bvj)
        g -= lam_j / (vj @ bvj) * (vi @ bvj) * (bii * bvj - (vi @ bvj) * bvi) / bii ** 2
    return g


# ---------------------------------------------------------------------------
# Alg. 1 — deterministic / full batch
# ---------------------------------------------------------------------------

def direction_alg1(i: int, V: np.ndarray, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Alg. 1 lines 5-8 (Eq. eq:update) with exact
    y_j = v_j / sqrt(<v_j, B v_j>)."""
    vi = V[i]
    avi, bvi = a @ vi, b @ vi
    rewards = (vi @ bvi) * avi - (vi @ avi) * bvi
    penalties = np.zeros_like(vi)
    for j in range(i):
        yj = V[j] / np.sqrt(V[j] @ b @ V[j])
        byj = b @ yj
        penalties += (vi @ (a @ yj)) * ((vi @ bvi) * byj - (vi @ byj) * bvi)
    return rewards - penalties


def step_alg1(V: np.ndarray, a: np.ndarray, b: np.ndarray, eta: float) -> np.ndarray:
    """One iteration of Alg. 1 (parfor over players from the iteration-start
    snapshot, then v_i <- v_i' / ||v_i'||, lines 9-10)."""
    grads = [direction_alg1(i, V, a, b) for i in range(V.shape[0])]
    out = np.empty_like(V)
    for i, g in enumerate(grads):
        vp = V[i] + eta * g
        out[i] = vp / np.linalg.norm(vp)
    return out


# ---------------------------------------------------------------------------
# Alg. 2 — stochastic with auxiliary [Bv] and rho clipping
# ---------------------------------------------------------------------------

def init_state(g: np.ndarray):
    """Alg. 2 lines 2-3: v_i ~ N(0,I) (the draws g are an input), v_i <- v_i/||v_i||;
    [Bv]_i <- v_i^0."""
    V = np.asarray(g, dtype=np.float64)
    V = V / np.linalg.norm(V, axis=1, keepdims=True)
    return V, V.copy()


def clip_denominator(v_j: np.ndarray, aux_j: np.ndarray, rho: float) -> float:
    """sqrt(max(<v_j, [Bv]_j>, rho)) — Alg. 2 lines 8-9."""
    return float(np.sqrt(max(float(v_j @ aux_j), rho)))


def direction_alg2(i: int, V: np.ndarray, AUX: np.ndarray, AV: np.ndarray,
                   BV: np.ndarray, rho: float) -> np.ndarray:
    """Alg. 2 lines 8-12 for player i:
      y_j = v_j / sqrt(max(<v_j,[Bv]_j>, rho))
      [By]_j = [Bv]_j / sqrt(max(<v_j,[Bv]_j>, rho))
      rewards = (v_i^T B_t v_i) A_t v_i - (v_i^T A_t v_i) B_t v_i
      penalties = sum_{j<i} (v_i^T A_t y_j) [<v_i, B_t v_i>[By]_j - <v_i,[By]_j> B_t v_i]
    with A_t y_j = (A_t v_j) / sqrt(.) by linearity."""
    vi = V[i]
    avi, bvi = AV[i], BV[i]
    rewards = (vi @ bvi) * avi - (vi @ avi) * bvi
    penalties = np.zeros_like(vi)
    for j in range(i):
        den = clip_denominator(V[j], AUX[j], rho)
        a_yj = AV[j] / den            # A_t y_j
        byj = AUX[j] / den            # [By]_j
        penalties += (vi @ a_yj) * ((vi @ bvi) * byj - (vi @ byj) * bvi)
    return rewards - penalties


def aux_direction(i: int, AUX: np.ndarray, BV: np.ndarray) -> np.ndarray:
    """Alg. 2 line 13: grad^{Bv}_i = B_t v_i - [Bv]_i."""
    return BV[i] - AUX[i]


def step_alg2(V: np.ndarray, AUX: np.ndarray, machines, eta: float, gamma: float,
              rho: float):
    """One iteration of Alg. 2.

    `machines` is a list of (AV_m, BV_m) pairs, the products of machine m's
    independent estimates A_tm, B_tm with every v_j.  Directions are averaged
    over m (lines 14, 17), then v_i' = v_i + eta grad_i, v_i <- v_i'/||v_i'||,
    [Bv]_i <- [Bv]_i + gamma grad^{Bv}_i.  All players read the
    iteration-start snapshot (parfor)."""
    k = V.shape[0]
    M = len(machines)
    V_new = np.empty_like(V)
    AUX_new = np.empty_like(AUX)
    for i in range(k):
        g = sum(direction_alg2(i, V, AUX, av, bv, rho) for av, bv in machines) / M
        gbv = sum(aux_direction(i, AUX, bv) for _, bv in machines) / M
        vp = V[i] + eta * g
        V_new[i] = vp / np.linalg.norm(vp)
        AUX_new[i] = AUX[i] + gamma * gbv
    return V_new, AUX_new


def step_alg2_matrices(V, AUX, a_t, b_t, eta, gamma, rho):
    """Alg. 2 iteration with explicit (symmetric) estimate matrices, M = 1."""
    return step_alg2(V, AUX, [(V @ a_t.T, V @ b_t.T)], eta, gamma, rho)


def step_alg2_appendix_f(V, AUX, machines, eta, gamma, rho):
    """Appendix F variant: the products A v_i, B v_i are
    estimated in parallel and AGGREGATED across machines first, then one
    update is formed from the aggregated products."""
    M = len(machines)
    av = sum(m[0] for m in machines) / M
    bv = sum(m[1] for m in machines) / M
    return step_alg2(V, AUX, [(av, bv)], eta, gamma, rho)


# ---------------------------------------------------------------------------
# Alg. 3 — smooth log-space variant (Appendix E)
# ---------------------------------------------------------------------------

def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def smooth_bracket(z: float, rho: float, nu: float) -> float:
    """[<v,Bv>]_j = exp(log rho + (log nu - log rho) sigmoid(z_j)) (Alg. 3 line 7)."""
    return float(np.exp(np.log(rho) + (np.log(nu) - np.log(rho)) * _sigmoid(z)))


def direction_alg3(i, V, AUX, Z, AV, BV, rho, nu):
    """Alg. 3 lines 8-12: as Alg. 2 but with the denominators
    sqrt([<v,Bv>]_j) from the sigmoid-parameterised bracket."""
    vi = V[i]
    avi, bvi = AV[i], BV[i]
    rewards = (vi @ bvi) * avi - (vi @ avi) * bvi
    penalties = np.zeros_like(vi)
    for j in range(i):
        den = np.sqrt(smooth_bracket(Z[j], rho, nu))
        a_yj = AV[j] / den
        byj = AUX[j] / den
        penalties += (vi @ a_yj) * ((vi @ bvi) * byj - (vi @ byj) * bvi)
    return rewards - penalties


def z_direction(i, V, AUX, Z, rho, nu):
    """Alg. 3 line 14: grad^z_i = (<v_i,[Bv]_i> - [<v,Bv>]_i) [<v,Bv>]_i
    (log nu - log rho) sigma(z_i)(1 - sigma(z_i)) — ascent sign as in the
    algorithm box (reading R6)."""
    br = smooth_bracket(Z[i], rho, nu)
    s = _sigmoid(Z[i])
    return (float(V[i] @ AUX[i]) - br) * br * (np.log(nu) - np.log(rho)) * s * (1 - s)


def step_alg3(V, AUX, Z, machines, eta, gamma, rho, nu):
    """One iteration of Alg. 3."""
    k = V.shape[0]
    M = len(machines)
    V_new, AUX_new, Z_new = np.empty_like(V), np.empty_like(AUX), np.array(Z, dtype=np.float64)
    for i in range(k):
        g = sum(direction_alg3(i, V, AUX, Z, av, bv, rho, nu) for av, bv in machines) / M
        gbv = sum(bv[i] - AUX[i] for _, bv in machines) / M
        gz = z_direction(i, V, AUX, Z, rho, nu)     # same for every machine
        vp = V[i] + eta * g
        V_new[i] = vp / np.linalg.norm(vp)
        AUX_new[i] = AUX[i] + gamma * gbv
        Z_new[i] = Z[i] + gamma * gz
    return V_new, AUX_new, Z_new


# ---------------------------------------------------------------------------
# Optimizer / schedules (Appendix H)
# ---------------------------------------------------------------------------

def adam_ascent(v, g, m, s, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    """Adam(b1=0.9, b2=0.999, eps=1e-8) ascent step on v_i,
    standard bias-corrected moments; returns (v + step, m, s).  The sphere
    retraction is applied by the caller."""
    m = b1 * m + (1 - b1) * g
    s = b2 * s + (1 - b2) * g * g
    mh = m / (1 - b1 ** t)
    sh = s / (1 - b2 ** t)
    return v + lr * mh / (np.sqrt(sh) + eps), m, s


def step_alg2_adam(V, AUX, Mom, Sec, t, machines, lr, gamma, rho, b1=0.9, b2=0.999, eps=1e-8):
    """One iteration of Alg. 2 with the ascent of line 16
    replaced by Adam on v_i (Appendix H: "Adam(b1=0.9,
    b2=0.999, eps=1e-8) was used for learning v_i"): the averaged direction of
    lines 10-14 is Adam's gradient, then the sphere retraction of line 17 and
    the aux update of line 19 as in step_alg2.  `t` is the 1-based step count
    of the bias corrections; Mom, Sec are the k x d moments.  Returns
    (V, AUX, Mom, Sec)."""
    k = V.shape[0]
    M = len(machines)
    V_new, AUX_new = np.empty_like(V), np.empty_like(AUX)
    Mom_new, Sec_new = np.empty_like(Mom), np.empty_like(Sec)
    for i in range(k):
        g = sum(direction_alg2(i, V, AUX, av, bv, rho) for av, bv in machines) / M
        gbv = sum(aux_direction(i, AUX, bv) for _, bv in machines) / M
        vp, Mom_new[i], Sec_new[i] = adam_ascent(V[i], g, Mom[i], Sec[i], t, lr, b1, b2, eps)
        V_new[i] = vp / np.linalg.norm(vp)
        AUX_new[i] = AUX[i] + gamma * gbv
    return V_new, AUX_new, Mom_new, Sec_new
