"""Pins for oracle/game.py against the paper's printed facts, its closed-form
propositions and independent mathematics (finite differences, fixed points)."""
import numpy as np
import pytest

from oracle import estimators, game, linalg
from synth import appendix_b_example, dense_gep_small, gaussian_init


def _planted(d, k, seed):
    a, b = dense_gep_small(seed, d)
    w, V = linalg.generalized_eigh(a, b, k)
    return a, b, w, V


# --- §2 utilities ----------------------------------------------------------

def test_fig1_utility_values():
    """Fig. 1 caption: player 2 aligned with the top
    eigenvector receives zero utility, aligned with the second eigenvector it
    receives the second eigenvalue."""
    a, b = appendix_b_example()
    w, V = linalg.generalized_eigh(a, b)
    at_top = np.stack([V[0], V[0]])
    assert abs(game.utility(1, at_top, a, b)) < 1e-12 * w[0]
    assert abs(game.utility(1, V, a, b) - w[1]) < 1e-10 * w[0]


def test_utility_forms_agree_and_first_player_is_rayleigh():
    rng = np.random.default_rng(0)
    a, b = dense_gep_small(1, 8)
    V = rng.standard_normal((4, 8))
    for i in range(4):
        assert np.isclose(game.utility(i, V, a, b), game.utility_y_form(i, V, a, b), rtol=1e-12)
    assert np.isclose(game.utility(0, V, a, b), game.rayleigh(V[0], a, b), rtol=1e-14)


def test_utility_simplex_form_lemma_well_posed():
    """Lemma well_posed_utils: with exact parents,
    u_i = sum_{j>=i} lambda_j z_j, z_j = w_j^2 <v_j,Bv_j> / sum_p w_p^2 <v_p,Bv_p>,
    where v_hat_i = sum_p w_p v_p (expansion in the generalized eigenbasis)."""
    a, b = dense_gep_small(2, 6)
    lam, Vall = linalg.generalized_eigh(a, b)           # all 6 pairs
    rng = np.random.default_rng(7)
    for i in range(4):
        vhat = rng.standard_normal(6)
        vhat /= np.linalg.norm(vhat)
        wcoef = np.linalg.solve(Vall.T, vhat)
        bnorm = np.einsum("pi,ij,pj->p", Vall, b, Vall)
        z = wcoef ** 2 * bnorm / np.sum(wcoef ** 2 * bnorm)
        V = np.vstack([Vall[:i], vhat[None]])
        assert np.isclose(game.utility(i, V, a, b), np.sum(lam[i:] * z[i:]), rtol=1e-7, atol=1e-10)


def test_utility_gradient_is_half_true_gradient():
    """Eq. eq:util_grad 'up to scaling factors' — it equals exactly 1/2 of the
    gradient of Eq. util_new; checked by central finite differences."""
    rng = np.random.default_rng(3)
    a, b = dense_gep_small(3, 5)
    V = rng.standard_normal((3, 5))
    for i in range(3):
        g = game.utility_gradient(i, V, a, b)
        fd = np.zeros(5)
        h = 1e-6
        for c in range(5):
            Vp, Vm = V.copy(), V.copy()
            Vp[i, c] += h
            Vm[i, c] -= h
            fd[c] = (game.utility(i, Vp, a, b) - game.utility(i, Vm, a, b)) / (2 * h)
        assert np.allclose(2 * g, fd, rtol=1e-6, atol=1e-8)


# --- §3 update direction -----------------------------------------------------

def test_direction_is_steepest_ascent_at_exact_parents():
    """Prop.: with exact parents, Eq. eq:update equals
    <v_i,Bv_i>^2 x Eq. eq:util_grad (relation (i)), i.e. a positive multiple
    of the utility gradient."""
    a, b, w, Vt = _planted(7, 4, 4)
    rng = np.random.default_rng(4)
    for i in range(1, 4):
        V = Vt.copy()
        V[i] = rng.standard_normal(7)
        V[i] /= np.linalg.norm(V[i])
        d1 = game.direction_alg1(i, V, a, b)
        g = game.utility_gradient(i, V, a, b)
        bii = V[i] @ b @ V[i]
        assert np.allclose(d1, bii ** 2 * g, rtol=1e-8, atol=1e-8)
        # same through Alg. 2 with exact estimates and exact aux
        av, bv = estimators.dense_products(a, b, V)
        d2 = game.direction_alg2(i, V, (b @ V.T).T, av, bv, rho=0.0)
        assert np.allclose(d2, d1, rtol=1e-12, atol=1e-12)


def test_equivalence_to_eigengame_unloaded_when_B_is_identity():
    """Prop. 'Equivalence to EigenGame Unloaded': with
    B = I the direction is (I - v_i v_i^T)[A v_i - sum_{j<i}(v_i^T A v_j) v_j]."""
    rng = np.random.default_rng(5)
    d, k = 9, 5
    a = rng.standard_normal((d, d))
    a = a + a.T
    V = rng.standard_normal((k, d))
    V /= np.linalg.norm(V, axis=1, keepdims=True)
    av, bv = estimators.dense_products(a, np.eye(d), V)
    for i in range(k):
        mu = a @ V[i] - sum((V[i] @ a @ V[j]) * V[j] for j in range(i))
        ref = mu - (V[i] @ mu) * V[i]
        got = game.direction_alg2(i, V, V.copy(), av, bv, rho=0.5)
        assert np.allclose(got, ref, atol=1e-12)


def test_direction_tangent_to_sphere():
    """Appendix D: the update already lives in the tangent
    space, <grad_i, v_i> = 0, for any state and any symmetric estimates."""
    rng = np.random.default_rng(6)
    d, k = 11, 6
    x, y = rng.standard_normal((40, 5)), rng.standard_normal((40, 6))
    V = rng.standard_normal((k, d))
    V /= np.linalg.norm(V, axis=1, keepdims=True)
    aux = rng.standard_normal((k, d))
    av, bv = estimators.cca_products(x, y, V)
    for i in range(k):
        g = game.direction_alg2(i, V, aux, av, bv, rho=0.1)
        assert abs(g @ V[i]) <= 1e-12 * max(1.0, np.linalg.norm(g))


def test_fixed_point_at_generalized_eigenvectors():
    """Lemma lemma:right_fp: exact expectations, exact
    auxiliaries [Bv]_j = B v_j, v_j = generalized eigenvectors => every
    direction and every aux direction vanishes."""
    a, b, w, Vt = _planted(10, 5, 6)
    assert np.all(w > 0)
    av, bv = estimators.dense_products(a, b, Vt)
    aux = bv.copy()
    scale = np.linalg.norm(a) * np.linalg.norm(b)
    for i in range(5):
        assert np.linalg.norm(game.direction_alg2(i, Vt, aux, av, bv, rho=1e-3)) < 1e-10 * scale
        assert np.linalg.norm(game.aux_direction(i, aux, bv)) == 0.0
    V2, A2 = game.step_alg2(Vt, aux, [(av, bv)], 0.1, 1.0, 1e-3)
    assert np.allclose(V2, Vt, atol=1e-12) and np.allclose(A2, aux)


def test_rho_clipping_branch():
    """Alg. 2 line 8: denominators use max(<v_j,[Bv]_j>, rho)."""
    v = np.array([1.0, 0.0])
    assert game.clip_denominator(v, np.array([4.0, 0.0]), 0.0) == 2.0
    assert game.clip_denominator(v, np.array([0.01, 0.0]), 0.5) == pytest.approx(np.sqrt(0.5))
    assert game.clip_denominator(v, np.array([-3.0, 0.0]), 0.25) == pytest.approx(0.5)


def test_step_alg2_sphere_and_aux_running_average():
    """Sphere preservation (Alg. 2 lines 16-17) and the aux update being an
    exact running average: with a frozen v and constant B_t, [Bv] -> B v at
    rate (1 - gamma) per step."""
    rng = np.random.default_rng(8)
    a, b = dense_gep_small(0)
    V, aux = game.init_state(gaussian_init(4, 16, 0))
    av, bv = estimators.dense_products(a, b, V)
    V2, aux2 = game.step_alg2(V, aux, [(av, bv)], 0.01, 0.3, 0.05)
    assert np.allclose(np.linalg.norm(V2, axis=1), 1.0, atol=1e-14)
    e0 = np.linalg.norm(aux - bv)
    e = aux.copy()
    for _ in range(10):
        e = e + 0.3 * (bv - e)
    assert np.isclose(np.linalg.norm(e - bv), 0.7 ** 10 * e0, rtol=1e-9)
    assert np.allclose(aux2, aux + 0.3 * (bv - aux))


def test_alg2_machine_average_and_appendix_f():
    """Alg. 2 lines 14-17: directions averaged over M machines; Appendix F
    aggregates products first.  With identical machines both reduce to M=1;
    the M=4 mean equals the mean of two M=2 means."""
    rng = np.random.default_rng(9)
    d, k = 8, 3
    V, aux = game.init_state(rng.standard_normal((k, d)))
    ms = []
    for _ in range(4):
        x, y = rng.standard_normal((20, 4)), rng.standard_normal((20, 4))
        ms.append(estimators.cca_products(x, y, V))
    one = game.step_alg2(V, aux, [ms[0]], 0.1, 0.5, 0.01)
    rep = game.step_alg2(V, aux, [ms[0]] * 3, 0.1, 0.5, 0.01)
    assert np.allclose(one[0], rep[0]) and np.allclose(one[1], rep[1])
    f = game.step_alg2_appendix_f(V, aux, [ms[0]] * 3, 0.1, 0.5, 0.01)
    assert np.allclose(one[0], f[0])
    g4 = [game.direction_alg2(1, V, aux, av, bv, 0.01) for av, bv in ms]
    assert np.allclose(np.mean(g4, 0), 0.5 * (np.mean(g4[:2], 0) + np.mean(g4[2:], 0)))


def test_alg2_reduces_to_alg1_direction_with_exact_aux():
    """Appendix C: Alg. 2 subsumes Alg. 1 (rho=0, exact
    estimates): with [Bv]_j = B v_j the two directions coincide."""
    rng = np.random.default_rng(10)
    a, b = dense_gep_small(1)
    V, _ = game.init_state(rng.standard_normal((4, 16)))
    av, bv = estimators.dense_products(a, b, V)
    for i in range(4):
        assert np.allclose(game.direction_alg2(i, V, bv, av, bv, 0.0),
                           game.direction_alg1(i, V, a, b), atol=1e-12)


# --- Alg. 3 (Appendix E) ----------------------------------------------------

def test_alg3_bracket_and_stationarity():
    rho, nu = 0.05, 20.0
    for z in [-50.0, -2.0, 0.0, 3.0, 50.0]:
        br = game.smooth_bracket(z, rho, nu)
        assert rho * (1 - 1e-12) <= br <= nu * (1 + 1e-12)
    assert np.isclose(game.smooth_bracket(0.0, rho, nu), np.sqrt(rho * nu))
    # z-gradient vanishes when <v,[Bv]> equals the bracket
    v = np.array([[1.0, 0.0]])
    br = game.smooth_bracket(0.7, rho, nu)
    aux = np.array([[br, 5.0]])
    assert abs(game.z_direction(0, v, aux, [0.7], rho, nu)) < 1e-14
    # ascent sign: bracket below target -> z increases
    assert game.z_direction(0, v, np.array([[br * 2, 0.0]]), [0.7], rho, nu) > 0


def test_alg3_tracks_alg2_on_exact_stream():
    """With exact matrices the smooth variant converges to the same
    solution as Alg. 2 (config 0 problem, rho < lambda_min(B) < lambda_max(B) < nu)."""
    a, b = dense_gep_small(0)
    ev = np.linalg.eigvalsh(b)
    rho, nu = 0.5 * ev[0], 2 * ev[-1]
    w, Vt = linalg.generalized_eigh(a, b, 3)
    V, aux = game.init_state(gaussian_init(3, 16, 0))
    z = np.zeros(3)
    for _ in range(3000):
        av, bv = estimators.dense_products(a, b, V)
        V, aux, z = game.step_alg3(V, aux, z, [(av, bv)], 0.05, 0.5, rho, nu)
    from oracle import metrics
    assert np.all(metrics.per_vector_angles(V, Vt) < 1e-3)


def test_adam_first_step():
    v = np.zeros(3)
    g = np.array([1.0, 0.0, -2.0])
    v1, m, s = game.adam_ascent(v, g, np.zeros(3), np.zeros(3), 1, 0.1)
    assert np.allclose(v1, 0.1 * np.sign(g), atol=1e-6)
    v2, m2, s2 = game.adam_ascent(v, np.zeros(3), np.zeros(3), np.zeros(3), 1, 0.1)
    assert np.allclose(v2, 0.0)


def test_alg2_adam_reduces_to_sign_ascent():
    """Pins of step_alg2_adam against closed forms: with b1 = b2 = eps = 0 (and,
    for any b1, b2, at t = 1 from zero moments) Adam's step is lr * sign(g)
    per coordinate, so the iteration equals normalize(v + lr sign(grad_i)) with
    the Alg. 2 direction; the aux update is that of step_alg2."""
    rng = np.random.default_rng(4)
    k, d = 3, 7
    A = rng.standard_normal((d, d)); A = A + A.T
    Bh = rng.standard_normal((d, d)); B = Bh @ Bh.T + d * np.eye(d)
    V, _ = game.init_state(rng.standard_normal((k, d)))
    AUX = V @ B.T + 0.1 * rng.standard_normal((k, d))
    machines = [(V @ A.T, V @ B.T)]
    lr, gamma, rho = 0.05, 0.5, 0.1
    Vs, As = game.step_alg2(V, AUX, machines, lr, gamma, rho)
    want = np.empty_like(V)
    for i in range(k):
        g = game.direction_alg2(i, V, AUX, machines[0][0], machines[0][1], rho)
        vp = V[i] + lr * np.sign(g)
        want[i] = vp / np.linalg.norm(vp)
    Z = np.zeros_like(V)
    for b1, b2, eps, t in [(0.0, 0.0, 0.0, 5), (0.9, 0.999, 0.0, 1)]:
        Va, Aa, Ma, Sa = game.step_alg2_adam(V, AUX, Z, Z, t, machines, lr, gamma, rho, b1, b2, eps)
        np.testing.assert_allclose(Va, want, rtol=0, atol=1e-12)
        np.testing.assert_allclose(Aa, As, rtol=0, atol=0)
    # the moments are the exponential averages of the direction
    Va, Aa, Ma, Sa = game.step_alg2_adam(V, AUX, Z, Z, 1, machines, lr, gamma, rho, 0.9, 0.999, 1e-8)
    g0 = game.direction_alg2(0, V, AUX, machines[0][0], machines[0][1], rho)
    np.testing.assert_allclose(Ma[0], 0.1 * g0, rtol=1e-12)
    np.testing.assert_allclose(Sa[0], 0.001 * g0 * g0, rtol=1e-12)


# --- round-2 pins: the auxiliary variable, the rho floor, Alg. 3's z-gradient ---

def _golden_hand_cases():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "alg2_hand_directions.txt")
    rows = []
    for line in open(path):
        if line.strip() and not line.startswith("#"):
            f = line.split()
            rows.append((f[0], np.array(f[1:4], float), np.array(f[4:7], float), np.array(f[7:10], float)))
    return rows


@pytest.mark.parametrize("case", _golden_hand_cases(), ids=lambda c: c[0])
def test_alg2_direction_hand_worked_example(case):
    """tests/golden/alg2_hand_directions.txt: Alg. 2 lines 8-12 worked by hand
    (k = 2, d = 3) with [Bv]_0 != B_t v_0 — unclipped, clipped by rho and
    with <v_0,[Bv]_0> negative (PAPER.md:991 'may not be positive ...
    clip the result to be greater than or equal to rho')."""
    name, aux0, g0, g1 = case
    V = np.array([[1.0, 0, 0], [0, 1.0, 0]])
    AV = np.array([[2.0, 1, 0], [1, 3, 1]])
    BV = np.array([[1.0, 0, 0], [0, 2, 1]])
    AUX = np.array([aux0, [1.0, 1, 1]])
    np.testing.assert_allclose(game.direction_alg2(0, V, AUX, AV, BV, 0.5), g0, rtol=0, atol=1e-14)
    np.testing.assert_allclose(game.direction_alg2(1, V, AUX, AV, BV, 0.5), g1, rtol=0, atol=1e-13)
    V2, A2 = game.step_alg2(V, AUX, [(AV, BV)], 0.1, 0.25, 0.5)
    np.testing.assert_allclose(A2, AUX + 0.25 * (BV - AUX), rtol=0, atol=1e-15)
    for i, g in enumerate((g0, g1)):
        vp = V[i] + 0.1 * g
        np.testing.assert_allclose(V2[i], vp / np.sqrt(vp @ vp), rtol=0, atol=1e-15)


def test_alg2_aux_scale_invariance():
    """PAPER.md:989-991 and Alg. 2 lines 8-9: the parents enter only through
    y_j = v_j / sqrt(<v_j,[Bv]_j>) and [By]_j = [Bv]_j / sqrt(<v_j,[Bv]_j>), so
    with exact A, B and aux = c * B v_j (any c with c <v_j,Bv_j> >= rho) the
    penalty is unchanged: c cancels between (v_i^T A y_j) ~ c^-1/2 and
    [By]_j ~ c^1/2, and Alg. 2's direction equals Alg. 1's (exact
    y_j = v_j / ||v_j||_B).  A direction that took [By]_j from anything but
    the auxiliary variable scales with c and fails."""
    a, b = dense_gep_small(4, 9)
    rng = np.random.default_rng(11)
    V, _ = game.init_state(rng.standard_normal((4, 9)))
    av, bv = estimators.dense_products(a, b, V)
    for c in (0.3, 1.0, 2.5, 7.0):
        aux = c * bv
        assert np.all(c * np.sum(V * bv, 1) > 0.01)
        for i in range(4):
            np.testing.assert_allclose(game.direction_alg2(i, V, aux, av, bv, 0.01),
                                       game.direction_alg1(i, V, a, b), rtol=1e-10, atol=1e-10)


def test_alg2_penalty_scales_with_the_clipped_denominator():
    """Alg. 2 line 8 (the red max(., rho)): with one parent j,
    grad_i = rewards_i - P_ij / max(<v_j,[Bv]_j>, rho) where P_ij does not
    depend on rho — both the A y_j and the [By]_j factor carry one
    1/sqrt(max(.)).  rewards_i is player i's direction without parents.  So
    (rewards - grad) * max(<v_j,[Bv]_j>, rho) must be the same vector for rho
    below the inner product (no clip), above it, and for a NEGATIVE inner
    product; and for rho below the inner product the direction must not
    depend on rho at all."""
    rng = np.random.default_rng(12)
    d = 7
    V, _ = game.init_state(rng.standard_normal((2, d)))
    AV, BV = rng.standard_normal((2, d)), rng.standard_normal((2, d))
    for ip in (0.8, 0.05, -0.6):
        aux0 = rng.standard_normal(d)
        aux0 += (ip - V[0] @ aux0) * V[0]          # <v_0, [Bv]_0> = ip exactly
        AUX = np.stack([aux0, rng.standard_normal(d)])
        rewards = game.direction_alg2(0, V[::-1].copy(), AUX[::-1].copy(), AV[::-1].copy(), BV[::-1].copy(), 1.0)
        P = []
        for rho in (0.01, 0.3, 1.7):
            g = game.direction_alg2(1, V, AUX, AV, BV, rho)
            P.append((rewards - g) * max(ip, rho))
        for p in P[1:]:
            np.testing.assert_allclose(p, P[0], rtol=1e-12, atol=1e-12)
        if ip > 0.3:
            np.testing.assert_allclose(game.direction_alg2(1, V, AUX, AV, BV, 0.01),
                                       game.direction_alg2(1, V, AUX, AV, BV, 0.3), rtol=1e-13, atol=1e-13)


def test_alg3_z_direction_is_the_negative_gradient_of_the_bracket_fit():
    """Appendix E: grad_z = -(<v_j,Bv_j> - [<v,Bv>]_j)
    [<v,Bv>]_j (log nu - log rho) sigma(z_j)(1 - sigma(z_j)) is the derivative
    of the fit loss 1/2 (<v_j,Bv_j> - [<v,Bv>]_j(z_j))^2 with
    [<v,Bv>]_j(z) = exp(log rho + (log nu - log rho) sigma(z)); the algorithm
    box drops the minus and ascends (line 21), i.e.
    z_direction = -dL/dz (reading R6).  Checked by central differences of
    the bracket itself at several z and targets, which pins the whole chain
    factor br (log nu - log rho) sigma (1 - sigma)."""
    rho, nu = 0.05, 20.0
    for z in (-3.0, -0.4, 0.0, 0.9, 2.5):
        for target in (0.01, 0.7, 4.0, 30.0):
            v = np.array([[1.0, 0.0]])
            aux = np.array([[target, 0.3]])
            loss = lambda zz: 0.5 * (target - game.smooth_bracket(zz, rho, nu)) ** 2
            h = 1e-5
            fd = -(loss(z + h) - loss(z - h)) / (2 * h)
            got = game.z_direction(0, v, aux, [z], rho, nu)
            assert abs(got - fd) <= 1e-7 * max(1.0, abs(fd)), (z, target, got, fd)


def test_alg3_bracket_limits_and_monotone():
    """Alg. 3 line 7: the bracket runs from rho (z -> -inf) to nu (z -> +inf),
    increasing in z, log-linear in sigma(z)."""
    rho, nu = 0.05, 20.0
    zs = np.linspace(-30, 30, 121)
    br = np.array([game.smooth_bracket(z, rho, nu) for z in zs])
    assert np.all(np.diff(br) > 0)
    assert abs(br[0] - rho) < 1e-10 and abs(br[-1] - nu) < 1e-9
    s = 1 / (1 + np.exp(-0.8))
    assert np.isclose(np.log(game.smooth_bracket(0.8, rho, nu)), np.log(rho) + (np.log(nu) - np.log(rho)) * s,
                      rtol=1e-14)


def test_alg3_direction_equals_alg2_where_the_bracket_matches():
    """Alg. 3 lines 7-12 differ from Alg. 2 lines 8-12
    only in the denominator: with z_j set so that the bracket
    [<v,Bv>]_j = exp(log rho + (log nu - log rho) sigma(z_j)) equals
    <v_j,[Bv]_j> (> rho, so Alg. 2 does not clip), the two directions agree
    for ANY auxiliary variables — and with rho > <v_j,[Bv]_j> and z -> -inf
    the bracket is rho, Alg. 2's clipped value."""
    rng = np.random.default_rng(13)
    k, d = 4, 8
    V, _ = game.init_state(rng.standard_normal((k, d)))
    AV, BV = rng.standard_normal((k, d)), rng.standard_normal((k, d))
    AUX = V * rng.uniform(0.5, 3.0, (k, 1)) + 0.2 * rng.standard_normal((k, d))
    ip = np.sum(V * AUX, 1)
    assert np.all(ip > 0.06)
    rho, nu = 0.05, 50.0
    s = (np.log(ip) - np.log(rho)) / (np.log(nu) - np.log(rho))
    Z = np.log(s / (1 - s))
    for i in range(k):
        np.testing.assert_allclose(game.direction_alg3(i, V, AUX, Z, AV, BV, rho, nu),
                                   game.direction_alg2(i, V, AUX, AV, BV, rho), rtol=1e-10, atol=1e-10)
    rho_hi = 1.05 * ip.max()
    Zlo = np.full(k, -60.0)
    for i in range(k):
        np.testing.assert_allclose(game.direction_alg3(i, V, AUX, Zlo, AV, BV, rho_hi, 10 * rho_hi),
                                   game.direction_alg2(i, V, AUX, AV, BV, rho_hi), rtol=1e-10, atol=1e-10)
