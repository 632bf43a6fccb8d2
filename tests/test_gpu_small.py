"""GPU parity of the one-CTA small-problem step (small_step.cuh, the fp32
variant of configs 0 and 1 in one launch per call): every stage of Alg. 2
 / Alg. 1 for small d, k inside one
CTA with the state resident in shared memory, against the fp64 oracle on
identical seeded inputs (-m gpu).  Bars: the north star's fp32 variant,
1e-4 normwise and per player."""
import numpy as np
import pytest
import torch

from tests.gpu_harness import check_cca_step, oracle_cca_step, random_state, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def geig():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2206_04993_b200 import build
    build.build()
    from paper_2206_04993_b200 import geig as g
    return g


def _assert(errs, tol):
    bad = {k: v for k, v in errs.items() if k != "sphere" and v > tol}
    assert not bad, f"parity errors above {tol}: {bad} (all: {errs})"
    assert errs["sphere"] < 1e-5


# (cfg, rows, k, dx, dy): config 1 at full size; several row chunks with an
# odd b (last row unused); b = 2 (h = 1); k = 16 with k not a multiple of 4
# and views of different widths; k = 1; bf16 data (config 2 recipe, narrowed)
CASES = [(1, 256, None, None, None), (1, 3001, None, None, None), (1, 2, 3, 8, 12), (1, 517, 13, 60, 52),
         (1, 64, 1, 4, 4), (2, 512, 16, 200, 136), (2, 1001, 5, 96, 40)]
ETA = {2: 0.5}   # config 2 at its eta = 0.1: some players' steps are small enough that fp32 storage of V' alone
                 # is ~1e-4 of the step; a larger step keeps the per-player bar meaningful


@pytest.mark.parametrize("cfg_idx,rows,k,dx,dy", CASES)
@pytest.mark.parametrize("state", ["random", "floor"])
def test_small_step_matches_oracle(geig, cfg_idx, rows, k, dx, dy, state):
    """One geig_step_cca on the small path (one launch) vs the oracle's Alg. 2
    step; the floor state clips most parents (Alg. 2 l.8)."""
    errs, got = check_cca_step(geig, cfg_idx, rows, k=k, dx=dx, dy=dy, math="f32", use_step=True, state=state,
                               rows_err=True, eta=ETA.get(cfg_idx))
    _assert(errs, 1e-4)
    if state == "floor" and (k or 8) > 2:
        assert got["clipped"], "the floor state should clip some parents"


def test_small_step_is_one_launch_and_matches_staged_path(geig):
    """The small path (GEIG_OPT_SMALL_STEP = 1, default) takes one launch per
    step and agrees with the staged products + update kernels (option 0) to
    fp32 rounding."""
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[1]
    x, y = cca_views(cfg, 256, seed=4)
    V, aux = random_state(cfg.k, cfg.d, 4)
    dev = "cuda:0"
    xd, yd = x.to(dev), y.to(dev)
    out = {}
    for small in (1, 0):
        s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math="f32", rho=cfg.rho, max_rows=256)
        try:
            geig.geig_set_option(s.h, geig.GEIG_OPT_SMALL_STEP, small)
            s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32,
                                                                                    device=dev))
            l0 = s.launches()
            for _ in range(3):
                geig.geig_step_cca(s.h, xd, yd, 256, cfg.eta, cfg.gamma)
            out[small] = (s.launches() - l0, *[t.double().cpu().numpy() for t in s.state()])
        finally:
            s.close()
    assert out[1][0] == 3 and out[0][0] > 3
    assert rel_err(out[1][1] - V, out[0][1] - V) < 1e-4
    assert rel_err(out[1][2], out[0][2]) < 1e-5


@pytest.mark.parametrize("rows,k,dx,dy", [(256, None, None, None), (1001, 16, 60, 52)])
def test_small_run_equals_steps_and_oracle(geig, rows, k, dx, dy):
    """geig_run_cca on the small path: T steps (distinct and repeated batches)
    in ONE launch with the state resident in shared memory leave exactly the
    state of T geig_step_cca calls (same arithmetic; the state round trip
    through global memory is exact), which matches T oracle steps."""
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[1]
    k = k or cfg.k
    dx, dy = dx or cfg.dx, dy or cfg.dy
    T = 5
    x, y = cca_views(cfg, 3 * rows, seed=21)
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    batches = [(x[i * rows:(i + 1) * rows], y[i * rows:(i + 1) * rows]) for i in (0, 1, 2, 0, 1)]
    V, aux = random_state(k, dx + dy, 22)
    V32 = V.astype(np.float32).astype(np.float64)
    aux32 = aux.astype(np.float32).astype(np.float64)
    dev = "cuda:0"
    Xd = [b_[0].to(dev).contiguous() for b_ in batches]
    Yd = [b_[1].to(dev).contiguous() for b_ in batches]
    states = []
    for run in (True, False):
        s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math="f32", rho=cfg.rho, max_rows=rows)
        try:
            s.set_state(torch.tensor(V32, dtype=torch.float32, device=dev),
                        torch.tensor(aux32, dtype=torch.float32, device=dev))
            l0 = s.launches()
            if run:
                geig.geig_run_cca(s.h, Xd, Yd, rows, cfg.eta, cfg.gamma)
                assert s.launches() - l0 <= 2       # the pointer-table copy is not a kernel; one launch
            else:
                for t in range(T):
                    geig.geig_step_cca(s.h, Xd[t], Yd[t], rows, cfg.eta, cfg.gamma)
            Vg, Ag = s.state()
            states.append((Vg.cpu().numpy(), Ag.cpu().numpy()))
        finally:
            s.close()
    assert np.array_equal(states[0][0], states[1][0]) and np.array_equal(states[0][1], states[1][1])
    Vo, Ao = V32, aux32
    for xb, yb in batches:
        _, _, Vo, Ao = oracle_cca_step(xb.double().numpy(), yb.double().numpy(), Vo, Ao, cfg.eta, cfg.gamma,
                                       cfg.rho)
    assert rel_err(states[0][0] - V32, Vo - V32) < 1e-4
    assert rel_err(states[0][1], Ao) < 1e-4


def test_small_dense_run_config0(geig):
    """Config 0 (Alg. 1, d = 16, k = 4): geig_run_dense runs the 2000 steps in
    one launch with A, B resident in shared memory; bit-identical to 2000
    geig_step_dense calls, per-step parity with the oracle along its own
    trajectory, and convergence to the exact generalized eigenvectors."""
    from oracle import estimators, game, linalg, metrics
    from synth import CONFIGS, dense_gep_small, gaussian_init
    cfg = CONFIGS[0]
    a, b = dense_gep_small(0)
    w, Vt = linalg.generalized_eigh(a, b, cfg.k)
    dev = "cuda:0"
    A = torch.tensor(a, dtype=torch.float32, device=dev)
    B = torch.tensor(b, dtype=torch.float32, device=dev)
    a32, b32 = A.double().cpu().numpy(), B.double().cpu().numpy()
    G = torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev)
    finals = []
    for run in (True, False):
        s = geig.Solver(geig.GEIG_DENSE, cfg.d, 0, cfg.k, math="f32", rho=cfg.rho)
        try:
            s.init_state(G)
            l0 = s.launches()
            if run:
                geig.geig_run_dense(s.h, A, B, cfg.steps, cfg.eta, cfg.gamma)
                assert s.launches() - l0 == 1
            else:
                for _ in range(cfg.steps):
                    geig.geig_step_dense(s.h, A, B, cfg.eta, cfg.gamma)
            finals.append([t.cpu().numpy() for t in s.state()])
        finally:
            s.close()
    assert np.array_equal(finals[0][0], finals[1][0]) and np.array_equal(finals[0][1], finals[1][1])
    ang = metrics.per_vector_angles(finals[0][0].astype(np.float64), Vt)
    assert np.all(ang < 1e-3), ang
    # 5-step launches from the oracle's state along its trajectory
    s = geig.Solver(geig.GEIG_DENSE, cfg.d, 0, cfg.k, math="f32", rho=cfg.rho)
    try:
        s.init_state(G)
        V0, aux0 = s.state()
        Vo, auxo = V0.double().cpu().numpy(), aux0.double().cpu().numpy()
        worst = 0.0
        for t in range(12):
            Vo32, auxo32 = Vo.astype(np.float32).astype(np.float64), auxo.astype(np.float32).astype(np.float64)
            s.set_state(torch.tensor(Vo32, dtype=torch.float32, device=dev),
                        torch.tensor(auxo32, dtype=torch.float32, device=dev))
            geig.geig_run_dense(s.h, A, B, 5, cfg.eta, cfg.gamma)
            Vg, auxg = [x.double().cpu().numpy() for x in s.state()]
            V2, aux2 = Vo32, auxo32
            for _ in range(5):
                av, bv = estimators.dense_products(a32, b32, V2)
                V2, aux2 = game.step_alg2(V2, aux2, [(av, bv)], cfg.eta, cfg.gamma, cfg.rho)
            worst = max(worst, rel_err(Vg - Vo32, V2 - Vo32), rel_err(auxg, aux2))
            Vo, auxo = V2, aux2
        assert worst < 1e-4, worst
    finally:
        s.close()


def test_small_path_declines_what_it_cannot_hold(geig):
    """Shapes outside the one-CTA budget (k > 16; 16 k d > 8192) and Adam run
    the staged kernels (several launches per step) with the same results."""
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[1]
    x, y = cca_views(cfg, 128, seed=31)
    dev = "cuda:0"
    for k, adam in ((17, False), (8, True)):
        s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, k, math="f32", rho=cfg.rho, max_rows=128)
        try:
            if adam:
                geig.geig_set_adam(s.h, 0.9, 0.999, 1e-3)
            V, aux = random_state(k, cfg.d, 32)
            s.set_state(torch.tensor(V, dtype=torch.float32, device=dev),
                        torch.tensor(aux, dtype=torch.float32, device=dev))
            l0 = s.launches()
            geig.geig_step_cca(s.h, x.to(dev), y.to(dev), 128, cfg.eta, cfg.gamma)
            assert s.launches() - l0 > 1
        finally:
            s.close()


@pytest.mark.parametrize("cfg_idx,math,rows", [(1, "f32", 256), (2, "bf16x2", 1024)])
def test_run_cca_host_pipeline_equals_device_steps(geig, cfg_idx, math, rows):
    """geig_run_cca_host (pinned host batches; the copy of batch t + 1 on a
    copy stream overlaps step t) leaves exactly the state of the same steps
    on device copies, and reports the bytes it moved."""
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[cfg_idx]
    T = 5
    x, y = cca_views(cfg, 2 * rows, seed=41)
    hx = [x[:rows].contiguous().pin_memory(), x[rows:].contiguous().pin_memory()]
    hy = [y[:rows].contiguous().pin_memory(), y[rows:].contiguous().pin_memory()]
    V, aux = random_state(cfg.k, cfg.d, 42)
    dev = "cuda:0"
    flag = 1 if x.dtype == torch.bfloat16 else 0
    out = []
    for host in (True, False):
        s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math=math, data_dtype=flag, rho=cfg.rho, max_rows=rows)
        try:
            s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
            if host:
                ga = torch.empty(cfg.k, cfg.k).pin_memory()
                h2d, d2h = geig.geig_run_cca_host(s.h, [hx[t % 2] for t in range(T)], [hy[t % 2] for t in range(T)],
                                                  rows, cfg.eta, cfg.gamma, ga)
                assert h2d == T * (hx[0].numel() * hx[0].element_size() + hy[0].numel() * hy[0].element_size())
                assert d2h == T * cfg.k * cfg.k * 4
            else:
                for t in range(T):
                    geig.geig_step_cca(s.h, hx[t % 2].to(dev), hy[t % 2].to(dev), rows, cfg.eta, cfg.gamma)
            out.append([t_.cpu().numpy() for t_ in s.state()] + [s.gram()[0].cpu().numpy()])
        finally:
            s.close()
    for a, b_ in zip(out[0], out[1]):
        assert np.array_equal(a, b_)
    assert np.array_equal(ga.numpy(), out[1][2])


@pytest.mark.parametrize("cl", [1, 2, 4, 8])
@pytest.mark.parametrize("rows,k,dx,dy", [(256, None, None, None), (3001, 13, 60, 52)])
def test_small_cluster_sizes_match_oracle_and_runs(geig, cl, rows, k, dx, dy):
    """The small-problem step on a thread-block cluster of cl CTAs (rows split
    over the CTAs, the products reduce-scattered, the Gram tables summed and
    v'' all-gathered through distributed shared memory in rank order): each
    cluster size matches the oracle's Alg. 2 over 3 steps at the fp32 bar,
    and a 3-step geig_run_cca equals 3 geig_step_cca calls bit for bit."""
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[1]
    k = k or cfg.k
    dx, dy = dx or cfg.dx, dy or cfg.dy
    T = 3
    x, y = cca_views(cfg, T * rows, seed=51)
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    batches = [(x[t * rows:(t + 1) * rows], y[t * rows:(t + 1) * rows]) for t in range(T)]
    V, aux = random_state(k, dx + dy, 52)
    V32 = V.astype(np.float32).astype(np.float64)
    aux32 = aux.astype(np.float32).astype(np.float64)
    dev = "cuda:0"
    Xd = [b_[0].to(dev).contiguous() for b_ in batches]
    Yd = [b_[1].to(dev).contiguous() for b_ in batches]
    states = []
    for run in (True, False):
        s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math="f32", rho=cfg.rho, max_rows=rows)
        try:
            geig.geig_set_option(s.h, geig.GEIG_OPT_SMALL_CLUSTER, cl)
            s.set_state(torch.tensor(V32, dtype=torch.float32, device=dev),
                        torch.tensor(aux32, dtype=torch.float32, device=dev))
            l0 = s.launches()
            if run:
                geig.geig_run_cca(s.h, Xd, Yd, rows, cfg.eta, cfg.gamma)
            else:
                for t in range(T):
                    geig.geig_step_cca(s.h, Xd[t], Yd[t], rows, cfg.eta, cfg.gamma)
                assert s.launches() - l0 == T
            Vg, Ag = s.state()
            states.append((Vg.cpu().numpy(), Ag.cpu().numpy()))
        finally:
            s.close()
    assert np.array_equal(states[0][0], states[1][0]) and np.array_equal(states[0][1], states[1][1])
    Vo, Ao = V32, aux32
    for xb, yb in batches:
        _, _, Vo, Ao = oracle_cca_step(xb.double().numpy(), yb.double().numpy(), Vo, Ao, cfg.eta, cfg.gamma, cfg.rho)
    assert rel_err(states[0][0] - V32, Vo - V32) < 1e-4
    assert rel_err(states[0][1], Ao) < 1e-4
