"""Column-owned multi-GPU step on one GPU, ranks emulated in one process
(the profiling guide: ranks whose kernels wait on one another must not run
as separate launches on one GPU; these do not wait on one another, and the
collectives are emulated exactly: the reduce-scatter as a sum of the
ranks' per-owner chunks, the all-gather as copies of the owners' shadow
blocks).  N ranks each own d / N columns; per step: geig_products_cca_owned
on the rank's rows -> sum of the chunks -> geig_update_owned -> shadow
blocks exchanged.  After T steps the assembled state must match the
oracle's Appendix-F step on the union of the ranks' rows,
and the replicated all-reduce path (geig_products_cca_tables +
geig_update_tables) to rounding."""
import numpy as np
import pytest
import torch

from tests.gpu_harness import floor_state, random_state, rel_err, row_rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def geig():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2206_04993_b200 import build
    build.build()
    from paper_2206_04993_b200 import geig as g
    return g


def _run_owned(geig, N, xs, ys, V, aux, k, dx, b, eta, gamma, rho, math):
    """xs[t][r], ys[t][r]: device batches of rank r at step t."""
    d = 2 * dx
    W = d // N
    dev = "cuda:0"
    ss = []
    for r in range(N):
        s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math=math, data_dtype=geig.GEIG_DATA_BF16, rho=rho, max_rows=b)
        s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
        geig.geig_set_partition(s.h, N, r)
        ss.append(s)
    try:
        chunk = geig.geig_owned_chunk_floats(ss[0].h)
        bufs = [torch.empty(N, chunk, device=dev) for _ in range(N)]
        shadows = [geig.shadow_tensor(s.h, N, k, W) for s in ss]
        for t in range(len(xs)):
            for r in range(N):
                geig.geig_products_cca_owned(ss[r].h, xs[t][r], ys[t][r], b, 1.0 / (N * (b // 2)), bufs[r])
            summed = [sum(bufs[q][r] for q in range(N)).contiguous() for r in range(N)]   # reduce-scatter
            for r in range(N):
                geig.geig_update_owned(ss[r].h, summed[r], eta, gamma)
            for r in range(N):                                                          # all-gather
                for q in range(N):
                    if q != r:
                        shadows[q][r].copy_(shadows[r][r])
        Vf = torch.empty(k, d, device=dev)
        Af = torch.empty_like(Vf)
        for r in range(N):
            Vr, Ar = ss[r].state()
            Vf[:, r * W:(r + 1) * W] = Vr[:, r * W:(r + 1) * W]
            Af[:, r * W:(r + 1) * W] = Ar[:, r * W:(r + 1) * W]
        torch.cuda.synchronize()
    finally:
        for s in ss:
            s.close()
    Vf = Vf / Vf.norm(dim=1, keepdim=True)
    return Vf.double().cpu().numpy(), Af.double().cpu().numpy()


@pytest.mark.parametrize("N,state,math", [(2, "floor", "bf16x2"), (3, "random", "bf16x2"), (2, "random", "bf16")])
def test_owned_step_matches_appendix_f(geig, N, state, math):
    from oracle import estimators, game
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[2]
    k, dx, b, T = 16, 768, 512, 3
    eta, gamma = 0.2, 0.5
    x, y = cca_views(cfg, T * N * b, seed=17)
    x, y = x[:, :dx].contiguous(), y[:, :dx].contiguous()
    V, aux = (floor_state if state == "floor" else (lambda k_, d_, s_, r_: random_state(k_, d_, s_)))(k, 2 * dx, 8, cfg.rho)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    dev = "cuda:0"
    rows = lambda t, r: slice((t * N + r) * b, (t * N + r + 1) * b)
    xs = [[x[rows(t, r)].to(dev).contiguous() for r in range(N)] for t in range(T)]
    ys = [[y[rows(t, r)].to(dev).contiguous() for r in range(N)] for t in range(T)]
    Vg, Ag = _run_owned(geig, N, xs, ys, V, aux, k, dx, b, eta, gamma, cfg.rho, math)
    Vo, Ao = V, aux
    for t in range(T):
        ms = [estimators.cca_products(x[rows(t, r)].double().numpy(), y[rows(t, r)].double().numpy(), Vo)
              for r in range(N)]
        Vo, Ao = game.step_alg2_appendix_f(Vo, Ao, ms, eta, gamma, cfg.rho)
    tol_s, tol_a = (1e-3, 1e-4) if math == "bf16x2" else (1e-2, 1e-2)
    es, ea = rel_err(Vg - V, Vo - V), rel_err(Ag, Ao)
    rs, ra = row_rel_err(Vg, Vo, V), row_rel_err(Ag, Ao)
    print(f"owned N={N} {state} {math}: step {es:.2e} (rows {rs:.2e}) aux {ea:.2e} (rows {ra:.2e})")
    assert es < tol_s and rs < 3 * tol_s, (es, rs)
    assert ea < tol_a and ra < 10 * tol_a, (ea, ra)


def test_owned_partition_errors_are_loud(geig):
    s = geig.Solver(geig.GEIG_CCA, 784, 784, 16, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=0.1, max_rows=64)
    try:
        with pytest.raises(geig.GeigError, match="64 world"):
            geig.geig_set_partition(s.h, 2, 0)            # d = 1568 is not a multiple of 128
        with pytest.raises(geig.GeigError):
            geig.geig_set_partition(s.h, 2, 2)            # rank out of range
        with pytest.raises(geig.GeigError, match="no partition"):
            geig.geig_update_owned(s.h, torch.zeros(64, device="cuda:0"), 0.1, 0.5)
    finally:
        s.close()
