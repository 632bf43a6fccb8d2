"""Peer-memory form of the column-owned multi-GPU step (geig_set_peers;
Appendix F: the products "aggregated ... across machines")
with the ranks emulated in one process on one GPU: every rank's receive
buffer, gathered shadow and flag words are plain device buffers whose
pointers the other "ranks" use as peer pointers.  The launches run in the
order a lockstep multi-GPU run completes them (every rank's products, then
every rank's update), so each kernel's flag waits are satisfied by kernels
that already finished: no kernel waits on one that has not started (the
profiling guide's rule for one GPU).

Checks: the state after T steps is BIT-IDENTICAL to the NCCL-style
column-owned step (geig_products_cca_owned + rank-order sum of the chunks +
geig_update_owned + copies of the shadow blocks) — the peer kernels store the
same numbers into the owners' slots and sum them in the same order — and it
matches the oracle's Appendix-F step; flags carry the step epoch."""
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


def _solvers(geig, N, V, aux, k, dx, b, rho, math):
    dev = "cuda:0"
    ss = []
    for r in range(N):
        s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math=math, data_dtype=geig.GEIG_DATA_BF16, rho=rho, max_rows=b)
        s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
        geig.geig_set_partition(s.h, N, r)
        ss.append(s)
    return ss


def _assemble(ss, N, W, k, d):
    Vf = torch.empty(k, d, device="cuda:0")
    Af = torch.empty_like(Vf)
    for r in range(N):
        Vr, Ar = ss[r].state()
        Vf[:, r * W:(r + 1) * W] = Vr[:, r * W:(r + 1) * W]
        Af[:, r * W:(r + 1) * W] = Ar[:, r * W:(r + 1) * W]
    torch.cuda.synchronize()
    return Vf.cpu().numpy(), Af.cpu().numpy()


def _run_peer(geig, N, xs, ys, V, aux, k, dx, b, eta, gamma, rho, math):
    d = 2 * dx
    W = d // N
    ss = _solvers(geig, N, V, aux, k, dx, b, rho, math)
    try:
        bufs = [geig.geig_peer_buffers(s.h) for s in ss]
        shadows = [geig.geig_shadow_buffer(s.h)[0] for s in ss]
        recv = [bb[0] for bb in bufs]
        flags = [bb[2] for bb in bufs]
        for s in ss:
            geig.geig_set_peers(s.h, recv, shadows, flags)
        scale = 1.0 / (N * (b // 2))
        for t in range(len(xs)):
            for r in range(N):
                geig.geig_products_cca_peer(ss[r].h, xs[t][r], ys[t][r], b, scale)
            for r in range(N):
                geig.geig_update_peer(ss[r].h, eta, gamma)
        out = _assemble(ss, N, W, k, d)
        # the flag words: step epochs len(xs) from every rank
        fl = torch.empty(2 * 8 * 32, dtype=torch.int32, device="cuda:0")
        lib_rt = __import__("ctypes").CDLL("libcudart.so.12")
        lib_rt.cudaMemcpy(__import__("ctypes").c_void_p(fl.data_ptr()), __import__("ctypes").c_void_p(flags[0]),
                          __import__("ctypes").c_size_t(fl.numel() * 4), 3)
        torch.cuda.synchronize()
        f = fl.view(16, 32)[:, 0].cpu().numpy()
        assert list(f[:N]) == [len(xs)] * N and list(f[8:8 + N]) == [len(xs)] * N, f
    finally:
        for s in ss:
            s.close()
    return out


def _run_owned_reference(geig, N, xs, ys, V, aux, k, dx, b, eta, gamma, rho, math):
    """The NCCL-style column-owned step with exact emulated collectives (rank-order sum)."""
    d = 2 * dx
    W = d // N
    dev = "cuda:0"
    ss = _solvers(geig, N, V, aux, k, dx, b, rho, math)
    try:
        chunk = geig.geig_owned_chunk_floats(ss[0].h)
        bufs = [torch.empty(N, chunk, device=dev) for _ in range(N)]
        shadows = [geig.shadow_tensor(s.h, N, k, W) for s in ss]
        for t in range(len(xs)):
            for r in range(N):
                geig.geig_products_cca_owned(ss[r].h, xs[t][r], ys[t][r], b, 1.0 / (N * (b // 2)), bufs[r])
            summed = [sum(bufs[q][r] for q in range(N)).contiguous() for r in range(N)]
            for r in range(N):
                geig.geig_update_owned(ss[r].h, summed[r], eta, gamma)
            for r in range(N):
                for q in range(N):
                    if q != r:
                        shadows[q][r].copy_(shadows[r][r])
        return _assemble(ss, N, W, k, d)
    finally:
        for s in ss:
            s.close()


@pytest.mark.parametrize("N,state,math", [(2, "floor", "bf16x2"), (3, "random", "bf16x2"), (4, "random", "bf16")])
def test_peer_step_matches_owned_step_and_appendix_f(geig, N, state, math):
    from oracle import estimators, game
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[2]
    k, dx, b, T = 16, 768, 512, 3
    eta, gamma = 0.2, 0.5
    x, y = cca_views(cfg, T * N * b, seed=23)
    x, y = x[:, :dx].contiguous(), y[:, :dx].contiguous()
    V, aux = (floor_state if state == "floor" else (lambda k_, d_, s_, r_: random_state(k_, d_, s_)))(k, 2 * dx, 9, cfg.rho)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    dev = "cuda:0"
    rows = lambda t, r: slice((t * N + r) * b, (t * N + r + 1) * b)
    xs = [[x[rows(t, r)].to(dev).contiguous() for r in range(N)] for t in range(T)]
    ys = [[y[rows(t, r)].to(dev).contiguous() for r in range(N)] for t in range(T)]
    Vp, Ap = _run_peer(geig, N, xs, ys, V, aux, k, dx, b, eta, gamma, cfg.rho, math)
    Vr, Ar = _run_owned_reference(geig, N, xs, ys, V, aux, k, dx, b, eta, gamma, cfg.rho, math)
    assert np.array_equal(Vp, Vr) and np.array_equal(Ap, Ar), (np.abs(Vp - Vr).max(), np.abs(Ap - Ar).max())
    Vp = Vp.astype(np.float64)
    Vp = Vp / np.linalg.norm(Vp, axis=1, keepdims=True)
    Vo, Ao = V, aux
    for t in range(T):
        ms = [estimators.cca_products(x[rows(t, r)].double().numpy(), y[rows(t, r)].double().numpy(), Vo)
              for r in range(N)]
        Vo, Ao = game.step_alg2_appendix_f(Vo, Ao, ms, eta, gamma, cfg.rho)
    tol_s, tol_a = (1e-3, 1e-4) if math == "bf16x2" else (1e-2, 1e-2)
    es, ea = rel_err(Vp - V, Vo - V), rel_err(Ap, Ao)
    rs = row_rel_err(Vp, Vo, V)
    assert es < tol_s and rs < 3 * tol_s, (es, rs)
    assert ea < tol_a, ea


def test_peer_calls_out_of_order_are_loud(geig):
    from synth import CONFIGS
    cfg = CONFIGS[2]
    V, aux = random_state(16, 1536, 1)
    ss = _solvers(geig, 2, V, aux, 16, 768, 64, cfg.rho, "bf16x2")
    try:
        with pytest.raises(geig.GeigError, match="no peers"):
            geig.geig_update_peer(ss[0].h, 0.1, 0.5)
        bufs = [geig.geig_peer_buffers(s.h) for s in ss]
        shadows = [geig.geig_shadow_buffer(s.h)[0] for s in ss]
        with pytest.raises(geig.GeigError, match="own buffers"):
            geig.geig_set_peers(ss[0].h, [bufs[1][0], bufs[0][0]], shadows, [b_[2] for b_ in bufs])
        geig.geig_set_peers(ss[0].h, [b_[0] for b_ in bufs], shadows, [b_[2] for b_ in bufs])
        with pytest.raises(geig.GeigError, match="without geig_products_cca_peer"):
            geig.geig_update_peer(ss[0].h, 0.1, 0.5)
    finally:
        for s in ss:
            s.close()
