"""GPU parity with the rho floor of Alg. 2 line 8 ACTIVE (PAPER.md:1013,
the red max(., rho); "the inner product <v_j,[Bv]_j> may not be
positive definite, therefore, we manually clip the result to be greater than
or equal to rho").  tests/gpu_harness.floor_state sets <v_j,[Bv]_j> to
1, -0.5, 0.5 rho, 2 rho, -0.05, 0.25 rho, 4 rho, 0 (cycling over j), so
most parents clip, some negative, some just above rho.  Every path that
applies the clip is covered: the fused single-launch step (bf16x2, config 3
full size, the bench's launch configuration), the persistent multi-step
launch, the staged fp32 FFMA path (config 1), the multi-GPU tables path,
Alg. 3 (no clip: the smooth bracket, but negative inner products in its
z-gradient) and the streamed k > 64 update (dense).  Besides the normwise
bars, every player's own row is held to a bar (row_* keys): V' relative to
the step that player took, [Bv]' and the Gram-table rows relative to their
own norms."""
import numpy as np
import pytest
import torch

from oracle import estimators, game
from synth import CONFIGS, cca_views
from tests.gpu_harness import (check_cca_step, floor_state, gram_ref, rel_err, row_rel_err, tri_row_rel_err)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def geig():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2206_04993_b200 import build
    build.build()
    from paper_2206_04993_b200 import geig as g
    return g


def _check(errs, got, bars, k):
    assert len(got["clipped"]) >= max(1, (k - 1) // 2), got["clipped"]    # the floor is active
    bad = {key: v for key, v in errs.items() if key != "sphere" and v > bars.get(key, bars["*"])}
    assert not bad, f"above the bars {bars}: {bad} (all: {errs})"
    assert errs["sphere"] < 1e-5


# fp32 exactness variant: products, tables and aux to 1e-4 per player; bf16x2:
# products/tables/aux 1e-4 (normwise) with the step at 1e-3
F32 = {"*": 1e-4}
BF16X2 = {"*": 1e-4, "step": 1e-3, "row_step": 1e-3, "row_ga": 1e-3, "row_gb": 1e-3, "row_aux": 1e-3}


def test_floor_fused_bf16x2_config3_full_size(geig):
    """Config 3 at full size (dx = dy = 8192, b = 4096, k = 64, bf16 data),
    the fused single-launch step in bench.py's arithmetic (bf16x2)."""
    errs, got = check_cca_step(geig, 3, 4096, math="bf16x2", use_step=True, state="floor", rows_err=True, eta=0.02)
    _check(errs, got, BF16X2, 64)


@pytest.mark.parametrize("cfg_idx,rows,k,dx,dy", [(2, 1024, None, None, None), (2, 300, 24, 200, 136),
                                                  (2, 130, 5, 64, 8)])
def test_floor_fused_bf16x2_ragged(geig, cfg_idx, rows, k, dx, dy):
    errs, got = check_cca_step(geig, cfg_idx, rows, k=k, dx=dx, dy=dy, math="bf16x2", use_step=True,
                               state="floor", rows_err=True, eta=0.5)
    _check(errs, got, BF16X2, k or CONFIGS[cfg_idx].k)


def test_floor_fused_bf16_config3(geig):
    """Plain bf16 operands: the 1e-2 bar of the north star, per player too."""
    errs, got = check_cca_step(geig, 3, 4096, math="bf16", use_step=True, state="floor", rows_err=True, eta=0.02)
    _check(errs, got, {"*": 1e-2}, 64)


@pytest.mark.parametrize("rows,k,dx,dy", [(256, None, None, None), (203, 5, 37, 50), (300, 33, 64, 64)])
def test_floor_staged_fp32_config1(geig, rows, k, dx, dy):
    """The staged fp32 FFMA path (products launches + cooperative update)."""
    errs, got = check_cca_step(geig, 1, rows, k=k, dx=dx, dy=dy, math="f32", state="floor", rows_err=True, eta=0.5)
    _check(errs, got, F32, k or 8)


def test_floor_tables_path(geig):
    """Multi-GPU form (geig_products_cca_tables + geig_update_tables: the
    update from aggregated tables) on two row shards with the floor active."""
    from paper_2206_04993_b200.parallel import product_buffers
    cfg = CONFIGS[2]
    k, dx, dy, rows, M = 16, 784, 784, 512, 2
    x, y = cca_views(cfg, M * rows, seed=3)
    d = dx + dy
    V, aux = floor_state(k, d, 5, cfg.rho)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    dev = "cuda:0"
    eta = 0.5
    s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho,
                    max_rows=rows)
    try:
        s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
        nt = geig.geig_table_floats(s.h)
        AV, BV, T = product_buffers(k, d, nt, device=dev)
        AV1, BV1, T1 = product_buffers(k, d, nt, device=dev)
        xd, yd = x.to(dev), y.to(dev)
        scale = 1.0 / (M * (rows // 2))
        geig.geig_products_cca_tables(s.h, xd[:rows].contiguous(), yd[:rows].contiguous(), rows, scale, AV, BV, T)
        geig.geig_products_cca_tables(s.h, xd[rows:].contiguous(), yd[rows:].contiguous(), rows, scale, AV1, BV1, T1)
        AV += AV1
        BV += BV1
        T += T1
        geig.geig_update_tables(s.h, AV, BV, T, eta, cfg.gamma)
        V2g, aux2g = s.state()
        ga, gb, gc = s.gram()
    finally:
        s.close()
    x64, y64 = x.double().numpy(), y.double().numpy()
    machines = [estimators.cca_products(x64[:rows], y64[:rows], V), estimators.cca_products(x64[rows:], y64[rows:], V)]
    V2, aux2 = game.step_alg2_appendix_f(V, aux, machines, eta, cfg.gamma, cfg.rho)
    av = sum(m[0] for m in machines) / M
    bv = sum(m[1] for m in machines) / M
    ga_r, gb_r, gc_r = gram_ref(V, aux, av, bv)
    V2g, aux2g = V2g.double().cpu().numpy(), aux2g.double().cpu().numpy()
    errs = dict(step=rel_err(V2g - V, V2 - V), aux=rel_err(aux2g, aux2), row_step=row_rel_err(V2g, V2, V),
                row_aux=row_rel_err(aux2g, aux2), row_ga=tri_row_rel_err(ga.double().cpu().numpy(), ga_r),
                row_gc=tri_row_rel_err(gc.double().cpu().numpy(), gc_r), sphere=0.0)
    got = {"clipped": [j for j in range(k - 1) if float(V[j] @ aux[j]) < cfg.rho]}
    _check(errs, got, BF16X2, k)


def test_floor_run_cca_multi_step(geig):
    """geig_run_cca (T = 3 steps, one launch) from a clipping state: the
    clip decisions move as [Bv] follows B_t v (gamma = 0.5) — vs 3 oracle steps."""
    cfg = CONFIGS[3]
    k, dx, dy, rows, T = 64, 2048, 1024, 1024, 3
    x, y = cca_views(cfg, T * rows, seed=21)
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    V, aux = floor_state(k, dx + dy, 6, cfg.rho)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    eta, dev = 0.02, "cuda:0"
    s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho,
                    max_rows=rows)
    try:
        s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
        Xd = [x[t * rows:(t + 1) * rows].to(dev).contiguous() for t in range(T)]
        Yd = [y[t * rows:(t + 1) * rows].to(dev).contiguous() for t in range(T)]
        geig.geig_run_cca(s.h, Xd, Yd, rows, eta, cfg.gamma)
        Vg, Ag = (t_.double().cpu().numpy() for t_ in s.state())
    finally:
        s.close()
    Vo, Ao = V, aux
    for t in range(T):
        av, bv = estimators.cca_products(x[t * rows:(t + 1) * rows].double().numpy(),
                                         y[t * rows:(t + 1) * rows].double().numpy(), Vo)
        Vo, Ao = game.step_alg2(Vo, Ao, [(av, bv)], eta, cfg.gamma, cfg.rho)
    assert rel_err(Vg - V, Vo - V) < 1e-3 and row_rel_err(Vg, Vo, V) < 1e-3
    assert rel_err(Ag, Ao) < 1e-4 and row_rel_err(Ag, Ao) < 1e-3


@pytest.mark.parametrize("math", ["f32", "bf16x2"])
def test_floor_smooth_alg3(geig, math):
    """Alg. 3 from a state with negative and tiny
    <v_j,[Bv]_j>: the bracket replaces the clip, the z-gradient sees
    <v_i,[Bv]_i> - bracket < 0."""
    cfg_idx, rows, k, dx, dy = (1, 256, 8, 64, 64) if math == "f32" else (2, 1000, 24, 200, 136)
    cfg = CONFIGS[cfg_idx]
    T, nu, eta = 2, 20.0, 0.2
    x, y = cca_views(cfg, T * rows, seed=7)
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    V, aux = floor_state(k, dx + dy, 5, cfg.rho)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    z0 = np.random.default_rng(6).standard_normal(k).astype(np.float32).astype(np.float64)
    dev = "cuda:0"
    flag = 1 if x.dtype == torch.bfloat16 else 0
    s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math=math, data_dtype=flag, rho=cfg.rho, max_rows=rows)
    try:
        s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
        geig.geig_set_smooth(s.h, nu)
        geig.geig_smooth_state(s.h, torch.tensor(z0, dtype=torch.float32, device=dev), None)
        for t in range(T):
            geig.geig_step_cca(s.h, x[t * rows:(t + 1) * rows].to(dev).contiguous(),
                               y[t * rows:(t + 1) * rows].to(dev).contiguous(), rows, eta, cfg.gamma)
        Vg, Ag = (t_.double().cpu().numpy() for t_ in s.state())
        zg = torch.empty(k, device=dev)
        geig.geig_smooth_state(s.h, None, zg)
        geig.geig_sync(s.h)
        zg = zg.double().cpu().numpy()
    finally:
        s.close()
    Vo, Ao, Zo = V, aux, z0
    for t in range(T):
        av, bv = estimators.cca_products(x[t * rows:(t + 1) * rows].double().numpy(),
                                         y[t * rows:(t + 1) * rows].double().numpy(), Vo)
        Vo, Ao, Zo = game.step_alg3(Vo, Ao, Zo, [(av, bv)], eta, cfg.gamma, cfg.rho, nu)
    tol = 1e-4 if math == "f32" else 1e-3
    assert rel_err(Vg - V, Vo - V) < tol and row_rel_err(Vg, Vo, V) < tol
    assert rel_err(Ag, Ao) < tol and row_rel_err(Ag, Ao) < tol
    assert rel_err(zg - z0, Zo - z0) < tol


@pytest.mark.parametrize("d,k", [(1000, 97), (517, 128)])
def test_floor_dense_streamed_update_k_over_64(geig, d, k):
    """The streamed update for k > 64 (update_kernel<2>) applies the clip in
    its own coefficient code: fp32 FFMA products, config 4's recipe."""
    from synth import dense_gep_large
    cfg = CONFIGS[4]
    a, b = dense_gep_large(d, seed=2, device="cuda:0")
    dev = "cuda:0"
    rho, eta, gamma = cfg.rho, 0.5, 0.5
    V, aux = floor_state(k, d, 3, rho)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    s = geig.Solver(geig.GEIG_DENSE, d, 0, k, math="f32", rho=rho)
    try:
        s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
        AV = torch.empty(k, d, device=dev)
        BV = torch.empty_like(AV)
        geig.geig_products_dense(s.h, a, b, 0, d, AV, BV)
        geig.geig_update(s.h, AV, BV, eta, gamma)
        V2g, aux2g = (t_.double().cpu().numpy() for t_ in s.state())
    finally:
        s.close()
    av, bv = estimators.dense_products(a.double().cpu().numpy(), b.double().cpu().numpy(), V)
    V2, aux2 = game.step_alg2(V, aux, [(av, bv)], eta, gamma, rho)
    assert sum(float(V[j] @ aux[j]) < rho for j in range(k - 1)) > k // 2
    assert rel_err(V2g - V, V2 - V) < 1e-4 and row_rel_err(V2g, V2, V) < 1e-4
    assert rel_err(aux2g, aux2) < 1e-4 and row_rel_err(aux2g, aux2) < 1e-4
