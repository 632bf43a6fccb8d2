"""GPU parity: the C-ABI CUDA path vs the fp64 oracle, element by element on
identical seeded inputs (-m gpu).  Tolerances (north star): relative 1e-4 for
the fp32 variant, 1e-2 for the bf16 variant; every output is compared
normwise (||got - ref||_F / ||ref||_F), the V update relative to the step
actually taken (||V'_gpu - V'_orc|| / ||V'_orc - V||), which is far stricter
than relative to ||V'||."""
import numpy as np
import pytest
import torch

from tests.gpu_harness import check_cca_step, gram_ref, oracle_cca_step, rel_err, random_state

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


# --- fp32 exactness variant (FFMA) --------------------------------------------

def test_cca_config1_fp32(geig):
    errs, got = check_cca_step(geig, 1, 256)
    _assert(errs, 1e-4)
    assert got["launches"] > 0


@pytest.mark.parametrize("rows,dx,dy,k", [(203, 37, 50, 5), (2, 3, 4, 1), (300, 129, 211, 33),
                                          (130, 300, 301, 64)])
def test_cca_ragged_fp32(geig, rows, dx, dy, k):
    """Ragged tails: odd b (last row unused), d not a multiple of the tiles,
    k crossing the 32-wide Gram tiles, b = 2 (h = 1), k = 1."""
    if dx <= 64 and dy <= 64:
        errs, _ = check_cca_step(geig, 1, rows, k=k, dx=dx, dy=dy)
    else:
        errs = _wide(geig, rows, dx, dy, k)
    _assert(errs, 1e-4)


def _wide(geig, rows, dx, dy, k):
    from synth import CONFIGS, cca_views
    from tests.gpu_harness import oracle_cca_step, run_gpu_cca_step, gram_ref
    cfg = CONFIGS[1]
    # a wider gaussian-view problem with the config-1 recipe: widen W by tiling seeds
    x1, y1 = cca_views(cfg, rows, seed=11)
    x2, y2 = cca_views(cfg, rows, seed=12)
    xs = torch.cat([x1, y1, x2, y2] * 3, 1)[:, :dx].contiguous()
    ys = torch.cat([y2, x2, y1, x1] * 3, 1)[:, :dy].contiguous()
    d = dx + dy
    V, aux = random_state(k, d, 3)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    got = run_gpu_cca_step(geig, xs, ys, V, aux, k, dx, dy, "f32", 0.05, 0.7, cfg.rho, 0)
    av, bv, V2, aux2 = oracle_cca_step(xs.double().numpy(), ys.double().numpy(), V, aux, 0.05, 0.7, cfg.rho)
    ga, gb, gc = gram_ref(V, aux, av, bv)
    return dict(av=rel_err(got["av"], av), bv=rel_err(got["bv"], bv), ga=rel_err(got["ga"], ga),
                gb=rel_err(got["gb"], gb), gc=rel_err(got["gc"], gc), step=rel_err(got["V"] - V, V2 - V),
                aux=rel_err(got["aux"], aux2),
                sphere=float(np.max(np.abs(np.linalg.norm(got["V"], axis=1) - 1))))


def test_cca_config2_bf16_data_fp32_math(geig):
    errs, _ = check_cca_step(geig, 2, 1024)
    _assert(errs, 1e-4)


def test_cca_config3_full_size_fp32_math(geig):
    """Config 3 at full size (dx=dy=8192, b=4096, k=64, bf16 data): one step
    through the FFMA exactness path vs the fp64 oracle.  eta = 0.02 (not the
    config's 1e-4): at 1e-4 the step (~0.1 of |V|) is resolved only to
    ~1.4e-4 by the fp32 storage of V' itself."""
    errs, _ = check_cca_step(geig, 3, 4096, eta=0.02)
    _assert(errs, 1e-4)


def test_dense_config0_trajectory(geig):
    """Config 0: per-step parity along the oracle's own trajectory (each GPU
    step starts from the oracle state) and convergence of the GPU iteration
    itself to the exact generalized eigenvectors (< 1e-3 rad)."""
    from oracle import estimators, game, linalg, metrics
    from synth import CONFIGS, dense_gep_small, gaussian_init
    cfg = CONFIGS[0]
    a, b = dense_gep_small(0)
    w, Vt = linalg.generalized_eigh(a, b, cfg.k)
    dev = "cuda:0"
    A = torch.tensor(a, dtype=torch.float32, device=dev)
    B = torch.tensor(b, dtype=torch.float32, device=dev)
    a32, b32 = A.double().cpu().numpy(), B.double().cpu().numpy()
    s = geig.Solver(geig.GEIG_DENSE, cfg.d, 0, cfg.k, math="f32", rho=cfg.rho)
    try:
        G = torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev)
        s.init_state(G)
        V0, aux0 = s.state()
        Vo, auxo = V0.double().cpu().numpy(), aux0.double().cpu().numpy()
        worst = 0.0
        for t in range(60):
            s.set_state(torch.tensor(Vo, dtype=torch.float32, device=dev),
                        torch.tensor(auxo, dtype=torch.float32, device=dev))
            geig.geig_step_dense(s.h, A, B, cfg.eta, cfg.gamma)
            Vg, auxg = s.state()
            Vo32 = Vo.astype(np.float32).astype(np.float64)
            auxo32 = auxo.astype(np.float32).astype(np.float64)
            av, bv = estimators.dense_products(a32, b32, Vo32)
            V2, aux2 = game.step_alg2(Vo32, auxo32, [(av, bv)], cfg.eta, cfg.gamma, cfg.rho)
            worst = max(worst, rel_err(Vg.double().cpu().numpy() - Vo32, V2 - Vo32),
                        rel_err(auxg.double().cpu().numpy(), aux2))
            Vo, auxo = V2, aux2
        assert worst < 1e-4
        # the GPU's own trajectory converges
        s.init_state(G)
        for t in range(cfg.steps):
            geig.geig_step_dense(s.h, A, B, cfg.eta, cfg.gamma)
        Vg, _ = s.state()
        ang = metrics.per_vector_angles(Vg.double().cpu().numpy(), Vt)
        assert np.all(ang < 1e-3), ang
    finally:
        s.close()


def test_init_state_matches_alg2_lines_2_3(geig):
    from oracle import game
    from synth import gaussian_init
    g = gaussian_init(7, 333, 5)
    s = geig.Solver(geig.GEIG_DENSE, 333, 0, 7, math="f32", rho=0.1)
    try:
        s.init_state(torch.tensor(g, dtype=torch.float32, device="cuda:0"))
        V, aux = s.state()
        Vo, auxo = game.init_state(g.astype(np.float32).astype(np.float64))
        assert rel_err(V.cpu().numpy(), Vo) < 1e-6 and rel_err(aux.cpu().numpy(), auxo) < 1e-6
    finally:
        s.close()


@pytest.mark.parametrize("d,k", [(333, 65), (1030, 97), (517, 128)])
def test_dense_streamed_update_k_over_64_fp32(geig, d, k):
    """The streamed update (k > 64, `update_kernel<2>`): the penalty sums
    sum_{j<i} L_ij [Bv]_j split over thread pairs (row groups q and 31 - q,
    alternating 4-blocks of j, shuffle-combined) — k not a multiple of 4
    (rows past k), k = 128, d not a multiple of the 32-column sub-chunk;
    fp32 FFMA products, so the step is held to the fp32 bar (PAPER.md:1017-1025,
    Alg. 2 l.12-19)."""
    from synth import dense_gep_small
    a, b = dense_gep_small(seed=3, d=d)
    _dense_step_check(geig, a, b, k, "f32", 0.1, 0.05, 0.5, seed=1, tol=1e-4)


def test_errors_are_loud(geig):
    with pytest.raises(geig.GeigError):
        geig.geig_create(geig.GEIG_CCA, 0, 4, 2, 0, 0, 0.1, 8, 0)
    with pytest.raises(geig.GeigError):
        geig.geig_create(geig.GEIG_CCA, 4, 4, 2, 0, 0, 0.1, 1, 0)
    s = geig.Solver(geig.GEIG_CCA, 4, 4, 2, math="f32", rho=0.1, max_rows=8)
    x = torch.zeros(16, 4, device="cuda:0")
    AV = torch.zeros(2, 8, device="cuda:0")
    with pytest.raises(geig.GeigError):
        geig.geig_products_cca(s.h, x, x, 16, 1.0, AV, AV)      # b > max_rows
    s.close()
    # unbuilt arithmetic variants are refused at creation, never silently wrong
    with pytest.raises(geig.GeigError, match="fp32 data"):
        geig.geig_create(geig.GEIG_CCA, 64, 64, 4, geig.GEIG_MATH_3XTF32, geig.GEIG_DATA_BF16, 0.1, 64, 0)
    with pytest.raises(geig.GeigError, match="fp32 data"):
        geig.geig_create(geig.GEIG_CCA, 64, 64, 4, geig.GEIG_MATH_TF32, geig.GEIG_DATA_BF16, 0.1, 64, 0)


# --- tensor-core variants (tcgen05): bf16 1e-2, tf32 1e-2 ---------------------

def test_cca_config2_bf16_tcgen05(geig):
    errs, got = check_cca_step(geig, 2, 1024, math="bf16")
    _assert(errs, 1e-2)


def test_cca_config3_full_size_bf16_tcgen05(geig):
    """Config 3 at full size, plain bf16 operands, through the products
    launch + update launch (AV, BV compared too).  The configuration
    bench.py times — bf16x2, geig_run_cca, CTA pairs — is held to the oracle
    by test_run_cca_matches_single_steps_and_oracle[bf16x2-3-4096-...] and
    test_fused_pairs_match_single_ctas."""
    errs, _ = check_cca_step(geig, 3, 4096, math="bf16")
    _assert(errs, 1e-2)


@pytest.mark.parametrize("rows,dx,dy,k", [(300, 200, 136, 24), (130, 64, 8, 5), (1000, 784, 784, 16),
                                          (258, 2048, 1024, 128)])
def test_cca_ragged_bf16_tcgen05(geig, rows, dx, dy, k):
    """Ragged for the TMA tiles: h not a multiple of 64 (zero-filled K tail),
    d not a multiple of 128 (masked M tail), k not a multiple of 16 (N pad),
    k = 128 (largest tile)."""
    cfg_idx = 2 if max(dx, dy) <= 784 else 3
    errs, _ = check_cca_step(geig, cfg_idx, rows, k=k, dx=dx, dy=dy, math="bf16")
    _assert(errs, 1e-2)


def _dense_step_check(geig, a, b, k, math, rho, eta, gamma, seed=0, tol=1e-2):
    """One dense step (products + update) vs the oracle.  eta = "auto":
    0.1 / max_i ||grad_i|| from the oracle's own Alg. 2 directions — the step
    is then ~0.1 of |v_i|, so fp32 storage of V' (6e-8 relative) resolves it
    to ~1e-6, and the comparison measures the direction's arithmetic (the
    step's cost and arithmetic do not depend on eta except the final axpy)."""
    from oracle import estimators, game
    dev = "cuda:0"
    d = a.shape[0]
    A = a.to(dev).float().contiguous() if isinstance(a, torch.Tensor) else torch.tensor(a, dtype=torch.float32, device=dev)
    B = b.to(dev).float().contiguous() if isinstance(b, torch.Tensor) else torch.tensor(b, dtype=torch.float32, device=dev)
    V, aux = random_state(k, d, seed)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    if isinstance(eta, str):
        a64, b64 = A.double().cpu().numpy(), B.double().cpu().numpy()
        av0, bv0 = estimators.dense_products(a64, b64, V)
        gmax = max(np.linalg.norm(game.direction_alg2(i, V, aux, av0, bv0, rho)) for i in range(k))
        eta = 0.1 / gmax
    s = geig.Solver(geig.GEIG_DENSE, d, 0, k, math=math, rho=rho)
    try:
        s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
        AV = torch.empty(k, d, device=dev)
        BV = torch.empty_like(AV)
        geig.geig_products_dense(s.h, A, B, 0, d, AV, BV)
        geig.geig_update(s.h, AV, BV, eta, gamma)
        V2g, aux2g = s.state()
        a64, b64 = A.double().cpu().numpy(), B.double().cpu().numpy()
        av, bv = estimators.dense_products(a64, b64, V)
        V2, aux2 = game.step_alg2(V, aux, [(av, bv)], eta, gamma, rho)
        errs = dict(av=rel_err(AV.double().cpu().numpy(), av), bv=rel_err(BV.double().cpu().numpy(), bv),
                    step=rel_err(V2g.double().cpu().numpy() - V, V2 - V),
                    aux=rel_err(aux2g.double().cpu().numpy(), aux2), sphere=0.0)
    finally:
        s.close()
    _assert(errs, tol)
    return errs


@pytest.mark.parametrize("cfg_idx,rows,k,dx,dy", [(1, 256, None, None, None), (2, 300, 24, 200, 136),
                                                  (2, 1024, 16, 784, 784), (3, 2048, 64, 1024, 512),
                                                  (2, 130, 5, 64, 8)])
def test_cca_tf32_tcgen05(geig, monkeypatch, cfg_idx, rows, k, dx, dy):
    """fp32 data on the tf32 tensor cores (staged path): forward K-major, the
    backward's X^T an MN-major tf32 operand (TMA 128B/32B-chunk swizzle,
    descriptor layout SWIZZLE_128B_BASE32B).  tf32 keeps 10 mantissa bits:
    the 1e-2 tensor-core bar; measured ~7e-4."""
    import tests.gpu_harness as gh
    cv = gh.cca_views
    monkeypatch.setattr(gh, "cca_views", lambda *a, **kw: tuple(t.float() for t in cv(*a, **kw)))
    errs, _ = gh.check_cca_step(geig, cfg_idx, rows, k=k, dx=dx, dy=dy, math="tf32")
    _assert(errs, 1e-2)
    assert errs["av"] < 3e-3 and errs["bv"] < 3e-3, errs


@pytest.mark.parametrize("cfg_idx,rows,k,dx,dy,eta", [(1, 256, None, None, None, None),
                                                      (2, 1024, 16, 784, 784, None),
                                                      (3, 2048, 64, 1024, 512, 0.02),
                                                      (2, 300, 24, 200, 136, 0.5), (2, 130, 5, 64, 8, 0.5)])
def test_cca_3xtf32_tcgen05(geig, monkeypatch, cfg_idx, rows, k, dx, dy, eta):
    """3xTF32: A split in shared memory into tf32 hi + lo by warps 2-3, B as
    hi / lo planes, three MMAs per K step (a_lo b_lo dropped): the fp32
    exactness bar of the FFMA variant on the configs (1e-4 everywhere),
    products, Gram tables and aux ~1e-6 (bar 1e-5) on all shapes.  On the
    tiny ragged shapes the step (a difference of O(1) terms, cancellation
    ~100-200x at a random state) gets the bf16x2 bar of 1e-3."""
    import tests.gpu_harness as gh
    cv = gh.cca_views
    monkeypatch.setattr(gh, "cca_views", lambda *a, **kw: tuple(t.float() for t in cv(*a, **kw)))
    errs, _ = gh.check_cca_step(geig, cfg_idx, rows, k=k, dx=dx, dy=dy, math="3xtf32", eta=eta)
    step = errs.pop("step")
    _assert(errs, 1e-5)
    assert step < (1e-3 if rows < 500 else 1e-4), (step, errs)   # tiny ragged shapes: the bf16x2 step bar


def test_dense_config0_3xtf32_tcgen05(geig):
    from synth import CONFIGS, dense_gep_small
    cfg = CONFIGS[0]
    a, b = dense_gep_small(0)
    errs = _dense_step_check(geig, a, b, cfg.k, "3xtf32", cfg.rho, cfg.eta, cfg.gamma, tol=1e-4)
    assert errs["av"] < 1e-5 and errs["bv"] < 1e-5, errs


def test_dense_config4_reduced_3xtf32_tcgen05(geig):
    """Config 4's recipe at d = 1000 (ragged tiles), k = 37, 3xTF32 (eta as
    in the fp32 test: the step must dominate the fp32 storage of V')."""
    from synth import CONFIGS, dense_gep_large
    cfg = CONFIGS[4]
    a, b = dense_gep_large(1000, seed=2, device="cuda:0")
    errs = _dense_step_check(geig, a, b, 37, "3xtf32", cfg.rho, 0.5, cfg.gamma, tol=1e-4)
    assert errs["av"] < 1e-5 and errs["bv"] < 1e-5, errs


def test_dense_config0_tf32_tcgen05(geig):
    from synth import CONFIGS, dense_gep_small
    cfg = CONFIGS[0]
    a, b = dense_gep_small(0)
    _dense_step_check(geig, a, b, cfg.k, "tf32", cfg.rho, cfg.eta, cfg.gamma)


def test_dense_config4_reduced_fp32(geig):
    from synth import CONFIGS, dense_gep_large
    cfg = CONFIGS[4]
    a, b = dense_gep_large(1000, seed=2, device="cuda:0")
    # eta = 0.5 so that the step (eta ||grad|| ~ 2e-2 ||V||) is resolved by
    # fp32 storage of V'; with the config's eta the fp32 rounding of V' alone
    # is 1.6e-4 of the step
    _dense_step_check(geig, a, b, 37, "f32", cfg.rho, 0.5, cfg.gamma, tol=1e-4)


def test_dense_config4_full_size_tf32_tcgen05(geig):
    """Config 4 at full size: d = 16384, k = 128, TF32 tensor cores."""
    from synth import CONFIGS, dense_gep_large
    cfg = CONFIGS[4]
    a, b = dense_gep_large(cfg.d, seed=0, device="cuda:0")
    _dense_step_check(geig, a, b, cfg.k, "tf32", cfg.rho, cfg.eta, cfg.gamma)


@pytest.mark.parametrize("math", ["3xtf32", "f32"])
def test_dense_config4_full_size_fp32_variant(geig, math):
    """Config 4 at full size (d = 16384, k = 128) in the fp32 variants —
    3xTF32 tensor cores (the products launch splits K in 4: 2 x 128 M tiles on
    148 SMs fill 7 waves instead of 2, atomic epilogue into the zeroed AV / BV
    rows) and FFMA — held to the north star's 1e-4 with eta = "auto" (the
    step resolved by fp32 storage, see _dense_step_check)."""
    from synth import CONFIGS, dense_gep_large
    cfg = CONFIGS[4]
    a, b = dense_gep_large(cfg.d, seed=1, device="cuda:0")
    _dense_step_check(geig, a, b, cfg.k, math, cfg.rho, "auto", cfg.gamma, tol=1e-4)


@pytest.mark.parametrize("math,tol", [("f32", 1e-5), ("3xtf32", 1e-5), ("tf32", 3e-3)])
@pytest.mark.parametrize("d,k,nshards", [(1000, 37, 3), (1000, 128, 2), (516, 64, 3), (517, 5, 3)])
def test_dense_row_shards_assemble_the_products(geig, math, tol, d, k, nshards):
    """Config 4's multi-GPU form on one GPU: A and B row-sharded
    (shard_rows: ragged, r0 > 0), each shard's geig_products_dense writes its
    columns [r0, r1) of AV, BV (the symmetric A's rows r0..r1 times every
    v_j), and the assembled products equal the oracle's A v_j, B v_j
    (Alg. 1 full batch; BASELINE config 4)."""
    from oracle import estimators
    from paper_2206_04993_b200.parallel import shard_rows
    from synth import CONFIGS, dense_gep_large
    if math != "f32" and d % 4:
        pytest.skip("the tensor-core path needs d % 4 == 0 (TMA 16-byte row strides); refused loudly")
    cfg = CONFIGS[4]
    dev = "cuda:0"
    a, b = dense_gep_large(d, seed=4, device=dev)
    V, aux = random_state(k, d, 6)
    V = V.astype(np.float32).astype(np.float64)
    s = geig.Solver(geig.GEIG_DENSE, d, 0, k, math=math, rho=cfg.rho)
    try:
        s.set_state(torch.tensor(V, dtype=torch.float32, device=dev))
        AV = torch.full((k, d), float("nan"), device=dev)
        BV = torch.full_like(AV, float("nan"))
        for r in range(nshards):
            r0, r1 = shard_rows(d, nshards, r)
            geig.geig_products_dense(s.h, a[r0:r1].contiguous(), b[r0:r1].contiguous(), r0, r1, AV, BV)
        geig.geig_sync(s.h)
    finally:
        s.close()
    av, bv = estimators.dense_products(a.double().cpu().numpy(), b.double().cpu().numpy(), V)
    ea, eb = rel_err(AV.double().cpu().numpy(), av), rel_err(BV.double().cpu().numpy(), bv)
    assert ea < tol and eb < tol, (ea, eb)


# --- the fused single-launch step (geig_step_cca on the bf16 path) -------------

@pytest.mark.parametrize("cfg_idx,rows,k,dx,dy", [(3, 4096, None, None, None), (2, 1024, None, None, None),
                                                  (2, 300, 24, 200, 136), (2, 130, 5, 64, 8),
                                                  (3, 1000, 64, 8192, 4096), (3, 2048, 32, 1024, 512),
                                                  (3, 1024, 64, 2048, 1024), (3, 512, 48, 256, 384)])
def test_fused_step_bf16(geig, cfg_idx, rows, k, dx, dy):
    """geig_step_cca runs forward GEMM, split-K reduction, backward GEMM, Gram
    tables and the update in ONE cooperative kernel; the step must match the
    oracle like the staged path."""
    errs, _ = check_cca_step(geig, cfg_idx, rows, k=k, dx=dx, dy=dy, math="bf16", use_step=True)
    _assert(errs, 1e-2)


@pytest.mark.parametrize("cfg_idx,rows,k,dx,dy,math", [(2, 1100, 24, 600, 328, "bf16"),
                                                       (2, 1200, 64, 400, 272, "bf16x2"),
                                                       (3, 4096, 16, 8192, 8192, "bf16x2")])
@pytest.mark.parametrize("tm", ["1", "2"])
def test_fused_step_forced_m_tiles(geig, cfg_idx, rows, k, dx, dy, math, tm):
    """Work items of two 128-row M tiles sharing each B-operand tile (the
    default at full size) and of one, forced on ragged shapes: a last item
    with a partial second M tile, a last item with a single M tile."""
    errs, _ = check_cca_step(geig, cfg_idx, rows, k=k, dx=dx, dy=dy, math=math, use_step=True,
                             options={geig.GEIG_OPT_FUSED_M_TILES: int(tm)})
    if math == "bf16":
        _assert(errs, 1e-2)
    else:
        step = errs.pop("step")
        _assert(errs, 1e-4)
        assert step < 1e-3, errs


def test_fused_step_matches_staged_path(geig):
    """Same inputs through the staged path (products + update) and the fused
    kernel: the states agree to bf16-product rounding order."""
    e1, g1 = check_cca_step(geig, 2, 1024, math="bf16", use_step=True)
    e2, g2 = check_cca_step(geig, 2, 1024, math="bf16", use_step=False)
    assert rel_err(g1["V"] - g2["V"] + 1.0, np.ones_like(g2["V"])) < 1e-3
    assert rel_err(g1["aux"], g2["aux"]) < 1e-3


# --- bf16x2: V and Z split into hi + lo bf16 operands (exact bf16 data) ------

@pytest.mark.parametrize("cfg_idx,rows,k,dx,dy,use_step", [(3, 4096, None, None, None, False),
                                                           (3, 4096, None, None, None, True),
                                                           (2, 1024, None, None, None, True),
                                                           (2, 300, 24, 200, 136, False)])
def test_bf16x2_fp32_level_parity(geig, cfg_idx, rows, k, dx, dy, use_step):
    """With the bf16 data exact and the V / Z operands carried as hi+lo bf16
    pairs, the tensor-core products, Gram tables and aux reach the fp32
    exactness-variant bar (1e-4); the step (a difference of O(1) terms,
    cancellation ~100x at a random state) gets 1e-3 — vs 1e-2 for plain bf16."""
    errs, _ = check_cca_step(geig, cfg_idx, rows, k=k, dx=dx, dy=dy, math="bf16x2", use_step=use_step)
    step = errs.pop("step")
    _assert(errs, 1e-4)
    assert step < 1e-3, errs


# --- Alg. 2's loop in one launch (geig_run_cca) --------------------------------

@pytest.mark.parametrize("math,cfg_idx,rows,k,dx,dy", [("bf16x2", 3, 4096, None, None, None),
                                                       ("bf16", 2, 1000, None, None, None),
                                                       ("bf16x2", 2, 300, 24, 200, 136)])
def test_run_cca_matches_single_steps_and_oracle(geig, math, cfg_idx, rows, k, dx, dy):
    """geig_run_cca (T steps in one persistent launch, distinct and repeated
    batches) leaves exactly the state of T geig_step_cca calls (same kernel
    code, deterministic reductions: bit-identical), and that state matches T
    oracle steps of Alg. 2."""
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[cfg_idx]
    k = k or cfg.k
    dx, dy = dx or cfg.dx, dy or cfg.dy
    T = 4
    x, y = cca_views(cfg, 2 * rows, seed=11)
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    batches = [(x[:rows], y[:rows]), (x[rows:], y[rows:]), (x[:rows], y[:rows]), (x[rows:], y[rows:])]
    V, aux = random_state(k, dx + dy, 3)
    V32 = V.astype(np.float32).astype(np.float64)
    aux32 = aux.astype(np.float32).astype(np.float64)
    flag = 1 if x.dtype == torch.bfloat16 else 0
    eta, gamma = cfg.eta, cfg.gamma
    dev = "cuda:0"
    Xd = [b_[0].to(dev).contiguous() for b_ in batches]
    Yd = [b_[1].to(dev).contiguous() for b_ in batches]
    states = []
    for run in (True, False):
        s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math=math, data_dtype=flag, rho=cfg.rho, max_rows=rows)
        try:
            s.set_state(torch.tensor(V32, dtype=torch.float32, device=dev),
                        torch.tensor(aux32, dtype=torch.float32, device=dev))
            if run:
                l0 = s.launches()
                geig.geig_run_cca(s.h, Xd, Yd, rows, eta, gamma)
                assert s.launches() - l0 == 1      # T steps, one persistent launch
            else:
                for t in range(T):
                    geig.geig_step_cca(s.h, Xd[t], Yd[t], rows, eta, gamma)
            Vg, Ag = s.state()
            states.append((Vg.cpu().numpy(), Ag.cpu().numpy()))
        finally:
            s.close()
    assert np.array_equal(states[0][0], states[1][0]) and np.array_equal(states[0][1], states[1][1])
    # oracle: T steps of Alg. 2 in fp64 on the same batches
    Vo, Ao = V32, aux32
    for t in range(T):
        _, _, Vo, Ao = oracle_cca_step(batches[t][0].double().numpy(), batches[t][1].double().numpy(), Vo, Ao,
                                       eta, gamma, cfg.rho)
    tol = 1e-2 if math == "bf16" else 1e-3
    assert rel_err(states[0][0] - V32, Vo - V32) < tol
    assert rel_err(states[0][1], Ao) < tol


def test_staged_tensor_core_products_still_match(geig):
    """geig_products_cca uses phases F, S, B of the fused kernel; the staged
    three-launch products (tc_gemm forward, zshuffle, tc_gemm backward — the
    path for k > 64 or d % 4 != 0, selected here with GEIG_OPT_STAGED_PRODUCTS)
    stay covered here."""
    for math, tol in (("bf16", 1e-2), ("bf16x2", 1e-3)):
        errs, _ = check_cca_step(geig, 3, 1024, k=64, dx=2048, dy=1024, math=math,
                                 options={geig.GEIG_OPT_STAGED_PRODUCTS: 1})
        _assert(errs, tol)


# --- multi-GPU form: products + Gram tables aggregated across ranks -------------

@pytest.mark.parametrize("math,tol_p,tol_s,k,dx,dy,rows", [("bf16x2", 1e-4, 1e-3, 16, 784, 784, 512),
                                                           ("bf16", 1e-2, 1e-2, 16, 784, 784, 512),
                                                           ("bf16x2", 1e-4, 1e-3, 24, 200, 136, 301),
                                                           ("bf16x2", 1e-4, 1e-3, 5, 64, 8, 130)])
def test_products_tables_two_shards_match_appendix_f(geig, math, tol_p, tol_s, k, dx, dy, rows):
    """Appendix F on one GPU: two row shards through
    geig_products_cca_tables (scale 1/(M h)), their products AND table partials
    summed (the all-reduce), then geig_update_tables — vs the oracle's
    aggregated-products step.  The tables (G^A, G^B of each shard's rows) must
    aggregate like the products."""
    from oracle import estimators, game
    from synth import CONFIGS, cca_views
    from paper_2206_04993_b200.parallel import product_buffers
    cfg = CONFIGS[2]
    M = 2
    x, y = cca_views(cfg, M * rows, seed=3)
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    d = dx + dy
    V, aux = random_state(k, d, 5)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    dev = "cuda:0"
    s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math=math, data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho, max_rows=rows)
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
        geig.geig_update_tables(s.h, AV, BV, T, cfg.eta, cfg.gamma)
        V2g, aux2g = s.state()
        ga, gb, gc = s.gram()
    finally:
        s.close()
    x64, y64 = x.double().numpy(), y.double().numpy()
    machines = [estimators.cca_products(x64[:rows], y64[:rows], V), estimators.cca_products(x64[rows:], y64[rows:], V)]
    V2, aux2 = game.step_alg2_appendix_f(V, aux, machines, cfg.eta, cfg.gamma, cfg.rho)
    av = sum(m[0] for m in machines) / M
    bv = sum(m[1] for m in machines) / M
    ga_r, gb_r, gc_r = gram_ref(V, aux, av, bv)
    errs = dict(av=rel_err(AV.double().cpu().numpy(), av), bv=rel_err(BV.double().cpu().numpy(), bv),
                ga=rel_err(ga.double().cpu().numpy(), ga_r), gb=rel_err(gb.double().cpu().numpy(), gb_r),
                gc=rel_err(gc.double().cpu().numpy(), gc_r), aux=rel_err(aux2g.double().cpu().numpy(), aux2))
    step = rel_err(V2g.double().cpu().numpy() - V, V2 - V)
    _assert(dict(errs, sphere=0.0), tol_p)
    assert step < tol_s, (step, errs)


@pytest.mark.parametrize("variant", ["alg2", "alg3", "adam"])
def test_products_tables_single_shard_equals_fused_step(geig, variant):
    """One rank: geig_products_cca_tables + geig_update_tables reproduce the
    fused single-launch step (same products, same tables, same update), for
    Alg. 2, Alg. 3 (smooth denominators) and Adam ascent, over 3 steps."""
    from synth import CONFIGS, cca_views
    from paper_2206_04993_b200.parallel import product_buffers
    cfg = CONFIGS[3]
    rows = 4096
    x, y = cca_views(cfg, rows, seed=7)
    V, aux = random_state(cfg.k, cfg.d, 2)
    dev = "cuda:0"
    out = []
    for mode in ("fused", "tables"):
        s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16,
                        rho=cfg.rho, max_rows=rows)
        try:
            # one CTA per item: the tables path's column partition (CTA pairs
            # re-partition the update's columns: test_fused_pairs_match_single_ctas)
            geig.geig_set_option(s.h, geig.GEIG_OPT_FUSED_PAIRS, 0)
            s.set_state(torch.tensor(V, dtype=torch.float32, device=dev),
                        torch.tensor(aux, dtype=torch.float32, device=dev))
            if variant == "alg3":
                geig.geig_set_smooth(s.h, 10.0)
            if variant == "adam":
                geig.geig_set_adam(s.h, 0.9, 0.999, 1e-8)
            xd, yd = x.to(dev), y.to(dev)
            for _ in range(3):
                if mode == "fused":
                    geig.geig_step_cca(s.h, xd, yd, rows, cfg.eta, cfg.gamma)
                else:
                    AV, BV, T = product_buffers(cfg.k, cfg.d, geig.geig_table_floats(s.h), device=dev)
                    geig.geig_products_cca_tables(s.h, xd, yd, rows, 1.0 / (rows // 2), AV, BV, T)
                    geig.geig_update_tables(s.h, AV, BV, T, cfg.eta, cfg.gamma)
            out.append([t.double().cpu().numpy() for t in s.state()])
        finally:
            s.close()
    (Vf, af), (Vt, at) = out
    assert rel_err(Vt - V, Vf - V) < 1e-5
    assert rel_err(at, af) < 1e-6


def test_mixed_call_sequence_keeps_the_launch_counters_consistent(geig):
    """The fused launches of a solver count the Gram reduction on a
    monotonic counter (early coefficients in phase B).  An arbitrary mix of
    single steps, multi-step launches, the multi-GPU tables path, standalone
    updates, state resets and stream switches must neither hang nor drift:
    two solvers driven by the same sequence end bit-identical, and the
    fused single step still matches the oracle afterwards."""
    from synth import CONFIGS, cca_views
    from paper_2206_04993_b200.parallel import product_buffers
    cfg = CONFIGS[2]
    k, dx, dy, rows = 16, 784, 784, 512
    x, y = cca_views(cfg, 4 * rows, seed=9)
    dev = "cuda:0"
    xs = [x[i * rows:(i + 1) * rows].to(dev).contiguous() for i in range(4)]
    ys = [y[i * rows:(i + 1) * rows].to(dev).contiguous() for i in range(4)]
    V, aux = random_state(k, dx + dy, 4)
    outs = []
    for rep in range(2):
        s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho,
                        max_rows=rows)
        try:
            Vd = torch.tensor(V, dtype=torch.float32, device=dev)
            Ad = torch.tensor(aux, dtype=torch.float32, device=dev)
            s.set_state(Vd, Ad)
            geig.geig_step_cca(s.h, xs[0], ys[0], rows, cfg.eta, cfg.gamma)
            geig.geig_run_cca(s.h, xs[:3], ys[:3], rows, cfg.eta, cfg.gamma)
            AV, BV, T = product_buffers(k, dx + dy, geig.geig_table_floats(s.h), device=dev)
            geig.geig_products_cca_tables(s.h, xs[1], ys[1], rows, 1.0 / (rows // 2), AV, BV, T)
            geig.geig_update_tables(s.h, AV, BV, T, cfg.eta, cfg.gamma)
            geig.geig_products_cca(s.h, xs[2], ys[2], rows, 1.0 / (rows // 2), AV, BV)
            geig.geig_update(s.h, AV, BV, cfg.eta, cfg.gamma)
            side = torch.cuda.Stream()
            geig.geig_set_stream(s.h, side.cuda_stream)
            geig.geig_run_cca(s.h, xs[1:4], ys[1:4], rows, cfg.eta, cfg.gamma)
            geig.geig_set_stream(s.h, torch.cuda.current_stream().cuda_stream)
            geig.geig_step_cca(s.h, xs[3], ys[3], rows, cfg.eta, cfg.gamma)
            outs.append([t.double().cpu().numpy() for t in s.state()])
        finally:
            s.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    errs, _ = check_cca_step(geig, 2, rows, k=k, dx=dx, dy=dy, math="bf16x2", use_step=True)
    step = errs.pop("step")
    _assert(errs, 1e-4)
    assert step < 1e-3


def _fuzz_cases(n=12, seed=2024):
    rng = np.random.default_rng(seed)
    cases = []
    for _ in range(n):
        k = int(rng.integers(1, 65))
        dx = int(rng.integers(1, 99)) * 8
        dy = int(rng.integers(1, 99)) * 8
        rows = int(rng.integers(2, 2600))
        math = "bf16x2" if rng.random() < 0.7 else "bf16"
        cases.append((k, dx, dy, rows, math))
    return cases


@pytest.mark.parametrize("k,dx,dy,rows,math", _fuzz_cases())
def test_fused_step_random_shapes(geig, k, dx, dy, rows, math):
    """Seeded random shapes through the fused single-launch step (k <= 64,
    d % 8 == 0, any b >= 2: ragged M tiles, odd b, k not a multiple of 16,
    split-K over few K blocks, the per-tile dependency counters) vs the
    fp64 oracle."""
    from synth import CONFIGS
    cfg = CONFIGS[2]
    if dx > cfg.dx or dy > cfg.dy:   # config 2's generator draws 784-column views
        pytest.skip("views wider than the recipe")
    errs, _ = check_cca_step(geig, 2, rows, k=k, dx=dx, dy=dy, math=math, use_step=True, eta=0.5)
    if math == "bf16":
        _assert(errs, 1e-2)
    else:
        step = errs.pop("step")
        _assert(errs, 1e-4)
        assert step < 1e-3, errs


def test_run_cca_large_batch_long_run_is_deterministic(geig):
    """Regression: the multi-step launch's phase-U tile barrier used to live
    in the smem ring (a TMA destination of phases F and B); re-initialising it
    there let phase U read partially landed tiles about once per 10^4 steps
    (non-finite v'' at b = 100k, config 1).  Two identical runs of 2000 steps
    in launches of 100 must stay finite and bit-identical."""
    from synth import CONFIGS, cca_views, gaussian_init
    cfg = CONFIGS[1]
    n, dx, k = 100_000, 64, 8
    x, y = cca_views(cfg, n, seed=3)
    x, y = x.to(torch.bfloat16).contiguous().cuda(), y.to(torch.bfloat16).contiguous().cuda()
    out = []
    for _ in range(2):
        s = geig.Solver(geig.GEIG_CCA, dx, dx, k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho,
                        max_rows=n)
        try:
            s.init_state(torch.tensor(gaussian_init(k, 2 * dx, 0), dtype=torch.float32, device="cuda:0"))
            for _ in range(20):
                geig.geig_run_cca(s.h, [x] * 100, [y] * 100, n, 0.0086, 1.0)
            out.append([t_.cpu() for t_ in s.state()])
        finally:
            s.close()
    assert all(torch.isfinite(t_).all() for t_ in out[0] + out[1])
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])


@pytest.mark.parametrize("variant", ["alg2", "alg3", "adam", "run"])
def test_fused_pairs_match_single_ctas(geig, variant):
    """The fused step on CTA pairs (thread-block clusters of 2: backward
    accumulators exchanged through distributed shared memory into the
    update's tiles, 128 update columns per CTA) against one CTA per item
    (AV, BV through global memory, 112 columns per CTA) over 3 steps at
    config 3: the same arithmetic up to the order of the Gram partial sums."""
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[3]
    rows = 4096
    x, y = cca_views(cfg, 2 * rows, seed=17)
    V, aux = random_state(cfg.k, cfg.d, 12)
    dev = "cuda:0"
    xs = [x[:rows].to(dev), x[rows:].to(dev), x[:rows].to(dev)]
    ys = [y[:rows].to(dev), y[rows:].to(dev), y[:rows].to(dev)]
    eta = 0.02
    out = []
    for pairs in (1, 0):
        s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16,
                        rho=cfg.rho, max_rows=rows)
        try:
            geig.geig_set_option(s.h, geig.GEIG_OPT_FUSED_PAIRS, pairs)
            s.set_state(torch.tensor(V, dtype=torch.float32, device=dev),
                        torch.tensor(aux, dtype=torch.float32, device=dev))
            if variant == "alg3":
                geig.geig_set_smooth(s.h, 10.0)
            if variant == "adam":
                geig.geig_set_adam(s.h, 0.9, 0.999, 1e-8)
            if variant == "run":
                geig.geig_run_cca(s.h, xs, ys, rows, eta, cfg.gamma)
            else:
                for t in range(3):
                    geig.geig_step_cca(s.h, xs[t], ys[t], rows, eta, cfg.gamma)
            out.append([t.double().cpu().numpy() for t in s.state()])
        finally:
            s.close()
    (Vp, ap), (Vs, as_) = out
    step, aux_e = rel_err(Vp - V, Vs - V), rel_err(ap, as_)
    assert step < 1e-5 and aux_e < 1e-5, (step, aux_e)


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("d,k", [(4096, 128), (3000, 100), (16384, 128)])
def test_gram_tensor_cores_match_ffma_gram(geig, math, d, k):
    """The streamed (k > 64) update's Gram tables G^A, G^C on the tensor
    cores (GEIG_OPT_GRAM_TC, split-K partial rows, one per update CTA)
    against the FFMA Gram of the update kernel, from the same products: the
    tables (geig_get_gram) and the step agree to the Gram arithmetic's
    precision (3xTF32: fp32 level; tf32: 10-bit operands), and the
    3xTF32 step matches the oracle at the fp32 bar (1e-4)."""
    from oracle import estimators, game
    from synth import dense_gep_large
    dev = "cuda:0"
    a, b = dense_gep_large(d, seed=3, device=dev)
    V, aux = random_state(k, d, 5)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    a64, b64 = a.double().cpu().numpy(), b.double().cpu().numpy()
    av0, bv0 = estimators.dense_products(a64, b64, V)
    rho = 5e-4
    eta = 0.1 / max(np.linalg.norm(game.direction_alg2(i, V, aux, av0, bv0, rho)) for i in range(k))
    out = {}
    for tc in (1, 0):
        s = geig.Solver(geig.GEIG_DENSE, d, 0, k, math=math, rho=rho)
        try:
            geig.geig_set_option(s.h, geig.GEIG_OPT_GRAM_TC, tc)
            s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
            AV = torch.empty(k, d, device=dev)
            BV = torch.empty_like(AV)
            geig.geig_products_dense(s.h, a, b, 0, d, AV, BV)
            l0 = s.launches()
            geig.geig_update(s.h, AV, BV, eta, 1.0)
            launches = s.launches() - l0
            V2, A2 = [x.double().cpu().numpy() for x in s.state()]
            ga, gb, gc = [x.double().cpu().numpy() for x in s.gram()]
            out[tc] = (V2, A2, ga, gb, gc, launches)
        finally:
            s.close()
    assert out[1][5] > out[0][5]            # the Gram launch (+ the 3xTF32 V split) ran
    tol = 1e-5 if math == "3xtf32" else 3e-3
    for j, name in ((2, "ga"), (4, "gc")):
        assert rel_err(out[1][j], out[0][j]) < tol, name
    assert rel_err(out[1][0] - V, out[0][0] - V) < 10 * tol
    if math == "3xtf32":
        V2, aux2 = game.step_alg2(V, aux, [(av0, bv0)], eta, 1.0, rho)
        assert rel_err(out[1][0] - V, V2 - V) < 1e-4
        assert rel_err(out[1][1], aux2) < 1e-4


@pytest.mark.parametrize("k,rows", [(40, 1000), (17, 2050), (64, 258)])
def test_fused_pairs_other_k_and_ragged_batches(geig, k, rows):
    """CTA pairs with k not a multiple of 32 (the drain reads TMEM columns
    past k, which must not reach the tiles) and ragged batches (h not a
    multiple of the 64-row K blocks): the pair step against one CTA per
    item and against the oracle."""
    from synth import CONFIGS, cca_views
    cfg = CONFIGS[3]
    x, y = cca_views(cfg, rows, seed=19)
    V, aux = random_state(k, cfg.d, 13)
    V32 = V.astype(np.float32).astype(np.float64)
    aux32 = aux.astype(np.float32).astype(np.float64)
    dev = "cuda:0"
    out = []
    for pairs in (1, 0):
        s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16,
                        rho=cfg.rho, max_rows=rows)
        try:
            geig.geig_set_option(s.h, geig.GEIG_OPT_FUSED_PAIRS, pairs)
            s.set_state(torch.tensor(V32, dtype=torch.float32, device=dev),
                        torch.tensor(aux32, dtype=torch.float32, device=dev))
            geig.geig_step_cca(s.h, x.to(dev), y.to(dev), rows, 0.02, cfg.gamma)
            out.append([t.double().cpu().numpy() for t in s.state()])
        finally:
            s.close()
    (Vp, ap), (Vs, as_) = out
    assert rel_err(Vp - V32, Vs - V32) < 1e-5 and rel_err(ap, as_) < 1e-5
    _, _, Vo, Ao = oracle_cca_step(x.double().numpy(), y.double().numpy(), V32, aux32, 0.02, cfg.gamma, cfg.rho)
    assert rel_err(Vp - V32, Vo - V32) < 1e-3
    assert rel_err(ap, Ao) < 1e-4
