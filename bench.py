#!/usr/bin/env python
"""bench.py — throughput of gamma-EigenGame updates on B200.

One step = one pass of the whole hot path (Alg. 2: minibatch products
A_t V, B_t V; Gram tables; penalty coefficients; fused ascent / retraction /
auxiliary update) over one minibatch of synthetic data already resident in
HBM.  Default workload: BASELINE.json configs[3] (CCA, dx=dy=8192, k=64,
batch 4096 rows per GPU, bf16 data, fp32 accumulate) — see DESIGN.md §Bench.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config I]
                    [--math bf16|f32|tf32|3xtf32] [--impl reference]

Multi-GPU (N > 1) is launched by torchrun; each rank owns its own batch
(weak scaling), products are combined by an NCCL all-reduce (Appendix F).
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/s of gamma-EigenGame updates (d,k)"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def _peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        # NVML at ~5 ms (the timed region is ~0.1 s); nvidia-smi as the fallback
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = (0x8, 0x40, 0x20, 0x4)   # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            def sample():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                try:
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
                self.rows.append([str(sm), str(smax)] + ["Active" if rs & b else "Not Active" for b in bits]
                                 + [str(util)])

            while not self._stop.is_set():
                try:
                    sample()
                except Exception:
                    pass
                self._stop.wait(float(os.environ.get("BENCH_CLOCK_INTERVAL", "0.005")))
            if not self.rows:
                sample()
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm, loaded = [], []
        smax = None
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
                if float(r[6]) > 0:
                    loaded.append(float(r[0]))
            except Exception:
                continue
            for n, v in zip(names, r[2:6]):
                if v.strip().lower() in ("active", "1", "0x1"):
                    reasons.add(n)
        use = loaded or sm
        return {"sm_mhz": statistics.median(use) if use else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def _dense_traffic(math, world):
    """DRAM bytes of one config-4 products launch from an ncu --set full
    capture (profiles/roofline_traffic_dense.json), for the captured math at
    N = 1; else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic_dense.json")) as f:
            tr = json.load(f)
        return tr["dram_bytes_per_launch"] if tr.get("math") == math and world == 1 else None
    except Exception:
        return None


def _workload(cfg, math):
    return {"workload": cfg.name, "problem": cfg.problem, "dx": cfg.dx, "dy": cfg.dy, "k": cfg.k,
            "batch_per_gpu": cfg.batch, "math": math, "data_dtype": cfg.dtype,
            "recipe": cfg.recipe}


# ---------------------------------------------------------------------------
# reference arm: the fp64 oracle on the host cores
# ---------------------------------------------------------------------------

def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


def oracle_sample(cfg, seconds: float, max_steps: int | None = None, seed: int = 0, rows_per_step: int | None = None):
    """Time the oracle (as it stands) on real steps of the workload until
    `seconds` of CPU work or `max_steps`; returns (rows/s, steps, rows).
    rows_per_step: a bounded sample of the batch (the first rows) per step."""
    import numpy as np
    from oracle import estimators, game
    from synth import cca_views, dense_gep_small, gaussian_init
    if cfg.problem == "cca":
        b = rows_per_step or cfg.batch
        x, y = cca_views(cfg, b, seed=seed)
        x64, y64 = x.double().numpy(), y.double().numpy()
        V, aux = game.init_state(gaussian_init(cfg.k, cfg.d, seed))
        n, rows, t0 = 0, 0, time.perf_counter()
        while True:
            av, bv = estimators.cca_products(x64, y64, V)
            V, aux = game.step_alg2(V, aux, [(av, bv)], cfg.eta, cfg.gamma, cfg.rho)
            n += 1
            rows += b
            el = time.perf_counter() - t0
            if el >= seconds or (max_steps and n >= max_steps):
                return rows / el, n, rows, el
    a, b = dense_gep_small(seed, cfg.d) if cfg.d <= 64 else (None, None)
    if a is None:
        # config 4's matrices at full size, drawn on the GPU when there is one
        # (the draw is input preparation, not timed); on a CPU-only host a
        # reduced d
        import torch
        from synth import dense_gep_large
        on_gpu = torch.cuda.is_available()
        at, bt = dense_gep_large(cfg.d if on_gpu else min(cfg.d, 2048), seed, device="cuda:0" if on_gpu else "cpu")
        a, b = at.double().cpu().numpy(), bt.double().cpu().numpy()
        del at, bt
    V, aux = game.init_state(gaussian_init(cfg.k, a.shape[0], seed))
    n, t0 = 0, time.perf_counter()
    while True:
        av, bv = estimators.dense_products(a, b, V)
        V, aux = game.step_alg2(V, aux, [(av, bv)], cfg.eta, cfg.gamma, cfg.rho)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or (max_steps and n >= max_steps):
            return n / el, n, n, el


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    # one untimed full step warms the BLAS threads up and sizes the run: the
    # K timed steps are full oracle steps when they fit ~120 s of host time,
    # else each step runs on a bounded sample of the batch (its first rows,
    # the oracle's cost being linear in the rows) so that EXACTLY K steps are
    # timed.  A dense step (full batch by definition) cannot be sampled: its
    # run is bounded in time and the line reports the steps run.
    _, _, _, t1 = oracle_sample(cfg, 0.0, max_steps=1)
    _, _, _, t1 = oracle_sample(cfg, 0.0, max_steps=1)
    rows_step = None
    sample = f"full oracle steps of {cfg.batch if cfg.problem == 'cca' else 'full-batch'} rows"
    full_rate = (cfg.batch / t1) if cfg.problem == "cca" else (1.0 / t1)
    if cfg.problem == "cca" and args.steps * t1 > 200.0:
        rows_step = max(64, int(cfg.batch * 200.0 / (args.steps * t1)) // 2 * 2)
        # (the oracle's per-step update cost does not shrink with the rows, so
        # the sampled rate is below the full-step rate reported beside it)
        sample = (f"oracle steps on the first {rows_step} of {cfg.batch} rows of the batch "
                  f"(one full step alone: {full_rate:.0f} samples/s)")
    v, n, rows, el = oracle_sample(cfg, 300.0 if rows_step else 150.0, max_steps=args.steps, rows_per_step=rows_step)
    unit = "samples/s" if cfg.problem == "cca" else "steps/s"
    cores = _blas_threads()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": unit, "n_gpus": world,
            "steps": n, "warmup": args.warmup, "ms_per_step": 1e3 * el / n, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _workload(cfg, "f64-oracle"),
            "cpu_baseline": {"value": v, "unit": unit, "cores": cores, "kind": "oracle",
                             "sample": f"{n} {sample}", "full_step_value": full_rate},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def _box_copy_gbs(dev, n=1 << 28, reps=5):
    """Best-of-`reps` bf16 device copy of n elements (read + write bytes) on
    this box, CUDA events; None if it cannot allocate."""
    import torch
    try:
        a = torch.empty(n, dtype=torch.bfloat16, device=dev).fill_(1.0)
        b = torch.empty_like(a)
        best = float("inf")
        for _ in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2 * n * 2 / (best / 1e3) / 1e9
    except Exception:
        return None

def run_gpu_dense(args, cfg, rank, world, dev, stream, peaks, peaks_src):
    """Dense full-batch GEP step (configs 0, 4; Alg. 2 with exact A, B =
    Alg. 1's direction): A and B row-sharded over the
    ranks (shard_rows), each rank's geig_products_dense forms its columns of
    AV, BV, one all-gather of the column blocks (dense_allgather_rows)
    assembles them, every rank applies geig_update to its replica of V and
    [Bv].  The unit is steps/s; the problem size is fixed as N grows
    (strong scaling)."""
    import torch
    import torch.distributed as dist
    from paper_2206_04993_b200 import geig
    from paper_2206_04993_b200.parallel import dense_allgather_rows, dense_wire_bytes, shard_rows
    from synth import dense_gep_large, dense_gep_small, gaussian_init
    math = args.math
    d, k = cfg.d, cfg.k
    if d <= 64:
        a64, b64 = dense_gep_small(0, d)
        A = torch.tensor(a64, dtype=torch.float32, device=dev)
        B = torch.tensor(b64, dtype=torch.float32, device=dev)
    else:
        A, B = dense_gep_large(d, seed=0, device=dev)
    r0, r1 = shard_rows(d, world, rank)
    Ar, Br = A[r0:r1].contiguous(), B[r0:r1].contiguous()
    if world > 1:
        del A, B
        torch.cuda.empty_cache()
    s = geig.Solver(geig.GEIG_DENSE, d, 0, k, math=math, rho=cfg.rho, device=dev.index, stream=stream.cuda_stream)
    s.init_state(torch.tensor(gaussian_init(k, d, 0), dtype=torch.float32, device=dev))
    AV = torch.empty(k, d, device=dev)
    BV = torch.empty_like(AV)
    ev = []

    def step(timed):
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        geig.geig_products_dense(s.h, Ar, Br, r0, r1, AV, BV)
        if timed:
            e1.record(stream)
            ev.append((e0, e1))
        if world > 1:
            dense_allgather_rows(AV, BV, d, world)
        geig.geig_update(s.h, AV, BV, cfg.eta, cfg.gamma)

    t_spin = time.perf_counter()
    while time.perf_counter() - t_spin < args.spinup:
        step(False)
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = s.launches()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_start.record(stream)
        for _ in range(args.steps):
            step(True)
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = s.launches() - l0
    elapsed_ms = t_start.elapsed_time(t_end)
    prod_ms = statistics.mean(a.elapsed_time(b_) for a, b_ in ev)
    if world > 1:
        t = torch.tensor([elapsed_ms, prod_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, prod_ms = t.tolist()
    value = args.steps / (elapsed_ms / 1e3)
    # roofline of the products launch (the dominant kernel): this rank's rows
    # of A and B read once, V read, its columns of AV, BV written
    esz = 4
    rows = r1 - r0
    alg_bytes = 2 * rows * d * esz + k * d * esz + 2 * k * rows * 4
    achieved = alg_bytes / (prod_ms / 1e3) / 1e9
    box_copy = _box_copy_gbs(dev)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks.get("hbm_gbs", 6650.0), "unit": "GB/s",
            "frac": achieved / peaks.get("hbm_gbs", 6650.0), "box_copy_gbs": box_copy,
            "frac_of_box_copy": (achieved / box_copy) if box_copy else None, "traffic": _dense_traffic(math, world),
            "algorithmic_bytes": alg_bytes, "peak_source": peaks_src,
            "kernel": f"tc_gemm products of the rank's rows of A and B ({math})", "ms_per_launch": prod_ms,
            "step_ms": elapsed_ms / args.steps, "products_share": prod_ms / (elapsed_ms / args.steps),
            "tensor_tflops": 4.0 * k * rows * d / (prod_ms / 1e3) / 1e12}
    e2e = None
    if not args.no_e2e:
        # end to end through the C ABI from pinned host memory: every step
        # copies this rank's rows of A and B host -> device, runs the step and
        # reads the k x k Gram table back
        hA, hB = Ar.cpu().pin_memory(), Br.cpu().pin_memory()
        ga = torch.empty(k, k).pin_memory()
        gd = torch.empty(3, k, k, device=dev)
        n_e2e = 3
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            Ar.copy_(hA, non_blocking=True)
            Br.copy_(hB, non_blocking=True)
            step(False)
            geig.geig_get_gram(s.h, gd[0], gd[1], gd[2])
            ga.copy_(gd[0])
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": n_e2e / el, "unit": "steps/s", "h2d_bytes_per_step": 2 * rows * d * esz,
               "d2h_bytes_per_step": k * k * 4, "steps": n_e2e, "timer": "host wall clock (synchronised)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, n, _, el = oracle_sample(cfg, args.cpu_seconds, seed=0)
        cpu = {"value": v, "unit": "steps/s", "cores": _blas_threads(), "kind": "oracle",
               "sample": f"{n} full fp64 oracle steps at d={d}, k={k} ({el:.1f} s)"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32" if math == "f32" else math,
                "data": "synthetic",
                "config": {"workload": cfg.name, "problem": "dense", "d": d, "k": k, "math": math,
                           "data_dtype": "f32", "recipe": cfg.recipe, "parallelism": f"rows{world}",
                           "rows_per_gpu": rows,
                           "collective": "all-gather of the column blocks of AV, BV" if world > 1 else None,
                           "wire_bytes_per_rank": dense_wire_bytes(k, d, world) if world > 1 else None,
                           "l2_policy": "A and B (2 x %.1f GiB) exceed the 126 MB L2; read once per step"
                                        % (rows * d * 4 / 2**30)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    s.close()


def run_gpu(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2206_04993_b200 import build
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    from paper_2206_04993_b200 import geig
    from paper_2206_04993_b200.parallel import allreduce_products, cca_scale, product_buffers
    from synth import cca_views, dense_gep_large, gaussian_init

    # (GEIG_BENCH_SHARE_GPU: functional check of the multi-rank path with
    # every rank on the available GPUs; never a measurement)
    ndev = torch.cuda.device_count()
    dev = torch.device(f"cuda:{local_rank % ndev if os.environ.get('GEIG_BENCH_SHARE_GPU') else local_rank}")
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    peaks, peaks_src = _peaks()

    if cfg.problem != "cca":
        return run_gpu_dense(args, cfg, rank, world, dev, stream, peaks, peaks_src)
    math = args.math
    data_bf16 = cfg.dtype == "bf16"
    dtype = torch.bfloat16 if data_bf16 else torch.float32
    # config 3 reads "batch 4096; rows sharded over 8 GPUs": --scaling weak
    # (default) gives every rank its own 4096-row batch (global N x 4096),
    # --scaling strong shards ONE 4096-row batch over the N ranks
    b = cfg.batch if args.scaling == "weak" else cfg.batch // world
    if b < 2:
        raise SystemExit("bench: --scaling strong leaves fewer than 2 rows per rank")
    esz = 2 if data_bf16 else 4
    batch_bytes = b * cfg.d * esz
    # ring of P distinct batches in HBM, larger than the 126 MB L2
    P = max(2, int((4 * 126e6) // batch_bytes) + 1)
    P = min(P, 64)
    X, Y = cca_views(cfg, P * b, seed=1000 + rank, device=dev, dtype=dtype)
    Xs = [X[i * b:(i + 1) * b] for i in range(P)]
    Ys = [Y[i * b:(i + 1) * b] for i in range(P)]
    s = geig.Solver(geig.GEIG_CCA, cfg.dx, cfg.dy, cfg.k, math=math,
                    data_dtype=geig.GEIG_DATA_BF16 if data_bf16 else geig.GEIG_DATA_F32,
                    rho=cfg.rho, max_rows=b, device=dev.index, stream=stream.cuda_stream)
    G = torch.tensor(gaussian_init(cfg.k, cfg.d, 0), dtype=torch.float32, device=dev)
    s.init_state(G)
    variant = "alg2"
    if args.smooth_nu is not None:                     # Alg. 3
        geig.geig_set_smooth(s.h, args.smooth_nu)
        variant = f"alg3(nu={args.smooth_nu:g})"
    if args.adam:                                      # Appendix H optimizer
        geig.geig_set_adam(s.h, 0.9, 0.999, 1e-8)
        variant += "+adam"
    scale = cca_scale(b, world)
    # multi-GPU step: the fused kernel's products + Gram-table partials in one
    # launch, ONE in-place all-reduce of [AV | BV | tables], then the update
    # from the aggregated tables (geig_products_cca_tables / geig_update_tables)
    tables = (world > 1 or args.split_step) and math in ("bf16", "bf16x2") and cfg.k <= 64 and not args.staged \
        and not args.no_tables
    # column-owned step (default at N > 1 where the partition fits): the
    # products launch writes per-owner chunks, ONE reduce-scatter, the update
    # of the rank's d / N columns, ONE all-gather of the bf16 shadow blocks
    owned = None
    peer = None
    if world > 1 and tables and args.multi == "peer":
        # the column-owned step over NVLink peer memory: no NCCL call on the
        # data path (buffers mapped by CUDA IPC, epoch flags)
        from paper_2206_04993_b200.parallel import PeerColumnOwnedStep, owned_wire_bytes
        geig.geig_set_partition(s.h, world, rank)
        peer = PeerColumnOwnedStep(geig, s, world, rank)
    if world > 1 and tables and args.multi == "owned":
        from paper_2206_04993_b200.parallel import (ColumnOwnedStep, allgather_blocks, owned_wire_bytes,
                                                    reduce_scatter_chunks)
        try:
            geig.geig_set_partition(s.h, world, rank)
            owned = ColumnOwnedStep(geig, s, world, rank)
        except geig.GeigError as e:
            if rank == 0:
                sys.stderr.write(f"bench: column-owned step unavailable ({e}); replicated all-reduce step\n")
    if tables:
        AV, BV, T = product_buffers(cfg.k, cfg.d, geig.geig_table_floats(s.h), device=dev)
    else:
        AV, BV = product_buffers(cfg.k, cfg.d, device=dev)   # one buffer: in-place all-reduce
        T = None

    ev = []

    fused = world == 1 and math in ("bf16", "bf16x2") and cfg.k <= 64 and not args.staged and not args.split_step
    # fp32 small problems (config 1): the one-CTA step kernel, state resident
    # in shared memory (small_step.cuh; k <= 16, KP d <= 8192, KP = 8 or 16)
    small = (world == 1 and math == "f32" and cfg.k <= 16 and (8 if cfg.k <= 8 else 16) * cfg.d <= 8192 and not args.staged
             and not args.split_step)
    fused = fused or small

    def step(i, timed):
        if timed:
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
        if fused:
            # one launch per step: forward GEMM, reshuffle, backward GEMM, Gram tables, update
            geig.geig_step_cca(s.h, Xs[i % P], Ys[i % P], b, cfg.eta, cfg.gamma)
            if timed:
                e1.record(stream)
        elif peer is not None:
            geig.geig_products_cca_peer(s.h, Xs[i % P], Ys[i % P], b, scale)
            if timed:
                e1.record(stream)
            geig.geig_update_peer(s.h, cfg.eta, cfg.gamma)
        elif owned is not None:
            geig.geig_products_cca_owned(s.h, Xs[i % P], Ys[i % P], b, scale, owned.buf)
            if timed:
                e1.record(stream)
            reduce_scatter_chunks(owned.buf, owned.mine)
            geig.geig_update_owned(s.h, owned.mine, cfg.eta, cfg.gamma)
            allgather_blocks(owned.shadow)
        elif tables:
            geig.geig_products_cca_tables(s.h, Xs[i % P], Ys[i % P], b, scale, AV, BV, T)
            if timed:
                e1.record(stream)
            if world > 1:
                allreduce_products(AV, BV, T=T)
            geig.geig_update_tables(s.h, AV, BV, T, cfg.eta, cfg.gamma)
        else:
            geig.geig_products_cca(s.h, Xs[i % P], Ys[i % P], b, scale, AV, BV)
            if timed:
                e1.record(stream)
            if world > 1:
                allreduce_products(AV, BV)
            geig.geig_update(s.h, AV, BV, cfg.eta, cfg.gamma)
        if timed:
            e2.record(stream)
            ev.append((e0, e1, e2))

    # fused path: Alg. 2's loop over the K timed steps is ONE persistent launch
    # (geig_run_cca); --per-step-launch times one geig_step_cca launch per step
    multi = fused and not args.per_step_launch

    def run_args(i0, n):   # marshalled outside the timed region
        return geig.cca_batches([Xs[(i0 + i) % P] for i in range(n)], [Ys[(i0 + i) % P] for i in range(n)])

    def run_steps(i0, n, args_=None):
        geig.geig_run_cca(s.h, None, None, b, cfg.eta, cfg.gamma, batches=args_ or run_args(i0, n))

    # spin the clocks up from idle (untimed, ~0.5 s), then the W warm-up steps
    t_spin = time.perf_counter()
    i_spin = 0
    while time.perf_counter() - t_spin < args.spinup:
        if multi:
            run_steps(i_spin, 20)
            i_spin += 20
        else:
            for _ in range(20):
                step(i_spin, False)
                i_spin += 1
        torch.cuda.synchronize()
    if multi:
        run_steps(0, args.warmup)
    else:
        for i in range(args.warmup):
            step(i, False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = s.launches()
    timed_args = run_args(args.warmup, args.steps) if multi else None
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_start.record(stream)
        if multi:
            run_steps(args.warmup, args.steps, timed_args)
        else:
            for i in range(args.steps):
                step(args.warmup + i, True)
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = s.launches() - l0
    elapsed_ms = t_start.elapsed_time(t_end)
    if multi:
        prod_ms = upd_ms = elapsed_ms / args.steps       # one launch: the kernel time per step
    else:
        prod_ms = statistics.mean(a.elapsed_time(b_) for a, b_, _ in ev)
        upd_ms = statistics.mean(b_.elapsed_time(c) for _, b_, c in ev)
    if world > 1:
        t = torch.tensor([elapsed_ms, prod_ms, upd_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, prod_ms, upd_ms = t.tolist()
    value = world * b * args.steps / (elapsed_ms / 1e3)

    # roofline of the dominant kernel.  Fused path: the single step kernel;
    # algorithmic bytes = the batch read once + the state (V, [Bv]) read and
    # written once + the bf16 shadow of V.  Staged path:
    # the products stage, algorithmic bytes = batch + V read + AV/BV written.
    kd = cfg.k * cfg.d
    if fused:
        alg_bytes = b * cfg.d * esz + 2 * kd * 4 + 2 * kd * 4 + kd * 2
        if small:
            kernel = ("small_step_kernel (one CTA: forward, backward, Gram, update, state in shared memory; "
                      + ("K steps in one launch via geig_run_cca)" if multi else "one launch per step)"))
            phases = {}
        else:
            kernel = ("cca_step_kernel (fused: forward GEMM, reshuffle, backward GEMM, Gram, update; "
                      + ("K steps in one persistent launch via geig_run_cca)" if multi else "one launch per step)"))
            ph = geig.geig_update_phase_ns(s.h)
            phases = {"forward_us": ph[3] / 1e3, "reshuffle_backward_us": ph[4] / 1e3, "gram_us": ph[0] / 1e3,
                      "reduce_us": ph[1] / 1e3, "coef_update_us": ph[2] / 1e3,
                      "source": "%globaltimer, CTA 0, last step"}
        k_ms = prod_ms
    else:
        alg_bytes = b * cfg.d * esz + kd * (2 if math in ("bf16", "bf16x2") else 4) + 2 * kd * 4
        kernel = ("cca_step_kernel products-only launch (phases F, S, B; multi-GPU: then all-reduce + update)"
                  if math in ("bf16", "bf16x2") and cfg.k <= 64 and not args.staged
                  else "products stage (tc_gemm forward + zshuffle + tc_gemm backward)")
        k_ms = prod_ms
        phases = {"products_ms": prod_ms, "update_ms": upd_ms}
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("workload") == cfg.name and tr.get("math") == math and tr.get("fused", False) == fused:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    # this box's own copy bandwidth (same method as MEASURED_PEAKS.json, after
    # the timed region): HBM bandwidth differs between boxes of the pool by
    # ~15%, so the line carries the denominator it was measured against too
    box_copy = _box_copy_gbs(dev)
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "box_copy_gbs": box_copy, "frac_of_box_copy": (achieved / box_copy) if box_copy else None,
            "frac": achieved / hbm_peak, "traffic": traffic, "algorithmic_bytes": alg_bytes,
            "kernel": kernel, "peak_source": peaks_src, "ms_per_launch": k_ms, "phases": phases,
            "flops_per_step": 4.0 * cfg.k * cfg.d * b,
            "tensor_tflops": 4.0 * cfg.k * cfg.d * b / (k_ms / 1e3) / 1e12}

    # end to end through the C ABI with HOST buffers (pinned), rank-local
    e2e = None
    if not args.no_e2e and world == 1:
        # one geig_run_cca_host call: the H2D copy of batch t + 1 (copy
        # stream, double-buffered staging) overlaps step t; every step's G^A
        # table is copied back; two distinct pinned host batches alternate
        hxs = [Xs[i % P].cpu().pin_memory() for i in range(2)]
        hys = [Ys[i % P].cpu().pin_memory() for i in range(2)]
        ga = torch.empty(cfg.k, cfg.k).pin_memory()
        n_e2e = max(3, min(args.steps, 20))
        geig.geig_run_cca_host(s.h, hxs, hys, b, cfg.eta, cfg.gamma, ga)   # warm: staging, copy stream
        t0 = time.perf_counter()
        h2d, d2h = geig.geig_run_cca_host(s.h, [hxs[i % 2] for i in range(n_e2e)], [hys[i % 2] for i in range(n_e2e)],
                                          b, cfg.eta, cfg.gamma, ga)
        el = time.perf_counter() - t0
        e2e = {"value": b * n_e2e / el, "unit": "samples/s", "h2d_bytes_per_step": h2d // n_e2e,
               "d2h_bytes_per_step": d2h // n_e2e, "steps": n_e2e,
               "timer": "host wall clock around one geig_run_cca_host call (it synchronises)",
               "pipeline": "H2D of batch t+1 on a copy stream overlaps step t"}
    elif not args.no_e2e:
        hx = Xs[0].cpu().pin_memory()
        hy = Ys[0].cpu().pin_memory()
        ga = torch.empty(cfg.k, cfg.k).pin_memory()
        n_e2e = max(3, min(args.steps, 20))
        # the Appendix-F step of every rank from its pinned host shard:
        # H2D copy, products, in-place all-reduce, update, D2H of the Gram
        # table (the same result the single-GPU host call reads back)
        xd, yd = torch.empty_like(Xs[0]), torch.empty_like(Ys[0])
        gd = torch.empty(3, cfg.k, cfg.k, device=dev)

        def e2e_step():
            xd.copy_(hx, non_blocking=True)
            yd.copy_(hy, non_blocking=True)
            if peer is not None:
                peer(xd, yd, b, cfg.eta, cfg.gamma)
            elif owned is not None:
                owned(xd, yd, b, cfg.eta, cfg.gamma)
            elif tables:
                geig.geig_products_cca_tables(s.h, xd, yd, b, scale, AV, BV, T)
                allreduce_products(AV, BV, T=T)
                geig.geig_update_tables(s.h, AV, BV, T, cfg.eta, cfg.gamma)
            else:
                geig.geig_products_cca(s.h, xd, yd, b, scale, AV, BV)
                allreduce_products(AV, BV)
                geig.geig_update(s.h, AV, BV, cfg.eta, cfg.gamma)
            geig.geig_get_gram(s.h, gd[0], gd[1], gd[2])
            ga.copy_(gd[0])
            return hx.numel() * hx.element_size() + hy.numel() * hy.element_size(), ga.numel() * 4
        e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            h2d, d2h = e2e_step()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": world * b * n_e2e / el, "unit": "samples/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": n_e2e, "timer": "host wall clock (call synchronises)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, n, rows, el = oracle_sample(cfg, args.cpu_seconds, seed=0)
        cpu = {"value": v, "unit": "samples/s", "cores": _blas_threads(), "kind": "oracle",
               "sample": f"{n} full fp64 oracle steps of {cfg.batch} rows ({el:.1f} s)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": "bf16" if math in ("bf16", "bf16x2") else ("f32" if math == "f32" else math),
                "data": "synthetic",
                "config": dict(_workload(cfg, math), batch_per_gpu=b, parallelism=f"dp{world}", global_batch=world * b,
                               batch_reading=("weak: every rank streams its own batch of %d rows (global N x %d); "
                                              "--scaling strong shards one %d-row batch over the N ranks"
                                              % (cfg.batch, cfg.batch, cfg.batch)) if args.scaling == "weak" else
                                             ("strong: one %d-row batch sharded over the N ranks (%d rows each); "
                                              "--scaling weak gives every rank its own %d-row batch"
                                              % (cfg.batch, b, cfg.batch)),
                               update=variant,
                               wire_bytes_per_rank=(owned_wire_bytes(cfg.k, cfg.d, world, geig.geig_table_floats(s.h))
                                                    if (owned is not None or peer is not None) else None),
                               step=("fused single launch (geig_run_cca)" if multi else
                                     "fused single launch per step" if fused else
                                     "column-owned over NVLink peer memory: products launch stores every column's "
                                     "AV|BV into its owner's slot, update sums the slots and stores its shadow block "
                                     "into every rank (epoch flags, no NCCL on the data path)" if peer is not None else
                                     "column-owned: products launch (per-owner chunks), reduce-scatter, update of "
                                     "the rank's d/N columns, all-gather of the bf16 shadow" if owned is not None else
                                     "products+tables launch, all-reduce, update_tables" if tables else
                                     "products launch, all-reduce, update"),
                               l2_policy=f"ring of {P} distinct batches ({P * batch_bytes / 2**20:.0f} MiB) "
                                         "> 126 MB L2, a new batch every step"),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    s.close()


def _free_port():
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--spinup", type=float, default=0.5, help="seconds of untimed steps before warm-up")
    ap.add_argument("--smooth-nu", type=float, default=None,
                    help="Alg. 3 (smooth gamma-EigenGame) with this nu upper bound of lambda_max(B)")
    ap.add_argument("--adam", action="store_true", help="Adam ascent on v_i (Appendix H)")
    ap.add_argument("--per-step-launch", action="store_true",
                    help="fused path: one geig_step_cca launch per step instead of geig_run_cca")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--multi", choices=("owned", "peer", "replicated"), default="owned",
                    help="N > 1: column-owned reduce-scatter / all-gather step (NCCL), the column-owned step over "
                         "NVLink peer memory (CUDA IPC, no NCCL on the data path), or the replicated all-reduce step")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="weak: cfg.batch rows per rank; strong: cfg.batch rows sharded over the ranks")
    ap.add_argument("--math", default=None)
    ap.add_argument("--impl", default="b200")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--staged", action="store_true", help="products + update as separate launches")
    ap.add_argument("--split-step", action="store_true",
                    help="N=1: the multi-GPU step structure (products launch, then update launch)")
    ap.add_argument("--no-tables", action="store_true",
                    help="multi-GPU / split step: update re-forms the Gram tables (geig_update) instead of "
                         "aggregating them with the products")
    args = ap.parse_args()
    from synth import CONFIGS
    cfg = CONFIGS[args.config]
    if args.math is None:
        # bf16 data: tensor cores with hi+lo bf16 operands (bf16x2) — same speed as
        # plain bf16 on this HBM-bound step, products ~fp32-accurate
        args.math = "bf16x2" if cfg.dtype == "bf16" else ("tf32" if cfg.problem == "dense" and cfg.d > 64 else "f32")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` without a launcher: re-exec under
        # torch.distributed.run, one rank per GPU (rank 0 prints the line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.stderr.write("bench: launching " + " ".join(cmd) + "\n")
        raise SystemExit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world} (launch one rank per GPU)")
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank % torch.cuda.device_count() if os.environ.get("GEIG_BENCH_SHARE_GPU")
                              else local_rank)
        dist.init_process_group(os.environ.get("GEIG_BENCH_BACKEND", "nccl"))
    run_gpu(args, cfg, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
