"""World-size-2 gloo tests of the multi-GPU host logic (parallel.py) on CPU:
row sharding, the Appendix-F all-reduce of partial products and identical
replicated updates.  The per-rank compute is injected (here: the oracle's
product form), exactly where the product path injects the CUDA binding."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_04993_b200.parallel import ShardedStep, cca_scale, dense_allgather_rows, product_buffers, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, x, y, V, aux, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import estimators, game
        b_local = x.shape[0] // world
        xs = x[rank * b_local:(rank + 1) * b_local]
        ys = y[rank * b_local:(rank + 1) * b_local]
        h = b_local // 2
        scale = cca_scale(b_local, world)
        state = {"V": V.copy(), "aux": aux.copy()}

        def products(AV, BV):
            # per-rank partial sums, scaled so that the SUM over ranks is the estimate
            av, bv = estimators.cca_products(xs.numpy(), ys.numpy(), state["V"])
            AV.copy_(torch.from_numpy(av * h * scale))
            BV.copy_(torch.from_numpy(bv * h * scale))

        def update(AV, BV):
            state["V"], state["aux"] = game.step_alg2(state["V"], state["aux"], [(AV.numpy(), BV.numpy())],
                                                      0.1, 0.5, 1e-3)

        step = ShardedStep(products, update)
        # rank 0: AV, BV halves of one buffer (in-place all-reduce); rank 1:
        # separate tensors (stacked all-reduce) -- both paths must agree
        if rank == 0:
            AV, BV = product_buffers(V.shape[0], V.shape[1], dtype=torch.float64)
            AV.zero_()
            BV.zero_()
        else:
            AV = torch.zeros(V.shape, dtype=torch.float64)
            BV = torch.zeros_like(AV)
        step(AV, BV)
        out_q.put((rank, AV.numpy().copy(), state["V"], state["aux"]))
        # dense row sharding: each rank writes its columns, all-reduce assembles
        d = 11                               # ragged: shards of 6 and 5 rows
        rng = np.random.default_rng(0)
        A = rng.standard_normal((d, d)); A = A + A.T
        W = rng.standard_normal((3, d))
        r0, r1 = shard_rows(d, world, rank)
        AVd = torch.full((3, d), float("nan"), dtype=torch.float64)   # other ranks' columns are filled by the gather
        BVd = torch.full_like(AVd, float("nan"))
        AVd[:, r0:r1] = torch.from_numpy((A[r0:r1] @ W.T).T)
        BVd[:, r0:r1] = torch.from_numpy((2 * A[r0:r1] @ W.T).T)
        dense_allgather_rows(AVd, BVd, d, world)
        out_q.put((rank + 100, AVd.numpy(), (A @ W.T).T, BVd.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_rows_partition():
    for n in [1, 7, 16, 4097]:
        for w in [1, 2, 3, 8]:
            rs = [shard_rows(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [r1 - r0 for r0, r1 in rs]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_world2_allreduce_matches_global_batch():
    from oracle import estimators, game
    world = 2
    rng = np.random.default_rng(3)
    b_local, dx, dy, k = 40, 6, 5, 3
    x = torch.from_numpy(rng.standard_normal((world * b_local, dx)))
    y = torch.from_numpy(rng.standard_normal((world * b_local, dy)))
    V, aux = game.init_state(rng.standard_normal((k, dx + dy)))
    aux = aux + 0.1 * rng.standard_normal(aux.shape)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, y, V, aux, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2 * world):
        r, a, b, c = q.get(timeout=120)
        res[r] = (a, b, c)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # global reference: A-halves of both ranks form the A batch, B-halves the B batch (reading R1)
    h = b_local // 2
    xa = torch.cat([x[r * b_local:r * b_local + h] for r in range(world)])
    xb = torch.cat([x[r * b_local + h:(r + 1) * b_local] for r in range(world)])
    ya = torch.cat([y[r * b_local:r * b_local + h] for r in range(world)])
    yb = torch.cat([y[r * b_local + h:(r + 1) * b_local] for r in range(world)])
    xg = torch.cat([xa, xb]).numpy()
    yg = torch.cat([ya, yb]).numpy()
    av, bv = estimators.cca_products(xg, yg, V)
    V2, aux2 = game.step_alg2(V, aux, [(av, bv)], 0.1, 0.5, 1e-3)
    for r in range(world):
        AVr, Vr, auxr = res[r]
        assert np.allclose(AVr, av, atol=1e-12)
        assert np.allclose(Vr, V2, atol=1e-12) and np.allclose(auxr, aux2, atol=1e-12)
    assert np.array_equal(res[0][1], res[1][1])        # replicas identical
    for r in range(world):
        got, ref, gotb = res[100 + r]
        assert np.allclose(got, ref, atol=1e-12)
        assert np.allclose(gotb, 2 * ref, atol=1e-12)


def _tables_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_04993_b200.parallel import allreduce_products
        k, d, nt = 3, 7, 12
        g = torch.Generator().manual_seed(100 + rank)
        # adjacent [AV | BV | T] in one buffer: ONE in-place all-reduce
        AV, BV, T = product_buffers(k, d, nt, dtype=torch.float64)
        AV.copy_(torch.randn(k, d, generator=g, dtype=torch.float64))
        BV.copy_(torch.randn(k, d, generator=g, dtype=torch.float64))
        T.copy_(torch.randn(nt, generator=g, dtype=torch.float64))
        mine = (AV.clone(), BV.clone(), T.clone())
        allreduce_products(AV, BV, T=T)
        # separate tensors: the stacked fallback
        AV2, BV2, T2 = mine[0].clone(), mine[1].clone(), mine[2].clone()
        allreduce_products(AV2, BV2, T=T2)
        out_q.put((rank, [t.numpy().copy() for t in mine], [t.numpy().copy() for t in (AV, BV, T)],
                   [t.numpy().copy() for t in (AV2, BV2, T2)]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_tables_buffer_allreduce():
    """The multi-GPU step's [AV | BV | T] buffer (product_buffers with
    n_tables > 0, T = the Gram-table partials of geig_products_cca_tables) is
    summed over ranks by allreduce_products — in place when adjacent, through
    a stacked copy otherwise — and every rank ends with the same sums
    (Appendix F)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tables_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, mine, inplace, stacked = q.get(timeout=120)
        res[r] = (mine, inplace, stacked)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [res[0][0][i] + res[1][0][i] for i in range(3)]
    for r in range(world):
        for i in range(3):
            np.testing.assert_allclose(res[r][1][i], want[i], rtol=0, atol=1e-14)
            np.testing.assert_allclose(res[r][2][i], want[i], rtol=0, atol=1e-14)


def _owned_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_04993_b200.parallel import allgather_blocks, reduce_scatter_chunks
        chunk = 7
        g = torch.Generator().manual_seed(200 + rank)
        buf = torch.randn(world * chunk, generator=g, dtype=torch.float64)
        mine = buf.clone()
        out = torch.empty(chunk, dtype=torch.float64)
        reduce_scatter_chunks(buf, out)
        blocks = torch.full((world, 2, 3, 5), -1.0, dtype=torch.float64)
        blocks[rank] = rank + torch.arange(30, dtype=torch.float64).view(2, 3, 5)
        allgather_blocks(blocks)
        out_q.put((rank, mine.numpy(), out.numpy(), blocks.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world3_column_owned_collectives():
    """Host plumbing of the column-owned step (parallel.ColumnOwnedStep):
    the reduce-scatter of per-owner chunks gives rank r the sum of every
    rank's chunk r; the all-gather of shadow blocks gives every rank every
    owner's block."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_owned_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, mine, out, blocks = q.get(timeout=120)
        res[r] = (mine, out, blocks)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    chunk = 7
    total = sum(res[r][0] for r in range(world))
    for r in range(world):
        np.testing.assert_allclose(res[r][1], total[r * chunk:(r + 1) * chunk], rtol=0, atol=1e-12)
        for q_ in range(world):
            np.testing.assert_array_equal(res[r][2][q_], q_ + np.arange(30.0).reshape(2, 3, 5))


def _peer_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_04993_b200.parallel import exchange_peer_pointers
        # stand-ins for CUDA IPC: a "handle" names (rank, pointer); opening it
        # maps to a distinct address so the assembled table is checkable
        local = [1000 * rank + 1, 1000 * rank + 2, 1000 * rank + 3]
        handle = lambda p: ("h", rank, p)
        opened_log = []

        def open_fn(h):
            opened_log.append(h)
            return 10 ** 6 + h[2]

        table, opened = exchange_peer_pointers(local, world, rank, handle, open_fn)
        out_q.put((rank, table, opened, opened_log))
    finally:
        dist.destroy_process_group()


def test_gloo_world3_peer_pointer_exchange():
    """Host plumbing of the peer exchange (parallel.exchange_peer_pointers):
    every rank ends with, per buffer kind, `world` pointers in rank order —
    its own pointers in its own slot, every other rank's handle opened once
    (the CUDA IPC calls are injected, exactly where PeerColumnOwnedStep
    passes geig_ipc_handle / geig_ipc_open)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, table, opened, log = q.get(timeout=120)
        res[r] = (table, opened, log)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        table, opened, log = res[r]
        for j in range(3):
            for q_ in range(world):
                want = 1000 * r + j + 1 if q_ == r else 10 ** 6 + 1000 * q_ + j + 1
                assert table[j][q_] == want
        assert len(opened) == 3 * (world - 1) and all(h[1] != r for h in log)
