"""Multi-GPU host logic (one process per GPU, torch.distributed over NCCL).

Appendix F: "we parallelized the estimation of the
matrix-vector products Av_i and Bv_i for all i and then aggregated this
information across machines".  Each rank owns a shard of the minibatch rows
(CCA) or of the matrix rows (dense), computes its partial products, and the
partials are combined by an all-reduce (sum); every rank then applies the
same update to its replica of V and [Bv].  The compute callables are
injected so the orchestration can be exercised on CPU with gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist


def product_buffers(k: int, d: int, n_tables: int = 0, **kw):
    """AV, BV as the two halves of ONE contiguous buffer, so the Appendix-F
    all-reduce runs in place on both (no stack / copy-back); with n_tables > 0
    a third view T of n_tables floats follows them in the same buffer (the
    Gram-table partials of geig_products_cca_tables) and is returned too."""
    kd = k * d
    buf = torch.empty(2 * kd + n_tables, **kw)
    AV, BV = buf[:kd].view(k, d), buf[kd:2 * kd].view(k, d)
    if n_tables:
        return AV, BV, buf[2 * kd:]
    return AV, BV


def allreduce_products(AV: torch.Tensor, BV: torch.Tensor, group=None, T: torch.Tensor | None = None):
    """SUM all-reduce of the partial products (and table partials T) of every
    rank: in place when AV, BV (, T) are adjacent in one buffer
    (product_buffers), else one fused all-reduce of a stacked copy."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return
    n = AV.numel()
    es = AV.element_size()
    adjacent = (AV.is_contiguous() and BV.is_contiguous() and AV.dtype == BV.dtype and BV.numel() == n
                and BV.data_ptr() == AV.data_ptr() + n * es)
    if T is not None:
        adjacent = adjacent and T.is_contiguous() and T.dtype == AV.dtype and T.data_ptr() == AV.data_ptr() + 2 * n * es
    if adjacent:
        flat = AV.as_strided((2 * n + (T.numel() if T is not None else 0),), (1,))
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    elif T is not None:
        flat = torch.cat([AV.reshape(-1), BV.reshape(-1), T.reshape(-1)])
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        AV.copy_(flat[:n].view_as(AV))
        BV.copy_(flat[n:2 * n].view_as(BV))
        T.copy_(flat[2 * n:])
    else:
        flat = torch.stack([AV, BV])
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        AV.copy_(flat[0])
        BV.copy_(flat[1])


def shard_rows(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range [r0, r1) of `rank`; sizes differ by at most one."""
    base, rem = divmod(n_rows, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


@dataclass
class ShardedStep:
    """One Appendix-F step.  products(AV, BV) writes this rank's partial
    products (already scaled so that the SUM over ranks is the global
    estimate); update(AV, BV) applies Alg. 2 lines 8-19 locally."""
    products: Callable[[torch.Tensor, torch.Tensor], None]
    update: Callable[[torch.Tensor, torch.Tensor], None]
    group: object = None

    def __call__(self, AV: torch.Tensor, BV: torch.Tensor):
        self.products(AV, BV)
        allreduce_products(AV, BV, self.group)   # one fused all-reduce of the two k x d products
        self.update(AV, BV)


def cca_scale(b_local: int, world: int) -> float:
    """Each rank holds b_local rows split into halves (reading R1); the global
    A_t / B_t average over world * (b_local // 2) rows per half."""
    return 1.0 / (world * (b_local // 2))


def dense_allgather_rows(AV: torch.Tensor, BV: torch.Tensor, d: int, world: int, group=None):
    """Dense row sharding (configs 0, 4: A, B row-sharded across ranks):
    rank r wrote columns [r0, r1) = shard_rows(d, world, r) of AV, BV (the
    products of its rows of A, B with every v_j, geig_products_dense).  One
    all-gather of the ranks' column blocks (packed contiguous, padded to
    ceil(d / world) columns) assembles the full k x d products on every rank:
    each rank sends 2 k (d / world) floats and receives the rest — half the
    wire bytes of a SUM all-reduce of zero-padded k x d buffers."""
    if world <= 1:
        return
    rank = dist.get_rank(group)
    k = AV.shape[0]
    w = (d + world - 1) // world
    r0, r1 = shard_rows(d, world, rank)
    send = torch.zeros(2, k, w, dtype=AV.dtype, device=AV.device)
    send[0, :, :r1 - r0] = AV[:, r0:r1]
    send[1, :, :r1 - r0] = BV[:, r0:r1]
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    for q in range(world):
        q0, q1 = shard_rows(d, world, q)
        if q != rank:
            AV[:, q0:q1] = recv[q][0, :, :q1 - q0]
            BV[:, q0:q1] = recv[q][1, :, :q1 - q0]


def dense_wire_bytes(k: int, d: int, world: int, elem: int = 4) -> dict:
    """Bytes each rank sends per dense step: all-gather of its column block
    of AV, BV vs the (ring) all-reduce of the full buffers it replaces."""
    w = (d + world - 1) // world
    return {"allgather_send": 2 * k * w * elem * (world - 1),
            "allreduce_ring_send": 2 * 2 * k * d * elem * (world - 1) // world}


# ---------------------------------------------------------------------------
# Column-owned step (geig_set_partition): reduce-scatter + all-gather
# ---------------------------------------------------------------------------

def reduce_scatter_chunks(buf: torch.Tensor, out: torch.Tensor, group=None):
    """Sum buf (world chunks, chunk r for rank r) over the ranks into `out`
    (this rank's summed chunk).  NCCL: one reduce-scatter; backends without
    it (gloo): an all-reduce of the buffer and a copy of the own chunk."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    chunks = buf.view(world, -1)
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, buf, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        out.copy_(chunks[rank])


def allgather_blocks(blocks: torch.Tensor, group=None):
    """blocks: [world, ...] with this rank's block current; afterwards every
    block is the owner's.  NCCL: one in-place all-gather; gloo: through
    host copies."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "nccl":
        # raw bytes: the shadow is an int16 view, a dtype torch's NCCL binding
        # does not map; the in-place form (input = this rank's slice of the
        # output) moves no local copy
        raw = blocks.view(torch.uint8) if blocks.element_size() == 2 else blocks
        dist.all_gather_into_tensor(raw.view(-1), raw[rank].reshape(-1), group=group)
    else:
        # host copies as raw bytes (gloo has no int16 / bf16 all-gather)
        raw = blocks.view(torch.uint8) if blocks.element_size() == 2 else blocks
        mine = raw[rank].cpu()
        got = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(got, mine, group=group)
        for q in range(world):
            if q != rank:
                raw[q].copy_(got[q])


def owned_wire_bytes(k: int, d: int, world: int, n_tables: int) -> dict:
    """Bytes each rank sends per step: reduce-scatter of [AV | BV | tables]
    chunks (fp32) + all-gather of the bf16 hi / lo shadow blocks, vs the
    ring all-reduce of [AV | BV | tables] of the replicated step."""
    W = d // world
    chunk = 2 * k * W + n_tables
    return {"reduce_scatter_send": 4 * chunk * (world - 1),
            "allgather_send": 2 * 2 * k * W * (world - 1),
            "allreduce_ring_send": 2 * 4 * (2 * k * d + n_tables) * (world - 1) // world}


class ColumnOwnedStep:
    """One column-owned multi-GPU step of Alg. 2 for a partitioned solver
    (geig_set_partition(world, rank)): products of the rank's rows (one
    launch) -> reduce-scatter of the per-owner chunks -> update of the own
    columns -> all-gather of the bf16 shadow blocks that the next forward
    reads (Appendix F)."""

    def __init__(self, geig, solver, world: int, rank: int, group=None):
        self.g, self.s, self.world, self.rank, self.group = geig, solver, world, rank, group
        self.k, self.d = solver.k, solver.d
        self.W = self.d // world
        self.chunk = geig.geig_owned_chunk_floats(solver.h)
        dev = f"cuda:{solver.device}"
        self.buf = torch.empty(world * self.chunk, device=dev)
        self.mine = torch.empty(self.chunk, device=dev)
        self.shadow = geig.shadow_tensor(solver.h, world, self.k, self.W, solver.device)

    def __call__(self, X, Y, b: int, eta: float, gamma: float):
        g = self.g
        g.geig_products_cca_owned(self.s.h, X, Y, b, cca_scale(b, self.world), self.buf)
        reduce_scatter_chunks(self.buf, self.mine, self.group)
        g.geig_update_owned(self.s.h, self.mine, eta, gamma)
        allgather_blocks(self.shadow, self.group)

    def gather_state(self):
        """The retracted V (unit rows) and [Bv] assembled from every rank's
        own columns (not on the hot path)."""
        V, AUX = self.s.state()
        Vb = V.view(self.k, self.world, self.W).permute(1, 0, 2).contiguous()
        Ab = AUX.view(self.k, self.world, self.W).permute(1, 0, 2).contiguous()
        allgather_blocks(Vb, self.group)
        allgather_blocks(Ab, self.group)
        V = Vb.permute(1, 0, 2).reshape(self.k, self.d)
        AUX = Ab.permute(1, 0, 2).reshape(self.k, self.d)
        return V / V.norm(dim=1, keepdim=True), AUX


def exchange_peer_pointers(local: list[int], world: int, rank: int, handle_fn, open_fn, group=None):
    """CUDA IPC handshake of the peer exchange: `local` holds this rank's
    device pointers (receive slots, gathered shadow, flag words); every
    rank's handles are all-gathered and every OTHER rank's are mapped into
    this process.  Returns (per buffer kind, a list of `world` pointers in
    rank order; this rank's entries are its own pointers) and the list of
    mapped pointers to unmap at the end."""
    mine = [handle_fn(p) for p in local]
    got = [None] * world
    dist.all_gather_object(got, mine, group=group)
    opened = []
    table = [[0] * world for _ in local]
    for q in range(world):
        for j in range(len(local)):
            if q == rank:
                table[j][q] = local[j]
            else:
                ptr = open_fn(got[q][j])
                table[j][q] = ptr
                opened.append(ptr)
    return table, opened


class PeerColumnOwnedStep:
    """The column-owned step over NVLink peer memory (geig_set_peers): one
    process per GPU; the products launch stores every column's AV | BV and
    the table row into the owner's receive slot, the update launch sums the
    slots and writes its shadow block into every rank's gathered shadow —
    no NCCL call on the data path (Appendix F)."""

    def __init__(self, geig, solver, world: int, rank: int, group=None):
        self.g, self.s, self.world, self.rank = geig, solver, world, rank
        recv, _, flags, _ = geig.geig_peer_buffers(solver.h)
        shadow, _ = geig.geig_shadow_buffer(solver.h)
        (self.recv, self.shadow, self.flags), self.opened = exchange_peer_pointers(
            [recv, shadow, flags], world, rank, geig.geig_ipc_handle, geig.geig_ipc_open, group)
        geig.geig_set_peers(solver.h, self.recv, self.shadow, self.flags)

    def __call__(self, X, Y, b: int, eta: float, gamma: float):
        self.g.geig_step_cca_peer(self.s.h, X, Y, b, cca_scale(b, self.world), eta, gamma)

    def close(self):
        for p in self.opened:
            self.g.geig_ipc_close(p)
        self.opened = []
