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
