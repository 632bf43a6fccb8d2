"""The NCCL calls of parallel.py executed on the one GPU there is: a
world-size-1 NCCL process group runs every collective wrapper of the
multi-GPU steps (in-place all-reduce of [AV | BV | T], reduce-scatter of the
per-owner chunks, in-place all-gather of the int16 shadow blocks, dense
all-gather of column blocks) with the dtypes, views and strides the bench
passes, so an argument the NCCL binding rejects (an unmapped dtype, a
non-contiguous view, a size mismatch) fails here and not on the 8-GPU box.
With one rank every collective is the identity, which is what is asserted;
the sums over ranks are covered by the gloo tests (test_parallel_gloo.py)
and the emulated-rank GPU tests (test_gpu_owned.py)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    assert torch.cuda.is_available()
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    yield
    dist.destroy_process_group()


def test_nccl_collective_wrappers_accept_the_bench_arguments(nccl_world1):
    from paper_2206_04993_b200 import parallel as par
    dev = "cuda:0"
    k, d, nt = 16, 512, 152
    g = torch.Generator(device=dev).manual_seed(3)

    # replicated step: one in-place all-reduce over AV | BV | T of one buffer.
    # (allreduce_products returns early at world 1, so call the collective on
    # the exact flat view it builds)
    AV, BV, T = par.product_buffers(k, d, nt, device=dev)
    for t in (AV, BV, T):
        t.copy_(torch.randn(t.shape, device=dev, generator=g))
    ref = torch.cat([AV.reshape(-1), BV.reshape(-1), T]).clone()
    flat = AV.as_strided((2 * k * d + nt,), (1,))
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    par.allreduce_products(AV, BV, T=T)
    torch.cuda.synchronize()
    assert torch.equal(flat, ref)

    # column-owned step: reduce-scatter of the chunks, all-gather of the
    # int16 shadow blocks [world, 2, k, W] in place
    chunk = 2 * k * d + nt
    buf = torch.randn(1 * chunk, device=dev, generator=g)
    mine = torch.empty(chunk, device=dev)
    par.reduce_scatter_chunks(buf, mine)
    shadow = torch.randint(-30000, 30000, (1, 2, k, d), dtype=torch.int16, device=dev, generator=g)
    want = shadow.clone()
    par.allgather_blocks(shadow)
    # fp32 blocks (gather_state)
    blocks = torch.randn(1, k, d, device=dev, generator=g)
    bwant = blocks.clone()
    par.allgather_blocks(blocks)
    torch.cuda.synchronize()
    assert torch.equal(mine, buf) and torch.equal(shadow, want) and torch.equal(blocks, bwant)

    # dense: all-gather of the ranks' column blocks (the wrapper returns early
    # at world 1; run its collective on the tensors it builds)
    send = torch.randn(2, k, d, device=dev, generator=g)
    recv = [torch.empty_like(send)]
    dist.all_gather(recv, send)
    t = torch.tensor([1.0, 2.0, 3.0], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)      # the bench's max-over-ranks timing
    dist.barrier()
    torch.cuda.synchronize()
    assert torch.equal(recv[0], send) and t.tolist() == [1.0, 2.0, 3.0]
