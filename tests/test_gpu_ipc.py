"""CUDA IPC plumbing of the peer-memory column-owned step with two processes
on one GPU (-m gpu): parallel.PeerColumnOwnedStep exchanges the handles of
every rank's receive slots, gathered shadow and flag words over gloo, maps
the other rank's buffers and hands the pointer tables to geig_set_peers.
Each process then writes a word into the OTHER rank's flag buffer through
the mapped pointer (a plain copy, no kernel that waits on the other
process: the two ranks' peer-step kernels would wait on each other and must
not share one GPU) and reads what the other wrote into its own buffer."""
import ctypes
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        from paper_2206_04993_b200 import geig
        from paper_2206_04993_b200.parallel import PeerColumnOwnedStep
        s = geig.Solver(geig.GEIG_CCA, 768, 768, 16, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=0.1,
                        max_rows=64)
        geig.geig_set_partition(s.h, 2, rank)
        step = PeerColumnOwnedStep(geig, s, 2, rank)
        rt = ctypes.CDLL("libcudart.so.12")
        val = ctypes.c_uint32(1000 + 7 * rank)
        # word 31 of the first flag line (padding, never a flag) of the other rank
        rt.cudaMemcpy(ctypes.c_void_p(step.flags[1 - rank] + 31 * 4), ctypes.byref(val), ctypes.c_size_t(4), 1)
        rt.cudaDeviceSynchronize()
        dist.barrier()
        got = ctypes.c_uint32(0)
        rt.cudaMemcpy(ctypes.byref(got), ctypes.c_void_p(step.flags[rank] + 31 * 4), ctypes.c_size_t(4), 2)
        own_ok = step.recv[rank] == geig.geig_peer_buffers(s.h)[0] and step.shadow[rank] == geig.geig_shadow_buffer(s.h)[0]
        dist.barrier()
        step.close()
        s.close()
        q.put((rank, got.value, own_ok, len(step.recv)))
    finally:
        dist.destroy_process_group()


def test_two_process_ipc_peer_setup():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2206_04993_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, got, own_ok, n = q.get(timeout=300)
        res[r] = (got, own_ok, n)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(2):
        got, own_ok, n = res[r]
        assert got == 1000 + 7 * (1 - r) and own_ok and n == 2
