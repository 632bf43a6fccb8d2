"""Two-rank Appendix-F step on ONE GPU (argv[1]: "replicated" — the
all-reduce of [AV | BV | tables] — or "owned" — the column-owned
reduce-scatter / all-gather step of parallel.ColumnOwnedStep) (launched by tests/test_gpu_multirank.py
through torch.distributed.run, gloo backend — a functional and parity check
of the multi-rank path, never a measurement).  Each rank owns half of the
minibatch rows, runs geig_products_cca_tables on its shard, the partial
[AV | BV | T] buffers are summed across ranks (allreduce_products), and
every rank applies geig_update_tables to its replica.  Rank 0 gathers the
replicas, runs the oracle's Appendix-F step on the same
rows, and prints one JSON line with the errors."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    from paper_2206_04993_b200 import geig
    from paper_2206_04993_b200.parallel import allreduce_products, cca_scale, product_buffers
    from synth import CONFIGS, cca_views
    from tests.gpu_harness import floor_state
    cfg = CONFIGS[2]
    k, dx, dy, b, T = 16, 768, 768, 512, 3
    eta = 0.2
    x, y = cca_views(cfg, world * b * T, seed=31)
    x, y = x[:, :dx].contiguous(), y[:, :dy].contiguous()
    V, aux = floor_state(k, dx + dy, 7, cfg.rho)
    V = V.astype(np.float32).astype(np.float64)
    aux = aux.astype(np.float32).astype(np.float64)
    dev = "cuda:0"
    s = geig.Solver(geig.GEIG_CCA, dx, dy, k, math="bf16x2", data_dtype=geig.GEIG_DATA_BF16, rho=cfg.rho,
                    max_rows=b)
    s.set_state(torch.tensor(V, dtype=torch.float32, device=dev), torch.tensor(aux, dtype=torch.float32, device=dev))
    mode = sys.argv[1] if len(sys.argv) > 1 else "replicated"
    scale = cca_scale(b, world)
    if mode == "owned":
        from paper_2206_04993_b200.parallel import ColumnOwnedStep
        geig.geig_set_partition(s.h, world, rank)
        step = ColumnOwnedStep(geig, s, world, rank)
        for t in range(T):
            r0 = (t * world + rank) * b
            step(x[r0:r0 + b].to(dev).contiguous(), y[r0:r0 + b].to(dev).contiguous(), b, eta, cfg.gamma)
            geig.geig_sync(s.h)
        Vg, Ag = (t_.cpu() for t_ in step.gather_state())
    else:
        AV, BV, Tt = product_buffers(k, dx + dy, geig.geig_table_floats(s.h), device=dev)
        for t in range(T):
            r0 = (t * world + rank) * b
            xs, ys = x[r0:r0 + b].to(dev).contiguous(), y[r0:r0 + b].to(dev).contiguous()
            geig.geig_products_cca_tables(s.h, xs, ys, b, scale, AV, BV, Tt)
            geig.geig_sync(s.h)
            allreduce_products(AV, BV, T=Tt)
            geig.geig_update_tables(s.h, AV, BV, Tt, eta, cfg.gamma)
        Vg, Ag = (t_.cpu() for t_ in s.state())
    s.close()
    Vs = [torch.empty_like(Vg) for _ in range(world)]
    dist.all_gather(Vs, Vg)
    if rank == 0:
        from oracle import estimators, game
        Vo, Ao = V, aux
        for t in range(T):
            ms = []
            for r in range(world):
                r0 = (t * world + r) * b
                ms.append(estimators.cca_products(x[r0:r0 + b].double().numpy(), y[r0:r0 + b].double().numpy(), Vo))
            Vo, Ao = game.step_alg2_appendix_f(Vo, Ao, ms, eta, cfg.gamma, cfg.rho)
        Vg = Vg.double().cpu().numpy()
        out = {"world": world, "mode": mode,
               "step_err": float(np.linalg.norm(Vg - Vo) / np.linalg.norm(Vo - V)),
               "aux_err": float(np.linalg.norm(Ag.double().cpu().numpy() - Ao) / np.linalg.norm(Ao)),
               "replicas_identical": all(bool(torch.equal(Vs[0], v)) for v in Vs)}
        print("MR_RESULT " + json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
