"""Multi-rank paths on one GPU (gloo; functional and parity checks, never a
measurement): the Appendix-F step with 2 ranks sharing
cuda:0 vs the oracle, and `bench.py --gpus 2` re-executing itself under
torch.distributed.run with rank 0 printing one JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


@pytest.mark.parametrize("mode", ["replicated", "owned"])
def test_two_ranks_appendix_f_step_matches_oracle(mode):
    assert torch.cuda.is_available()
    from paper_2206_04993_b200 import build
    build.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "mr_step.py"), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = next(l for l in r.stdout.splitlines() if l.startswith("MR_RESULT "))
    res = json.loads(line[len("MR_RESULT "):])
    assert res["replicas_identical"], res
    assert res["step_err"] < 1e-3 and res["aux_err"] < 1e-4, res


def test_bench_gpus2_reexecs_under_torchrun():
    env = dict(os.environ, GEIG_BENCH_SHARE_GPU="1", GEIG_BENCH_BACKEND="gloo")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--spinup", "0", "--no-e2e", "--no-cpu-baseline", "--config", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["config"]["parallelism"] == "dp2"
    assert "torch.distributed.run" in r.stderr
