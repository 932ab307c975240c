"""Multi-process parity of the distributed executors (tests/dist_exec_check.py
under torchrun): 1.5D SAGE in every fetch mode (NCCL row fetch,
owner-computes, peer-memory owner sampling, batch split), LADIES race on the
grid and the NCCL / peer-memory feature fetch, all bit-identical to the
single-GPU results, on block-only partitions (gb_rmat_block).  With >= 2
GPUs over NCCL; on any GPU box also two processes sharing one GPU over gloo
(exchanges staged through host memory: the message-based modes)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _gpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("procs", [2, 4])
def test_distributed_executors_processes_sharing_one_gpu(procs):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={procs}",
           "--master-addr", "127.0.0.1", "--master-port", str(29593 + procs),
           os.path.join(HERE, "dist_exec_check.py")]
    env = dict(os.environ, GB_DIST_BACKEND="gloo")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(HERE), env=env)
    assert r.returncode == 0 and "ALL PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.skipif(_gpus() < 2, reason="needs at least 2 GPUs")
def test_distributed_executors_match_serial():
    n = 4 if _gpus() >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29591",
           os.path.join(HERE, "dist_exec_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(HERE))
    assert r.returncode == 0 and "ALL PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
