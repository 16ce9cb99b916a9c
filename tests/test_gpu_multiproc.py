"""GPU: the sharded path as real processes (torchrun, 2 ranks) on one B200.

The gpurun pool gives one GPU, so both ranks share it (NCCL refuses two ranks
on one device): the process group is gloo and tpx_cluster_run_sharded uses
the library's host-callback transport (sharded.HostComm + TorchAdapter); the
kernels, the halo / pair / partial-record protocol and the process-level
plumbing are the ones a multi-GPU NCCL run uses.  Rank 0 checks the
concatenated outputs against the oracle bit for bit (tools/sharded_check.py).
"""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,preset,n", [(2, "mixed", 1_500_000), (3, "lowflux", 600_000)])
def test_torchrun_sharded_processes(world, preset, n):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, TPX_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "sharded_check.py"), str(n), preset]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout
