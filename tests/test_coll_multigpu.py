"""Real NVLink multi-GPU parity (skipped unless >= 2 GPUs are visible)."""
import os
import socket
import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("nvls", [0, 1])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_real_multigpu_parity(world, nvls):
    """nvls=1: buffers in a multicast region, so TREE AllReduce runs inside
    the NVSwitch (int32 and movement bit-exact; fp sums within the stated
    tolerance, since the switch accumulates in fp32 in its own order)."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, LAGOM_NVLS="1") if nvls else dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_coll_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("world", [2, 4])
def test_real_multigpu_parity_one_hop_allgather_reducescatter(world):
    """TREE AllGather (peer stores) and ReduceScatter (peer loads, ring order;
    LAGOM_ONE_HOP=1) instead of
    the switch: bit-exact (the ReduceScatter combines in the ring order)."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, LAGOM_NVLS="1", LAGOM_ONE_HOP="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_coll_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
