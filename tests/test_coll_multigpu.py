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


@pytest.mark.parametrize("variant", ["p2p", "nvls", "nvls-deep", "nvls-a2a-lsu"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_real_multigpu_parity(world, variant):
    """nvls: buffers in a multicast region, so TREE AllReduce runs inside
    the NVSwitch (int32 and movement bit-exact; fp sums within the stated
    bound of the fp64 exact sum, since the switch accumulates in fp32 in its
    own order). nvls = the co-resident kernels (default), nvls-deep = the
    deep-unroll ones (coresident = 0), nvls-a2a-lsu = the vector-store AllToAll
    at every NT (a2a_tma = 0; the default moves large-NT AllToAll with TMA)."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ)
    if variant != "p2p":
        env["LAGOM_NVLS"] = "1"
    if variant == "nvls-deep":
        env["LAGOM_CORESIDENT"] = "0"
    if variant == "nvls-a2a-lsu":
        env["LAGOM_A2A_TMA"] = "0"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_coll_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("a2a_tma", [1, 0])
@pytest.mark.parametrize("world", [2, 4])
def test_real_multigpu_parity_one_hop_allgather_reducescatter(world, a2a_tma):
    """TREE AllGather and ReduceScatter over the peer mappings instead of the
    switch (LAGOM_ONE_HOP=1): bit-exact (the ReduceScatter combines in the
    ring order). a2a_tma = 1: TMA bulk stores (AG) and the TMA pull (RS) at
    NT > 256, vector stores / the push into the owners' scratch at NT <= 256;
    a2a_tma = 0: the vector kernels at every NT."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, LAGOM_NVLS="1", LAGOM_ONE_HOP="1", LAGOM_A2A_TMA=str(a2a_tma))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_coll_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("one_hop", [0, 1])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_real_multigpu_parity_bench_sizes(world, one_hop):
    """The bench's own collectives at BASELINE sizes on real peers with NVLS
    on (TREE = in-switch AR/AG/RS, or with one_hop the peer-store AllGather
    and the TMA pull ReduceScatter at NT 512; one-hop A2A; RING = P2P rings),
    NC 8/16, NT 512, C 2 MiB: bit-exact, or within the fp64-exact-sum bound
    for the switch's fp32 sums."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, LAGOM_NVLS="1", LAGOM_BENCH_SIZES="1", LAGOM_ONE_HOP=str(one_hop))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_coll_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1800, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
