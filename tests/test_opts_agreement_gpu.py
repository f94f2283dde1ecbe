"""Every rank of a communicator must run the same kernel for the same launch,
so the kernel-selecting options (lagom_comm_opts_t: coresident, one_hop,
a2a_tma, use_tma, steps, max_channels, max_chunk_bytes) must agree: the
import step compares each peer's heap header with its own and fails loudly
on a mismatch (instead of two ranks waiting on flags the other never
writes). Two processes share one GPU here; no kernel is launched."""
import os
import socket

import pytest

from tests.conftest import cuda_available

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, mismatch, q):
    import torch.distributed as dist
    from paper_2602_20656_b200 import coll as C
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    kw = {"coresident": rank} if mismatch else {}
    comm = C.Communicator(rank, 2, 0, max_channels=4, max_chunk_bytes=1 << 20, **kw)
    handles = [None, None]
    dist.all_gather_object(handles, comm.export_handle())
    try:
        comm.import_handles(handles)
        q.put((rank, "ok"))
    except C.LagomError as e:
        q.put((rank, e.code + ": " + str(e)))
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mismatch", [False, True])
def test_peer_options_must_agree(mismatch):
    if not cuda_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, mismatch, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    got = dict(q.get(timeout=10) for _ in range(2))
    if mismatch:
        for r in range(2):
            assert got[r].startswith("INVALID_INPUT") and "different options" in got[r], got
    else:
        assert got == {0: "ok", 1: "ok"}
