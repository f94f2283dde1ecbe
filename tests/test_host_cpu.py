"""CPU-side tests of the B200 layer's host code: the C-ABI library loads and
exports every symbol include/lagom_coll.h declares (no compute without a GPU),
argument accounting, and the multi-rank host path (shm coordinator) at
world_size 2 with a gloo rendezvous."""
import ctypes
import json
import os
import re
import secrets

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.conftest import ROOT


def header_symbols():
    with open(os.path.join(ROOT, "include", "lagom_coll.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(lagom_\w+)\(", text, re.M)))


def test_coll_library_exports_every_declared_symbol():
    from paper_2602_20656_b200 import coll as C
    lib = C.library()
    syms = header_symbols()
    assert len(syms) >= 17
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(C.EXPORTED_SYMBOLS) <= set(syms)
    assert lib.lagom_coll_abi_version() == 2


def test_other_libraries_load():
    for so in ("liblagom.so", "liblagom_b200.so"):
        ctypes.CDLL(os.path.join(ROOT, "paper_2602_20656_b200", so))
    from paper_2602_20656_b200 import _lagom_py as L
    assert L.version == "0.1.0"


def test_bus_bytes_accounting():
    from paper_2602_20656_b200 import coll as C
    assert C.coll_bytes(C.ALL_REDUCE, C.BF16, 1000, 8) == (2000, pytest.approx(2 * 7 / 8))
    assert C.coll_bytes(C.ALL_GATHER, C.F32, 10, 4) == (160, pytest.approx(3 / 4))
    assert C.coll_bytes(C.REDUCE_SCATTER, C.I32, 10, 2) == (80, pytest.approx(0.5))
    assert C.coll_bytes(C.ALL_TO_ALL, C.F16, 8, 8) == (128, pytest.approx(7 / 8))


def test_status_strings_and_errors_without_gpu():
    from paper_2602_20656_b200 import coll as C
    lib = C.library()
    assert lib.lagom_status_string(0) == b"ok"
    assert b"timeout" in lib.lagom_status_string(4)
    with pytest.raises(C.LagomError) as e:
        C.Communicator(5, 2, 0)  # rank out of range: rejected before touching CUDA
    assert e.value.code == "INVALID_INPUT"
    # NVLS peer-mapping entry points reject a null communicator without CUDA
    blob = ctypes.create_string_buffer(64)
    assert lib.lagom_comm_nvls_export_peer(None, blob) == 1
    assert lib.lagom_comm_nvls_import_peers(None, blob) == 1
    assert lib.lagom_comm_nvls_use_peers(None, 1) == 1


def test_config_mapping_from_reference_json():
    from paper_2602_20656_b200 import coll as C
    cfg = C.CollConfig.from_reference({"algorithm": "TREE", "protocol": "LL128", "transport": "P2P",
                                       "num_channels": 17, "num_threads": 640, "chunk_size": 289792})
    assert (cfg.algorithm, cfg.protocol, cfg.num_channels, cfg.num_threads, cfg.chunk_size) == \
           (C.TREE, C.LL128, 17, 640, 289792)
    with pytest.raises(C.LagomError):
        C.CollConfig.from_reference({"algorithm": "RING", "protocol": "LL", "transport": "NET",
                                     "num_channels": 1, "num_threads": 64, "chunk_size": 32768})


def _coord_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tok = [secrets.token_hex(6) if rank == 0 else None]
    dist.broadcast_object_list(tok, src=0)
    from paper_2602_20656_b200 import _lagom_py as L
    out = json.loads(L.coord_selftest(f"lagom_test_{tok[0]}", rank, world, 4))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shm_coordinator_multiprocess(world):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_coord_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, rounds in results.items():
        for k, rec in enumerate(rounds):
            assert rec["msg"] == f"round-{k}-of-{world}"
            assert rec["gathered"] == [100 * q_ + k for q_ in range(world)]
            assert rec["max"] == [world - 1, 0.0, 1.5 * (world - 1) + k]


def test_reference_arm_times_every_comm_op(root):
    """bench.py --impl reference: the reference's CPU path (the CPU collective
    restatement over every comm op of the iteration, prefaulted rotating
    buffers) prints the bench line contract with the Lagom arm's metric,
    unit and workload config, and a cpu_baseline describing the run."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    sys.path.insert(0, root)
    import bench
    from paper_2602_20656_b200 import dags
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == "ms"
    assert line["config"] == bench.workload_config(dags.BUILDERS["gpt2-1.3b-dp"](1))
    assert line["value"] > 0 and line["higher_is_better"] is False
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert "all 96 comm ops" in cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
