"""Bit-exact parity of the sm_100a collective kernels against the CPU oracle,
on one GPU with all ranks emulated (virtual mode: one cooperative launch per
collective, every rank's CTAs co-resident, per-rank heaps on the device).

Parity bar: every output byte equals the oracle's for every dtype (fp32,
bf16, fp16 and int32), because the oracle reproduces the kernels' fixed
reduction order (oracle/coll_oracle.c header)."""
import numpy as np
import pytest

from tests.conftest import cuda_available
from tests import coll_cases
from tests.oracle_ref import collective as oracle_collective, out_elems

pytestmark = pytest.mark.gpu

CASES = coll_cases.cases([1, 2, 3, 4, 8], seed=1234, per_combo=1)


@pytest.fixture(scope="module")
def vcomms():
    if not cuda_available():
        pytest.skip("no CUDA device")
    from paper_2602_20656_b200 import coll as C
    comms = {n: C.VirtualCommunicator(n, 0, max_channels=32, max_chunk_bytes=1 << 20, timeout_ms=5000)
             for n in (1, 2, 3, 4, 8)}
    yield comms
    for c in comms.values():
        c.close()


GUARD = 4096  # bytes of canary on both sides of every output buffer


def run_virtual(vc, c, sends_np):
    """One virtual launch. Besides the result it checks what compute-sanitizer
    would (closed on this pool): no byte outside an output buffer is written
    (canary bands on both sides) and no input byte changes."""
    import torch
    from paper_2602_20656_b200 import coll as C
    n = c["n"]
    dev = [torch.from_numpy(s).cuda() for s in sends_np]
    nbytes = out_elems(c["coll"], n, c["count"]) * sends_np[0].itemsize
    bases = [torch.full((GUARD + nbytes + GUARD,), 0x5A, dtype=torch.uint8, device="cuda") for _ in range(n)]
    for b in bases:
        b[GUARD:GUARD + nbytes].fill_(0xAB)  # poison: every byte must be written
    outs = [b[GUARD:GUARD + nbytes].view(dev[0].dtype) for b in bases]
    cfg = C.CollConfig(c["algo"], c["proto"], c["nc"], c["nt"], c["chunk"])
    vc.launch(c["coll"], cfg, c["dtype"], c["count"], [t.data_ptr() for t in dev],
              [t.data_ptr() for t in outs], torch.cuda.current_stream().cuda_stream, c["op"])
    torch.cuda.synchronize()
    vc.check()
    for r, b in enumerate(bases):
        assert bool((b[:GUARD] == 0x5A).all()) and bool((b[GUARD + nbytes:] == 0x5A).all()), \
            f"rank {r}: write outside the output buffer"
        assert dev[r].cpu().numpy().tobytes() == sends_np[r].tobytes(), f"rank {r}: input modified"
    return [o.cpu().numpy() for o in outs]


@pytest.mark.parametrize("case", CASES, ids=[coll_cases.case_id(c) for c in CASES])
def test_virtual_parity(vcomms, case):
    sends = coll_cases.inputs(case)
    want = oracle_collective(case["coll"], case["algo"], case["dtype"], case["op"], sends)
    got = run_virtual(vcomms[case["n"]], case, sends)
    for r in range(case["n"]):
        assert got[r].tobytes() == want[r].tobytes(), f"rank {r} differs"


def test_counters_stay_in_lockstep_across_configs(vcomms):
    """Back-to-back launches with changing NC/NT/C/protocol on the same comm
    (what the tuner does between profile calls) keep every connection's step
    counters consistent."""
    from paper_2602_20656_b200 import coll as C
    rng = np.random.default_rng(5)
    for i in range(40):
        nc, nt, ch = coll_cases.CONFIGS[i % len(coll_cases.CONFIGS)]
        c = dict(coll=C.ALL_REDUCE, algo=i % 2, proto=i % 3, n=4, dtype=0, op=0, nc=min(nc, 32),
                 nt=nt, chunk=ch, count=int(rng.integers(1, 200000)), seed=i)
        sends = coll_cases.inputs(c)
        want = oracle_collective(c["coll"], c["algo"], 0, 0, sends)
        got = run_virtual(vcomms[4], c, sends)
        assert got[0].tobytes() == want[0].tobytes()


def test_invalid_configs_fail_loudly(vcomms):
    from paper_2602_20656_b200 import coll as C
    vc = vcomms[2]
    for bad in (C.CollConfig(C.RING, C.SIMPLE, 0, 64, 32768),
                C.CollConfig(C.RING, C.SIMPLE, 33, 64, 32768),
                C.CollConfig(C.RING, C.SIMPLE, 1, 100, 32768),
                C.CollConfig(C.RING, C.SIMPLE, 1, 64, 1000),
                C.CollConfig(C.RING, C.SIMPLE, 1, 64, 2 << 20)):
        with pytest.raises(C.LagomError) as e:
            vc.launch(C.ALL_REDUCE, bad, 0, 16, [0, 0], [0, 0])
        assert e.value.code == "INVALID_WORKLOAD"


TMA_CASES = [c for c in coll_cases.cases([2, 4], seed=77, per_combo=1) if c["proto"] == 0]


@pytest.mark.parametrize("use_tma", [0, 2])
@pytest.mark.parametrize("case", TMA_CASES, ids=[coll_cases.case_id(c) for c in TMA_CASES])
def test_virtual_parity_data_paths(case, use_tma):
    """SIMPLE with the data path forced: 0 = vector ld/st only, 2 = TMA bulk
    copies for copy AND reduction steps (warp-specialized smem pipeline)."""
    if not cuda_available():
        pytest.skip("no CUDA device")
    from paper_2602_20656_b200 import coll as C
    vc = C.VirtualCommunicator(case["n"], 0, max_channels=32, max_chunk_bytes=1 << 20, timeout_ms=5000,
                               use_tma=use_tma)
    try:
        sends = coll_cases.inputs(case)
        want = oracle_collective(case["coll"], case["algo"], case["dtype"], case["op"], sends)
        got = run_virtual(vc, case, sends)
        for r in range(case["n"]):
            assert got[r].tobytes() == want[r].tobytes(), f"rank {r} differs"
    finally:
        vc.close()


@pytest.mark.parametrize("offset_elems", [1, 3, 8])
@pytest.mark.parametrize("proto", [0, 1, 2])
@pytest.mark.parametrize("coll,algo", [(0, 0), (0, 1), (1, 0), (2, 0), (3, 0)])
def test_misaligned_user_buffers(vcomms, coll, algo, proto, offset_elems):
    """User buffers that start off a 16-byte boundary (torch views at an
    element offset) take the byte-granular load/store paths and bypass TMA;
    results must still be bit-exact."""
    import torch
    from paper_2602_20656_b200 import coll as C
    from tests.oracle_ref import in_elems
    n, dtype, count = 3, C.BF16, 5000 + 7
    rng = np.random.default_rng(coll * 100 + proto * 10 + offset_elems)
    from tests.oracle_ref import random_input
    sends = [random_input(dtype, in_elems(coll, n, count), rng) for _ in range(n)]
    want = oracle_collective(coll, algo, dtype, 0, sends)
    dev, outs, guards = [], [], []
    for s in sends:
        base = torch.zeros(s.size + offset_elems, dtype=torch.uint16, device="cuda")
        base[offset_elems:] = torch.from_numpy(s).cuda()
        dev.append(base[offset_elems:])
        m = out_elems(coll, n, count)
        ob = torch.full((m + offset_elems + 64,), 0xABAB, dtype=torch.uint16, device="cuda")
        ob[:offset_elems] = 0x5A5A
        ob[offset_elems + m:] = 0x5A5A  # canaries on both sides
        guards.append(ob)
        outs.append(ob[offset_elems:offset_elems + m])
    cfg = C.CollConfig(algo, proto, 4, 256, 8192)
    vcomms[n].launch(coll, cfg, dtype, count, [t.data_ptr() for t in dev], [t.data_ptr() for t in outs],
                     torch.cuda.current_stream().cuda_stream, 0)
    torch.cuda.synchronize()
    vcomms[n].check()
    for r in range(n):
        assert outs[r].cpu().numpy().tobytes() == want[r].tobytes()
        g = guards[r].cpu().numpy()
        assert (g[:offset_elems] == 0x5A5A).all() and (g[offset_elems + outs[r].numel():] == 0x5A5A).all()


def test_zero_count_is_a_no_op(vcomms):
    from paper_2602_20656_b200 import coll as C
    for coll in range(4):
        vcomms[2].launch(coll, C.CollConfig(C.RING, C.SIMPLE, 2, 64, 32768), C.F32, 0, [0, 0], [0, 0])
    vcomms[2].check()


NT_CLASSES = [64, 128, 192, 256, 384, 512, 576, 640]


@pytest.mark.parametrize("nt", NT_CLASSES)
@pytest.mark.parametrize("coll", [0, 1, 2, 3])
def test_single_rank_real_mode_is_a_copy(coll, nt):
    """nranks == 1 (the bench's N = 1 line): every collective is a copy of
    count elements through the co-resident copy kernel (local.cu), bit-exact
    against the oracle at n = 1, for every thread-count class, with src/dst
    co-aligned, mutually misaligned, and ragged byte counts."""
    if not cuda_available():
        pytest.skip("no CUDA device")
    import torch
    from paper_2602_20656_b200 import coll as C
    comm = C.Communicator(0, 1, 0, max_channels=64)
    try:
        rng = np.random.default_rng(coll * 1000 + nt)
        for dtype, count, soff, doff, nc in [(1, 25 << 19, 0, 0, 8), (0, 300003, 0, 0, 3), (1, 4099, 1, 1, 2),
                                             (2, 100001, 1, 3, 64), (3, 7, 0, 0, 1), (1, 1 << 20, 0, 5, 17)]:
            from tests.oracle_ref import random_input
            x = random_input(dtype, count, rng)
            want = oracle_collective(coll, 0, dtype, 0, [x])[0]
            esz = x.itemsize
            sbase = torch.zeros((count + soff + 8) * esz, dtype=torch.uint8, device="cuda")
            src = sbase[soff * esz:(soff + count) * esz]
            src.copy_(torch.from_numpy(x.view(np.uint8)).cuda())
            dbase = torch.full(((count + doff + 64) * esz,), 0x5A, dtype=torch.uint8, device="cuda")
            dst = dbase[doff * esz:(doff + count) * esz]
            dst.fill_(0xAB)
            comm.launch(coll, C.CollConfig(C.TREE, C.SIMPLE, nc, nt, 2 << 20), dtype, count, src.data_ptr(),
                        dst.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            comm.check()
            assert dst.cpu().numpy().tobytes() == want.view(np.uint8).tobytes()
            g = dbase.cpu().numpy()
            assert (g[:doff * esz] == 0x5A).all() and (g[(doff + count) * esz:] == 0x5A).all()
        # in place: no launch, data untouched
        buf = torch.arange(1000, dtype=torch.int32, device="cuda")
        comm.launch(coll, C.CollConfig(C.RING, C.SIMPLE, 4, nt, 1 << 20), C.I32, 1000, buf.data_ptr(),
                    buf.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(buf, torch.arange(1000, dtype=torch.int32, device="cuda"))
    finally:
        comm.close()


def test_launches_on_one_comm_keep_issue_order_across_streams(vcomms):
    """Two collectives on one communicator issued on two streams: the second
    waits for the first (they share step counters), both bit-exact."""
    import torch
    from paper_2602_20656_b200 import coll as C
    vc = vcomms[4]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs, wants = [], []
    for i, st in enumerate((s1, s2, s1, s2)):
        c = dict(coll=C.ALL_REDUCE, algo=C.RING, proto=i % 3, n=4, dtype=0, op=0, nc=4, nt=256, chunk=65536,
                 count=200003, seed=40 + i)
        sends = coll_cases.inputs(c)
        wants.append(oracle_collective(C.ALL_REDUCE, C.RING, 0, 0, sends)[0])
        dev = [torch.from_numpy(s).cuda() for s in sends]
        torch.cuda.synchronize()
        out = [torch.empty_like(d) for d in dev]
        vc.launch(C.ALL_REDUCE, C.CollConfig(C.RING, i % 3, 4, 256, 65536), 0, 200003,
                  [t.data_ptr() for t in dev], [t.data_ptr() for t in out], st.cuda_stream, 0)
        outs.append((dev, out))
    torch.cuda.synchronize()
    vc.check()
    for (dev, out), want in zip(outs, wants):
        assert out[0].cpu().numpy().tobytes() == want.tobytes()
