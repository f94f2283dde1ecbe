"""Real multi-GPU parity check (one process per GPU, CUDA-IPC peer heaps over
NVLink/NVSwitch). Launched by tests/test_coll_multigpu.py via torchrun; every
rank rebuilds all ranks' seeded inputs, runs the kernel, and compares its own
output with the oracle bit for bit. Exit code = number of failing cases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_20656_b200 import coll as C  # noqa: E402
from tests import coll_cases  # noqa: E402
from tests.oracle_ref import collective as oracle_collective, in_elems, out_elems  # noqa: E402


# One ulp of the output type relative to |S| (2^-7 bf16, 2^-10 f16, 2^-23
# f32): the switch accumulates in fp32 (.acc::f32) but its conversion of the
# sum to bf16 is faithful, not correctly rounded — measured on 2xB200 up to
# 0.8 ulp off the fp64 sum, where round-to-nearest would be
# at most 0.5 ulp.
ULP = {0: 2.0 ** -23, 1: 2.0 ** -7, 2: 2.0 ** -10}


def within_tolerance(got, sends, c):
    """In-switch (NVLS) sums against the EXACT fp64 sum S of the inputs:
    |got - S| <= ulp_rel * |S| + n * 2^-23 * sum|x| — one faithful rounding
    to the output type plus fp32 accumulation of n terms."""
    from tests.test_oracle_cpu import to_f32
    g = to_f32(got, c["dtype"]).astype(np.float64)
    n = len(sends)
    if c["coll"] == C.ALL_REDUCE:
        parts = [to_f32(s, c["dtype"]).astype(np.float64) for s in sends]
    else:
        r = int(os.environ["RANK"])
        k = c["count"]
        parts = [to_f32(s[r * k:(r + 1) * k], c["dtype"]).astype(np.float64) for s in sends]
    exact = np.sum(parts, axis=0)
    mag = np.sum(np.abs(parts), axis=0)
    tol = ULP[c["dtype"]] * np.abs(exact) + n * 2.0 ** -23 * mag
    ok = bool(np.all(np.abs(g - exact) <= tol))
    if not ok:
        bad = np.flatnonzero(np.abs(g - exact) > tol)
        i = bad[np.argmax((np.abs(g - exact) / np.maximum(tol, 1e-30))[bad])]
        print(f"[tolerance] {bad.size} of {g.size} outside: worst i={i} got={g[i]!r} exact={exact[i]!r} "
              f"err/|S|={abs(g[i] - exact[i]) / max(abs(exact[i]), 1e-30):.3e} tol={tol[i]:.3e}", flush=True)
    return ok


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    use_tma = int(os.environ.get("LAGOM_USE_TMA", "1"))
    # kernel-selecting options, identical on every rank (checked at import)
    comm = C.Communicator.from_process_group(device=local, max_channels=32, max_chunk_bytes=4 << 20,
                                             timeout_ms=5000, use_tma=use_tma,
                                             one_hop=int(os.environ.get("LAGOM_ONE_HOP", "0")),
                                             a2a_tma=int(os.environ.get("LAGOM_A2A_TMA", "1")),
                                             coresident=int(os.environ.get("LAGOM_CORESIDENT", "1")))
    stream = torch.cuda.current_stream().cuda_stream
    nvls = bool(os.environ.get("LAGOM_NVLS")) and comm.nvls_supported()
    fails, checked = 0, 0
    cases = coll_cases.cases([world], seed=int(os.environ.get("LAGOM_CASE_SEED", "99")), per_combo=2,
                             tree_extra=True)
    for c in cases:
        c["nc"] = max(1, min(32, c["nc"] * 2))  # real mode: no co-residency cap
    if os.environ.get("LAGOM_BIG"):
        # large messages: many TMA tiles per step, many pieces per channel
        cases = [dict(coll=coll, algo=0, proto=0, n=world, dtype=dt, op=0, nc=nc, nt=640, chunk=ch,
                      count=cnt, seed=1000 + i)
                 for i, (coll, dt, nc, ch, cnt) in enumerate(
                     (coll, dt, nc, ch, cnt) for coll in (C.ALL_REDUCE, C.REDUCE_SCATTER, C.ALL_GATHER)
                     for dt in (0, 1) for nc in (8, 32) for ch in (1 << 20, 4 << 20)
                     for cnt in (3 << 20, (8 << 20) + 5))]
        # TREE keys: in-switch AG/RS and the one-hop AllToAll (NVLS region)
        cases += [dict(coll=coll, algo=C.TREE, proto=0, n=world, dtype=dt, op=0, nc=nc, nt=nt, chunk=1 << 20,
                       count=cnt, seed=2000 + i)
                  for i, (coll, dt, nc, nt, cnt) in enumerate(
                      (coll, dt, nc, nt, cnt) for coll in (C.ALL_TO_ALL, C.ALL_GATHER, C.REDUCE_SCATTER)
                      for dt in (1, 3) for nc, nt in ((4, 256), (8, 640)) for cnt in (1 << 20, (2 << 20) + 8))]
    if os.environ.get("LAGOM_BENCH_SIZES"):
        # exactly what bench.py replays (BASELINE configs 2-5) with its seed
        # pick TREE/SIMPLE NC8 NT512 C2M (NVLS / one-hop when LAGOM_NVLS):
        # 25 MiB bf16 buckets, 64 MiB AG/RS, 8 MiB-per-peer (n=8) A2A, and
        # the Llama-70B FSDP layer's AG/RS at n <= 2 (1.71 GB per rank)
        n = world
        fsdp = 8192 * (64 + 16) * 128 + 64 * 128 * 8192 + 3 * 8192 * 28672
        sizes = [(C.ALL_REDUCE, 25 << 19), (C.ALL_GATHER, (8192 // n) * 4096),
                 (C.REDUCE_SCATTER, (8192 // n) * 4096), (C.ALL_TO_ALL, 8192 * 4096 // n)]
        if n <= 2:
            sizes += [(C.ALL_GATHER, fsdp // n), (C.REDUCE_SCATTER, fsdp // n)]
        cases = [dict(coll=coll, algo=algo, proto=0, n=n, dtype=1, op=0, nc=nc, nt=512, chunk=2 << 20,
                      count=cnt, seed=3000 + i)
                 for i, (coll, cnt, algo, nc) in enumerate(
                     (coll, cnt, algo, nc) for coll, cnt in sizes for algo in (C.TREE, C.RING) for nc in (8, 16))]
    # Buffers inside the multicast region are carved once (same offsets on
    # every rank) and reused by every case: the region is a bump allocator.
    # A canary band after the output catches writes past its end.
    band = 4096
    nbytes = max(4 * max(in_elems(c["coll"], world, c["count"]), out_elems(c["coll"], world, c["count"]))
                 for c in cases) + band
    one_hop = int(os.environ.get("LAGOM_ONE_HOP", "0"))
    rs_slot = max([2 * c["count"] * 4 for c in cases if c["coll"] == C.REDUCE_SCATTER] + [0])
    if nvls:
        comm.enable_nvls(max(1 << 30, 2 * nbytes + (64 << 20) + world * rs_slot))
        if one_hop and rs_slot:
            comm.nvls_scratch(rs_slot)  # push-based one-hop ReduceScatter
        xbuf = comm.nvls_tensor(nbytes, torch.uint8)
        ybuf = comm.nvls_tensor(nbytes, torch.uint8)
    else:
        xbuf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        ybuf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for c in cases:
        sends = coll_cases.inputs(c)
        want = oracle_collective(c["coll"], c["algo"], c["dtype"], c["op"], sends)[rank]
        xs = torch.from_numpy(sends[rank].view(np.uint8).copy()).cuda()
        xbuf[:xs.numel()].copy_(xs)
        out_b = want.nbytes
        ybuf[:out_b + band].fill_(0xAB)
        cfg = C.CollConfig(c["algo"], c["proto"], c["nc"], c["nt"], c["chunk"])
        comm.launch(c["coll"], cfg, c["dtype"], c["count"], xbuf.data_ptr(), ybuf.data_ptr(), stream, c["op"])
        torch.cuda.synchronize()
        comm.check()
        got = ybuf[:out_b].cpu().numpy().view(want.dtype)
        canary_ok = bool((ybuf[out_b:out_b + band] == 0xAB).all())
        # The in-switch sum runs only for TREE SUM on whole 16-byte blocks
        # (lagom_nvls_prepare); the one-hop ReduceScatter and every P2P
        # fallback (ragged blocks, MAX/MIN) reduce in the oracle's fixed order,
        # so they are compared bit for bit.
        esz = 2 if c["dtype"] in (C.BF16, C.F16) else 4
        in_switch = (nvls and c["algo"] == C.TREE and c["dtype"] != C.I32 and c["op"] == C.SUM
                     and (c["count"] * esz) % 16 == 0
                     and (c["coll"] == C.ALL_REDUCE or (c["coll"] == C.REDUCE_SCATTER and not one_hop)))
        exact = not in_switch
        if not exact:  # switch-side fp32 accumulation: stated tolerance, not bits
            ok = within_tolerance(got, sends, c)
        else:
            ok = got.tobytes() == want.tobytes()
        ok = ok and canary_ok
        checked += 1
        if not ok:
            fails += 1
            print(f"[rank {rank}] MISMATCH {coll_cases.case_id(c)} canary_ok={canary_ok}", flush=True)
    t = torch.tensor([fails])
    dist.all_reduce(t)
    if rank == 0:
        print(f"mp_coll_check: world={world} nvls={int(nvls)} cases={len(cases)} checked={checked} "
              f"failing(sum over ranks)={int(t)}", flush=True)
    assert checked == len(cases)
    comm.close()
    dist.destroy_process_group()
    sys.exit(min(int(t), 100))


if __name__ == "__main__":
    main()
