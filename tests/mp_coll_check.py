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
from tests.oracle_ref import collective as oracle_collective, out_elems  # noqa: E402


def nvls_tensor(comm, t):
    out = comm.nvls_tensor(t.numel(), t.dtype)
    out.copy_(t)
    return out


def within_tolerance(got, want, sends, c):
    from tests.test_oracle_cpu import to_f32
    g, w = to_f32(got, c["dtype"]).astype(np.float64), to_f32(want, c["dtype"]).astype(np.float64)
    n = len(sends)
    if c["coll"] == C.ALL_REDUCE:
        mag = np.sum([np.abs(to_f32(s, c["dtype"]).astype(np.float64)) for s in sends], axis=0)
    else:
        r = int(os.environ["RANK"])
        k = c["count"]
        mag = np.sum([np.abs(to_f32(s[r * k:(r + 1) * k], c["dtype"]).astype(np.float64)) for s in sends], axis=0)
    tol = (1e-5 if c["dtype"] == 0 else 2.0 ** -7 * n) * mag + 1e-30
    return bool(np.all(np.abs(g - w) <= 2 * tol))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    use_tma = int(os.environ.get("LAGOM_USE_TMA", "1"))
    comm = C.Communicator.from_process_group(device=local, max_channels=32, max_chunk_bytes=4 << 20,
                                             timeout_ms=5000, use_tma=use_tma)
    stream = torch.cuda.current_stream().cuda_stream
    nvls = bool(os.environ.get("LAGOM_NVLS")) and comm.nvls_supported()
    if nvls:
        comm.enable_nvls(1 << 30)
    fails = 0
    cases = coll_cases.cases([world], seed=int(os.environ.get("LAGOM_CASE_SEED", "99")), per_combo=2)
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
        sends = coll_cases.inputs(c)
        want = oracle_collective(c["coll"], c["algo"], c["dtype"], c["op"], sends)[rank]
        x = torch.from_numpy(sends[rank]).cuda()
        y = torch.empty(out_elems(c["coll"], world, c["count"]), dtype=x.dtype, device="cuda")
        if nvls:  # buffers inside the multicast region (same offsets on every rank)
            x = nvls_tensor(comm, x)
            y = nvls_tensor(comm, y)
        y.view(torch.uint8).fill_(0xAB)
        cfg = C.CollConfig(c["algo"], c["proto"], c["nc"], c["nt"], c["chunk"])
        comm.launch(c["coll"], cfg, c["dtype"], c["count"], x.data_ptr(), y.data_ptr(), stream, c["op"])
        torch.cuda.synchronize()
        comm.check()
        got = y.cpu().numpy()
        exact = not (nvls and c["algo"] == C.TREE and c["dtype"] != C.I32 and c["coll"] != C.ALL_GATHER)
        if not exact:  # switch-side fp32 accumulation: stated tolerance, not bits
            ok = within_tolerance(got, want, sends, c)
        else:
            ok = got.tobytes() == want.tobytes()
        if not ok:
            fails += 1
            print(f"[rank {rank}] MISMATCH {coll_cases.case_id(c)}", flush=True)
    t = torch.tensor([fails])
    dist.all_reduce(t)
    if rank == 0:
        print(f"mp_coll_check: world={world} cases={len(cases)} failing(sum over ranks)={int(t)}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(min(int(t), 100))


if __name__ == "__main__":
    main()
