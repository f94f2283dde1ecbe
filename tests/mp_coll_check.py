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


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = C.Communicator.from_process_group(device=local, max_channels=32, max_chunk_bytes=1 << 20,
                                             timeout_ms=5000)
    stream = torch.cuda.current_stream().cuda_stream
    fails = 0
    cases = coll_cases.cases([world], seed=int(os.environ.get("LAGOM_CASE_SEED", "99")), per_combo=2)
    for c in cases:
        c["nc"] = max(1, min(32, c["nc"] * 2))  # real mode: no co-residency cap
        sends = coll_cases.inputs(c)
        want = oracle_collective(c["coll"], c["algo"], c["dtype"], c["op"], sends)[rank]
        x = torch.from_numpy(sends[rank]).cuda()
        y = torch.empty(out_elems(c["coll"], world, c["count"]), dtype=x.dtype, device="cuda")
        y.view(torch.uint8).fill_(0xAB)
        cfg = C.CollConfig(c["algo"], c["proto"], c["nc"], c["nt"], c["chunk"])
        comm.launch(c["coll"], cfg, c["dtype"], c["count"], x.data_ptr(), y.data_ptr(), stream, c["op"])
        torch.cuda.synchronize()
        comm.check()
        if y.cpu().numpy().tobytes() != want.tobytes():
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
