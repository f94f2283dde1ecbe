"""Where does a switch collective's time go? Per-channel phase stamps of the
NVLS kernels (LAGOM_PHASE_STAMPS=1, lagom_comm_phase_stamps) for back-to-back
launches, one process per GPU:

  LAGOM_PHASE_STAMPS=1 python -m torch.distributed.run --nproc-per-node 4 \\
      --master-addr 127.0.0.1 tools/nvls_phases.py --out gpurun_out/phases.jsonl

Per (collective, size, NC/NT): the event time per launch over a batch, and for
the last launch of the batch the phases per channel (median / max over
channels and ranks): entry barrier, data loop, system fence, exit barrier;
the kernel span (first channel entry to last channel exit) and the gap
between the previous launch's last exit and this launch's first entry.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_20656_b200 import coll as C  # noqa: E402


def size_of(s):
    s = s.strip().upper()
    mul = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}.get(s[-1], 1)
    return int(float(s[:-1] if s[-1] in "KMG" else s) * mul)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1M,25M,256M")
    ap.add_argument("--colls", default="AR,AG")
    ap.add_argument("--configs", default="8:512,16:512,64:128")
    ap.add_argument("--batch", type=int, default=20)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    assert os.environ.get("LAGOM_PHASE_STAMPS") == "1", "run with LAGOM_PHASE_STAMPS=1"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    MAXC = 64
    comm = C.Communicator.from_process_group(device=local, max_channels=MAXC)
    sizes = [size_of(s) for s in a.sizes.split(",")]
    big = max(sizes) * world + 4096
    comm.enable_nvls(2 * big + (64 << 20))
    xb, yb = comm.nvls_tensor(big, torch.uint8), comm.nvls_tensor(big, torch.uint8)
    stream = torch.cuda.current_stream()
    names = {"AR": C.ALL_REDUCE, "AG": C.ALL_GATHER, "RS": C.REDUCE_SCATTER}
    rows = []
    for size in sizes:
        for cn in a.colls.split(","):
            coll = names[cn]
            count = size // 2 if coll == C.ALL_REDUCE else size // 2 // world
            n_in = count if coll in (C.ALL_REDUCE, C.ALL_GATHER) else count * world
            n_out = count if coll in (C.ALL_REDUCE, C.REDUCE_SCATTER) else count * world
            x = xb[:2 * n_in].view(torch.bfloat16)
            y = yb[:2 * n_out].view(torch.bfloat16)
            x.normal_()
            for spec in a.configs.split(","):
                nc, nt = (int(v) for v in spec.split(":"))
                cfg = C.CollConfig(C.TREE, C.SIMPLE, nc, nt, 2 << 20)

                def fn():
                    comm.launch(coll, cfg, C.BF16, count, x.data_ptr(), y.data_ptr(), stream.cuda_stream)
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(a.batch):
                    fn()
                e1.record(stream)
                e1.synchronize()
                comm.check()
                ev_us = e0.elapsed_time(e1) * 1e3 / a.batch
                st = comm.phase_stamps(MAXC)[:nc]
                # per channel (channels have their own epochs): the slot of the
                # last launch and of the one before (epochs step by 2 per launch)
                last = [max(st[c][k][5] for k in range(2)) for c in range(nc)]
                cur = [st[c][(last[c] >> 1) & 1] for c in range(nc)]
                prev = [st[c][((last[c] - 2) >> 1) & 1] for c in range(nc)]
                ph = {
                    "entry_barrier": [s[1] - s[0] for s in cur],
                    "data": [s[2] - s[1] for s in cur],
                    "fence": [s[3] - s[2] for s in cur],
                    "exit_barrier": [s[4] - s[3] for s in cur],
                    "total": [s[4] - s[0] for s in cur],
                    "entry_skew": [s[0] - min(t[0] for t in cur) for s in cur],
                }
                mine = {k: [statistics.median(v), max(v)] for k, v in ph.items()}
                mine["span"] = max(s[4] for s in cur) - min(s[0] for s in cur)
                mine["gap_prev"] = min(s[0] for s in cur) - max(s[4] for s in prev)
                mine["ev_us"] = ev_us
                allr = [None] * world
                dist.all_gather_object(allr, mine)
                if rank == 0:
                    row = {"coll": cn, "bytes": size, "nc": nc, "nt": nt, "n": world, "batch": a.batch,
                           "ev_us": max(m["ev_us"] for m in allr),
                           "span_us": [m["span"] / 1e3 for m in allr],
                           "gap_prev_us": [m["gap_prev"] / 1e3 for m in allr]}
                    for k in ph:
                        row[k + "_us"] = {"median": statistics.median(m[k][0] for m in allr) / 1e3,
                                          "max": max(m[k][1] for m in allr) / 1e3}
                    rows.append(row)
                    print(json.dumps(row), flush=True)
    if rank == 0 and a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
