"""Replays one workload DAG with hand-written per-group configs, interleaved
with the NCCL-default arm and the compute-only replay — for exploring the
config space around the tuner's picks (not a bench line).

  python tools/fixed_configs.py --workload gpt2-1.3b-dp \
      --sets "T:1:256:1M|T:32:640:4M" "T:2:256:1M|T:32:640:4M" --steps 5

A set is '<body>|<tail>': <body> is the config of every comm op that compute
can still hide, <tail> the config of the last layer's (exposed) comm ops.
Each config is ALGO:NC:NT:C with ALGO R (ring) or T (tree).
"""
import argparse
import json
import os
import random
import secrets
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import dist_env  # noqa: E402


def parse_cfg(s):
    a, nc, nt, c = s.split(":")
    mul = {"K": 1 << 10, "M": 1 << 20}.get(c[-1].upper(), 1)
    return {"algorithm": {"R": "RING", "T": "TREE"}[a], "protocol": "SIMPLE", "transport": "P2P",
            "num_channels": int(nc), "num_threads": int(nt),
            "chunk_size": int(float(c[:-1] if c[-1].upper() in "KM" else c) * mul)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt2-1.3b-dp")
    ap.add_argument("--sets", nargs="+", required=True)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--sm-reserve", type=int, default=1, help="SM partition: 0 none, 1 auto, 2 all")
    ap.add_argument("--coresident", type=int, default=1)
    ap.add_argument("--nvls", type=int, default=1)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rank, world, local = dist_env()
    import torch
    import torch.distributed as dist

    from paper_2602_20656_b200 import _lagom_py as L
    from paper_2602_20656_b200 import dags
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
        tok = [secrets.token_hex(6) if rank == 0 else None]
        dist.broadcast_object_list(tok, src=0)
        token = tok[0]
    else:
        token = secrets.token_hex(6)
    dag = dags.with_nc_max(dags.BUILDERS[a.workload](world), 64)
    last = dag["compute_ops"][-1]["id"]
    eng = L.ReplayEngine(json.dumps(dag), f"fx_{token}", rank, world, local, repeats=1, warmup=0, nccl=True,
                         sm_partition=int(a.sm_reserve), max_channels=64, nvls=bool(a.nvls),
                         coresident=bool(a.coresident))
    if rank != 0:
        eng.serve()
        eng.close()
        dist.barrier()
        return
    docs = {}
    for s in a.sets:
        body, tail = (s.split("|") + [s])[:2]
        cb, ct = parse_cfg(body), parse_cfg(tail)
        docs[s] = json.dumps({"configs": [ct if c.get("ready_after") == last else cb for c in dag["comm_ops"]]})
    arms = {s: (lambda d=d: eng.run(d)) for s, d in docs.items()}
    arms["nccl"] = eng.run_nccl
    arms["compute"] = eng.run_compute_only
    for _ in range(2):
        for fn in arms.values():
            fn()
    res = {k: [] for k in arms}
    names = list(arms)
    rng = random.Random(20260219)
    for s in range(a.steps):  # a fresh random order per step: no arm keeps a fixed predecessor
        perm = names[:]
        rng.shuffle(perm)
        for k in perm:
            res[k].append(json.loads(arms[k]()))
    eng.stop()
    eng.close()
    if world > 1:
        dist.barrier()
    rows = []
    for k, rs in res.items():
        z = statistics.median(r["Z"] for r in rs) / 1e3
        y = statistics.median(r["Y"] for r in rs) / 1e3
        x = statistics.median(r["X"] for r in rs) / 1e3
        rows.append({"arm": k, "Z_ms": round(z, 3), "Y_ms": round(y, 3), "X_ms": round(x, 3),
                     "Zs": [round(r["Z"] / 1e3, 2) for r in rs]})
        print(json.dumps(rows[-1]), flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(json.dumps({"workload": dag["name"], "sm_reserve": a.sm_reserve, "rows": rows}) + "\n")


if __name__ == "__main__":
    main()
