"""CUPTI PM-sampling capture of full-iteration replays (the contention
profiler's counter source): every rank samples its own GPU — DRAM read/write
bytes, NVLink tx/rx bytes, SM active cycles, tensor-pipe active cycles, L2
bytes — every --interval-ns of GPU time while the replay's GEMMs and
collectives run concurrently (no kernel replay, no serialisation).

  python tools/pm_probe.py --workload gpt2-1.3b-dp --config T:8:512:2M \
      --out gpurun_out/pm_gpt2_n1.json
  python -m torch.distributed.run --nproc-per-node 2 ... tools/pm_probe.py ...

Writes, per replay mode (compute-only, comm-only, Lagom-overlapped, NCCL),
rank 0's samples, the replay timeline (reference trace schema) and the
%globaltimer origin of the timeline, plus per-op window sums
(tools/pm_analyze.py) printed as one JSON line per mode.
"""
import argparse
import json
import os
import secrets
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import dist_env  # noqa: E402
from tools.fixed_configs import parse_cfg  # noqa: E402
from tools.pm_analyze import summarize  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt2-1.3b-dp")
    ap.add_argument("--config", nargs="+", default=["T:8:512:2M"],
                    help="ALGO:NC:NT:C configs, one measured set each (every comm op gets it)")
    ap.add_argument("--interval-ns", type=int, default=20000)
    ap.add_argument("--layers", type=int, default=0, help="truncate the DAG (0 = full)")
    ap.add_argument("--sm-partition", type=int, default=1)
    ap.add_argument("--nvls", type=int, default=1)
    ap.add_argument("--nccl", type=int, default=1)
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
    dag = dags.BUILDERS[a.workload](world)
    if a.layers:
        keep = {c["id"] for c in dag["compute_ops"][:a.layers]}
        dag["compute_ops"] = dag["compute_ops"][:a.layers]
        dag["comm_ops"] = [c for c in dag["comm_ops"] if c.get("ready_after") in keep or
                           (c.get("ready_after") is None and c is dag["comm_ops"][0])]
    eng = L.ReplayEngine(json.dumps(dag), f"pm_{token}", rank, world, local, repeats=1, warmup=1,
                         nccl=bool(a.nccl), sm_partition=a.sm_partition, max_channels=64, nvls=bool(a.nvls),
                         pm_interval_ns=a.interval_ns)
    if rank != 0:
        eng.serve()
        eng.close()
        dist.barrier()
        return
    eng.set_pm_sampling(True)
    out = {"workload": dag["name"], "n": world, "interval_ns": a.interval_ns, "modes": {}}
    runs = [("compute", eng.run_compute_only)]
    for c in a.config:
        doc = json.dumps({"configs": [parse_cfg(c)] * len(dag["comm_ops"])})
        runs += [(f"comm:{c}", lambda d=doc: eng.run_comm_only(d)), (f"lagom:{c}", lambda d=doc: eng.run(d))]
    if a.nccl:
        runs.append(("nccl", eng.run_nccl))
    for name, fn in runs:
        m = json.loads(fn())
        out["modes"][name] = {k: m[k] for k in ("pm", "trace", "x", "x_ev", "y", "X", "Y", "Z")}
        s = summarize(m, dag)
        print(json.dumps({"mode": name, **s["totals"], "Z_us": m["Z"]}), flush=True)
        out["modes"][name]["summary"] = s
    eng.set_pm_sampling(False)
    eng.stop()
    eng.close()
    if world > 1:
        dist.barrier()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f)


if __name__ == "__main__":
    main()
