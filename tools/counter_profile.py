"""Counter-backed contention profile of one workload (CUPTI PM sampling on
every rank; tools/pm_analyze.py integrates the samples over op windows).

  python -m torch.distributed.run --nproc-per-node N ... tools/counter_profile.py \
      --workload gpt2-1.3b-dp --out profiles/round2_counters_n2_gpt2-1.3b-dp.json

For the workload's own DAG (bench.py's replay) it measures:
  * compute-only replays: y_i and the HBM bytes of every compute op — the
    reference ComputeOp.bytes_per_block D (model.hpp:27-35) is bytes / blocks;
  * per config set (every comm op gets the config; ALGO:NC:NT:C):
      comm-only replays  -> x_j (kernel span), HBM bytes and NVLink tx/rx
                            bytes in each comm window: the footprint V
                            (reference mem_footprint, commperf.cpp:127-135)
                            is HBM bytes / x_j; NVLink bytes / x_j is the wire
                            rate the roofline claims;
      overlapped replays -> X, Y, Z and the SM / tensor-pipe activity inside
                            the comm windows (SM-occupancy loss of the victim).
Rank 0 writes one JSON; tools/predict_vs_measured.py --counters fits the
reference model from it and predicts every config set's overlapped Z.
"""
import argparse
import json
import os
import secrets
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import dist_env  # noqa: E402
from tools.fixed_configs import parse_cfg  # noqa: E402
from tools.pm_analyze import summarize  # noqa: E402

DEFAULT_SETS = ["T:8:512:2M", "T:16:512:2M", "T:4:640:2M", "T:32:256:2M", "T:64:128:2M", "T:16:256:2M",
                "T:64:64:2M", "R:8:512:2M"]
DRAM = ("dram__bytes_read.sum", "dram__bytes_write.sum")


def op_rows(summary, cat):
    return [o for o in summary["ops"] if o["cat"] == cat]


def med(vals):
    return statistics.median(vals) if vals else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt2-1.3b-dp")
    ap.add_argument("--sets", nargs="+", default=DEFAULT_SETS)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--interval-ns", type=int, default=20000)
    ap.add_argument("--nvls", type=int, default=1)
    ap.add_argument("--sm-partition", type=int, default=1)
    ap.add_argument("--one-hop", type=int, default=0,
                    help="lagom_comm_opts_t.one_hop (0: the setting of the committed round-2 counter profiles)")
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
    eng = L.ReplayEngine(json.dumps(dag), f"cp_{token}", rank, world, local, repeats=1, warmup=1, nccl=False,
                         sm_partition=a.sm_partition, max_channels=64, nvls=bool(a.nvls),
                         one_hop=a.one_hop, pm_interval_ns=a.interval_ns)
    if rank != 0:
        eng.serve()
        eng.close()
        dist.barrier()
        return
    eng.set_pm_sampling(True)
    out = {"workload": dag["name"], "n": world, "interval_ns": a.interval_ns, "nvls": bool(eng.nvls_active),
           "sm_partition": a.sm_partition, "compute_ops": [], "sets": {}}

    def runs(fn, k):
        res = []
        for _ in range(k):
            m = json.loads(fn())
            s = summarize(m, dag)
            res.append((m, s))
        return res

    # 1. compute only: y_i and HBM bytes per compute op. One replay here and
    # one after every set below (medians over all of them), so the power-
    # capped part's clock drift affects the isolated and overlapped
    # measurements alike.
    comp = runs(eng.run_compute_only, 1)

    def compute_only_summary():
        out["compute_ops"] = []
        for i, c in enumerate(dag["compute_ops"]):
            rows = [op_rows(s, "compute")[i] for _, s in comp]
            out["compute_ops"].append({"id": c["id"], "y_us": med([m["y"][i] for m, _ in comp]),
                                       "dram_bytes": med([r[DRAM[0]] + r[DRAM[1]] for r in rows]),
                                       "tensor_active": med([r["sm__pipe_tensor_cycles_active_realtime.avg"]
                                                             for r in rows]),
                                       "sm_elapsed": med([r["sm__cycles_elapsed.avg"] for r in rows])})
        out["compute_Y_us"] = med([m["Y"] for m, _ in comp])
        out["compute_Z_us"] = med([m["Z"] for m, _ in comp])
        out["compute_replays"] = len(comp)

    # 2. per config set: comm alone and overlapped
    for spec in a.sets:
        cfg = parse_cfg(spec)
        doc = json.dumps({"configs": [cfg] * len(dag["comm_ops"])})
        alone = runs(lambda: eng.run_comm_only(doc), a.reps)
        over = runs(lambda: eng.run(doc), a.reps)
        comm = []
        for j, c in enumerate(dag["comm_ops"]):
            rows = [op_rows(s, "comm")[j] for _, s in alone]
            x = med([m["x"][j] for m, _ in alone])
            comm.append({"id": c["id"], "x_us": x, "x_ev_us": med([m["x_ev"][j] for m, _ in alone]),
                         "dram_bytes": med([r[DRAM[0]] + r[DRAM[1]] for r in rows]),
                         "nvltx_bytes": med([r["nvltx__bytes.sum"] for r in rows]),
                         "nvlrx_bytes": med([r["nvlrx__bytes.sum"] for r in rows])})
        # victim activity inside the comm windows of the overlapped replays
        ov = []
        for m, s in over:
            cw = op_rows(s, "comm")
            t = sum(o["dur_us"] for o in cw) or 1.0
            ov.append({"Z": m["Z"], "Y": m["Y"], "X": m["X"], "y": m["y"], "x": m["x"],
                       "tensor_active_per_us_in_comm": sum(o["sm__pipe_tensor_cycles_active_realtime.avg"]
                                                           for o in cw) / t,
                       "dram_GBps_in_comm": sum(o[DRAM[0]] + o[DRAM[1]] for o in cw) / t / 1e3})
        entry = {"config": cfg, "comm_ops": comm,
                 "comm_only": {"X_us": med([m["X"] for m, _ in alone]), "Z_us": med([m["Z"] for m, _ in alone])},
                 "overlapped": {k: med([o[k] for o in ov]) for k in ("Z", "Y", "X", "tensor_active_per_us_in_comm",
                                                                    "dram_GBps_in_comm")},
                 "overlapped_y": [med([o["y"][i] for o in ov]) for i in range(len(dag["compute_ops"]))],
                 "overlapped_x": [med([o["x"][j] for o in ov]) for j in range(len(dag["comm_ops"]))]}
        out["sets"][spec] = entry
        comp += runs(eng.run_compute_only, 1)
        xs = sum(c["x_us"] for c in comm)
        print(json.dumps({"set": spec, "X_alone_us": xs,
                          "V_GBps": sum(c["dram_bytes"] for c in comm) / xs / 1e3,
                          "nvltx_GBps": sum(c["nvltx_bytes"] for c in comm) / xs / 1e3,
                          "Z_over_us": entry["overlapped"]["Z"], "Y_over_us": entry["overlapped"]["Y"]}),
              flush=True)
    compute_only_summary()
    print(json.dumps({"mode": "compute", "Y_us": out["compute_Y_us"], "replays": len(comp),
                      "dram_GB": sum(o["dram_bytes"] for o in out["compute_ops"]) / 1e9}), flush=True)
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
