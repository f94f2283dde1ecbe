#!/usr/bin/env python3
"""lagom-b200 benchmark — overlapped iteration time with Lagom-tuned sm_100a
collectives vs NCCL-default, on BASELINE.json's config 2 (GPT-2 1.3B, DP)
by default.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      bench.py --gpus N ...            (N > 1: one process per GPU)
  python bench.py --impl reference    (the reference's CPU path, rank 0)

One step = one replay of the whole iteration DAG (every layer's backward
GEMMs on the compute stream, every gradient-bucket AllReduce on the comm
stream, gated on its layer) through the native C++ replay engine. Timing is
device-side (CUDA events on the engine's streams), max over ranks. The
Lagom configs are searched first by the C++ tuner (tune(start=min), the
reference's Alg. 1/2, bit-identical picks) with the GPU replay as its
ProfileFn replaying the full iteration; comm ops of one role (the k-th
bucket of every layer) share a config.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import secrets
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["_source"] = "measured"
        return d
    d = dict(PEAKS_FALLBACK)
    d["_source"] = "fallback"
    return d


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        # nvidia-smi numbers physical GPUs: map the CUDA ordinal through
        # CUDA_VISIBLE_DEVICES when it is set
        vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
        if vis and device < len(vis) and vis[device].strip().isdigit():
            device = int(vis[device])
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(self.rows)}


def tune_speed(binary: str):
    """Runs tests/cpp/tune_speed.cpp (product: build/tune_speed; reference
    build: oracle/_ref/tune_speed_ref) pinned to one core; None if absent."""
    if not os.path.exists(binary):
        return None
    cmd = [binary, "7"]
    if subprocess.run(["which", "taskset"], capture_output=True).returncode == 0:
        cmd = ["taskset", "-c", "0"] + cmd
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, check=True).stdout
        d = json.loads(out)
    except Exception as e:  # reported, never fatal
        return {"failed": str(e)}
    return {"unit": "us per tune(start=min), simulator ProfileFn, budget 500, best of 7",
            "cores": 1, "workloads": {k: {"us": v["us"], "calls": v["calls"], "us_per_call": v["us_per_call"]}
                                      for k, v in d.items()}}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


# ----------------------------------------------------------------- reference
def workload_config(dag: dict) -> dict:
    """The workload identity shared by both arms' `config` (no engine knobs)."""
    return {"workload": dag["name"], "compute_ops": len(dag["compute_ops"]), "comm_ops": len(dag["comm_ops"]),
            "parallelism": dag.get("parallelism", "")}


METRIC = "overlapped iteration ms (collectives + compute, one training-step DAG)"


def reference_arm(args, world):
    """The reference's CPU path on the host cores. The reference has no
    data-path collective (a collective there is only comm_time,
    commperf.cpp:112-125) and no compute path, so its CPU counterpart of the
    iteration is the CPU collective restatement (oracle/coll_oracle.c,
    OpenMP over all host threads) executing EVERY comm op of the iteration
    in order over n rank buffers in host memory. Buffers are allocated and
    first-touched before the timed region (ops of the same shape share
    them); each timed step runs all ops back to back."""
    import collections
    import ctypes

    import numpy as np

    from paper_2602_20656_b200 import dags
    lib_path = os.path.join(ROOT, "oracle", "_ref", "libcoll_oracle.so")
    if not os.path.exists(lib_path):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "coll"], check=True, capture_output=True)
    lib = ctypes.CDLL(lib_path)
    lib.lagom_oracle_collective.restype = ctypes.c_int
    lib.lagom_oracle_collective.argtypes = [ctypes.c_int] * 5 + [ctypes.c_longlong, ctypes.c_void_p,
                                                                 ctypes.c_void_p]
    lib.lagom_oracle_threads.restype = ctypes.c_int
    n = max(1, world)
    dag = dags.BUILDERS[args.workload](n)
    ops = dag["comm_ops"]
    coll_codes = {"ALL_REDUCE": 0, "ALL_GATHER": 1, "REDUCE_SCATTER": 2, "ALL_TO_ALL": 3}
    rng = np.random.default_rng(0)
    # Prefaulted host buffers: per (collective, count) a pool of buffer sets
    # that ops of that shape rotate through, sized so consecutive ops never
    # find their data in the last-level cache (>= 1.5 GiB per pool, or one
    # set per op).
    bufs, uses = {}, collections.Counter((c["collective"], c["count"]) for c in ops)
    for c in ops:
        key = (c["collective"], c["count"])
        if key in bufs:
            continue
        code = coll_codes[c["collective"]]
        nin = c["count"] * (n if code in (2, 3) else 1)
        nout = c["count"] * (n if code in (1, 3) else 1)
        set_bytes = 2 * n * (nin + nout)
        pool = []
        for _ in range(max(1, min(uses[key], -(-(3 << 29) // set_bytes)))):
            sends = [rng.integers(0x3000, 0x3f80, size=nin, dtype=np.uint16) for _ in range(n)]  # finite bf16
            outs = [np.ones(nout, dtype=np.uint16) for _ in range(n)]  # written: pages faulted in
            pool.append((sends, outs, (ctypes.c_void_p * n)(*[a.ctypes.data for a in sends]),
                         (ctypes.c_void_p * n)(*[a.ctypes.data for a in outs])))
        bufs[key] = (code, pool)
    turn = collections.Counter()

    def step():
        t0 = time.perf_counter()
        for c in ops:
            key = (c["collective"], c["count"])
            code, pool = bufs[key]
            _, _, s, r = pool[turn[key] % len(pool)]
            turn[key] += 1
            # ring order (algorithm 0) and bf16 (dtype 1), sum
            if lib.lagom_oracle_collective(code, 0, n, 1, 0, c["count"], s, r) != 0:
                raise RuntimeError("oracle collective failed")
        return time.perf_counter() - t0

    for _ in range(max(1, args.warmup)):
        step()
    steps = [step() for _ in range(args.steps)]
    ms = statistics.median(steps) * 1e3
    cores = lib.lagom_oracle_threads()
    sample = (f"all {len(ops)} comm ops of one iteration per step (the whole workload), bf16 sum, ring order, "
              f"n={n} rank buffers in host memory (prefaulted, rotated so no op finds its data in cache), OpenMP "
              f"over {cores} threads; the iteration's GEMMs are not executed (the reference has no compute path)")
    line = {"metric": METRIC, "impl": "reference",
            "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": max(1, args.warmup),
            "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic", "config": workload_config(dag),
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- lagom
def nccl_log_env(tag: str) -> str | None:
    """NCCL_DEBUG=INFO with INIT/TUNING to a per-process file, unless the
    user set NCCL_DEBUG: the channels and algorithms NCCL chose for the
    baseline go into the bench line."""
    if os.environ.get("NCCL_DEBUG", "").upper() in ("INFO", "TRACE") and not os.environ.get("NCCL_DEBUG_FILE"):
        return None  # the user asked for NCCL's log on stderr
    path = f"/tmp/lagom_nccl_{tag}_%p.log"
    os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,TUNING,NVLS", NCCL_DEBUG_FILE=path)
    return path.replace("%p", str(os.getpid()))


def nccl_log_summary(path: str | None) -> dict:
    import re
    if not path:
        return {"log": None}
    if not os.path.exists(path):  # NCCL expands %p itself; take this process's file if the pid differs
        import glob
        cands = sorted(glob.glob(path.rsplit("_", 1)[0] + "_*.log"))
        if not cands:
            return {"log": None}
        path = cands[0]
    text = open(path, errors="replace").read()
    out = {"log": path}
    m = re.search(r"(\d+) coll channels, (\d+) collnet channels, (\d+) nvls channels, (\d+) p2p channels", text)
    if m:
        out.update(coll_channels=int(m.group(1)), nvls_channels=int(m.group(3)), p2p_channels=int(m.group(4)))
    algo = [ln.split("NCCL INFO", 1)[-1].strip() for ln in text.splitlines()
            if re.search(r"(AllReduce|AllGather|ReduceScatter|SendRecv|Broadcast).*(Algo|algorithm|proto)", ln)]
    out["tuning"] = sorted(set(algo))[:12]
    out["version"] = (re.search(r"NCCL version ([\w.+]+)", text) or [None, None])[1]
    return out


def wire_bytes(op: dict, n: int, cfg: dict, nvls: bool, one_hop_a2a: bool, one_hop_agrs: bool = False
               ) -> tuple[float, str]:
    """Bytes that cross NVLink per rank, per direction, for one launch of the
    config's schedule, and the schedule's name. n = 1: HBM
    bytes (read + write of the local copy)."""
    e = 2 if op["dtype"] in (1, 2) else 4
    coll = op["collective"]
    S = op["count"] * e * (1 if coll == "ALL_REDUCE" else n)  # nccl-tests algorithmic bytes
    if n == 1:
        return 2.0 * op["count"] * e, "local copy (HBM read + write)"
    tree = cfg["algorithm"] == "TREE"
    if tree and nvls and one_hop_agrs and coll in ("ALL_GATHER", "REDUCE_SCATTER"):
        return S * (n - 1) / n, "one hop (peer stores / pushes): (n-1)/n S egress"
    if tree and nvls and coll == "ALL_REDUCE":
        # ld_reduce: every GPU serves each rank's S/n share (S out); multimem.st:
        # the switch delivers every share to every GPU (S in), plus the own share
        # each way: S (1 + 1/n) per rank on either direction
        return S * (n + 1) / n, "NVLS AllReduce (in-switch): S (1 + 1/n) per rank per direction"
    if tree and nvls and coll in ("ALL_GATHER", "REDUCE_SCATTER"):
        return float(S), "NVLS (in-switch): S per rank on the busier direction"
    if tree and coll == "ALL_TO_ALL" and one_hop_a2a:
        return S * (n - 1) / n, "one-hop AllToAll: (n-1)/n S egress"
    f = 2.0 * (n - 1) / n if coll == "ALL_REDUCE" else (n - 1) / n
    return S * f, "ring: busbw bytes"


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lagom", choices=["lagom", "reference"])
    ap.add_argument("--workload", default="gpt2-1.3b-dp")
    ap.add_argument("--budget", type=int, default=120)
    ap.add_argument("--start", default="best", choices=["min", "nccl-default", "coresident", "best"],
                    help="tune() seed: the reference CLI's min / nccl-default, or coresident (NC 64, NT 128: "
                         "the co-resident kernel regime); best = run all three, keep the lowest final Z "
                         "(head to head)")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--nc-max", type=int, default=64, help="per-op CommBounds.nc_max for the search")
    ap.add_argument("--nvls", type=int, default=1, help="comm buffers in an NVLS region (TREE = in-switch)")
    ap.add_argument("--params", default=os.path.join(ROOT, "profiles", "fitted_params_b200_n4.json"),
                    help="subspace params fitted on B200 by tools/contention_profile.py (reference JSON "
                         "schema); '' = the reference's synthetic defaults")
    ap.add_argument("--sm-partition", type=int, default=1, choices=[0, 1, 2],
                    help="GEMMs a collective can overlap run on num_sms - NC SMs: 0 never, 1 only for "
                         "collectives whose CTAs cannot share an SM with a GEMM CTA (default), 2 always")
    ap.add_argument("--coresident", type=int, default=1,
                    help="NVLS / one-hop / single-rank kernels sized to co-reside with GEMM CTAs")
    ap.add_argument("--one-hop", type=int, default=2,
                    help="lagom_comm_opts_t.one_hop: TREE AG/RS through the switch (0), one hop (1), one hop at "
                         "n = 2 (2, default: the switch echoes the own block, so at n = 2 it moves twice the bytes)")
    ap.add_argument("--a2a-tma", type=int, default=1,
                    help="lagom_comm_opts_t.a2a_tma (one-hop AllToAll / AllGather / ReduceScatter via TMA)")
    ap.add_argument("--ablations", type=int, default=1,
                    help="also time: our kernels at the seed with the SM partition forced on, and (N > 1) NCCL "
                         "with the GEMMs on num_sms - NCCL's channels")
    ap.add_argument("--order-seed", type=int, default=20260219, help="seed of the per-step arm permutation")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, world, local = dist_env()

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, world)
        return

    import random

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
    nccl_log = nccl_log_env(token) if not args.no_nccl else None
    peaks = load_peaks()
    n_sms = torch.cuda.get_device_properties(local).multi_processor_count
    gpu_json = json.dumps({"num_sms": n_sms, "peak_mem_bw": peaks["hbm_gbs"] * 1e3,
                           "link_bw": NVLINK_PEER_GBS * 1e3, "comm_bw_cap_fraction": 0.6})

    dag = dags.with_nc_max(dags.BUILDERS[args.workload](world), args.nc_max)
    # Comm roles recur in every layer; the last layer's comms are exposed (no
    # compute left to hide them), so they get groups of their own.
    last_compute = dag["compute_ops"][-1]["id"]
    nroles = 1 + max(int(c.get("role", 0)) for c in dag["comm_ops"])
    groups = [int(c.get("role", 0)) + (nroles if c.get("ready_after") == last_compute else 0)
              for c in dag["comm_ops"]]
    present = sorted(set(groups))
    groups = [present.index(g) for g in groups]

    # One engine for the whole run: rank 0 drives (search + measured replays),
    # the other ranks serve replay commands until rank 0 stops them.
    T_in_bytes = 8192 * 2048 * 2
    eng = L.ReplayEngine(json.dumps(dag), f"lagom_{token}", rank, world, local, repeats=1, warmup=0,
                         nccl=not args.no_nccl, e2e_in_bytes=T_in_bytes, e2e_out_bytes=4096,
                         sm_partition=args.sm_partition, max_channels=max(32, args.nc_max),
                         nvls=bool(args.nvls), coresident=bool(args.coresident), one_hop=args.one_hop,
                         a2a_tma=bool(args.a2a_tma))
    nvls_state = {"requested": bool(args.nvls) and world > 1, "active": bool(eng.nvls_active),
                  "peer_mappings": bool(eng.nvls_peers_active)}
    result, tuned, tune_wall_s, tune_runs = None, None, 0.0, {}
    if rank != 0:
        eng.serve()
    else:
        # ---- 1. Lagom search (C++ tune(), reference Alg. 1/2) with the GPU
        # replay of the FULL iteration as ProfileFn; comm ops of the same role
        # (k-th bucket of every layer) share one config.
        t_tune = time.perf_counter()
        eng.run_compute_only()  # first-touch / clocks settle before the search
        starts = ["min", "nccl-default", "coresident"] if args.start == "best" else [args.start]
        eng.set_partition(args.sm_partition, 0)
        eng.set_measurement(5, 2)  # each profile call: median of 5 replays after 2 warmups
        params_doc = open(args.params).read() if args.params and os.path.exists(args.params) else ""
        if params_doc:
            pj = json.loads(params_doc)
            params_doc = json.dumps(pj.get("params", pj))  # accept a profile file or a bare table
        runs = {st: json.loads(eng.tune(gpu_json, st, args.budget, params_doc, groups)) for st in starts}
        tune_wall_s = time.perf_counter() - t_tune
        eng.set_measurement(1, 0)
        # The replays are noisy under the 1 kW power cap, so the starts' final
        # assignments are compared head to head (interleaved) before choosing.
        docs = {st: json.dumps({"configs": [r["configs"][g] for g in groups]}) for st, r in runs.items()}
        zsel = {st: [] for st in runs}
        order = list(runs)
        sel_rng = random.Random(args.order_seed + 1)
        # 12 rounds: with 6, identical-config spreads of a few % let the pick flip between sessions
        for i in range(12 if len(runs) > 1 else 0):  # random order per round: no start keeps a predecessor
            perm = order[:]
            sel_rng.shuffle(perm)
            for st in perm:
                zsel[st].append(json.loads(eng.run(docs[st]))["Z"])
        best_start = min(runs, key=lambda st: statistics.median(zsel[st]) if zsel[st] else 0.0)
        tune_runs = runs
        tuned = runs[best_start]
        tuned["start"] = best_start
        tuned["other_starts"] = {st: {"Z_tune": r["final"]["Z"], "Z_select": zsel[st], "calls": r["profile_calls"],
                                      "boundary": r["boundary_condition"]}
                                 for st, r in runs.items()}
        full_cfgs = [tuned["configs"][g] for g in groups]
        seed_full = [dict(tuned["initial"][g], num_channels=8, num_threads=512, chunk_size=2 << 20)
                     for g in groups]
        cfg_doc = json.dumps({"configs": full_cfgs})
        ncc_doc = json.dumps({"configs": seed_full})

        # ---- 2. measured full-iteration replays. Every step runs every arm
        # once, in a fresh seeded random order (a power-capped B200 runs a
        # replay faster right after a lighter one, so no arm may keep a fixed
        # predecessor); compute-only is one of the arms.
        nccl_reserve = 0

        def with_partition(part, nccl_res, fn):
            def run():
                eng.set_partition(part, nccl_res)
                return fn()
            return run

        arms = {"lagom": with_partition(args.sm_partition, 0, lambda: eng.run(cfg_doc)),
                "e2e": with_partition(args.sm_partition, 0, lambda: eng.run_e2e(cfg_doc)),
                "seed": with_partition(args.sm_partition, 0, lambda: eng.run(ncc_doc)),
                "compute": eng.run_compute_only}
        if args.ablations:
            arms["seed_partition_all"] = with_partition(2, 0, lambda: eng.run(ncc_doc))
        if not args.no_nccl:
            arms["nccl"] = with_partition(args.sm_partition, 0, eng.run_nccl)
            eng.run_nccl()  # NCCL initialises its channels on the first collective
            nccl_info = nccl_log_summary(nccl_log)
            if args.ablations and world > 1:
                nccl_reserve = int(nccl_info.get("nvls_channels") or nccl_info.get("coll_channels") or 0) \
                    if nvls_state["active"] else int(nccl_info.get("coll_channels") or 0)
                if nccl_reserve > 0:
                    arms["nccl_partition"] = with_partition(args.sm_partition, nccl_reserve, eng.run_nccl)
        else:
            nccl_info = {}
        for _ in range(args.warmup):
            for fn in arms.values():
                fn()
        runs = {k: [] for k in arms}
        names = list(arms)
        rng = random.Random(args.order_seed)
        orders = []
        with ClockSampler(local) as clk:
            for s in range(args.steps):
                perm = names[:]
                rng.shuffle(perm)
                orders.append(perm)
                for k in perm:
                    runs[k].append(json.loads(arms[k]()))
        eng.set_partition(args.sm_partition, 0)
        comm_only = [json.loads(eng.run_comm_only(cfg_doc)) for _ in range(max(3, args.steps // 3))]
        eng.stop()
        result = dict(runs, comm=comm_only, clocks=clk.summary(), orders=orders, nccl_reserve=nccl_reserve,
                      nccl_info=nccl_info)
    eng.close()  # collective: NCCL teardown on every rank at the same point
    if world > 1:
        dist.barrier()
    if rank != 0:
        return

    # ---- 3. report
    med = lambda rs, k="Z": statistics.median(r[k] for r in rs) if rs else None  # noqa: E731
    ms = {k: med(result[k]) / 1e3 for k in arms}
    y = {k: med(result[k], "Y") / 1e3 for k in arms}
    ms_nccl = ms.get("nccl")
    y_iso = y["compute"]

    # dominant kernel: the config group (comm ops sharing one tuned config)
    # with the largest summed x over the DAG; its first op, timed alone at the
    # tuned config (comm-only replay), is the roofline's launch
    import collections
    x_sum = collections.defaultdict(float)
    for r in result["lagom"]:
        for j, x in enumerate(r["x"]):
            x_sum[groups[j]] += x
    g_dom = max(x_sum, key=x_sum.get) if x_sum else 0
    j_dom = groups.index(g_dom)
    op = dag["comm_ops"][j_dom]
    cfg_dom = full_cfgs[j_dom]
    t_ev = statistics.median(r["x_ev"][j_dom] for r in result["comm"])    # CUDA events, us
    t_span = statistics.median(r["x"][j_dom] for r in result["comm"])     # kernel's own span, us
    one_hop_agrs = nvls_state["peer_mappings"] and (
        args.one_hop == 1 or (args.one_hop == 2 and world == 2 and cfg_dom["num_channels"] >= 16))
    wb, sched = wire_bytes(op, world, cfg_dom, nvls_state["active"], nvls_state["peer_mappings"], one_hop_agrs)
    e = 2 if op["dtype"] in (1, 2) else 4
    S = op["count"] * e * (1 if op["collective"] == "ALL_REDUCE" else world)
    if world > 1:
        achieved = wb / (t_ev * 1e-6) / 1e9
        busf = 2.0 * (world - 1) / world if op["collective"] == "ALL_REDUCE" else (world - 1) / world
        roof = {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                "frac": achieved / NVLINK_PEER_GBS, "traffic": None,
                "busbw": S * busf / (t_ev * 1e-6) / 1e9,
                "note": f"{op['collective']} {S / 2**20:.1f} MiB at its tuned config, timed alone with CUDA "
                        f"events (comm-only replay); achieved = wire bytes per rank on the busier direction "
                        f"({sched}) / time; peak = measured NVLink peer copy per direction (900 nominal)"}
    else:
        achieved = wb / (t_ev * 1e-6) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                "note": f"n=1: the collective is a local copy of {S / 2**20:.1f} MiB ({sched}), timed alone with "
                        f"CUDA events at the tuned config; peak = {peaks['_source']} copy bandwidth"}
    nc_dom = int(cfg_dom["num_channels"])
    roof.update(config=f"{cfg_dom['algorithm']}/{cfg_dom['protocol']}/NC{nc_dom}/NT{cfg_dom['num_threads']}",
                kernel_span_us=t_span, event_us=t_ev, achieved_per_cta=roof["achieved"] / max(1, nc_dom))
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as f:
            tr = json.load(f).get(f"{dag['name']}")
        for t in (tr if isinstance(tr, list) else [tr]):  # one ncu capture per kernel config
            if isinstance(t, dict) and t.get("config") == roof["config"]:
                roof["traffic"] = t.get("bytes")

    gemm_flops = dags.flops(dag)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            out = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference",
                                  "--steps", "3", "--warmup", "1", "--workload", args.workload],
                                 capture_output=True, text=True, timeout=600)
            cpu = json.loads(out.stdout.strip().splitlines()[-1])["cpu_baseline"]
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "ms", "cores": None, "kind": "port", "sample": f"failed: {e}"}
        # Search speed (the north star's N = 1 figure of merit): tune(start=min)
        # with the simulator ProfileFn on the reference's sample workloads,
        # one pinned host core, best of 7 — the reference build's tuner
        # (oracle/_ref, the CPU baseline) next to the product's.
        cpu["reference_tuner"] = tune_speed(os.path.join(ROOT, "oracle", "_ref", "tune_speed_ref"))
    search_speed = tune_speed(os.path.join(ROOT, "build", "tune_speed")) if world == 1 else None

    same_cfg = full_cfgs == seed_full
    our_arms = [k for k in ("lagom", "e2e", "seed", "seed_partition_all") if k in arms]
    launches_per_replay = sum(1 for c in dag["comm_ops"] if c["count"] > 0)
    line = {
        "metric": METRIC,
        "value": ms["lagom"], "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms["lagom"], "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights/activations on device)",
        "config": workload_config(dag),
        "speedup_vs_nccl_default": (ms_nccl / ms["lagom"]) if ms_nccl else None,
        "arms_ms": ms,
        "ablation": {
            "nccl_default": ms_nccl,
            "nccl_with_sm_partition": ms.get("nccl_partition"),
            "nccl_reserved_sms": result["nccl_reserve"] or None,
            {0: "ours_at_seed_no_partition", 1: "ours_at_seed_auto_partition", 2: "ours_at_seed"}[args.sm_partition]:
                ms["seed"],
            "ours_at_seed_partition_all": ms.get("seed_partition_all"),
            "ours_tuned": ms["lagom"],
            "tuned_equals_seed": same_cfg,
            "noise_floor_ms": abs(ms["lagom"] - ms["seed"]) if same_cfg else None,
            "order": "seeded random permutation of all arms per step (compute-only included)",
        },
        "compute": {"isolated_ms": y_iso, "overlapped_ms": y["lagom"], "overlapped_nccl_ms": y.get("nccl"),
                    "slowdown": y["lagom"] / y_iso, "slowdown_nccl": (y["nccl"] / y_iso) if "nccl" in y else None,
                    "tflops_isolated": gemm_flops / (y_iso * 1e-3) / 1e12,
                    "frac_of_sustained_bf16": gemm_flops / (y_iso * 1e-3) / 1e12 / peaks["bf16_tflops_sustained"]},
        "roofline": roof,
        "lagom": {"sm_partition": ["none", "auto (non-co-resident kernels only)", "all"][args.sm_partition],
                  "coresident_kernels": bool(args.coresident), "one_hop": args.one_hop,
                  "params": os.path.relpath(args.params, ROOT) if args.params else "reference defaults",
                  "nvls": nvls_state, "nccl": result["nccl_info"],
                  "l2": "inputs larger than L2 (weights+activations per step >> 126 MB)",
                  "tune": {"start": tuned["start"], "others": tuned["other_starts"], "groups": len(tuned["configs"]),
                           "profile_calls": tuned["profile_calls"], "boundary": tuned["boundary_condition"],
                           "search_wall_s": round(tune_wall_s, 3),
                           "search_calls_total": sum(r["profile_calls"] for r in tune_runs.values()),
                           "ms_per_profile_call": round(1e3 * tune_wall_s /
                                                        max(1, sum(r["profile_calls"] for r in tune_runs.values())), 3),
                           "picks": [f"{c['algorithm']}/{c['protocol']}/NC{c['num_channels']}/NT"
                                     f"{c['num_threads']}/C{c['chunk_size'] // 1024}K" for c in tuned["configs"]]}},
        "search_speed": search_speed,
        "e2e": {"value": ms["e2e"], "unit": "ms", "h2d_bytes_per_step": T_in_bytes, "d2h_bytes_per_step": 4096},
        "gpu_launches": args.steps * len(our_arms) * launches_per_replay,
        "gpu_launches_note": f"our collective kernels in the timed region: {launches_per_replay} per replay x "
                             f"{len(our_arms)} arms ({', '.join(our_arms)}) x {args.steps} steps",
        "clocks": result["clocks"],
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if args.out:
        # measured Chrome traces (reference trace schema) of one Lagom and one NCCL step
        for arm in ("lagom", "nccl"):
            if result.get(arm):
                with open(args.out.replace(".json", f"_trace_{arm}.json"), "w") as f:
                    json.dump(result[arm][len(result[arm]) // 2].get("trace", []), f)
        for arm in list(arms) + ["comm"]:
            for r in result[arm]:
                r.pop("trace", None)
        with open(args.out, "w") as f:
            json.dump({"line": line, "tune": tuned, "tune_runs": tune_runs, "raw": result}, f)


if __name__ == "__main__":
    main()
