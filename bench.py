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
def reference_arm(args, world):
    """The reference's CPU path on the host cores: the CPU collective
    restatement (oracle/coll_oracle.c; the reference has no data-path
    collective — a collective there is only comm_time, commperf.cpp:112-125)
    executing the iteration's collectives over `n` rank buffers in host
    memory, OpenMP over all host threads. Bounded sample: one layer's comm
    ops (or at least one op), extrapolated linearly to the whole iteration."""
    import ctypes

    import numpy as np

    from paper_2602_20656_b200 import dags
    sys.path.insert(0, os.path.join(ROOT, "tests"))
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
    layer_ops = [c for c in ops if c.get("ready_after") in (None, dag["compute_ops"][0]["id"])] or ops[:1]
    rng = np.random.default_rng(0)

    def run_op(c):
        code = coll_codes[c["collective"]]
        cnt = c["count"]
        nin = cnt if code in (0, 1) else cnt * n
        nout = cnt if code in (0, 2) else cnt * n
        sends = [rng.integers(0, 1 << 16, size=nin, dtype=np.uint16) for _ in range(n)]
        outs = [np.empty(nout, dtype=np.uint16) for _ in range(n)]
        s = (ctypes.c_void_p * n)(*[a.ctypes.data for a in sends])
        r = (ctypes.c_void_p * n)(*[a.ctypes.data for a in outs])
        t0 = time.perf_counter()
        rc = lib.lagom_oracle_collective(code, 0, n, 1, 0, cnt, s, r)
        dt = time.perf_counter() - t0
        assert rc == 0
        return dt

    scale = len(ops) / len(layer_ops)
    for _ in range(min(1, args.warmup)):
        run_op(layer_ops[0])
    steps = []
    for _ in range(args.steps):
        steps.append(sum(run_op(c) for c in layer_ops) * scale)
    ms = statistics.median(steps) * 1e3
    cores = lib.lagom_oracle_threads()
    sample = (f"{len(layer_ops)} of {len(ops)} comm ops (one layer) per step, x{scale:.0f} to the "
              f"iteration; n={n} rank buffers in host memory; no GEMMs (the reference path has none)")
    line = {"metric": "overlapped iteration ms (Lagom-tuned collectives + compute)", "impl": "reference",
            "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": dag["name"], "comm_ops": len(ops), "parallelism": f"dp{world}"},
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- lagom
def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lagom", choices=["lagom", "reference"])
    ap.add_argument("--workload", default="gpt2-1.3b-dp")
    ap.add_argument("--budget", type=int, default=120)
    ap.add_argument("--start", default="best", choices=["min", "nccl-default", "best"],
                    help="tune() seed (reference CLI --start); best = run both, keep the lower final Z")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--nc-max", type=int, default=64, help="per-op CommBounds.nc_max for the search")
    ap.add_argument("--nvls", type=int, default=1, help="comm buffers in an NVLS region (TREE = in-switch)")
    ap.add_argument("--params", default=os.path.join(ROOT, "profiles", "fitted_params_b200_n4.json"),
                    help="subspace params fitted on B200 by tools/contention_profile.py (reference JSON "
                         "schema); '' = the reference's synthetic defaults")
    ap.add_argument("--sm-reserve", type=int, default=1,
                    help="Lagom replays run each compute op's GEMMs on num_sms - max NC of the collectives "
                         "that can overlap it (cuBLASLt SM count target)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, world, local = dist_env()

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, world)
        return

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
                         reserve_comm_sms=bool(args.sm_reserve), max_channels=max(32, args.nc_max),
                         nvls=bool(args.nvls))
    result, tuned, tune_wall_s, tune_runs = None, None, 0.0, {}
    if rank != 0:
        eng.serve()
    else:
        # ---- 1. Lagom search (C++ tune(), reference Alg. 1/2) with the GPU
        # replay of the FULL iteration as ProfileFn; comm ops of the same role
        # (k-th bucket of every layer) share one config.
        t_tune = time.perf_counter()
        eng.run_compute_only()  # first-touch / clocks settle before the search
        starts = ["min", "nccl-default"] if args.start == "best" else [args.start]
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
        for i in range(6 if len(runs) > 1 else 0):  # alternating order, so neither keeps a predecessor
            for st in (order if i % 2 == 0 else order[::-1]):
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

        def series(fn, k):
            return [json.loads(fn()) for _ in range(k)]

        # ---- 2. measured full-iteration replays. The arms are interleaved
        # step by step (lagom, nccl, seed, e2e, ...) so that clock/power drift
        # of the power-capped part affects every arm alike.
        arms = {"lagom": lambda: eng.run(cfg_doc), "e2e": lambda: eng.run_e2e(cfg_doc),
                "seed": lambda: eng.run(ncc_doc)}
        if not args.no_nccl:
            arms["nccl"] = eng.run_nccl
        for _ in range(args.warmup):
            for fn in arms.values():
                fn()
        runs = {k: [] for k in arms}
        # The arm order rotates every step: on a power-capped part a replay
        # runs faster right after a lighter one, so no arm keeps a fixed
        # predecessor.
        names = list(arms)
        with ClockSampler(local) as clk:
            for s in range(args.steps):
                for k in names[s % len(names):] + names[:s % len(names)]:
                    runs[k].append(json.loads(arms[k]()))
        lagom_runs, e2e_runs, seed_runs = runs["lagom"], runs["e2e"], runs["seed"]
        nccl_runs = runs.get("nccl", [])
        compute_only = series(eng.run_compute_only, max(3, args.steps // 3))
        comm_only = series(lambda: eng.run_comm_only(cfg_doc), max(3, args.steps // 3))
        eng.stop()
        result = dict(lagom=lagom_runs, e2e=e2e_runs, compute=compute_only, comm=comm_only,
                      seed=seed_runs, nccl=nccl_runs, clocks=clk.summary())
    eng.close()  # collective: NCCL teardown on every rank at the same point
    if world > 1:
        dist.barrier()
    if rank != 0:
        return

    # ---- 3. report
    med = lambda rs, k="Z": statistics.median(r[k] for r in rs) if rs else None  # noqa: E731
    ms = med(result["lagom"]) / 1e3
    ms_e2e = med(result["e2e"]) / 1e3
    ms_nccl = med(result["nccl"]) / 1e3 if result["nccl"] else None
    ms_seed = med(result["seed"]) / 1e3
    y_iso = med(result["compute"], "Y") / 1e3
    y_lagom = med(result["lagom"], "Y") / 1e3
    y_nccl = med(result["nccl"], "Y") / 1e3 if result["nccl"] else None

    # dominant kernel: the comm op with the largest summed x over the DAG
    import collections
    x_sum = collections.defaultdict(float)
    for r in result["lagom"]:
        for j, x in enumerate(r["x"]):
            x_sum[j] += x
    j_dom = max(x_sum, key=x_sum.get) if x_sum else 0
    op = dag["comm_ops"][j_dom]
    x_dom_us = statistics.median(r["x"][j_dom] for r in result["lagom"])
    x_dom_iso = statistics.median(r["x"][j_dom] for r in result["comm"])
    S = op["count"] * 2 * (1 if op["collective"] == "ALL_REDUCE" else world)
    fac = {"ALL_REDUCE": 2.0 * (world - 1) / world}.get(op["collective"], (world - 1) / world) if world > 1 else 0
    if world > 1:
        achieved = S * fac / (x_dom_iso * 1e-6) / 1e9
        roof = {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                "frac": achieved / NVLINK_PEER_GBS, "traffic": None,
                "frac_of_nominal_900": achieved / 900.0,
                "note": "busbw of the dominant collective timed alone (comm-only replay, CUDA events); "
                        "peak = measured NVLink peer copy per direction (900 GB/s nominal)"}
    else:
        # n = 1: the collective is a local copy, HBM-bound (read + write)
        achieved = 2 * S / (x_dom_iso * 1e-6) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                "note": f"n=1 collective = local copy; peak = {peaks['_source']} copy bandwidth"}
    # The Lagom picks run the collective on a few SMs by design; the per-SM
    # rate against the per-SM share of the peak shows how hard those SMs work.
    nc_dom = int(tuned["configs"][groups[j_dom]]["num_channels"])
    roof["channels"] = nc_dom
    roof["achieved_per_sm"] = roof["achieved"] / max(1, nc_dom)
    if world == 1:  # HBM is shared by all SMs: compare with one SM's share
        roof["peak_per_sm_share"] = roof["peak"] / n_sms
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as f:
            roof["traffic"] = json.load(f).get(f"{dag['name']}", None)

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

    line = {
        "metric": "overlapped iteration ms (Lagom-tuned collectives + compute)",
        "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights/activations on device)",
        "config": {"workload": dag["name"], "compute_ops": len(dag["compute_ops"]),
                   "comm_ops": len(dag["comm_ops"]), "parallelism": dag.get("parallelism", f"dp{world}"),
                   "l2": "inputs larger than L2 (weights+activations per step >> 126 MB)",
                   "sm_partition": "per compute op: GEMMs on num_sms - max NC of overlappable collectives"
                   if args.sm_reserve else "none",
                   "params": os.path.relpath(args.params, ROOT) if args.params else "reference defaults",
                   "nvls": bool(args.nvls) and world > 1,
                   "tune": {"start": tuned["start"], "others": tuned["other_starts"],
                            "groups": len(tuned["configs"]),
                            "profile_calls": tuned["profile_calls"], "boundary": tuned["boundary_condition"],
                            "search_wall_s": round(tune_wall_s, 3),
                            "search_calls_total": sum(r["profile_calls"] for r in tune_runs.values()),
                            "ms_per_profile_call": round(1e3 * tune_wall_s /
                                                         max(1, sum(r["profile_calls"] for r in tune_runs.values())), 3),
                            "picks": [f"{c['algorithm']}/{c['protocol']}/NC{c['num_channels']}/NT"
                                      f"{c['num_threads']}/C{c['chunk_size'] // 1024}K" for c in tuned["configs"]]}},
        "nccl_default_ms": ms_nccl,
        "speedup_vs_nccl_default": (ms_nccl / ms) if ms_nccl else None,
        "lagom_kernels_nccl_seed_ms": ms_seed,
        "compute": {"isolated_ms": y_iso, "overlapped_ms": y_lagom, "overlapped_nccl_ms": y_nccl,
                    "slowdown": y_lagom / y_iso, "slowdown_nccl": (y_nccl / y_iso) if y_nccl else None,
                    "tflops_isolated": gemm_flops / (y_iso * 1e-3) / 1e12,
                    "frac_of_sustained_bf16": gemm_flops / (y_iso * 1e-3) / 1e12 / peaks["bf16_tflops_sustained"]},
        "roofline": roof,
        "search_speed": search_speed,
        "e2e": {"value": ms_e2e, "unit": "ms", "h2d_bytes_per_step": T_in_bytes, "d2h_bytes_per_step": 4096},
        "gpu_launches": args.steps * len(dag["comm_ops"]),
        "clocks": result["clocks"],
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if args.out:
        # measured Chrome traces (reference trace schema) of one Lagom and one NCCL step
        for arm in ("lagom", "nccl"):
            if result[arm]:
                with open(args.out.replace(".json", f"_trace_{arm}.json"), "w") as f:
                    json.dump(result[arm][len(result[arm]) // 2].get("trace", []), f)
        for arm in ("lagom", "e2e", "seed", "nccl", "compute", "comm"):
            for r in result[arm]:
                r.pop("trace", None)
        with open(args.out, "w") as f:
            json.dump({"line": line, "tune": tuned, "tune_runs": tune_runs, "raw": result}, f)


if __name__ == "__main__":
    main()
