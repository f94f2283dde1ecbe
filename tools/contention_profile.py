"""Contention profiler: measures the sm_100a collectives and a victim GEMM
stream on B200 and fits the reference cost model's coefficients
(reference commperf.cpp:108-135 comm_time / mem_footprint, contention.cpp:22-44
wave_count / wave_time) — writing them in the reference's own params JSON
schema (docs/formats.md "Subspace parameters") plus a fitted GpuSpec.

  python -m torch.distributed.run --nproc-per-node 2 ... tools/contention_profile.py \
      --out profiles/fitted_params_n2.json

Measurements (rank 0 drives the native replay engine; other ranks serve):
  1. comm alone: x(NC, NT, C, m) for RING/SIMPLE, RING/LL, RING/LL128 and
     TREE/SIMPLE AllReduce (kernel active span, %globaltimer);
  2. victim alone: y of one GEMM op (cuBLASLt bf16);
  3. overlapped: y(NC, C) with the comm running (SM partition on): the
     compute-side slowdown the footprint V and the lost SMs cause.
Fits (least squares):
  comm_time   x = alpha + zeta*NC + ceil(m/(NC*C))*c_over + m/min(NC*b_chan*eta(NT), link)
  thread eff. eta(NT) = eta0 + (1-eta0)*NT/640   (eta0 by 1-D search)
  footprint   V(NC, C) = kappa*NC*C/(C+C_knee)*b_chan  (from the overlapped slowdown)
Then reports per-point predicted vs measured x.
"""
import argparse
import itertools
import json
import math
import os
import secrets
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

KIB = 1024
MIB = 1 << 20


COLLS = ("ALL_REDUCE", "ALL_GATHER", "REDUCE_SCATTER", "ALL_TO_ALL")


def dag_for(sizes_mib, gemm, nranks):
    """Comm ops: every collective at every size (message_bytes = s MiB: the
    AR buffer, the AG output, the RS input, the A2A send), AllReduce first."""
    comm = []
    for coll in COLLS:
        for s in sizes_mib:
            count = s * MIB // 2 // (1 if coll == "ALL_REDUCE" else nranks)
            comm.append({"id": f"{coll.lower()}{s}", "collective": coll, "dtype": 1, "count": count,
                         "ready_after": None, "role": len(comm)})
    return {"name": "contention-probe", "compute_ops": [{"id": "victim", "gemms": [gemm] * 8}],
            "comm_ops": comm}


def fit_factor(co, link, pts):
    """The reference's collective_factors (default_params.json:164-169) scale
    message bytes inside comm_time; fit one factor per collective against the
    subspace's AllReduce-fitted coefficients (median relative error)."""
    best = None
    for f in np.geomspace(0.2, 5.0, 241):
        rel = [abs(predict(co, link, nc, nt, c, m * f) - x) / x for nc, nt, c, m, x in pts]
        err = float(np.median(rel))
        if best is None or err < best[0]:
            best = (err, float(f), float(np.percentile(rel, 90)))
    return best


def cfg(algo, proto, nc, nt, c):
    return {"algorithm": algo, "protocol": proto, "transport": "P2P", "num_channels": nc,
            "num_threads": nt, "chunk_size": c}


def fit_comm(points, link_guess):
    """points: list of (nc, nt, c, m_eff, x_us). Returns coeffs dict + link."""
    best = None
    for eta0 in np.linspace(0.3, 1.0, 15):
        for link in [link_guess * f for f in (0.8, 0.9, 1.0, 1.1, 1.25, 1.5)]:
            # x - m/min(nc*b*eta, link) is nonlinear in b; search b too
            for b in np.geomspace(2e3, 1.2e5, 40):  # bytes/us per channel
                rows, ys = [], []
                for nc, nt, c, m, x in points:
                    eta = eta0 + (1 - eta0) * nt / 640.0
                    bw = min(nc * b * eta, link)
                    rows.append([1.0, nc, math.ceil(m / (nc * c))])
                    ys.append(x - m / bw)
                A, y = np.array(rows), np.array(ys)
                coef, *_ = np.linalg.lstsq(A, y, rcond=None)
                coef = np.maximum(coef, 0.0)
                res = A @ coef - y
                err = float(np.sqrt(np.mean((res / np.maximum(1.0, np.array([p[4] for p in points]))) ** 2)))
                if best is None or err < best[0]:
                    best = (err, eta0, link, b, coef)
    err, eta0, link, b, coef = best
    return {"base_latency": float(coef[0]), "per_channel_setup": float(coef[1]),
            "per_chunk_overhead": float(coef[2]), "per_channel_bw": float(b), "nt_floor": float(eta0)}, \
        float(link), err


def predict(co, link, nc, nt, c, m):
    eta = co["nt_floor"] + (1 - co["nt_floor"]) * nt / 640.0
    return co["base_latency"] + co["per_channel_setup"] * nc + math.ceil(m / (nc * c)) * co["per_chunk_overhead"] + \
        m / min(nc * co["per_channel_bw"] * eta, link)


def fit_footprint(over, y0, lam, b_chan, peak):
    """SM loss lambda/(lambda-NC) explains part of the victim's slowdown; the
    remainder is attributed to the comm's HBM footprint V (wave_time's
    blocks*D/(B - V) term) -> kappa, C_knee of the subspace (reference
    mem_footprint, commperf.cpp:127-135)."""
    rows = []
    for nc, c, y, _ in over:
        sm_part = y0 * lam / (lam - nc)
        rows.append((nc, c, max(0.0, y / sm_part - 1.0)))
    best = None
    for knee in [32 * KIB, 64 * KIB, 128 * KIB, 256 * KIB, 512 * KIB, 1 * MIB]:
        X = np.array([[nc * c / (c + knee)] for nc, c, _ in rows])
        Y = np.array([e for *_, e in rows])
        k, *_ = np.linalg.lstsq(X, Y, rcond=None)
        err = float(np.sum((X @ k - Y) ** 2))
        if best is None or err < best[0]:
            best = (err, knee, float(k[0]))
    _, knee, slope = best
    # slope ~ V/(B - V) per (NC*sat) ~= kappa*b_chan/B for V << B
    return max(0.0, slope * peak / b_chan), int(knee)


def fit_all(meas, meas_coll, over, y0, lam, over_tree=()):
    """Fits the reference cost model's coefficients from the measurements
    (median-relative-error least squares, tools/predict_vs_measured.fit)."""
    from tools.predict_vs_measured import fit as fit_model
    params, report = {}, {}
    for key, pts in meas.items():
        co, link, rep = fit_model(pts)
        co.update({"mem_coeff": 0.5, "chunk_knee": 128 * KIB})
        params[key] = co
        report[key] = dict(rep, link_bw=link)
    peak = 6434.2e3  # bytes/us, measured copy bandwidth (MEASURED_PEAKS.json)
    for key, ov in (("RING/SIMPLE/P2P", over), ("TREE/SIMPLE/P2P", over_tree)):
        if ov and key in params:
            kappa, knee = fit_footprint(ov, y0, lam, params[key]["per_channel_bw"], peak)
            params[key]["mem_coeff"] = kappa
            params[key]["chunk_knee"] = knee
    # Per-collective traffic factors, fitted on the TREE key (the subspace
    # the search selects on an NVSwitch box).
    factors, factor_report = {"ALL_REDUCE": 2.0}, {}
    if "TREE/SIMPLE/P2P" in params and meas_coll.get("TREE/SIMPLE/P2P"):
        co, lk = params["TREE/SIMPLE/P2P"], report["TREE/SIMPLE/P2P"]["link_bw"]
        for coll, pts in meas_coll["TREE/SIMPLE/P2P"].items():
            err, f, p90 = fit_factor(co, lk, [tuple(p) for p in pts])
            factors[coll] = f
            factor_report[coll] = {"factor": f, "median_rel_err": err, "p90_rel_err": p90, "points": len(pts)}
    for coll in COLLS[1:]:
        factors.setdefault(coll, 1.0)
    params["collective_factors"] = factors
    gpu = {"num_sms": lam, "peak_mem_bw": peak, "link_bw": max(r["link_bw"] for r in report.values()),
           "comm_bw_cap_fraction": 0.6, "compute_on_comm_slowdown": 0.0}
    return params, gpu, report, factor_report


def validate(L, gpu, params):
    """Loads the params document with the product loader (reference schema)."""
    L.tune_sim(json.dumps({"gpu": gpu, "compute_ops": [{"id": "c", "total_blocks": 1, "blocks_per_sm": 1,
                                                        "bytes_per_block": 0, "base_wave_time": 1.0}],
                           "comm_ops": [{"id": "k", "collective": "ALL_REDUCE", "message_bytes": 1 << 20}]}),
               "min", 5, json.dumps(params))


def refit(path, out):
    """GPU-free: recomputes every fit from a stored profile's measurements."""
    from paper_2602_20656_b200 import _lagom_py as L
    prof = json.load(open(path))
    meas = {k: [tuple(p) for p in v] for k, v in prof["measurements"].items()}
    params, gpu, report, factor_report = fit_all(meas, prof.get("measurements_other", {}),
                                                 prof["victim"]["overlapped"], prof["victim"]["y_alone_us"],
                                                 prof["gpu"]["num_sms"], prof["victim"].get("overlapped_tree", ()))
    validate(L, gpu, params)
    prof.update(params=params, gpu=gpu, fit_report=report, factor_report=factor_report)
    with open(out, "w") as f:
        json.dump(prof, f, indent=1)
    print(json.dumps({"fit_report": report, "factor_report": factor_report}, indent=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/fitted_params.json")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--nvls", type=int, default=1, help="TREE = in-switch (NVLS) when the box supports it")
    ap.add_argument("--refit", default="", help="recompute the fits of a stored profile (no GPU) into --out")
    a = ap.parse_args()
    if a.refit:
        return refit(a.refit, a.out)
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    import torch
    import torch.distributed as dist

    from paper_2602_20656_b200 import _lagom_py as L
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
        tok = [secrets.token_hex(6) if rank == 0 else None]
        dist.broadcast_object_list(tok, src=0)
        token = tok[0]
    else:
        token = secrets.token_hex(6)
    sizes = [1, 8, 32] if a.quick else [1, 4, 16, 64, 256]
    gemm = [8192, 8192, 2048]  # a 275 GFLOP compute-bound victim op (x8 per replay)
    dag = dag_for(sizes, gemm, world)
    dag_ar = dict(dag, comm_ops=[op for op in dag["comm_ops"] if op["collective"] == "ALL_REDUCE"])

    def engine(d, tag):
        return L.ReplayEngine(json.dumps(d), f"lagom_cp{tag}_{token}", rank, world, local, repeats=3, warmup=1,
                              nccl=False, sm_partition=2, nvls=bool(a.nvls), max_channels=64)
    eng = engine(dag, "a")
    if rank != 0:  # serve phase 1 (comm alone), then phase 2 (victim overlapped)
        eng.serve()
        eng.close()
        eng = engine(dag_ar, "b")
        eng.serve()
        eng.close()
        if world > 1:
            dist.barrier()
        return
    ncs = [1, 2, 4, 8, 16, 32, 64]
    nts = [64, 256, 640]
    chunks = [32 * KIB, 256 * KIB, 1 * MIB, 4 * MIB]
    keys = [("RING", "SIMPLE"), ("RING", "LL"), ("RING", "LL128"), ("TREE", "SIMPLE")]
    if a.quick:
        ncs, nts, chunks, keys = [1, 4, 16], [256, 640], [256 * KIB, 2 * MIB], keys[:2]
    meas, meas_coll = {}, {}
    factor = 2.0  # AllReduce traffic factor (reference collective_factors)
    nops = len(dag["comm_ops"])
    for (algo, proto) in keys:
        pts, other = [], {c: [] for c in COLLS[1:]}
        for nc, nt, c in itertools.product(ncs, nts, chunks):
            if proto == "LL" and c > 1 * MIB:
                continue
            r = json.loads(eng.run_comm_only(json.dumps({"configs": [cfg(algo, proto, nc, nt, c)] * nops})))
            for op, x in zip(dag["comm_ops"], r["x"]):
                s = int(op["id"].lstrip("abcdefghijklmnopqrstuvwxyz_"))
                if op["collective"] == "ALL_REDUCE":
                    pts.append((nc, nt, c, s * MIB * factor, x))
                else:
                    other[op["collective"]].append((nc, nt, c, s * MIB, x))
        meas[f"{algo}/{proto}/P2P"] = pts
        meas_coll[f"{algo}/{proto}/P2P"] = other
        print(f"[profile] {algo}/{proto}: {len(pts)} AllReduce points (+ AG/RS/A2A)", flush=True)
    eng.stop()
    eng.close()
    # victim alone and overlapped (AllReduce ops only)
    eng = engine(dag_ar, "b")
    y0 = json.loads(eng.run_compute_only())["Y"]
    over, over_tree = [], []
    for nc, c in itertools.product([1, 2, 4, 8, 16, 32], [64 * KIB, 1 * MIB, 4 * MIB]):
        r = json.loads(eng.run(json.dumps({"configs": [cfg("RING", "SIMPLE", nc, 512, c)] * len(sizes)})))
        over.append((nc, c, r["Y"], r["X"]))
    if ("TREE", "SIMPLE") in keys:  # the in-switch (NVLS) kernels' footprint on the victim
        for nc, c in itertools.product([1, 2, 4, 8, 16, 32], [64 * KIB, 1 * MIB, 4 * MIB]):
            r = json.loads(eng.run(json.dumps({"configs": [cfg("TREE", "SIMPLE", nc, 512, c)] * len(sizes)})))
            over_tree.append((nc, c, r["Y"], r["X"]))
    eng.stop()
    eng.close()

    lam = torch.cuda.get_device_properties(local).multi_processor_count
    params, gpu, report, factor_report = fit_all(meas, meas_coll, over, y0, lam, over_tree)
    from paper_2602_20656_b200 import _lagom_py as L2
    validate(L2, gpu, params)
    out = {"nranks": world, "params": params, "gpu": gpu, "fit_report": report, "factor_report": factor_report,
           "victim": {"y_alone_us": y0, "overlapped": over, "overlapped_tree": over_tree}, "measurements": meas,
           "measurements_other": meas_coll}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({"fit_report": report, "factor_report": factor_report, "gpu": gpu,
                      "RING/SIMPLE": params["RING/SIMPLE/P2P"]}), flush=True)
    if world > 1:
        dist.barrier()


if __name__ == "__main__":
    main()
