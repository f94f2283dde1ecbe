"""Predicted (model) vs measured (B200 replay) overlapped-iteration time.

  python tools/predict_vs_measured.py --profile profiles/round1_contention_profile_n4.json \
      --bench profiles/round1_bench_n4_gpt2-1.3b-dp.json --out profiles/round1_predict_vs_measured.json

1. Refits the reference cost model (comm_time, reference commperf.cpp:112-125)
   to the contention profiler's comm-alone measurements, per subspace, and
   writes the coefficients in the reference params schema.
2. Builds the model Workload of the bench DAG: comm ops from their message
   sizes; each compute op calibrated from its measured isolated time y_i
   (mu = lambda x W CTAs, TB = 1, theta = y_i / W, D from the fitted HBM
   footprint), so the wave model's lambda - NC term carries the SM partition.
3. simulate() (the product simulator, bit-identical to the reference's) with
   the tuned configs -> predicted X, Y, Z; compares with the bench's measured
   medians and states the relative error.
"""
import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

KIB = 1024
MIB = 1 << 20


def fit(points):
    """Least squares on x = a + z*NC + ceil(m/(NC*C))*o + m/min(NC*b*eta(NT), link)."""
    xs = np.array([p[4] for p in points])
    best = None
    link_hi = max(p[3] / p[4] for p in points)
    for eta0 in np.linspace(0.05, 1.0, 20):
        for link in link_hi * np.array([0.9, 1.0, 1.1, 1.3, 1.6]):
            for b in np.geomspace(2e3, 1e6, 70):  # bytes/us per channel (NVLS channels reach ~2e5)
                A = np.array([[1.0, p[0], math.ceil(p[3] / (p[0] * p[2]))] for p in points])
                bw = np.array([min(p[0] * b * (eta0 + (1 - eta0) * p[1] / 640.0), link) for p in points])
                y = xs - np.array([p[3] for p in points]) / bw
                coef, *_ = np.linalg.lstsq(A, y, rcond=None)
                coef = np.maximum(coef, 0.0)
                pred = A @ coef + np.array([p[3] for p in points]) / bw
                err = float(np.median(np.abs(pred - xs) / xs))
                if best is None or err < best[0]:
                    best = (err, eta0, link, b, coef, pred)
    err, eta0, link, b, coef, pred = best
    rel = np.abs(pred - xs) / xs
    return ({"base_latency": float(coef[0]), "per_channel_bw": float(b), "per_chunk_overhead": float(coef[2]),
             "per_channel_setup": float(coef[1]), "mem_coeff": 0.0, "chunk_knee": 128 * KIB, "nt_floor": float(eta0)},
            float(link), {"median_rel_err": float(np.median(rel)), "p90_rel_err": float(np.percentile(rel, 90)),
                          "max_rel_err": float(rel.max()), "points": len(points)})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", default="")
    ap.add_argument("--bench", default="")
    ap.add_argument("--counters", default="", help="a counter profile (tools/counter_profile.py): fit the "
                    "model from CUPTI counters and predict its measured config sets")
    ap.add_argument("--out", default="")
    ap.add_argument("--waves", type=int, default=16)
    ap.add_argument("--fit-cache", default="", help="reuse (or write) the comm-model fit of --profile")
    ap.add_argument("--hbm-share", type=float, default=0.0,
                    help="fraction of each isolated wave time put in the wave model's HBM term "
                         "blocks*D/(B - V) (reference contention.cpp:35-44), the rest in theta; "
                         "0 = no HBM term (the comm footprint V then has no effect)")
    a = ap.parse_args()
    if a.counters:
        res = counter_model(a.counters, a.waves, a.out)
        for r in res["rows"]:
            print(json.dumps({"set": r["set"], "coresident": r["coresident"], "Z_pred": round(r["predicted"]["Z"], 1),
                              "Z_meas": round(r["measured"]["Z"], 1), "Z_err": round(r["rel_err"]["Z"], 4),
                              "Y_err": round(r["rel_err"]["Y"], 4), "V_GBps": round(r["V_GBps"], 1)}))
        return
    from paper_2602_20656_b200 import _lagom_py as L
    from paper_2602_20656_b200 import dags

    prof = json.load(open(a.profile))
    params, report, link = {}, {}, None
    if a.fit_cache and os.path.exists(a.fit_cache):  # the same profile's fit, computed once
        with open(a.fit_cache) as f:
            params, report, link = (lambda d: (d["params"], d["report"], d["link"]))(json.load(f))
    else:
        for key, pts in prof["measurements"].items():
            co, lk, rep = fit(pts)
            params[key] = co
            report[key] = dict(rep, link_bw=lk)
            if key == "RING/SIMPLE/P2P":
                link = lk
        if a.fit_cache:
            with open(a.fit_cache, "w") as f:
                json.dump({"params": params, "report": report, "link": link}, f)
    # footprint from the overlapped-victim sweeps (reference mem_footprint form)
    for key in ("RING/SIMPLE/P2P", "TREE/SIMPLE/P2P"):
        if key in params and key in prof["params"]:
            params[key]["mem_coeff"] = prof["params"][key]["mem_coeff"]
            params[key]["chunk_knee"] = prof["params"][key]["chunk_knee"]
    params["collective_factors"] = prof["params"].get(
        "collective_factors", {"ALL_REDUCE": 2.0, "ALL_GATHER": 1.0, "REDUCE_SCATTER": 1.0, "ALL_TO_ALL": 1.0})

    bench = json.load(open(a.bench))
    line, raw = bench["line"], bench["raw"]
    nranks = line["n_gpus"]
    dag = dags.BUILDERS[line["config"]["workload"].rsplit("-", 1)[0] if False else _builder(line)](nranks)
    groups = _groups(dag)
    cfgs = [bench["tune"]["configs"][g] for g in groups]
    # The reference model has ONE link cap (GpuSpec.link_bw, commperf.cpp:112-125):
    # take the fitted cap of the subspace the tuned configs run in.
    keys = {f"{c['algorithm']}/{c['protocol']}/{c['transport']}" for c in cfgs}
    if len(keys) == 1 and next(iter(keys)) in report:
        link = report[next(iter(keys))]["link_bw"]
    y_iso = np.median([r["y"] for r in raw["compute"]], axis=0)
    lam = prof["gpu"]["num_sms"]
    W = a.waves
    # delta (reference GpuSpec.compute_on_comm_slowdown): comm progresses at
    # 1/(1+delta) while a compute wave runs — fitted as the ratio of the comm
    # kernels' active time overlapped vs alone in the same bench run.
    x_alone = float(np.median([r["X"] for r in raw["comm"]]))
    x_over = float(np.median([r["X"] for r in raw["lagom"]]))
    delta = max(0.0, x_over / x_alone - 1.0)
    gpu = dict(prof["gpu"], link_bw=link, compute_on_comm_slowdown=delta)
    work = {"units": {"time": "us", "size": "bytes", "bandwidth": "bytes_per_us"}, "gpu": gpu,
            "compute_ops": [compute_op(c["id"], float(y), lam, W, gpu["peak_mem_bw"], a.hbm_share)
                            for c, y in zip(dag["compute_ops"], y_iso)],
            "comm_ops": []}
    for c in dag["comm_ops"]:
        e = 2 if c.get("dtype", 1) in (1, 2) else 4
        mb = c["count"] * e * (1 if c["collective"] == "ALL_REDUCE" else nranks)
        op = {"id": c["id"], "collective": c["collective"], "message_bytes": mb}
        if c.get("ready_after"):
            op["ready_after"] = c["ready_after"]
        work["comm_ops"].append(op)
    sim = json.loads(L.simulate(json.dumps(work), json.dumps({"configs": cfgs}), json.dumps(params)))
    meas = {k: float(np.median([r[k] for r in raw["lagom"]])) for k in ("X", "Y", "Z")}
    out = {"fit_report": report, "params": params, "gpu": gpu,
           "predicted": {"X": sim["X"], "Y": sim["Y"], "Z": sim["Z"]}, "measured": meas,
           "rel_err": {k: (sim[k] - meas[k]) / meas[k] for k in ("X", "Y", "Z")},
           "workload": line["config"]["workload"], "n_gpus": nranks,
           "delta_fit": {"x_alone_us": x_alone, "x_overlapped_us": x_over, "delta": delta},
           "note": "X = sum of kernel active spans (measured) vs sum of comm_time (model); Y, Z in us"}
    print(json.dumps({k: out[k] for k in ("predicted", "measured", "rel_err", "fit_report")}, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)
        with open(a.out.replace(".json", "_params.json"), "w") as f:
            json.dump(params, f, indent=2)


def compute_op(op_id, y_iso, lam, waves, peak, hbm_share):
    """A compute op calibrated to its isolated time: `waves` full waves of
    lambda CTAs; a share of each wave's time goes to the HBM term so the
    comm's footprint V can slow it (f = theta + blocks*D/(B - V))."""
    f = y_iso / waves
    d = hbm_share * f * peak / lam  # blocks * D / B = hbm_share * f at V = 0
    return {"id": op_id, "total_blocks": lam * waves, "blocks_per_sm": 1,
            "bytes_per_block": int(round(d)), "base_wave_time": f - lam * int(round(d)) / peak}


def _builder(line):
    w = line["config"]["workload"]
    for k in ("gpt2-1.3b-dp", "llama3-8b-tp", "llama3-70b", "mixtral-8x7b-ep"):
        if w.startswith(k):
            return {"llama3-8b-tp": "llama3-8b-tp-sp", "llama3-70b": "llama3-70b-fsdp"}.get(k, k)
    raise SystemExit(f"unknown workload {w}")


def _groups(dag):
    last = dag["compute_ops"][-1]["id"]
    nroles = 1 + max(int(c.get("role", 0)) for c in dag["comm_ops"])
    g = [int(c.get("role", 0)) + (nroles if c.get("ready_after") == last else 0) for c in dag["comm_ops"]]
    present = sorted(set(g))
    return [present.index(x) for x in g]



# ------------------------------------------------------------------ counters
def counter_model(profile_path, waves=16, out=""):
    """Predicted vs measured from one counter profile (tools/counter_profile.py):
    the reference model calibrated from CUPTI counters, then simulate()
    (bit-identical to the reference's) predicts every measured config set's
    overlapped Z, which the same run measured.

      comm_time  (commperf.cpp:112-125): fitted per subspace to the sets'
                 comm-alone kernel spans x_j;
      V          (mem_footprint, commperf.cpp:127-135): mem_coeff / chunk_knee
                 fitted to each set's measured HBM bytes per us of comm;
      D          (ComputeOp.bytes_per_block): each compute op's measured HBM
                 bytes / its blocks (lambda x waves CTAs); theta so that the
                 isolated time is matched: f = theta + blocks*D/(B - V);
      delta      (compute_on_comm_slowdown): median over sets of overlapped /
                 alone comm span - 1;
      sm_occupancy (SimOptions): False for sets whose kernels ride along the
                 GEMMs (co-resident regime), True where they take SMs."""
    from paper_2602_20656_b200 import _lagom_py as L
    from paper_2602_20656_b200 import dags
    prof = json.load(open(profile_path))
    n = prof["n"]
    wl = prof["workload"]
    dag = dags.BUILDERS[_builder({"config": {"workload": wl}})](n)
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else {}
    B = peaks.get("hbm_gbs", 6540.8) * 1e3  # bytes/us
    lam = 148
    sizes = []
    for c in dag["comm_ops"]:
        e = 2 if c.get("dtype", 1) in (1, 2) else 4
        sizes.append(c["count"] * e * (1 if c["collective"] == "ALL_REDUCE" else n))
    # comm_time fit per subspace over every set's comm-alone spans
    by_key = {}
    for spec, st in prof["sets"].items():
        cfg = st["config"]
        key = f"{cfg['algorithm']}/{cfg['protocol']}/P2P"
        for j, co in enumerate(st["comm_ops"]):
            f = 2.0 if dag["comm_ops"][j]["collective"] == "ALL_REDUCE" else 1.0
            by_key.setdefault(key, []).append((cfg["num_channels"], cfg["num_threads"], cfg["chunk_size"],
                                               sizes[j] * f, co["x_us"]))
    params, report, links = {}, {}, {}
    for key, pts in by_key.items():
        co, lk, rep = fit(pts)
        params[key], links[key] = co, lk
        report[key] = dict(rep, link_bw=lk)
    # footprint V per set (HBM bytes per us of comm), fitted per subspace
    for key in by_key:
        vpts = []
        for spec, st in prof["sets"].items():
            cfg = st["config"]
            if f"{cfg['algorithm']}/{cfg['protocol']}/P2P" != key:
                continue
            xs = sum(c["x_us"] for c in st["comm_ops"])
            vpts.append((cfg["num_channels"], cfg["chunk_size"], sum(c["dram_bytes"] for c in st["comm_ops"]) / xs))
        bch = params[key]["per_channel_bw"]
        best = None
        for knee in (KIB, 16 * KIB, 64 * KIB, 256 * KIB, MIB):
            num = sum(v * nc * c / (c + knee) * bch for nc, c, v in vpts)
            den = sum((nc * c / (c + knee) * bch) ** 2 for nc, c, v in vpts)
            kappa = num / den if den else 0.0
            err = sum((kappa * nc * c / (c + knee) * bch - v) ** 2 for nc, c, v in vpts)
            if best is None or err < best[0]:
                best = (err, kappa, knee)
        params[key]["mem_coeff"] = float(best[1])
        params[key]["chunk_knee"] = int(best[2])
        report[key]["V_points"] = vpts
    for key in ("RING/SIMPLE/P2P", "RING/LL/P2P", "RING/LL128/P2P", "TREE/SIMPLE/P2P", "TREE/LL/P2P",
                "TREE/LL128/P2P"):
        params.setdefault(key, dict(next(iter(params.values()))))
    params["collective_factors"] = {"ALL_REDUCE": 2.0, "ALL_GATHER": 1.0, "REDUCE_SCATTER": 1.0, "ALL_TO_ALL": 1.0}
    # delta: comm slowdown under compute
    ratios = [sum(st["overlapped_x"]) / sum(c["x_us"] for c in st["comm_ops"]) for st in prof["sets"].values()]
    delta = max(0.0, float(np.median(ratios)) - 1.0)
    rows = []
    for spec, st in prof["sets"].items():
        cfg = st["config"]
        key = f"{cfg['algorithm']}/{cfg['protocol']}/P2P"
        coresident = cfg["algorithm"] == "TREE" and cfg["num_threads"] <= 256 and prof.get("nvls", False)
        gpu = {"num_sms": lam, "peak_mem_bw": B, "link_bw": links[key], "comm_bw_cap_fraction": 0.6,
               "compute_on_comm_slowdown": delta}
        comps = []
        for i, c in enumerate(dag["compute_ops"]):
            co = prof["compute_ops"][i]
            D = co["dram_bytes"] / (lam * waves)
            f = co["y_us"] / waves
            comps.append({"id": c["id"], "total_blocks": lam * waves, "blocks_per_sm": 1,
                          "bytes_per_block": int(round(D)), "base_wave_time": max(1e-3, f - lam * round(D) / B)})
        work = {"units": {"time": "us", "size": "bytes", "bandwidth": "bytes_per_us"}, "gpu": gpu,
                "compute_ops": comps, "comm_ops": []}
        for j, c in enumerate(dag["comm_ops"]):
            op = {"id": c["id"], "collective": c["collective"], "message_bytes": sizes[j], "bounds": {"nc_max": 64}}
            if c.get("ready_after"):
                op["ready_after"] = c["ready_after"]
            work["comm_ops"].append(op)
        sim = json.loads(L.simulate(json.dumps(work), json.dumps({"configs": [cfg] * len(sizes)}),
                                    json.dumps(params), not coresident))
        meas = st["overlapped"]
        rows.append({"set": spec, "coresident": coresident, "predicted": {k: sim[k] for k in ("X", "Y", "Z")},
                     "measured": {k: meas[k] for k in ("X", "Y", "Z")},
                     "rel_err": {k: (sim[k] - meas[k]) / meas[k] for k in ("X", "Y", "Z")},
                     "V_GBps": sum(c["dram_bytes"] for c in st["comm_ops"]) / sum(c["x_us"] for c in st["comm_ops"])
                     / 1e3})
    res = {"workload": wl, "n": n, "params": params, "fit_report": report, "delta": delta,
           "hbm_bytes_per_us": B, "waves": waves, "rows": rows,
           "max_abs_Z_err": max(abs(r["rel_err"]["Z"]) for r in rows)}
    if out:
        with open(out, "w") as f:
            json.dump(res, f, indent=1)
    return res


if __name__ == "__main__":
    main()
