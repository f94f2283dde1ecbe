"""Counter-backed contention model for one GPU count: the reference's cost
and contention model (commperf.cpp:108-135, contention.cpp:22-72) fitted to
CUPTI-counter profiles of every workload (tools/counter_profile.py), then
simulate() — the product's, bit-identical to the reference's — predicts

  * every profiled config set's overlapped Z (the profile measured it), and
  * every bench row's overlapped Z at the tuned picks (bench.py --out),

and states the error against the measurement.

  python tools/counter_fit.py --n 2 --profiles gpurun_out/r2_counters_n2_*.json \
      --bench gpurun_out/r2_final_n2_*.json --out profiles/round2_model_n2.json

Calibration (no GPU; every input is a measurement in the files):
  comm_time   per subspace, least squares over every set's comm-alone kernel
              spans x_j (all workloads; m = message bytes x collective factor);
  V           mem_footprint's mem_coeff / chunk_knee per subspace, from each
              set's measured HBM bytes per us of comm;
  D, theta    per compute op: HBM bytes (compute-only replay) / blocks, blocks
              = lambda x waves; theta matches the isolated time at V = 0;
  regime      a set whose kernels ride along the GEMMs (co-resident: TREE with
              NT <= 256 on NVLS) holds no SMs (SimOptions.sm_occupancy =
              false); dedicated sets lose their NC SMs (sm_occupancy = true);
              each regime's bandwidth B (reference wave_time's peak_mem_bw -
              V, with theta refitted so the isolated time is unchanged) is
              fitted;
  delta       compute_on_comm_slowdown, one per regime;
four global parameters (delta and the effective bandwidth B of each regime)
fitted by grid search over all sets of all workloads (median |Z error|): the
bandwidth the overlapped victims see is below the HBM copy peak once the
collective's traffic shares the L2 and the SMs' memory pipes, and the fit
states how far.
"""
import argparse
import glob
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tools.contention_profile import predict as comm_predict  # noqa: E402
from tools.predict_vs_measured import KIB, MIB, _builder, fit  # noqa: E402

LAMBDA, WAVES = 148, 16


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return (json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6540.8) * 1e3  # bytes/us


# At two ranks the product runs TREE AllGather / ReduceScatter one hop from
# ONE_HOP_MIN_NC channels up (lagom_comm_opts_t.one_hop = 2), and through the
# switch below: two schedules inside one reference subspace, which one
# comm_time curve cannot fit. With --one-hop-min-nc the one-hop configs get
# their own subspace key (transport SHM: the reference's Transport enum, used
# here as the "peer mappings, not the switch" label) in the fitted params and
# in the configs handed to simulate(). None: one key per (algorithm, protocol).
ONE_HOP_MIN_NC = None


def key_of(cfg, coll=None, n=None):
    if (ONE_HOP_MIN_NC and n == 2 and cfg["algorithm"] == "TREE" and coll in ("ALL_GATHER", "REDUCE_SCATTER")
            and cfg["num_channels"] >= ONE_HOP_MIN_NC):
        return f"{cfg['algorithm']}/{cfg['protocol']}/SHM"
    return f"{cfg['algorithm']}/{cfg['protocol']}/P2P"


def with_key(cfg, coll, n):
    """cfg as simulate() must see it: transport per key_of."""
    return dict(cfg, transport=key_of(cfg, coll, n).split("/")[2])


def coresident(cfg, nvls):
    return cfg["algorithm"] == "TREE" and cfg["num_threads"] <= 256 and nvls


class Workload:
    def __init__(self, prof):
        from paper_2602_20656_b200 import dags
        self.prof = prof
        self.n = prof["n"]
        self.dag = dags.BUILDERS[_builder({"config": {"workload": prof["workload"]}})](self.n)
        self.sizes = []
        for c in self.dag["comm_ops"]:
            e = 2 if c.get("dtype", 1) in (1, 2) else 4
            self.sizes.append(c["count"] * e * (1 if c["collective"] == "ALL_REDUCE" else self.n))

    def work(self, gpu, bw, y_iso=None):
        """The reference Workload; y_iso (optional) overrides the isolated
        compute times (a bench run's own compute-only replays)."""
        comps = []
        for i, c in enumerate(self.dag["compute_ops"]):
            co = self.prof["compute_ops"][i]
            d = co["dram_bytes"] / (LAMBDA * WAVES)
            f = (y_iso[i] if y_iso is not None else co["y_us"]) / WAVES
            comps.append({"id": c["id"], "total_blocks": LAMBDA * WAVES, "blocks_per_sm": 1,
                          "bytes_per_block": int(round(d)),
                          "base_wave_time": max(1e-3, f - LAMBDA * round(d) / bw)})
        w = {"units": {"time": "us", "size": "bytes", "bandwidth": "bytes_per_us"}, "gpu": dict(gpu, peak_mem_bw=bw),
             "compute_ops": comps, "comm_ops": []}
        for j, c in enumerate(self.dag["comm_ops"]):
            op = {"id": c["id"], "collective": c["collective"], "message_bytes": self.sizes[j],
                  "bounds": {"nc_max": 64}}
            if c.get("ready_after"):
                op["ready_after"] = c["ready_after"]
            w["comm_ops"].append(op)
        return w


COLLS = ("ALL_REDUCE", "ALL_GATHER", "REDUCE_SCATTER", "ALL_TO_ALL")


def fit_params(wls, extra=()):
    """comm_time per subspace on its AllReduce points (or its most measured
    collective), then the reference's collective_factors
    (default_params.json:164-169) — one message-size factor per collective —
    by 1-D search against those coefficients (median relative error).
    extra: (key, collective, nc, nt, c, bytes, x) comm-alone points measured
    elsewhere (the bench runs' comm-only replays at the tuned picks)."""
    by_key = {}
    for key, coll, *pt in extra:
        by_key.setdefault(key, {}).setdefault(coll, []).append(tuple(pt))
    for wl in wls:
        for st in wl.prof["sets"].values():
            cfg = st["config"]
            for j, co in enumerate(st["comm_ops"]):
                coll = wl.dag["comm_ops"][j]["collective"]
                by_key.setdefault(key_of(cfg, coll, wl.n), {}).setdefault(coll, []).append(
                    (cfg["num_channels"], cfg["num_threads"], cfg["chunk_size"], wl.sizes[j], co["x_us"]))
    params, report, links = {}, {}, {}
    factors = {"ALL_REDUCE": 2.0}
    main_key = max(by_key, key=lambda k: sum(len(v) for v in by_key[k].values()))
    # the main subspace first: its collective factors scale the other subspaces' base points
    for key, colls in sorted(by_key.items(), key=lambda kv: kv[0] != main_key):
        base = "ALL_REDUCE" if "ALL_REDUCE" in colls else max(colls, key=lambda c: len(colls[c]))
        bf = 2.0 if base == "ALL_REDUCE" else (factors.get(base, 1.0) if key != main_key else 1.0)
        co, lk, rep = fit([(nc, nt, c, m * bf, x) for nc, nt, c, m, x in colls[base]])
        params[key], links[key] = co, lk
        report[key] = dict(rep, link_bw=lk, base_collective=base)
        if key != main_key:
            continue
        factors[base] = bf
        for coll, pts in colls.items():
            if coll == base:
                continue
            best = None
            for f in np.geomspace(0.1, 10.0, 241):
                rel = [abs(comm_predict(co, lk, nc, nt, c, m * f) - x) / x for nc, nt, c, m, x in pts]
                err = float(np.median(rel))
                if best is None or err < best[0]:
                    best = (err, float(f))
            factors[coll] = best[1]
            report[key][f"factor_{coll}"] = {"factor": best[1], "median_rel_err": best[0], "points": len(pts)}
    for key in by_key:  # footprint V: HBM bytes per us of comm, per set
        vpts = []
        for wl in wls:
            for st in wl.prof["sets"].values():
                cfg = st["config"]
                if key_of(cfg, wl.dag["comm_ops"][0]["collective"], wl.n) == key:
                    xs = sum(c["x_us"] for c in st["comm_ops"])
                    vpts.append((cfg["num_channels"], cfg["chunk_size"],
                                 sum(c["dram_bytes"] for c in st["comm_ops"]) / xs))
        bch = params[key]["per_channel_bw"]
        best = None
        for knee in (KIB, 16 * KIB, 64 * KIB, 256 * KIB, MIB):
            basis = [nc * c / (c + knee) * bch for nc, c, _ in vpts]
            den = sum(b * b for b in basis)
            kappa = sum(b * v for b, (_, _, v) in zip(basis, vpts)) / den if den else 0.0
            err = sum((kappa * b - v) ** 2 for b, (_, _, v) in zip(basis, vpts))
            if best is None or err < best[0]:
                best = (err, kappa, knee)
        params[key]["mem_coeff"], params[key]["chunk_knee"] = float(best[1]), int(best[2])
        report[key]["V_points_GBps"] = [round(v / 1e3, 1) for _, _, v in vpts]
    base = next(iter(params.values()))
    for key in ("RING/SIMPLE/P2P", "RING/LL/P2P", "RING/LL128/P2P", "TREE/SIMPLE/P2P", "TREE/LL/P2P",
                "TREE/LL128/P2P"):
        params.setdefault(key, dict(base))
    params["collective_factors"] = {c: factors.get(c, 1.0) for c in COLLS}
    return params, report, links


def predict(wl, cfgs, params, links, g, nvls, y_iso=None):
    from paper_2602_20656_b200 import _lagom_py as L
    co = all(coresident(c, nvls) for c in cfgs)
    cfgs = [with_key(c, op["collective"], wl.n) for c, op in zip(cfgs, wl.dag["comm_ops"])]
    key = "/".join((cfgs[0]["algorithm"], cfgs[0]["protocol"], cfgs[0]["transport"]))
    bw = g["B_co"] if co else g["B_ded"]
    gpu = {"num_sms": LAMBDA, "link_bw": links.get(key, next(iter(links.values()))), "comm_bw_cap_fraction": 0.6,
           "compute_on_comm_slowdown": g["delta_co"] if co else g["delta_ded"]}
    sim = json.loads(L.simulate(json.dumps(wl.work(gpu, bw, y_iso)), json.dumps({"configs": cfgs}),
                                json.dumps(params), not co))
    return sim, co


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--profiles", nargs="+", required=True)
    ap.add_argument("--bench", nargs="*", default=[])
    ap.add_argument("--out", default="")
    ap.add_argument("--globals", default="", help="take the four global parameters from this model file "
                    "instead of the grid search (re-derives its rows; tests/test_model_fit_cpu.py)")
    ap.add_argument("--one-hop-min-nc", type=int, default=0,
                    help="two-rank TREE AG/RS at >= this NC get their own subspace (the product's one_hop = 2 "
                         "threshold, 16; 0 = off). Taken from --globals' file when it records one")
    a = ap.parse_args()
    global ONE_HOP_MIN_NC
    ONE_HOP_MIN_NC = a.one_hop_min_nc or None
    if a.globals:
        ONE_HOP_MIN_NC = json.load(open(a.globals)).get("one_hop_min_nc") or ONE_HOP_MIN_NC
    profs = [json.load(open(p)) for f in a.profiles for p in sorted(glob.glob(f))]
    wls = [Workload(p) for p in profs if p["n"] == a.n]
    benches = []
    for f in a.bench:
        for p in sorted(glob.glob(f)):
            if p.endswith("_lagom.json") or p.endswith("_nccl.json"):
                continue
            b = json.load(open(p))
            if b["line"]["n_gpus"] == a.n:
                benches.append(b)
    # the bench runs' comm-only replays at the tuned picks join the comm fit
    extra = []
    for b in benches:
        wl = next((w for w in wls if w.prof["workload"] == b["line"]["config"]["workload"]), None)
        if wl is None:
            continue
        cfgs = [b["tune"]["configs"][gi] for gi in _groups(wl.dag)]
        xs = np.median([r["x"] for r in b["raw"]["comm"]], axis=0)
        for j, cfg in enumerate(cfgs):
            extra.append((key_of(cfg, wl.dag["comm_ops"][j]["collective"], a.n), wl.dag["comm_ops"][j]["collective"],
                          cfg["num_channels"], cfg["num_threads"],
                          cfg["chunk_size"], wl.sizes[j], float(xs[j])))
    params, report, links = fit_params(wls, extra)
    B = hbm_peak()
    sets = [(wl, spec, st) for wl in wls for spec, st in wl.prof["sets"].items()]

    def errors(g):
        out = []
        for wl, spec, st in sets:
            sim, co = predict(wl, [st["config"]] * len(wl.sizes), params, links, g, wl.prof.get("nvls", False))
            out.append((sim["Z"] - st["overlapped"]["Z"]) / st["overlapped"]["Z"])
        return out

    best = None
    fractions = (1.0, 1 / 1.5, 1 / 2, 1 / 3, 1 / 4, 1 / 6)
    if a.globals:
        g0 = json.load(open(a.globals))["global"]
        best = (float(np.median(np.abs(errors(g0)))), g0)
    for dd in (() if a.globals else (0.0, 0.1, 0.2, 0.3, 0.5)):
        for dc in (0.0, 0.1, 0.2, 0.3, 0.5, 0.8):
            for fd in fractions:
                for fc in fractions:
                    g = {"B": B, "B_ded": B * fd, "B_co": B * fc, "delta_ded": dd, "delta_co": dc}
                    e = errors(g)
                    score = float(np.median(np.abs(e)))
                    if best is None or score < best[0]:
                        best = (score, g)
    g = best[1]
    rows = []
    for wl, spec, st in sets:
        sim, co = predict(wl, [st["config"]] * len(wl.sizes), params, links, g, wl.prof.get("nvls", False))
        m = st["overlapped"]
        rows.append({"workload": wl.prof["workload"], "set": spec, "coresident": co,
                     "Z_pred": sim["Z"], "Z_meas": m["Z"], "Z_err": (sim["Z"] - m["Z"]) / m["Z"],
                     "Y_err": (sim["Y"] - m["Y"]) / m["Y"]})
    bench_rows = []
    for b in benches:
        line = b["line"]
        wname = line["config"]["workload"]
        wl = next((w for w in wls if w.prof["workload"] == wname), None)
        if wl is None:
            continue
        cfgs = [b["tune"]["configs"][gi] for gi in _groups(wl.dag)]
        nvls = line["lagom"]["nvls"]["active"]
        # isolated compute times from the bench run's own interleaved compute-only arm
        y_iso = [float(v) for v in np.median([r["y"] for r in b["raw"]["compute"]], axis=0)]
        sim, co = predict(wl, cfgs, params, links, g, nvls, y_iso)
        meas = line["arms_ms"]["lagom"] * 1e3
        bench_rows.append({"workload": wname, "n": a.n, "picks": sorted(set(line["lagom"]["tune"]["picks"])),
                           "coresident": co, "Z_pred": sim["Z"], "Z_meas": meas, "Z_err": (sim["Z"] - meas) / meas,
                           "Y_pred": sim["Y"], "Y_meas": line["compute"]["overlapped_ms"] * 1e3})
    res = {"n": a.n, "one_hop_min_nc": ONE_HOP_MIN_NC, "global": g, "fit_score_median_abs_Z_err": best[0],
           "params": params, "fit_report": report,
           "sets": rows, "bench_rows": bench_rows,
           "note": "sets: the profile's own overlapped replays (every comm op at one config); bench_rows: bench.py's "
                   "Lagom arm at the tuned picks, measured in a separate run"}
    for r in rows:
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}))
    for r in bench_rows:
        print("BENCH", json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}))
    print(json.dumps({"global": g, "median_abs_Z_err": best[0]}))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


def _groups(dag):
    last = dag["compute_ops"][-1]["id"]
    nroles = 1 + max(int(c.get("role", 0)) for c in dag["comm_ops"])
    g = [int(c.get("role", 0)) + (nroles if c.get("ready_after") == last else 0) for c in dag["comm_ops"]]
    present = sorted(set(g))
    return [present.index(x) for x in g]


if __name__ == "__main__":
    main()
