"""Prints DESIGN.md §6's result tables from the committed round-2 files:
bench lines (profiles/round2_final_n{N}_{workload}.json, and the same
session's repeat round2_final_rep2_n{N}_{workload}.json) and the
counter-backed models (profiles/round2_model_n{N}.json over the final
kernels' counters and bench lines; round2_model_session3_n{N}.json over
session 3's). No GPU.

  python tools/results_tables.py
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {"gpt2-1.3b-dp": "GPT-2 1.3B DP (2)", "llama3-8b-tp-sp": "Llama-3 8B TP-SP (3)",
         "llama3-70b-fsdp": "Llama-3 70B-layer FSDP (4)", "mixtral-8x7b-ep": "Mixtral 8x7B EP (5)"}


def load(name):
    p = os.path.join(ROOT, "profiles", name)
    return json.load(open(p)) if os.path.exists(p) else None


def picks(line):
    ps = sorted(set(line["lagom"]["tune"]["picks"]))
    ncs = sorted({int(p.split("/NC")[1].split("/")[0]) for p in ps})
    nts = sorted({int(p.split("/NT")[1].split("/")[0]) for p in ps})
    nc = f"NC{ncs[0]}" if len(ncs) == 1 else f"NC{ncs[0]}–{ncs[-1]}"
    nt = f"NT{nts[0]}" if len(nts) == 1 else f"NT{nts[0]}–{nts[-1]}"
    return f"{ps[0].split('/')[0]} {nc} {nt}"


def dominant_roofline(d, n):
    """The roofline of the config group with the largest summed x (bench.py's
    definition), recomputed from the line's raw replays: wire bytes per rank
    on the busier direction / CUDA-event time in the comm-only replay."""
    import statistics
    import sys
    sys.path.insert(0, ROOT)
    import bench
    from paper_2602_20656_b200 import dags
    line, raw = d["line"], d["raw"]
    w = next(k for k in NAMES if line["config"]["workload"].startswith(k.split("-")[0] + "-" + k.split("-")[1]))
    dag = dags.BUILDERS[w](n)
    last = dag["compute_ops"][-1]["id"]
    nroles = 1 + max(int(c.get("role", 0)) for c in dag["comm_ops"])
    g = [int(c.get("role", 0)) + (nroles if c.get("ready_after") == last else 0) for c in dag["comm_ops"]]
    present = sorted(set(g))
    groups = [present.index(x) for x in g]
    xs = {}
    for r in raw["lagom"]:
        for j, x in enumerate(r["x"]):
            xs[groups[j]] = xs.get(groups[j], 0.0) + x
    gd = max(xs, key=xs.get)
    j = groups.index(gd)
    cfg = d["tune"]["configs"][gd]
    t = statistics.median(r["x_ev"][j] for r in raw["comm"])
    nv = line["lagom"]["nvls"]
    oh = line["lagom"].get("one_hop", 0)
    hop = nv["peer_mappings"] and (oh == 1 or (oh == 2 and n == 2 and cfg["num_channels"] >= 16))
    wb, _ = bench.wire_bytes(dag["comm_ops"][j], n, cfg, nv["active"], nv["peer_mappings"], hop)
    peak = line["roofline"]["peak"]
    return wb / (t * 1e-6) / 1e9 / peak, f"{cfg['algorithm']} NC{cfg['num_channels']}/NT{cfg['num_threads']}"


def fmt(v, nd=2):
    return "—" if v is None else f"{v:.{nd}f}"


def bench_rows():
    out = ["| workload (BASELINE config) | N | Lagom-tuned | NCCL-default | speedup | ours @ seed | "
           "ours @ seed, partition always | NCCL + SM partition | compute only | picks | compute slowdown "
           "(Lagom / NCCL) | roofline frac (dominant group) | repeat: speedup, picks |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for n in (4, 2, 1):
        for w, name in NAMES.items():
            d = load(f"round2_final_n{n}_{w}.json")
            if not d:
                continue
            line = d["line"]
            a, c = line["arms_ms"], line["compute"]
            sp = line["speedup_vs_nccl_default"]
            sps = f"**{sp:.3f}×**" if sp and sp >= 1.07 else f"{sp:.3f}×"
            frac, dcfg = dominant_roofline(d, n)
            d2 = load(f"round2_final_rep2_n{n}_{w}.json")
            rep = "—"
            if d2:
                sp2 = d2["line"]["speedup_vs_nccl_default"]
                rep = (f"**{sp2:.3f}×**" if sp2 >= 1.07 else f"{sp2:.3f}×") + f", {picks(d2['line'])}"
            out.append(f"| {name} | {n} | {a['lagom']:.2f} | {fmt(a.get('nccl'))} | {sps} | {fmt(a.get('seed'))} | "
                       f"{fmt(a.get('seed_partition_all'))} | {fmt(a.get('nccl_partition'))} | {a['compute']:.2f} | "
                       f"{picks(line)} | {c['slowdown']:.3f} / {fmt(c.get('slowdown_nccl'), 3)} | "
                       f"{frac:.3f} ({dcfg}) | {rep} |")
    return "\n".join(out)


def model_rows(model="round2_model_n{n}.json"):
    out = ["| workload | N | picks | predicted Z (ms) | measured Z (ms) | error |", "|---|---|---|---|---|---|"]
    for n in (4, 2):
        m = load(model.format(n=n))
        if not m:
            continue
        for r in m["bench_rows"]:
            w = next((k for k in NAMES if r["workload"].startswith(k.split("-")[0] + "-" + k.split("-")[1])),
                     r["workload"])
            out.append(f"| {NAMES.get(w, r['workload'])} | {n} | {len(r['picks'])} configs | {r['Z_pred'] / 1e3:.2f} | "
                       f"{r['Z_meas'] / 1e3:.2f} | {r['Z_err'] * 100:+.1f} % |")
    return "\n".join(out)


def model_set_summary(model="round2_model_n{n}.json"):
    out = ["| N | sets | median abs Z error | within 5 % | delta (dedicated / co-resident) |", "|---|---|---|---|---|"]
    for n in (4, 2):
        m = load(model.format(n=n))
        if not m:
            continue
        errs = sorted(abs(r["Z_err"]) for r in m["sets"])
        within = sum(e <= 0.05 for e in errs)
        g = m["global"]
        out.append(f"| {n} | {len(errs)} | {errs[len(errs) // 2] * 100:.1f} % | {within} / {len(errs)} | "
                   f"{g['delta_ded']} / {g['delta_co']} |")
    return "\n".join(out)


if __name__ == "__main__":
    print(bench_rows())
    for tag, model in (("final kernels before the L2 prefetch, session B bench lines", "round2_model_n{n}.json"),
                       ("session 3 kernels", "round2_model_session3_n{n}.json")):
        print()
        print(f"model ({tag}):")
        print(model_rows(model))
        print()
        print(model_set_summary(model))
