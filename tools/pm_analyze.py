"""Window sums over CUPTI PM samples (tools/pm_probe.py, bench/profiler
replays with set_pm_sampling): integrates every sampled counter over a
replay's compute-op and comm-op windows.

A replay's timeline (reference trace schema: ts/dur in us from the replay
start) is placed on the samples' clock through the replay's %globaltimer
origin (pm.t0_ns, written by lagom_timestamp right after the replay's start
event). A sample [s, e) contributes value * |[s, e) ∩ window| / (e - s) to a
window (counts spread uniformly over the sample).
"""
from __future__ import annotations


def _cols(pm):
    return {m: i + 2 for i, m in enumerate(pm["metrics"])}


def window_sum(pm: dict, a_ns: float, b_ns: float) -> dict:
    cols = _cols(pm)
    tot = {m: 0.0 for m in cols}
    for row in pm["samples"]:
        s, e = row[0], row[1]
        if e <= a_ns or s >= b_ns or e <= s:
            continue
        f = (min(e, b_ns) - max(s, a_ns)) / (e - s)
        for m, c in cols.items():
            tot[m] += row[c] * f
    return tot


def activity_origin(pm: dict) -> float:
    """The replay's start on the samples' clock. CUPTI stamps samples with
    host-synchronised wall-clock time, which is offset from %globaltimer (by
    ~190 ms on the B200 boxes), so the origin is found from the counters: the
    start of the first sample with SM (else DRAM) activity above 5 % of its
    peak — every replay mode starts with work at t = 0 (the sampler is
    started right before the replay's first launch)."""
    cols = _cols(pm)
    key = next((k for k in ("sm__cycles_active.avg", "dram__bytes_read.sum", "dram__bytes.sum") if k in cols), None)
    rows = pm["samples"]
    if key is None:
        return float(rows[0][0])
    c = cols[key]
    peak = max(r[c] for r in rows) or 1.0
    for r in rows:
        if r[c] > 0.05 * peak:
            # counts are spread over the sample: place the start where the
            # sample's activity fraction says work began
            frac = min(1.0, r[c] / peak)
            return float(r[1] - frac * (r[1] - r[0]))
    return float(rows[0][0])


def summarize(m: dict, dag: dict) -> dict:
    """Per-op and whole-replay counter totals of one measurement JSON (the
    engine's measurement with a "pm" block)."""
    pm = m.get("pm")
    if not pm or not pm.get("samples"):
        return {"totals": {"samples": 0}, "ops": []}
    t0 = activity_origin(pm)
    ops = []
    for ev in m.get("trace", []):
        if ev.get("ph") != "X":
            continue
        a = t0 + ev["ts"] * 1e3
        b = a + ev["dur"] * 1e3
        w = window_sum(pm, a, b)
        ops.append({"name": ev["name"], "cat": ev.get("cat"), "ts_us": ev["ts"], "dur_us": ev["dur"],
                    **{k: v for k, v in w.items()}})
    z_end = t0 + m["Z"] * 1e3
    whole = window_sum(pm, t0, z_end)
    first, last = pm["samples"][0], pm["samples"][-1]
    totals = {"samples": len(pm["samples"]), "first_sample_offset_us": (first[0] - t0) / 1e3,
              "last_sample_offset_us": (last[1] - t0) / 1e3, "sample_us": (first[1] - first[0]) / 1e3,
              "clock_offset_ms": (t0 - pm["t0_ns"]) / 1e6}
    for k, v in whole.items():
        totals[k] = v
    dur_s = m["Z"] * 1e-6
    if "dram__bytes_read.sum" in whole:
        totals["dram_GBps"] = (whole["dram__bytes_read.sum"] + whole["dram__bytes_write.sum"]) / dur_s / 1e9
    if "nvltx__bytes.sum" in whole:
        totals["nvltx_GBps"] = whole["nvltx__bytes.sum"] / dur_s / 1e9
        totals["nvlrx_GBps"] = whole["nvlrx__bytes.sum"] / dur_s / 1e9
    return {"totals": totals, "ops": ops}
