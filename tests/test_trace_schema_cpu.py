"""Measured step timelines (Chrome trace JSON written by bench.py --out from
the replay engine's timeline) use the reference's trace schema exactly:
trace_to_json (reference json_io.cpp:243-257) — one complete ("X") event per
op with name, cat, ph, ts, dur, pid, tid (1 compute / 2 comm) and, for
compute events, args.blocks. The schema is taken from a trace the product
simulate() emits (bit-identical to the reference's) and every committed
measured trace is checked against it, plus the stream invariants a replay
guarantees (compute events back to back in DAG order, comm events in issue
order, names = the DAG's op ids)."""
import glob
import json
import os

import pytest

from tests.conftest import ROOT

TRACES = sorted(glob.glob(os.path.join(ROOT, "profiles", "traces", "*.json")))


@pytest.fixture(scope="module")
def reference_schema():
    from paper_2602_20656_b200 import _lagom_py as L
    w = L.gen("allreduce-pair")
    cfgs = L.seed_configs(w, "min", "")
    tr = json.loads(L.simulate(w, cfgs, ""))["trace"]
    comp = next(e for e in tr if e["cat"] == "compute")
    comm = next(e for e in tr if e["cat"] == "comm")
    return {"compute": set(comp), "comm": set(comm), "args": set(comp["args"]),
            "tid": {"compute": comp["tid"], "comm": comm["tid"]}, "pid": comp["pid"], "ph": comp["ph"]}


def _dag_ids(name):
    from paper_2602_20656_b200 import dags
    n = int(name.split("_")[-3][1:]) if name.startswith("round") else int(name.split("_")[0][1:])
    w = next(k for k in dags.BUILDERS if k in name)
    dag = dags.BUILDERS[w](n)
    return [c["id"] for c in dag["compute_ops"]], [c["id"] for c in dag["comm_ops"]]


def test_traces_committed():
    assert len(TRACES) >= 8


@pytest.mark.parametrize("path", TRACES, ids=[os.path.basename(p) for p in TRACES])
def test_measured_trace_matches_reference_schema(reference_schema, path):
    ev = json.load(open(path))
    assert isinstance(ev, list) and ev
    s = reference_schema
    for e in ev:
        assert e["cat"] in ("compute", "comm")
        assert set(e) == s[e["cat"]], (e, s[e["cat"]])
        assert e["ph"] == s["ph"] and e["pid"] == s["pid"] and e["tid"] == s["tid"][e["cat"]]
        assert isinstance(e["name"], str)
        assert isinstance(e["ts"], (int, float)) and isinstance(e["dur"], (int, float))
        assert e["ts"] >= 0 and e["dur"] >= 0
        if e["cat"] == "compute":
            assert set(e["args"]) == s["args"] and isinstance(e["args"]["blocks"], int) and e["args"]["blocks"] > 0
    comp = [e for e in ev if e["cat"] == "compute"]
    comm = [e for e in ev if e["cat"] == "comm"]
    cids, kids = _dag_ids(os.path.basename(path))
    assert [e["name"] for e in comp] == cids
    if comm:
        assert [e["name"] for e in comm] == kids
    # one stream each: compute ops start in order, one after the other
    for a, b in zip(comp, comp[1:]):
        assert b["ts"] >= a["ts"] + a["dur"] * 0.999 - 1.0
    for a, b in zip(comm, comm[1:]):
        assert b["ts"] >= a["ts"] - 1.0
