"""Given the same profile table, the same picks (north star): profile tables
recorded on 4xB200 by bench.py (the grouped GPU ProfileFn replaying the full
GPT-2 1.3B DP iteration, tests/golden/gpu_table_n4_*.json) are replayed
through tune() — the product's, and the reference build's when
/root/reference is present — via a table-backed ProfileFn. Both must
reproduce the picks the live GPU search made, bit for bit."""
import glob
import json
import os
import subprocess

import pytest

from tests.conftest import ROOT

TABLES = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "gpu_table_*.json")))


@pytest.fixture(scope="module")
def product_tool():
    subprocess.run(["make", "-C", ROOT, "build/table_tune"], check=True, capture_output=True)
    return os.path.join(ROOT, "build", "table_tune")


@pytest.mark.parametrize("path", TABLES, ids=[os.path.basename(p) for p in TABLES])
def test_recorded_gpu_table_reproduces_live_picks(product_tool, path):
    want = json.load(open(path))["expected"]
    got = json.loads(subprocess.run([product_tool, path], check=True, capture_output=True, text=True).stdout)
    assert got["table_misses"] == 0
    assert got["configs"] == want["configs"]
    assert got["profile_calls"] == want["profile_calls"]
    assert got["boundary_condition"] == want["boundary_condition"]


@pytest.mark.parametrize("path", TABLES, ids=[os.path.basename(p) for p in TABLES])
def test_python_binding_table_replay(path):
    from paper_2602_20656_b200 import _lagom_py as L
    doc = json.load(open(path))
    r = json.loads(L.tune_table(json.dumps(doc["workload"]), json.dumps(doc["initial"]),
                                json.dumps(doc["table"]), doc["budget"]))
    assert r["configs"] == doc["expected"]["configs"]


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj"), reason="/root/reference not present")
@pytest.mark.parametrize("path", TABLES, ids=[os.path.basename(p) for p in TABLES])
def test_reference_tuner_makes_identical_picks(product_tool, path):
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True, capture_output=True)
    ref = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "table_tune_ref"), path], check=True,
                         capture_output=True, text=True).stdout
    mine = subprocess.run([product_tool, path], check=True, capture_output=True, text=True).stdout
    assert ref == mine
