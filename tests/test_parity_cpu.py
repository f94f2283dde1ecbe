"""Bit-identical parity of the product tuner library with the reference.

Three layers of evidence:
  1. the product parity driver's output matches the committed golden digests
     generated from the reference build (runs anywhere, incl. the GPU box);
  2. when /root/reference is present: the driver compiled against the
     reference (oracle/_ref) and against the product print identical bytes;
  3. when /root/reference is present: the reference's own unit suites and its
     acceptance suite compile unmodified against the product headers/library
     and pass (tests/cpp/Makefile, doctest shim).
"""
import hashlib
import json
import os
import subprocess

import pytest

from tests.conftest import ROOT

GOLDEN = os.path.join(ROOT, "tests", "golden", "parity_ref.digests")
DRIVER = os.path.join(ROOT, "build", "parity_driver")
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "parity_driver_ref")
REF_TESTS = "/root/reference/proj/tests"


@pytest.fixture(scope="module")
def product_lines():
    subprocess.run(["make", "-C", ROOT, "build/parity_driver"], check=True, capture_output=True)
    out = subprocess.run([DRIVER], check=True, capture_output=True, text=True).stdout
    return out.splitlines()


def _case(line):
    return line[len('{"case":"'):].split('"', 1)[0]


def test_product_matches_golden_digests(product_lines):
    want = {}
    with open(GOLDEN) as f:
        for ln in f:
            case, digest = ln.rsplit(" ", 1)
            want[case] = digest.strip()
    got = {_case(l): hashlib.sha256(l.encode()).hexdigest() for l in product_lines}
    assert len(got) == len(product_lines), "case names must be unique"
    assert set(got) == set(want)
    bad = [c for c in want if got[c] != want[c]]
    assert not bad, f"{len(bad)} cases differ from the reference, e.g. {bad[:5]}"


def test_golden_covers_every_boundary_condition(product_lines):
    seen = set()
    for l in product_lines:
        if _case(l).startswith("tune/"):
            d = json.loads(l)
            if "boundary" in d:
                seen.add(d["boundary"])
    assert seen == {0, 1, 2, 3}


def test_key_cases_match_survey_appendix_a():
    """allreduce-pair, start=min: 13 calls, boundary 2,
    X = 178322.42; nccl-default: 21 calls."""
    from paper_2602_20656_b200 import _lagom_py as L
    w = L.gen("allreduce-pair")
    r = json.loads(L.tune_sim(w, "min", 500, ""))
    assert r["profile_calls"] == 13 and r["boundary_condition"] == 2
    assert r["final"]["X"] == pytest.approx(178322.42, rel=1e-12)
    assert [c["num_channels"] for c in r["configs"]] == [17, 32]
    r = json.loads(L.tune_sim(w, "nccl-default", 500, ""))
    assert r["profile_calls"] == 21 and r["boundary_condition"] == 2


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="/root/reference not present")
def test_product_bytes_equal_reference_build(product_lines):
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True, capture_output=True)
    ref = subprocess.run([REF_DRIVER], check=True, capture_output=True, text=True).stdout.splitlines()
    assert len(ref) == len(product_lines)
    diff = [(_case(a)) for a, b in zip(ref, product_lines) if a != b]
    assert not diff, f"differs from the reference on {diff[:5]}"


SUITES = ["test_model", "test_commperf", "test_contention", "test_simulator", "test_tuner",
          "test_oracle", "test_workloads", "test_cli"]


@pytest.fixture(scope="module")
def conformance_build():
    if not os.path.isdir(REF_TESTS):
        pytest.skip("/root/reference not present")
    subprocess.run(["make", "-C", ROOT, "host", "cli"], check=True, capture_output=True)
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp"), "-j8"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return os.path.join(ROOT, "build", "conformance")


@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_passes_against_product(conformance_build, suite):
    # test_cli drives our `lagom` binary (reference tests/CMakeLists.txt:20-25 sets LAGOM_BIN)
    env = dict(os.environ, LAGOM_DATA=os.path.join(ROOT, "data"), LAGOM_BIN=os.path.join(ROOT, "build", "lagom"))
    r = subprocess.run([os.path.join(conformance_build, suite)], capture_output=True, text=True, env=env,
                       timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_reference_acceptance_suite_passes_against_product(conformance_build):
    env = dict(os.environ, LAGOM_DATA=os.path.join(ROOT, "data"))
    r = subprocess.run([os.path.join(conformance_build, "acceptance_main")], capture_output=True, text=True,
                       env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 8
