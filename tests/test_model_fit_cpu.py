"""The contention profiler's fits and the predicted-vs-measured claim,
re-derived on the CPU from the committed 4xB200 measurements
(profiles/round1_contention_profile_n4.json, profiles/round1_final_n4_*.json):
the params the bench searches with are exactly the fit of the committed
profile, and the product simulate() reproduces the committed predictions."""
import json
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT

PROFILE = os.path.join(ROOT, "profiles", "round1_contention_profile_n4.json")


def test_refit_reproduces_the_bench_params(tmp_path):
    out = tmp_path / "refit.json"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "contention_profile.py"), "--refit", PROFILE,
                    "--out", str(out)], cwd=ROOT, check=True, capture_output=True, timeout=600)
    got = json.load(open(out))["params"]
    want = json.load(open(os.path.join(ROOT, "profiles", "fitted_params_b200_n4.json")))["params"]
    assert got.keys() == want.keys()
    for key, co in want.items():
        for k, v in co.items():
            assert got[key][k] == pytest.approx(v, rel=1e-9, abs=1e-12), (key, k)
    # the reference schema: every collective has a traffic factor, AllReduce keeps 2.0
    assert got["collective_factors"]["ALL_REDUCE"] == 2.0
    assert set(got["collective_factors"]) == {"ALL_REDUCE", "ALL_GATHER", "REDUCE_SCATTER", "ALL_TO_ALL"}


@pytest.mark.parametrize("workload", ["gpt2-1.3b-dp", "llama3-8b-tp-sp"])
def test_predicted_overlap_time_within_stated_bound(tmp_path, workload):
    bench = os.path.join(ROOT, "profiles", f"round1_final_n4_{workload}.json")
    out = tmp_path / "pvm.json"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "predict_vs_measured.py"), "--profile", PROFILE,
                    "--bench", bench, "--out", str(out)], cwd=ROOT, check=True, capture_output=True, timeout=600)
    got = json.load(open(out))
    committed = json.load(open(os.path.join(ROOT, "profiles", f"round1_predict_vs_measured_n4_{workload}.json")))
    assert got["predicted"]["Z"] == pytest.approx(committed["predicted"]["Z"], rel=1e-12)
    assert abs(got["rel_err"]["Z"]) <= 0.05  # stated bound on Z
