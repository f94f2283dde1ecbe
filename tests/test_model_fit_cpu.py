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


ROWS = [(n, w) for n in (4, 2) for w in ("gpt2-1.3b-dp", "llama3-8b-tp-sp", "llama3-70b-fsdp", "mixtral-8x7b-ep")]
# Stated bound: |predicted Z - measured Z| <= 5 % of measured.
# Rows the round-1 model misses are pinned at their real errors, not skipped.
OUT_OF_BOUND = {(4, "llama3-70b-fsdp"), (4, "mixtral-8x7b-ep"), (2, "llama3-70b-fsdp"), (2, "mixtral-8x7b-ep")}


@pytest.fixture(scope="module")
def fit_cache(tmp_path_factory):
    return str(tmp_path_factory.mktemp("fit") / "fit.json")


@pytest.mark.parametrize("n,workload", ROWS, ids=[f"n{n}-{w}" for n, w in ROWS])
def test_predicted_overlap_time_all_rows(tmp_path, fit_cache, n, workload):
    """Every (config, N) row of DESIGN.md §6 re-derived from the committed
    profile and bench files: the prediction is reproduced bit for bit, the
    relative Z error equals the committed one, and it is inside the stated
    5 % bound exactly for the rows DESIGN.md says are inside."""
    bench = os.path.join(ROOT, "profiles", f"round1_final_n{n}_{workload}.json")
    out = tmp_path / "pvm.json"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "predict_vs_measured.py"), "--profile", PROFILE,
                    "--bench", bench, "--out", str(out), "--fit-cache", fit_cache], cwd=ROOT, check=True,
                   capture_output=True, timeout=600)
    got = json.load(open(out))
    committed = json.load(open(os.path.join(ROOT, "profiles", f"round1_predict_vs_measured_n{n}_{workload}.json")))
    assert got["predicted"]["Z"] == pytest.approx(committed["predicted"]["Z"], rel=1e-12)
    assert got["rel_err"]["Z"] == pytest.approx(committed["rel_err"]["Z"], rel=1e-9)
    assert (abs(got["rel_err"]["Z"]) <= 0.05) == ((n, workload) not in OUT_OF_BOUND)


# Round 2's counter-backed models: (tag, N, model file, counter profiles, bench lines). "session3":
# fitted to the counters and bench lines taken with the round-2 kernels before the barrier rework;
# "final": the same fit over the counters and bench lines (session B) of the final kernels before the
# L2 prefetch of the local-read kernels.
ROUND2 = []
for _tag, _model, _counters, _bench in (
        ("session3", "round2_model_session3_n{n}.json", "round2_counters_session3_n{n}_*.json",
         "round2_session3_n{n}_*.json"),
        ("final", "round2_model_n{n}.json", "round2_counters_n{n}_*.json", "round2_final_sessB_n{n}_*.json"),
        # the same with the two-rank one-hop schedules in their own subspace (counter_fit --one-hop-min-nc)
        ("final-onehop", "round2_model_onehop_n{n}.json", "round2_counters_n{n}_*.json",
         "round2_final_sessB_n{n}_*.json")):
    for _n in (4, 2):
        if os.path.exists(os.path.join(ROOT, "profiles", _model.format(n=_n))):
            ROUND2.append((_tag, _n, _model.format(n=_n), _counters.format(n=_n), _bench.format(n=_n)))


@pytest.mark.parametrize("tag,n,model,counters,bench", ROUND2, ids=[f"{r[0]}-n{r[1]}" for r in ROUND2])
def test_counter_model_rows_reproduce(tmp_path, tag, n, model, counters, bench):
    """Round 2's counter-backed model (tools/counter_fit.py) re-derived from
    the committed CUPTI counter profiles and bench lines with the committed
    global parameters: every config set's and every bench row's predicted Z
    is reproduced, so the errors DESIGN.md §7 states are the real ones —
    inside and outside the 5 % bound alike."""
    out = tmp_path / "model.json"
    committed_path = os.path.join(ROOT, "profiles", model)
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "counter_fit.py"), "--n", str(n),
                    "--profiles", os.path.join(ROOT, "profiles", counters),
                    "--bench", os.path.join(ROOT, "profiles", bench),
                    "--globals", committed_path, "--out", str(out)], cwd=ROOT, check=True, capture_output=True,
                   timeout=900)
    got, committed = json.load(open(out)), json.load(open(committed_path))
    assert len(got["sets"]) == len(committed["sets"]) and len(got["bench_rows"]) == len(committed["bench_rows"])
    for a, b in zip(got["sets"] + got["bench_rows"], committed["sets"] + committed["bench_rows"]):
        assert a["Z_pred"] == pytest.approx(b["Z_pred"], rel=1e-9)
        assert a["Z_err"] == pytest.approx(b["Z_err"], rel=1e-9, abs=1e-12)
