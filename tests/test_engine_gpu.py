"""The replay engine on one GPU: a two-layer GPT-2 backward DAG with its
bucket AllReduces (n = 1), tuned through the C++ tune() with the GPU
ProfileFn, then replayed in every mode. Checks the measurement contract
(x per comm op, y per compute op, X = sum x, Y = sum y, Z >= max parts) and
that a recorded profile table replays to the same picks."""
import json
import os

import pytest

from tests.conftest import cuda_available

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    if not cuda_available():
        pytest.skip("no CUDA device")
    from paper_2602_20656_b200 import _lagom_py as L
    from paper_2602_20656_b200 import dags
    dag = dags.gpt2_dp(1, layers=2)
    eng = L.ReplayEngine(json.dumps(dag), f"lagom_test_{os.getpid()}", 0, 1, 0, repeats=1, warmup=0,
                         nccl=True, e2e_in_bytes=1 << 20, e2e_out_bytes=4096, sm_partition=1)
    yield eng, dag
    eng.stop()
    eng.close()


def test_tune_and_replay_modes(engine):
    from paper_2602_20656_b200 import _lagom_py as L
    eng, dag = engine
    groups = [int(c["role"]) for c in dag["comm_ops"]]
    t = json.loads(eng.tune("", "min", 12, "", groups))
    assert 1 <= t["profile_calls"] <= 12
    assert len(t["configs"]) == max(groups) + 1
    cfgs = json.dumps({"configs": [t["configs"][g] for g in groups]})
    for fn in (lambda: eng.run(cfgs), lambda: eng.run_e2e(cfgs), eng.run_nccl, eng.run_compute_only,
               lambda: eng.run_comm_only(cfgs)):
        m = json.loads(fn())
        assert len(m["x"]) == len(dag["comm_ops"]) and len(m["y"]) == len(dag["compute_ops"])
        assert m["X"] == pytest.approx(sum(m["x"]), rel=1e-9)
        assert m["Y"] == pytest.approx(sum(m["y"]), rel=1e-9)
        assert m["Z"] > 0
    # the recorded table replays to the same picks through tune()
    r = json.loads(L.tune_table(json.dumps(t["workload"]), json.dumps(t["initial"]),
                                json.dumps(t["profile_table"]), 12))
    assert r["configs"] == t["configs"]


def test_cli_tune_with_gpu_profiler(engine, tmp_path):
    """`lagom tune --profiler gpu` (the reference CLI surface with the replay
    engine as profiler) on one GPU."""
    import subprocess
    from tests.conftest import ROOT
    eng, dag = engine
    w = tmp_path / "w.json"
    d = tmp_path / "d.json"
    w.write_text(eng.workload(""))
    d.write_text(json.dumps(dag))
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", LAGOM_JOB=f"clitest{os.getpid()}")
    r = subprocess.run([os.path.join(ROOT, "build", "lagom"), "tune", "--workload", str(w), "--dag", str(d),
                        "--profiler", "gpu", "--budget", "4", "--start", "nccl-default"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode in (0, 4), r.stderr[-2000:]
    rep = json.loads(r.stdout)
    assert rep["command"] == "tune" and 1 <= rep["profile_calls"] <= 4
    assert len(rep["configs"]) == len(dag["comm_ops"])


def test_gpu_batched_exhaustive_matches_cpu_oracle():
    """exhaustive() with one GPU thread per joint grid point
    returns the CPU oracle's bits (makespan, evaluations, argmin configs)."""
    if not cuda_available():
        pytest.skip("no CUDA device")
    from paper_2602_20656_b200 import _lagom_py as L
    cases = [L.gen("allreduce-pair"), L.gen("fsdp", layers=1, seed=5), L.gen("tp", layers=2, seed=3)]
    cases += [L.gen("random", seed=s, m=1 + s % 4, n=1 + s % 3) for s in range(20)]
    for s in (3, 7):  # delta > 0 exercises the stretch integration
        w = json.loads(L.gen("random", seed=100 + s, m=3, n=2))
        w["gpu"]["compute_on_comm_slowdown"] = 0.2 * s
        cases.append(json.dumps(w))
    for w in cases:
        cpu = json.loads(L.oracle(w, "", 10 ** 7))
        gpu = json.loads(L.oracle_gpu(w, "", 10 ** 7, 0))
        assert gpu["evaluations"] == cpu["evaluations"]
        assert gpu["Z"] == cpu["Z"]  # bit-identical doubles
        assert gpu["configs"] == cpu["configs"]


def test_cli_sweep_and_compare_on_hardware(tmp_path, root):
    """`lagom sweep|compare --profiler gpu --dag`: the reference CLI's
    one-parameter sweep and its method comparison with every value / grid
    point a measured replay; the CSVs keep the reference schemas
    (sweep: value,x_comm,Y,Z — reference sweep.cpp:53-61; compare:
    method,Z,evaluations — reference lagom_main.cpp:333-360)."""
    import subprocess
    if not cuda_available():
        pytest.skip("no CUDA device")
    from paper_2602_20656_b200 import _lagom_py as L
    from paper_2602_20656_b200 import dags
    dag = dags.gpt2_dp(1, layers=1)
    eng = L.ReplayEngine(json.dumps(dag), f"lagom_cli_wl_{os.getpid()}", 0, 1, 0, nccl=False)
    work = eng.workload("")
    eng.stop()
    eng.close()
    (tmp_path / "w.json").write_text(work)
    (tmp_path / "d.json").write_text(json.dumps(dag))
    cli = os.path.join(root, "build", "lagom")
    env = dict(os.environ, LAGOM_JOB=f"clitest{os.getpid()}")
    comm = dag["comm_ops"][0]["id"]
    r = subprocess.run([cli, "sweep", "--workload", str(tmp_path / "w.json"), "--dag", str(tmp_path / "d.json"),
                        "--profiler", "gpu", "--comm", comm, "--param", "nc", "--values", "1,4,16"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "value,x_comm,Y,Z" and [ln.split(",")[0] for ln in lines[1:]] == ["1", "4", "16"]
    for ln in lines[1:]:
        v, x, y, z = (float(t) for t in ln.split(","))
        assert x > 0 and y > 0 and z >= max(y, x) * 0.999
    r = subprocess.run([cli, "compare", "--workload", str(tmp_path / "w.json"), "--dag", str(tmp_path / "d.json"),
                        "--profiler", "gpu", "--grid", "nc=1,8;nt=128;c=1M", "--budget", "8"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode in (0, 4), r.stderr
    rows = r.stdout.strip().splitlines()
    assert rows[0] == "method,Z,evaluations"
    methods = {ln.split(",")[0]: float(ln.split(",")[1]) for ln in rows[1:]}
    assert set(methods) == {"exhaustive", "tune", "naive"} and all(z > 0 for z in methods.values())
    n_ops = len(dag["comm_ops"])
    assert int(rows[1].split(",")[2]) == 2 ** n_ops  # every joint grid point replayed
