"""Per-SM rate of the single-rank (n = 1) collective path — the local copy
every collective degenerates to on one GPU — over NC x NT x algorithm, plus
the 2-rank-emulated push path, on ONE GPU. CUDA events, median of reps.

  python tools/copy_rate_sweep.py --bytes 25M --out gpurun_out/copy_rate.jsonl
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2602_20656_b200 import coll as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", default="25M")
    ap.add_argument("--ncs", default="1,2,4,8,16,32")
    ap.add_argument("--nts", default="64,256,512,640")
    ap.add_argument("--colls", default="AR")
    ap.add_argument("--algos", default="0,1")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    s = a.bytes.upper()
    nbytes = int(float(s[:-1]) * {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}[s[-1]]) if s[-1] in "KMG" else int(s)
    count = nbytes // 2
    stream = torch.cuda.current_stream()
    comm = C.Communicator(0, 1, torch.cuda.current_device())
    x = torch.randn(count, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(count, device="cuda", dtype=torch.bfloat16)
    codes = {"AR": C.ALL_REDUCE, "AG": C.ALL_GATHER, "RS": C.REDUCE_SCATTER, "A2A": C.ALL_TO_ALL}
    out = open(a.out, "a") if a.out else None
    for coll in a.colls.split(","):
        for algo in [int(v) for v in a.algos.split(",")]:
            if algo == 1 and coll != "AR":
                continue
            for nc in [int(v) for v in a.ncs.split(",")]:
                for nt in [int(v) for v in a.nts.split(",")]:
                    cfg = C.CollConfig(algo, C.SIMPLE, nc, nt, 2 << 20)
                    launch = lambda: comm.launch(codes[coll], cfg, C.BF16, count, x.data_ptr(),  # noqa: E731
                                                 y.data_ptr(), stream.cuda_stream)
                    for _ in range(3):
                        launch()
                    ts = []
                    for _ in range(a.reps):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        launch()
                        e1.record(stream)
                        e1.synchronize()
                        ts.append(e0.elapsed_time(e1) * 1e-3)
                    comm.check()
                    assert torch.equal(x, y), (coll, algo, nc, nt)
                    t = statistics.median(ts)
                    row = {"coll": coll, "algo": algo, "nc": nc, "nt": nt, "bytes": nbytes, "us": t * 1e6,
                           "copy_gbs": nbytes / t / 1e9, "per_sm_gbs": nbytes / t / 1e9 / nc}
                    print(json.dumps(row), flush=True)
                    if out:
                        out.write(json.dumps(row) + "\n")
    comm.close()


if __name__ == "__main__":
    main()
