"""Small collective workload for compute-sanitizer (memcheck / racecheck):
every algorithm x protocol x data path on 2 virtual ranks plus the n = 1
paths, checked against the CPU oracle. Generous watchdog (sanitized kernels
run orders of magnitude slower)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_20656_b200 import coll as C  # noqa: E402
from tests.oracle_ref import collective, in_elems, out_elems, random_input  # noqa: E402


def main():
    bad = 0
    rng = np.random.default_rng(0)
    for n in (1, 2):
        for use_tma in (1, 2, 0):
            vc = C.VirtualCommunicator(n, 0, max_channels=4, max_chunk_bytes=64 << 10, timeout_ms=600000,
                                       use_tma=use_tma)
            for coll, algo in [(0, 0), (0, 1), (1, 0), (2, 0), (3, 0)]:
                for proto in (0, 1, 2):
                    if use_tma != 1 and proto != 0:
                        continue
                    count = 3000 + 5
                    sends = [random_input(1, in_elems(coll, n, count), rng) for _ in range(n)]
                    want = collective(coll, algo, 1, 0, sends)
                    dev = [torch.from_numpy(s).cuda() for s in sends]
                    outs = [torch.empty(out_elems(coll, n, count), dtype=dev[0].dtype, device="cuda") for _ in range(n)]
                    vc.launch(coll, C.CollConfig(algo, proto, 2, 128, 4096), C.BF16, count,
                              [t.data_ptr() for t in dev], [t.data_ptr() for t in outs],
                              torch.cuda.current_stream().cuda_stream)
                    torch.cuda.synchronize()
                    vc.check()
                    for r in range(n):
                        if outs[r].cpu().numpy().tobytes() != want[r].tobytes():
                            bad += 1
                            print("MISMATCH", n, use_tma, coll, algo, proto, r, flush=True)
            vc.close()
    print(f"sanitize_colls: mismatches={bad}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
