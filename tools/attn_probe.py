"""One replay engine over a one-op DAG with a fused attention (cuDNN SDPA)
victim: builds, replays compute-only, prints y. Debugging aid."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2602_20656_b200 import _lagom_py as L
    torch.cuda.set_device(0)
    bwd = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    dag = {"name": "attn", "compute_ops": [{"id": "a0", "gemms": [[1024, 1024, 1024]],
                                            "attention": [[2, 16, 1024, 128, 1, bwd]]}],
           "comm_ops": [{"id": "c0", "collective": "ALL_REDUCE", "dtype": 1, "count": 1 << 20,
                         "ready_after": "a0"}]}
    print("creating engine", flush=True)
    eng = L.ReplayEngine(json.dumps(dag), f"attn_{os.getpid()}", 0, 1, 0, nccl=False)
    print("created", flush=True)
    m = json.loads(eng.run_compute_only())
    print("y", m["y"], flush=True)
    eng.stop()
    eng.close()


if __name__ == "__main__":
    main()
