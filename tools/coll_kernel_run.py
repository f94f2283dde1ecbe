"""Launches one collective configuration repeatedly on ONE GPU — the target
for `ncu --set full` captures (never wrap a multi-rank command in ncu).

  python tools/coll_kernel_run.py --coll AR --ranks 1 --count 13107200 \
      --nc 8 --nt 512 --chunk 2M --proto 0 --iters 20

--ranks 1 uses a real single-rank communicator (the n=1 path of the bench);
--ranks >1 emulates the ranks on this GPU (virtual mode, cooperative launch)
so the staging/flag protocol shows up in the profile. Prints the CUDA-event
time per launch and the implied bandwidth.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2602_20656_b200 import coll as C  # noqa: E402


def size(s):
    s = s.upper()
    mul = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}.get(s[-1], 1)
    return int(float(s[:-1] if s[-1] in "KMG" else s) * mul)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--coll", default="AR", choices=["AR", "AG", "RS", "A2A"])
    ap.add_argument("--algo", type=int, default=0)
    ap.add_argument("--proto", type=int, default=0)
    ap.add_argument("--ranks", type=int, default=1)
    ap.add_argument("--count", type=int, default=13107200)
    ap.add_argument("--nc", type=int, default=8)
    ap.add_argument("--nt", type=int, default=512)
    ap.add_argument("--chunk", default="2M")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    coll = {"AR": C.ALL_REDUCE, "AG": C.ALL_GATHER, "RS": C.REDUCE_SCATTER, "A2A": C.ALL_TO_ALL}[a.coll]
    n = a.ranks
    nin = a.count if coll in (C.ALL_REDUCE, C.ALL_GATHER) else a.count * n
    nout = a.count if coll in (C.ALL_REDUCE, C.REDUCE_SCATTER) else a.count * n
    cfg = C.CollConfig(a.algo, a.proto, a.nc, a.nt, size(a.chunk))
    stream = torch.cuda.current_stream()
    xs = [torch.randn(nin, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
    ys = [torch.empty(nout, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
    if n == 1:
        comm = C.Communicator(0, 1, torch.cuda.current_device(), max_channels=64)
        launch = lambda: comm.launch(coll, cfg, C.BF16, a.count, xs[0].data_ptr(), ys[0].data_ptr(),  # noqa: E731
                                     stream.cuda_stream)
    else:
        comm = C.VirtualCommunicator(n, torch.cuda.current_device(), max_channels=64)
        launch = lambda: comm.launch(coll, cfg, C.BF16, a.count, [x.data_ptr() for x in xs],  # noqa: E731
                                     [y.data_ptr() for y in ys], stream.cuda_stream)
    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(stream)
    for _ in range(a.iters):
        launch()
    ev[1].record(stream)
    torch.cuda.synchronize()
    comm.check()
    t = ev[0].elapsed_time(ev[1]) / a.iters * 1e-3
    moved = (nin + nout) * 2 * n  # bytes read + written by all ranks' kernels (local view)
    print(f"{a.coll} ranks={n} count={a.count} NC={a.nc} NT={a.nt} C={a.chunk} proto={a.proto}: "
          f"{t * 1e6:.1f} us/launch, {moved / t / 1e9:.1f} GB/s read+write", flush=True)
    comm.close()


if __name__ == "__main__":
    main()
