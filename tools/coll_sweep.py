"""Collective bandwidth sweep: lagom sm_100a kernels vs NCCL (torch.distributed),
one process per GPU. Run under torchrun:

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      tools/coll_sweep.py --sizes 1M,64M,512M --out gpurun_out/sweep.jsonl

Each row: collective, protocol, NC, NT, C, bytes, time (max over ranks, CUDA
events, median of reps), algbw and busbw (nccl-tests accounting).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_20656_b200 import coll as C  # noqa: E402


def parse_size(s):
    s = s.strip().upper()
    mul = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}.get(s[-1], 1)
    return int(float(s[:-1] if s[-1] in "KMG" else s) * mul)


def time_it(fn, reps, warm, stream, batch=1):
    """Median over reps of one timed group of `batch` back-to-back launches,
    per launch (batch > 1 hides the launch latency and the barrier's rank
    skew, leaving the kernels' own back-to-back rate)."""
    for _ in range(warm):
        fn()
    times = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(batch):
            fn()
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b) / 1e3 / batch)
    times.sort()
    t = torch.tensor([times[len(times) // 2]], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1M,16M,128M,1G")
    ap.add_argument("--colls", default="AR,AG,RS,A2A")
    ap.add_argument("--configs", default="8:512:2M:0,16:512:1M:0,32:640:1M:0,32:640:4M:0,8:512:64K:1,8:512:64K:2,16:640:512K:2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warm", type=int, default=2)
    ap.add_argument("--nccl", type=int, default=1)
    ap.add_argument("--batch", type=int, default=1, help="launches per timed group (per-launch time reported)")
    ap.add_argument("--one-hop", type=int, default=0, help="lagom_comm_opts_t.one_hop (TREE AG/RS over peer mappings)")
    ap.add_argument("--lagom", type=int, default=1, help="0: NCCL rows only (e.g. under NCCL_ALGO=NVLS)")
    ap.add_argument("--out", default="")
    ap.add_argument("--nvls", type=int, default=0, help="buffers in an NVLS region (TREE runs in-switch)")
    ap.add_argument("--use-tma", type=int, default=1, help="SIMPLE data path: 0 LSU, 1 TMA copies, 2 TMA also reduces")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = C.Communicator.from_process_group(device=local, max_channels=64, use_tma=args.use_tma,
                                             one_hop=args.one_hop)
    stream = torch.cuda.current_stream()
    s_ptr = stream.cuda_stream
    sizes = [parse_size(s) for s in args.sizes.split(",")]
    if args.nvls:
        # the region is a bump allocator: carve the largest send/recv once and reuse views
        big = max(sizes) * world + 4096
        comm.enable_nvls(2 * big + (64 << 20))
        xbig, ybig = comm.nvls_tensor(big, torch.uint8), comm.nvls_tensor(big, torch.uint8)
    names = {"AR": C.ALL_REDUCE, "AG": C.ALL_GATHER, "RS": C.REDUCE_SCATTER, "A2A": C.ALL_TO_ALL}
    rows = []
    for size in sizes:
        for cn in args.colls.split(","):
            coll = names[cn]
            # size = algorithmic bytes S (nccl-tests): AR buffer; AG/RS/A2A total
            count = size // 2 if coll == C.ALL_REDUCE else size // 2 // world
            n_in = count if coll in (C.ALL_REDUCE, C.ALL_GATHER) else count * world
            n_out = count if coll in (C.ALL_REDUCE, C.REDUCE_SCATTER) else count * world
            x = torch.randn(n_in, device="cuda", dtype=torch.bfloat16)
            y = torch.empty(n_out, device="cuda", dtype=torch.bfloat16)
            if args.nvls:
                xn = xbig[:2 * n_in].view(torch.bfloat16)
                y = ybig[:2 * n_out].view(torch.bfloat16)
                xn.copy_(x)
                x = xn
            s_bytes, fac = C.coll_bytes(coll, C.BF16, count, world)
            # Data check of every config: movement collectives exactly against
            # NCCL; sums against an fp32 NCCL reference within the stated bf16
            # tolerance 2^-7 * n * sum|x| (orders differ, so bits may too).
            if coll in (C.ALL_GATHER, C.ALL_TO_ALL):
                y_ref = torch.empty_like(y)
                (dist.all_gather_into_tensor if coll == C.ALL_GATHER else dist.all_to_all_single)(y_ref, x)
                mag = None
            else:
                xf, xa = x.float(), x.float().abs()
                if coll == C.ALL_REDUCE:
                    y_ref, mag = xf.clone(), xa.clone()
                    dist.all_reduce(y_ref)
                    dist.all_reduce(mag)
                else:
                    y_ref = torch.empty(n_out, device="cuda")
                    mag = torch.empty(n_out, device="cuda")
                    dist.reduce_scatter_tensor(y_ref, xf)
                    dist.reduce_scatter_tensor(mag, xa)
            for spec in (args.configs.split(",") if args.lagom else []):
                f = spec.split(":")
                nc, nt, ch, proto = f[:4]
                algo = int(f[4]) if len(f) > 4 else C.RING
                cfg = C.CollConfig(algo, int(proto), int(nc), int(nt), parse_size(ch))
                fn = lambda: comm.launch(coll, cfg, C.BF16, count, x.data_ptr(), y.data_ptr(), s_ptr)
                t = time_it(fn, args.reps, args.warm, stream, args.batch)
                comm.check()
                if mag is None:
                    ok = bool(torch.equal(y, y_ref))
                else:
                    ok = bool(((y.float() - y_ref).abs() <= (2.0 ** -7) * world * mag + 1e-6).all())
                rows.append(dict(impl="lagom", ok=ok, one_hop=args.one_hop, coll=cn, algo=int(algo), proto=int(proto), nc=int(nc), nt=int(nt),
                                 use_tma=args.use_tma, nvls=args.nvls, batch=args.batch,
                                 chunk=parse_size(ch), bytes=s_bytes, t_s=t, algbw=s_bytes / t / 1e9,
                                 busbw=s_bytes / t * fac / 1e9))
                if rank == 0:
                    print(json.dumps(rows[-1]), flush=True)
            if args.nccl:
                if coll == C.ALL_REDUCE:
                    fn = lambda: dist.all_reduce(y)
                elif coll == C.ALL_GATHER:
                    fn = lambda: dist.all_gather_into_tensor(y, x)
                elif coll == C.REDUCE_SCATTER:
                    fn = lambda: dist.reduce_scatter_tensor(y, x)
                else:
                    fn = lambda: dist.all_to_all_single(y, x)
                t = time_it(fn, args.reps, args.warm, stream, args.batch)
                rows.append(dict(impl="nccl", algo_env=os.environ.get("NCCL_ALGO", ""), batch=args.batch, coll=cn,
                                 bytes=s_bytes, t_s=t, algbw=s_bytes / t / 1e9,
                                 busbw=s_bytes / t * fac / 1e9))
                if rank == 0:
                    print(json.dumps(rows[-1]), flush=True)
    if rank == 0 and args.out:
        with open(args.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
