"""Shared parity-case generator for the collective kernels (virtual and real
multi-GPU tests). Every case is seeded, so each rank can rebuild every other
rank's input and compute the oracle output locally."""
import itertools

import numpy as np

from paper_2602_20656_b200 import coll as C

# (collective, algorithm) pairs of the kernel family
FAMILY = [(C.ALL_REDUCE, C.RING), (C.ALL_REDUCE, C.TREE), (C.ALL_GATHER, C.RING),
          (C.REDUCE_SCATTER, C.RING), (C.ALL_TO_ALL, C.RING)]
# TREE keys of the other collectives: in-switch (NVLS) AllGather/ReduceScatter
# and the one-hop AllToAll when the buffers live in an NVLS region; elsewhere
# they run the ring schedule.
TREE_EXTRA = [(C.ALL_GATHER, C.TREE), (C.REDUCE_SCATTER, C.TREE), (C.ALL_TO_ALL, C.TREE)]
PROTOS = [C.SIMPLE, C.LL, C.LL128]
NAMES = {0: "AR", 1: "AG", 2: "RS", 3: "A2A"}
DT_NAMES = {0: "f32", 1: "bf16", 2: "f16", 3: "i32"}

# (NC, NT, C): includes the tuner's minimum config (1, 64, 32 KiB) and configs
# whose chunk is smaller than the data so the slot ring wraps many times.
CONFIGS = [(1, 64, 1024), (2, 128, 4096), (3, 192, 32768), (5, 320, 8192),
           (8, 512, 65536), (16, 640, 1 << 20)]
COUNTS = [1, 7, 100, 1000, 4099, 65536 + 3, 300000]


def cases(nranks_list, seed=0, per_combo=2, tree_extra=False):
    rng = np.random.default_rng(seed)
    out = []
    for (coll, algo), proto in itertools.product(FAMILY + (TREE_EXTRA if tree_extra else []), PROTOS):
        for n in nranks_list:
            for dtype in (0, 1, 3) + ((2,) if coll == C.ALL_REDUCE else ()):
                for _ in range(per_combo):
                    nc, nt, ch = CONFIGS[rng.integers(len(CONFIGS))]
                    if n * nc > 128:  # virtual mode: all CTAs must be co-resident
                        nc = max(1, 128 // n)
                    count = int(COUNTS[rng.integers(len(COUNTS))])
                    op = int(rng.integers(3)) if coll in (C.ALL_REDUCE, C.REDUCE_SCATTER) else 0
                    out.append(dict(coll=coll, algo=algo, proto=proto, n=n, dtype=dtype, op=op,
                                    nc=int(nc), nt=int(nt), chunk=int(ch), count=count,
                                    seed=int(rng.integers(1 << 30))))
    return out


def case_id(c):
    return (f"{NAMES[c['coll']]}{'-tree' if c['algo'] else ''}-p{c['proto']}-n{c['n']}-"
            f"{DT_NAMES[c['dtype']]}-op{c['op']}-nc{c['nc']}-nt{c['nt']}-c{c['chunk']}-{c['count']}")


def inputs(c):
    from tests.oracle_ref import in_elems, random_input
    n = c["n"]
    return [random_input(c["dtype"], in_elems(c["coll"], n, c["count"]),
                         np.random.default_rng(c["seed"] + 7919 * r)) for r in range(n)]
