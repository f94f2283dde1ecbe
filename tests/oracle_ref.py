"""Loader for the CPU collective oracle (oracle/coll_oracle.c) — TEST
INFRASTRUCTURE. Used only as the checker; never by the product path."""
import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "_ref", "libcoll_oracle.so")

NP_DTYPE = {0: np.float32, 1: np.uint16, 2: np.uint16, 3: np.int32}  # bf16/f16 as raw bits
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "coll"], check=True,
                           capture_output=True)
        _lib = ctypes.CDLL(LIB)
        _lib.lagom_oracle_collective.restype = ctypes.c_int
        _lib.lagom_oracle_collective.argtypes = [ctypes.c_int] * 5 + [ctypes.c_longlong,
                                                                     ctypes.c_void_p, ctypes.c_void_p]
        _lib.lagom_oracle_ring_block.restype = ctypes.c_longlong
        _lib.lagom_oracle_ring_block.argtypes = [ctypes.c_longlong, ctypes.c_int, ctypes.c_int]
        _lib.lagom_oracle_threads.restype = ctypes.c_int
    return _lib


def out_elems(coll: int, n: int, count: int) -> int:
    return count if coll in (0, 2) else n * count


def in_elems(coll: int, n: int, count: int) -> int:
    return count if coll in (0, 1) else n * count


def collective(coll, algo, dtype, op, sends):
    """sends: list of numpy arrays (one per rank). Returns list of outputs."""
    n = len(sends)
    count = sends[0].size if coll in (0, 1) else sends[0].size // n
    outs = [np.zeros(out_elems(coll, n, count), dtype=sends[0].dtype) for _ in range(n)]
    sarr = (ctypes.c_void_p * n)(*[s.ctypes.data for s in sends])
    rarr = (ctypes.c_void_p * n)(*[o.ctypes.data for o in outs])
    rc = lib().lagom_oracle_collective(coll, algo, n, dtype, op, count, sarr, rarr)
    assert rc == 0
    return outs


def random_input(dtype, nelems, rng):
    if dtype == 3:
        return rng.integers(-(1 << 20), 1 << 20, size=nelems, dtype=np.int32)
    x = rng.standard_normal(nelems).astype(np.float32)
    if dtype == 0:
        return x
    import torch
    t = torch.from_numpy(x).to(torch.bfloat16 if dtype == 1 else torch.float16)
    return t.view(torch.int16).numpy().view(np.uint16).copy()
