"""Pins the CPU collective oracle (oracle/coll_oracle.c).

The reference has no data-path collective, so the oracle's parity with the
reference is UNPINNED; what is checked here is that it
implements the standard collective semantics and the documented reduction
order, against an independent numpy restatement:
  * AllGather / AllToAll: exact data movement;
  * int32 sums: exact (order-free, wrap-around);
  * fp32 / bf16 / fp16: bit-exact against numpy evaluating the same ring or
    tree order one rounding per hop (torch for bf16 rounding), and within
    a stated tolerance of the fp64 sum (fp32: 1e-5 x sum|x|; bf16: 2^-7 x n x
    sum|x|) — the tolerance the north star asks to state;
  * edge cases: count 0, count 1, ragged counts, n = 1..8.
"""
import numpy as np
import pytest
import torch

from tests import oracle_ref as O

AR, AG, RS, A2A = 0, 1, 2, 3


def to_f32(x, dtype):
    if dtype == 0:
        return x.astype(np.float32)
    t = torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16 if dtype == 1 else torch.float16)
    return t.float().numpy()


def from_f32(v, dtype):
    if dtype == 0:
        return np.float32(v)
    t = torch.tensor([v], dtype=torch.float32).to(torch.bfloat16 if dtype == 1 else torch.float16)
    return t.view(torch.int16).numpy().view(np.uint16)[0]


def ring_ref(sends, dtype, k_of_elem, n, offs):
    """acc = x_{k+1}; acc = x_{k+h} + acc for h = 2..n (one rounding per hop)."""
    out = np.empty(len(k_of_elem), dtype=sends[0].dtype)
    f = [to_f32(s, dtype) for s in sends] if dtype != 3 else sends
    for i, k in enumerate(k_of_elem):
        if dtype == 3:
            acc = np.int64(sends[(k + 1) % n][offs + i])
            for h in range(2, n + 1):
                acc = acc + np.int64(sends[(k + h) % n][offs + i])
            out[i] = np.int64(acc).astype(np.int32) if -2**31 <= acc < 2**31 else np.int32(((acc + 2**31) % 2**32) - 2**31)
            continue
        acc = from_f32(f[(k + 1) % n][offs + i], dtype)
        for h in range(2, n + 1):
            a = to_f32(np.array([acc]), dtype)[0] if dtype else acc
            acc = from_f32(np.float32(f[(k + h) % n][offs + i]) + np.float32(a), dtype)
        out[i] = acc
    return out


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("count", [0, 1, 7, 33])
def test_allgather_alltoall_exact(n, count):
    rng = np.random.default_rng(n * 100 + count)
    sends = [O.random_input(0, count, rng) for _ in range(n)]
    outs = O.collective(AG, 0, 0, 0, sends)
    for r in range(n):
        assert np.array_equal(outs[r], np.concatenate(sends))
    sends = [O.random_input(3, n * count, rng) for _ in range(n)]
    outs = O.collective(A2A, 0, 3, 0, sends)
    for r in range(n):
        want = np.concatenate([sends[q][r * count:(r + 1) * count] for q in range(n)])
        assert np.array_equal(outs[r], want)


@pytest.mark.parametrize("n", [1, 2, 4, 7])
@pytest.mark.parametrize("dtype", [0, 1, 2, 3])
def test_reducescatter_ring_order(n, dtype):
    rng = np.random.default_rng(7 * n + dtype)
    count = 29
    sends = [O.random_input(dtype, n * count, rng) for _ in range(n)]
    outs = O.collective(RS, 0, dtype, 0, sends)
    for r in range(n):
        want = ring_ref(sends, dtype, [r] * count, n, r * count)
        assert outs[r].tobytes() == want.tobytes()


@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("dtype", [0, 1, 3])
def test_allreduce_ring_blocks_and_tolerance(n, dtype):
    rng = np.random.default_rng(11 * n + dtype)
    count = 101  # ragged: ring blocks of whole 16-byte packs
    sends = [O.random_input(dtype, count, rng) for _ in range(n)]
    outs = O.collective(AR, 0, dtype, 0, sends)
    blk = O.lib().lagom_oracle_ring_block(count, n, dtype)
    pack = 16 // (2 if dtype in (1, 2) else 4)
    assert blk % pack == 0 and blk * n >= count
    want = ring_ref(sends, dtype, [i // blk for i in range(count)], n, 0)
    for r in range(n):
        assert outs[r].tobytes() == want.tobytes()
    if dtype != 3:
        exact = np.sum([to_f32(s, dtype).astype(np.float64) for s in sends], axis=0)
        mag = np.sum([np.abs(to_f32(s, dtype).astype(np.float64)) for s in sends], axis=0)
        tol = 1e-5 * mag if dtype == 0 else (2.0 ** -7) * n * mag
        assert np.all(np.abs(to_f32(outs[0], dtype) - exact) <= tol + 1e-30)


def test_int32_sum_wraps_exactly():
    n = 4
    sends = [np.full(5, 2**30, dtype=np.int32) for _ in range(n)]
    out = O.collective(AR, 0, 3, 0, sends)[0]
    assert np.all(out == np.int32(0))  # 4 * 2^30 wraps to 0


def test_tree_allreduce_order():
    n, count = 6, 17
    rng = np.random.default_rng(3)
    sends = [O.random_input(0, count, rng) for _ in range(n)]
    out = O.collective(AR, 1, 0, 0, sends)[0]

    def val(v, i):
        acc = np.float32(sends[v][i])
        for c in (2 * v + 1, 2 * v + 2):
            if c < n:
                acc = np.float32(acc + val(c, i))
        return acc
    want = np.array([val(0, i) for i in range(count)], dtype=np.float32)
    assert out.tobytes() == want.tobytes()


@pytest.mark.parametrize("op", [1, 2])
def test_max_min(op):
    n, count = 3, 40
    rng = np.random.default_rng(op)
    sends = [O.random_input(0, count, rng) for _ in range(n)]
    out = O.collective(AR, 0, 0, op, sends)[0]
    want = np.max(sends, axis=0) if op == 1 else np.min(sends, axis=0)
    assert np.array_equal(out, want)
