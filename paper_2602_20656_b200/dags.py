"""Replay DAGs for BASELINE.json's configs 2-5.

Each DAG is the reference Workload's overlap shape (ordered compute stream,
serialized comm stream, ``ready_after`` gates — reference model.hpp:78-96 and
the generator shapes of reference workloads.cpp:59-109) with real kernels
attached: cuBLASLt bf16 GEMMs [m, n, k(, batch)] and fused cuDNN SDPA
attention [batch, heads, seq, head_dim, causal, backward] per compute op, and one
collective per comm op (bf16, counts per include/lagom_coll.h). Shapes follow
the public model cards; data is synthetic (random-init on device).

Every comm op carries a ``role`` (its position in the layer: the k-th
gradient bucket, the attention/MLP AG or RS, dispatch/combine): bench.py
tunes one config per role against the full iteration (the reference tuner
over grouped comm ops, lagom::b200::make_grouped_gpu_profiler).
"""
from __future__ import annotations

import json

BF16 = 1
MiB = 1 << 20


def _sdpa(batch, heads, seq, d, backward, causal=True):
    """A fused attention (cuDNN SDPA, flash-style) entry of a compute op:
    [batch, heads, seq, head_dim, causal, backward]."""
    return [batch, heads, seq, d, int(causal), int(backward)]


def gpt2_dp(nranks: int, layers: int = 24):
    """Config 2 — GPT-2 1.3B, DP: layer backward + bucketed (25 MiB, DDP
    default) gradient AllReduce gated on the layer's backward."""
    h, T, s, d, heads, mb = 2048, 8192, 1024, 128, 16, 8
    layer_params = 12 * h * h + 13 * h
    layer_bytes = 2 * layer_params
    bucket = 25 * MiB
    gemms = [[T, 4 * h, h], [h, 4 * h, T],       # fc2 dgrad / wgrad
             [T, h, 4 * h], [4 * h, h, T],       # fc1
             [T, h, h], [h, h, T]]               # attention out-proj
    gemms += [[T, h, 3 * h], [3 * h, h, T]]      # qkv
    attention = [_sdpa(mb, heads, s, d, backward=True)]  # attention core backward (fused)
    compute, comm = [], []
    for l in range(layers):
        compute.append({"id": f"bwd{l}", "gemms": gemms, "attention": attention})
        left, b = layer_bytes, 0
        while left > 0:
            nbytes = min(bucket, left)
            comm.append({"id": f"ar{l}_{b}", "collective": "ALL_REDUCE", "dtype": BF16,
                         "count": nbytes // 2, "ready_after": f"bwd{l}", "role": b})
            left -= nbytes
            b += 1
    return {"name": f"gpt2-1.3b-dp{nranks}", "parallelism": f"dp{nranks}", "compute_ops": compute,
            "comm_ops": comm}


def llama8b_tp_sp(nranks: int, layers: int = 32):
    """Config 3 — Llama-3 8B, TP=n with sequence parallelism (forward):
    per layer AG(seq-sharded activations) -> attention block -> RS, then
    AG -> MLP -> RS, overlapped Domino-style (comms gated on the producing
    compute, overlapping the next compute)."""
    n = nranks
    h, T, ffn, hd = 4096, 8192, 14336, 128
    q_heads, kv_heads = 32, 8
    shard = T // n
    compute, comm = [], []
    for l in range(layers):
        qkv = (q_heads + 2 * kv_heads) * hd // n
        attn = [[T, qkv, h], [T, h, q_heads * hd // n]]
        mlp = [[T, 2 * ffn // n, h], [T, h, ffn // n]]
        # this rank's q heads, causal, full sequence (K/V expanded to the q heads)
        compute.append({"id": f"attn{l}", "gemms": attn,
                        "attention": [_sdpa(1, max(1, q_heads // n), T, hd, backward=False)]})
        compute.append({"id": f"mlp{l}", "gemms": mlp})
        comm.append({"id": f"rs_attn{l}", "collective": "REDUCE_SCATTER", "dtype": BF16,
                     "count": shard * h, "ready_after": f"attn{l}", "role": 0})
        comm.append({"id": f"ag_mlp{l}", "collective": "ALL_GATHER", "dtype": BF16,
                     "count": shard * h, "ready_after": f"attn{l}", "role": 1})
        comm.append({"id": f"rs_mlp{l}", "collective": "REDUCE_SCATTER", "dtype": BF16,
                     "count": shard * h, "ready_after": f"mlp{l}", "role": 2})
        comm.append({"id": f"ag_attn{l + 1}", "collective": "ALL_GATHER", "dtype": BF16,
                     "count": shard * h, "ready_after": f"mlp{l}", "role": 3})
    return {"name": f"llama3-8b-tp{n}-sp", "parallelism": f"tp{n}-sp", "compute_ops": compute, "comm_ops": comm}


def llama70b_fsdp(nranks: int, layers: int = 4):
    """Config 4 — Llama-3 70B-shaped layers, FSDP/ZeRO-3 (fwd): per layer a
    parameter AllGather (prefetched after the previous layer), the layer's
    GEMMs, and the gradient ReduceScatter gated on it (reference gen_fsdp
    shape, workloads.cpp:59-76)."""
    n = nranks
    h, T, ffn, hd = 8192, 4096, 28672, 128
    q_heads, kv_heads = 64, 8
    layer_params = h * (q_heads + 2 * kv_heads) * hd + q_heads * hd * h + 3 * h * ffn
    shard = layer_params // n
    compute, comm = [], []
    for l in range(layers):
        g = [[T, (q_heads + 2 * kv_heads) * hd, h], [T, h, q_heads * hd], [T, 2 * ffn, h], [T, h, ffn]]
        ag = {"id": f"ag{l}", "collective": "ALL_GATHER", "dtype": BF16, "count": shard, "role": 0}
        if l > 0:
            ag["ready_after"] = f"layer{l - 1}"
        comm.append(ag)
        compute.append({"id": f"layer{l}", "gemms": g, "attention": [_sdpa(1, q_heads, T, hd, backward=False)]})
        comm.append({"id": f"rs{l}", "collective": "REDUCE_SCATTER", "dtype": BF16, "count": shard,
                     "ready_after": f"layer{l}", "role": 1})
    return {"name": f"llama3-70b-layers-fsdp{n}", "parallelism": f"fsdp{n}", "compute_ops": compute,
            "comm_ops": comm}


def mixtral_ep(nranks: int, layers: int = 32):
    """Config 5 — Mixtral 8x7B, EP=n (dual micro-batch): per layer dispatch
    AllToAll, expert GEMMs, combine AllToAll (reference gen_ep_dualbatch
    shape, workloads.cpp:92-109). 4096 tokens x top-2 = 8192 slots/rank."""
    n = nranks
    h, ffn, slots = 4096, 14336, 8192
    experts_per_rank = max(1, 8 // n)
    compute, comm = [], []
    per_peer = slots * h // n
    for l in range(layers):
        g = [[slots // experts_per_rank, 2 * ffn, h], [slots // experts_per_rank, h, ffn]] * experts_per_rank
        disp = {"id": f"a2a_in{l}", "collective": "ALL_TO_ALL", "dtype": BF16, "count": per_peer, "role": 0}
        if l > 0:
            disp["ready_after"] = f"ex{l - 1}"
        comm.append(disp)
        compute.append({"id": f"ex{l}", "gemms": g})
        comm.append({"id": f"a2a_out{l}", "collective": "ALL_TO_ALL", "dtype": BF16, "count": per_peer,
                     "ready_after": f"ex{l}", "role": 1})
    return {"name": f"mixtral-8x7b-ep{n}", "parallelism": f"ep{n}", "compute_ops": compute, "comm_ops": comm}


def with_nc_max(dag: dict, nc_max: int) -> dict:
    """Per-op resource bounds (reference CommBounds, model.hpp:70-76): the
    reference default nc_max = 32 was sized for its modeled 64-SM device; on
    a 148-SM B200 the search may use up to 64 channels."""
    for c in dag["comm_ops"]:
        c.setdefault("bounds", {})["nc_max"] = nc_max
    return dag


BUILDERS = {"gpt2-1.3b-dp": gpt2_dp, "llama3-8b-tp-sp": llama8b_tp_sp,
            "llama3-70b-fsdp": llama70b_fsdp, "mixtral-8x7b-ep": mixtral_ep}


def attention_flops(a) -> float:
    """Forward 4*b*h*s^2*d (QK^T and PV), backward 2.5x; causal halves it
    (replay.cpp attention_flops)."""
    b, h, s, d = a[0], a[1], a[2], a[3]
    causal = a[4] if len(a) > 4 else 1
    bwd = a[5] if len(a) > 5 else 0
    fwd = 4.0 * b * h * s * s * d * (0.5 if causal else 1.0)
    return 2.5 * fwd if bwd else fwd


def flops(dag: dict) -> float:
    tot = 0.0
    for c in dag["compute_ops"]:
        for g in c["gemms"]:
            b = g[3] if len(g) > 3 else 1
            tot += 2.0 * g[0] * g[1] * g[2] * b
        tot += sum(attention_flops(a) for a in c.get("attention", []))
    return tot


def to_json(dag: dict) -> str:
    return json.dumps(dag)
