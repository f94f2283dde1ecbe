// lagom-b200 — deterministic fixture workloads (drop-in for reference
// proj/include/lagom/workloads.hpp:8-39). Draws use std::mt19937_64 (fully
// specified by the standard) with explicit modulo / 53-bit arithmetic, so the
// generated workloads are bit-identical to the reference's on every platform.
#pragma once

#include <cstdint>

#include "lagom/model.hpp"

namespace lagom {

// 64 SMs, 600 B/us HBM, 400 B/us link, phi = 0.6, delta = 0.
GpuSpec default_gpu();

// Per layer: AllGather (after previous layer), compute, ReduceScatter (after it).
Workload gen_fsdp(int layers, std::uint64_t seed);

// Per layer: compute, then an AllReduce gated on it.
Workload gen_tp_domino(int layers, std::uint64_t seed);

// Per layer: dispatch AlltoAll, expert compute, combine AlltoAll.
Workload gen_ep_dualbatch(int layers, std::uint64_t seed);

// Two ungated AllReduces (2 MiB "ar_a", 32 MiB "ar_b") against 7 matmuls.
Workload gen_allreduce_pair();

Workload gen_random(int num_compute, int num_comm, std::uint64_t seed);

}  // namespace lagom
