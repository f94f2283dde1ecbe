// Single-rank collectives (nranks == 1): every collective of
// include/lagom_coll.h degenerates to a copy of count elements from send to
// recv (AllReduce / ReduceScatter of one rank's data, AllGather / AllToAll
// of one block). In place it is a no-op (no launch), as in NCCL.
//
// The copy is HBM-bound (read S + write S). It is built to share an SM with
// the training step's GEMM CTAs instead of taking SMs from them: sm_100
// cuBLASLt bf16 GEMM CTAs use 256 threads x 168 registers and ~214 KB of
// shared memory (ncu launch statistics, profiles/round2_coresidence.md), so
// each SM keeps ~22.5 K registers and ~19 KB of shared memory free. This
// kernel uses no shared memory and is compiled per thread-count class with
// __launch_bounds__(MAXT, 3), i.e. <= 65536/3 = 21.8 K registers per CTA at
// NT = MAXT: its CTAs are dispatched next to running GEMM CTAs (measured:
// 25 MiB copies run at the same rate with and without the GEMM loop,
// tools/coresident_probe.cu) and the tuner's NC costs the GEMMs no SMs.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "comm_internal.h"
#include "device.cuh"

namespace {

using lagom_dev::globaltimer;

struct LocalParams {
  const char* src;
  char* dst;
  int64_t bytes;
  unsigned long long* span;
};

// U 16-byte loads in flight per thread before the stores: ~32 KB per CTA in
// every class (the per-SM copy rate is set by the bytes in flight).
template <int MAXT, int U, bool PF>
__global__ void __launch_bounds__(MAXT, 3) local_copy_kernel(const __grid_constant__ LocalParams P) {
  const char* __restrict__ src = P.src;
  char* __restrict__ dst = P.dst;
  const int64_t bytes = P.bytes;
  unsigned long long* span = P.span;
  if (threadIdx.x == 0 && span) atomicMin(span, static_cast<unsigned long long>(globaltimer()));
  const int64_t nt = blockDim.x, stride = nt * gridDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * nt + threadIdx.x;
  // head bytes up to dst's 16 B boundary; the body is vectorised when src
  // shares dst's alignment, element-wise otherwise
  const int64_t head = lagom_dev::lmin(bytes, static_cast<int64_t>((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15));
  const bool vec = ((reinterpret_cast<uintptr_t>(src) ^ reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (tid < head) dst[tid] = src[tid];
  const int64_t body = vec ? (bytes - head) / 16 : 0;
  // pointer-stepped so the unrolled body carries no 64-bit index math (keeps
  // the register-capped classes free of spills)
  const uint4* s = reinterpret_cast<const uint4*>(src + head) + tid;
  uint4* d = reinterpret_cast<uint4*>(dst + head) + tid;
  int64_t left = body - tid;  // units from this thread's position to the end
  // The CTA's next batch is U chunks of nt units, `stride` apart: threads
  // 0..U-1 each ask the TMA unit to prefetch one into L2 (no registers, no
  // shared memory), so the batch's loads wait on L2 instead of HBM.
  const int64_t chunk_bytes = nt * 16;
  const int64_t cta_left = left + threadIdx.x;  // units from the CTA's first position to the end
  const uint4* cta_src = s - threadIdx.x;
  for (; left > (U - 1) * stride; left -= U * stride) {
    if (PF && gridDim.x == 1) {
      // one CTA: the next batch is one contiguous run of U chunks, one prefetch
      if (threadIdx.x == 0 && left > U * stride)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s + U * stride),
                     "r"(static_cast<uint32_t>(lagom_dev::lmin(U * stride, left - U * stride) * 16))
                     : "memory");
    } else if (PF && threadIdx.x < U) {
      const int64_t at = (U + static_cast<int64_t>(threadIdx.x)) * stride;  // chunk of the next batch
      const int64_t done = (body - tid) - left;                             // units this CTA passed
      if (cta_left - done - at >= nt)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(cta_src + done + at),
                     "r"(static_cast<uint32_t>(chunk_bytes))
                     : "memory");
    }
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u, s += stride) v[u] = __ldcs(s);
#pragma unroll
    for (int u = 0; u < U; ++u, d += stride) __stcs(d, v[u]);
  }
  for (; left > 0; left -= stride, s += stride, d += stride) __stcs(d, __ldcs(s));  // < U units left
  // tail (and the whole range when src and dst are not co-aligned)
  for (int64_t b = head + body * 16 + tid; b < bytes; b += stride) dst[b] = src[b];
  if (span) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(span + 1, static_cast<unsigned long long>(globaltimer()));
  }
}

// the thread-count class that holds NT (NT is a multiple of 64 in [64, 640])
template <bool PF>
const void* pick_pf(int nt) {
  if (nt <= 64) return reinterpret_cast<const void*>(&local_copy_kernel<64, 32, PF>);
  if (nt <= 128) return reinterpret_cast<const void*>(&local_copy_kernel<128, 16, PF>);
  if (nt <= 256) return reinterpret_cast<const void*>(&local_copy_kernel<256, 7, PF>);
  if (nt <= 384) return reinterpret_cast<const void*>(&local_copy_kernel<384, 4, PF>);
  if (nt <= 512) return reinterpret_cast<const void*>(&local_copy_kernel<512, 3, PF>);
  return reinterpret_cast<const void*>(&local_copy_kernel<640, 2, PF>);
}
// L2 prefetch of the next batch: on unless LAGOM_COPY_PREFETCH=0 (single
// rank only, so a per-process choice needs no agreement)
const void* pick(int nt) {
  static const bool pf = [] {
    const char* e = std::getenv("LAGOM_COPY_PREFETCH");
    return !(e && e[0] == '0');
  }();
  return pf ? pick_pf<true>(nt) : pick_pf<false>(nt);
}

}  // namespace

int lagom_local_select(const lagom_comm* c, const lagom_coll_args_t* a, const void* send, void* recv,
                       LaunchPlan* plan) {
  (void)c;
  const int64_t bytes = a->count * (a->dtype == LAGOM_BF16 || a->dtype == LAGOM_F16 ? 2 : 4);
  if (send == recv || bytes == 0) {  // in place: nothing to move, no launch
    plan->kernel = nullptr;
    return LAGOM_OK;
  }
  LocalParams p{static_cast<const char*>(send), static_cast<char*>(recv), bytes,
                static_cast<unsigned long long*>(a->span_out)};
  static_assert(sizeof p <= sizeof plan->params, "launch plan too small");
  std::memcpy(plan->params, &p, sizeof p);
  plan->kernel = pick(a->num_threads);
  plan->smem = 0;
  return LAGOM_OK;
}
