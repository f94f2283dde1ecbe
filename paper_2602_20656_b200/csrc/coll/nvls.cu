// NVLS: collectives reduced / broadcast inside the NVSwitch (NVLink SHARP).
//
// On an NVSwitch box every rank reaches every other through the switch, so
// the reference's TREE algorithm (Algorithm::Tree, model.hpp:37) is realized
// with the switch as the tree's root: a multicast object spans one region of
// every rank's HBM, `multimem.ld_reduce` returns the element-wise sum of all
// ranks' copies (accumulated in fp32 for bf16/f16, in the switch), and
// `multimem.st` writes one value into every rank's copy. Per GPU this moves
// S bytes over NVLink for an AllReduce instead of the ring's 2(n-1)/n S
// through the SMs, so far fewer channels (SMs) reach a given bandwidth —
// which is exactly what the Lagom search trades against compute.
//
// Set-up is collective and transport-agnostic like the IPC heap: rank 0
// creates the multicast object and exports a POSIX fd, peers duplicate it
// with pidfd_getfd (blob = {pid, fd, size}), every rank adds its device, and
// after a caller barrier every rank binds physical memory and maps both the
// unicast and the multicast views. Buffers allocated from the region
// (lagom_comm_nvls_alloc) have identical offsets on every rank.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "comm_internal.h"
#include "device.cuh"

namespace {

// Driver entry points are resolved at run time (cudaGetDriverEntryPoint), so
// liblagom_coll.so loads on machines without a driver (CPU tests, build box).
void* driver_sym(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return fn;
}
// decltype() names the prototype without referencing the symbol.
#define DRV(fn) (reinterpret_cast<decltype(&fn)>(driver_sym(#fn)))


constexpr uint64_t kBlobMagic = 0x4c41474f4d4e564cull;  // "LAGOMNVL"
constexpr uint64_t kPeerMagic = 0x4c41474f4d504552ull;  // "LAGOMPER"
struct Blob {
  uint64_t magic;
  int64_t pid;
  int64_t fd;
  int64_t size;
};

int drv_fail(CUresult r, const char* what) {
  const char* s = nullptr;
  DRV(cuGetErrorString)(r, &s);
  return lagom_fail(LAGOM_ERR_CUDA, std::string(what) + ": " + (s ? s : "?"));
}
#define LAGOM_DRV(call)                                  \
  do {                                                   \
    CUresult r_ = (call);                                \
    if (r_ != CUDA_SUCCESS) return drv_fail(r_, #call);  \
  } while (0)

size_t granularity(int nranks) {
  CUmulticastObjectProp prop{};
  prop.numDevices = static_cast<unsigned>(nranks);
  prop.size = 2u << 20;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  if (DRV(cuMulticastGetGranularity)(&g, &prop, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS || g == 0)
    g = 2u << 20;
  return g;
}

// --------------------------------------------------------------- kernels ---
using lagom_dev::globaltimer;
using lagom_dev::ld_acquire_sys;

struct NvlsParams {
  char* heap[LAGOM_MAX_RANKS];
  int rank, nranks;
  int64_t count;        // elements, lagom_coll.h semantics
  int elem_bytes;
  const char* send_uc;  // local views
  char* recv_uc;
  char* send_mc;        // multicast views (send/recv inside the NVLS region)
  char* recv_mc;
  int64_t off_nvbar, off_nvep;
  int64_t off_nvpiece, off_nvpbase;        // push RS: piece flags [ch][src], piece count [ch]
  int64_t piece_units;                     // push RS: 16 B units per pipelined piece (chunk C)
  unsigned int* abort_flag;
  uint64_t timeout_ns;
  unsigned long long* span;
  char* peer_recv[LAGOM_MAX_RANKS];        // one-hop A2A / AG: recv in every rank's region;
                                           // push RS: every rank's scratch slot for me
  const char* peer_send[LAGOM_MAX_RANKS];  // one-hop RS (pull): send in every rank's region
  char* scratch;                           // push RS: my scratch (slot q holds rank q's partial)
  int64_t scratch_slot;                    // bytes per scratch slot
  uint64_t* phase;                         // diagnostics: [ch][parity][LAGOM_PHASE_STAMPS] or null
};

// Thread 0 records stamp k of this channel's launch (lagom_comm_phase_stamps);
// epochs advance by 2 per launch, so (ep >> 1) & 1 alternates.
__device__ __forceinline__ void phase_stamp(const NvlsParams& P, int ch, uint64_t ep, int k) {
  if (P.phase) P.phase[(static_cast<int64_t>(ch) * 2 + ((ep >> 1) & 1)) * LAGOM_PHASE_STAMPS + k] = globaltimer();
}

// Polls *p (relaxed) until it reaches v; the caller then reads it once with
// ld.acquire (acquire pattern). false on abort or timeout.
__device__ bool nv_wait(const uint64_t* p, uint64_t v, const NvlsParams& P) {
  uint64_t t0 = 0;
  unsigned it = 0;
  while (lagom_dev::ld_relaxed_sys(p) < v) {
    if ((++it & 255u) == 0) {
      if (*reinterpret_cast<volatile unsigned*>(P.abort_flag)) return false;
      const uint64_t now = globaltimer();
      if (!t0) t0 = now;
      if (now - t0 > P.timeout_ns) {
        atomicExch(P.abort_flag, 1u);
        return false;
      }
    }
  }
  return true;
}

// All ranks' CTA `ch` meet. Every thread of the CTA calls it. Threads
// 0..n-2 work in parallel: thread t posts `ep` into peer p = r+1+t's flag
// [ch][me] (relaxed) and polls its own flag [ch][p] (relaxed), then reads it
// once more with ld.acquire (the peer's writes before its post). With
// `release` (exit barriers), thread 0 first runs ONE system fence for the
// CTA after a __syncthreads, which releases every thread's earlier writes
// (multimem / peer stores) before any post. System fences are the expensive
// part and contend across SMs (tools/flag_latency.cu on 4xB200, per barrier:
// a fence per post as in st.release 5.5 us at 64 CTAs, relaxed posts 1.6 us,
// one fence per CTA 4.4-5.6 us at 8-64 CTAs; profiles/round2_nvls_phases.md).
__device__ bool nv_barrier(const NvlsParams& P, int ch, uint64_t ep, int* s_ok, bool release) {
  const int n = P.nranks, r = P.rank, t = threadIdx.x;
  __syncthreads();
  if (t == 0) {
    *s_ok = 1;
    if (release) lagom_dev::fence_acq_rel_sys();
  }
  __syncthreads();
  if (t < n - 1) {
    const int p = (r + 1 + t) % n;
    const uint64_t* mine = reinterpret_cast<const uint64_t*>(P.heap[r] + P.off_nvbar + (static_cast<int64_t>(ch) * n + p) * 128);
    lagom_dev::st_relaxed_sys(reinterpret_cast<uint64_t*>(P.heap[p] + P.off_nvbar + (static_cast<int64_t>(ch) * n + r) * 128), ep);
    if (!nv_wait(mine, ep, P)) *s_ok = 0;
    else (void)ld_acquire_sys(mine);
  }
  __syncthreads();
  return *s_ok != 0;
}

template <typename T> struct Mm;
template <> struct Mm<float> {
  __device__ static uint4 ld_reduce(const void* p) {
    uint4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
  }
};
template <> struct Mm<__nv_bfloat16> {
  __device__ static uint4 ld_reduce(const void* p) {
    uint4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
  }
};
template <> struct Mm<__half> {
  __device__ static uint4 ld_reduce(const void* p) {
    uint4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
  }
};
template <> struct Mm<int32_t> {
  __device__ static uint4 ld_reduce(const void* p) {
    const uint32_t* q = static_cast<const uint32_t*>(p);
    uint4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.x) : "l"(q) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.y) : "l"(q + 1) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.z) : "l"(q + 2) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.w) : "l"(q + 3) : "memory");
    return v;
  }
};
__device__ __forceinline__ void mm_store(void* p, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// MINB = 3 (co-resident variants): <= 65536 / (3 x MAXT) registers per
// thread, i.e. <= 21.8 K registers per CTA at NT = MAXT, which fits next to
// an sm_100 cuBLASLt GEMM CTA (256 x 168 registers, ~214 KB shared memory)
// on one SM. MINB = 1: the deep-unroll variants of round 1.
template <int KIND, typename T, int U, int MAXT, int MINB = 1>
__global__ void __launch_bounds__(MAXT, MINB) nvls_kernel(const __grid_constant__ NvlsParams P) {
  __shared__ int s_ok;
  const int ch = blockIdx.x, nch = gridDim.x, n = P.nranks, r = P.rank;
  if (threadIdx.x == 0 && P.span) atomicMin(P.span, static_cast<unsigned long long>(globaltimer()));
  uint64_t* ep_home = reinterpret_cast<uint64_t*>(P.heap[r] + P.off_nvep + static_cast<int64_t>(ch) * 8);
  const uint64_t ep = *reinterpret_cast<volatile uint64_t*>(ep_home) + 1;
  if (threadIdx.x == 0) phase_stamp(P, ch, ep, 0);
  if (!nv_barrier(P, ch, ep, &s_ok, false)) return;  // every rank's inputs are ready
  if (threadIdx.x == 0) phase_stamp(P, ch, ep, 1);

  // 16 B units: AR/RS reduce the whole buffer / own block through the switch,
  // AG broadcasts the own block, A2A (KIND 3) writes block p straight into
  // rank p's recv. Channel c owns a contiguous slice; in AR each rank further
  // takes 1/n of it (its stores reach every rank).
  const int64_t E = P.elem_bytes;
  const int64_t B = P.count;  // elements per block (AR: the whole buffer)
  const int64_t units = B * E / 16;
  const int64_t per_ch = (units + nch - 1) / nch;
  int64_t lo = lagom_dev::lmin(units, per_ch * ch), hi = lagom_dev::lmin(units, per_ch * (ch + 1));
  const int64_t nt = blockDim.x;
  if constexpr (KIND == 3) {
    // One hop through the switch: step k sends block r+k to rank r+k, so at
    // every step the ranks' destinations form a permutation (no receiver is
    // the target of two senders at once); k = 0 is the local block.
    for (int k = 0; k < n; ++k) {
      const int p = (r + k) % n;
      const char* in = P.send_uc + static_cast<int64_t>(p) * units * 16;
      char* out = P.peer_recv[p] + static_cast<int64_t>(r) * units * 16;
      int64_t u0 = lo + threadIdx.x;
      for (; u0 + (U - 1) * nt < hi; u0 += nt * U) {
        if (threadIdx.x == 0 && u0 + nt * U < hi)  // the CTA's next batch into L2
          lagom_dev::prefetch_l2(in + (u0 + nt * U) * 16, lagom_dev::lmin(nt * U, hi - u0 - nt * U) * 16);
        const char* src = in + u0 * 16;
        char* dst = out + u0 * 16;
        uint4 v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = *reinterpret_cast<const uint4*>(src + j * nt * 16);
#pragma unroll
        for (int j = 0; j < U; ++j) *reinterpret_cast<uint4*>(dst + j * nt * 16) = v[j];
      }
      if (u0 < hi) {  // the rest as one predicated batch
        uint4 v[U];
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (u0 + j * nt < hi) v[j] = *reinterpret_cast<const uint4*>(in + (u0 + j * nt) * 16);
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (u0 + j * nt < hi) *reinterpret_cast<uint4*>(out + (u0 + j * nt) * 16) = v[j];
      }
    }
  } else if constexpr (KIND == 4) {
    // One-hop AllGather (n = 2 default): load the own block once, store it
    // into every rank's recv (the local copy plus one NVLink write per peer).
    // A multicast store would also carry the sender's own copy through the
    // switch, which caps NVLS AllGather at (n-1)/n of the link per GPU.
    const char* in = P.send_uc;
    const int64_t at = static_cast<int64_t>(r) * units * 16;
    int64_t u0 = lo + threadIdx.x;
    for (; u0 + (U - 1) * nt < hi; u0 += nt * U) {
      if (threadIdx.x == 0 && u0 + nt * U < hi)  // the CTA's next batch into L2
        lagom_dev::prefetch_l2(in + (u0 + nt * U) * 16, lagom_dev::lmin(nt * U, hi - u0 - nt * U) * 16);
      uint4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = *reinterpret_cast<const uint4*>(in + (u0 + j * nt) * 16);
      for (int k = 1; k <= n; ++k) {
        char* out = P.peer_recv[(r + k) % n] + at;
#pragma unroll
        for (int j = 0; j < U; ++j) *reinterpret_cast<uint4*>(out + (u0 + j * nt) * 16) = v[j];
      }
    }
    if (u0 < hi) {  // the rest as one predicated batch
      uint4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (u0 + j * nt < hi) v[j] = *reinterpret_cast<const uint4*>(in + (u0 + j * nt) * 16);
      for (int k = 1; k <= n; ++k) {
        char* out = P.peer_recv[(r + k) % n] + at;
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (u0 + j * nt < hi) *reinterpret_cast<uint4*>(out + (u0 + j * nt) * 16) = v[j];
      }
    }
  } else if constexpr (KIND == 6) {
    // Push-based one-hop ReduceScatter, pipelined in pieces of C bytes (the
    // config's chunk): my partial of piece i of every other rank's block goes
    // straight into that rank's scratch slot for me (posted NVLink writes, no
    // round trip), then a flag per (channel, source) counts the pieces that
    // landed; the owner reduces piece i in the ring order — acc = x_{r+1},
    // then x_{r+2}, ..., ending with its own x_r, rounding to the element
    // type at every combine — as soon as every peer's piece i is there, so
    // the result is bit-identical to the ring schedule and its oracle. Piece
    // i+1 is pushed before piece i is reduced.
    using R = lagom_dev::Red<T, LAGOM_SUM>;
    __shared__ int s_go;
    const int64_t pu = P.piece_units > 0 ? P.piece_units : 1;
    const int64_t npieces = (hi - lo + pu - 1) / pu;
    uint64_t* pbase_home = reinterpret_cast<uint64_t*>(P.heap[r] + P.off_nvpbase + static_cast<int64_t>(ch) * 8);
    const uint64_t pbase = *reinterpret_cast<volatile uint64_t*>(pbase_home);
    const char* own = P.send_uc + static_cast<int64_t>(r) * units * 16;
    auto part = [&](int q) -> const uint4* {
      return reinterpret_cast<const uint4*>(q == r ? own : P.scratch + static_cast<int64_t>(q) * P.scratch_slot);
    };
    auto push = [&](int64_t i) {
      const int64_t a = lo + i * pu, b = lagom_dev::lmin(hi, a + pu);
      for (int k = 1; k < n; ++k) {
        const int p = (r + k) % n;
        const uint4* src = reinterpret_cast<const uint4*>(P.send_uc + static_cast<int64_t>(p) * units * 16) + a;
        uint4* dst = reinterpret_cast<uint4*>(P.peer_recv[p]) + a;
        int64_t left = b - a - threadIdx.x;
        src += threadIdx.x;
        dst += threadIdx.x;
        for (; left > (U - 1) * nt; left -= U * nt) {
          if (threadIdx.x == 0 && left > U * nt)  // the CTA's next batch into L2
            lagom_dev::prefetch_l2(src + U * nt, lagom_dev::lmin(U * nt, left - U * nt) * 16);
          uint4 v[U];
#pragma unroll
          for (int j = 0; j < U; ++j) v[j] = src[j * nt];
#pragma unroll
          for (int j = 0; j < U; ++j) dst[j * nt] = v[j];
          src += U * nt;
          dst += U * nt;
        }
        for (; left > 0; left -= nt, src += nt, dst += nt) *dst = *src;
      }
      __syncthreads();
      if (threadIdx.x == 0) lagom_dev::fence_acq_rel_sys();  // the piece's peer stores (every thread's) before its flag
      __syncthreads();
      if (threadIdx.x < n - 1) {  // post piece i to every peer, one thread per peer
        const int p = (r + 1 + threadIdx.x) % n;
        lagom_dev::st_relaxed_sys(reinterpret_cast<uint64_t*>(P.heap[p] + P.off_nvpiece + (static_cast<int64_t>(ch) * n + r) * 128),
                                  pbase + static_cast<uint64_t>(i) + 1);
      }
    };
    if (threadIdx.x == 0) s_go = 1;  // published by push(0)'s __syncthreads
    if (npieces > 0) push(0);
    for (int64_t i = 0; i < npieces; ++i) {
      if (i + 1 < npieces) push(i + 1);
      if (threadIdx.x < n - 1) {  // every peer's piece i landed in my scratch
        const int q = (r + 1 + threadIdx.x) % n;
        const uint64_t* f = reinterpret_cast<const uint64_t*>(P.heap[r] + P.off_nvpiece + (static_cast<int64_t>(ch) * n + q) * 128);
        if (!nv_wait(f, pbase + static_cast<uint64_t>(i) + 1, P)) s_go = 0;
        else (void)ld_acquire_sys(f);
      }
      __syncthreads();
      if (!s_go) return;
      const int64_t a = lo + i * pu, b = lagom_dev::lmin(hi, a + pu);
      uint4* out = reinterpret_cast<uint4*>(P.recv_uc);
      for (int64_t u = a + threadIdx.x; u < b; u += nt * U) {
        if (threadIdx.x < n && u - threadIdx.x + nt * U < b) {  // every part's next batch into L2
          const int64_t nb = u - threadIdx.x + nt * U;
          lagom_dev::prefetch_l2(part((r + 1 + threadIdx.x) % n) + nb, lagom_dev::lmin(nt * U, b - nb) * 16);
        }
        uint4 acc[U];
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (u + j * nt < b) acc[j] = part((r + 1) % n)[u + j * nt];
        for (int k = 2; k <= n; ++k) {
          const uint4* x = part((r + k) % n);
#pragma unroll
          for (int j = 0; j < U; ++j)
            if (u + j * nt < b) acc[j] = lagom_dev::red4<R>(x[u + j * nt], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (u + j * nt < b) out[u + j * nt] = acc[j];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      *reinterpret_cast<volatile uint64_t*>(pbase_home) = pbase + static_cast<uint64_t>(npieces);
      // No exit barrier: my output is mine alone, and the next launch's entry
      // barrier keeps peers from overwriting my scratch while I still read it.
      *reinterpret_cast<volatile uint64_t*>(ep_home) = ep + 1;
      if (P.span) atomicMax(P.span + 1, static_cast<unsigned long long>(globaltimer()));
    }
    return;
  } else if constexpr (KIND == 5) {
    // One-hop ReduceScatter: pull block r of every rank's send through the
    // peer mappings and combine in the ring order (x_{r+1}, then x_{r+2}, ...,
    // ending with the own x_r; every combine rounds to the element type), so
    // the result is bit-identical to the ring schedule and its oracle. No
    // switch echo: a rank's ingress is its (n-1) peers' blocks only.
    using R = lagom_dev::Red<T, LAGOM_SUM>;
    const int64_t at = static_cast<int64_t>(r) * units * 16;
    int64_t u0 = lo + threadIdx.x;
    for (; u0 + (U - 1) * nt < hi; u0 += nt * U) {
      uint4 acc[U];
      const char* s1 = P.peer_send[(r + 1) % n] + at;
#pragma unroll
      for (int j = 0; j < U; ++j) acc[j] = *reinterpret_cast<const uint4*>(s1 + (u0 + j * nt) * 16);
      for (int k = 2; k <= n; ++k) {
        const char* sp = P.peer_send[(r + k) % n] + at;
        uint4 v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = *reinterpret_cast<const uint4*>(sp + (u0 + j * nt) * 16);
#pragma unroll
        for (int j = 0; j < U; ++j) acc[j] = lagom_dev::red4<R>(v[j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) *reinterpret_cast<uint4*>(P.recv_uc + (u0 + j * nt) * 16) = acc[j];
    }
    if (u0 < hi) {  // the rest as one predicated batch (one round trip per peer)
      uint4 acc[U];
      const char* s1 = P.peer_send[(r + 1) % n] + at;
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (u0 + j * nt < hi) acc[j] = *reinterpret_cast<const uint4*>(s1 + (u0 + j * nt) * 16);
      for (int k = 2; k <= n; ++k) {
        const char* sp = P.peer_send[(r + k) % n] + at;
        uint4 v[U];
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (u0 + j * nt < hi) v[j] = *reinterpret_cast<const uint4*>(sp + (u0 + j * nt) * 16);
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (u0 + j * nt < hi) acc[j] = lagom_dev::red4<R>(v[j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (u0 + j * nt < hi) *reinterpret_cast<uint4*>(P.recv_uc + (u0 + j * nt) * 16) = acc[j];
    }
  } else {
  if (KIND == 0) {  // AR: my 1/n share of the channel slice
    const int64_t len = hi - lo, per_r = (len + n - 1) / n;
    const int64_t a = lo + lagom_dev::lmin(len, per_r * r), b = lo + lagom_dev::lmin(len, per_r * (r + 1));
    lo = a;
    hi = b;
  }
  // multimem loads are remote: U x 16 B in flight per thread
  const int64_t blk = KIND == 0 ? 0 : static_cast<int64_t>(r) * units;  // block offset in units
  // Pointers are advanced per batch so the unrolled body needs no 64-bit
  // index math or bounds checks (keeps U = 16 free of spills at 640 threads).
  const char* in = KIND == 1 ? P.send_uc : P.send_mc + blk * 16;
  char* out = KIND == 2 ? P.recv_uc : P.recv_mc + blk * 16;
  auto load = [&](const char* p) -> uint4 {
    if (KIND == 1) return *reinterpret_cast<const uint4*>(p);
    return Mm<T>::ld_reduce(p);
  };
  auto store = [&](char* p, uint4 v) {
    if (KIND == 2) *reinterpret_cast<uint4*>(p) = v;  // RS: my block, local
    else mm_store(p, v);                              // AR / AG: to every rank
  };
  int64_t u0 = lo + threadIdx.x;
  for (; u0 + (U - 1) * nt < hi; u0 += nt * U) {
    if (KIND == 1 && threadIdx.x == 0 && u0 + nt * U < hi)  // AG reads locally: next batch into L2
      lagom_dev::prefetch_l2(in + (u0 + nt * U) * 16, lagom_dev::lmin(nt * U, hi - u0 - nt * U) * 16);
    const char* src = in + u0 * 16;
    char* dst = out + u0 * 16;
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = load(src + k * nt * 16);
#pragma unroll
    for (int k = 0; k < U; ++k) store(dst + k * nt * 16, v[k]);
  }
  // The rest (< U units per thread) as one predicated batch: its loads are
  // all in flight together, so it costs one round trip through the switch
  // instead of one per unit.
  if (u0 < hi) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (u0 + k * nt < hi) v[k] = load(in + (u0 + k * nt) * 16);
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (u0 + k * nt < hi) store(out + (u0 + k * nt) * 16, v[k]);
  }
  }
  if (P.phase) {
    __syncthreads();
    if (threadIdx.x == 0) phase_stamp(P, ch, ep, 2);
  }
  // my multimem / peer stores are visible everywhere before any rank moves
  // on: nobody reads results or reuses inputs early
  const bool done = nv_barrier(P, ch, ep + 1, &s_ok, true);
  if (threadIdx.x == 0) {
    if (done) *reinterpret_cast<volatile uint64_t*>(ep_home) = ep + 1;
    phase_stamp(P, ch, ep, 3);
    phase_stamp(P, ch, ep, 4);
    if (P.phase) P.phase[(static_cast<int64_t>(ch) * 2 + ((ep >> 1) & 1)) * LAGOM_PHASE_STAMPS + 5] = ep;
  }
  if (threadIdx.x == 0 && P.span) atomicMax(P.span + 1, static_cast<unsigned long long>(globaltimer()));
}

// One-hop AllToAll through the TMA engine: thread 0 streams every (peer,
// tile) of the channel slice through a ring of kA2aStages smem stages — bulk
// load from the local send block, bulk store into the destination rank's recv
// (one NVLink write per byte). A single SM's TMA engine pushes ~50 GB/s to a
// peer against ~35 GB/s for 640 threads of vector ld/st (tools/tma_probe.cu),
// and the rate does not depend on NT.
constexpr int kA2aStages = 4;
constexpr int kA2aTile = 48 * 1024;
constexpr int kA2aSmem = kA2aStages * kA2aTile;

__global__ void __launch_bounds__(640) a2a_tma_kernel(const __grid_constant__ NvlsParams P) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ uint64_t full[kA2aStages];
  __shared__ int s_ok;
  const int ch = blockIdx.x, nch = gridDim.x, n = P.nranks, r = P.rank;
  if (threadIdx.x == 0 && P.span) atomicMin(P.span, static_cast<unsigned long long>(globaltimer()));
  uint64_t* ep_home = reinterpret_cast<uint64_t*>(P.heap[r] + P.off_nvep + static_cast<int64_t>(ch) * 8);
  const uint64_t ep = *reinterpret_cast<volatile uint64_t*>(ep_home) + 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kA2aStages; ++s) lagom_dev::mbar_init(&full[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!nv_barrier(P, ch, ep, &s_ok, false)) return;  // every rank's recv is free
  if (threadIdx.x == 0) {
    const int64_t blk = P.count * P.elem_bytes;  // bytes per block (16 B multiple)
    const int64_t units = blk / 16, per_ch = (units + nch - 1) / nch;
    const int64_t lo = lagom_dev::lmin(units, per_ch * ch) * 16, hi = lagom_dev::lmin(units, per_ch * (ch + 1)) * 16;
    const int64_t per_peer = (hi - lo + kA2aTile - 1) / kA2aTile, ntiles = per_peer * n;
    // tile i: step k = i / per_peer sends block r+k to rank r+k (a permutation
    // of destinations at every step; k = 0 is the local block)
    auto src_of = [&](int64_t i, uint32_t* len) -> const char* {
      const int p = static_cast<int>((r + i / per_peer) % n);
      const int64_t off = lo + (i % per_peer) * kA2aTile;
      *len = static_cast<uint32_t>(lagom_dev::lmin(kA2aTile, hi - off));
      return P.send_uc + p * blk + off;
    };
    auto dst_of = [&](int64_t i) -> char* {
      const int p = static_cast<int>((r + i / per_peer) % n);
      return P.peer_recv[p] + r * blk + lo + (i % per_peer) * kA2aTile;
    };
    auto issue = [&](int64_t i) {
      uint32_t len;
      const char* src = src_of(i, &len);
      const int st = static_cast<int>(i % kA2aStages);
      lagom_dev::mbar_expect(&full[st], len);
      lagom_dev::bulk_load(ring + st * kA2aTile, src, len, &full[st]);
    };
    for (int64_t i = 0; i < ntiles && i < kA2aStages; ++i) issue(i);
    for (int64_t i = 0; i < ntiles; ++i) {
      const int st = static_cast<int>(i % kA2aStages);
      lagom_dev::mbar_wait(&full[st], static_cast<uint32_t>((i / kA2aStages) & 1));
      uint32_t len;
      src_of(i, &len);
      lagom_dev::bulk_store(dst_of(i), ring + st * kA2aTile, len);
      lagom_dev::bulk_commit();
      if (i >= 1 && i - 1 + kA2aStages < ntiles) {
        lagom_dev::bulk_wait_read1();  // tile i-1's store has read its stage
        issue(i - 1 + kA2aStages);
      }
    }
    lagom_dev::bulk_wait_all();        // every bulk store performed
    lagom_dev::fence_proxy_global();   // async-proxy writes -> generic proxy
  }
  const bool done = nv_barrier(P, ch, ep + 1, &s_ok, true);  // every peer's writes into my recv landed
  if (threadIdx.x == 0) {
    if (done) *reinterpret_cast<volatile uint64_t*>(ep_home) = ep + 1;
    if (P.span) atomicMax(P.span + 1, static_cast<unsigned long long>(globaltimer()));
  }
}

// One-hop AllGather through the TMA engine (one_hop with the TMA data path):
// thread 0 loads each tile of the own block once into a ring of smem stages
// and bulk-stores it into every rank's recv (the peers' over NVLink, its own
// last), one bulk group per tile. (n-1)/n S leaves each GPU, against S for
// the switch's multicast, which also echoes the own block.
__global__ void __launch_bounds__(640) ag_tma_kernel(const __grid_constant__ NvlsParams P) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ uint64_t full[kA2aStages];
  __shared__ int s_ok;
  const int ch = blockIdx.x, nch = gridDim.x, n = P.nranks, r = P.rank;
  if (threadIdx.x == 0 && P.span) atomicMin(P.span, static_cast<unsigned long long>(globaltimer()));
  uint64_t* ep_home = reinterpret_cast<uint64_t*>(P.heap[r] + P.off_nvep + static_cast<int64_t>(ch) * 8);
  const uint64_t ep = *reinterpret_cast<volatile uint64_t*>(ep_home) + 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kA2aStages; ++s) lagom_dev::mbar_init(&full[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!nv_barrier(P, ch, ep, &s_ok, false)) return;  // every rank's recv is free
  if (threadIdx.x == 0) {
    const int64_t blk = P.count * P.elem_bytes;
    const int64_t units = blk / 16, per_ch = (units + nch - 1) / nch;
    const int64_t lo = lagom_dev::lmin(units, per_ch * ch) * 16, hi = lagom_dev::lmin(units, per_ch * (ch + 1)) * 16;
    const int64_t ntiles = (hi - lo + kA2aTile - 1) / kA2aTile;
    auto issue = [&](int64_t i) {
      const int64_t off = lo + i * kA2aTile;
      const uint32_t len = static_cast<uint32_t>(lagom_dev::lmin(kA2aTile, hi - off));
      const int st = static_cast<int>(i % kA2aStages);
      lagom_dev::mbar_expect(&full[st], len);
      lagom_dev::bulk_load(ring + st * kA2aTile, P.send_uc + off, len, &full[st]);
    };
    for (int64_t i = 0; i < ntiles && i < kA2aStages; ++i) issue(i);
    for (int64_t i = 0; i < ntiles; ++i) {
      const int st = static_cast<int>(i % kA2aStages);
      const int64_t off = lo + i * kA2aTile;
      const uint32_t len = static_cast<uint32_t>(lagom_dev::lmin(kA2aTile, hi - off));
      lagom_dev::mbar_wait(&full[st], static_cast<uint32_t>((i / kA2aStages) & 1));
      for (int k = 1; k <= n; ++k) lagom_dev::bulk_store(P.peer_recv[(r + k) % n] + r * blk + off, ring + st * kA2aTile, len);
      lagom_dev::bulk_commit();
      if (i >= 1 && i - 1 + kA2aStages < ntiles) {
        lagom_dev::bulk_wait_read1();  // tile i-1's stores have read its stage
        issue(i - 1 + kA2aStages);
      }
    }
    lagom_dev::bulk_wait_all();
    lagom_dev::fence_proxy_global();
  }
  const bool done = nv_barrier(P, ch, ep + 1, &s_ok, true);  // every peer's stores into my recv landed
  if (threadIdx.x == 0) {
    if (done) *reinterpret_cast<volatile uint64_t*>(ep_home) = ep + 1;
    if (P.span) atomicMax(P.span + 1, static_cast<unsigned long long>(globaltimer()));
  }
}

// One-hop ReduceScatter pulled through the TMA engine: thread 0 bulk-loads,
// per tile of the own block r, every rank's partial (the peers' over
// NVLink, from their send buffers in the region) into one smem stage, up to
// kA2aStages tiles ahead — up to 192 KB of remote reads in flight per SM
// without registers, where vector loads would be latency-bound. All threads
// then combine the stage in the ring order (acc = x_{r+1}, then x_{r+2}, ...,
// ending with the own x_r, rounding to the element type at every combine),
// so the result is bit-identical to the ring schedule and its oracle, and
// store it to recv. (n-1)/n S enters each GPU; nothing is pushed.
template <typename T>
__global__ void __launch_bounds__(640) rs_tma_kernel(const __grid_constant__ NvlsParams P) {
  using R = lagom_dev::Red<T, LAGOM_SUM>;
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ uint64_t full[kA2aStages];
  __shared__ int s_ok;
  const int ch = blockIdx.x, nch = gridDim.x, n = P.nranks, r = P.rank;
  if (threadIdx.x == 0 && P.span) atomicMin(P.span, static_cast<unsigned long long>(globaltimer()));
  uint64_t* ep_home = reinterpret_cast<uint64_t*>(P.heap[r] + P.off_nvep + static_cast<int64_t>(ch) * 8);
  const uint64_t ep = *reinterpret_cast<volatile uint64_t*>(ep_home) + 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kA2aStages; ++s) lagom_dev::mbar_init(&full[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!nv_barrier(P, ch, ep, &s_ok, false)) return;  // every rank's partials are ready
  const int64_t blk = P.count * P.elem_bytes;
  const int64_t units = blk / 16, per_ch = (units + nch - 1) / nch;
  const int64_t lo = lagom_dev::lmin(units, per_ch * ch) * 16, hi = lagom_dev::lmin(units, per_ch * (ch + 1)) * 16;
  const int64_t tile = (kA2aTile / n) & ~static_cast<int64_t>(127);  // per partial; n of them per stage
  const int64_t ntiles = (hi - lo + tile - 1) / tile;
  auto src = [&](int k) -> const char* {  // partial x_{r+k} of my block
    const int q = (r + k) % n;
    return (q == r ? P.send_uc : P.peer_send[q]) + r * blk;
  };
  auto issue = [&](int64_t i) {
    const int64_t off = lo + i * tile;
    const uint32_t len = static_cast<uint32_t>(lagom_dev::lmin(tile, hi - off));
    const int st = static_cast<int>(i % kA2aStages);
    lagom_dev::mbar_expect(&full[st], len * static_cast<uint32_t>(n));
    for (int k = 1; k <= n; ++k)
      lagom_dev::bulk_load(ring + st * kA2aTile + (k - 1) * tile, src(k) + off, len, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int64_t i = 0; i < ntiles && i < kA2aStages; ++i) issue(i);
  for (int64_t i = 0; i < ntiles; ++i) {
    const int st = static_cast<int>(i % kA2aStages);
    const int64_t off = lo + i * tile;
    const int64_t len = lagom_dev::lmin(tile, hi - off);
    lagom_dev::mbar_wait(&full[st], static_cast<uint32_t>((i / kA2aStages) & 1));
    const uint4* x = reinterpret_cast<const uint4*>(ring + st * kA2aTile);
    const int64_t tu = tile / 16;
    uint4* out = reinterpret_cast<uint4*>(P.recv_uc + off);
    for (int64_t u = threadIdx.x; u < len / 16; u += blockDim.x) {
      uint4 acc = x[u];
      for (int k = 2; k <= n; ++k) acc = lagom_dev::red4<R>(x[(k - 1) * tu + u], acc);
      out[u] = acc;
    }
    __syncthreads();  // the stage is consumed
    if (threadIdx.x == 0 && i + kA2aStages < ntiles) issue(i + kA2aStages);
  }
  // my loads of the peers' send buffers completed (their mbarrier fired):
  // the peers may reuse them once every rank posted; no writes to release
  const bool done = nv_barrier(P, ch, ep + 1, &s_ok, false);
  if (threadIdx.x == 0) {
    if (done) *reinterpret_cast<volatile uint64_t*>(ep_home) = ep + 1;
    if (P.span) atomicMax(P.span + 1, static_cast<unsigned long long>(globaltimer()));
  }
}

const void* pick_rs_tma(int dtype) {
  switch (dtype) {
    case LAGOM_F32: return reinterpret_cast<const void*>(&rs_tma_kernel<float>);
    case LAGOM_BF16: return reinterpret_cast<const void*>(&rs_tma_kernel<__nv_bfloat16>);
    case LAGOM_F16: return reinterpret_cast<const void*>(&rs_tma_kernel<__half>);
    case LAGOM_I32: return reinterpret_cast<const void*>(&rs_tma_kernel<int32_t>);
  }
  return nullptr;
}

// the 192 KB dynamic smem ring of a TMA kernel, enabled once per kernel
// (communicators may launch from several host threads)
bool tma_smem_ok(const void* k) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, bool>> done;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == k) return d.second;
  const bool ok = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kA2aSmem) == cudaSuccess;
  done.emplace_back(k, ok);
  return ok;
}

template <int KIND, int U, int MAXT, int MINB = 1>
const void* pick_nvls_u(int dtype) {
  // the copy kinds (AG, A2A, one-hop AG) move bytes: one instantiation
  if (KIND == 1 || KIND == 3 || KIND == 4)
    return reinterpret_cast<const void*>(&nvls_kernel<KIND, int32_t, U, MAXT, MINB>);
  switch (dtype) {
    case LAGOM_F32: return reinterpret_cast<const void*>(&nvls_kernel<KIND, float, U, MAXT, MINB>);
    case LAGOM_BF16: return reinterpret_cast<const void*>(&nvls_kernel<KIND, __nv_bfloat16, U, MAXT, MINB>);
    case LAGOM_F16: return reinterpret_cast<const void*>(&nvls_kernel<KIND, __half, U, MAXT, MINB>);
    case LAGOM_I32: return reinterpret_cast<const void*>(&nvls_kernel<KIND, int32_t, U, MAXT, MINB>);
  }
  return nullptr;
}
// Requests in flight per thread. multimem.ld_reduce is a round trip through
// the switch, so AR / RS throughput per SM is set by the bytes in flight,
// NT x U x 16 B (measured on 4xB200: AR 25 MiB at NC = 4, NT = 512 goes from
// 232 to 411 GB/s busbw with U = 16 instead of 8).
//   coresident (default), NT <= 256: the CTA fits next to a GEMM CTA on one
//     SM (<= 21.8 K registers): U = 32 / 16 / 8 at NT = 64 / 128 / 256, i.e.
//     32 KB in flight per CTA (one-hop RS and the A2A take half where the full
//     unroll would spill under the cap);
//   NT > 256, or coresident = 0: the deep unrolls of round 1 (U = 16, U = 8
//     for the copy kinds; NT <= 256 -> U = 32 with a 256-thread launch bound),
//     whose CTAs take an SM of their own (the replay's SM partition reserves
//     their NC). The tuner's NT thus also picks the regime: many light CTAs
//     riding along the GEMMs, or few heavy CTAs on dedicated SMs.
template <int KIND>
const void* pick_nvls(int dtype, int nt, bool coresident) {
  if (coresident && nt <= 256) {
    constexpr int H = (KIND == 5 || KIND == 6) ? 2 : 1, H3 = KIND == 3 ? 2 : 1;
    if (nt <= 64) return pick_nvls_u<KIND, 32 / H / H3, 64, 3>(dtype);
    if (nt <= 128) return pick_nvls_u<KIND, 16 / H, 128, 3>(dtype);
    return pick_nvls_u<KIND, 8 / H, 256, 3>(dtype);
  }
  if (KIND == 5 || KIND == 6)  // one-hop RS holds acc[U] + v[U]: half the unroll of ld_reduce
    return nt <= 256 ? pick_nvls_u<KIND, 16, 256>(dtype) : pick_nvls_u<KIND, 8, 640>(dtype);
  if (nt <= 256) return pick_nvls_u<KIND, 32, 256>(dtype);
  return (KIND == 1 || KIND == 3 || KIND == 4) ? pick_nvls_u<KIND, 8, 640>(dtype) : pick_nvls_u<KIND, 16, 640>(dtype);
}

bool inside(const lagom_comm* c, const void* p, int64_t bytes) {
  const char* q = static_cast<const char*>(p);
  return c->nvls_ready && q >= c->nvls_uc && q + bytes <= c->nvls_uc + c->nvls_bytes;
}

int ebytes(int dtype) { return (dtype == LAGOM_BF16 || dtype == LAGOM_F16) ? 2 : 4; }

}  // namespace

// Used by lagom_coll_launch: 1 if this launch runs on the switch / the peer
// mappings, with *kernel/params filled in; 0 to run the P2P kernels; -1 (with
// lagom_last_error set) if it must run there but cannot.
//
// TREE AllGather / ReduceScatter through the peer mappings (peer stores /
// peer loads) instead of the switch (opts.one_hop). At n = 2 the multicast
// echo of the own block caps NVLS AllGather and ReduceScatter at ~330 GB/s
// busbw from NC = 8 upward, while the one-hop schedules keep scaling with the
// channels (AllGather on a 4xB200 pair, 1 GiB: NC 8: 216 vs 322; NC 15: 355
// vs 278; NC 32: 569 vs 342 GB/s; profiles/round1_ag_one_hop_n2.jsonl).
// one_hop = 2: one hop at n = 2 from kOneHopMinChannels channels up, where
// the per-SM rate of the peer copies (~55 GB/s with TMA) overtakes the
// switch (n = 2, AG / RS 64 MiB, profiles/round2_onehop_scan_*_n2.jsonl:
// NC 8: 161 / 202 us one hop vs 109 / 120 us switch; NC 16: 88 / 109 vs
// 110 / 116; NC 24: 64 / 81 vs 116 / 121). Every rank has the same n and
// launches the same config, so every rank makes the same choice.
constexpr int kOneHopMinChannels = 16;
bool one_hop(const lagom_comm* c, int nc) {
  const int mode = c->opts.one_hop;
  return c->nvls_peers_ready && (mode == 1 || (mode == 2 && c->nranks == 2 && nc >= kOneHopMinChannels));
}

int lagom_nvls_prepare(const lagom_comm* c, const lagom_coll_args_t* a, const void* send, void* recv,
                       const void** kernel, void* params_out, size_t* params_bytes, int* smem_bytes) {
  *smem_bytes = 0;
  if (!c->nvls_ready || a->algorithm != LAGOM_TREE || a->redop != LAGOM_SUM || c->virt) return 0;
  const int64_t e = ebytes(a->dtype), n = c->nranks;
  const bool co = c->opts.coresident != 0, hop = one_hop(c, a->num_channels);
  // TMA data path for the one-hop kernels (one elected thread, 192 KB smem
  // ring: an SM of its own) unless the config asks for the co-resident
  // regime (NT <= 256)
  const bool tma = c->opts.a2a_tma && !(co && a->num_threads <= 256);
  const void* rs_tma = hop && tma && a->collective == LAGOM_REDUCE_SCATTER ? pick_rs_tma(a->dtype) : nullptr;
  if (rs_tma && !tma_smem_ok(rs_tma)) rs_tma = nullptr;
  const bool push_rs = hop && !rs_tma && c->nvls_scratch && a->count * ebytes(a->dtype) <= c->nvls_scratch_slot;
  int64_t in_b = 0, out_b = 0;
  const void* k = nullptr;
  switch (a->collective) {
    case LAGOM_ALL_REDUCE: in_b = out_b = a->count * e; k = pick_nvls<0>(a->dtype, a->num_threads, co); break;
    case LAGOM_ALL_GATHER:
      in_b = a->count * e;
      out_b = a->count * e * n;
      if (hop && tma && tma_smem_ok(reinterpret_cast<const void*>(&ag_tma_kernel))) {
        k = reinterpret_cast<const void*>(&ag_tma_kernel);
        *smem_bytes = kA2aSmem;
        break;
      }
      k = hop ? pick_nvls<4>(a->dtype, a->num_threads, co) : pick_nvls<1>(a->dtype, a->num_threads, co);
      break;
    case LAGOM_REDUCE_SCATTER:
      in_b = a->count * e * n;
      out_b = a->count * e;
      // one hop: TMA pull when allowed; else push (partials into the owners'
      // scratch, local reduce) when a scratch slot fits the block, else pull
      // with vector loads (latency-bound)
      if (rs_tma) {
        k = rs_tma;
        *smem_bytes = kA2aSmem;
        break;
      }
      k = !hop ? pick_nvls<2>(a->dtype, a->num_threads, co)
          : push_rs ? pick_nvls<6>(a->dtype, a->num_threads, co) : pick_nvls<5>(a->dtype, a->num_threads, co);
      break;
    case LAGOM_ALL_TO_ALL:
      if (!c->nvls_peers_ready) return 0;
      in_b = out_b = a->count * e * n;
      if (tma && tma_smem_ok(reinterpret_cast<const void*>(&a2a_tma_kernel))) {
        k = reinterpret_cast<const void*>(&a2a_tma_kernel);
        *smem_bytes = kA2aSmem;
        break;
      }
      k = pick_nvls<3>(a->dtype, a->num_threads, co);
      break;
    default: return 0;
  }
  // Whole 16 B units per block: a property of (collective, count, dtype),
  // identical on every rank, so every rank falls back to P2P together.
  if ((a->count * e) % 16 != 0) return 0;
  // peer-store kernels (one-hop AllToAll / AllGather) write into peer_recv,
  // the one-hop RS reads peer_send: both buffers must be in the region too
  const bool a2a = a->collective == LAGOM_ALL_TO_ALL || (a->collective == LAGOM_ALL_GATHER && hop);
  const bool send_mc = a->collective != LAGOM_ALL_GATHER && !a2a, recv_mc = a->collective != LAGOM_REDUCE_SCATTER;
  const bool need_send = send_mc || (a->collective == LAGOM_REDUCE_SCATTER && hop && !push_rs);
  const bool need_recv = recv_mc || a2a;
  // Buffer placement is per rank: a rank that fell back to P2P here while
  // its peers ran the switch kernel would wait on flags nobody writes, so a
  // misplaced buffer is an error, not a fallback.
  if ((reinterpret_cast<uintptr_t>(send) | reinterpret_cast<uintptr_t>(recv)) & 15)
    return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "TREE with NVLS bound: buffers must be 16-byte aligned"), -1;
  if ((need_send && !inside(c, send, in_b)) || (need_recv && !inside(c, recv, out_b)))
    return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT,
                      "TREE with NVLS bound: send/recv must lie in the NVLS region (lagom_comm_nvls_alloc)"),
           -1;
  NvlsParams p{};
  for (int r = 0; r < c->nranks; ++r) p.heap[r] = c->heap[r];
  p.rank = c->rank;
  p.nranks = c->nranks;
  p.count = a->count;
  p.elem_bytes = static_cast<int>(e);
  p.send_uc = static_cast<const char*>(send);
  p.recv_uc = static_cast<char*>(recv);
  p.send_mc = send_mc ? c->nvls_mc + (static_cast<const char*>(send) - c->nvls_uc) : nullptr;
  p.recv_mc = recv_mc && !a2a ? c->nvls_mc + (static_cast<char*>(recv) - c->nvls_uc) : nullptr;
  if (a2a)
    for (int q = 0; q < c->nranks; ++q) p.peer_recv[q] = c->nvls_peer[q] + (static_cast<char*>(recv) - c->nvls_uc);
  if (a->collective == LAGOM_REDUCE_SCATTER && hop && !push_rs)
    for (int q = 0; q < c->nranks; ++q)
      p.peer_send[q] = c->nvls_peer[q] + (static_cast<const char*>(send) - c->nvls_uc);
  if (a->collective == LAGOM_REDUCE_SCATTER && push_rs) {
    const int64_t at = (c->nvls_scratch - c->nvls_uc) + static_cast<int64_t>(c->rank) * c->nvls_scratch_slot;
    for (int q = 0; q < c->nranks; ++q) p.peer_recv[q] = c->nvls_peer[q] + at;  // my slot in q's scratch
    p.scratch = c->nvls_scratch;
    p.scratch_slot = c->nvls_scratch_slot;
  }
  p.off_nvbar = c->off_nvbar;
  p.off_nvep = c->off_nvep;
  p.off_nvpiece = c->off_nvpiece;
  p.off_nvpbase = c->off_nvpbase;
  p.piece_units = a->chunk_bytes / 16;
  p.abort_flag = c->abort_dev;
  p.timeout_ns = static_cast<uint64_t>(c->opts.timeout_ms) * 1000000ull;
  p.span = static_cast<unsigned long long*>(a->span_out);
  p.phase = c->phase_stamps ? reinterpret_cast<uint64_t*>(c->heap[c->rank] + c->off_phase) : nullptr;
  std::memcpy(params_out, &p, sizeof p);
  *params_bytes = sizeof p;
  *kernel = k;
  return 1;
}

extern "C" {

int lagom_comm_nvls_supported(lagom_comm_t c) {
  if (!c || c->virt || c->nranks < 2) return 0;
  CUdevice dev;
  int mc = 0;
  if (DRV(cuDeviceGet)(&dev, c->device) != CUDA_SUCCESS) return 0;
  if (DRV(cuDeviceGetAttribute)(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return 0;
  return mc ? 1 : 0;
}

int lagom_comm_nvls_export(lagom_comm_t c, int64_t bytes, void* blob) {
  if (!c || !blob || bytes <= 0) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_export: bad arguments");
  std::memset(blob, 0, LAGOM_HANDLE_BYTES);
  if (!lagom_comm_nvls_supported(c)) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "NVLS multicast unsupported");
  if (c->rank != 0) return LAGOM_OK;
  cudaSetDevice(c->device);
  const size_t g = granularity(c->nranks);
  CUmulticastObjectProp prop{};
  prop.numDevices = static_cast<unsigned>(c->nranks);
  prop.size = (static_cast<size_t>(bytes) + g - 1) / g * g;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mc;
  LAGOM_DRV(DRV(cuMulticastCreate)(&mc, &prop));
  int fd = -1;
  LAGOM_DRV(DRV(cuMemExportToShareableHandle)(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  c->nvls_mc_handle = mc;
  c->nvls_bytes = static_cast<int64_t>(prop.size);
  c->nvls_export_fd = fd;
  Blob b{kBlobMagic, static_cast<int64_t>(getpid()), fd, static_cast<int64_t>(prop.size)};
  std::memcpy(blob, &b, sizeof b);
  return LAGOM_OK;
}

int lagom_comm_nvls_import(lagom_comm_t c, const void* blob) {
  if (!c || !blob) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_import: bad arguments");
  Blob b;
  std::memcpy(&b, blob, sizeof b);
  if (b.magic != kBlobMagic) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_import: not an NVLS blob");
  cudaSetDevice(c->device);
  if (c->rank != 0) {
    const int pidfd = static_cast<int>(syscall(SYS_pidfd_open, static_cast<pid_t>(b.pid), 0));
    if (pidfd < 0) return lagom_fail(LAGOM_ERR_CUDA, "pidfd_open failed");
    const int fd = static_cast<int>(syscall(SYS_pidfd_getfd, pidfd, static_cast<int>(b.fd), 0));
    close(pidfd);
    if (fd < 0) return lagom_fail(LAGOM_ERR_CUDA, "pidfd_getfd failed (ptrace permission?)");
    CUmemGenericAllocationHandle mc;
    const CUresult r = DRV(cuMemImportFromShareableHandle)(&mc, reinterpret_cast<void*>(static_cast<intptr_t>(fd)),
                                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fd);
    if (r != CUDA_SUCCESS) return drv_fail(r, "cuMemImportFromShareableHandle");
    c->nvls_mc_handle = mc;
    c->nvls_bytes = b.size;
  }
  CUdevice dev;
  LAGOM_DRV(DRV(cuDeviceGet)(&dev, c->device));
  LAGOM_DRV(DRV(cuMulticastAddDevice)(static_cast<CUmemGenericAllocationHandle>(c->nvls_mc_handle), dev));
  return LAGOM_OK;
}

int lagom_comm_nvls_bind(lagom_comm_t c) {
  if (!c || !c->nvls_mc_handle) return lagom_fail(LAGOM_ERR_NOT_READY, "nvls_bind before import");
  cudaSetDevice(c->device);
  const size_t size = static_cast<size_t>(c->nvls_bytes), g = granularity(c->nranks);
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mem;
  LAGOM_DRV(DRV(cuMemCreate)(&mem, size, &ap, 0));
  c->nvls_mem_handle = mem;
  const auto mc = static_cast<CUmemGenericAllocationHandle>(c->nvls_mc_handle);
  LAGOM_DRV(DRV(cuMulticastBindMem)(mc, 0, mem, 0, size, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = c->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mcv = 0;
  LAGOM_DRV(DRV(cuMemAddressReserve)(&uc, size, g, 0, 0));
  LAGOM_DRV(DRV(cuMemMap)(uc, size, 0, mem, 0));
  LAGOM_DRV(DRV(cuMemSetAccess)(uc, size, &acc, 1));
  LAGOM_DRV(DRV(cuMemAddressReserve)(&mcv, size, g, 0, 0));
  LAGOM_DRV(DRV(cuMemMap)(mcv, size, 0, mc, 0));
  LAGOM_DRV(DRV(cuMemSetAccess)(mcv, size, &acc, 1));
  c->nvls_uc = reinterpret_cast<char*>(uc);
  c->nvls_mc = reinterpret_cast<char*>(mcv);
  if (cudaMemset(c->nvls_uc, 0, size) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return lagom_fail(LAGOM_ERR_CUDA, "nvls region init");
  c->nvls_used = 0;
  c->nvls_ready = true;
  // Binding is collective (every rank imported before anyone binds), so the
  // exported fd has served its purpose.
  if (c->nvls_export_fd >= 0) {
    close(c->nvls_export_fd);
    c->nvls_export_fd = -1;
  }
  return LAGOM_OK;
}

int lagom_comm_nvls_alloc(lagom_comm_t c, int64_t bytes, void** ptr) {
  if (!c || !ptr || bytes < 0) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_alloc: bad arguments");
  if (!c->nvls_ready) return lagom_fail(LAGOM_ERR_NOT_READY, "NVLS region not bound");
  const int64_t off = (c->nvls_used + 4095) / 4096 * 4096;
  if (off + bytes > c->nvls_bytes) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "NVLS region exhausted");
  c->nvls_used = off + bytes;
  *ptr = c->nvls_uc + off;
  return LAGOM_OK;
}

int64_t lagom_comm_nvls_bytes(lagom_comm_t c) { return c && c->nvls_ready ? c->nvls_bytes : 0; }

int lagom_comm_nvls_scratch(lagom_comm_t c, int64_t slot_bytes) {
  if (!c || slot_bytes <= 0) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_scratch: bad arguments");
  if (c->nvls_scratch) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_scratch: already reserved");
  const int64_t slot = (slot_bytes + 4095) / 4096 * 4096;
  void* p = nullptr;
  if (int s = lagom_comm_nvls_alloc(c, slot * c->nranks, &p)) return s;
  c->nvls_scratch = static_cast<char*>(p);
  c->nvls_scratch_slot = slot;
  return LAGOM_OK;
}

int lagom_comm_nvls_export_peer(lagom_comm_t c, void* blob) {
  if (!c || !blob) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_export_peer: bad arguments");
  if (!c->nvls_ready) return lagom_fail(LAGOM_ERR_NOT_READY, "nvls_export_peer before nvls_bind");
  std::memset(blob, 0, LAGOM_HANDLE_BYTES);
  cudaSetDevice(c->device);
  if (c->nvls_peer_fd < 0) {
    int fd = -1;
    LAGOM_DRV(DRV(cuMemExportToShareableHandle)(&fd, static_cast<CUmemGenericAllocationHandle>(c->nvls_mem_handle),
                                                CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    c->nvls_peer_fd = fd;
  }
  Blob b{kPeerMagic, static_cast<int64_t>(getpid()), c->nvls_peer_fd, c->nvls_bytes};
  std::memcpy(blob, &b, sizeof b);
  return LAGOM_OK;
}

int lagom_comm_nvls_import_peers(lagom_comm_t c, const void* blobs) {
  if (!c || !blobs) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_import_peers: bad arguments");
  if (!c->nvls_ready) return lagom_fail(LAGOM_ERR_NOT_READY, "nvls_import_peers before nvls_bind");
  cudaSetDevice(c->device);
  const size_t g = granularity(c->nranks);
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = c->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      c->nvls_peer[q] = c->nvls_uc;
      continue;
    }
    if (c->nvls_peer[q]) continue;
    Blob b;
    std::memcpy(&b, static_cast<const unsigned char*>(blobs) + static_cast<size_t>(q) * LAGOM_HANDLE_BYTES, sizeof b);
    if (b.magic != kPeerMagic || b.size != c->nvls_bytes)
      return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_import_peers: blob of rank " + std::to_string(q));
    const int pidfd = static_cast<int>(syscall(SYS_pidfd_open, static_cast<pid_t>(b.pid), 0));
    if (pidfd < 0) return lagom_fail(LAGOM_ERR_CUDA, "pidfd_open failed");
    const int fd = static_cast<int>(syscall(SYS_pidfd_getfd, pidfd, static_cast<int>(b.fd), 0));
    close(pidfd);
    if (fd < 0) return lagom_fail(LAGOM_ERR_CUDA, "pidfd_getfd failed (ptrace permission?)");
    CUmemGenericAllocationHandle h;
    const CUresult r = DRV(cuMemImportFromShareableHandle)(&h, reinterpret_cast<void*>(static_cast<intptr_t>(fd)),
                                                           CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fd);
    if (r != CUDA_SUCCESS) return drv_fail(r, "cuMemImportFromShareableHandle (peer)");
    CUdeviceptr va = 0;
    const size_t size = static_cast<size_t>(b.size);
    CUresult m = DRV(cuMemAddressReserve)(&va, size, g, 0, 0);
    const bool reserved = m == CUDA_SUCCESS;
    bool mapped = false;
    if (m == CUDA_SUCCESS) mapped = (m = DRV(cuMemMap)(va, size, 0, h, 0)) == CUDA_SUCCESS;
    DRV(cuMemRelease)(h);  // the mapping holds its own reference
    if (m == CUDA_SUCCESS) m = DRV(cuMemSetAccess)(va, size, &acc, 1);
    if (m != CUDA_SUCCESS) {  // undo this peer's partial mapping; earlier peers stay for release
      if (mapped) DRV(cuMemUnmap)(va, size);
      if (reserved) DRV(cuMemAddressFree)(va, size);
      return drv_fail(m, "map peer NVLS region");
    }
    c->nvls_peer[q] = reinterpret_cast<char*>(va);
  }
  c->nvls_peers_mapped = true;
  return LAGOM_OK;
}

int lagom_comm_nvls_use_peers(lagom_comm_t c, int on) {
  if (!c) return lagom_fail(LAGOM_ERR_INVALID_ARGUMENT, "nvls_use_peers: null comm");
  if (on && !c->nvls_peers_mapped) return lagom_fail(LAGOM_ERR_NOT_READY, "nvls_use_peers before import_peers");
  c->nvls_peers_ready = on != 0;
  return LAGOM_OK;
}

}  // extern "C"

void lagom_nvls_release(lagom_comm* c) {
  if (!c) return;
  for (int q = 0; q < LAGOM_MAX_RANKS; ++q) {
    if (c->nvls_peer[q] && q != c->rank) {
      DRV(cuMemUnmap)(reinterpret_cast<CUdeviceptr>(c->nvls_peer[q]), static_cast<size_t>(c->nvls_bytes));
      DRV(cuMemAddressFree)(reinterpret_cast<CUdeviceptr>(c->nvls_peer[q]), static_cast<size_t>(c->nvls_bytes));
    }
    c->nvls_peer[q] = nullptr;
  }
  c->nvls_peers_ready = c->nvls_peers_mapped = false;
  if (c->nvls_peer_fd >= 0) {
    close(c->nvls_peer_fd);
    c->nvls_peer_fd = -1;
  }
  if (c->nvls_export_fd >= 0) {
    close(c->nvls_export_fd);
    c->nvls_export_fd = -1;
  }
  if (c->nvls_mc) {
    DRV(cuMemUnmap)(reinterpret_cast<CUdeviceptr>(c->nvls_mc), static_cast<size_t>(c->nvls_bytes));
    DRV(cuMemAddressFree)(reinterpret_cast<CUdeviceptr>(c->nvls_mc), static_cast<size_t>(c->nvls_bytes));
  }
  if (c->nvls_uc) {
    DRV(cuMemUnmap)(reinterpret_cast<CUdeviceptr>(c->nvls_uc), static_cast<size_t>(c->nvls_bytes));
    DRV(cuMemAddressFree)(reinterpret_cast<CUdeviceptr>(c->nvls_uc), static_cast<size_t>(c->nvls_bytes));
  }
  if (c->nvls_mc_handle && c->nvls_mem_handle) {
    CUdevice dev;
    if (DRV(cuDeviceGet)(&dev, c->device) == CUDA_SUCCESS)
      DRV(cuMulticastUnbind)(static_cast<CUmemGenericAllocationHandle>(c->nvls_mc_handle), dev, 0,
                        static_cast<size_t>(c->nvls_bytes));
  }
  if (c->nvls_mem_handle) DRV(cuMemRelease)(static_cast<CUmemGenericAllocationHandle>(c->nvls_mem_handle));
  if (c->nvls_mc_handle) DRV(cuMemRelease)(static_cast<CUmemGenericAllocationHandle>(c->nvls_mc_handle));
  c->nvls_mc = c->nvls_uc = nullptr;
  c->nvls_scratch = nullptr;
  c->nvls_scratch_slot = 0;
  c->nvls_ready = false;
}
