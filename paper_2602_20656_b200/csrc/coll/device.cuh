// sm_100a collective kernels: protocol primitives and algorithm bodies.
//
// Realizes the reference's modeled collective (comm_time over CommConfig,
// reference commperf.cpp:112-125 / model.hpp:37-67) as real kernels over
// NVLink 5 / NVSwitch peer memory:
//   * one CTA per channel (NC), NT threads, C-byte pipeline steps;
//   * a "connection" = ordered rank pair (src -> dst) per channel, with
//     `steps` staging slots living in dst's memory (written remotely by src),
//     a ready counter in dst's memory and a freed counter in src's memory;
//   * protocols SIMPLE (bulk 16 B vector stores + release/acquire counters),
//     LL (16 B lines = 8 B payload + two 4 B flags; no fence) and LL128
//     (128 B lines = 112 B payload + 8 B flag, relying on 128 B store
//     atomicity over NVLink like NCCL's LL128);
//   * reductions in the element type with a fixed, documented order so the
//     CPU oracle (oracle/coll_oracle.c) reproduces every result bit for bit.
// No tensor cores: the collectives are not a contraction.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "lagom_coll.h"

namespace lagom_dev {

constexpr int kUnroll = 4;

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }
constexpr unsigned kFull = 0xffffffffu;

// --------------------------------------------------------------- params ----
// Heap layout (identical on every rank, offsets in bytes from heap base):
//   ready[ch][src]     128 B apart   written by src (Simple data-ready count)
//   freed[ch][dst]     128 B apart   written by dst (slots consumed count)
//   sstep[ch][dst]     8 B           my send-step counter (local only)
//   rstep[ch][src]     8 B           my recv-step counter (local only)
//   slots[ch][src][k]  slot_bytes    staging written by src, k < steps
struct KParams {
  char* heap[LAGOM_MAX_RANKS];
  const char* send[LAGOM_MAX_RANKS];
  char* recv[LAGOM_MAX_RANKS];
  int rank;  // real mode: this rank; virtual mode: -1 (rank = blockIdx.y)
  int nranks;
  int elem_bytes;
  int steps;
  int64_t count;
  int64_t chunk_bytes;
  int64_t slot_bytes;
  int64_t off_ready, off_freed, off_sstep, off_rstep, off_slots;
  unsigned int* abort_flag;  // host-mapped, sticky
  uint64_t timeout_ns;
  unsigned long long* span;  // optional {min start, max end} in globaltimer ns
  int tma;                   // SIMPLE data path through TMA bulk copies
  int tma_stages;            // smem ring depth per group
  int tile_bytes;            // bytes per TMA tile (per input buffer)
  int tma_reduce;            // also route reduction steps through the TMA ring
  // Copy steps split their bytes between the TMA engine (warp 0) and the LSU
  // threads of the other warps, in proportion to measured rates: the TMA
  // engine of one SM moves as much as `tma_share_*` LSU threads (local copy /
  // push to a peer). 0: the TMA ring takes the whole 16 B aligned body.
  int tma_share_local;
  int tma_share_push;
};

// ------------------------------------------------------------------ TMA ----
// 1-D bulk copies (cp.async.bulk): one elected thread per group keeps
// `tma_stages` tiles of every input in flight (mbarrier complete_tx), the
// group combines them in shared memory, and bulk stores push the result to
// the peer's staging slot / the local output. A single CTA sustains ~50 GB/s
// this way against ~35 GB/s (push) / ~11 GB/s (pull) with 640 threads of
// vector ld/st (tools/tma_probe.cu, measured on B200).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAGOM_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAGOM_WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
// Asks the TMA unit to pull [p, p + bytes) into L2 (16 B aligned, 16 B
// multiple): no registers or shared memory held, so register-capped kernels
// get their next batch's loads served from L2 instead of HBM.
__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
  if (bytes > 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(static_cast<uint32_t>(bytes)) : "memory");
}
__device__ __forceinline__ void mbar_init_count(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Order generic-proxy accesses (flags, peer writes) against async-proxy ones.
__device__ __forceinline__ void fence_proxy_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// --------------------------------------------------------- memory model ----
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Relaxed flag accesses for release / acquire patterns with an explicit
// fence: one fence covers several flag stores (or many polls).
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ uint4 ld_volatile_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_v4(uint4* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
// Staging reads bypass L1 (slots are rewritten by a peer every `steps` steps).
__device__ __forceinline__ uint4 ld_stage(const uint4* p) { return __ldcg(p); }
__device__ __forceinline__ void st_stage(uint4* p, uint4 v) { __stcg(p, v); }
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// User buffers: 16 B vectors when aligned and whole, else byte-granular.
__device__ __forceinline__ uint4 load_user(const char* p, int nb, bool aligned) {
  if (aligned && nb == 16) return *reinterpret_cast<const uint4*>(p);
  uint4 v = make_uint4(0, 0, 0, 0);
  unsigned char* d = reinterpret_cast<unsigned char*>(&v);
  for (int i = 0; i < nb; ++i) d[i] = static_cast<unsigned char>(p[i]);
  return v;
}
__device__ __forceinline__ void store_user(char* p, uint4 v, int nb, bool aligned) {
  if (aligned && nb == 16) {
    *reinterpret_cast<uint4*>(p) = v;
    return;
  }
  const unsigned char* s = reinterpret_cast<const unsigned char*>(&v);
  for (int i = 0; i < nb; ++i) p[i] = static_cast<char>(s[i]);
}

// ------------------------------------------------------------ reductions ----
// Element-wise op on 4-byte words. bf16/f16 are widened to f32, combined and
// rounded back to nearest-even — exactly what oracle/coll_oracle.c does.
struct NoRed {};
template <typename T, int OP> struct Red;

template <int OP> struct Red<float, OP> {
  __device__ static uint32_t w(uint32_t a, uint32_t b) {
    const float x = __uint_as_float(a), y = __uint_as_float(b);
    return __float_as_uint(OP == LAGOM_SUM ? __fadd_rn(x, y) : OP == LAGOM_MAX ? fmaxf(x, y) : fminf(x, y));
  }
};
template <int OP> struct Red<int32_t, OP> {
  __device__ static uint32_t w(uint32_t a, uint32_t b) {
    const int32_t x = static_cast<int32_t>(a), y = static_cast<int32_t>(b);
    const int32_t r = OP == LAGOM_SUM ? static_cast<int32_t>(a + b) : OP == LAGOM_MAX ? max(x, y) : min(x, y);
    return static_cast<uint32_t>(r);
  }
};
template <int OP> struct Red<__nv_bfloat16, OP> {
  __device__ static uint32_t h(uint32_t a, uint32_t b) {
    const float x = __uint_as_float(a << 16), y = __uint_as_float(b << 16);
    const float r = OP == LAGOM_SUM ? __fadd_rn(x, y) : OP == LAGOM_MAX ? fmaxf(x, y) : fminf(x, y);
    return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(r)));
  }
  __device__ static uint32_t w(uint32_t a, uint32_t b) {
    return h(a & 0xffffu, b & 0xffffu) | (h(a >> 16, b >> 16) << 16);
  }
};
template <int OP> struct Red<__half, OP> {
  __device__ static uint32_t h(uint32_t a, uint32_t b) {
    const float x = __half2float(__ushort_as_half(static_cast<unsigned short>(a)));
    const float y = __half2float(__ushort_as_half(static_cast<unsigned short>(b)));
    const float r = OP == LAGOM_SUM ? __fadd_rn(x, y) : OP == LAGOM_MAX ? fmaxf(x, y) : fminf(x, y);
    return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(r)));
  }
  __device__ static uint32_t w(uint32_t a, uint32_t b) {
    return h(a & 0xffffu, b & 0xffffu) | (h(a >> 16, b >> 16) << 16);
  }
};

template <class R>
__device__ __forceinline__ uint4 red4(uint4 a, uint4 b) {
  return make_uint4(R::w(a.x, b.x), R::w(a.y, b.y), R::w(a.z, b.z), R::w(a.w, b.w));
}
template <>
__device__ __forceinline__ uint4 red4<NoRed>(uint4 a, uint4) {
  return a;
}

// ------------------------------------------------------------ groups -------
// A group of warps sharing a named barrier (ring/A2A: the whole CTA; tree:
// the reduce-up half and the broadcast-down half).
struct Grp {
  int tid;
  int n;
  int bar;
  volatile int* abort;  // shared memory, CTA-wide
  unsigned char* smem = nullptr;  // TMA tile ring: stages x 3 buffers x tile_bytes
  uint64_t* bars = nullptr;       // "full": one mbarrier per stage (TMA loads landed)
  uint64_t* reds = nullptr;       // "reduced": per stage, one arrival per consumer warp
  uint32_t* tiles = nullptr;      // tiles this group has cycled through the ring
  uint32_t* redpar = nullptr;     // producer-private: next parity per stage of `reds`
  int copy_stage = 0;             // bytes per stage for one-input (copy) steps; 0 = 3 x tile_bytes
  __device__ void sync() const { asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(n) : "memory"); }
};

// --------------------------------------------------------------- links -----
struct SendLink {
  char* slots;            // dst's staging for (ch, me)
  uint64_t* ready;        // dst's ready counter for (ch, me)
  const uint64_t* freed;  // my freed counter for (ch, dst)
  uint64_t* step_home;    // my persisted send-step counter
  uint64_t step;
};
struct RecvLink {
  const char* slots;      // my staging for (ch, src)
  const uint64_t* ready;  // my ready counter for (ch, src)
  uint64_t* freed;        // src's freed counter for (ch, me)
  uint64_t* step_home;
  uint64_t step;
};

__device__ __forceinline__ SendLink make_send(const KParams& P, int me, int ch, int dst) {
  const int64_t n = P.nranks;
  SendLink l;
  l.slots = P.heap[dst] + P.off_slots + (ch * n + me) * P.steps * P.slot_bytes;
  l.ready = reinterpret_cast<uint64_t*>(P.heap[dst] + P.off_ready + (ch * n + me) * 128);
  l.freed = reinterpret_cast<const uint64_t*>(P.heap[me] + P.off_freed + (ch * n + dst) * 128);
  l.step_home = reinterpret_cast<uint64_t*>(P.heap[me] + P.off_sstep + (ch * n + dst) * 8);
  l.step = *reinterpret_cast<volatile uint64_t*>(l.step_home);
  return l;
}
__device__ __forceinline__ RecvLink make_recv(const KParams& P, int me, int ch, int src) {
  const int64_t n = P.nranks;
  RecvLink l;
  l.slots = P.heap[me] + P.off_slots + (ch * n + src) * P.steps * P.slot_bytes;
  l.ready = reinterpret_cast<const uint64_t*>(P.heap[me] + P.off_ready + (ch * n + src) * 128);
  l.freed = reinterpret_cast<uint64_t*>(P.heap[src] + P.off_freed + (ch * n + me) * 128);
  l.step_home = reinterpret_cast<uint64_t*>(P.heap[me] + P.off_rstep + (ch * n + src) * 8);
  l.step = *reinterpret_cast<volatile uint64_t*>(l.step_home);
  return l;
}

// ------------------------------------------------------------- waiting -----
// Bounded spin: aborts (sticky host flag) after timeout_ns or when any other
// CTA / group already aborted, so a lost peer can never hang the GPU.
struct Watch {
  uint64_t t0 = 0;
  unsigned it = 0;
  __device__ bool expired(const KParams& P, volatile int* abort) {
    if ((++it & 127u) != 0) return false;
    if (*abort) return true;
    if (*reinterpret_cast<volatile unsigned*>(P.abort_flag)) return true;
    const uint64_t now = globaltimer();
    if (t0 == 0) t0 = now;
    if (now - t0 > P.timeout_ns) {
      atomicExch(P.abort_flag, 1u);
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ bool wait_geq(const uint64_t* p, uint64_t target, const KParams& P,
                                         volatile int* abort) {
  Watch w;
  while (ld_acquire_sys(p) < target)
    if (w.expired(P, abort)) return false;
  return true;
}

// ---------------------------------------------------------------- step -----
// One pipeline step of a group: optionally receive from NR links, combine with
// own data (SRC), write the result to user memory (DST) and forward it on NS
// links. Combine order: v = own; v = op(v, recv[0]); v = op(v, recv[1]).
// Every participant of a connection executes the same sequence of steps with
// the same byte counts, which keeps the step counters in lockstep.
template <int PROTO, class R, int NR, bool SRC, bool DST, int NS>
__device__ __noinline__ bool step(const Grp& g, const KParams& P, RecvLink* rl, SendLink* sl,
                     const char* src, char* dst, int64_t nbytes) {
  const int S = P.steps;
  // 1. flow control: slot free on every send link; data ready (SIMPLE).
  if (g.tid == 0) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < NS; ++i)
      if (ok && sl[i].step >= static_cast<uint64_t>(S))
        ok = wait_geq(sl[i].freed, sl[i].step - S + 1, P, g.abort);
    if (PROTO == LAGOM_SIMPLE) {
#pragma unroll
      for (int i = 0; i < NR; ++i)
        if (ok) ok = wait_geq(rl[i].ready, rl[i].step + 1, P, g.abort);
    }
    if (!ok) *g.abort = 1;
  }
  g.sync();
  if (*g.abort) return false;

  const char* rs[NR > 0 ? NR : 1];
  char* ss[NS > 0 ? NS : 1];
#pragma unroll
  for (int i = 0; i < NR; ++i) rs[i] = rl[i].slots + static_cast<int64_t>(rl[i].step % S) * P.slot_bytes;
#pragma unroll
  for (int i = 0; i < NS; ++i) ss[i] = sl[i].slots + static_cast<int64_t>(sl[i].step % S) * P.slot_bytes;
  const bool src_al = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  const bool dst_al = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  const int64_t units = (nbytes + 15) >> 4;
  bool ok = true;

  int64_t lsu_from = 0;  // units already moved by the TMA path
  int ltid = g.tid, ln = g.n;  // the LSU part's threads (all, or warps 1..)
  if constexpr (PROTO == LAGOM_SIMPLE) {
    constexpr int NIN = NR + (SRC ? 1 : 0);
    // TMA moves copy steps (one input); reduction steps use it only when
    // P.tma_reduce is set (measured slower than the LSU path on B200 so far).
    if (P.tma && g.smem && NIN > 0 && (NIN == 1 || P.tma_reduce) && (!SRC || src_al) && (!DST || dst_al) &&
        nbytes >= 16) {
      int64_t main = nbytes & ~static_cast<int64_t>(15);
      if (NIN == 1) {
        const int share = NS > 0 ? P.tma_share_push : P.tma_share_local;
        if (share > 0 && g.n >= 64) {  // warp 0 drives TMA, warps 1.. run the LSU loop
          main = (main * share / (share + g.n - 32)) & ~static_cast<int64_t>(15);
          ltid = g.tid - 32;
          ln = g.n - 32;
        }
      }
      // A copy step (one input) owns the stage's three buffers as one tile:
      // 3x the bytes in flight, which is what bounds a single SM's TMA rate.
      const int T = NIN == 1 ? (g.copy_stage ? g.copy_stage : 3 * P.tile_bytes) : P.tile_bytes;
      const int ST = P.tma_stages;
      const int64_t ntiles = (main + T - 1) / T;
      const uint32_t base = *reinterpret_cast<volatile uint32_t*>(g.tiles);
      auto buf = [&](uint32_t stage, int b) {
        return g.smem + (static_cast<int64_t>(stage) * 3 + b) * P.tile_bytes;
      };
      auto input = [&](int b, int64_t off) -> const char* {
        if (SRC) return b == 0 ? src + off : rs[b > 0 ? b - 1 : 0] + off;
        return rs[b] + off;
      };
      auto issue = [&](int64_t i) {
        const uint32_t stg = (base + static_cast<uint32_t>(i)) % ST;
        const uint32_t len = static_cast<uint32_t>(lmin(T, main - i * T));
        mbar_expect(&g.bars[stg], len * NIN);
#pragma unroll
        for (int b = 0; b < NIN; ++b) bulk_load(buf(stg, b), input(b, i * T), len, &g.bars[stg]);
      };
      if (g.tid == 0) {
        fence_proxy_global();  // staging data acquired through the ready flag
        for (int64_t i = 0; i < ntiles && i < ST; ++i) issue(i);
      }
      const int nwarps = g.n >> 5;
      if (NIN >= 2 && nwarps >= 2 && g.reds) {
        // Warp-specialized: warp 0 lane 0 produces (bulk loads ahead, bulk
        // stores behind), warps 1.. reduce; "full" and "reduced" mbarriers
        // hand tiles back and forth so the reduction of tile i overlaps the
        // stores of tile i-1 and the loads of tiles i+1..i+ST-1.
        const int warp = g.tid >> 5, lane = g.tid & 31;
        if (warp == 0) {
          if (lane == 0) {
            // `reds` only completes phases for tiles that went through this
            // path (copy steps skip it), so its parity is tracked per stage.
            uint32_t rp = *g.redpar;
            for (int64_t i = 0; i < ntiles; ++i) {
              const uint32_t gi = base + static_cast<uint32_t>(i);
              const uint32_t stg = gi % ST;
              const uint32_t len = static_cast<uint32_t>(lmin(T, main - i * T));
              mbar_wait(&g.reds[stg], (rp >> stg) & 1u);
              rp ^= 1u << stg;
#pragma unroll
              for (int s = 0; s < NS; ++s) bulk_store(ss[s] + i * T, buf(stg, 0), len);
              if (DST) bulk_store(dst + i * T, buf(stg, 0), len);
              bulk_commit();
              if (i >= 1 && i - 1 + ST < ntiles) {
                bulk_wait_read1();
                issue(i - 1 + ST);
              }
            }
            *g.redpar = rp;
          }
        } else {
          const int cth = g.n - 32, ctid = g.tid - 32;
          for (int64_t i = 0; i < ntiles; ++i) {
            const uint32_t gi = base + static_cast<uint32_t>(i);
            const uint32_t stg = gi % ST, parity = (gi / ST) & 1u;
            const uint32_t len = static_cast<uint32_t>(lmin(T, main - i * T));
            mbar_wait(&g.bars[stg], parity);
            uint4* a = reinterpret_cast<uint4*>(buf(stg, 0));
            const uint4* b1 = reinterpret_cast<const uint4*>(buf(stg, 1));
            const uint4* b2 = reinterpret_cast<const uint4*>(buf(stg, 2));
            for (uint32_t u = ctid; u < len / 16; u += cth) {
              uint4 v = red4<R>(a[u], b1[u]);
              if (NIN == 3) v = red4<R>(v, b2[u]);
              a[u] = v;
            }
            fence_proxy_shared();
            __syncwarp();
            if (lane == 0) mbar_arrive(&g.reds[stg]);
          }
        }
      } else
      for (int64_t i = 0; i < ntiles; ++i) {
        const uint32_t gi = base + static_cast<uint32_t>(i);
        const uint32_t stg = gi % ST, parity = (gi / ST) & 1u;
        const uint32_t len = static_cast<uint32_t>(lmin(T, main - i * T));
        if constexpr (NIN >= 2) {
          mbar_wait(&g.bars[stg], parity);
          uint4* a = reinterpret_cast<uint4*>(buf(stg, 0));
          const uint4* b1 = reinterpret_cast<const uint4*>(buf(stg, 1));
          const uint4* b2 = reinterpret_cast<const uint4*>(buf(stg, 2));
          for (uint32_t u = g.tid; u < len / 16; u += g.n) {
            uint4 v = red4<R>(a[u], b1[u]);
            if (NIN == 3) v = red4<R>(v, b2[u]);
            a[u] = v;
          }
          fence_proxy_shared();  // generic smem writes -> async-proxy bulk store
          g.sync();
        } else {
          if (g.tid == 0) mbar_wait(&g.bars[stg], parity);
        }
        if (g.tid == 0) {
#pragma unroll
          for (int s = 0; s < NS; ++s) bulk_store(ss[s] + i * T, buf(stg, 0), len);
          if (DST) bulk_store(dst + i * T, buf(stg, 0), len);
          bulk_commit();
          if (i >= 1 && i - 1 + ST < ntiles) {
            bulk_wait_read1();  // tile i-1's stores have read their stage
            issue(i - 1 + ST);
          }
        }
      }
      if (g.tid == 0) {
        bulk_wait_all();
        fence_proxy_global();
        *reinterpret_cast<volatile uint32_t*>(g.tiles) = base + static_cast<uint32_t>(ntiles);
      }
      lsu_from = main >> 4;
    }
  }
  if (PROTO == LAGOM_SIMPLE && ltid < 0) {
    // TMA driver warp of a split copy: its bytes are done (thread 0 waited).
  } else if constexpr (PROTO == LAGOM_SIMPLE) {
    // Fast path (all user pointers 16 B aligned): batches of U whole units per
    // thread, every load of the batch issued before any combine or store so
    // each thread keeps U (or 2U) 16 B requests in flight.
    constexpr int U = (NR + (SRC ? 1 : 0) >= 2) ? 4 : 8;
    const int64_t whole = nbytes >> 4;
    int64_t u0 = lsu_from + ltid;
    if ((!SRC || src_al) && (!DST || dst_al)) {
      const int64_t stride = static_cast<int64_t>(ln) * U;
      for (; u0 + static_cast<int64_t>(U - 1) * ln < whole; u0 += stride) {
        uint4 own[U];
        uint4 in[NR > 0 ? NR : 1][U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t u = u0 + static_cast<int64_t>(k) * ln;
          if (SRC) own[k] = reinterpret_cast<const uint4*>(src)[u];
#pragma unroll
          for (int i = 0; i < NR; ++i) in[i][k] = ld_stage(reinterpret_cast<const uint4*>(rs[i]) + u);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t u = u0 + static_cast<int64_t>(k) * ln;
          uint4 v = SRC ? own[k] : in[0][k];
#pragma unroll
          for (int i = SRC ? 0 : 1; i < NR; ++i) v = red4<R>(v, in[i][k]);
          if (DST) reinterpret_cast<uint4*>(dst)[u] = v;
#pragma unroll
          for (int i = 0; i < NS; ++i) st_stage(reinterpret_cast<uint4*>(ss[i]) + u, v);
        }
      }
    }
    // Remainder, partial last unit, misaligned user buffers.
    for (int64_t u = u0; u < units; u += ln) {
      const int nb = static_cast<int>(lmin(16, nbytes - u * 16));
      uint4 v = make_uint4(0, 0, 0, 0);
      if (SRC) v = load_user(src + u * 16, nb, src_al);
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const uint4 r = ld_stage(reinterpret_cast<const uint4*>(rs[i]) + u);
        v = (SRC || i > 0) ? red4<R>(v, r) : r;
      }
      if (DST) store_user(dst + u * 16, v, nb, dst_al);
#pragma unroll
      for (int i = 0; i < NS; ++i) st_stage(reinterpret_cast<uint4*>(ss[i]) + u, v);
    }
  } else if constexpr (PROTO == LAGOM_LL) {
    // Unit u (16 B payload) <-> two 16 B lines {d0,f,d1,f},{d2,f,d3,f}.
    // Each thread issues the loads of U units at once, then validates flags
    // (re-polling only the lines that have not landed yet).
    constexpr int U = 2;
    uint32_t rflag[NR > 0 ? NR : 1];
    uint32_t sflag[NS > 0 ? NS : 1];
#pragma unroll
    for (int i = 0; i < NR; ++i) rflag[i] = static_cast<uint32_t>(rl[i].step + 1);
#pragma unroll
    for (int i = 0; i < NS; ++i) sflag[i] = static_cast<uint32_t>(sl[i].step + 1);
    for (int64_t u0 = g.tid; u0 < units && ok; u0 += static_cast<int64_t>(g.n) * U) {
      uint4 v[U];
      uint4 la[NR > 0 ? NR : 1][U], lb[NR > 0 ? NR : 1][U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t u = u0 + static_cast<int64_t>(k) * g.n;
        v[k] = make_uint4(0, 0, 0, 0);
        if (u < units) {
          if (SRC) v[k] = load_user(src + u * 16, static_cast<int>(lmin(16, nbytes - u * 16)), src_al);
#pragma unroll
          for (int i = 0; i < NR; ++i) {
            const uint4* line = reinterpret_cast<const uint4*>(rs[i]) + 2 * u;
            la[i][k] = ld_volatile_v4(line);
            lb[i][k] = ld_volatile_v4(line + 1);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t u = u0 + static_cast<int64_t>(k) * g.n;
        if (u >= units) continue;
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          const uint4* line = reinterpret_cast<const uint4*>(rs[i]) + 2 * u;
          Watch w;
          while (!(la[i][k].y == rflag[i] && la[i][k].w == rflag[i] && lb[i][k].y == rflag[i] &&
                   lb[i][k].w == rflag[i])) {
            if (w.expired(P, g.abort)) {
              ok = false;
              break;
            }
            la[i][k] = ld_volatile_v4(line);
            lb[i][k] = ld_volatile_v4(line + 1);
          }
        }
      }
      if (!ok) break;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t u = u0 + static_cast<int64_t>(k) * g.n;
        if (u >= units) continue;
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          const uint4 got = make_uint4(la[i][k].x, la[i][k].z, lb[i][k].x, lb[i][k].z);
          v[k] = (SRC || i > 0) ? red4<R>(v[k], got) : got;
        }
        if (DST) store_user(dst + u * 16, v[k], static_cast<int>(lmin(16, nbytes - u * 16)), dst_al);
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          uint4* line = reinterpret_cast<uint4*>(ss[i]) + 2 * u;
          st_volatile_v4(line, make_uint4(v[k].x, sflag[i], v[k].y, sflag[i]));
          st_volatile_v4(line + 1, make_uint4(v[k].z, sflag[i], v[k].w, sflag[i]));
        }
      }
    }
    if (!ok) *g.abort = 1;
  } else {
    // LL128: line l = 8 x 16 B; lanes j<7 carry payload units 7l+j, lane 7
    // carries {0, 0, flag_lo, flag_hi}. A warp writes 4 whole lines per
    // store instruction; a line is consumed only when its flag matches. Each
    // warp iteration covers U line-quads with all loads issued up front.
    constexpr int U = 4;
    const int lane = g.tid & 31, warp = g.tid >> 5, nwarps = g.n >> 5;
    const int j = lane & 7;
    const int64_t lines = (units + 6) / 7;
    const int64_t quad_stride = static_cast<int64_t>(nwarps) * 4;
    uint64_t rflag[NR > 0 ? NR : 1];
    uint64_t sflag[NS > 0 ? NS : 1];
#pragma unroll
    for (int i = 0; i < NR; ++i) rflag[i] = rl[i].step + 1;
#pragma unroll
    for (int i = 0; i < NS; ++i) sflag[i] = sl[i].step + 1;
    for (int64_t base = static_cast<int64_t>(warp) * 4; base < lines; base += quad_stride * U) {
      uint4 v[U];
      uint4 d[NR > 0 ? NR : 1][U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t l = base + k * quad_stride + (lane >> 3);
        const int64_t u = 7 * l + j;
        const bool payload = l < lines && j < 7 && u < units;
        v[k] = make_uint4(0, 0, 0, 0);
        if (SRC && payload) v[k] = load_user(src + u * 16, static_cast<int>(lmin(16, nbytes - u * 16)), src_al);
#pragma unroll
        for (int i = 0; i < NR; ++i)
          d[i][k] = l < lines ? ld_volatile_v4(reinterpret_cast<const uint4*>(rs[i]) + 8 * l + j)
                              : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t l = base + k * quad_stride + (lane >> 3);
        const bool act = l < lines;
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          const uint4* cell = reinterpret_cast<const uint4*>(rs[i]) + 8 * l + j;
          uint64_t f = __shfl_sync(kFull, (static_cast<uint64_t>(d[i][k].w) << 32) | d[i][k].z, (lane & ~7) | 7);
          bool need = act && f != rflag[i];
          Watch w;
          while (__any_sync(kFull, need)) {
            if (__any_sync(kFull, w.expired(P, g.abort))) {
              ok = false;
              break;
            }
            if (need) d[i][k] = ld_volatile_v4(cell);
            f = __shfl_sync(kFull, (static_cast<uint64_t>(d[i][k].w) << 32) | d[i][k].z, (lane & ~7) | 7);
            need = act && f != rflag[i];
          }
        }
      }
      if (!ok) break;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t l = base + k * quad_stride + (lane >> 3);
        const int64_t u = 7 * l + j;
        const bool act = l < lines;
        const bool payload = act && j < 7 && u < units;
#pragma unroll
        for (int i = 0; i < NR; ++i) v[k] = (SRC || i > 0) ? red4<R>(v[k], d[i][k]) : d[i][k];
        if (DST && payload) store_user(dst + u * 16, v[k], static_cast<int>(lmin(16, nbytes - u * 16)), dst_al);
        if (!act) continue;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const uint4 out = j < 7 ? v[k]
                                  : make_uint4(0u, 0u, static_cast<uint32_t>(sflag[i]),
                                               static_cast<uint32_t>(sflag[i] >> 32));
          st_volatile_v4(reinterpret_cast<uint4*>(ss[i]) + 8 * l + j, out);
        }
      }
    }
    if (!ok) *g.abort = 1;
  }

  // 3. publish: data ready (SIMPLE) and slots consumed (all protocols).
  g.sync();
  if (*g.abort) return false;
  if (g.tid == 0) {
    if (PROTO == LAGOM_SIMPLE) {
      __threadfence_system();
#pragma unroll
      for (int i = 0; i < NS; ++i) st_release_sys(sl[i].ready, sl[i].step + 1);
    }
#pragma unroll
    for (int i = 0; i < NR; ++i) st_release_sys(rl[i].freed, rl[i].step + 1);
  }
#pragma unroll
  for (int i = 0; i < NS; ++i) ++sl[i].step;
#pragma unroll
  for (int i = 0; i < NR; ++i) ++rl[i].step;
  return true;
}

// Plain local copy by a group (own block of AllToAll / single-rank cases).
// With the TMA ring (SIMPLE, P.tma) one elected thread streams part of the
// 16 B aligned body through the smem stages (bulk load -> bulk store) while
// warps 1.. copy the rest with 8 x 16 B loads in flight per thread; the split
// follows P.tma_share_local, so small CTAs (the Lagom search starts at
// NT = 64) still move ~50 GB/s and large ones add the LSU rate on top.
__device__ __forceinline__ void group_copy(const Grp& g, const KParams& P, const char* src, char* dst,
                                           int64_t nbytes) {
  constexpr int U = 8;
  const bool al = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  int64_t done = 0;  // bytes moved by the TMA ring
  int ltid = g.tid, ln = g.n;
  if (P.tma && g.smem && al && nbytes >= 16) {
    done = nbytes & ~static_cast<int64_t>(15);
    if (P.tma_share_local > 0 && g.n >= 64) {
      done = (done * P.tma_share_local / (P.tma_share_local + g.n - 32)) & ~static_cast<int64_t>(15);
      ltid = g.tid - 32;
      ln = g.n - 32;
    }
    if (g.tid == 0 && done > 0) {
      const int T = g.copy_stage ? g.copy_stage : 3 * P.tile_bytes, ST = P.tma_stages;
      const int64_t ntiles = (done + T - 1) / T;
      const uint32_t base = *reinterpret_cast<volatile uint32_t*>(g.tiles);
      auto buf = [&](uint32_t stage) { return g.smem + static_cast<int64_t>(stage) * T; };
      auto issue = [&](int64_t i) {
        const uint32_t stg = (base + static_cast<uint32_t>(i)) % ST;
        const uint32_t len = static_cast<uint32_t>(lmin(T, done - i * T));
        mbar_expect(&g.bars[stg], len);
        bulk_load(buf(stg), src + i * T, len, &g.bars[stg]);
      };
      for (int64_t i = 0; i < ntiles && i < ST; ++i) issue(i);
      for (int64_t i = 0; i < ntiles; ++i) {
        const uint32_t gi = base + static_cast<uint32_t>(i);
        const uint32_t stg = gi % ST;
        mbar_wait(&g.bars[stg], (gi / ST) & 1u);
        bulk_store(dst + i * T, buf(stg), static_cast<uint32_t>(lmin(T, done - i * T)));
        bulk_commit();
        if (i >= 1 && i - 1 + ST < ntiles) {
          bulk_wait_read1();  // tile i-1's store has read its stage
          issue(i - 1 + ST);
        }
      }
      bulk_wait_all();
      *reinterpret_cast<volatile uint32_t*>(g.tiles) = base + static_cast<uint32_t>(ntiles);
    }
  }
  const int64_t units = (nbytes + 15) >> 4, whole = nbytes >> 4;
  if (ltid < 0) return;  // TMA driver warp
  int64_t u0 = (done >> 4) + ltid;
  if (al) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (; u0 + static_cast<int64_t>(U - 1) * ln < whole; u0 += static_cast<int64_t>(ln) * U) {
      uint4 v[U];
#pragma unroll
      for (int k = 0; k < U; ++k) v[k] = s4[u0 + static_cast<int64_t>(k) * ln];
#pragma unroll
      for (int k = 0; k < U; ++k) d4[u0 + static_cast<int64_t>(k) * ln] = v[k];
    }
  }
  for (int64_t u = u0; u < units; u += ln) {
    const int nb = static_cast<int>(lmin(16, nbytes - u * 16));
    store_user(dst + u * 16, load_user(src + u * 16, nb, al), nb, al);
  }
}

// ---------------------------------------------------------- decomposition --
// Shared with oracle/coll_oracle.c (lagom_piece_plan): a block of B elements
// is cut into NC channel slices of whole 16 B packs, and each slice into
// pieces of C / elem_bytes elements. Every element's route — and so its
// reduction order — depends only on the block it belongs to.
struct Slice {
  int64_t lo, hi;
};
__device__ __forceinline__ Slice channel_slice(int64_t B, int E, int nch, int ch) {
  const int64_t pack = 16 / E;
  const int64_t packs = (B + pack - 1) / pack;
  const int64_t per = (packs + nch - 1) / nch;
  Slice s;
  s.lo = lmin(B, static_cast<int64_t>(ch) * per * pack);
  s.hi = lmin(B, static_cast<int64_t>(ch + 1) * per * pack);
  return s;
}
// AllReduce ring block: ceil(N / n) rounded up to whole packs.
__device__ __forceinline__ int64_t ring_block(int64_t N, int n, int E) {
  const int64_t pack = 16 / E;
  const int64_t per = (N + n - 1) / n;
  return (per + pack - 1) / pack * pack;
}

// ------------------------------------------------------------- algorithms --
template <class Link>
__device__ __forceinline__ void persist(const Grp& g, const Link& l) {
  if (g.tid == 0) *l.step_home = l.step;
}

// Ring AllGather: block r travels r -> r+1 -> ... (n-1 steps).
template <int PROTO>
__device__ void ring_allgather(const Grp& g, const KParams& P, int r, int ch, int nch) {
  const int n = P.nranks, E = P.elem_bytes;
  const int64_t B = P.count, ce = P.chunk_bytes / E;
  const char* send = P.send[P.rank < 0 ? r : 0];
  char* recv = P.recv[P.rank < 0 ? r : 0];
  const Slice sl = channel_slice(B, E, nch, ch);
  if (n == 1) {
    group_copy(g, P, send + sl.lo * E, recv + sl.lo * E, (sl.hi - sl.lo) * E);
    return;
  }
  RecvLink in = make_recv(P, r, ch, (r + n - 1) % n);
  SendLink out = make_send(P, r, ch, (r + 1) % n);
  for (int64_t off = sl.lo; off < sl.hi; off += ce) {
    const int64_t nb = lmin(ce, sl.hi - off) * E;
    if (!step<PROTO, NoRed, 0, true, true, 1>(g, P, &in, &out, send + off * E, recv + (r * B + off) * E, nb)) return;
    for (int s = 1; s < n - 1; ++s) {
      const int k = (r - s + n) % n;
      if (!step<PROTO, NoRed, 1, false, true, 1>(g, P, &in, &out, nullptr, recv + (k * B + off) * E, nb)) return;
    }
    const int k = (r + 1) % n;
    if (!step<PROTO, NoRed, 1, false, true, 0>(g, P, &in, &out, nullptr, recv + (k * B + off) * E, nb)) return;
  }
  persist(g, in);
  persist(g, out);
}

// Ring ReduceScatter: the partial of block k starts at rank k+1 and ends,
// fully reduced, at rank k (n-1 steps). Order: x_{k+1}, then + x_{k+2}, ...
template <int PROTO, class R>
__device__ void ring_reducescatter(const Grp& g, const KParams& P, int r, int ch, int nch) {
  const int n = P.nranks, E = P.elem_bytes;
  const int64_t B = P.count, ce = P.chunk_bytes / E;
  const char* send = P.send[P.rank < 0 ? r : 0];
  char* recv = P.recv[P.rank < 0 ? r : 0];
  const Slice sl = channel_slice(B, E, nch, ch);
  if (n == 1) {
    group_copy(g, P, send + sl.lo * E, recv + sl.lo * E, (sl.hi - sl.lo) * E);
    return;
  }
  RecvLink in = make_recv(P, r, ch, (r + n - 1) % n);
  SendLink out = make_send(P, r, ch, (r + 1) % n);
  for (int64_t off = sl.lo; off < sl.hi; off += ce) {
    const int64_t nb = lmin(ce, sl.hi - off) * E;
    int k = (r + n - 1) % n;
    if (!step<PROTO, R, 0, true, false, 1>(g, P, &in, &out, send + (k * B + off) * E, nullptr, nb)) return;
    for (int s = 1; s < n - 1; ++s) {
      k = (r - s - 1 + 2 * n) % n;
      if (!step<PROTO, R, 1, true, false, 1>(g, P, &in, &out, send + (k * B + off) * E, nullptr, nb)) return;
    }
    if (!step<PROTO, R, 1, true, true, 0>(g, P, &in, &out, send + (r * B + off) * E, recv + off * E, nb)) return;
  }
  persist(g, in);
  persist(g, out);
}

// Ring AllReduce = ring ReduceScatter over n blocks of ring_block() elements
// fused with ring AllGather of the reduced blocks (2(n-1) steps).
template <int PROTO, class R>
__device__ void ring_allreduce(const Grp& g, const KParams& P, int r, int ch, int nch) {
  const int n = P.nranks, E = P.elem_bytes;
  const int64_t N = P.count, ce = P.chunk_bytes / E;
  const char* send = P.send[P.rank < 0 ? r : 0];
  char* recv = P.recv[P.rank < 0 ? r : 0];
  if (n == 1) {
    const Slice sl = channel_slice(N, E, nch, ch);
    group_copy(g, P, send + sl.lo * E, recv + sl.lo * E, (sl.hi - sl.lo) * E);
    return;
  }
  const int64_t B = ring_block(N, n, E);
  const Slice sl = channel_slice(B, E, nch, ch);
  RecvLink in = make_recv(P, r, ch, (r + n - 1) % n);
  SendLink out = make_send(P, r, ch, (r + 1) % n);
  auto bytes_of = [&](int k, int64_t off, int64_t len) -> int64_t {
    const int64_t valid = lmin(lmax(N - k * B, 0), B);
    return lmax(0, lmin(len, valid - off)) * E;
  };
  for (int64_t off = sl.lo; off < sl.hi; off += ce) {
    const int64_t len = lmin(ce, sl.hi - off);
    int k = (r + n - 1) % n;
    if (!step<PROTO, R, 0, true, false, 1>(g, P, &in, &out, send + (k * B + off) * E, nullptr, bytes_of(k, off, len))) return;
    for (int s = 1; s < n - 1; ++s) {
      k = (r - s - 1 + 2 * n) % n;
      if (!step<PROTO, R, 1, true, false, 1>(g, P, &in, &out, send + (k * B + off) * E, nullptr, bytes_of(k, off, len))) return;
    }
    k = r;
    if (!step<PROTO, R, 1, true, true, 1>(g, P, &in, &out, send + (k * B + off) * E, recv + (k * B + off) * E, bytes_of(k, off, len))) return;
    for (int s = 1; s < n - 1; ++s) {
      k = (r - s + n) % n;
      if (!step<PROTO, R, 1, false, true, 1>(g, P, &in, &out, nullptr, recv + (k * B + off) * E, bytes_of(k, off, len))) return;
    }
    k = (r + 1) % n;
    if (!step<PROTO, R, 1, false, true, 0>(g, P, &in, &out, nullptr, recv + (k * B + off) * E, bytes_of(k, off, len))) return;
  }
  persist(g, in);
  persist(g, out);
}

// Tree AllReduce over a binary tree (parent (r-1)/2, children 2r+1, 2r+2).
// Half the CTA reduces up (children + own -> parent; the root writes the
// result and starts the broadcast), the other half broadcasts down, so the
// two directions pipeline against each other. Order at a node:
// own, then + child 2r+1, then + child 2r+2.
template <int PROTO, class R, int NC_>
__device__ bool tree_up(const Grp& g, const KParams& P, int r, RecvLink* kids, SendLink* up,
                        SendLink* down, const char* send, char* recv, int64_t off, int64_t nb) {
  const int E = P.elem_bytes;
  if (r == 0)
    return step<PROTO, R, NC_, true, true, NC_>(g, P, kids, down, send + off * E, recv + off * E, nb);
  return step<PROTO, R, NC_, true, false, 1>(g, P, kids, up, send + off * E, nullptr, nb);
}
template <int PROTO, class R, int NC_>
__device__ bool tree_down(const Grp& g, const KParams& P, RecvLink* parent, SendLink* kids,
                          char* recv, int64_t off, int64_t nb) {
  return step<PROTO, R, 1, false, true, NC_>(g, P, parent, kids, nullptr, recv + off * P.elem_bytes, nb);
}

template <int PROTO, class R>
__device__ void tree_allreduce(const KParams& P, int r, int ch, int nch, volatile int* aborts,
                               unsigned char* smem, uint64_t (*bars)[16], uint64_t (*reds)[16],
                               uint32_t* tiles, uint32_t* redpar) {
  const int n = P.nranks, E = P.elem_bytes;
  const int64_t N = P.count, ce = P.chunk_bytes / E;
  const char* send = P.send[P.rank < 0 ? r : 0];
  char* recv = P.recv[P.rank < 0 ? r : 0];
  const Slice sl = channel_slice(N, E, nch, ch);
  if (n == 1) {
    Grp all{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x), 1, aborts};
    if (smem) {  // the whole ring (both halves' buffers) for the copy
      all.smem = smem;
      all.bars = bars[0];
      all.tiles = tiles;
      all.copy_stage = 6 * P.tile_bytes;
    }
    group_copy(all, P, send + sl.lo * E, recv + sl.lo * E, (sl.hi - sl.lo) * E);
    return;
  }
  const int half = blockDim.x / 2;
  const bool is_up = static_cast<int>(threadIdx.x) < half;
  // Each half has its own abort word: a flag raised by the other half must
  // not be observed mid-way between one half's barrier and its check.
  Grp g{is_up ? static_cast<int>(threadIdx.x) : static_cast<int>(threadIdx.x) - half, half,
        is_up ? 1 : 2, aborts + (is_up ? 0 : 1)};
  if (smem) {  // each half owns half of the TMA tile ring
    const int gi = is_up ? 0 : 1;
    g.smem = smem + static_cast<int64_t>(gi) * P.tma_stages * 3 * P.tile_bytes;
    g.bars = bars[gi];
    g.reds = reds[gi];
    g.tiles = tiles + gi;
    g.redpar = redpar + gi;
  }
  const int nkids = (2 * r + 1 < n) + (2 * r + 2 < n);
  RecvLink kin[2];
  SendLink kout[2];
  for (int i = 0; i < nkids; ++i) {
    if (is_up) kin[i] = make_recv(P, r, ch, 2 * r + 1 + i);
    if (is_up ? r == 0 : true) kout[i] = make_send(P, r, ch, 2 * r + 1 + i);
  }
  if (is_up) {
    SendLink up;
    if (r > 0) up = make_send(P, r, ch, (r - 1) / 2);
    for (int64_t off = sl.lo; off < sl.hi; off += ce) {
      const int64_t nb = lmin(ce, sl.hi - off) * E;
      bool ok = nkids == 0   ? tree_up<PROTO, R, 0>(g, P, r, kin, &up, kout, send, recv, off, nb)
                : nkids == 1 ? tree_up<PROTO, R, 1>(g, P, r, kin, &up, kout, send, recv, off, nb)
                             : tree_up<PROTO, R, 2>(g, P, r, kin, &up, kout, send, recv, off, nb);
      if (!ok) return;
    }
    for (int i = 0; i < nkids; ++i) {
      persist(g, kin[i]);
      if (r == 0) persist(g, kout[i]);
    }
    if (r > 0) persist(g, up);
  } else if (r > 0) {
    RecvLink par = make_recv(P, r, ch, (r - 1) / 2);
    for (int64_t off = sl.lo; off < sl.hi; off += ce) {
      const int64_t nb = lmin(ce, sl.hi - off) * E;
      bool ok = nkids == 0   ? tree_down<PROTO, R, 0>(g, P, &par, kout, recv, off, nb)
                : nkids == 1 ? tree_down<PROTO, R, 1>(g, P, &par, kout, recv, off, nb)
                             : tree_down<PROTO, R, 2>(g, P, &par, kout, recv, off, nb);
      if (!ok) return;
    }
    persist(g, par);
    for (int i = 0; i < nkids; ++i) persist(g, kout[i]);
  }
}

// AllToAll: per piece, copy the own block locally, then for p = 1..n-1 send
// block (r+p) to rank r+p and receive block (r-p) from rank r-p.
template <int PROTO>
__device__ void alltoall(const Grp& g, const KParams& P, int r, int ch, int nch) {
  const int n = P.nranks, E = P.elem_bytes;
  const int64_t B = P.count, ce = P.chunk_bytes / E;
  const char* send = P.send[P.rank < 0 ? r : 0];
  char* recv = P.recv[P.rank < 0 ? r : 0];
  const Slice sl = channel_slice(B, E, nch, ch);
  SendLink out[LAGOM_MAX_RANKS];
  RecvLink in[LAGOM_MAX_RANKS];
  for (int p = 1; p < n; ++p) {
    out[p] = make_send(P, r, ch, (r + p) % n);
    in[p] = make_recv(P, r, ch, (r - p + n) % n);
  }
  for (int64_t off = sl.lo; off < sl.hi; off += ce) {
    const int64_t nb = lmin(ce, sl.hi - off) * E;
    group_copy(g, P, send + (r * B + off) * E, recv + (r * B + off) * E, nb);
    for (int p = 1; p < n; ++p) {
      const int d = (r + p) % n, s = (r - p + n) % n;
      if (!step<PROTO, NoRed, 0, true, false, 1>(g, P, nullptr, &out[p], send + (d * B + off) * E, nullptr, nb)) return;
      if (!step<PROTO, NoRed, 1, false, true, 0>(g, P, &in[p], nullptr, nullptr, recv + (s * B + off) * E, nb)) return;
    }
  }
  for (int p = 1; p < n; ++p) {
    persist(g, out[p]);
    persist(g, in[p]);
  }
}

// ----------------------------------------------------------------- kernel --
enum Kind { kRingAG = 0, kRingRS = 1, kRingAR = 2, kTreeAR = 3, kA2A = 4 };

template <int KIND, int PROTO, class R>
__global__ void __launch_bounds__(640) coll_kernel(const __grid_constant__ KParams P) {
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  __shared__ int s_abort[2];
  __shared__ uint64_t s_bars[2][16];
  __shared__ uint64_t s_reds[2][16];
  __shared__ uint32_t s_tiles[2];
  __shared__ uint32_t s_redpar[2];
  constexpr bool kTma = PROTO == LAGOM_SIMPLE;
  if (threadIdx.x < 2) {
    s_abort[threadIdx.x] = 0;
    s_tiles[threadIdx.x] = 0;
    s_redpar[threadIdx.x] = 0;
  }
  if (kTma && P.tma && threadIdx.x == 0) {
    // consumer warps per group: all warps but the producer's (tree: per half)
    const int gwarps = (KIND == kTreeAR ? static_cast<int>(blockDim.x) / 2 : static_cast<int>(blockDim.x)) / 32;
    for (int g = 0; g < 2; ++g)
      for (int s = 0; s < P.tma_stages; ++s) {
        mbar_init(&s_bars[g][s]);
        mbar_init_count(&s_reds[g][s], gwarps > 1 ? static_cast<uint32_t>(gwarps - 1) : 1u);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x == 0 && P.span) atomicMin(P.span, static_cast<unsigned long long>(globaltimer()));
  __syncthreads();
  const int r = P.rank < 0 ? static_cast<int>(blockIdx.y) : P.rank;
  const int ch = blockIdx.x, nch = gridDim.x;
  Grp all{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x), 1, s_abort};
  unsigned char* tma_smem = (kTma && P.tma) ? dyn_smem : nullptr;
  if (tma_smem) {
    all.smem = tma_smem;
    all.bars = s_bars[0];
    all.reds = s_reds[0];
    all.tiles = s_tiles;
    all.redpar = s_redpar;
  }
  if constexpr (KIND == kRingAG) ring_allgather<PROTO>(all, P, r, ch, nch);
  else if constexpr (KIND == kRingRS) ring_reducescatter<PROTO, R>(all, P, r, ch, nch);
  else if constexpr (KIND == kRingAR) ring_allreduce<PROTO, R>(all, P, r, ch, nch);
  else if constexpr (KIND == kTreeAR) tree_allreduce<PROTO, R>(P, r, ch, nch, s_abort, tma_smem, s_bars, s_reds, s_tiles, s_redpar);
  else alltoall<PROTO>(all, P, r, ch, nch);
  if (P.span) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(P.span + 1, static_cast<unsigned long long>(globaltimer()));
  }
}

}  // namespace lagom_dev
