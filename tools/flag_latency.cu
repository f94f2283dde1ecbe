// How long does a cross-GPU flag barrier take over NVLink / NVSwitch?
// One process, every visible GPU, peer access enabled; one kernel per GPU
// (launched concurrently) runs K barriers in a row among all GPUs, each
// barrier the all-to-all flag exchange of the switch kernels (nvls.cu
// nv_barrier) in several variants:
//   0 serial:   thread 0 posts to every peer with st.release.sys, then polls
//               each peer's flag with ld.acquire.sys      (round-1 form)
//   1 parallel: thread t < n-1 posts to one peer (fence.acq_rel.sys +
//               st.relaxed.sys), polls one flag relaxed, fences (round-2 form)
//   2 parallel, no fences (lower bound: relaxed post + relaxed poll)
//   3 parallel, volatile st / ld (st.volatile / ld.volatile)
//   4 parallel, post with red.release.sys.add (atomic) and poll relaxed
//   5 exit form: thread 0 runs one fence.acq_rel.sys for the CTA, then
//     thread t < n-1 posts relaxed and polls relaxed
//   6 entry form: relaxed post, relaxed poll, then one ld.acquire.sys of
//     the flag that was seen
//   7 parallel st.release.sys (a fence per posting thread), relaxed poll
//   8 exit form with fence.sc.sys (__threadfence_system) instead
// and with G CTAs per GPU doing independent barriers (the channels).
// Prints us per barrier (max over GPUs of the kernel time / K).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/flag_latency tools/flag_latency.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

constexpr int kMaxGpu = 8;
struct Args {
  uint64_t* flags[kMaxGpu];  // per GPU: [cta][src] flags, 128 B apart
  int me, n, iters;
};

__device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_rlx(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_vol(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rlx(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_vol(uint64_t* p, uint64_t v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_rel(uint64_t* p, uint64_t v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int MODE>
__global__ void barrier_kernel(Args a, unsigned long long* out) {
  const int n = a.n, r = a.me, g = blockIdx.x, t = threadIdx.x;
  __shared__ unsigned long long t0;
  auto flag = [&](int owner, int src) { return a.flags[owner] + (static_cast<int64_t>(g) * kMaxGpu + src) * 16; };
  if (t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  __syncthreads();
  for (int it = 1; it <= a.iters; ++it) {
    const uint64_t ep = static_cast<uint64_t>(it);
    if (MODE == 0) {
      if (t == 0) {
        for (int p = 0; p < n; ++p)
          if (p != r) st_rel(flag(p, r), ep);
        for (int p = 0; p < n; ++p)
          if (p != r)
            while (ld_acq(flag(r, p)) < ep) {
            }
      }
    } else if (MODE != 5 && MODE != 8 && t < n - 1) {
      const int p = (r + 1 + t) % n;
      if (MODE == 1) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        st_rlx(flag(p, r), ep);
        while (ld_rlx(flag(r, p)) < ep) {
        }
        asm volatile("fence.acq_rel.sys;" ::: "memory");
      } else if (MODE == 2) {
        st_rlx(flag(p, r), ep);
        while (ld_rlx(flag(r, p)) < ep) {
        }
      } else if (MODE == 3) {
        st_vol(flag(p, r), ep);
        while (ld_vol(flag(r, p)) < ep) {
        }
      } else if (MODE == 4) {
        red_rel(flag(p, r), 1);
        while (ld_rlx(flag(r, p)) < ep) {
        }
      } else if (MODE == 6) {
        st_rlx(flag(p, r), ep);
        while (ld_rlx(flag(r, p)) < ep) {
        }
        (void)ld_acq(flag(r, p));
      } else if (MODE == 7) {
        st_rel(flag(p, r), ep);
        while (ld_rlx(flag(r, p)) < ep) {
        }
      }
    }
    if (MODE == 5 || MODE == 8) {
      if (t == 0) {
        if (MODE == 5) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else __threadfence_system();
      }
      __syncthreads();
      if (t < n - 1) {
        const int p = (r + 1 + t) % n;
        st_rlx(flag(p, r), ep);
        while (ld_rlx(flag(r, p)) < ep) {
        }
      }
    }
    __syncthreads();
  }
  if (t == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    atomicMax(out, t1 - t0);
  }
}

template <int MODE>
int run(const std::vector<uint64_t*>& flags, const std::vector<unsigned long long*>& outs, int n, int grid,
        int iters, const char* name) {
  const size_t fbytes = 64 * kMaxGpu * 128;
  std::vector<cudaStream_t> st(n);
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMemset(flags[d], 0, fbytes));
    CK(cudaMemset(outs[d], 0, 8));
    CK(cudaStreamCreate(&st[d]));
  }
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceSynchronize());
  }
  for (int d = 0; d < n; ++d) {
    Args a{};
    for (int q = 0; q < n; ++q) a.flags[q] = flags[q];
    a.me = d;
    a.n = n;
    a.iters = iters;
    CK(cudaSetDevice(d));
    barrier_kernel<MODE><<<grid, 128, 0, st[d]>>>(a, outs[d]);
    CK(cudaGetLastError());
  }
  unsigned long long worst = 0;
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaStreamSynchronize(st[d]));
    unsigned long long v = 0;
    CK(cudaMemcpy(&v, outs[d], 8, cudaMemcpyDeviceToHost));
    worst = v > worst ? v : worst;
    CK(cudaStreamDestroy(st[d]));
  }
  printf("{\"gpus\": %d, \"mode\": \"%s\", \"ctas\": %d, \"iters\": %d, \"us_per_barrier\": %.3f}\n", n, name, grid,
         iters, worst / 1e3 / iters);
  return 0;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("need >= 2 GPUs\n");
    return 0;
  }
  if (n > kMaxGpu) n = kMaxGpu;
  std::vector<uint64_t*> flags(n);
  std::vector<unsigned long long*> outs(n);
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    for (int q = 0; q < n; ++q)
      if (q != d) CK(cudaDeviceEnablePeerAccess(q, 0));
    CK(cudaMalloc(&flags[d], 64 * kMaxGpu * 128));
    CK(cudaMalloc(&outs[d], 8));
  }
  const int iters = 2000;
  for (int grid : {1, 8, 64}) {
    if (run<0>(flags, outs, n, grid, iters, "serial_release_acquire")) return 1;
    if (run<1>(flags, outs, n, grid, iters, "parallel_fenced")) return 1;
    if (run<2>(flags, outs, n, grid, iters, "parallel_relaxed")) return 1;
    if (run<3>(flags, outs, n, grid, iters, "parallel_volatile")) return 1;
    if (run<4>(flags, outs, n, grid, iters, "parallel_red_release")) return 1;
    if (run<5>(flags, outs, n, grid, iters, "exit_one_fence_acq_rel")) return 1;
    if (run<6>(flags, outs, n, grid, iters, "entry_relaxed_then_acquire")) return 1;
    if (run<7>(flags, outs, n, grid, iters, "parallel_st_release")) return 1;
    if (run<8>(flags, outs, n, grid, iters, "exit_one_fence_sc")) return 1;
  }
  // the same with 2 GPUs when more are visible
  if (n > 2)
    for (int grid : {1, 8})
      if (run<1>(flags, outs, 2, grid, iters, "parallel_fenced")) return 1;
  return 0;
}
