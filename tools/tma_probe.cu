// Per-CTA NVLink throughput with 1-D TMA bulk copies (cp.async.bulk) vs LSU
// vector copies. Single process, 2 GPUs (peer access). One elected thread per
// CTA drives an S-stage smem ring: bulk load (mbarrier complete_tx) -> bulk
// store (bulk_group). Modes: push (local -> peer), pull (peer -> local),
// local (local -> local).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(dst_smem)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(dst), "r"(smem_addr(src_smem)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int S>
__global__ void tma_copy(const char* __restrict__ src, char* __restrict__ dst, size_t bytes, uint32_t tile) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t per_cta = (bytes / gridDim.x) / tile * tile;
  const char* s0 = src + per_cta * blockIdx.x;
  char* d0 = dst + per_cta * blockIdx.x;
  const size_t n = per_cta / tile;
  for (size_t i = 0; i < n && i < S; ++i) {
    mbar_expect(&bars[i], tile);
    bulk_load(smem + i * tile, s0 + i * tile, tile, &bars[i]);
  }
  for (size_t i = 0; i < n; ++i) {
    const int s = static_cast<int>(i % S);
    mbar_wait(&bars[s], static_cast<uint32_t>((i / S) & 1));
    bulk_store(d0 + i * tile, smem + s * tile, tile);
    if (i >= 1 && i - 1 + S < n) {
      bulk_wait_read<1>();  // store i-1 has finished reading its buffer
      const int sp = static_cast<int>((i - 1) % S);
      mbar_expect(&bars[sp], tile);
      bulk_load(smem + sp * tile, s0 + (i - 1 + S) * tile, tile, &bars[sp]);
    }
  }
  bulk_wait_all();
}

template <int U>
__global__ void lsu_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n_units) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t base = ((size_t)blockIdx.x * blockDim.x) * U + threadIdx.x; base < n_units; base += stride) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      size_t i = base + (size_t)k * blockDim.x;
      if (i < n_units) v[k] = src[i];
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      size_t i = base + (size_t)k * blockDim.x;
      if (i < n_units) dst[i] = v[k];
    }
  }
}

template <typename F>
float timeit(F f, size_t bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return -1; }
  return (float)(bytes * 5.0 / (ms * 1e-3) / 1e9);
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = 1ull << 30;
  void *a0, *b0, *a1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMemset(a1, 1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 2, bytes));
  const int smem_max = 200 * 1024;
  CK(cudaFuncSetAttribute(tma_copy<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
  CK(cudaFuncSetAttribute(tma_copy<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
  printf("mode,engine,grid,tile_or_block,stages_or_unroll,GBps,GBps_per_cta\n");
  const char* names[3] = {"push", "pull", "local"};
  const char* srcs[3] = {(const char*)a0, (const char*)a1, (const char*)a0};
  char* dsts[3] = {(char*)a1, (char*)b0, (char*)b0};
  for (int mode = 0; mode < 3; ++mode)
    for (int g : {1, 2, 4, 8, 16, 32}) {
      for (uint32_t tile : {8192u, 16384u, 24576u, 49152u}) {
        if (tile * 4 <= (uint32_t)smem_max) {
          float r = timeit([&] { tma_copy<4><<<g, 32, tile * 4>>>(srcs[mode], dsts[mode], bytes, tile); }, bytes);
          printf("%s,tma,%d,%u,4,%.1f,%.1f\n", names[mode], g, tile, r, r / g);
        }
        if (tile * 8 <= (uint32_t)smem_max) {
          float r = timeit([&] { tma_copy<8><<<g, 32, tile * 8>>>(srcs[mode], dsts[mode], bytes, tile); }, bytes);
          printf("%s,tma,%d,%u,8,%.1f,%.1f\n", names[mode], g, tile, r, r / g);
        }
      }
      float r = timeit([&] { lsu_copy<8><<<g, 640>>>((const uint4*)srcs[mode], (uint4*)dsts[mode], bytes / 16); }, bytes);
      printf("%s,lsu,%d,640,8,%.1f,%.1f\n", names[mode], g, r, r / g);
    }
  return 0;
}
