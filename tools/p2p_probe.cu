// NVLink peer-memory probe (single process, 2 GPUs, cudaDeviceEnablePeerAccess):
// per-CTA push (local ld -> peer st) and pull (peer ld -> local st) bandwidth
// as a function of CTAs, threads and unroll. Used to size the collective
// kernels' inner loops. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe p2p_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U, int MODE>
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n_units) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t base = ((size_t)blockIdx.x * blockDim.x) * U + threadIdx.x; base < n_units; base += stride) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      size_t i = base + (size_t)k * blockDim.x;
      if (i < n_units) v[k] = MODE == 1 ? __ldcg(src + i) : src[i];
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      size_t i = base + (size_t)k * blockDim.x;
      if (i < n_units) {
        if (MODE == 2) __stcg(dst + i, v[k]);
        else if (MODE == 3) __stwt(dst + i, v[k]);
        else dst[i] = v[k];
      }
    }
  }
}

template <int U, int MODE>
float run(const uint4* src, uint4* dst, size_t units, int grid, int block) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  copy_kernel<U, MODE><<<grid, block>>>(src, dst, units);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) copy_kernel<U, MODE><<<grid, block>>>(src, dst, units);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return (float)(units * 16.0 * 5 / (ms * 1e-3) / 1e9);
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = 1ull << 30, units = bytes / 16;
  void *a0, *b0, *a1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMemset(a1, 1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 2, bytes));
  const int grids[] = {1, 4, 16, 32, 64, 148, 296};
  const int blocks[] = {256, 512, 640};
  printf("mode,grid,block,unroll,GBps\n");
  for (int g : grids)
    for (int bl : blocks) {
      printf("push_st,%d,%d,4,%.1f\n", g, bl, run<4, 0>((uint4*)a0, (uint4*)a1, units, g, bl));
      printf("push_st,%d,%d,8,%.1f\n", g, bl, run<8, 0>((uint4*)a0, (uint4*)a1, units, g, bl));
      printf("push_stcg,%d,%d,8,%.1f\n", g, bl, run<8, 2>((uint4*)a0, (uint4*)a1, units, g, bl));
      printf("pull_ld,%d,%d,4,%.1f\n", g, bl, run<4, 0>((uint4*)a1, (uint4*)b0, units, g, bl));
      printf("pull_ld,%d,%d,8,%.1f\n", g, bl, run<8, 0>((uint4*)a1, (uint4*)b0, units, g, bl));
      printf("pull_ldcg,%d,%d,16,%.1f\n", g, bl, run<16, 1>((uint4*)a1, (uint4*)b0, units, g, bl));
      printf("local,%d,%d,8,%.1f\n", g, bl, run<8, 0>((uint4*)a0, (uint4*)b0, units, g, bl));
    }
  CK(cudaDeviceSynchronize());
  printf("cudaMemcpyPeer:");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf(" %.1f GB/s\n", bytes * 5.0 / (ms * 1e-3) / 1e9);
  return 0;
}
