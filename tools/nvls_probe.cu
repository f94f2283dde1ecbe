// Does this box support NVLink multicast (NVLS)? Prints the device attribute
// and the multicast granularity; tries a single-process multicast object over
// all visible GPUs, binds memory, and runs multimem.ld_reduce / multimem.st.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)

__global__ void nvls_allreduce(float* mc, size_t n, int rank, int nranks) {
  // each rank reduces its 1/nranks slice through the switch and multicasts it back
  size_t per = n / nranks, lo = per * rank;
  for (size_t i = lo + (blockIdx.x * blockDim.x + threadIdx.x) * 4; i < lo + per; i += (size_t)gridDim.x * blockDim.x * 4) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + i) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(mc + i), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
  }
}

int main() {
  CK(cuInit(0));
  int ndev = 0;
  CK(cuDeviceGetCount(&ndev));
  for (int d = 0; d < ndev; ++d) {
    CUdevice dev; CK(cuDeviceGet(&dev, d));
    int mc = 0; CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("device %d multicast_supported=%d\n", d, mc);
  }
  if (ndev < 2) return 0;
  CUmulticastObjectProp prop = {};
  prop.numDevices = ndev;
  prop.size = 0;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  prop.size = 64 << 20;
  CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("multicast granularity %zu\n", gran);
  prop.size = ((64ull << 20) + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mch;
  CK(cuMulticastCreate(&mch, &prop));
  std::vector<CUcontext> ctx(ndev);
  for (int d = 0; d < ndev; ++d) { CUdevice dev; CK(cuDeviceGet(&dev, d)); CK(cuMulticastAddDevice(mch, dev)); CK(cuDevicePrimaryCtxRetain(&ctx[d], dev)); }
  std::vector<CUdeviceptr> uc(ndev), mcva(ndev);
  for (int d = 0; d < ndev; ++d) {
    CK(cuCtxSetCurrent(ctx[d]));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle mh;
    CK(cuMemCreate(&mh, prop.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mh, 0, prop.size, 0));
    CUmemAccessDesc acc = {}; acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc.location.id = d; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemAddressReserve(&uc[d], prop.size, gran, 0, 0));
    CK(cuMemMap(uc[d], prop.size, 0, mh, 0));
    CK(cuMemSetAccess(uc[d], prop.size, &acc, 1));
    CK(cuMemAddressReserve(&mcva[d], prop.size, gran, 0, 0));
    CK(cuMemMap(mcva[d], prop.size, 0, mch, 0));
    CK(cuMemSetAccess(mcva[d], prop.size, &acc, 1));
    std::vector<float> h(prop.size / 4, (float)(d + 1));
    CK(cuMemcpyHtoD(uc[d], h.data(), prop.size));
  }
  size_t n = prop.size / 4;
  for (int d = 0; d < ndev; ++d) { CK(cuCtxSetCurrent(ctx[d])); nvls_allreduce<<<132, 512>>>((float*)mcva[d], n, d, ndev); }
  for (int d = 0; d < ndev; ++d) { CK(cuCtxSetCurrent(ctx[d])); CK(cuCtxSynchronize()); }
  float want = ndev * (ndev + 1) / 2.0f;
  for (int d = 0; d < ndev; ++d) {
    CK(cuCtxSetCurrent(ctx[d]));
    std::vector<float> h(n); CK(cuMemcpyDtoH(h.data(), uc[d], prop.size));
    size_t bad = 0; for (float v : h) bad += v != want;
    printf("device %d: %zu of %zu elements != %.0f\n", d, bad, n, want);
  }
  // bandwidth: 256 MiB... reuse 64 MiB, 20 iterations
  cudaEvent_t e0, e1; CK(cuCtxSetCurrent(ctx[0])); cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it)
    for (int d = 0; d < ndev; ++d) { CK(cuCtxSetCurrent(ctx[d])); nvls_allreduce<<<32, 512>>>((float*)mcva[d], n, d, ndev); }
  CK(cuCtxSetCurrent(ctx[0])); cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it)
    for (int d = 0; d < ndev; ++d) { CK(cuCtxSetCurrent(ctx[d])); nvls_allreduce<<<32, 512>>>((float*)mcva[d], n, d, ndev); }
  for (int d = 0; d < ndev; ++d) { CK(cuCtxSetCurrent(ctx[d])); CK(cuCtxSynchronize()); }
  CK(cuCtxSetCurrent(ctx[0])); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double S = prop.size, t = ms / 20 * 1e-3;
  printf("NVLS allreduce 32 CTAs/GPU, %zu MiB: %.1f us, algbw %.1f GB/s, busbw %.1f GB/s (no inter-GPU sync: indicative)\n",
         prop.size >> 20, t * 1e6, S / t / 1e9, S / t * 2.0 * (ndev - 1) / ndev / 1e9);
  return 0;
}
