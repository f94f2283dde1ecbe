// Deterministic on-device synthetic data (replay-engine weights/activations
// and collective payloads). Counter-based: value(i) = hash(seed, i).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "lagom_coll.h"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void fill_kernel(void* p, int64_t n, int dtype, uint64_t seed, float scale) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h = mix64(seed * 0x100000001b3ull + static_cast<uint64_t>(i));
    const float u = static_cast<float>(h >> 40) * (1.0f / 16777216.0f);  // [0, 1)
    const float v = (2.0f * u - 1.0f) * scale;
    switch (dtype) {
      case LAGOM_F32: static_cast<float*>(p)[i] = v; break;
      case LAGOM_BF16: static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v); break;
      case LAGOM_F16: static_cast<__half*>(p)[i] = __float2half_rn(v); break;
      default: static_cast<int32_t*>(p)[i] = static_cast<int32_t>(h >> 43) - (1 << 20); break;
    }
  }
}

}  // namespace

extern "C" int lagom_fill_random(void* ptr, int64_t nelems, int dtype, uint64_t seed, float scale,
                                 void* stream) {
  if (nelems <= 0) return LAGOM_OK;
  if (!ptr || dtype < LAGOM_F32 || dtype > LAGOM_I32) return LAGOM_ERR_INVALID_ARGUMENT;
  const int64_t blocks64 = (nelems + 255) / 256;
  const int blocks = static_cast<int>(blocks64 < 148 * 16 ? blocks64 : 148 * 16);
  fill_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, nelems, dtype, seed, scale);
  return cudaGetLastError() == cudaSuccess ? LAGOM_OK : LAGOM_ERR_CUDA;
}

namespace {
__global__ void timestamp_kernel(unsigned long long* dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  *dst = t;
}
}  // namespace

extern "C" int lagom_timestamp(void* dst, void* stream) {
  if (!dst) return LAGOM_ERR_INVALID_ARGUMENT;
  timestamp_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<unsigned long long*>(dst));
  return cudaGetLastError() == cudaSuccess ? LAGOM_OK : LAGOM_ERR_CUDA;
}
