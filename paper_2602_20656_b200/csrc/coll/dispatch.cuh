// Kernel table for one protocol: (algorithm kind, dtype, redop) -> kernel.
#pragma once
#include "device.cuh"

namespace lagom_dev {

template <int K, int P>
const void* pick_red(int dtype, int op) {
#define LAGOM_RED(T)                                                          \
  switch (op) {                                                               \
    case LAGOM_SUM: return reinterpret_cast<const void*>(&coll_kernel<K, P, Red<T, LAGOM_SUM>>); \
    case LAGOM_MAX: return reinterpret_cast<const void*>(&coll_kernel<K, P, Red<T, LAGOM_MAX>>); \
    case LAGOM_MIN: return reinterpret_cast<const void*>(&coll_kernel<K, P, Red<T, LAGOM_MIN>>); \
  }                                                                           \
  return nullptr;
  switch (dtype) {
    case LAGOM_F32: { LAGOM_RED(float) }
    case LAGOM_BF16: { LAGOM_RED(__nv_bfloat16) }
    case LAGOM_F16: { LAGOM_RED(__half) }
    case LAGOM_I32: { LAGOM_RED(int32_t) }
  }
#undef LAGOM_RED
  return nullptr;
}

template <int P>
const void* pick_proto(int kind, int dtype, int op) {
  switch (kind) {
    case kRingAG: return reinterpret_cast<const void*>(&coll_kernel<kRingAG, P, NoRed>);
    case kA2A: return reinterpret_cast<const void*>(&coll_kernel<kA2A, P, NoRed>);
    case kRingRS: return pick_red<kRingRS, P>(dtype, op);
    case kRingAR: return pick_red<kRingAR, P>(dtype, op);
    case kTreeAR: return pick_red<kTreeAR, P>(dtype, op);
  }
  return nullptr;
}

}  // namespace lagom_dev
