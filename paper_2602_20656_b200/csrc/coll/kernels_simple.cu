// LAGOM_SIMPLE instantiations of the collective-kernel family (see device.cuh).
#include "dispatch.cuh"

const void* lagom_pick_simple(int kind, int dtype, int op) {
  return lagom_dev::pick_proto<LAGOM_SIMPLE>(kind, dtype, op);
}
