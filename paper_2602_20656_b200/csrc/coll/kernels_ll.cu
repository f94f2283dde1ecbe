// LAGOM_LL instantiations of the collective-kernel family (see device.cuh).
#include "dispatch.cuh"

const void* lagom_pick_ll(int kind, int dtype, int op) {
  return lagom_dev::pick_proto<LAGOM_LL>(kind, dtype, op);
}
