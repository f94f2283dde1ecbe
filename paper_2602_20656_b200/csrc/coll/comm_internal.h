// Internal: the communicator object shared by comm.cu and nvls.cu.
#pragma once
#include <cstdint>
#include <string>

#include "lagom_coll.h"

// Stamps per channel and launch recorded by the switch kernels when
// LAGOM_PHASE_STAMPS=1 (lagom_comm_phase_stamps): entry, entry barrier done,
// data done, fence done, exit barrier done, epoch.
constexpr int LAGOM_PHASE_STAMPS = 8;

struct lagom_comm {
  int rank = 0;
  int nranks = 1;
  int device = 0;
  bool virt = false;
  bool ready = false;
  lagom_comm_opts_t opts{};

  int64_t slot_bytes = 0;
  int64_t off_ready = 0, off_freed = 0, off_sstep = 0, off_rstep = 0, off_slots = 0;
  int64_t heap_bytes = 0;
  char* heap[LAGOM_MAX_RANKS] = {};  // mapped bases (own + peers / all virtual ranks)
  bool imported[LAGOM_MAX_RANKS] = {};
  unsigned int* abort_host = nullptr;
  unsigned int* abort_dev = nullptr;
  bool broken = false;
  void* order_ev = nullptr;                 // cudaEvent_t: the last launch (issue order)
  int64_t off_hdr = 0;                      // heap header: options peers must agree on
  // NVLS (NVLink SHARP multicast): a symmetric region bound to a multicast
  // object spanning every rank's GPU (nvls.cu).
  unsigned long long nvls_mc_handle = 0;    // CUmemGenericAllocationHandle (multicast)
  unsigned long long nvls_mem_handle = 0;   // CUmemGenericAllocationHandle (physical)
  char* nvls_uc = nullptr;                  // unicast mapping of this rank's memory
  char* nvls_mc = nullptr;                  // multicast mapping (all ranks)
  int64_t nvls_bytes = 0;
  int64_t nvls_used = 0;
  char* nvls_scratch = nullptr;             // push-based one-hop RS: n slots of scratch_slot bytes
  int64_t nvls_scratch_slot = 0;
  bool nvls_ready = false;
  int64_t off_nvbar = 0, off_nvep = 0;      // NVLS barrier flags / epochs in the heap
  int64_t off_nvpiece = 0, off_nvpbase = 0; // push RS piece flags / per-channel piece counts
  int64_t off_phase = 0;                    // phase stamps of the switch kernels (diagnostics)
  int phase_stamps = 0;                     // LAGOM_PHASE_STAMPS=1 at creation: kernels record them
  int nvls_export_fd = -1;                  // rank 0's exported fd, closed once bound
  // Peer (unicast) mappings of every rank's region: one-hop AllToAll writes
  // straight into the destination rank's recv buffer.
  char* nvls_peer[LAGOM_MAX_RANKS] = {};    // own entry = nvls_uc
  bool nvls_peers_mapped = false;          // every peer region mapped here
  bool nvls_peers_ready = false;           // ... and agreed on by all ranks (use_peers)
  int nvls_peer_fd = -1;                    // this rank's exported physical-memory fd
};

// Records `what` as lagom_last_error() and returns `status`.
int lagom_fail(int status, const std::string& what);
// One launch, decided but not issued: kernel (nullptr = nothing to launch),
// its single by-value parameter block, dynamic shared memory.
struct LaunchPlan {
  const void* kernel = nullptr;
  alignas(16) unsigned char params[512];
  int smem = 0;
};
// nranks == 1: the copy kernel of local.cu (no launch in place).
int lagom_local_select(const lagom_comm* c, const lagom_coll_args_t* a, const void* send, void* recv,
                       LaunchPlan* plan);
