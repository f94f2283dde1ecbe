// Host side of the collective C-ABI (include/lagom_coll.h): communicator
// lifetime, symmetric-heap allocation, CUDA-IPC peer mapping over
// NVLink/NVSwitch, argument validation and kernel dispatch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "device.cuh"
#include "lagom_coll.h"

using lagom_dev::KParams;

#include "comm_internal.h"

namespace {

thread_local std::string g_last_error;

int fail(int status, const std::string& what) {
  g_last_error = what;
  return status;
}
}  // namespace
int lagom_fail(int status, const std::string& what) { return fail(status, what); }
namespace {

int cuda_fail(cudaError_t e, const char* where) {
  return fail(LAGOM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define LAGOM_CUDA(call)                                  \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
  } while (0)

// Heap header: the options every rank must agree on (they select kernels
// and the heap layout), written at creation, compared at import.
struct HeapHeader {
  uint64_t magic;
  int64_t nranks, max_channels, steps, max_chunk_bytes, use_tma, coresident, one_hop, a2a_tma;
};
constexpr uint64_t kHeapMagic = 0x4c41474f4d484452ull;  // "LAGOMHDR"

HeapHeader header_of(const lagom_comm* c) {
  return HeapHeader{kHeapMagic, c->nranks, c->opts.max_channels, c->opts.steps, c->opts.max_chunk_bytes,
                    c->opts.use_tma, c->opts.coresident, c->opts.one_hop, c->opts.a2a_tma};
}

void layout(lagom_comm* c) {
  const int64_t n = c->nranks, ch = c->opts.max_channels;
  c->slot_bytes = 2 * c->opts.max_chunk_bytes;  // LL doubles the payload
  int64_t off = 0;
  c->off_hdr = off;
  off += 256;
  c->off_ready = off;
  off += ch * n * 128;
  c->off_freed = off;
  off += ch * n * 128;
  c->off_sstep = off;
  off += ch * n * 8;
  c->off_rstep = off;
  off += ch * n * 8;
  c->off_nvbar = off;  // NVLS entry/exit barrier flags [ch][src], 128 B apart
  off += ch * n * 128;
  c->off_nvep = off;   // NVLS per-channel epoch (local)
  off += ch * 8;
  c->off_nvpiece = off;  // push RS: pieces landed [ch][src], 128 B apart (written by src)
  off += ch * n * 128;
  c->off_nvpbase = off;  // push RS: pieces completed per channel so far (local)
  off += ch * 8;
  c->off_phase = off;  // diagnostics: per-channel phase stamps, 2 launches (local)
  off += ch * 2 * LAGOM_PHASE_STAMPS * 8;
  off = (off + 4095) / 4096 * 4096;
  c->off_slots = off;
  off += ch * n * c->opts.steps * c->slot_bytes;
  c->heap_bytes = off;
}

int check_opts(lagom_comm_opts_t* o) {
  if (o->max_channels < 1 || o->max_channels > LAGOM_MAX_CHANNELS)
    return fail(LAGOM_ERR_INVALID_ARGUMENT, "max_channels out of range");
  if (o->steps < 1 || o->steps > 64) return fail(LAGOM_ERR_INVALID_ARGUMENT, "steps out of range");
  if (o->max_chunk_bytes < 1024 || o->max_chunk_bytes % 1024 != 0)
    return fail(LAGOM_ERR_INVALID_ARGUMENT, "max_chunk_bytes must be a positive 1 KiB multiple");
  if (o->timeout_ms < 1) return fail(LAGOM_ERR_INVALID_ARGUMENT, "timeout_ms must be >= 1");
  if (o->use_tma < 0 || o->use_tma > 2) return fail(LAGOM_ERR_INVALID_ARGUMENT, "use_tma must be 0, 1 or 2");
  if (o->coresident < 0 || o->coresident > 1) return fail(LAGOM_ERR_INVALID_ARGUMENT, "coresident must be 0 or 1");
  if (o->one_hop < 0 || o->one_hop > 2) return fail(LAGOM_ERR_INVALID_ARGUMENT, "one_hop must be 0, 1 or 2");
  if (o->a2a_tma < 0 || o->a2a_tma > 1) return fail(LAGOM_ERR_INVALID_ARGUMENT, "a2a_tma must be 0 or 1");
  return LAGOM_OK;
}

int alloc_common(lagom_comm* c) {
  LAGOM_CUDA(cudaSetDevice(c->device));
  LAGOM_CUDA(cudaHostAlloc(&c->abort_host, sizeof(unsigned int), cudaHostAllocMapped));
  *c->abort_host = 0;
  LAGOM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->abort_dev), c->abort_host, 0));
  cudaEvent_t ev;
  LAGOM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  c->order_ev = ev;
  const char* ps = std::getenv("LAGOM_PHASE_STAMPS");
  c->phase_stamps = ps && std::atoi(ps) > 0 ? 1 : 0;
  return LAGOM_OK;
}

int elem_bytes_of(int dtype) {
  switch (dtype) {
    case LAGOM_F32: return 4;
    case LAGOM_BF16: return 2;
    case LAGOM_F16: return 2;
    case LAGOM_I32: return 4;
  }
  return 0;
}

// ------------------------------------------------------------ dispatch ----
// One translation unit per protocol (kernels_simple.cu, kernels_ll.cu,
// kernels_ll128.cu) so the 114 kernel instantiations compile in parallel.
}  // namespace
const void* lagom_pick_simple(int kind, int dtype, int op);
int lagom_nvls_prepare(const lagom_comm* c, const lagom_coll_args_t* a, const void* send, void* recv,
                       const void** kernel, void* params_out, size_t* params_bytes, int* smem_bytes);
void lagom_nvls_release(lagom_comm* c);
const void* lagom_pick_ll(int kind, int dtype, int op);
const void* lagom_pick_ll128(int kind, int dtype, int op);
namespace {

const void* pick_kernel(const lagom_coll_args_t* a) {
  using namespace lagom_dev;
  int kind = -1;
  switch (a->collective) {
    case LAGOM_ALL_GATHER: kind = kRingAG; break;
    case LAGOM_REDUCE_SCATTER: kind = kRingRS; break;
    case LAGOM_ALL_TO_ALL: kind = kA2A; break;
    case LAGOM_ALL_REDUCE: kind = a->algorithm == LAGOM_TREE ? kTreeAR : kRingAR; break;
  }
  switch (a->protocol) {
    case LAGOM_SIMPLE: return lagom_pick_simple(kind, a->dtype, a->redop);
    case LAGOM_LL: return lagom_pick_ll(kind, a->dtype, a->redop);
    case LAGOM_LL128: return lagom_pick_ll128(kind, a->dtype, a->redop);
  }
  return nullptr;
}

int validate(const lagom_comm* c, const lagom_coll_args_t* a) {
  if (!c || !a) return fail(LAGOM_ERR_INVALID_ARGUMENT, "null comm or args");
  if (a->collective < 0 || a->collective > LAGOM_ALL_TO_ALL)
    return fail(LAGOM_ERR_INVALID_ARGUMENT, "unknown collective");
  if (a->algorithm != LAGOM_RING && a->algorithm != LAGOM_TREE)
    return fail(LAGOM_ERR_INVALID_ARGUMENT, "unknown algorithm");
  if (a->protocol < LAGOM_SIMPLE || a->protocol > LAGOM_LL128)
    return fail(LAGOM_ERR_INVALID_ARGUMENT, "unknown protocol");
  if (elem_bytes_of(a->dtype) == 0) return fail(LAGOM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (a->redop < LAGOM_SUM || a->redop > LAGOM_MIN) return fail(LAGOM_ERR_INVALID_ARGUMENT, "unknown redop");
  if (a->count < 0) return fail(LAGOM_ERR_INVALID_ARGUMENT, "count must be >= 0");
  if (a->num_channels < 1 || a->num_channels > c->opts.max_channels)
    return fail(LAGOM_ERR_INVALID_CONFIG, "num_channels must lie in [1, " +
                                              std::to_string(c->opts.max_channels) + "]");
  if (a->num_threads < 64 || a->num_threads > 640 || a->num_threads % 64 != 0)
    return fail(LAGOM_ERR_INVALID_CONFIG, "num_threads must be one of {64, 128, ..., 640}");
  if (a->chunk_bytes < 1024 || a->chunk_bytes % 1024 != 0 || a->chunk_bytes > c->opts.max_chunk_bytes)
    return fail(LAGOM_ERR_INVALID_CONFIG, "chunk_size must be a 1 KiB multiple in [1 KiB, " +
                                              std::to_string(c->opts.max_chunk_bytes) + "]");
  // Tree is an AllReduce schedule (reference keys TREE/* for any collective;
  // the other collectives fall back to their ring schedule, as NCCL does).
  return LAGOM_OK;
}

constexpr int kTmaStages = 4;
constexpr int kTmaSmemBytes = 192 * 1024;

// Dynamic shared memory for the TMA tile ring; the opt-in above 48 KB is set
// once per kernel.
int smem_for(const KParams& p, const lagom_coll_args_t* a, const void* kernel) {
  if (!p.tma) return 0;
  static std::mutex mu;
  static std::vector<const void*> done;
  std::lock_guard<std::mutex> lock(mu);
  if (std::find(done.begin(), done.end(), kernel) == done.end()) {
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmemBytes) != cudaSuccess)
      return -1;
    done.push_back(kernel);
  }
  const int groups = (a->collective == LAGOM_ALL_REDUCE && a->algorithm == LAGOM_TREE) ? 2 : 1;
  return groups * kTmaStages * 3 * p.tile_bytes;
}

// TMA share of a split copy step in LSU-thread equivalents (device.cuh,
// KParams::tma_share_*); environment overrides for experiments.
int tma_share(const char* env, int dflt) {
  const char* e = std::getenv(env);
  return e ? std::max(0, std::atoi(e)) : dflt;
}

KParams make_params(const lagom_comm* c, const lagom_coll_args_t* a) {
  KParams p{};
  for (int r = 0; r < c->nranks; ++r) p.heap[r] = c->heap[r];
  p.rank = c->virt ? -1 : c->rank;
  p.nranks = c->nranks;
  p.elem_bytes = elem_bytes_of(a->dtype);
  p.steps = c->opts.steps;
  p.count = a->count;
  p.chunk_bytes = a->chunk_bytes;
  p.slot_bytes = c->slot_bytes;
  p.off_ready = c->off_ready;
  p.off_freed = c->off_freed;
  p.off_sstep = c->off_sstep;
  p.off_rstep = c->off_rstep;
  p.off_slots = c->off_slots;
  p.abort_flag = c->abort_dev;
  p.timeout_ns = static_cast<uint64_t>(c->opts.timeout_ms) * 1000000ull;
  p.span = static_cast<unsigned long long*>(a->span_out);
  p.tma = (c->opts.use_tma && a->protocol == LAGOM_SIMPLE) ? 1 : 0;
  p.tma_stages = kTmaStages;
  p.tma_reduce = c->opts.use_tma >= 2 ? 1 : 0;
  p.tma_share_local = tma_share("LAGOM_TMA_SHARE_LOCAL", 0);
  p.tma_share_push = tma_share("LAGOM_TMA_SHARE_PUSH", 0);
  // 192 KB of tile ring per CTA: 3 buffers x stages per group (2 groups for tree)
  const int groups = (a->collective == LAGOM_ALL_REDUCE && a->algorithm == LAGOM_TREE) ? 2 : 1;
  p.tile_bytes = kTmaSmemBytes / (groups * kTmaStages * 3) / 1024 * 1024;
  return p;
}

int launch_real(lagom_comm* c, const lagom_coll_args_t* a, const void* sendbuf, void* recvbuf, cudaStream_t stream);
int select_real(lagom_comm* c, const lagom_coll_args_t* a, const void* sendbuf, void* recvbuf, LaunchPlan* plan);

}  // namespace

extern "C" {

int lagom_coll_abi_version(void) { return LAGOM_COLL_ABI_VERSION; }

const char* lagom_status_string(int s) {
  switch (s) {
    case LAGOM_OK: return "ok";
    case LAGOM_ERR_INVALID_ARGUMENT: return "invalid argument";
    case LAGOM_ERR_INVALID_CONFIG: return "invalid config";
    case LAGOM_ERR_CUDA: return "cuda error";
    case LAGOM_ERR_TIMEOUT: return "peer timeout";
    case LAGOM_ERR_NOT_READY: return "peers not imported";
    case LAGOM_ERR_BROKEN: return "communicator broken by an earlier abort";
  }
  return "unknown status";
}

const char* lagom_last_error(void) { return g_last_error.c_str(); }

void lagom_comm_default_opts(lagom_comm_opts_t* o) {
  o->max_channels = 32;
  o->steps = 4;
  o->max_chunk_bytes = 4 << 20;
  o->timeout_ms = 10000;
  o->use_tma = 1;
  o->coresident = 1;
  o->one_hop = 2;
  o->a2a_tma = 1;
}

int lagom_comm_create(int rank, int nranks, int device, const lagom_comm_opts_t* opts,
                      lagom_comm_t* out) {
  if (!out) return fail(LAGOM_ERR_INVALID_ARGUMENT, "null out");
  if (nranks < 1 || nranks > LAGOM_MAX_RANKS || rank < 0 || rank >= nranks)
    return fail(LAGOM_ERR_INVALID_ARGUMENT, "rank/nranks out of range");
  auto* c = new lagom_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  if (opts) c->opts = *opts; else lagom_comm_default_opts(&c->opts);
  if (int s = check_opts(&c->opts)) { delete c; return s; }
  layout(c);
  if (int s = alloc_common(c)) { delete c; return s; }
  void* h = nullptr;
  cudaError_t e = cudaMalloc(&h, static_cast<size_t>(c->heap_bytes));
  if (e == cudaSuccess) e = cudaMemset(h, 0, static_cast<size_t>(c->heap_bytes));
  const HeapHeader hdr = header_of(c);
  if (e == cudaSuccess) e = cudaMemcpy(static_cast<char*>(h) + c->off_hdr, &hdr, sizeof hdr, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (h) cudaFree(h);
    cudaFreeHost(c->abort_host);
    if (c->order_ev) cudaEventDestroy(static_cast<cudaEvent_t>(c->order_ev));
    delete c;
    return cuda_fail(e, "heap allocation");
  }
  c->heap[rank] = static_cast<char*>(h);
  c->imported[rank] = true;
  c->ready = nranks == 1;
  *out = c;
  return LAGOM_OK;
}

int lagom_comm_export_handle(lagom_comm_t c, void* handle) {
  if (!c || !handle || c->virt) return fail(LAGOM_ERR_INVALID_ARGUMENT, "export needs a real-mode comm");
  LAGOM_CUDA(cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  LAGOM_CUDA(cudaIpcGetMemHandle(&h, c->heap[c->rank]));
  std::memcpy(handle, &h, sizeof h);
  return LAGOM_OK;
}

int lagom_comm_import_handles(lagom_comm_t c, const void* handles) {
  if (!c || !handles || c->virt) return fail(LAGOM_ERR_INVALID_ARGUMENT, "import needs a real-mode comm");
  LAGOM_CUDA(cudaSetDevice(c->device));
  const char* base = static_cast<const char*>(handles);
  for (int r = 0; r < c->nranks; ++r) {
    if (r == c->rank || c->imported[r]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, base + static_cast<size_t>(r) * LAGOM_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    LAGOM_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->heap[r] = static_cast<char*>(p);
    c->imported[r] = true;
  }
  // every peer must have been created with the same kernel-selecting options
  const HeapHeader mine = header_of(c);
  for (int r = 0; r < c->nranks; ++r) {
    if (r == c->rank) continue;
    HeapHeader peer{};
    LAGOM_CUDA(cudaMemcpy(&peer, c->heap[r] + c->off_hdr, sizeof peer, cudaMemcpyDefault));
    if (std::memcmp(&peer, &mine, sizeof mine) != 0)
      return fail(LAGOM_ERR_INVALID_ARGUMENT,
                  "rank " + std::to_string(r) + " was created with different options (nranks, max_channels, steps, "
                  "max_chunk_bytes, use_tma, coresident, one_hop, a2a_tma must match on every rank)");
  }
  c->ready = true;
  return LAGOM_OK;
}

int lagom_comm_create_virtual(int nranks, int device, const lagom_comm_opts_t* opts,
                              lagom_comm_t* out) {
  if (!out) return fail(LAGOM_ERR_INVALID_ARGUMENT, "null out");
  if (nranks < 1 || nranks > LAGOM_MAX_RANKS) return fail(LAGOM_ERR_INVALID_ARGUMENT, "nranks out of range");
  auto* c = new lagom_comm();
  c->rank = 0;
  c->nranks = nranks;
  c->device = device;
  c->virt = true;
  if (opts) c->opts = *opts; else lagom_comm_default_opts(&c->opts);
  if (int s = check_opts(&c->opts)) { delete c; return s; }
  layout(c);
  if (int s = alloc_common(c)) { delete c; return s; }
  for (int r = 0; r < nranks; ++r) {
    void* h = nullptr;
    cudaError_t e = cudaMalloc(&h, static_cast<size_t>(c->heap_bytes));
    if (e == cudaSuccess) e = cudaMemset(h, 0, static_cast<size_t>(c->heap_bytes));
    if (e != cudaSuccess) {
      lagom_comm_destroy(c);
      return cuda_fail(e, "virtual heap allocation");
    }
    c->heap[r] = static_cast<char*>(h);
    c->imported[r] = true;
  }
  LAGOM_CUDA(cudaDeviceSynchronize());
  c->ready = true;
  *out = c;
  return LAGOM_OK;
}

int lagom_comm_destroy(lagom_comm_t c) {
  if (!c) return LAGOM_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < c->nranks; ++r) {
    if (!c->heap[r]) continue;
    if (c->virt || r == c->rank) cudaFree(c->heap[r]);
    else cudaIpcCloseMemHandle(c->heap[r]);
  }
  lagom_nvls_release(c);
  if (c->abort_host) cudaFreeHost(c->abort_host);
  if (c->order_ev) cudaEventDestroy(static_cast<cudaEvent_t>(c->order_ev));
  delete c;
  return LAGOM_OK;
}

int lagom_comm_info(lagom_comm_t c, int* rank, int* nranks, int* device, int* is_virtual) {
  if (!c) return fail(LAGOM_ERR_INVALID_ARGUMENT, "null comm");
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->nranks;
  if (device) *device = c->device;
  if (is_virtual) *is_virtual = c->virt ? 1 : 0;
  return LAGOM_OK;
}

int64_t lagom_comm_heap_bytes(lagom_comm_t c) { return c ? c->heap_bytes : -1; }

int lagom_comm_check(lagom_comm_t c) {
  if (!c) return fail(LAGOM_ERR_INVALID_ARGUMENT, "null comm");
  if (c->broken) return fail(LAGOM_ERR_BROKEN, "communicator broken by an earlier abort");
  if (*reinterpret_cast<volatile unsigned int*>(c->abort_host) != 0) {
    c->broken = true;
    return fail(LAGOM_ERR_TIMEOUT, "a collective kernel timed out waiting for a peer");
  }
  return LAGOM_OK;
}

int lagom_coll_validate(lagom_comm_t c, const lagom_coll_args_t* a) { return validate(c, a); }

int lagom_coll_launch(lagom_comm_t c, const lagom_coll_args_t* a, const void* sendbuf,
                      void* recvbuf, void* stream) {
  if (int s = validate(c, a)) return s;
  if (c->virt) return fail(LAGOM_ERR_INVALID_ARGUMENT, "virtual comm: use lagom_coll_launch_virtual");
  if (!c->ready) return fail(LAGOM_ERR_NOT_READY, "peer heaps not imported");
  if (c->broken || *reinterpret_cast<volatile unsigned int*>(c->abort_host)) {
    c->broken = true;
    return fail(LAGOM_ERR_BROKEN, "communicator broken by an earlier abort");
  }
  if (a->count == 0) return LAGOM_OK;
  // Issue order across streams: this launch waits for the previous one on
  // this communicator (they share step counters, slots and NVLS epochs).
  const auto st = static_cast<cudaStream_t>(stream);
  const auto order = static_cast<cudaEvent_t>(c->order_ev);
  LAGOM_CUDA(cudaStreamWaitEvent(st, order, 0));
  const int s = launch_real(c, a, sendbuf, recvbuf, st);
  if (s != LAGOM_OK) return s;
  LAGOM_CUDA(cudaEventRecord(order, st));
  return LAGOM_OK;
}

}  // extern "C"

namespace {
int select_real(lagom_comm* c, const lagom_coll_args_t* a, const void* sendbuf, void* recvbuf, LaunchPlan* plan) {
  if (c->nranks == 1) return lagom_local_select(c, a, sendbuf, recvbuf, plan);
  {  // TREE on an NVSwitch box with NVLS bound: the switch-rooted schedule
    size_t nv_bytes = 0;
    const int prep = lagom_nvls_prepare(c, a, sendbuf, recvbuf, &plan->kernel, plan->params, &nv_bytes, &plan->smem);
    if (prep < 0) return LAGOM_ERR_INVALID_ARGUMENT;  // reason recorded by lagom_nvls_prepare
    if (prep == 1) return LAGOM_OK;
  }
  KParams p = make_params(c, a);
  p.send[0] = static_cast<const char*>(sendbuf);
  p.recv[0] = static_cast<char*>(recvbuf);
  static_assert(sizeof p <= sizeof plan->params, "launch plan too small");
  const void* k = pick_kernel(a);
  if (!k) return fail(LAGOM_ERR_INVALID_ARGUMENT, "no kernel for this combination");
  const int smem = smem_for(p, a, k);
  if (smem < 0) return fail(LAGOM_ERR_CUDA, "cannot enable the TMA shared-memory ring");
  std::memcpy(plan->params, &p, sizeof p);
  plan->kernel = k;
  plan->smem = smem;
  return LAGOM_OK;
}

int launch_real(lagom_comm* c, const lagom_coll_args_t* a, const void* sendbuf, void* recvbuf, cudaStream_t stream) {
  LaunchPlan plan;
  if (int s = select_real(c, a, sendbuf, recvbuf, &plan)) return s;
  if (!plan.kernel) return LAGOM_OK;
  void* args[] = {plan.params};
  LAGOM_CUDA(cudaLaunchKernel(plan.kernel, dim3(a->num_channels, 1, 1), dim3(a->num_threads, 1, 1), args,
                              static_cast<size_t>(plan.smem), stream));
  return LAGOM_OK;
}
}  // namespace

extern "C" {

int lagom_coll_launch_virtual(lagom_comm_t c, const lagom_coll_args_t* a,
                              const void* const* sendbufs, void* const* recvbufs, void* stream) {
  if (int s = validate(c, a)) return s;
  if (!c->virt) return fail(LAGOM_ERR_INVALID_ARGUMENT, "real comm: use lagom_coll_launch");
  if (c->broken || *reinterpret_cast<volatile unsigned int*>(c->abort_host)) {
    c->broken = true;
    return fail(LAGOM_ERR_BROKEN, "communicator broken by an earlier abort");
  }
  if (a->count == 0) return LAGOM_OK;
  KParams p = make_params(c, a);
  for (int r = 0; r < c->nranks; ++r) {
    p.send[r] = static_cast<const char*>(sendbufs[r]);
    p.recv[r] = static_cast<char*>(recvbufs[r]);
  }
  const void* k = pick_kernel(a);
  if (!k) return fail(LAGOM_ERR_INVALID_ARGUMENT, "no kernel for this combination");
  void* args[] = {&p};
  const int smem = smem_for(p, a, k);
  if (smem < 0) return fail(LAGOM_ERR_CUDA, "cannot enable the TMA shared-memory ring");
  // Ranks spin on one another: a cooperative launch guarantees that every
  // rank's CTAs are co-resident (or fails loudly instead of hanging).
  const auto st = static_cast<cudaStream_t>(stream);
  const auto order = static_cast<cudaEvent_t>(c->order_ev);
  LAGOM_CUDA(cudaStreamWaitEvent(st, order, 0));
  LAGOM_CUDA(cudaLaunchCooperativeKernel(k, dim3(a->num_channels, c->nranks, 1),
                                         dim3(a->num_threads, 1, 1), args, static_cast<size_t>(smem), st));
  LAGOM_CUDA(cudaEventRecord(order, st));
  return LAGOM_OK;
}

int lagom_coll_footprint(lagom_comm_t c, const lagom_coll_args_t* a, const void* sendbuf, void* recvbuf,
                         int* regs_per_thread, int* smem_bytes) {
  if (int s = validate(c, a)) return s;
  if (c->virt) return fail(LAGOM_ERR_INVALID_ARGUMENT, "footprint needs a real-mode comm");
  if (!regs_per_thread || !smem_bytes) return fail(LAGOM_ERR_INVALID_ARGUMENT, "null output");
  *regs_per_thread = 0;
  *smem_bytes = 0;
  if (a->count == 0) return LAGOM_OK;
  LaunchPlan plan;
  if (int s = select_real(c, a, sendbuf, recvbuf, &plan)) return s;
  if (!plan.kernel) return LAGOM_OK;
  cudaFuncAttributes fa;
  LAGOM_CUDA(cudaFuncGetAttributes(&fa, plan.kernel));
  *regs_per_thread = fa.numRegs;
  *smem_bytes = static_cast<int>(fa.sharedSizeBytes) + plan.smem;
  return LAGOM_OK;
}

int lagom_coll_bytes(const lagom_coll_args_t* a, int nranks, int64_t* alg_bytes, double* bus_factor) {
  if (!a || nranks < 1) return fail(LAGOM_ERR_INVALID_ARGUMENT, "bad arguments");
  const int64_t e = elem_bytes_of(a->dtype);
  const double n = nranks;
  int64_t s = 0;
  double f = 0;
  switch (a->collective) {
    case LAGOM_ALL_REDUCE: s = a->count * e; f = 2.0 * (n - 1) / n; break;
    case LAGOM_ALL_GATHER:
    case LAGOM_REDUCE_SCATTER:
    case LAGOM_ALL_TO_ALL: s = a->count * e * nranks; f = (n - 1) / n; break;
    default: return fail(LAGOM_ERR_INVALID_ARGUMENT, "unknown collective");
  }
  if (alg_bytes) *alg_bytes = s;
  if (bus_factor) *bus_factor = f;
  return LAGOM_OK;
}

}  // extern "C"

extern "C" int lagom_comm_phase_stamps(lagom_comm_t comm, uint64_t* out, int max_values) {
  if (!comm || !out || max_values < 0) return fail(LAGOM_ERR_INVALID_ARGUMENT, "phase_stamps: bad argument");
  const int64_t total = static_cast<int64_t>(comm->opts.max_channels) * 2 * LAGOM_PHASE_STAMPS;
  const int64_t n = std::min<int64_t>(total, max_values);
  LAGOM_CUDA(cudaSetDevice(comm->device));
  LAGOM_CUDA(cudaDeviceSynchronize());
  LAGOM_CUDA(cudaMemcpy(out, comm->heap[comm->virt ? 0 : comm->rank] + comm->off_phase, n * 8, cudaMemcpyDeviceToHost));
  return LAGOM_OK;
}
