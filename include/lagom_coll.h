/* lagom-b200 — C-ABI of the sm_100a collective-kernel family (below the
 * tuner's ProfileFn seam).
 *
 * The reference has no device code: a collective there is the analytic
 * formula comm_time (reference proj/src/commperf.cpp:112-125) over the
 * tunable tuple CommConfig (reference proj/include/lagom/model.hpp:58-67).
 * This header is the boundary that turns that tuple into a real launch:
 *
 *   CommConfig.algorithm    -> lagom_coll_args_t.algorithm  (RING | TREE)
 *   CommConfig.protocol     -> lagom_coll_args_t.protocol   (SIMPLE | LL | LL128)
 *   CommConfig.transport    -> P2P only (NVLink 5 / NVSwitch peer memory)
 *   CommConfig.num_channels -> grid size  (one CTA per channel)
 *   CommConfig.num_threads  -> block size (threads per CTA, 64..640 step 64)
 *   CommConfig.chunk_size   -> bytes of payload per pipeline step per channel
 *
 * Every value the reference tuner can emit (reference tuner.cpp:47-76 with
 * CommBounds defaults, model.hpp:70-76) is accepted.
 *
 * Conventions: plain C, POD structs, no exceptions, no torch types. Every
 * entry point returns lagom_status_t; lagom::b200 (C++) maps non-zero codes
 * to lagom::Error (reference error.hpp:9-18). Streams are cudaStream_t passed
 * as void*. One communicator per process per GPU (real mode), or one
 * communicator emulating all ranks on one GPU (virtual mode, for testing the
 * protocols without NVLink). The library owns the peer mappings; the caller
 * owns streams and buffers.
 */
#ifndef LAGOM_COLL_H_
#define LAGOM_COLL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAGOM_COLL_ABI_VERSION 2
#define LAGOM_MAX_RANKS 8
#define LAGOM_MAX_CHANNELS 64
#define LAGOM_HANDLE_BYTES 64 /* == sizeof(cudaIpcMemHandle_t) */

typedef enum {
  LAGOM_OK = 0,
  LAGOM_ERR_INVALID_ARGUMENT = 1, /* -> ErrorCode::InvalidInput        */
  LAGOM_ERR_INVALID_CONFIG = 2,   /* -> ErrorCode::InvalidWorkload     */
  LAGOM_ERR_CUDA = 3,             /* -> ErrorCode::IoFailure           */
  LAGOM_ERR_TIMEOUT = 4,          /* peer never answered: IoFailure     */
  LAGOM_ERR_NOT_READY = 5,        /* peers not imported yet             */
  LAGOM_ERR_BROKEN = 6            /* an earlier launch aborted          */
} lagom_status_t;

/* Enum values equal the reference's enum order (model.hpp:37-40). */
typedef enum { LAGOM_ALL_REDUCE = 0, LAGOM_ALL_GATHER = 1, LAGOM_REDUCE_SCATTER = 2, LAGOM_ALL_TO_ALL = 3 } lagom_collective_t;
typedef enum { LAGOM_RING = 0, LAGOM_TREE = 1 } lagom_algorithm_t;
typedef enum { LAGOM_SIMPLE = 0, LAGOM_LL = 1, LAGOM_LL128 = 2 } lagom_protocol_t;
typedef enum { LAGOM_F32 = 0, LAGOM_BF16 = 1, LAGOM_F16 = 2, LAGOM_I32 = 3 } lagom_dtype_t;
typedef enum { LAGOM_SUM = 0, LAGOM_MAX = 1, LAGOM_MIN = 2 } lagom_redop_t;

typedef struct {
  int max_channels;        /* channels provisioned (<= LAGOM_MAX_CHANNELS); default 32 */
  int steps;               /* pipeline slots per connection; default 4                 */
  int64_t max_chunk_bytes; /* largest chunk_size accepted; default 4 MiB                */
  int64_t timeout_ms;      /* spin-wait watchdog; default 10000                         */
  int use_tma;             /* SIMPLE copy steps use TMA bulk copies (1, default); 2 also
                              routes reduction steps through the TMA smem ring; 0 off  */
  /* Options below change which kernel a launch runs, so every rank of a
   * communicator must use the same values: lagom_comm_import_handles checks
   * them against every peer's and fails with LAGOM_ERR_INVALID_ARGUMENT. */
  int coresident;          /* 1 (default): at NT <= 256 the NVLS and one-hop kernels,
                              and the single-rank copy at any NT, fit next to a GEMM
                              CTA on one SM (<= 21.8 K registers per CTA, no dynamic
                              shared memory), so their NC costs no SMs; larger NT runs
                              the deep-unroll kernels that take an SM each. 0: deep
                              unrolls at every NT (lagom_coll_footprint tells which) */
  int one_hop;             /* TREE AllGather / ReduceScatter with NVLS bound: 0 through
                              the switch, 1 one hop over the peer mappings
                              (AG: peer stores; RS: TMA pull of the peers' partials, or
                              pushes into the owners' scratch with vector stores, see
                              lagom_comm_nvls_scratch), 2 (default) one hop at nranks == 2
                              from 16 channels up (the multicast echo doubles the
                              switch's bytes there; fewer SMs move less one hop)      */
  int a2a_tma;             /* 1 (default): the one-hop kernels (AllToAll, and with one_hop
                              the AllGather / ReduceScatter) move data with TMA bulk copies
                              (one elected thread, 192 KB smem ring: the CTA takes an SM)
                              except in the co-resident regime (coresident and NT <= 256),
                              which keeps vector loads / stores; 0: vector always     */
} lagom_comm_opts_t;

typedef struct {
  int collective;       /* lagom_collective_t */
  int algorithm;        /* lagom_algorithm_t (TREE: the binary tree for ALL_REDUCE; with
                           NVLS bound, in-switch AR/AG/RS and the one-hop AllToAll;
                           otherwise the other collectives run their ring schedule) */
  int protocol;         /* lagom_protocol_t */
  int num_channels;     /* NC: CTAs */
  int num_threads;      /* NT: threads per CTA */
  int64_t chunk_bytes;  /* C */
  int dtype;            /* lagom_dtype_t */
  int redop;            /* lagom_redop_t (ignored for ALL_GATHER / ALL_TO_ALL) */
  /* count semantics (NCCL-compatible):
   *   ALL_REDUCE     send[count]          -> recv[count]
   *   ALL_GATHER     send[count]          -> recv[nranks*count]
   *   REDUCE_SCATTER send[nranks*count]   -> recv[count]
   *   ALL_TO_ALL     send[nranks*count]   -> recv[nranks*count]            */
  int64_t count;
  /* Optional device pointer to two uint64 {first CTA start, last CTA end}
   * (%globaltimer, ns), combined with atomicMin/atomicMax: initialise to
   * {UINT64_MAX, 0}. The kernel's active span, excluding time the launch
   * spent queued behind other kernels — what the cost model calls x. */
  void* span_out;
} lagom_coll_args_t;

typedef struct lagom_comm* lagom_comm_t;

/* Library / ABI identity. */
int lagom_coll_abi_version(void);
const char* lagom_status_string(int status);
/* Human-readable detail of the last failure on this thread. */
const char* lagom_last_error(void);

void lagom_comm_default_opts(lagom_comm_opts_t* opts);

/* Real mode: one rank of an nranks job on `device` (cudaSetDevice'd by the
 * library). Allocates this rank's symmetric heap (staging slots + flags). */
int lagom_comm_create(int rank, int nranks, int device, const lagom_comm_opts_t* opts,
                      lagom_comm_t* out);
/* Writes this rank's cudaIpcMemHandle (LAGOM_HANDLE_BYTES) into `handle`. */
int lagom_comm_export_handle(lagom_comm_t comm, void* handle);
/* `handles` = nranks * LAGOM_HANDLE_BYTES, rank order (own entry ignored).
 * Maps every peer heap; after this the comm is ready. */
int lagom_comm_import_handles(lagom_comm_t comm, const void* handles);

/* Virtual mode: all `nranks` ranks live on `device` in this process; one
 * cooperative launch runs every rank's CTAs (grid = NC x nranks). */
int lagom_comm_create_virtual(int nranks, int device, const lagom_comm_opts_t* opts,
                              lagom_comm_t* out);

int lagom_comm_destroy(lagom_comm_t comm);
int lagom_comm_info(lagom_comm_t comm, int* rank, int* nranks, int* device, int* is_virtual);
/* Bytes of device memory this rank's heap occupies. */
int64_t lagom_comm_heap_bytes(lagom_comm_t comm);
/* LAGOM_OK, or LAGOM_ERR_TIMEOUT/BROKEN if a launched kernel aborted. Call
 * after synchronizing the stream of the launch. */
int lagom_comm_check(lagom_comm_t comm);

/* Validates (collective, algorithm, protocol, NC, NT, C) against this comm
 * without launching. */
int lagom_coll_validate(lagom_comm_t comm, const lagom_coll_args_t* args);

/* Real mode: enqueue one collective on `stream` (cudaStream_t). Launches on
 * one communicator are ordered in issue order even across streams (each
 * launch waits for the previous one through an event the communicator
 * keeps), because consecutive launches share the per-connection step
 * counters and the NVLS epochs. With nranks == 1 every collective is a copy
 * of count elements (none in place). */
int lagom_coll_launch(lagom_comm_t comm, const lagom_coll_args_t* args, const void* sendbuf,
                      void* recvbuf, void* stream);
/* Virtual mode: sendbufs/recvbufs hold nranks device pointers, rank order. */
int lagom_coll_launch_virtual(lagom_comm_t comm, const lagom_coll_args_t* args,
                              const void* const* sendbufs, void* const* recvbufs, void* stream);

/* The per-CTA footprint of the kernel this launch would run (nothing is
 * launched): registers per thread and shared memory per CTA (static +
 * dynamic); both 0 when nothing would launch (count 0, in-place nranks 1).
 * NT x regs and smem tell whether the CTAs fit next to a GEMM CTA on one SM
 * (sm_100 cuBLASLt bf16 GEMMs leave ~22.5 K registers and ~19 KB free). */
int lagom_coll_footprint(lagom_comm_t comm, const lagom_coll_args_t* args, const void* sendbuf,
                         void* recvbuf, int* regs_per_thread, int* smem_bytes);

/* Algorithmic and bus bytes of one launch (nccl-tests accounting):
 * algbw bytes S and busbw factor, so busbw = S / t * factor. */
int lagom_coll_bytes(const lagom_coll_args_t* args, int nranks, int64_t* alg_bytes,
                     double* bus_factor);

/* NVLS (NVLink SHARP multicast) on NVSwitch boxes. With a bound region,
 * TREE AllReduce / AllGather / ReduceScatter (sum) whose buffers live in the
 * region run reduced/broadcast inside the switch (multimem.ld_reduce /
 * multimem.st); other launches keep the P2P kernels. Collective set-up:
 *   rank 0: lagom_comm_nvls_export(bytes, blob)  -> broadcast blob
 *   all:    lagom_comm_nvls_import(blob); <barrier>; lagom_comm_nvls_bind()
 * Allocations (same sequence on every rank) have identical offsets. */
int lagom_comm_nvls_supported(lagom_comm_t comm);
int lagom_comm_nvls_export(lagom_comm_t comm, int64_t bytes, void* blob /* LAGOM_HANDLE_BYTES */);
int lagom_comm_nvls_import(lagom_comm_t comm, const void* blob);
int lagom_comm_nvls_bind(lagom_comm_t comm);
int lagom_comm_nvls_alloc(lagom_comm_t comm, int64_t bytes, void** ptr);
int64_t lagom_comm_nvls_bytes(lagom_comm_t comm);
/* One-hop AllToAll through the switch: after nvls_bind, every rank exports
 * its region's physical allocation (blob), the blobs are all-gathered in rank
 * order (nranks * LAGOM_HANDLE_BYTES), every rank maps every peer's region,
 * and all ranks switch it on (nvls_use_peers). Then ALL_TO_ALL with algorithm TREE and recvbuf in the region
 * stores each block straight into its destination rank's recvbuf (one NVLink
 * write per byte, no staging). The exporter keeps its fd open until
 * lagom_comm_destroy, so peers may import at any time before that. */
int lagom_comm_nvls_export_peer(lagom_comm_t comm, void* blob /* LAGOM_HANDLE_BYTES */);
int lagom_comm_nvls_import_peers(lagom_comm_t comm, const void* blobs);
/* Reserves the push-based one-hop ReduceScatter's scratch in the NVLS region:
 * nranks slots of slot_bytes (slot q receives rank q's partial of this
 * rank's block). Same call order on every rank (symmetric offsets, like
 * lagom_comm_nvls_alloc). Without it (or for blocks larger than a slot) the
 * one-hop ReduceScatter pulls peers' partials instead of receiving pushes. */
int lagom_comm_nvls_scratch(lagom_comm_t comm, int64_t slot_bytes);
/* Switches the one-hop AllToAll on (1) or off (0). Must be agreed on by all
 * ranks (call it with the same value everywhere once every rank imported),
 * since sender and receiver must use the same schedule. */
int lagom_comm_nvls_use_peers(lagom_comm_t comm, int on);

/* Synthetic data: fills `nelems` elements of `dtype` with uniform values in
 * [-scale, scale) (int32: integers in [-2^20, 2^20)) from a counter-based
 * hash of (seed, index) — deterministic and identical on every GPU. */
int lagom_fill_random(void* ptr, int64_t nelems, int dtype, uint64_t seed, float scale,
                      void* stream);

/* Enqueues a one-thread kernel on `stream` that writes the GPU's
 * %globaltimer (ns; the clock of span_out and of CUPTI's PM samples) to the
 * device uint64 at `dst`: aligns stream timelines with counter samples. */
int lagom_timestamp(void* dst, void* stream);

/* Diagnostics. With LAGOM_PHASE_STAMPS=1 in the environment at communicator
 * creation, the switch kernels (NVLS AR / AG / RS, one hop) record per channel
 * for the last two launches 8 uint64 values: %globaltimer at entry, after the entry
 * barrier, after the data loop, after the system fence, after the exit
 * barrier, then the launch's epoch. Synchronizes the device and copies
 * min(max_values, max_channels * 16) of them, [channel][(epoch/2)%2][8], into
 * `out`. */
int lagom_comm_phase_stamps(lagom_comm_t comm, uint64_t* out, int max_values);

#ifdef __cplusplus
}
#endif

#endif /* LAGOM_COLL_H_ */
