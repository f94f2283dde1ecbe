// lagom-b200 — B200 layer under the tuner's ProfileFn seam (new, additive API;
// no reference counterpart — the reference's profiler is the simulator,
// reference proj/include/lagom/tuner.hpp:15-20 / simulator.hpp:26-43).
//
//   ReplayDag        the iteration DAG to execute: the reference Workload's
//                    shape (ordered compute stream + serialized comm stream +
//                    ready_after gates, model.hpp:78-96) with real kernels
//                    attached — cuBLASLt bf16 GEMMs (victims) and collectives.
//   Coordinator      host-side rank coordination (broadcast / all-gather /
//                    max-reduce / barrier). make_shm_coordinator() is the
//                    native one-box implementation over POSIX shared memory.
//   ReplayEngine     per rank: owns the streams, events, cuBLASLt plans, the
//                    collective communicator (include/lagom_coll.h) and an
//                    NCCL communicator for the NCCL-default baseline.
//   make_gpu_profiler  the measured twin of make_sim_profiler: rank 0 calls it
//                    from tune(); every other rank sits in ReplayEngine::serve().
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "lagom/model.hpp"
#include "lagom/oracle.hpp"
#include "lagom/simulator.hpp"
#include "lagom/sweep.hpp"
#include "lagom/tuner.hpp"

namespace lagom::b200 {

// ------------------------------------------------------------------- DAG ---
struct GemmShape {
  std::int64_t m = 0, n = 0, k = 0;  // D[m,n] = A[m,k] * B[k,n], bf16 in/out, fp32 accumulate
  std::int64_t batch = 1;            // > 1: strided-batched (attention cores)
};

// Fused scaled-dot-product attention (cuDNN SDPA, flash-style): Q, K, V
// [batch, heads, seq, head_dim] bf16, fp32 softmax; forward or backward.
struct AttentionShape {
  std::int64_t batch = 1, heads = 1, seq = 0, head_dim = 128;
  bool causal = true;
  bool backward = false;
};

struct ReplayComputeOp {
  std::string id;
  std::vector<GemmShape> gemms;           // executed back to back on the compute stream,
  std::vector<AttentionShape> attention;  // then these
};

// Element type codes are lagom_dtype_t (include/lagom_coll.h).
struct ReplayCommOp {
  std::string id;
  Collective collective = Collective::AllReduce;
  int dtype = 1;             // LAGOM_BF16
  std::int64_t count = 0;    // per lagom_coll.h count semantics
  std::optional<std::string> ready_after;
  CommBounds bounds;
};

struct ReplayDag {
  std::string name;
  std::vector<ReplayComputeOp> compute_ops;
  std::vector<ReplayCommOp> comm_ops;
};

// Bytes one comm op's message carries in the model (CommOp.message_bytes):
// the per-rank buffer the collective moves (AR: the buffer; AG/RS/A2A: the
// full n-block buffer).
std::int64_t message_bytes(const ReplayCommOp& op, int nranks);
// FLOPs of one compute op (2*m*n*k*batch summed).
double compute_flops(const ReplayComputeOp& op);

// The tuner's view of the DAG. Compute ops get wave-model parameters
// estimated from their GEMM shapes (the contention profiler refits them).
Workload to_workload(const ReplayDag& dag, const GpuSpec& gpu, int nranks);
// The replay DAG JSON (paper_2602_20656_b200/dags.py): compute_ops with
// "gemms" [[m, n, k(, batch)], ...] and "attention" [[batch, heads, seq,
// head_dim, causal, backward], ...]; comm_ops with collective, dtype, count,
// ready_after and bounds.
ReplayDag replay_dag_from_json(const std::string& text);

// ------------------------------------------------------------ coordinator --
class Coordinator {
 public:
  virtual ~Coordinator() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual void barrier() = 0;
  virtual void broadcast(void* buf, std::size_t bytes, int root) = 0;
  // out = concat over ranks of `bytes` from each rank (rank order).
  virtual void allgather(const void* in, std::size_t bytes, void* out) = 0;
  virtual void allreduce_max(double* values, std::size_t n) = 0;
};

std::unique_ptr<Coordinator> make_single_coordinator();
// All ranks pass the same unique `name` (e.g. derived from a job token).
// Rank 0 creates the segment; the others attach (waiting up to timeout_s).
std::unique_ptr<Coordinator> make_shm_coordinator(const std::string& name, int rank, int size,
                                                  double timeout_s = 300.0);

// ---------------------------------------------------------------- engine ---
// Per-SM resources an sm_100 cuBLASLt bf16 GEMM CTA leaves free (256 threads
// x 168 registers, ~214 KB shared memory; profiles/round2_coresidence.md).
constexpr int kCoresidentRegs = 21845;      // 65536 / 3
constexpr int kCoresidentSmem = 16 * 1024;
enum : int { kPartitionNone = 0, kPartitionAuto = 1, kPartitionAll = 2 };

struct ReplayOptions {
  int device = 0;
  int repeats = 3;           // replays per profile call; medians are reported
  int warmup = 1;            // unrecorded replays before the measured ones
  bool enable_nccl = true;   // create an NCCL communicator for the baseline
  std::int64_t max_chunk_bytes = 4 << 20;
  int max_channels = 32;
  std::uint64_t seed = 1234;
  // End-to-end mode (run_e2e): every replay first copies `e2e_in_bytes` from
  // pinned host memory into the first GEMM's input operand (the step's
  // activations) and finally reads `e2e_out_bytes` of the last comm op's
  // result back to pinned host memory; both copies are inside Z.
  std::int64_t e2e_in_bytes = 0;
  std::int64_t e2e_out_bytes = 0;
  // SM partition of Lagom replays: the GEMMs that a collective can overlap
  // run with cuBLASLt's SM count target = num_sms - the NC it reserves
  // (the contention model's lambda - NC made explicit).
  //   kPartitionNone: no SMs reserved;
  //   kPartitionAuto: only collectives whose CTAs cannot share an SM with a
  //     GEMM CTA reserve their NC (lagom_coll_footprint: NT x registers >
  //     kCoresidentRegs or shared memory > kCoresidentSmem) — the
  //     co-resident NVLS / one-hop / single-rank kernels take no SMs;
  //   kPartitionAll: every collective reserves its NC (round 1).
  // NCCL-baseline replays keep cuBLASLt's default (see nccl_reserve_sms).
  int sm_partition = 1;
  // Ablation: NCCL-baseline replays run the GEMMs that a collective can
  // overlap on num_sms - nccl_reserve_sms SMs (0: cuBLASLt's default).
  int nccl_reserve_sms = 0;
  // SIMPLE collectives move data with TMA bulk copies (lagom_comm_opts_t.use_tma).
  bool use_tma = true;
  // Victim GEMMs run the fastest of cuBLASLt's top-8 heuristic algorithms
  // for their shape and SM budget (timed once); false: the first candidate.
  bool autotune_gemms = true;
  // PM sampling: metrics (empty = default_pm_metrics()) and interval.
  std::vector<std::string> pm_metrics;
  std::uint64_t pm_interval_ns = 20000;
  // lagom_comm_opts_t.coresident / one_hop / a2a_tma (kernel selection; the
  // same on every rank).
  bool coresident = true;
  int one_hop = 2;
  bool a2a_tma = true;
  // NVSwitch multicast: comm buffers live in an NVLS region, so TREE
  // AllReduce/AllGather/ReduceScatter run reduced/broadcast in the switch.
  bool nvls = false;
};

// CUPTI PM sampling (pm_sampler.cpp): counters sampled every `interval_ns`
// of GPU time while kernels run concurrently — no kernel replay, no
// serialisation. One sampler per process and device.
struct PmSample {
  std::uint64_t start_ns = 0, end_ns = 0;  // GPU timestamps (%globaltimer clock)
  std::vector<double> values;              // one per metric
};
class PmSampler {
 public:
  // metrics empty: default_pm_metrics()
  PmSampler(int device, std::vector<std::string> metrics = {}, std::uint64_t interval_ns = 20000,
            std::size_t max_samples = 20000);
  ~PmSampler();
  PmSampler(const PmSampler&) = delete;
  PmSampler& operator=(const PmSampler&) = delete;
  const std::vector<std::string>& metrics() const;
  void start();
  std::vector<PmSample> stop();  // every completed sample since start()

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};
// DRAM read/write bytes, NVLink tx/rx bytes, SM active and elapsed cycles,
// tensor-pipe active cycles, L2 bytes.
std::vector<std::string> default_pm_metrics();

// One measured replay, max over ranks (median over repeats).
struct ReplayMeasurement {
  ProfileResult profile;           // x_j, X = sum x_j, Y = sum y_i, Z
  std::vector<double> comp_times;  // y_i
  // x_j from CUDA events on the comm stream (launch to completion, including
  // time queued behind other kernels), next to profile.comm_times, which is
  // the kernel's own active span for the Lagom kernels
  std::vector<double> comm_event_times;
  // PM sampling (set_pm_sampling): this rank's samples over its last
  // replay, and the %globaltimer instant of the replay's start (the origin
  // of the timeline's start offsets).
  std::vector<std::string> pm_metrics;
  std::vector<PmSample> pm_samples;
  std::uint64_t pm_t0_ns = 0;
  double wall_us = 0.0;            // host wall time of the profile call
  // This rank's last replay as a timeline (one event per compute op on the
  // "compute" stream, one per comm op on "comm"), start offsets from the
  // replay start — exportable with trace_to_json (reference json_io.hpp:36).
  std::vector<TimelineEvent> timeline;
};

class ReplayEngine {
 public:
  ReplayEngine(const ReplayDag& dag, Coordinator& coord, const ReplayOptions& opts);
  ~ReplayEngine();
  ReplayEngine(const ReplayEngine&) = delete;
  ReplayEngine& operator=(const ReplayEngine&) = delete;

  const ReplayDag& dag() const;
  int rank() const;
  int nranks() const;

  // Collective-call functions: every rank must call them in the same order.
  // Lagom kernels with one CommConfig per comm op.
  ReplayMeasurement run(const std::vector<CommConfig>& configs);
  // Same, end to end (host->device input and device->host result per replay).
  ReplayMeasurement run_e2e(const std::vector<CommConfig>& configs);
  // Same DAG, every comm through NCCL with its default parameters.
  ReplayMeasurement run_nccl();
  // Compute stream only (isolated victim times y_i).
  ReplayMeasurement run_compute_only();
  // Comm stream only with the given configs (isolated x_j).
  ReplayMeasurement run_comm_only(const std::vector<CommConfig>& configs);

  // Command protocol for make_gpu_profiler: rank 0 drives, others serve().
  // Returns when rank 0 calls stop().
  void serve();
  void stop();  // rank 0 only
  ReplayMeasurement remote_run(const std::vector<CommConfig>& configs);      // rank 0 only
  ReplayMeasurement remote_run_e2e(const std::vector<CommConfig>& configs);  // rank 0 only
  ReplayMeasurement remote_run_nccl();                                       // rank 0 only
  ReplayMeasurement remote_run_compute_only();                               // rank 0 only
  ReplayMeasurement remote_run_comm_only(const std::vector<CommConfig>& c);  // rank 0 only

  // Number of replay measurements performed.
  int calls() const;
  // Rank 0: replays per measurement and unrecorded warmups for the following
  // remote_* calls (sent along with each command to the serving ranks).
  void set_measurement(int repeats, int warmup);
  // Rank 0: the SM partition of the following remote_* calls (sent along
  // with each command): Lagom replays reserve max NC SMs from the GEMMs that
  // a collective can overlap (lagom_partition), NCCL replays reserve
  // `nccl_reserve_sms` (0 = none).
  void set_partition(int sm_partition, int nccl_reserve_sms);
  // Rank 0: CUPTI PM sampling on every rank during the following remote_*
  // calls (each rank samples its own GPU; rank 0's samples are returned).
  void set_pm_sampling(bool on);
  // Whether the NVLS region (in-switch TREE) and the peer mappings (one-hop
  // AllToAll / AllGather / ReduceScatter) are in use — what set-up achieved,
  // not what was requested.
  bool nvls_active() const;
  bool nvls_peers_active() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// The measured ProfileFn (rank 0): broadcasts the configs, every rank replays
// the DAG, results are max-reduced over ranks. Measurements are not pure
// (noise), so `record` (optional) receives every (configs, result) pair — a
// profile table that replays bit-identically through any tuner.
ProfileFn make_gpu_profiler(ReplayEngine& engine,
                            std::vector<std::pair<std::vector<CommConfig>, ProfileResult>>* record = nullptr);

// Role-tied search: comm ops with the same group id share one config (e.g.
// the k-th gradient bucket of every layer). The tuner sees one comm op per
// group (grouped_workload); the profiler replays the FULL DAG with the group
// configs expanded to every op and reports x_g = sum of its ops' x_j, so X,
// Y and Z are those of the real iteration.
Workload grouped_workload(const ReplayDag& dag, const std::vector<int>& group_of_op, const GpuSpec& gpu,
                          int nranks);
ProfileFn make_grouped_gpu_profiler(ReplayEngine& engine, std::vector<int> group_of_op,
                                    std::vector<std::pair<std::vector<CommConfig>, ProfileResult>>* record = nullptr);

// exhaustive() (reference oracle.cpp:12-63) with one GPU thread per joint
// grid point; bit-identical result (FP64, no FMA contraction, host argmin in
// enumeration order). Falls back to the CPU oracle for what it does not cover
// (more than 64 ops, invalid grid entries, grids beyond `limit`).
lagom::OracleResult exhaustive_gpu(const Workload& workload, const std::vector<std::vector<CommConfig>>& grids,
                            const SubspaceParams& params, std::int64_t limit, int device = 0);

// exhaustive() / run_sweep() (reference oracle.cpp:12-63, sweep.cpp:11-61)
// with any ProfileFn — with make_gpu_profiler every grid point / sweep value
// is a measured replay. Same enumeration order and tie rule as the
// simulated versions.
OracleResult exhaustive_with(const ProfileFn& profile_fn, const Workload& workload,
                             const std::vector<std::vector<CommConfig>>& grids, std::int64_t limit);
std::vector<SweepRow> sweep_with(const ProfileFn& profile_fn, const Workload& workload,
                                 const std::vector<CommConfig>& base, const std::string& comm_id, SweepParam param,
                                 const std::vector<std::int64_t>& values);

// A ProfileFn that answers from a recorded table (exact config-vector match;
// throws Error(InvalidInput) on a miss). Used to prove that two tuners make
// identical picks given the same profile table.
ProfileFn make_table_profiler(std::vector<std::pair<std::vector<CommConfig>, ProfileResult>> table);

}  // namespace lagom::b200
