// Iteration-replay engine: the measured twin of the reference's simulate()
// (reference simulator.cpp:32-166). It executes the DAG with the same
// scheduling contract the model assumes —
//   * compute ops back to back on one stream (cuBLASLt bf16 GEMMs);
//   * comm ops strictly in order on a second stream, comm j starting after
//     comm j-1 and after its ready_after compute op (cudaStreamWaitEvent);
// — and measures with CUDA events: y_i per compute op, x_j per comm op (from
// the instant the comm stream reaches it to its end, i.e. the model's
// start/end), Z = last event - start. Results are max-reduced over ranks and
// the median over `repeats` replays is reported.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <unordered_map>

#include "attention.hpp"
#include "lagom/b200.hpp"
#include "lagom/error.hpp"
#include "lagom/json_io.hpp"
#include "lagom_coll.h"
#include "nccl_dl.hpp"

namespace lagom::b200 {

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(ErrorCode::IoFailure, "cuda", std::string(what) + ": " + cudaGetErrorString(e));
}
void lt_check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS)
    throw Error(ErrorCode::IoFailure, "cublasLt", std::string(what) + " failed with status " + std::to_string(s));
}
void coll_check(int s, const char* what) {
  if (s != LAGOM_OK) {
    const ErrorCode code = s == LAGOM_ERR_INVALID_CONFIG ? ErrorCode::InvalidWorkload
                           : s == LAGOM_ERR_INVALID_ARGUMENT ? ErrorCode::InvalidInput
                                                             : ErrorCode::IoFailure;
    throw Error(code, what, lagom_last_error());
  }
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(ErrorCode::IoFailure, "nccl", std::string(what) + ": " + nccl().GetErrorString(r));
}

int elem_bytes(int dtype) { return (dtype == LAGOM_BF16 || dtype == LAGOM_F16) ? 2 : 4; }

int coll_code(Collective c) {
  switch (c) {
    case Collective::AllReduce: return LAGOM_ALL_REDUCE;
    case Collective::AllGather: return LAGOM_ALL_GATHER;
    case Collective::ReduceScatter: return LAGOM_REDUCE_SCATTER;
    case Collective::AllToAll: return LAGOM_ALL_TO_ALL;
  }
  return LAGOM_ALL_REDUCE;
}

ncclDataType_t nccl_type(int dtype) {
  switch (dtype) {
    case LAGOM_F32: return ncclFloat32;
    case LAGOM_BF16: return ncclBfloat16;
    case LAGOM_F16: return ncclFloat16;
    default: return ncclInt32;
  }
}

// LAGOM_TRACE=1: one stderr line per measurement / command, per rank.
bool trace_on() {
  static const bool on = [] {
    const char* e = std::getenv("LAGOM_TRACE");
    return e && *e && *e != '0';
  }();
  return on;
}
double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

enum class Mode : int { Lagom = 1, Nccl = 2, ComputeOnly = 3, CommOnly = 4, Stop = 5, LagomE2E = 6 };

struct Plan {
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatmulAlgo_t algo{};
};

struct Gemm {
  GemmShape shape;
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, d = nullptr;
  cublasLtMatmulAlgo_t algo{};
  void *A = nullptr, *B = nullptr, *D = nullptr;
  std::map<int, Plan> by_sm_target;  // plans restricted to a number of SMs
};

struct Comm {
  ReplayCommOp op;
  int dep = -1;
  void* send = nullptr;
  void* recv = nullptr;
  std::int64_t in_elems = 0, out_elems = 0;
  bool nvls = false;
};

template <typename T>
T median_of(std::vector<T> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

// Command broadcast from rank 0 to the serving ranks.
struct WireConfig {
  std::int32_t algorithm, protocol, transport, num_channels, num_threads, pad;
  std::int64_t chunk_size;
};

}  // namespace

// ------------------------------------------------------------- DAG helpers --

std::int64_t message_bytes(const ReplayCommOp& op, int nranks) {
  const std::int64_t e = elem_bytes(op.dtype);
  return op.collective == Collective::AllReduce ? op.count * e : op.count * e * nranks;
}

double attention_flops(const AttentionShape& a) {
  // forward: QK^T and PV, 2 x 2*b*h*s*s*d; backward 2.5x (dV, dP, dQ, dK + recompute of S);
  // causal masks half of the score matrix
  const double fwd = 4.0 * static_cast<double>(a.batch * a.heads) * static_cast<double>(a.seq) *
                     static_cast<double>(a.seq) * static_cast<double>(a.head_dim) * (a.causal ? 0.5 : 1.0);
  return a.backward ? 2.5 * fwd : fwd;
}

double compute_flops(const ReplayComputeOp& op) {
  double f = 0;
  for (const GemmShape& g : op.gemms)
    f += 2.0 * static_cast<double>(g.m) * static_cast<double>(g.n) * static_cast<double>(g.k) *
         static_cast<double>(g.batch);
  for (const AttentionShape& a : op.attention) f += attention_flops(a);
  return f;
}

ReplayDag replay_dag_from_json(const std::string& text) {
  const Json d = parse_json(text, "dag");
  ReplayDag dag;
  dag.name = d.value("name", std::string("dag"));
  for (const Json& c : d.at("compute_ops")) {
    ReplayComputeOp op;
    op.id = c.at("id").get<std::string>();
    for (const Json& g : c.value("gemms", Json::array()))
      op.gemms.push_back({g.at(0).get<std::int64_t>(), g.at(1).get<std::int64_t>(), g.at(2).get<std::int64_t>(),
                          g.size() > 3 ? g.at(3).get<std::int64_t>() : 1});
    for (const Json& a : c.value("attention", Json::array()))
      op.attention.push_back({a.at(0).get<std::int64_t>(), a.at(1).get<std::int64_t>(), a.at(2).get<std::int64_t>(),
                              a.at(3).get<std::int64_t>(), a.size() > 4 ? a.at(4).get<int>() != 0 : true,
                              a.size() > 5 ? a.at(5).get<int>() != 0 : false});
    dag.compute_ops.push_back(op);
  }
  for (const Json& c : d.at("comm_ops")) {
    ReplayCommOp op;
    op.id = c.at("id").get<std::string>();
    op.collective = collective_from_string(c.at("collective").get<std::string>());
    op.dtype = c.value("dtype", 1);
    op.count = c.at("count").get<std::int64_t>();
    if (c.contains("ready_after") && !c["ready_after"].is_null()) op.ready_after = c["ready_after"].get<std::string>();
    if (c.contains("bounds")) {
      const Json& b = c["bounds"];
      op.bounds.nc_max = b.value("nc_max", op.bounds.nc_max);
      op.bounds.c_min = b.value("c_min", op.bounds.c_min);
      op.bounds.c_max = b.value("c_max", op.bounds.c_max);
    }
    dag.comm_ops.push_back(op);
  }
  return dag;
}

Workload to_workload(const ReplayDag& dag, const GpuSpec& gpu, int nranks) {
  Workload w;
  w.gpu = gpu;
  for (const ReplayComputeOp& c : dag.compute_ops) {
    ComputeOp op;
    op.id = c.id;
    // One CTA per 256x128 output tile, one resident CTA per SM (sm_100
    // cuBLASLt bf16 tiles); D = operand + result bytes per tile; theta =
    // a tile's FLOPs at 1/148 of the measured dense bf16 rate (~1.43 PF/s
    // sustained) — starting values the contention profiler refits.
    std::int64_t tiles = 0;
    double bytes = 0;
    for (const GemmShape& g : c.gemms) {
      tiles += ((g.m + 255) / 256) * ((g.n + 127) / 128) * g.batch;
      bytes += 2.0 * static_cast<double>(g.batch) *
               static_cast<double>(g.m * g.k + g.k * g.n + g.m * g.n);
    }
    for (const AttentionShape& a : c.attention) {  // one CTA per 128-row query tile
      tiles += a.batch * a.heads * ((a.seq + 127) / 128);
      bytes += 2.0 * static_cast<double>(a.batch * a.heads * a.seq * a.head_dim) * (a.backward ? 8.0 : 4.0);
    }
    op.total_blocks = std::max<std::int64_t>(1, tiles);
    op.blocks_per_sm = 1;
    op.bytes_per_block = static_cast<std::int64_t>(bytes / static_cast<double>(op.total_blocks));
    const double flops_per_tile = compute_flops(c) / static_cast<double>(op.total_blocks);
    op.base_wave_time = flops_per_tile / (1.43e15 / 148.0) * 1e6;  // us
    w.compute_ops.push_back(op);
  }
  for (const ReplayCommOp& c : dag.comm_ops) {
    CommOp op;
    op.id = c.id;
    op.collective = c.collective;
    op.message_bytes = std::max<std::int64_t>(1, message_bytes(c, nranks));
    op.ready_after = c.ready_after;
    op.bounds = c.bounds;
    w.comm_ops.push_back(op);
  }
  return w;
}

// ------------------------------------------------------------------ engine --

struct ReplayEngine::Impl {
  ReplayDag dag;
  Coordinator& coord;
  ReplayOptions opts;
  int rank = 0, n = 1;
  int num_sms = 148;
  cudaStream_t cs = nullptr, ks = nullptr;
  cublasLtHandle_t lt = nullptr;
  void* workspace = nullptr;
  std::size_t workspace_bytes = 64ull << 20;
  std::vector<std::vector<Gemm>> gemms;  // per compute op
  void* cudnn = nullptr;                 // cuDNN handle (attention victims)
  std::vector<std::unique_ptr<Attention>> attn_pool;  // one per distinct shape (shared by layers)
  std::vector<std::vector<Attention*>> attention;     // per compute op
  void* attn_workspace = nullptr;
  std::map<std::tuple<std::int64_t, std::int64_t, std::int64_t, std::int64_t>, std::array<void*, 3>> operands;
  std::vector<Comm> comms;
  lagom_comm_t lcomm = nullptr;
  ncclComm_t ncomm = nullptr;
  cudaEvent_t ev_start = nullptr, ev_cend = nullptr, ev_kend = nullptr;
  std::vector<cudaEvent_t> ev_cb, ev_ce, ev_kb, ev_ke;
  unsigned long long* spans = nullptr;  // device: [start_j...][end_j...]
  std::vector<unsigned long long> spans_host;
  void* host_in = nullptr;   // pinned
  void* host_out = nullptr;  // pinned
  int calls = 0;
  bool pm_on = false;
  std::vector<std::int64_t> model_blocks;  // per compute op: the CTAs to_workload models (trace args.blocks)
  std::unique_ptr<PmSampler> sampler;  // created on first use (each rank, its own GPU)
  unsigned long long* stamp = nullptr;  // device: %globaltimer at the replay start
  bool nvls_on = false;
  bool nvls_peers_on = false;
  std::vector<TimelineEvent> last_timeline;

  Impl(const ReplayDag& d, Coordinator& c, const ReplayOptions& o) : dag(d), coord(c), opts(o) {
    rank = coord.rank();
    n = coord.size();
    cuda_check(cudaSetDevice(opts.device), "cudaSetDevice");
    cuda_check(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, opts.device), "sm count");
    cuda_check(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream");
    // The comm stream has the highest priority (every arm, NCCL included):
    // a collective launched while the victims' CTAs fill the GPU gets the
    // next SM that frees up instead of queueing behind the rest of a GEMM or
    // attention grid.
    int prio_lo = 0, prio_hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "priority range");
    cuda_check(cudaStreamCreateWithPriority(&ks, cudaStreamNonBlocking, prio_hi), "stream");
    lt_check(cublasLtCreate(&lt), "cublasLtCreate");
    cuda_check(cudaMalloc(&workspace, workspace_bytes), "workspace");
    build_gemms();
    build_attention();
    for (const ComputeOp& op : to_workload(dag, GpuSpec{}, n).compute_ops) model_blocks.push_back(op.total_blocks);
    build_comm_backends();
    build_comms();
    auto mk = [](cudaEvent_t* e) { cuda_check(cudaEventCreate(e), "event"); };
    mk(&ev_start);
    mk(&ev_cend);
    mk(&ev_kend);
    ev_cb.resize(dag.compute_ops.size());
    ev_ce.resize(dag.compute_ops.size());
    ev_kb.resize(dag.comm_ops.size());
    ev_ke.resize(dag.comm_ops.size());
    for (auto* v : {&ev_cb, &ev_ce, &ev_kb, &ev_ke})
      for (auto& e : *v) mk(&e);
    if (opts.e2e_in_bytes > 0) {
      if (dag.compute_ops.empty() || gemms[0].empty())
        throw Error(ErrorCode::InvalidInput, "e2e", "end-to-end mode needs a compute op");
      const Gemm& g0 = gemms[0][0];
      const std::int64_t cap = g0.shape.k * g0.shape.m * g0.shape.batch * 2;
      opts.e2e_in_bytes = std::min(opts.e2e_in_bytes, cap);
      cuda_check(cudaHostAlloc(&host_in, opts.e2e_in_bytes, cudaHostAllocDefault), "pinned in");
      // synthetic step input, generated once on the device and parked on the host
      cuda_check(cudaMemcpy(host_in, g0.A, opts.e2e_in_bytes, cudaMemcpyDeviceToHost), "seed host input");
    }
    if (opts.e2e_out_bytes > 0) {
      if (comms.empty()) throw Error(ErrorCode::InvalidInput, "e2e", "end-to-end mode needs a comm op");
      const Comm& last = comms.back();
      opts.e2e_out_bytes = std::min<std::int64_t>(opts.e2e_out_bytes, last.out_elems * elem_bytes(last.op.dtype));
      cuda_check(cudaHostAlloc(&host_out, opts.e2e_out_bytes, cudaHostAllocDefault), "pinned out");
    }
    if (!comms.empty()) {
      cuda_check(cudaMalloc(&spans, 2 * comms.size() * sizeof(unsigned long long)), "spans");
      spans_host.resize(2 * comms.size());
    }
    cuda_check(cudaDeviceSynchronize(), "init sync");
    coord.barrier();
  }

  ~Impl() {
    cudaSetDevice(opts.device);
    cudaDeviceSynchronize();
    for (auto& ops : gemms)
      for (Gemm& g : ops) {
        for (auto& [t, pl] : g.by_sm_target) cublasLtMatmulDescDestroy(pl.desc);
        if (g.desc) cublasLtMatmulDescDestroy(g.desc);
        if (g.a) cublasLtMatrixLayoutDestroy(g.a);
        if (g.b) cublasLtMatrixLayoutDestroy(g.b);
        if (g.d) cublasLtMatrixLayoutDestroy(g.d);
      }
    for (auto& [k, p] : operands)
      for (void* q : p) cudaFree(q);
    attention.clear();
    attn_pool.clear();
    if (attn_workspace) cudaFree(attn_workspace);
    destroy_cudnn_handle(cudnn);
    for (Comm& c : comms) {
      if (c.nvls) continue;  // owned by the communicator's NVLS region
      cudaFree(c.send);
      cudaFree(c.recv);
    }
    if (spans) cudaFree(spans);
    if (stamp) cudaFree(stamp);
    if (host_in) cudaFreeHost(host_in);
    if (host_out) cudaFreeHost(host_out);
    if (ncomm) nccl().CommDestroy(ncomm);
    if (lcomm) lagom_comm_destroy(lcomm);
    for (auto* v : {&ev_cb, &ev_ce, &ev_kb, &ev_ke})
      for (auto& e : *v) cudaEventDestroy(e);
    cudaEventDestroy(ev_start);
    cudaEventDestroy(ev_cend);
    cudaEventDestroy(ev_kend);
    if (lt) cublasLtDestroy(lt);
    cudaFree(workspace);
    cudaStreamDestroy(cs);
    cudaStreamDestroy(ks);
  }

  void fill(void* p, std::int64_t elems, int dtype, std::uint64_t salt) {
    coll_check(lagom_fill_random(p, elems, dtype, opts.seed * 1000003ull + salt + 7919ull * rank, 0.02f, cs),
               "fill");
  }

  void build_gemms() {
    std::uint64_t salt = 1;
    gemms.resize(dag.compute_ops.size());
    for (std::size_t i = 0; i < dag.compute_ops.size(); ++i) {
      for (const GemmShape& s : dag.compute_ops[i].gemms) {
        Gemm g;
        g.shape = s;
        // TN (the fast sm_100 layout): A stored k x m (transposed), B k x n,
        // D m x n, all column-major bf16; fp32 compute.
        lt_check(cublasLtMatmulDescCreate(&g.desc, CUBLAS_COMPUTE_32F, CUDA_R_32F), "desc");
        const cublasOperation_t opA = CUBLAS_OP_T, opB = CUBLAS_OP_N;
        lt_check(cublasLtMatmulDescSetAttribute(g.desc, CUBLASLT_MATMUL_DESC_TRANSA, &opA, sizeof opA), "transa");
        lt_check(cublasLtMatmulDescSetAttribute(g.desc, CUBLASLT_MATMUL_DESC_TRANSB, &opB, sizeof opB), "transb");
        lt_check(cublasLtMatrixLayoutCreate(&g.a, CUDA_R_16BF, s.k, s.m, s.k), "layout a");
        lt_check(cublasLtMatrixLayoutCreate(&g.b, CUDA_R_16BF, s.k, s.n, s.k), "layout b");
        lt_check(cublasLtMatrixLayoutCreate(&g.d, CUDA_R_16BF, s.m, s.n, s.m), "layout d");
        if (s.batch > 1) {
          const int32_t bc = static_cast<int32_t>(s.batch);
          const int64_t sa = s.k * s.m, sb = s.k * s.n, sd = s.m * s.n;
          for (auto [lay, stride] : {std::pair{g.a, sa}, std::pair{g.b, sb}, std::pair{g.d, sd}}) {
            lt_check(cublasLtMatrixLayoutSetAttribute(lay, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof bc), "batch");
            lt_check(cublasLtMatrixLayoutSetAttribute(lay, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &stride,
                                                      sizeof stride),
                     "stride");
          }
        }
        // Operands are shared between GEMMs of identical shape (all layers of
        // a model): the values are synthetic and these GEMMs are compute-bound,
        // so sharing only bounds memory (a 32-layer DAG fits in HBM).
        const auto key = std::make_tuple(s.m, s.n, s.k, s.batch);
        auto hit = operands.find(key);
        if (hit == operands.end()) {
          const std::int64_t na = s.k * s.m * s.batch, nb = s.k * s.n * s.batch, nd = s.m * s.n * s.batch;
          std::array<void*, 3> p{};
          cuda_check(cudaMalloc(&p[0], na * 2), "gemm A");
          cuda_check(cudaMalloc(&p[1], nb * 2), "gemm B");
          cuda_check(cudaMalloc(&p[2], nd * 2), "gemm D");
          fill(p[0], na, LAGOM_BF16, salt++);
          fill(p[1], nb, LAGOM_BF16, salt++);
          hit = operands.emplace(key, p).first;
        }
        g.A = hit->second[0];
        g.B = hit->second[1];
        g.D = hit->second[2];
        g.algo = fastest_algo(g, g.desc, 0);
        gemms[i].push_back(g);
      }
    }
  }

  void build_attention() {
    attention.resize(dag.compute_ops.size());
    std::int64_t ws = 0;
    for (std::size_t i = 0; i < dag.compute_ops.size(); ++i)
      for (const AttentionShape& a : dag.compute_ops[i].attention) {
        if (!cudnn) cudnn = create_cudnn_handle();
        Attention* hit = nullptr;
        for (auto& p : attn_pool) {
          const AttentionShape& s = p->shape();
          if (s.batch == a.batch && s.heads == a.heads && s.seq == a.seq && s.head_dim == a.head_dim &&
              s.causal == a.causal && s.backward == a.backward)
            hit = p.get();
        }
        if (!hit) {
          attn_pool.push_back(std::make_unique<Attention>(a, cudnn, opts.seed * 7777 + attn_pool.size() + 97 * rank, cs));
          hit = attn_pool.back().get();
          ws = std::max(ws, hit->workspace_bytes());
        }
        attention[i].push_back(hit);
      }
    ensure_attn_workspace(ws);
  }

  std::int64_t attn_ws_bytes = 0;
  void ensure_attn_workspace(std::int64_t bytes) {
    if (bytes <= attn_ws_bytes) return;
    cuda_check(cudaDeviceSynchronize(), "sync");
    if (attn_workspace) cudaFree(attn_workspace);
    cuda_check(cudaMalloc(&attn_workspace, static_cast<std::size_t>(bytes)), "attention workspace");
    attn_ws_bytes = bytes;
  }

  void build_comms() {
    std::unordered_map<std::string, int> index;
    for (std::size_t i = 0; i < dag.compute_ops.size(); ++i) index[dag.compute_ops[i].id] = static_cast<int>(i);
    std::uint64_t salt = 1ull << 32;
    for (const ReplayCommOp& op : dag.comm_ops) {
      Comm c;
      c.op = op;
      if (op.ready_after) {
        auto it = index.find(*op.ready_after);
        if (it == index.end())
          throw Error(ErrorCode::InvalidWorkload, op.id + ".ready_after", "names no compute op");
        c.dep = it->second;
      }
      const bool in_full = op.collective == Collective::ReduceScatter || op.collective == Collective::AllToAll;
      const bool out_full = op.collective == Collective::AllGather || op.collective == Collective::AllToAll;
      c.in_elems = op.count * (in_full ? n : 1);
      c.out_elems = op.count * (out_full ? n : 1);
      const int e = elem_bytes(op.dtype);
      const std::int64_t in_b = std::max<std::int64_t>(16, c.in_elems * e);
      const std::int64_t out_b = std::max<std::int64_t>(16, c.out_elems * e);
      if (nvls_on) {  // symmetric multicast region: TREE runs in the switch
        coll_check(lagom_comm_nvls_alloc(lcomm, in_b, &c.send), "nvls alloc");
        coll_check(lagom_comm_nvls_alloc(lcomm, out_b, &c.recv), "nvls alloc");
        c.nvls = true;
      } else {
        cuda_check(cudaMalloc(&c.send, in_b), "comm send");
        cuda_check(cudaMalloc(&c.recv, out_b), "comm recv");
      }
      fill(c.send, c.in_elems, op.dtype, salt++);
      comms.push_back(c);
    }
  }

  void build_comm_backends() {
    lagom_comm_opts_t o;
    lagom_comm_default_opts(&o);
    o.max_channels = opts.max_channels;
    o.max_chunk_bytes = opts.max_chunk_bytes;
    o.use_tma = opts.use_tma ? 1 : 0;
    o.coresident = opts.coresident ? 1 : 0;
    o.one_hop = opts.one_hop;
    o.a2a_tma = opts.a2a_tma ? 1 : 0;
    coll_check(lagom_comm_create(rank, n, opts.device, &o, &lcomm), "lagom_comm_create");
    if (n > 1) {
      unsigned char mine[LAGOM_HANDLE_BYTES];
      coll_check(lagom_comm_export_handle(lcomm, mine), "export");
      std::vector<unsigned char> all(static_cast<std::size_t>(n) * LAGOM_HANDLE_BYTES);
      coord.allgather(mine, LAGOM_HANDLE_BYTES, all.data());
      coll_check(lagom_comm_import_handles(lcomm, all.data()), "import");
    }
    // NVLS region sized for every comm op's send + recv buffers (4 KiB aligned).
    if (opts.nvls && n > 1 && lagom_comm_nvls_supported(lcomm)) {
      std::int64_t need = 1 << 20, rs_slot = 0;
      for (const ReplayCommOp& op : dag.comm_ops)
        if (op.collective == Collective::ReduceScatter)
          rs_slot = std::max<std::int64_t>(rs_slot, op.count * elem_bytes(op.dtype));
      if (opts.one_hop && rs_slot > 0) need += (rs_slot + 4095) / 4096 * 4096 * n + 4096;  // push-RS scratch
      for (const ReplayCommOp& op : dag.comm_ops) {
        const bool in_full = op.collective == Collective::ReduceScatter || op.collective == Collective::AllToAll;
        const bool out_full = op.collective == Collective::AllGather || op.collective == Collective::AllToAll;
        const std::int64_t e = elem_bytes(op.dtype);
        need += (op.count * e * (in_full ? n : 1) + 8191) / 4096 * 4096;
        need += (op.count * e * (out_full ? n : 1) + 8191) / 4096 * 4096;
      }
      // Every step is agreed on by all ranks (max-reduce of a failure flag):
      // if any rank cannot create, import or bind the multicast region, all
      // ranks fall back to the P2P kernels together instead of hanging.
      auto agree = [&](bool ok) {
        double bad = ok ? 0.0 : 1.0;
        coord.allreduce_max(&bad, 1);
        return bad == 0.0;
      };
      unsigned char blob[LAGOM_HANDLE_BYTES];
      bool ok = agree(lagom_comm_nvls_export(lcomm, need, blob) == LAGOM_OK);
      if (ok) {
        coord.broadcast(blob, sizeof blob, 0);
        ok = agree(lagom_comm_nvls_import(lcomm, blob) == LAGOM_OK);
      }
      if (ok) ok = agree(lagom_comm_nvls_bind(lcomm) == LAGOM_OK);
      // push ReduceScatter scratch (co-resident one-hop configs) only where one hop applies
      const bool hop = opts.one_hop == 1 || (opts.one_hop == 2 && n == 2);
      if (ok && hop && rs_slot > 0) coll_check(lagom_comm_nvls_scratch(lcomm, rs_slot), "nvls scratch");
      nvls_on = ok;
      if (ok) {  // peer mappings: one-hop AllToAll (TREE) into the peers' recv buffers
        unsigned char mine[LAGOM_HANDLE_BYTES];
        bool pok = agree(lagom_comm_nvls_export_peer(lcomm, mine) == LAGOM_OK);
        if (pok) {
          std::vector<unsigned char> all(static_cast<std::size_t>(n) * LAGOM_HANDLE_BYTES);
          coord.allgather(mine, LAGOM_HANDLE_BYTES, all.data());
          pok = agree(lagom_comm_nvls_import_peers(lcomm, all.data()) == LAGOM_OK);
        }
        if (pok) coll_check(lagom_comm_nvls_use_peers(lcomm, 1), "nvls peers");
        nvls_peers_on = pok;
        if (!pok && rank == 0 && trace_on())
          std::fprintf(stderr, "[lagom] NVLS peer mappings unavailable (%s); AllToAll stays staged\n",
                       lagom_last_error());
      }
      if (!ok && rank == 0 && trace_on())
        std::fprintf(stderr, "[lagom] NVLS unavailable (%s); TREE uses the P2P kernels\n", lagom_last_error());
    }
    if (opts.enable_nccl) {
      ncclUniqueId id{};
      if (rank == 0) nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
      coord.broadcast(&id, sizeof id, 0);
      nccl_check(nccl().CommInitRank(&ncomm, n, id, rank), "ncclCommInitRank");
    }
  }

  // The fastest of cuBLASLt's top heuristic candidates for this shape and SM
  // target, timed here once (cached per shape and target). Every arm —
  // isolated compute, NCCL, Lagom with or without the SM partition — thus
  // runs the best GEMM kernel cuBLASLt has for its SM budget, so no arm gains
  // or loses from a heuristic's mispick (the first candidate is not always
  // the fastest on sm_100: e.g. Mixtral's expert GEMMs ran faster under an
  // SM count target than at the full GPU with the first candidate).
  std::map<std::tuple<std::int64_t, std::int64_t, std::int64_t, std::int64_t, int>, cublasLtMatmulAlgo_t> algo_cache;
  cublasLtMatmulAlgo_t fastest_algo(Gemm& g, cublasLtMatmulDesc_t desc, int sm_target) {
    const auto key = std::make_tuple(g.shape.m, g.shape.n, g.shape.k, g.shape.batch, sm_target);
    if (auto it = algo_cache.find(key); it != algo_cache.end()) return it->second;
    cublasLtMatmulPreference_t pref;
    lt_check(cublasLtMatmulPreferenceCreate(&pref), "pref");
    lt_check(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &workspace_bytes,
                                                  sizeof workspace_bytes),
             "pref ws");
    constexpr int kCands = 8;
    cublasLtMatmulHeuristicResult_t res[kCands]{};
    int found = 0;
    lt_check(cublasLtMatmulAlgoGetHeuristic(lt, desc, g.a, g.b, g.d, g.d, pref, kCands, res, &found), "heuristic");
    cublasLtMatmulPreferenceDestroy(pref);
    if (found < 1) throw Error(ErrorCode::IoFailure, "cublasLt", "no algorithm for the GEMM shape");
    // Rank 0 times the candidates and every rank takes its pick (identical
    // candidate lists: same device, same cuBLASLt): ranks that ran different
    // GEMM kernels would drift apart within a layer, and the gated
    // collectives would then wait for the slowest rank at every step.
    std::int32_t best = 0;
    if (found > 1 && opts.autotune_gemms && rank == 0) {
      cudaEvent_t e0, e1;
      cuda_check(cudaEventCreate(&e0), "event");
      cuda_check(cudaEventCreate(&e1), "event");
      float best_ms = 1e30f;
      const float alpha = 1.0f, beta = 0.0f;
      for (int c = 0; c < found; ++c) {
        if (res[c].state != CUBLAS_STATUS_SUCCESS) continue;
        auto run = [&] {
          return cublasLtMatmul(lt, desc, &alpha, g.A, g.a, g.B, g.b, &beta, g.D, g.d, g.D, g.d, &res[c].algo,
                                workspace, workspace_bytes, cs);
        };
        if (run() != CUBLAS_STATUS_SUCCESS) continue;  // warm-up (and skip algos that refuse)
        cuda_check(cudaEventRecord(e0, cs), "record");
        for (int r = 0; r < 5; ++r) lt_check(run(), "cublasLtMatmul (autotune)");
        cuda_check(cudaEventRecord(e1, cs), "record");
        cuda_check(cudaEventSynchronize(e1), "sync");
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
        if (ms < best_ms) {
          best_ms = ms;
          best = c;
        }
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    if (opts.autotune_gemms && n > 1) coord.broadcast(&best, sizeof best, 0);
    if (best >= found) best = 0;
    return algo_cache.emplace(key, res[best].algo).first->second;
  }

  // A plan for `sm_target` SMs (0 = the whole GPU): the SM partition that
  // leaves the collective's NC channels their own SMs (the contention
  // model's lambda - NC). Cached per target.
  const Plan& plan_for(Gemm& g, int sm_target) {
    auto it = g.by_sm_target.find(sm_target);
    if (it != g.by_sm_target.end()) return it->second;
    Plan p;
    lt_check(cublasLtMatmulDescCreate(&p.desc, CUBLAS_COMPUTE_32F, CUDA_R_32F), "desc");
    const cublasOperation_t opA = CUBLAS_OP_T, opB = CUBLAS_OP_N;
    lt_check(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_TRANSA, &opA, sizeof opA), "transa");
    lt_check(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_TRANSB, &opB, sizeof opB), "transb");
    const int32_t target = sm_target;
    lt_check(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_SM_COUNT_TARGET, &target, sizeof target),
             "sm target");
    p.algo = fastest_algo(g, p.desc, sm_target);
    return g.by_sm_target.emplace(sm_target, p).first->second;
  }

  void launch_gemm(Gemm& g, int sm_target) {
    const float alpha = 1.0f, beta = 0.0f;
    const cublasLtMatmulDesc_t desc = sm_target > 0 ? plan_for(g, sm_target).desc : g.desc;
    const cublasLtMatmulAlgo_t* algo = sm_target > 0 ? &plan_for(g, sm_target).algo : &g.algo;
    lt_check(cublasLtMatmul(lt, desc, &alpha, g.A, g.a, g.B, g.b, &beta, g.D, g.d, g.D, g.d, algo, workspace,
                            workspace_bytes, cs),
             "cublasLtMatmul");
  }

  lagom_coll_args_t coll_args(const Comm& c, const CommConfig& cfg, unsigned long long* span) const {
    lagom_coll_args_t a{};
    a.collective = coll_code(c.op.collective);
    a.algorithm = cfg.algorithm == Algorithm::Tree ? LAGOM_TREE : LAGOM_RING;
    a.protocol = static_cast<int>(cfg.protocol);
    a.num_channels = cfg.num_channels;
    a.num_threads = cfg.num_threads;
    a.chunk_bytes = cfg.chunk_size;
    a.dtype = c.op.dtype;
    a.redop = LAGOM_SUM;
    a.count = c.op.count;
    a.span_out = span;
    return a;
  }

  // Whether comm j's kernel at `cfg` fits next to a GEMM CTA on one SM
  // (lagom_coll_footprint), cached per (op, config).
  std::map<std::tuple<std::size_t, int, int, int, int>, bool> fits_cache;
  bool coresident(std::size_t j, const CommConfig& cfg) {
    const auto key = std::make_tuple(j, static_cast<int>(cfg.algorithm), static_cast<int>(cfg.protocol),
                                     cfg.num_channels, cfg.num_threads);
    auto it = fits_cache.find(key);
    if (it != fits_cache.end()) return it->second;
    const lagom_coll_args_t a = coll_args(comms[j], cfg, nullptr);
    int regs = 0, smem = 0;
    coll_check(lagom_coll_footprint(lcomm, &a, comms[j].send, comms[j].recv, &regs, &smem), "footprint");
    const bool fits = regs * cfg.num_threads <= kCoresidentRegs && smem <= kCoresidentSmem;
    return fits_cache.emplace(key, fits).first->second;
  }

  void launch_comm_lagom(const Comm& c, const CommConfig& cfg, unsigned long long* span) {
    const lagom_coll_args_t a = coll_args(c, cfg, span);
    coll_check(lagom_coll_launch(lcomm, &a, c.send, c.recv, ks), c.op.id.c_str());
  }

  void launch_comm_nccl(const Comm& c) {
    const NcclApi& api = nccl();
    const ncclDataType_t t = nccl_type(c.op.dtype);
    const std::size_t cnt = static_cast<std::size_t>(c.op.count);
    switch (c.op.collective) {
      case Collective::AllReduce:
        nccl_check(api.AllReduce(c.send, c.recv, cnt, t, ncclSum, ncomm, ks), "ncclAllReduce");
        break;
      case Collective::AllGather:
        nccl_check(api.AllGather(c.send, c.recv, cnt, t, ncomm, ks), "ncclAllGather");
        break;
      case Collective::ReduceScatter:
        nccl_check(api.ReduceScatter(c.send, c.recv, cnt, t, ncclSum, ncomm, ks), "ncclReduceScatter");
        break;
      case Collective::AllToAll: {
        const std::size_t bytes = cnt * elem_bytes(c.op.dtype);
        nccl_check(api.GroupStart(), "group");
        for (int p = 0; p < n; ++p) {
          nccl_check(api.Send(static_cast<char*>(c.send) + p * bytes, cnt, t, p, ncomm, ks), "send");
          nccl_check(api.Recv(static_cast<char*>(c.recv) + p * bytes, cnt, t, p, ncomm, ks), "recv");
        }
        nccl_check(api.GroupEnd(), "group");
        break;
      }
    }
  }

  // One replay on this rank; returns [x_0..x_{N-1}, y_0..y_{M-1}, Z,
  // xev_0..xev_{N-1}] in us (x: kernel span for Lagom kernels, else events;
  // xev: events).
  std::vector<double> replay(Mode mode, const std::vector<CommConfig>* cfgs) {
    const bool do_compute = mode != Mode::CommOnly;
    const bool do_comm = mode != Mode::ComputeOnly;
    const std::size_t M = dag.compute_ops.size(), N = comms.size();
    // SM partition (opts.reserve_comm_sms): in Lagom modes compute op i runs
    // its GEMMs on num_sms - (max NC of the collectives that can overlap it),
    // so those CTAs never queue behind the GEMMs. Collective j, gated on
    // compute op d (or ungated, d = -1), can only run during ops i > d; ops
    // no collective can overlap (e.g. before the first gate) keep the whole
    // GPU, and collectives gated on the last op cost the GEMMs nothing.
    std::vector<int> sm_target(M, 0);
    const bool lagom_part =
        opts.sm_partition != kPartitionNone && cfgs && (mode == Mode::Lagom || mode == Mode::LagomE2E);
    const bool nccl_part = opts.nccl_reserve_sms > 0 && mode == Mode::Nccl;
    if (lagom_part || nccl_part) {
      std::vector<int> reserve(M, 0);
      for (std::size_t j = 0; j < N; ++j) {
        const int r = nccl_part ? opts.nccl_reserve_sms
                      : (opts.sm_partition == kPartitionAll || !coresident(j, (*cfgs)[j])) ? (*cfgs)[j].num_channels
                                                                                          : 0;
        for (std::size_t i = static_cast<std::size_t>(comms[j].dep + 1); i < M; ++i)
          reserve[i] = std::max(reserve[i], r);
      }
      for (std::size_t i = 0; i < M; ++i)
        if (reserve[i] > 0) sm_target[i] = std::max(1, num_sms - reserve[i]);
    }
    // Plans for new SM targets are built (and their algorithms timed) here,
    // before the barrier and the start event — never inside the measurement.
    if (do_compute)
      for (std::size_t i = 0; i < M; ++i)
        if (sm_target[i] > 0) {
          for (Gemm& g : gemms[i]) plan_for(g, sm_target[i]);
          for (Attention* at : attention[i]) {
            at->prepare(cudnn, sm_target[i]);
            ensure_attn_workspace(at->workspace_bytes());
          }
        }
    coord.barrier();
    const bool e2e = mode == Mode::LagomE2E;
    cuda_check(cudaEventRecord(ev_start, cs), "record");
    if (pm_on) coll_check(lagom_timestamp(stamp, cs), "timestamp");
    if (e2e && host_in)
      cuda_check(cudaMemcpyAsync(gemms[0][0].A, host_in, opts.e2e_in_bytes, cudaMemcpyHostToDevice, cs), "h2d");
    cuda_check(cudaStreamWaitEvent(ks, ev_start, 0), "wait");
    const bool spans_on = do_comm && spans && mode != Mode::Nccl;
    if (spans_on) {
      // {start, end} pairs: start <- UINT64_MAX, end <- 0
      cuda_check(cudaMemset2DAsync(spans, 2 * sizeof(unsigned long long), 0xff, sizeof(unsigned long long), N, ks),
                 "span init");
      cuda_check(cudaMemset2DAsync(spans + 1, 2 * sizeof(unsigned long long), 0, sizeof(unsigned long long), N, ks),
                 "span init");
    }
    if (do_compute) {
      for (std::size_t i = 0; i < M; ++i) {
        cuda_check(cudaEventRecord(ev_cb[i], cs), "record");
        for (Gemm& g : gemms[i]) launch_gemm(g, sm_target[i]);
        for (Attention* at : attention[i]) at->launch(cudnn, cs, attn_workspace, sm_target[i]);
        cuda_check(cudaEventRecord(ev_ce[i], cs), "record");
      }
    }
    if (do_comm) {
      for (std::size_t j = 0; j < N; ++j) {
        if (do_compute && comms[j].dep >= 0) cuda_check(cudaStreamWaitEvent(ks, ev_ce[comms[j].dep], 0), "wait");
        cuda_check(cudaEventRecord(ev_kb[j], ks), "record");
        if (mode == Mode::Nccl) launch_comm_nccl(comms[j]);
        else launch_comm_lagom(comms[j], (*cfgs)[j], spans ? spans + 2 * j : nullptr);
        cuda_check(cudaEventRecord(ev_ke[j], ks), "record");
      }
    }
    cuda_check(cudaEventRecord(ev_kend, ks), "record");
    if (e2e && host_out) {
      cuda_check(cudaStreamWaitEvent(cs, ev_kend, 0), "wait");
      cuda_check(cudaMemcpyAsync(host_out, comms.back().recv, opts.e2e_out_bytes, cudaMemcpyDeviceToHost, cs), "d2h");
    }
    cuda_check(cudaEventRecord(ev_cend, cs), "record");
    cuda_check(cudaEventSynchronize(ev_cend), "sync");
    cuda_check(cudaEventSynchronize(ev_kend), "sync");
    coll_check(lagom_comm_check(lcomm), "collective watchdog");

    std::vector<double> out(N + M + 1 + N, 0.0);
    auto us = [](cudaEvent_t a, cudaEvent_t b) {
      float ms = 0.f;
      cuda_check(cudaEventElapsedTime(&ms, a, b), "elapsed");
      return static_cast<double>(ms) * 1e3;
    };
    double z = 0.0;
    if (do_comm)
      for (std::size_t j = 0; j < N; ++j) out[j] = out[N + M + 1 + j] = us(ev_kb[j], ev_ke[j]);
    if (spans_on) {
      // x_j = the kernel's active span (first CTA start .. last CTA end):
      // excludes time the launch sat queued behind persistent GEMM CTAs.
      cuda_check(cudaMemcpy(spans_host.data(), spans, 2 * N * sizeof(unsigned long long), cudaMemcpyDeviceToHost),
                 "spans");
      for (std::size_t j = 0; j < N; ++j) {
        const unsigned long long a = spans_host[2 * j], b = spans_host[2 * j + 1];
        if (b >= a && a != ~0ull) out[j] = static_cast<double>(b - a) * 1e-3;
      }
    }
    if (do_compute)
      for (std::size_t i = 0; i < M; ++i) out[N + i] = us(ev_cb[i], ev_ce[i]);
    z = std::max(us(ev_start, ev_cend), us(ev_start, ev_kend));
    out[N + M] = z;
    last_timeline.clear();
    if (do_compute)
      for (std::size_t i = 0; i < M; ++i)
        last_timeline.push_back({"compute", dag.compute_ops[i].id, us(ev_start, ev_cb[i]), out[N + i],
                                 model_blocks[i]});
    if (do_comm)
      for (std::size_t j = 0; j < N; ++j)
        last_timeline.push_back({"comm", dag.comm_ops[j].id, us(ev_start, ev_kb[j]), out[j], 0});
    return out;
  }

  ReplayMeasurement measure(Mode mode, const std::vector<CommConfig>* cfgs) {
    return measure(mode, cfgs, opts.repeats, opts.warmup);
  }

  ReplayMeasurement measure(Mode mode, const std::vector<CommConfig>* cfgs, int repeats, int warmup) {
    const auto t0 = std::chrono::steady_clock::now();
    if (trace_on())
      std::fprintf(stderr, "[lagom rank %d %.3f] measure mode=%d repeats=%d warmup=%d\n", rank, now_s(),
                   static_cast<int>(mode), repeats, warmup);
    if (cfgs && cfgs->size() != comms.size())
      throw Error(ErrorCode::InvalidWorkload, "configs",
                  "expected " + std::to_string(comms.size()) + " configs, got " + std::to_string(cfgs->size()));
    if (pm_on && !sampler) {
      sampler = std::make_unique<PmSampler>(opts.device, opts.pm_metrics, opts.pm_interval_ns);
      cuda_check(cudaMalloc(&stamp, sizeof(unsigned long long)), "stamp");
    }
    for (int w = 0; w < warmup; ++w) replay(mode, cfgs);
    const std::size_t N = comms.size(), M = dag.compute_ops.size();
    std::vector<std::vector<double>> reps;
    std::vector<PmSample> samples;
    std::uint64_t t0_ns = 0;
    for (int r = 0; r < std::max(1, repeats); ++r) {
      if (pm_on) sampler->start();
      std::vector<double> v = replay(mode, cfgs);
      if (pm_on) {
        samples = sampler->stop();  // the last repeat's samples are reported
        cuda_check(cudaMemcpy(&t0_ns, stamp, sizeof t0_ns, cudaMemcpyDeviceToHost), "stamp");
      }
      coord.allreduce_max(v.data(), v.size());
      reps.push_back(std::move(v));
    }
    ReplayMeasurement m;
    if (pm_on) {
      m.pm_metrics = sampler->metrics();
      m.pm_samples = std::move(samples);
      m.pm_t0_ns = t0_ns;
    }
    m.profile.comm_times.resize(N);
    m.comp_times.resize(M);
    std::vector<double> col(reps.size());
    auto med = [&](std::size_t k) {
      for (std::size_t r = 0; r < reps.size(); ++r) col[r] = reps[r][k];
      return median_of(col);
    };
    for (std::size_t j = 0; j < N; ++j) m.profile.comm_times[j] = med(j);
    for (std::size_t i = 0; i < M; ++i) m.comp_times[i] = med(N + i);
    m.profile.total_comm = 0.0;
    for (double x : m.profile.comm_times) m.profile.total_comm += x;
    m.profile.total_compute = 0.0;
    for (double y : m.comp_times) m.profile.total_compute += y;
    m.profile.makespan = med(N + M);
    m.comm_event_times.resize(N);
    for (std::size_t j = 0; j < N; ++j) m.comm_event_times[j] = med(N + M + 1 + j);
    m.timeline = last_timeline;
    ++calls;
    m.wall_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    if (trace_on())
      std::fprintf(stderr, "[lagom rank %d %.3f] done mode=%d Z=%.1fus wall=%.1fms\n", rank, now_s(),
                   static_cast<int>(mode), m.profile.makespan, m.wall_us / 1e3);
    return m;
  }

  // rank-0 side of the command protocol
  ReplayMeasurement remote(Mode mode, const std::vector<CommConfig>* cfgs) {
    if (rank != 0) throw Error(ErrorCode::InvalidInput, "engine", "remote_* is rank 0 only");
    std::vector<WireConfig> wire(comms.size() + 1);
    wire[0].algorithm = static_cast<std::int32_t>(mode);
    wire[0].protocol = opts.repeats;  // measurement settings travel with the command
    wire[0].transport = opts.warmup;
    wire[0].num_channels = opts.sm_partition;
    wire[0].num_threads = opts.nccl_reserve_sms;
    wire[0].pad = pm_on ? 1 : 0;
    if (cfgs) {
      if (cfgs->size() != comms.size())
        throw Error(ErrorCode::InvalidWorkload, "configs", "one config per comm op expected");
      for (std::size_t j = 0; j < cfgs->size(); ++j) {
        const CommConfig& c = (*cfgs)[j];
        wire[j + 1] = WireConfig{static_cast<std::int32_t>(c.algorithm), static_cast<std::int32_t>(c.protocol),
                                 static_cast<std::int32_t>(c.transport), c.num_channels, c.num_threads, 0,
                                 c.chunk_size};
      }
    }
    coord.broadcast(wire.data(), wire.size() * sizeof(WireConfig), 0);
    if (mode == Mode::Stop) return {};
    return measure(mode, cfgs, opts.repeats, opts.warmup);
  }
};

ReplayEngine::ReplayEngine(const ReplayDag& dag, Coordinator& coord, const ReplayOptions& opts)
    : impl_(std::make_unique<Impl>(dag, coord, opts)) {}
ReplayEngine::~ReplayEngine() = default;

const ReplayDag& ReplayEngine::dag() const { return impl_->dag; }
int ReplayEngine::rank() const { return impl_->rank; }
int ReplayEngine::nranks() const { return impl_->n; }
int ReplayEngine::calls() const { return impl_->calls; }
void ReplayEngine::set_measurement(int repeats, int warmup) {
  impl_->opts.repeats = std::max(1, repeats);
  impl_->opts.warmup = std::max(0, warmup);
}
void ReplayEngine::set_partition(int sm_partition, int nccl_reserve_sms) {
  if (sm_partition < kPartitionNone || sm_partition > kPartitionAll)
    throw Error(ErrorCode::InvalidInput, "sm_partition", "must be 0 (none), 1 (auto) or 2 (all)");
  impl_->opts.sm_partition = sm_partition;
  impl_->opts.nccl_reserve_sms = std::max(0, std::min(nccl_reserve_sms, impl_->num_sms - 1));
}
bool ReplayEngine::nvls_active() const { return impl_->nvls_on; }
void ReplayEngine::set_pm_sampling(bool on) { impl_->pm_on = on; }
bool ReplayEngine::nvls_peers_active() const { return impl_->nvls_peers_on; }

ReplayMeasurement ReplayEngine::run(const std::vector<CommConfig>& configs) {
  return impl_->measure(Mode::Lagom, &configs);
}
ReplayMeasurement ReplayEngine::run_e2e(const std::vector<CommConfig>& configs) {
  return impl_->measure(Mode::LagomE2E, &configs);
}
ReplayMeasurement ReplayEngine::run_nccl() {
  if (!impl_->ncomm) throw Error(ErrorCode::InvalidInput, "engine", "NCCL baseline disabled");
  return impl_->measure(Mode::Nccl, nullptr);
}
ReplayMeasurement ReplayEngine::run_compute_only() { return impl_->measure(Mode::ComputeOnly, nullptr); }
ReplayMeasurement ReplayEngine::run_comm_only(const std::vector<CommConfig>& configs) {
  return impl_->measure(Mode::CommOnly, &configs);
}

void ReplayEngine::serve() {
  Impl& I = *impl_;
  if (I.rank == 0) return;
  for (;;) {
    std::vector<WireConfig> wire(I.comms.size() + 1);
    I.coord.broadcast(wire.data(), wire.size() * sizeof(WireConfig), 0);
    const Mode mode = static_cast<Mode>(wire[0].algorithm);
    if (mode == Mode::Stop) return;
    std::vector<CommConfig> cfgs(I.comms.size());
    for (std::size_t j = 0; j < cfgs.size(); ++j) {
      const WireConfig& w = wire[j + 1];
      cfgs[j] = CommConfig{static_cast<Algorithm>(w.algorithm), static_cast<Protocol>(w.protocol),
                           static_cast<Transport>(w.transport), w.num_channels, w.num_threads, w.chunk_size};
    }
    I.opts.sm_partition = wire[0].num_channels;
    I.opts.nccl_reserve_sms = wire[0].num_threads;
    I.pm_on = wire[0].pad != 0;
    const bool with_cfg = mode == Mode::Lagom || mode == Mode::CommOnly || mode == Mode::LagomE2E;
    I.measure(mode, with_cfg ? &cfgs : nullptr, wire[0].protocol, wire[0].transport);
  }
}

void ReplayEngine::stop() {
  if (impl_->rank == 0 && impl_->n > 1) impl_->remote(Mode::Stop, nullptr);
}
ReplayMeasurement ReplayEngine::remote_run(const std::vector<CommConfig>& c) { return impl_->remote(Mode::Lagom, &c); }
ReplayMeasurement ReplayEngine::remote_run_e2e(const std::vector<CommConfig>& c) {
  return impl_->remote(Mode::LagomE2E, &c);
}
ReplayMeasurement ReplayEngine::remote_run_nccl() {
  if (!impl_->ncomm) throw Error(ErrorCode::InvalidInput, "engine", "NCCL baseline disabled");
  return impl_->remote(Mode::Nccl, nullptr);
}
ReplayMeasurement ReplayEngine::remote_run_compute_only() { return impl_->remote(Mode::ComputeOnly, nullptr); }
ReplayMeasurement ReplayEngine::remote_run_comm_only(const std::vector<CommConfig>& c) {
  return impl_->remote(Mode::CommOnly, &c);
}

// --------------------------------------------------------------- profilers --

ProfileFn make_gpu_profiler(ReplayEngine& engine,
                            std::vector<std::pair<std::vector<CommConfig>, ProfileResult>>* record) {
  return [&engine, record](const std::vector<CommConfig>& configs) {
    ReplayMeasurement m = engine.remote_run(configs);
    if (record) record->emplace_back(configs, m.profile);
    return m.profile;
  };
}

Workload grouped_workload(const ReplayDag& dag, const std::vector<int>& group_of_op, const GpuSpec& gpu,
                          int nranks) {
  if (group_of_op.size() != dag.comm_ops.size())
    throw Error(ErrorCode::InvalidInput, "groups", "one group id per comm op expected");
  const Workload full = to_workload(dag, gpu, nranks);
  Workload w;
  w.gpu = full.gpu;
  w.compute_ops = full.compute_ops;
  const int groups = group_of_op.empty() ? 0 : *std::max_element(group_of_op.begin(), group_of_op.end()) + 1;
  for (int g = 0; g < groups; ++g) {
    const auto it = std::find(group_of_op.begin(), group_of_op.end(), g);
    if (it == group_of_op.end()) throw Error(ErrorCode::InvalidInput, "groups", "group ids must be dense");
    CommOp op = full.comm_ops[static_cast<std::size_t>(it - group_of_op.begin())];
    op.id = "group" + std::to_string(g) + ":" + op.id;
    w.comm_ops.push_back(op);
  }
  return w;
}

ProfileFn make_grouped_gpu_profiler(ReplayEngine& engine, std::vector<int> group_of_op,
                                    std::vector<std::pair<std::vector<CommConfig>, ProfileResult>>* record) {
  return [&engine, groups = std::move(group_of_op), record](const std::vector<CommConfig>& gcfg) {
    std::vector<CommConfig> full(groups.size());
    for (std::size_t j = 0; j < groups.size(); ++j) full[j] = gcfg.at(static_cast<std::size_t>(groups[j]));
    const ReplayMeasurement m = engine.remote_run(full);
    ProfileResult r;
    r.comm_times.assign(gcfg.size(), 0.0);
    for (std::size_t j = 0; j < groups.size(); ++j) r.comm_times[static_cast<std::size_t>(groups[j])] += m.profile.comm_times[j];
    r.total_comm = 0.0;
    for (double x : r.comm_times) r.total_comm += x;
    r.total_compute = m.profile.total_compute;
    r.makespan = m.profile.makespan;
    if (record) record->emplace_back(gcfg, r);
    return r;
  };
}

ProfileFn make_table_profiler(std::vector<std::pair<std::vector<CommConfig>, ProfileResult>> table) {
  auto shared = std::make_shared<decltype(table)>(std::move(table));
  return [shared](const std::vector<CommConfig>& configs) -> ProfileResult {
    for (const auto& [cfg, res] : *shared)
      if (cfg == configs) return res;
    throw Error(ErrorCode::InvalidInput, "profile_table", "no recorded entry for this config vector");
  };
}

}  // namespace lagom::b200
