// GPU-batched exhaustive oracle: the reference's joint grid
// search (reference oracle.cpp:12-63) with one thread per joint grid point.
//
// simulate() is pure (reference SPEC.md:255), so every point is independent.
// Each thread replays the overlap simulator's event loop (overlap_sim.cpp,
// itself the reference's simulator.cpp:32-166 restated) in FP64 with the same
// operations in the same order; this file is compiled with --fmad=false, so
// no multiply-add is contracted and every makespan is bit-identical to the
// CPU's. Per-(comm, grid entry) durations and footprints come from the host's
// comm_time / mem_footprint; the argmin runs on the host in enumeration order
// with the reference's strict-< tie break.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <unordered_map>

#include "lagom/b200.hpp"
#include "lagom/commperf.hpp"
#include "lagom/error.hpp"
#include "lagom/oracle.hpp"

namespace lagom::b200 {

namespace {

constexpr int kMaxOps = 64;  // compute ops and comm ops per workload on the GPU path

struct DevComp {
  long long total_blocks, blocks_per_sm, bytes_per_block;
  double base_wave_time;
};

struct DevArgs {
  int n_comp, n_comm, num_sms;
  double peak_mem_bw, stretch;
  const DevComp* comp;
  const int* gate;            // [n_comm] compute-op index or -1
  const int* grid_size;       // [n_comm]
  const long long* grid_off;  // [n_comm] offset into the flattened tables
  const double* dur;          // comm_time per (comm, entry)
  const double* foot;         // mem_footprint per (comm, entry)
  const int* occ;             // occupied SMs per (comm, entry)
  long long points, first;
  double* out;                // makespan per point
};

__device__ double wave_time_d(const DevComp& op, long long blocks, double footprint, double peak) {
  const double left = peak - footprint;
  const double moved = static_cast<double>(blocks) * static_cast<double>(op.bytes_per_block);
  return op.base_wave_time + moved / left;
}

__global__ void grid_kernel(DevArgs A) {
  const long long p = A.first + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= A.first + A.points) return;
  const double kNever = __longlong_as_double(0x7ff0000000000000LL);
  int entry[kMaxOps];
  long long rest = p;
  for (int j = A.n_comm - 1; j >= 0; --j) {  // odometer: last comm fastest
    entry[j] = static_cast<int>(rest % A.grid_size[j]);
    rest /= A.grid_size[j];
  }
  double work[kMaxOps], start[kMaxOps], end[kMaxOps], op_done[kMaxOps];
  bool finished[kMaxOps];
  for (int j = 0; j < A.n_comm; ++j) {
    work[j] = A.dur[A.grid_off[j] + entry[j]];
    start[j] = end[j] = 0.0;
    finished[j] = false;
  }
  for (int i = 0; i < A.n_comp; ++i) op_done[i] = kNever;
  int next = 0, active = -1;

  auto start_ready = [&](double now) {
    while (active < 0 && next < A.n_comm) {
      const double prev_end = next == 0 ? 0.0 : (finished[next - 1] ? end[next - 1] : kNever);
      const double gate_end = A.gate[next] < 0 ? 0.0 : op_done[A.gate[next]];
      const double s = fmax(prev_end, gate_end);
      if (s > now) return;
      start[next] = s;
      active = next++;
    }
  };
  auto progress = [&](double from, double to, double rate) {
    double t = from;
    start_ready(t);
    while (active >= 0 && t < to) {
      const double need = work[active] / rate;
      if (t + need <= to) {
        t += need;
        work[active] = 0.0;
        finished[active] = true;
        end[active] = t;
        active = -1;
        start_ready(t);
      } else {
        work[active] -= (to - t) * rate;
        t = to;
      }
    }
  };

  double t = 0.0, Y = 0.0;
  double comp_times[kMaxOps];
  for (int i = 0; i < A.n_comp; ++i) {
    const DevComp op = A.comp[i];
    const double begin = t;
    long long left = op.total_blocks;
    while (left > 0) {
      start_ready(t);
      int nc = 0;
      double v = 0.0;
      if (active >= 0) {
        nc = A.occ[A.grid_off[active] + entry[active]];
        v = A.foot[A.grid_off[active] + entry[active]];
      }
      const long long cap = static_cast<long long>(A.num_sms - nc) * op.blocks_per_sm;
      const long long blocks = left < cap ? left : cap;
      const double f = wave_time_d(op, blocks, v, A.peak_mem_bw);
      progress(t, t + f, A.stretch);
      t += f;
      left -= blocks;
    }
    op_done[i] = t;
    comp_times[i] = t - begin;
  }
  const double compute_end = t;
  double ft = compute_end;
  for (;;) {
    start_ready(ft);
    if (active < 0) break;
    ft += work[active];
    work[active] = 0.0;
    finished[active] = true;
    end[active] = ft;
    active = -1;
  }
  double last_end = 0.0, X = 0.0;
  double ct[kMaxOps];
  for (int j = 0; j < A.n_comm; ++j) {
    ct[j] = end[j] - start[j];
    last_end = fmax(last_end, end[j]);
  }
  for (int i = 0; i < A.n_comp; ++i) Y += comp_times[i];
  for (int j = 0; j < A.n_comm; ++j) X += ct[j];
  // std::max({compute_end, last_end, Y, X}): first maximum wins; all are
  // non-negative and finite here, so fmax chains give the same bits.
  A.out[p - A.first] = fmax(fmax(fmax(compute_end, last_end), Y), X);
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(ErrorCode::IoFailure, "cuda", std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

OracleResult exhaustive_gpu(const Workload& w, const std::vector<std::vector<CommConfig>>& grids,
                            const SubspaceParams& params, std::int64_t limit, int device) {
  validate(w);
  const std::size_t N = w.comm_ops.size(), M = w.compute_ops.size();
  // Anything the kernel does not cover (sizes, invalid configs whose error
  // order matters, the empty grid) goes to the CPU oracle unchanged.
  bool gpu_ok = N > 0 && N <= kMaxOps && M <= kMaxOps && grids.size() == N;
  for (std::size_t j = 0; gpu_ok && j < N; ++j) {
    if (grids[j].empty()) gpu_ok = false;
    for (const CommConfig& c : grids[j]) {
      try {
        validate_config(c, w.comm_ops[j], w.gpu);
        (void)params.at(subspace_key(c));
      } catch (const Error&) {
        gpu_ok = false;
      }
    }
  }
  long double points_ld = 1;
  for (const auto& g : grids) points_ld *= static_cast<long double>(g.empty() ? 1 : g.size());
  if (!gpu_ok || limit < 0 || points_ld > static_cast<long double>(limit)) return exhaustive(w, grids, params, limit);
  const long long points = static_cast<long long>(points_ld);

  std::unordered_map<std::string, int> idx;
  for (std::size_t i = 0; i < M; ++i) idx[w.compute_ops[i].id] = static_cast<int>(i);
  std::vector<DevComp> comp(M);
  for (std::size_t i = 0; i < M; ++i) {
    const ComputeOp& c = w.compute_ops[i];
    comp[i] = {c.total_blocks, c.blocks_per_sm, c.bytes_per_block, c.base_wave_time};
  }
  std::vector<int> gate(N), gsize(N), occ;
  std::vector<long long> goff(N);
  std::vector<double> dur, foot;
  for (std::size_t j = 0; j < N; ++j) {
    const CommOp& op = w.comm_ops[j];
    gate[j] = op.ready_after ? idx.at(*op.ready_after) : -1;
    gsize[j] = static_cast<int>(grids[j].size());
    goff[j] = static_cast<long long>(dur.size());
    for (const CommConfig& c : grids[j]) {
      dur.push_back(comm_time(op, c, w.gpu, params));
      foot.push_back(mem_footprint(c, w.gpu, params));
      occ.push_back(c.num_channels);
    }
  }
  check(cudaSetDevice(device), "cudaSetDevice");
  auto up = [](const auto& v, auto** d) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    check(cudaMalloc(reinterpret_cast<void**>(d), std::max<std::size_t>(1, v.size()) * sizeof(T)), "malloc");
    if (!v.empty()) check(cudaMemcpy(*d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "h2d");
  };
  DevComp* d_comp = nullptr;
  int *d_gate = nullptr, *d_gsize = nullptr, *d_occ = nullptr;
  long long* d_goff = nullptr;
  double *d_dur = nullptr, *d_foot = nullptr, *d_out = nullptr;
  up(comp, &d_comp);
  up(gate, &d_gate);
  up(gsize, &d_gsize);
  up(goff, &d_goff);
  up(dur, &d_dur);
  up(foot, &d_foot);
  up(occ, &d_occ);
  const long long batch = std::min<long long>(points, 1 << 22);
  check(cudaMalloc(&d_out, static_cast<std::size_t>(batch) * sizeof(double)), "malloc");
  std::vector<double> z(static_cast<std::size_t>(batch));
  OracleResult best;
  best.makespan = std::numeric_limits<double>::infinity();
  long long best_p = -1;
  for (long long first = 0; first < points; first += batch) {
    const long long cnt = std::min(batch, points - first);
    DevArgs a{static_cast<int>(M), static_cast<int>(N), w.gpu.num_sms, w.gpu.peak_mem_bw,
              1.0 / (1.0 + w.gpu.compute_on_comm_slowdown), d_comp, d_gate, d_gsize, d_goff, d_dur, d_foot, d_occ,
              cnt, first, d_out};
    grid_kernel<<<static_cast<unsigned>((cnt + 127) / 128), 128>>>(a);
    check(cudaGetLastError(), "grid_kernel");
    check(cudaMemcpy(z.data(), d_out, static_cast<std::size_t>(cnt) * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
    for (long long k = 0; k < cnt; ++k)
      if (z[static_cast<std::size_t>(k)] < best.makespan) {  // strict: earliest optimum
        best.makespan = z[static_cast<std::size_t>(k)];
        best_p = first + k;
      }
  }
  for (void* p : {static_cast<void*>(d_comp), static_cast<void*>(d_gate), static_cast<void*>(d_gsize),
                  static_cast<void*>(d_goff), static_cast<void*>(d_dur), static_cast<void*>(d_foot),
                  static_cast<void*>(d_occ), static_cast<void*>(d_out)})
    cudaFree(p);
  best.evaluations = points;
  best.configs.resize(N);
  long long rest = best_p;
  for (std::size_t j = N; j-- > 0;) {
    best.configs[j] = grids[j][static_cast<std::size_t>(rest % gsize[j])];
    rest /= gsize[j];
  }
  return best;
}

}  // namespace lagom::b200
