// Overlap predictor: one compute stream (wave by wave) against one serialized
// comm stream, event-driven. Reference: simulator.cpp:32-174.
//
// Re-designed for speed (this is the tuner's inner loop when the model is the
// profiler, and the exhaustive oracle's only cost): op-id lookups are resolved
// to indices once, config validation builds no strings unless it fails, and
// profile() never materialises the timeline. The floating-point operations and
// their order are exactly the reference's, so every result is bit-identical.
#include <algorithm>
#include <limits>
#include <unordered_map>

#include "lagom/contention.hpp"
#include "lagom/error.hpp"
#include "lagom/simulator.hpp"

namespace lagom {

namespace {

constexpr double kNever = std::numeric_limits<double>::infinity();

struct CommLane {
  double footprint = 0.0;  // V while running
  int occupancy = 0;       // SMs held while running
  int gate = -1;           // index of the ready_after compute op, -1 = none
  bool finished = false;
  double start = 0.0;
  double end = 0.0;
  double work_left = 0.0;  // remaining contention-free duration
};

bool config_ok(const CommConfig& c, const CommOp& op, const GpuSpec& gpu) {
  return c.num_channels >= 1 && c.num_channels <= max_channels(op, gpu) &&
         in_thread_ladder(c.num_threads) && c.chunk_size % kKiB == 0 &&
         c.chunk_size >= op.bounds.c_min && c.chunk_size <= op.bounds.c_max;
}

// The engine. `Trace` selects whether timeline events are recorded.
template <bool Trace>
class OverlapRun {
 public:
  OverlapRun(const Workload& w, const std::vector<CommConfig>& configs,
             const SubspaceParams& params, const SimOptions& opt)
      : w_(w), gpu_(w.gpu) {
    validate(w);
    const std::size_t n = w.comm_ops.size();
    if (configs.size() != n)
      throw Error(ErrorCode::InvalidWorkload, "configs",
                  "expected " + std::to_string(n) + " configs, got " +
                      std::to_string(configs.size()));
    lanes_.resize(n);
    const bool gated = std::any_of(w.comm_ops.begin(), w.comm_ops.end(),
                                   [](const CommOp& c) { return c.ready_after.has_value(); });
    std::unordered_map<std::string_view, int> by_id;
    if (gated) {
      by_id.reserve(w.compute_ops.size());
      for (std::size_t i = 0; i < w.compute_ops.size(); ++i)
        by_id.emplace(w.compute_ops[i].id, static_cast<int>(i));
    }
    for (std::size_t j = 0; j < n; ++j) {
      const CommOp& op = w.comm_ops[j];
      if (!config_ok(configs[j], op, gpu_))
        validate_config(configs[j], op, gpu_, "configs[" + std::to_string(j) + "]");
      CommLane& L = lanes_[j];
      L.work_left = comm_time(op, configs[j], gpu_, params);
      L.footprint = mem_footprint(configs[j], gpu_, params);
      L.occupancy = opt.sm_occupancy ? configs[j].num_channels : 0;
      if (op.ready_after) L.gate = by_id.find(*op.ready_after)->second;
    }
    op_done_.assign(w.compute_ops.size(), kNever);
  }

  void run(std::vector<double>& comp_times, std::vector<double>& comm_times,
           double& Y, double& X, double& Z, std::vector<TimelineEvent>* tl) {
    const double stretch = 1.0 / (1.0 + gpu_.compute_on_comm_slowdown);
    const std::size_t m = w_.compute_ops.size();
    comp_times.assign(m, 0.0);

    double t = 0.0;
    for (std::size_t i = 0; i < m; ++i) {
      const ComputeOp& op = w_.compute_ops[i];
      const double begin = t;
      std::int64_t left = op.total_blocks;
      while (left > 0) {
        start_ready(t);  // a comm becoming startable exactly now is visible
        std::optional<ActiveComm> ac;
        if (active_ >= 0) ac = ActiveComm{lanes_[active_].occupancy, lanes_[active_].footprint};
        const int nc = ac ? ac->num_channels : 0;
        if (nc >= gpu_.num_sms)
          throw Error(ErrorCode::SmExhaustion, op.id, "communication occupies all SMs");
        const std::int64_t cap = static_cast<std::int64_t>(gpu_.num_sms - nc) * op.blocks_per_sm;
        const std::int64_t blocks = std::min(left, cap);
        const double f = wave_time(op, blocks, ac, gpu_);
        if constexpr (Trace) tl->push_back({"compute", op.id, t, f, blocks});
        progress(t, t + f, stretch);
        t += f;
        left -= blocks;
      }
      op_done_[i] = t;
      comp_times[i] = t - begin;
    }
    const double compute_end = t;

    // Compute stream drained: the rest of the comm chain runs at full rate.
    double ft = compute_end;
    for (;;) {
      start_ready(ft);
      if (active_ < 0) break;
      CommLane& L = lanes_[active_];
      ft += L.work_left;
      L.work_left = 0.0;
      L.finished = true;
      L.end = ft;
      active_ = -1;
    }

    const std::size_t n = lanes_.size();
    comm_times.assign(n, 0.0);
    double last_end = 0.0;
    for (std::size_t j = 0; j < n; ++j) {
      comm_times[j] = lanes_[j].end - lanes_[j].start;
      if constexpr (Trace)
        tl->push_back({"comm", w_.comm_ops[j].id, lanes_[j].start, comm_times[j], 0});
      last_end = std::max(last_end, lanes_[j].end);
    }
    Y = 0.0;
    for (double y : comp_times) Y += y;
    X = 0.0;
    for (double x : comm_times) X += x;
    Z = std::max({compute_end, last_end, Y, X});
  }

 private:
  // Start every comm whose chain predecessor finished and whose gate op has
  // completed by `now`; the start instant is the event that enabled it.
  void start_ready(double now) {
    while (active_ < 0 && next_ < lanes_.size()) {
      CommLane& L = lanes_[next_];
      const double prev_end =
          next_ == 0 ? 0.0 : (lanes_[next_ - 1].finished ? lanes_[next_ - 1].end : kNever);
      const double gate_end = L.gate < 0 ? 0.0 : op_done_[static_cast<std::size_t>(L.gate)];
      const double s = std::max(prev_end, gate_end);
      if (s > now) return;
      L.start = s;
      active_ = static_cast<int>(next_++);
    }
  }

  // Integrate comm progress over [from, to] at `rate`, chaining completions.
  void progress(double from, double to, double rate) {
    double t = from;
    start_ready(t);
    while (active_ >= 0 && t < to) {
      CommLane& L = lanes_[active_];
      const double need = L.work_left / rate;
      if (t + need <= to) {
        t += need;
        L.work_left = 0.0;
        L.finished = true;
        L.end = t;
        active_ = -1;
        start_ready(t);
      } else {
        L.work_left -= (to - t) * rate;
        t = to;
      }
    }
  }

  const Workload& w_;
  const GpuSpec& gpu_;
  std::vector<CommLane> lanes_;
  std::vector<double> op_done_;
  std::size_t next_ = 0;
  int active_ = -1;
};

}  // namespace

SimResult simulate(const Workload& workload, const std::vector<CommConfig>& configs,
                   const SubspaceParams& params, const SimOptions& options) {
  OverlapRun<true> run(workload, configs, params, options);
  SimResult r;
  r.timeline.reserve(workload.comm_ops.size() + 4 * workload.compute_ops.size());
  run.run(r.comp_times, r.comm_times, r.total_compute, r.total_comm, r.makespan,
          &r.timeline);
  return r;
}

ProfileResult profile(const Workload& workload, const std::vector<CommConfig>& configs,
                      const SubspaceParams& params, const SimOptions& options) {
  OverlapRun<false> run(workload, configs, params, options);
  ProfileResult p;
  std::vector<double> comp;
  run.run(comp, p.comm_times, p.total_compute, p.total_comm, p.makespan, nullptr);
  return p;
}

}  // namespace lagom
