// Lagom search: H priority (Eq. 7), resource stepping (Alg. 2), the co-tuning
// loop (Alg. 1) and the terminal-state audit. Reference: tuner.cpp:12-353.
//
// This is the caller of the ProfileFn seam and must make the reference's picks
// bit for bit given the same profile results. The behaviours that matter
// are each marked "parity:" below.
#include <algorithm>
#include <cmath>
#include <limits>

#include "lagom/error.hpp"
#include "lagom/tuner.hpp"

namespace lagom {

ProfileFn make_sim_profiler(const Workload& workload, const SubspaceParams& params) {
  // Own copies: the returned callable may outlive the caller's objects.
  return [w = workload, p = params](const std::vector<CommConfig>& cfgs) {
    return profile(w, cfgs, p);
  };
}

std::optional<double> compute_h(double y_before, double y_after, double x_old,
                                double x_new) {
  if (x_old <= x_new) return std::nullopt;  // already at its optimum
  return (y_after - y_before) / (x_old - x_new);
}

StepBounds bounds_for(const CommOp& op, const GpuSpec& gpu) {
  StepBounds b;
  b.nc_min = 1;
  b.nc_max = max_channels(op, gpu);
  b.nt_min = kThreadLadder[0];
  b.c_min = op.bounds.c_min;
  b.c_max = op.bounds.c_max;
  return b;
}

CommConfig minimum_config(const SubspaceKey& key, const StepBounds& b) {
  CommConfig c;
  c.algorithm = key.algorithm;
  c.protocol = key.protocol;
  c.transport = key.transport;
  c.num_channels = b.nc_min;
  c.num_threads = b.nt_min;
  c.chunk_size = b.c_min;
  return c;
}

CommConfig grow_config(const CommConfig& cur, double lr, const StepBounds& b) {
  const double k = 1.0 + lr;
  CommConfig nxt = cur;

  // parity: std::llround = round half away from zero.
  const std::int64_t nc_target = std::llround(static_cast<double>(cur.num_channels) * k);
  const std::int64_t nc_floor = static_cast<std::int64_t>(cur.num_channels) + 1;
  nxt.num_channels =
      static_cast<int>(std::min<std::int64_t>(b.nc_max, std::max(nc_floor, nc_target)));

  // First ladder rung at or above NT*(1+lr); the top rung when none is.
  const double nt_target = static_cast<double>(cur.num_threads) * k;
  const auto rung = std::find_if(kThreadLadder.begin(), kThreadLadder.end(),
                                 [&](int v) { return static_cast<double>(v) >= nt_target; });
  nxt.num_threads = rung == kThreadLadder.end() ? kThreadLadder.back() : *rung;

  const std::int64_t c_target =
      std::llround(static_cast<double>(cur.chunk_size) * k / 1024.0) * kKiB;
  nxt.chunk_size = std::min<std::int64_t>(b.c_max, std::max(cur.chunk_size + kKiB, c_target));
  return nxt;
}

StepResult step_resource(const CommConfig& cur, double x_prev, double x_new,
                         double X_after, double Y_after, const StepBounds& b) {
  // parity: guard order is regression, crossing, growth, no-move.
  if (x_new - x_prev > 0) return {StepOutcome::DoneRegression, cur};
  if (X_after < Y_after) return {StepOutcome::DoneCrossing, cur};
  const double lr = x_new > 0 ? (x_prev - x_new) / x_new : 0.0;
  const CommConfig nxt = grow_config(cur, lr, b);
  if (nxt == cur) return {StepOutcome::DoneNoMove, cur};
  return {StepOutcome::Grow, nxt};
}

const char* to_string(DoneReason reason) {
  switch (reason) {
    case DoneReason::NotDone: return "not_done";
    case DoneReason::Regression: return "regression";
    case DoneReason::Crossing: return "crossing";
    case DoneReason::NoMove: return "no_move";
    case DoneReason::AlreadyOptimal: return "already_optimal";
  }
  return "?";
}

SubspaceKey select_subspace(const CommOp& op, const GpuSpec& gpu,
                            const SubspaceParams& params) {
  if (params.empty())
    throw Error(ErrorCode::UnknownSubspace, "params", "no subspaces defined");
  const StepBounds b = bounds_for(op, gpu);
  const std::vector<SubspaceKey> keys = params.keys();
  // parity: strict <, so ties keep the first key in map order.
  SubspaceKey pick = keys.front();
  double pick_time = comm_time(op, minimum_config(pick, b), gpu, params);
  for (std::size_t i = 1; i < keys.size(); ++i) {
    const double t = comm_time(op, minimum_config(keys[i], b), gpu, params);
    if (t < pick_time) {
      pick = keys[i];
      pick_time = t;
    }
  }
  return pick;
}

int check_boundary(const std::vector<CommConfig>& initial, const TuneResult& res) {
  const double X = res.final_profile.total_comm;
  const double Y = res.final_profile.total_compute;
  const double tol = 1e-9 * (X + Y + 1.0);
  const std::size_t n = res.configs.size();

  // 1: nothing grew and the comm stream is not the bottleneck.
  bool untouched = true;
  for (std::size_t j = 0; j < n; ++j) untouched = untouched && res.configs[j] == initial[j];
  if (untouched && X <= Y + tol) return 1;

  // 2: comm-bound, everything done, every grown comm at its standalone optimum.
  bool grown_at_optimum = true;
  for (std::size_t j = 0; j < n; ++j) {
    if (res.configs[j] == initial[j]) continue;
    const DoneReason r = res.states[j].reason;
    grown_at_optimum = grown_at_optimum &&
                       (r == DoneReason::Regression || r == DoneReason::NoMove ||
                        r == DoneReason::AlreadyOptimal);
  }
  if (X > Y && grown_at_optimum && !res.states.empty() &&
      std::all_of(res.states.begin(), res.states.end(),
                  [](const CommTuneState& s) { return s.done; }))
    return 2;

  // 3: |X - Y| within the largest observed single-step move of (X, Y),
  // including the jump from the last logged call to the final assignment.
  double largest = 0.0;
  for (std::size_t k = 1; k < res.log.size(); ++k) {
    const double dx = std::abs(res.log[k].total_comm - res.log[k - 1].total_comm);
    const double dy = std::abs(res.log[k].total_compute - res.log[k - 1].total_compute);
    largest = std::max(largest, dx + dy);
  }
  if (!res.log.empty()) {
    const TuneRecord& tail = res.log.back();
    largest = std::max(largest, std::abs(X - tail.total_comm) + std::abs(Y - tail.total_compute));
  }
  return std::abs(X - Y) <= largest + tol ? 3 : 0;
}

namespace {

// Not-done comm with the least H; ties go to the lowest index.
int pick_next(const std::vector<CommTuneState>& st) {
  int best = -1;
  for (int j = 0; j < static_cast<int>(st.size()); ++j) {
    if (st[j].done) continue;
    if (best < 0 || st[j].priority < st[best].priority) best = j;
  }
  return best;
}

DoneReason freeze_reason(StepOutcome o) {
  switch (o) {
    case StepOutcome::DoneRegression: return DoneReason::Regression;
    case StepOutcome::DoneCrossing: return DoneReason::Crossing;
    case StepOutcome::DoneNoMove: return DoneReason::NoMove;
    default: return DoneReason::NotDone;
  }
}

class CoTuner {
 public:
  CoTuner(const Workload& w, const std::vector<CommConfig>& init, const ProfileFn& f,
          int budget)
      : w_(w), n_(w.comm_ops.size()), profiler_(f), budget_(budget), cur_(init) {}

  TuneResult run(const std::vector<CommConfig>& init) {
    for (const CommOp& op : w_.comm_ops) bounds_.push_back(bounds_for(op, w_.gpu));
    st_.resize(n_);
    for (std::size_t j = 0; j < n_; ++j) st_[j].current = st_[j].best_config = init[j];

    const ProfileResult probe = measure(std::nullopt);
    out_.initial_makespan = probe.makespan;
    for (std::size_t j = 0; j < n_; ++j) {
      CommTuneState& s = st_[j];
      s.x_previous = s.x_current = probe.comm_times[j];
      s.last_total_comm = probe.total_comm;
      s.last_total_compute = probe.total_compute;
      s.best_makespan = probe.makespan;
      s.history.push_back(
          {s.current, probe.comm_times[j], probe.total_comm, probe.total_compute, probe.makespan});
    }
    best_vec_ = cur_;
    best_ = probe;
    last_ = probe;

    for (int picked; (picked = pick_next(st_)) >= 0;) {
      const auto j = static_cast<std::size_t>(picked);
      CommTuneState& s = st_[j];
      // parity: the crossing guard reads this comm's own (possibly stale)
      // last X'/Y', not the global last profile.
      const StepResult step = step_resource(s.current, s.x_previous, s.x_current,
                                            s.last_total_comm, s.last_total_compute,
                                            bounds_[j]);
      if (step.outcome != StepOutcome::Grow) {
        s.done = true;
        s.reason = freeze_reason(step.outcome);
        // parity: a regression found lazily reverts without a profile call.
        if (step.outcome == StepOutcome::DoneRegression) cur_[j] = s.current = s.best_config;
        continue;
      }
      // parity: the budget is checked only once a growth step exists.
      if (calls_ >= budget_) {
        out_.budget_exhausted = true;
        break;
      }
      s.x_previous = s.x_current;
      s.current = step.next;
      s.grown = true;
      cur_[j] = step.next;

      const ProfileResult r = measure(picked);
      s.x_current = r.comm_times[j];
      s.last_total_comm = r.total_comm;
      s.last_total_compute = r.total_compute;
      s.history.push_back({step.next, r.comm_times[j], r.total_comm, r.total_compute, r.makespan});
      if (r.makespan < s.best_makespan) {
        s.best_makespan = r.makespan;
        s.best_config = step.next;
      }
      if (r.makespan < best_.makespan) {
        best_vec_ = cur_;
        best_ = r;
      }
      // parity: H uses the *global* previous profile's Y.
      const std::optional<double> h =
          compute_h(last_.total_compute, r.total_compute, s.x_previous, s.x_current);
      TuneRecord& rec = out_.log.back();
      rec.priority_after = h;
      if (h) {
        s.priority = *h;
      } else {
        rec.already_optimal = true;
        // parity: only an exact stall freezes here; a strict regression is
        // left to step_resource at the comm's next selection.
        if (s.x_current == s.x_previous) {
          s.done = true;
          s.reason = DoneReason::AlreadyOptimal;
          cur_[j] = s.current = s.best_config;
        }
      }
      last_ = r;
    }

    // Final verification with the never-worse fallback.
    if (out_.budget_exhausted) {
      cur_ = best_vec_;
      out_.final_profile = best_;
    } else {
      ProfileResult fin;
      if (cur_ == last_profiled_) {
        fin = last_;
      } else if (calls_ < budget_) {
        fin = measure(std::nullopt);
      } else {
        cur_ = best_vec_;
        fin = best_;
      }
      if (fin.makespan > best_.makespan) {
        cur_ = best_vec_;
        fin = best_;
      }
      out_.final_profile = std::move(fin);
    }
    out_.configs = cur_;
    out_.profile_calls = calls_;
    out_.states = std::move(st_);
    out_.boundary_condition = check_boundary(init, out_);
    return std::move(out_);
  }

 private:
  ProfileResult measure(std::optional<int> comm) {
    ProfileResult r = profiler_(cur_);
    ++calls_;
    TuneRecord rec;
    rec.iteration = calls_;
    rec.comm_index = comm;
    if (comm) {
      rec.config = cur_[static_cast<std::size_t>(*comm)];
      rec.comm_time = r.comm_times[static_cast<std::size_t>(*comm)];
    }
    rec.total_comm = r.total_comm;
    rec.total_compute = r.total_compute;
    rec.makespan = r.makespan;
    rec.priorities.resize(n_);
    rec.done.resize(n_);
    for (std::size_t k = 0; k < n_; ++k) {
      rec.priorities[k] = st_[k].priority;
      rec.done[k] = st_[k].done;
    }
    out_.log.push_back(std::move(rec));
    last_profiled_ = cur_;
    return r;
  }

  const Workload& w_;
  std::size_t n_;
  const ProfileFn& profiler_;
  int budget_;
  std::vector<CommConfig> cur_;
  std::vector<CommConfig> last_profiled_;
  std::vector<CommConfig> best_vec_;
  std::vector<StepBounds> bounds_;
  std::vector<CommTuneState> st_;
  ProfileResult best_, last_;
  int calls_ = 0;
  TuneResult out_;
};

}  // namespace

TuneResult tune(const Workload& workload, const std::vector<CommConfig>& initial,
                const ProfileFn& profiler, int budget) {
  const std::size_t n = workload.comm_ops.size();
  if (initial.size() != n) {
    throw Error(ErrorCode::InvalidWorkload, "configs",
                "expected " + std::to_string(n) + " initial configs, got " +
                    std::to_string(initial.size()));
  }
  if (n == 0) {
    TuneResult r;
    r.configs = initial;
    r.boundary_condition = 1;
    return r;
  }
  if (budget < 1) {
    TuneResult r;
    r.configs = initial;
    r.budget_exhausted = true;
    return r;
  }
  return CoTuner(workload, initial, profiler, budget).run(initial);
}

}  // namespace lagom
