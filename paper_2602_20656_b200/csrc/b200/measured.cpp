// The reference's offline studies on hardware: the exhaustive joint-grid
// oracle (reference oracle.cpp:12-63) and the one-parameter sweep (reference
// sweep.cpp:11-61) with a ProfileFn — the measured replay
// (make_gpu_profiler) instead of the simulator. Same enumeration order, same
// strict-< tie rule, same row schema (sweep_csv), so `lagom sweep|compare
// --profiler gpu` emit the reference CSV with measured numbers.
#include "lagom/b200.hpp"
#include "lagom/error.hpp"
#include "lagom/sweep.hpp"

#include <limits>

namespace lagom::b200 {

OracleResult exhaustive_with(const ProfileFn& profile_fn, const Workload& workload,
                             const std::vector<std::vector<CommConfig>>& grids, std::int64_t limit) {
  const std::size_t n = grids.size();
  if (n != workload.comm_ops.size())
    throw Error(ErrorCode::InvalidWorkload, "grids", "expected one grid per comm op");
  long double points = 1;
  for (std::size_t j = 0; j < n; ++j) {
    if (grids[j].empty())
      throw Error(ErrorCode::InvalidWorkload, "grids[" + std::to_string(j) + "]", "grid must be non-empty");
    points *= static_cast<long double>(grids[j].size());
  }
  if (limit < 0 || points > static_cast<long double>(limit))
    throw Error(ErrorCode::GridTooLarge, "grid",
                "joint grid has " + std::to_string(static_cast<double>(points)) + " points, limit is " +
                    std::to_string(limit));
  OracleResult best;
  best.makespan = std::numeric_limits<double>::infinity();
  std::vector<std::size_t> digit(n, 0);
  std::vector<CommConfig> point(n);
  for (;;) {
    for (std::size_t j = 0; j < n; ++j) point[j] = grids[j][digit[j]];
    const double z = profile_fn(point).makespan;
    ++best.evaluations;
    if (z < best.makespan) {  // strict: the earliest optimum wins
      best.makespan = z;
      best.configs = point;
    }
    std::size_t pos = n;  // odometer, last comm fastest
    bool wrapped = true;
    while (pos-- > 0) {
      if (++digit[pos] < grids[pos].size()) {
        wrapped = false;
        break;
      }
      digit[pos] = 0;
    }
    if (wrapped) break;
  }
  return best;
}

std::vector<SweepRow> sweep_with(const ProfileFn& profile_fn, const Workload& workload,
                                 const std::vector<CommConfig>& base, const std::string& comm_id, SweepParam param,
                                 const std::vector<std::int64_t>& values) {
  std::size_t target = workload.comm_ops.size();
  for (std::size_t j = 0; j < workload.comm_ops.size(); ++j)
    if (workload.comm_ops[j].id == comm_id) target = j;
  if (target == workload.comm_ops.size())
    throw Error(ErrorCode::InvalidWorkload, "comm", "no comm op with id '" + comm_id + "'");
  std::vector<SweepRow> rows;
  std::vector<CommConfig> cfg = base;
  for (const std::int64_t v : values) {
    CommConfig& c = cfg[target];
    c = base[target];
    if (param == SweepParam::NumChannels) c.num_channels = static_cast<int>(v);
    else if (param == SweepParam::ChunkSize) c.chunk_size = v;
    else c.num_threads = static_cast<int>(v);
    const ProfileResult r = profile_fn(cfg);
    rows.push_back({v, r.comm_times.at(target), r.total_compute, r.makespan});
  }
  return rows;
}

}  // namespace lagom::b200
