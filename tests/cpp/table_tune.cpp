// Table-tune driver — TEST INFRASTRUCTURE.
//
// Reads a recorded GPU profile table (configs -> ProfileResult, as bench.py
// stores it from make_grouped_gpu_profiler) and runs tune() against it
// through a table-backed ProfileFn. Compiled twice — against the reference
// build (oracle/_ref/table_tune_ref, namespace lagom_ref) and against the
// product (build/table_tune) — so a test can show that, given the same
// measured profile table, both tuners make bit-identical picks.
//
// usage: table_tune <doc.json>   doc = {"workload": {...}, "initial": [...],
//                                       "table": [{"configs": [...], "result": {x, X, Y, Z}}], "budget": N}
#include <cstdio>
#include <iostream>

#include "lagom/json_io.hpp"
#include "lagom/tuner.hpp"

using namespace lagom;

int main(int argc, char** argv) {
  if (argc != 2) {
    std::cerr << "usage: table_tune doc.json\n";
    return 2;
  }
  const Json doc = parse_json(read_file(argv[1]), argv[1]);
  const Workload w = workload_from_json(doc.at("workload"));
  const std::vector<CommConfig> init = configs_from_json(doc.at("initial"));
  std::vector<std::pair<std::vector<CommConfig>, ProfileResult>> table;
  for (const Json& e : doc.at("table")) {
    ProfileResult r;
    r.comm_times = e.at("result").at("x").get<std::vector<double>>();
    r.total_comm = e.at("result").at("X").get<double>();
    r.total_compute = e.at("result").at("Y").get<double>();
    r.makespan = e.at("result").at("Z").get<double>();
    table.emplace_back(configs_from_json(e.at("configs")), r);
  }
  int misses = 0;
  const ProfileFn f = [&](const std::vector<CommConfig>& c) {
    for (const auto& [k, v] : table)
      if (k == c) return v;
    ++misses;
    return ProfileResult{std::vector<double>(c.size(), 1e300), 1e300, 0.0, 1e300};
  };
  const TuneResult r = tune(w, init, f, doc.at("budget").get<int>());
  Json out;
  out["configs"] = configs_to_json(r.configs)["configs"];
  out["profile_calls"] = r.profile_calls;
  out["boundary_condition"] = r.boundary_condition;
  out["budget_exhausted"] = r.budget_exhausted;
  out["table_misses"] = misses;
  char buf[64];
  Json log = Json::array();
  for (const TuneRecord& rec : r.log) {
    std::snprintf(buf, sizeof buf, "%a", rec.makespan);
    Json j = {{"iter", rec.iteration}, {"comm", rec.comm_index ? *rec.comm_index : -1}, {"Z", buf}};
    if (rec.comm_index) j["config"] = config_to_json(rec.config);
    if (rec.priority_after) {
      std::snprintf(buf, sizeof buf, "%a", *rec.priority_after);
      j["H_after"] = buf;
    }
    log.push_back(j);
  }
  out["log"] = log;
  Json states = Json::array();
  for (const CommTuneState& s : r.states) states.push_back(to_string(s.reason));
  out["reasons"] = states;
  std::cout << out.dump() << "\n";
  return 0;
}
