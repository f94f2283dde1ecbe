// Python bindings (pybind11) of the C++ API — used by tests/ and bench.py.
// JSON in, JSON out, in the reference's own file formats (reference
// docs/formats.md: workload / configs / params documents, tune-log records),
// so everything Python sees is exactly what the reference CLI would emit.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <execinfo.h>
#include <unistd.h>

#include <chrono>
#include <csignal>
#include <cstdlib>
#include <memory>

#include "lagom/b200.hpp"
#include "lagom/error.hpp"
#include "lagom/json_io.hpp"
#include "lagom/oracle.hpp"
#include "lagom/simulator.hpp"
#include "lagom/sweep.hpp"
#include "lagom/tuner.hpp"
#include "lagom/version.hpp"
#include "lagom/workloads.hpp"

namespace py = pybind11;
using namespace lagom;
using lagom::b200::ReplayDag;

namespace {

Json parse(const std::string& s) { return parse_json(s, "<python>"); }

SubspaceParams params_or_default(const std::string& p) {
  return p.empty() ? SubspaceParams::defaults() : params_from_json(parse(p));
}

Json profile_json(const ProfileResult& p) {
  return Json{{"x", p.comm_times}, {"X", p.total_comm}, {"Y", p.total_compute}, {"Z", p.makespan}};
}

// Reference CLI seeds (lagom_main.cpp:181-198): min or nccl-default.
std::vector<CommConfig> seed_configs(const Workload& w, const SubspaceParams& params,
                                     const std::string& start) {
  // min / nccl-default: the reference CLI's starts (lagom_main.cpp --start).
  // coresident (B200 addition): many light channels that ride along the
  // GEMMs (NC 64, NT 128 — the co-resident kernel regime of the NVLS, one-hop
  // and single-rank kernels, lagom_coll.h), a region neither reference start
  // reaches, since Alg. 2 only grows resources (tuner.cpp:47-76).
  if (start != "min" && start != "nccl-default" && start != "coresident")
    throw Error(ErrorCode::InvalidInput, "start", "expected min|nccl-default|coresident");
  std::vector<CommConfig> out;
  for (const CommOp& op : w.comm_ops) {
    const StepBounds b = bounds_for(op, w.gpu);
    CommConfig c = minimum_config(select_subspace(op, w.gpu, params), b);
    if (start == "nccl-default") {
      c.num_channels = std::min(8, b.nc_max);
      c.num_threads = 512;
      c.chunk_size = std::clamp<std::int64_t>(2048 * kKiB, b.c_min, b.c_max);
    } else if (start == "coresident") {
      c.num_channels = std::min(64, b.nc_max);
      c.num_threads = 128;
      c.chunk_size = std::clamp<std::int64_t>(2048 * kKiB, b.c_min, b.c_max);
    }
    out.push_back(c);
  }
  return out;
}

// Tune log records in the reference CLI schema (lagom_main.cpp:204-236).
Json tune_json(const Workload& w, const TuneResult& r, double wall_us) {
  Json log = Json::array();
  for (const TuneRecord& rec : r.log) {
    Json j;
    j["iter"] = rec.iteration;
    j["comm_id"] = rec.comm_index ? Json(w.comm_ops[*rec.comm_index].id) : Json(nullptr);
    j["config"] = rec.comm_index ? config_to_json(rec.config) : Json(nullptr);
    j["x"] = rec.comm_index ? Json(rec.comm_time) : Json(nullptr);
    j["X"] = rec.total_comm;
    j["Y"] = rec.total_compute;
    j["Z"] = rec.makespan;
    Json h, done = Json::array();
    for (std::size_t k = 0; k < rec.priorities.size(); ++k) {
      h[w.comm_ops[k].id] = rec.priorities[k];
      if (rec.done[k]) done.push_back(w.comm_ops[k].id);
    }
    j["H_table"] = h;
    j["done"] = done;
    if (rec.priority_after) j["H_after"] = *rec.priority_after;
    else if (rec.comm_index) j["H_after"] = nullptr;
    j["already_optimal"] = rec.already_optimal;
    log.push_back(j);
  }
  Json states = Json::array();
  for (const CommTuneState& s : r.states)
    states.push_back({{"config", config_to_json(s.current)}, {"reason", to_string(s.reason)},
                      {"done", s.done}, {"grown", s.grown}, {"priority", s.priority}});
  return Json{{"configs", configs_to_json(r.configs)["configs"]},
              {"final", profile_json(r.final_profile)},
              {"initial_Z", r.initial_makespan},
              {"profile_calls", r.profile_calls},
              {"budget_exhausted", r.budget_exhausted},
              {"boundary_condition", r.boundary_condition},
              {"wall_us", wall_us},
              {"log", log},
              {"states", states}};
}

GpuSpec gpu_from_json(const std::string& s) {
  GpuSpec g;
  if (s.empty()) return g;
  const Json j = parse(s);
  g.num_sms = j.value("num_sms", g.num_sms);
  g.peak_mem_bw = j.value("peak_mem_bw", g.peak_mem_bw);
  g.link_bw = j.value("link_bw", g.link_bw);
  g.comm_bw_cap_fraction = j.value("comm_bw_cap_fraction", g.comm_bw_cap_fraction);
  g.compute_on_comm_slowdown = j.value("compute_on_comm_slowdown", g.compute_on_comm_slowdown);
  return g;
}

Json pm_json(const b200::ReplayMeasurement& m) {
  if (m.pm_metrics.empty()) return nullptr;
  Json rows = Json::array();
  for (const b200::PmSample& s : m.pm_samples) {
    Json row = Json::array({s.start_ns, s.end_ns});
    for (double v : s.values) row.push_back(v);
    rows.push_back(row);
  }
  return Json{{"metrics", m.pm_metrics}, {"t0_ns", m.pm_t0_ns}, {"samples", rows}};
}

Json measurement_json(const b200::ReplayMeasurement& m) {
  SimResult tl;
  tl.timeline = m.timeline;
  return Json{{"x", m.profile.comm_times}, {"x_ev", m.comm_event_times}, {"y", m.comp_times}, {"X", m.profile.total_comm},
              {"Y", m.profile.total_compute}, {"Z", m.profile.makespan}, {"wall_us", m.wall_us},
              {"trace", trace_to_json(tl)}, {"pm", pm_json(m)}};
}

std::vector<CommConfig> configs_arg(const std::string& s) { return configs_from_json(parse(s)); }

class PyEngine {
 public:
  PyEngine(const std::string& dag_json, const std::string& coord_name, int rank, int size, int device,
           int repeats, int warmup, bool nccl, std::int64_t max_chunk, int max_channels,
           std::int64_t e2e_in, std::int64_t e2e_out, int sm_partition, bool nvls, bool coresident, int one_hop,
           bool a2a_tma, std::uint64_t pm_interval_ns)
      : dag_(b200::replay_dag_from_json(dag_json)) {
    coord_ = b200::make_shm_coordinator(coord_name, rank, size);
    b200::ReplayOptions o;
    o.device = device;
    o.repeats = repeats;
    o.warmup = warmup;
    o.enable_nccl = nccl;
    o.max_chunk_bytes = max_chunk;
    o.max_channels = max_channels;
    o.e2e_in_bytes = e2e_in;
    o.e2e_out_bytes = e2e_out;
    o.sm_partition = sm_partition;
    o.nvls = nvls;
    o.coresident = coresident;
    o.one_hop = one_hop;
    o.a2a_tma = a2a_tma;
    o.pm_interval_ns = pm_interval_ns;
    engine_ = std::make_unique<b200::ReplayEngine>(dag_, *coord_, o);
  }
  std::string workload(const std::string& gpu_json) const {
    return workload_to_json(b200::to_workload(dag_, gpu_from_json(gpu_json), coord_->size())).dump();
  }
  std::string run(const std::string& cfgs) {
    alive();
    py::gil_scoped_release nogil;
    return measurement_json(engine_->remote_run(configs_arg(cfgs))).dump();
  }
  std::string run_e2e(const std::string& cfgs) {
    py::gil_scoped_release nogil;
    return measurement_json(engine_->remote_run_e2e(configs_arg(cfgs))).dump();
  }
  std::string run_nccl() {
    py::gil_scoped_release nogil;
    return measurement_json(engine_->remote_run_nccl()).dump();
  }
  std::string run_compute_only() {
    py::gil_scoped_release nogil;
    return measurement_json(engine_->remote_run_compute_only()).dump();
  }
  std::string run_comm_only(const std::string& cfgs) {
    py::gil_scoped_release nogil;
    return measurement_json(engine_->remote_run_comm_only(configs_arg(cfgs))).dump();
  }
  // Lagom search with the measured profiler (rank 0). Also returns the
  // recorded profile table for bit-identical offline replays.
  std::string tune(const std::string& gpu_json, const std::string& start, int budget,
                   const std::string& params_json, const std::vector<int>& groups) {
    py::gil_scoped_release nogil;
    const GpuSpec gpu = gpu_from_json(gpu_json);
    const bool grouped = !groups.empty();
    const Workload w = grouped ? b200::grouped_workload(dag_, groups, gpu, coord_->size())
                               : b200::to_workload(dag_, gpu, coord_->size());
    const SubspaceParams params = params_or_default(params_json);
    const std::vector<CommConfig> init = seed_configs(w, params, start);
    std::vector<std::pair<std::vector<CommConfig>, ProfileResult>> table;
    const ProfileFn f = grouped ? b200::make_grouped_gpu_profiler(*engine_, groups, &table)
                                : b200::make_gpu_profiler(*engine_, &table);
    const auto t0 = std::chrono::steady_clock::now();
    const TuneResult r = tune_impl(w, init, f, budget);
    const double wall = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    Json out = tune_json(w, r, wall);
    out["initial"] = configs_to_json(init)["configs"];
    Json tab = Json::array();
    for (const auto& [cfg, res] : table)
      tab.push_back({{"configs", configs_to_json(cfg)["configs"]}, {"result", profile_json(res)}});
    out["profile_table"] = tab;
    out["workload"] = workload_to_json(w);
    return out.dump();
  }
  void serve() {
    py::gil_scoped_release nogil;
    engine_->serve();
  }
  void stop() { engine_->stop(); }
  // Collective: every rank must call it (NCCL communicator teardown).
  void close() {
    py::gil_scoped_release nogil;
    engine_.reset();
  }
  void set_measurement(int repeats, int warmup) { engine_->set_measurement(repeats, warmup); }
  void set_partition(int sm_partition, int nccl_reserve) { engine_->set_partition(sm_partition, nccl_reserve); }
  bool nvls_active() const { return engine_->nvls_active(); }
  void set_pm_sampling(bool on) { engine_->set_pm_sampling(on); }
  bool nvls_peers_active() const { return engine_->nvls_peers_active(); }
  int rank() const { return engine_->rank(); }
  int nranks() const { return engine_->nranks(); }
  void barrier() {
    py::gil_scoped_release nogil;
    coord_->barrier();
  }

 private:
  void alive() const {
    if (!engine_) throw Error(ErrorCode::InvalidInput, "engine", "engine is closed");
  }
  static TuneResult tune_impl(const Workload& w, const std::vector<CommConfig>& init, const ProfileFn& f,
                              int budget) {
    return lagom::tune(w, init, f, budget);
  }
  ReplayDag dag_;
  std::unique_ptr<b200::Coordinator> coord_;
  std::unique_ptr<b200::ReplayEngine> engine_;
};

}  // namespace

namespace {
// LAGOM_BACKTRACE=1: native backtrace on SIGABRT / SIGSEGV (debugging aid;
// the boxes have no debugger).
void backtrace_handler(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  const char msg[] = "[lagom] native backtrace:\n";
  (void)!write(2, msg, sizeof msg - 1);
  backtrace_symbols_fd(frames, n, 2);
  std::signal(sig, SIG_DFL);
  std::raise(sig);
}
}  // namespace

PYBIND11_MODULE(_lagom_py, m) {
  if (const char* e = std::getenv("LAGOM_BACKTRACE"); e && *e == '1') {
    std::signal(SIGABRT, backtrace_handler);
    std::signal(SIGSEGV, backtrace_handler);
  }
  m.doc() = "lagom-b200 C++ API (JSON in/out in the reference formats)";
  m.attr("version") = kVersion;
  py::register_exception<Error>(m, "LagomError");

  m.def("default_params", [] { return params_to_json(SubspaceParams::defaults()).dump(); });
  m.def("gen", [](const std::string& pattern, int layers, std::uint64_t seed, int mcount, int ncount) {
    Workload w;
    if (pattern == "fsdp") w = gen_fsdp(layers, seed);
    else if (pattern == "tp") w = gen_tp_domino(layers, seed);
    else if (pattern == "ep") w = gen_ep_dualbatch(layers, seed);
    else if (pattern == "allreduce-pair") w = gen_allreduce_pair();
    else if (pattern == "random") w = gen_random(mcount, ncount, seed);
    else throw Error(ErrorCode::InvalidInput, "pattern", "unknown pattern '" + pattern + "'");
    return workload_to_json(w).dump();
  }, py::arg("pattern"), py::arg("layers") = 4, py::arg("seed") = 1, py::arg("m") = 4, py::arg("n") = 2);
  m.def("seed_configs", [](const std::string& w, const std::string& start, const std::string& p) {
    return configs_to_json(seed_configs(workload_from_json(parse(w)), params_or_default(p), start)).dump();
  }, py::arg("workload"), py::arg("start") = "min", py::arg("params") = "");
  m.def("simulate", [](const std::string& w, const std::string& c, const std::string& p, bool sm_occupancy) {
    SimOptions opt;
    opt.sm_occupancy = sm_occupancy;  // false: running comms hold no SMs (co-resident kernels)
    const SimResult r = simulate(workload_from_json(parse(w)), configs_arg(c), params_or_default(p), opt);
    return Json{{"x", r.comm_times}, {"y", r.comp_times}, {"X", r.total_comm}, {"Y", r.total_compute},
                {"Z", r.makespan}, {"trace", trace_to_json(r)}}.dump();
  }, py::arg("workload"), py::arg("configs"), py::arg("params") = "", py::arg("sm_occupancy") = true);
  m.def("tune_sim", [](const std::string& w, const std::string& start, int budget, const std::string& p) {
    const Workload wl = workload_from_json(parse(w));
    const SubspaceParams params = params_or_default(p);
    const auto init = seed_configs(wl, params, start);
    const auto t0 = std::chrono::steady_clock::now();
    const TuneResult r = tune(wl, init, make_sim_profiler(wl, params), budget);
    const double wall = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    Json out = tune_json(wl, r, wall);
    out["initial"] = configs_to_json(init)["configs"];
    return out.dump();
  }, py::arg("workload"), py::arg("start") = "min", py::arg("budget") = 500, py::arg("params") = "");
  m.def("tune_table", [](const std::string& w, const std::string& init, const std::string& table, int budget) {
    const Workload wl = workload_from_json(parse(w));
    std::vector<std::pair<std::vector<CommConfig>, ProfileResult>> t;
    for (const Json& e : parse(table)) {
      ProfileResult r;
      r.comm_times = e["result"]["x"].get<std::vector<double>>();
      r.total_comm = e["result"]["X"].get<double>();
      r.total_compute = e["result"]["Y"].get<double>();
      r.makespan = e["result"]["Z"].get<double>();
      t.emplace_back(configs_from_json(e["configs"]), r);
    }
    const TuneResult r = tune(wl, configs_arg(init), b200::make_table_profiler(std::move(t)), budget);
    return tune_json(wl, r, 0.0).dump();
  }, py::arg("workload"), py::arg("initial"), py::arg("table"), py::arg("budget") = 500);
  m.def("oracle_gpu", [](const std::string& w, const std::string& p, std::int64_t limit, int device) {
    const Workload wl = workload_from_json(parse(w));
    const SubspaceParams params = params_or_default(p);
    py::gil_scoped_release nogil;
    const OracleResult o = b200::exhaustive_gpu(wl, default_grids(wl, params), params, limit, device);
    return Json{{"Z", o.makespan}, {"evaluations", o.evaluations},
                {"configs", configs_to_json(o.configs)["configs"]}}.dump();
  }, py::arg("workload"), py::arg("params") = "", py::arg("limit") = 1000000, py::arg("device") = 0);
  m.def("oracle", [](const std::string& w, const std::string& p, std::int64_t limit) {
    const Workload wl = workload_from_json(parse(w));
    const SubspaceParams params = params_or_default(p);
    const OracleResult o = exhaustive(wl, default_grids(wl, params), params, limit);
    return Json{{"Z", o.makespan}, {"evaluations", o.evaluations},
                {"configs", configs_to_json(o.configs)["configs"]}}.dump();
  }, py::arg("workload"), py::arg("params") = "", py::arg("limit") = 1000000);

  // Exercises the native shm coordinator (CPU only): barrier, broadcast from
  // rank 0, all-gather of rank ids, max-reduction. Used by the world_size-2
  // CPU tests of the multi-rank host path.
  m.def("coord_selftest", [](const std::string& name, int rank, int size, int rounds) {
    py::gil_scoped_release nogil;
    auto c = b200::make_shm_coordinator(name, rank, size, 60.0);
    Json out = Json::array();
    for (int k = 0; k < rounds; ++k) {
      c->barrier();
      char msg[32] = {0};
      if (rank == 0) std::snprintf(msg, sizeof msg, "round-%d-of-%d", k, size);
      c->broadcast(msg, sizeof msg, 0);
      std::int64_t mine = 100 * rank + k, all[8] = {0};
      c->allgather(&mine, sizeof mine, all);
      double v[3] = {static_cast<double>(rank), -static_cast<double>(rank), 1.5 * rank + k};
      c->allreduce_max(v, 3);
      out.push_back({{"msg", std::string(msg)}, {"gathered", std::vector<std::int64_t>(all, all + size)},
                     {"max", std::vector<double>(v, v + 3)}});
    }
    return out.dump();
  }, py::arg("name"), py::arg("rank"), py::arg("size"), py::arg("rounds") = 3);

  py::class_<PyEngine>(m, "ReplayEngine")
      .def(py::init<const std::string&, const std::string&, int, int, int, int, int, bool, std::int64_t, int,
                    std::int64_t, std::int64_t, int, bool, bool, int, bool, std::uint64_t>(),
           py::arg("dag"), py::arg("coord_name"), py::arg("rank"), py::arg("size"), py::arg("device"),
           py::arg("repeats") = 3, py::arg("warmup") = 1, py::arg("nccl") = true,
           py::arg("max_chunk_bytes") = 4 << 20, py::arg("max_channels") = 32, py::arg("e2e_in_bytes") = 0,
           py::arg("e2e_out_bytes") = 0, py::arg("sm_partition") = 1, py::arg("nvls") = false,
           py::arg("coresident") = true, py::arg("one_hop") = 2, py::arg("a2a_tma") = true,
           py::arg("pm_interval_ns") = 20000)
      .def("workload", &PyEngine::workload, py::arg("gpu") = "")
      .def("run", &PyEngine::run)
      .def("run_e2e", &PyEngine::run_e2e)
      .def("run_nccl", &PyEngine::run_nccl)
      .def("run_compute_only", &PyEngine::run_compute_only)
      .def("run_comm_only", &PyEngine::run_comm_only)
      .def("tune", &PyEngine::tune, py::arg("gpu") = "", py::arg("start") = "min", py::arg("budget") = 200,
           py::arg("params") = "", py::arg("groups") = std::vector<int>{})
      .def("serve", &PyEngine::serve)
      .def("stop", &PyEngine::stop)
      .def("close", &PyEngine::close)
      .def("set_measurement", &PyEngine::set_measurement, py::arg("repeats"), py::arg("warmup") = 0)
      .def("barrier", &PyEngine::barrier)
      .def("set_partition", &PyEngine::set_partition, py::arg("sm_partition"), py::arg("nccl_reserve_sms") = 0)
      .def_property_readonly("nvls_active", &PyEngine::nvls_active)
      .def("set_pm_sampling", &PyEngine::set_pm_sampling, py::arg("on"))
      .def_property_readonly("nvls_peers_active", &PyEngine::nvls_peers_active)
      .def_property_readonly("rank", &PyEngine::rank)
      .def_property_readonly("nranks", &PyEngine::nranks);
}
