// `lagom` command-line front end — the reference CLI's surface
// (reference proj/tools/lagom_main.cpp:421-504, docs/formats.md "Reports" and
// "Exit codes"): simulate | tune | oracle | compare | sweep | gen, the same
// flags, report schemas, tune-log records, parameter resolution
// (--params > $LAGOM_PARAMS > defaults) and exit codes (0 ok, 2 validation,
// 3 I/O, 4 budget exhausted, 5 grid too large).
//
// B200 addition: `tune | sweep | compare --profiler gpu --dag DAG.json`
// replace the simulator with the iteration-replay engine (lagom/b200.hpp):
// every profile call, sweep value and grid point is a measured replay, and
// the reports / CSV keep the reference schemas. One process per GPU:
// RANK / WORLD_SIZE / LOCAL_RANK come from the environment (torchrun), the
// ranks meet in a shared-memory coordinator named by $LAGOM_JOB (or
// $MASTER_PORT); rank 0 runs the search and writes the report, the other
// ranks serve replays.
#include <chrono>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <string>
#include <vector>

#include "lagom/b200.hpp"
#include "lagom/error.hpp"
#include "lagom/json_io.hpp"
#include "lagom/oracle.hpp"
#include "lagom/simulator.hpp"
#include "lagom/sweep.hpp"
#include "lagom/tuner.hpp"
#include "lagom/version.hpp"
#include "lagom/workloads.hpp"

using lagom::Json;

namespace {

enum Exit { kOk = 0, kValidation = 2, kIo = 3, kBudget = 4, kGrid = 5, kUsage = 106 };

// ------------------------------------------------------------- arguments ---
struct Args {
  std::string command;
  std::map<std::string, std::string> opt;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
};

const std::map<std::string, std::set<std::string>> kFlags = {
    {"simulate", {"workload", "configs", "params", "trace", "out"}},
    {"tune", {"workload", "params", "start", "budget", "log", "out", "profiler", "dag", "gpu"}},
    {"oracle", {"workload", "params", "grid", "limit", "out"}},
    {"compare", {"workload", "params", "grid", "limit", "budget", "profiler", "dag"}},
    {"sweep", {"workload", "configs", "params", "comm", "param", "values", "out", "profiler", "dag"}},
    {"gen", {"pattern", "layers", "seed", "m", "n", "out"}},
};
const std::map<std::string, std::set<std::string>> kRequired = {
    {"simulate", {"workload", "configs"}}, {"tune", {"workload"}},   {"oracle", {"workload"}},
    {"compare", {"workload"}},            {"sweep", {"workload", "comm", "param", "values"}},
    {"gen", {"pattern"}},
};

int usage(const std::string& why) {
  std::cerr << why << "\nusage: lagom {simulate|tune|oracle|compare|sweep|gen} [--option value ...]\n";
  return kUsage;
}

std::optional<Args> parse(int argc, char** argv, int& rc) {
  if (argc < 2) {
    rc = usage("a subcommand is required");
    return std::nullopt;
  }
  Args a;
  a.command = argv[1];
  if (!kFlags.count(a.command)) {
    rc = usage("unknown subcommand '" + a.command + "'");
    return std::nullopt;
  }
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) {
      rc = usage("unexpected argument '" + k + "'");
      return std::nullopt;
    }
    k = k.substr(2);
    std::string v;
    if (const auto eq = k.find('='); eq != std::string::npos) {
      v = k.substr(eq + 1);
      k = k.substr(0, eq);
    } else if (i + 1 < argc) {
      v = argv[++i];
    } else {
      rc = usage("--" + k + " needs a value");
      return std::nullopt;
    }
    if (!kFlags.at(a.command).count(k)) {
      rc = usage("unknown option --" + k + " for " + a.command);
      return std::nullopt;
    }
    a.opt[k] = v;
  }
  for (const auto& r : kRequired.at(a.command))
    if (!a.has(r)) {
      rc = usage("--" + r + " is required");
      return std::nullopt;
    }
  if (a.command == "tune" && a.has("start") && a.get("start") != "min" && a.get("start") != "nccl-default") {
    rc = usage("--start: expected min|nccl-default");
    return std::nullopt;
  }
  for (const char* num : {"budget"})
    if (a.has(num)) {
      char* end = nullptr;
      const long v = std::strtol(a.get(num).c_str(), &end, 10);
      if (*end || v <= 0) {
        rc = usage(std::string("--") + num + " must be a positive number");
        return std::nullopt;
      }
    }
  return a;
}

// ---------------------------------------------------------------- helpers ---
struct Inputs {
  std::string workload, configs, params;
};

lagom::SubspaceParams resolve_params(Inputs& in) {
  if (!in.params.empty()) return lagom::load_params(in.params);
  if (const char* env = std::getenv("LAGOM_PARAMS"); env && *env) {
    in.params = env;
    return lagom::load_params(in.params);
  }
  return lagom::SubspaceParams::defaults();
}

Json header(const std::string& command, const Inputs& in) {
  Json d;
  d["version"] = lagom::kVersion;
  d["command"] = command;
  Json digests;
  if (!in.workload.empty()) digests["workload"] = lagom::file_digest(in.workload);
  if (!in.configs.empty()) digests["configs"] = lagom::file_digest(in.configs);
  if (!in.params.empty()) digests["params"] = lagom::file_digest(in.params);
  d["inputs"] = digests;
  return d;
}

void emit(const Json& doc, const std::string& out) {
  if (out.empty()) std::cout << doc.dump(2) << '\n';
  else lagom::save_json(doc, out);
}

std::int64_t parse_size(const std::string& t) {
  if (t.empty()) throw lagom::Error(lagom::ErrorCode::InvalidInput, "value", "empty value");
  std::int64_t scale = 1;
  std::string digits = t;
  const char last = t.back();
  if (last == 'K' || last == 'k') scale = lagom::kKiB;
  if (last == 'M' || last == 'm') scale = lagom::kKiB * lagom::kKiB;
  if (scale != 1) digits.pop_back();
  std::size_t used = 0;
  std::int64_t v = 0;
  try {
    v = std::stoll(digits, &used);
  } catch (...) {
    used = 0;
  }
  if (used == 0 || used != digits.size())
    throw lagom::Error(lagom::ErrorCode::InvalidInput, "value", "cannot parse '" + t + "'");
  return v * scale;
}

std::vector<std::int64_t> parse_list(const std::string& csv) {
  std::vector<std::int64_t> out;
  std::size_t b = 0;
  while (b <= csv.size()) {
    const std::size_t e = csv.find(',', b);
    const std::string tok = csv.substr(b, e == std::string::npos ? std::string::npos : e - b);
    if (!tok.empty()) out.push_back(parse_size(tok));
    if (e == std::string::npos) break;
    b = e + 1;
  }
  return out;
}

struct Grid {
  std::vector<std::int64_t> nc{1, 2, 4, 8, 16};
  std::vector<std::int64_t> c{64 * lagom::kKiB, 256 * lagom::kKiB, 1024 * lagom::kKiB, 2048 * lagom::kKiB};
  std::vector<std::int64_t> nt{128};
};

Grid parse_grid(const std::string& spec) {
  Grid g;
  std::size_t b = 0;
  while (b < spec.size()) {
    std::size_t e = spec.find(';', b);
    if (e == std::string::npos) e = spec.size();
    const std::string part = spec.substr(b, e - b);
    const std::size_t eq = part.find('=');
    if (eq == std::string::npos)
      throw lagom::Error(lagom::ErrorCode::InvalidInput, "grid", "expected name=v1,v2,... in '" + part + "'");
    const std::string name = part.substr(0, eq);
    auto vals = parse_list(part.substr(eq + 1));
    if (name == "nc") g.nc = vals;
    else if (name == "c") g.c = vals;
    else if (name == "nt") g.nt = vals;
    else throw lagom::Error(lagom::ErrorCode::InvalidInput, "grid", "unknown grid parameter '" + name + "'");
    b = e + 1;
  }
  return g;
}

std::vector<std::vector<lagom::CommConfig>> grids_for(const lagom::Workload& w, const lagom::SubspaceParams& p,
                                                      const Grid& spec) {
  std::vector<std::vector<lagom::CommConfig>> out;
  for (const lagom::CommOp& op : w.comm_ops) {
    const auto key = lagom::select_subspace(op, w.gpu, p);
    const auto b = lagom::bounds_for(op, w.gpu);
    std::vector<lagom::CommConfig> g;
    for (std::int64_t nc : spec.nc) {
      if (nc < b.nc_min || nc > b.nc_max) continue;
      for (std::int64_t c : spec.c) {
        if (c < b.c_min || c > b.c_max) continue;
        for (std::int64_t nt : spec.nt) {
          if (!lagom::in_thread_ladder(static_cast<int>(nt))) continue;
          lagom::CommConfig cfg = lagom::minimum_config(key, b);
          cfg.num_channels = static_cast<int>(nc);
          cfg.num_threads = static_cast<int>(nt);
          cfg.chunk_size = c;
          g.push_back(cfg);
        }
      }
    }
    if (g.empty())
      throw lagom::Error(lagom::ErrorCode::InvalidInput, "grid", "grid excludes every config for comm '" + op.id + "'");
    out.push_back(std::move(g));
  }
  return out;
}

std::vector<lagom::CommConfig> seeds(const lagom::Workload& w, const lagom::SubspaceParams& p,
                                     const std::string& start) {
  std::vector<lagom::CommConfig> out;
  for (const lagom::CommOp& op : w.comm_ops) {
    const auto b = lagom::bounds_for(op, w.gpu);
    lagom::CommConfig c = lagom::minimum_config(lagom::select_subspace(op, w.gpu, p), b);
    if (start == "nccl-default") {
      c.num_channels = std::min(8, b.nc_max);
      c.num_threads = 512;
      c.chunk_size = std::clamp<std::int64_t>(2048 * lagom::kKiB, b.c_min, b.c_max);
    }
    out.push_back(c);
  }
  return out;
}

Json log_record(const lagom::Workload& w, const lagom::TuneRecord& r) {
  Json j;
  j["iter"] = r.iteration;
  j["comm_id"] = r.comm_index ? Json(w.comm_ops[*r.comm_index].id) : Json(nullptr);
  j["config"] = r.comm_index ? lagom::config_to_json(r.config) : Json(nullptr);
  j["x"] = r.comm_index ? Json(r.comm_time) : Json(nullptr);
  j["X"] = r.total_comm;
  j["Y"] = r.total_compute;
  j["Z"] = r.makespan;
  Json h, done = Json::array();
  for (std::size_t k = 0; k < r.priorities.size(); ++k) {
    h[w.comm_ops[k].id] = r.priorities[k];
    if (r.done[k]) done.push_back(w.comm_ops[k].id);
  }
  j["H_table"] = h;
  j["done"] = done;
  if (r.priority_after) j["H_after"] = *r.priority_after;
  else if (r.comm_index) j["H_after"] = nullptr;
  j["already_optimal"] = r.already_optimal;
  return j;
}

Json configs_with_ids(const lagom::Workload& w, const std::vector<lagom::CommConfig>& cs) {
  Json arr = Json::array();
  for (std::size_t j = 0; j < cs.size(); ++j) {
    Json c = lagom::config_to_json(cs[j]);
    c["comm_id"] = w.comm_ops[j].id;
    arr.push_back(c);
  }
  return arr;
}

// ---------------------------------------------------------------- commands --
int cmd_simulate(const Args& a) {
  Inputs in{a.get("workload"), a.get("configs"), a.get("params")};
  const lagom::Workload w = lagom::validate(lagom::load_workload(in.workload));
  const auto configs = lagom::load_configs(in.configs);
  const auto params = resolve_params(in);
  const lagom::SimResult r = lagom::simulate(w, configs, params);
  if (a.has("trace")) lagom::export_trace(r, a.get("trace"));
  Json d = header("simulate", in);
  d["result"] = {{"X", r.total_comm}, {"Y", r.total_compute}, {"Z", r.makespan}};
  Json comp = Json::array(), comm = Json::array();
  for (std::size_t i = 0; i < w.compute_ops.size(); ++i)
    comp.push_back({{"id", w.compute_ops[i].id}, {"time_us", r.comp_times[i]}});
  for (std::size_t j = 0; j < w.comm_ops.size(); ++j)
    comm.push_back({{"id", w.comm_ops[j].id}, {"time_us", r.comm_times[j]}});
  d["result"]["compute"] = comp;
  d["result"]["comm"] = comm;
  emit(d, a.get("out"));
  return kOk;
}

// GPU profiler: every rank builds the replay engine over the DAG; rank 0
// drives (tune / sweep / grid), the other ranks serve replay commands.
struct GpuSession {
  std::unique_ptr<lagom::b200::Coordinator> coord;
  std::unique_ptr<lagom::b200::ReplayEngine> engine;
  bool driver() const { return engine->rank() == 0; }
};

std::unique_ptr<GpuSession> gpu_session(const Args& a, const lagom::Workload& w) {
  if (!a.has("dag")) throw lagom::Error(lagom::ErrorCode::InvalidInput, "dag", "--profiler gpu needs --dag");
  const auto env_int = [](const char* k, int d) {
    const char* v = std::getenv(k);
    return v && *v ? std::atoi(v) : d;
  };
  const int rank = env_int("RANK", 0), world = env_int("WORLD_SIZE", 1), local = env_int("LOCAL_RANK", rank);
  const char* job = std::getenv("LAGOM_JOB");
  const char* port = std::getenv("MASTER_PORT");
  const std::string name = std::string("lagom_cli_") + (job ? job : (port ? port : "0"));
  const lagom::b200::ReplayDag dag = lagom::b200::replay_dag_from_json(lagom::read_file(a.get("dag")));
  if (dag.comm_ops.size() != w.comm_ops.size())
    throw lagom::Error(lagom::ErrorCode::InvalidInput, "dag", "the DAG must have one comm op per workload comm op");
  auto s = std::make_unique<GpuSession>();
  s->coord = lagom::b200::make_shm_coordinator(name, rank, world);
  lagom::b200::ReplayOptions o;
  o.device = local;
  o.sm_partition = lagom::b200::kPartitionAuto;
  o.enable_nccl = false;
  o.nvls = world > 1;
  s->engine = std::make_unique<lagom::b200::ReplayEngine>(dag, *s->coord, o);
  if (!s->driver()) s->engine->serve();  // returns when the driver stops the engine
  return s;
}

int cmd_tune(const Args& a) {
  Inputs in{a.get("workload"), "", a.get("params")};
  const lagom::Workload w = lagom::validate(lagom::load_workload(in.workload));
  const auto params = resolve_params(in);
  const std::string start = a.get("start", "min");
  const int budget = std::atoi(a.get("budget", "500").c_str());
  const auto init = seeds(w, params, start);
  const std::string profiler = a.get("profiler", "sim");
  lagom::TuneResult r;
  if (profiler == "gpu") {
    auto gs = gpu_session(a, w);
    if (!gs->driver()) return kOk;  // a serving rank, done
    r = lagom::tune(w, init, lagom::b200::make_gpu_profiler(*gs->engine), budget);
    gs->engine->stop();
  } else if (profiler == "sim") {
    r = lagom::tune(w, init, lagom::make_sim_profiler(w, params), budget);
  } else {
    throw lagom::Error(lagom::ErrorCode::InvalidInput, "profiler", "expected sim|gpu");
  }
  if (a.has("log")) {
    std::ofstream log(a.get("log"), std::ios::binary);
    if (!log) throw lagom::Error(lagom::ErrorCode::IoFailure, a.get("log"), "cannot open for writing");
    for (const auto& rec : r.log) log << log_record(w, rec).dump() << '\n';
  }
  Json d = header("tune", in);
  d["start"] = start;
  d["budget"] = budget;
  d["profile_calls"] = r.profile_calls;
  d["budget_exhausted"] = r.budget_exhausted;
  d["boundary_condition"] = r.boundary_condition;
  d["initial_Z"] = r.initial_makespan;
  d["final"] = {{"X", r.final_profile.total_comm}, {"Y", r.final_profile.total_compute},
                {"Z", r.final_profile.makespan}};
  d["configs"] = configs_with_ids(w, r.configs);
  emit(d, a.get("out"));
  return r.budget_exhausted ? kBudget : kOk;
}

int cmd_oracle(const Args& a) {
  Inputs in{a.get("workload"), "", a.get("params")};
  const lagom::Workload w = lagom::validate(lagom::load_workload(in.workload));
  const auto params = resolve_params(in);
  const auto grids = grids_for(w, params, parse_grid(a.get("grid")));
  const std::int64_t limit = a.has("limit") ? parse_size(a.get("limit")) : 1000000;
  const auto t0 = std::chrono::steady_clock::now();
  const lagom::OracleResult r = lagom::exhaustive(w, grids, params, limit);
  const auto us =
      std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count();
  Json d = header("oracle", in);
  d["best_Z"] = r.makespan;
  d["evaluations"] = r.evaluations;
  d["wall_time_us"] = us;
  d["best_configs"] = configs_with_ids(w, r.configs);
  emit(d, a.get("out"));
  return kOk;
}

int cmd_compare(const Args& a) {
  Inputs in{a.get("workload"), "", a.get("params")};
  const lagom::Workload w = lagom::validate(lagom::load_workload(in.workload));
  const auto params = resolve_params(in);
  const auto grids = grids_for(w, params, parse_grid(a.get("grid")));
  const std::int64_t limit = a.has("limit") ? parse_size(a.get("limit")) : 1000000;
  const int budget = std::atoi(a.get("budget", "500").c_str());
  const std::string profiler = a.get("profiler", "sim");
  if (profiler == "gpu") {
    // Measured: the grid and the tuner profile on the GPU replay; the naive
    // strawman's picks (it reads the model directly, reference oracle.cpp:85-88)
    // are measured once. Same CSV rows as the simulated compare.
    auto gs = gpu_session(a, w);
    if (!gs->driver()) return kOk;
    const lagom::ProfileFn f = lagom::b200::make_gpu_profiler(*gs->engine);
    const auto ex = lagom::b200::exhaustive_with(f, w, grids, limit);
    const auto tu = lagom::tune(w, seeds(w, params, "min"), f, budget);
    const auto nv = lagom::sequential_naive(w, params);
    const double nv_z = f(nv.configs).makespan;
    gs->engine->stop();
    std::cout.precision(17);
    std::cout << "method,Z,evaluations\n"
              << "exhaustive," << ex.makespan << ',' << ex.evaluations << '\n'
              << "tune," << tu.final_profile.makespan << ',' << tu.profile_calls << '\n'
              << "naive," << nv_z << ',' << nv.profile_calls << '\n';
    return tu.budget_exhausted ? kBudget : kOk;
  }
  if (profiler != "sim") throw lagom::Error(lagom::ErrorCode::InvalidInput, "profiler", "expected sim|gpu");
  const auto ex = lagom::exhaustive(w, grids, params, limit);
  const auto tu = lagom::tune(w, seeds(w, params, "min"), lagom::make_sim_profiler(w, params), budget);
  const auto nv = lagom::sequential_naive(w, params);
  std::cout.precision(17);
  std::cout << "method,Z,evaluations\n"
            << "exhaustive," << ex.makespan << ',' << ex.evaluations << '\n'
            << "tune," << tu.final_profile.makespan << ',' << tu.profile_calls << '\n'
            << "naive," << nv.makespan << ',' << nv.profile_calls << '\n';
  return tu.budget_exhausted ? kBudget : kOk;
}

int cmd_sweep(const Args& a) {
  Inputs in{a.get("workload"), a.get("configs"), a.get("params")};
  const lagom::Workload w = lagom::validate(lagom::load_workload(in.workload));
  const auto params = resolve_params(in);
  std::vector<lagom::CommConfig> base;
  if (!in.configs.empty()) {
    base = lagom::load_configs(in.configs);
  } else {
    base = seeds(w, params, "min");
    for (std::size_t j = 0; j < base.size(); ++j) {
      const auto b = lagom::bounds_for(w.comm_ops[j], w.gpu);
      base[j].num_channels = std::min(4, b.nc_max);
      base[j].num_threads = 128;
      base[j].chunk_size = std::clamp<std::int64_t>(1024 * lagom::kKiB, b.c_min, b.c_max);
    }
  }
  const std::string profiler = a.get("profiler", "sim");
  const auto param = lagom::sweep_param_from_string(a.get("param"));
  std::vector<lagom::SweepRow> rows;
  if (profiler == "gpu") {  // every value a measured replay of the DAG
    auto gs = gpu_session(a, w);
    if (!gs->driver()) return kOk;
    rows = lagom::b200::sweep_with(lagom::b200::make_gpu_profiler(*gs->engine), w, base, a.get("comm"), param,
                                   parse_list(a.get("values")));
    gs->engine->stop();
  } else if (profiler == "sim") {
    rows = lagom::run_sweep(w, base, params, a.get("comm"), param, parse_list(a.get("values")));
  } else {
    throw lagom::Error(lagom::ErrorCode::InvalidInput, "profiler", "expected sim|gpu");
  }
  const std::string csv = lagom::sweep_csv(rows);
  if (!a.has("out")) {
    std::cout << csv;
  } else {
    std::ofstream out(a.get("out"), std::ios::binary);
    if (!out) throw lagom::Error(lagom::ErrorCode::IoFailure, a.get("out"), "cannot open for writing");
    out << csv;
  }
  return kOk;
}

int cmd_gen(const Args& a) {
  const std::string pattern = a.get("pattern");
  const int layers = std::atoi(a.get("layers", "4").c_str());
  const std::uint64_t seed = std::strtoull(a.get("seed", "1").c_str(), nullptr, 10);
  lagom::Workload w;
  if (pattern == "fsdp") w = lagom::gen_fsdp(layers, seed);
  else if (pattern == "tp") w = lagom::gen_tp_domino(layers, seed);
  else if (pattern == "ep") w = lagom::gen_ep_dualbatch(layers, seed);
  else if (pattern == "allreduce-pair") w = lagom::gen_allreduce_pair();
  else if (pattern == "random")
    w = lagom::gen_random(std::atoi(a.get("m", "4").c_str()), std::atoi(a.get("n", "2").c_str()), seed);
  else
    throw lagom::Error(lagom::ErrorCode::InvalidInput, "pattern",
                       "expected fsdp|tp|ep|allreduce-pair|random, got '" + pattern + "'");
  lagom::validate(w);
  const Json d = lagom::workload_to_json(w);
  if (!a.has("out")) std::cout << d.dump(2) << '\n';
  else lagom::save_json(d, a.get("out"));
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  int rc = 0;
  const auto args = parse(argc, argv, rc);
  if (!args) return rc;
  try {
    const std::string& c = args->command;
    if (c == "simulate") return cmd_simulate(*args);
    if (c == "tune") return cmd_tune(*args);
    if (c == "oracle") return cmd_oracle(*args);
    if (c == "compare") return cmd_compare(*args);
    if (c == "sweep") return cmd_sweep(*args);
    return cmd_gen(*args);
  } catch (const lagom::Error& e) {
    std::cerr << e.what() << '\n';
    return e.code() == lagom::ErrorCode::IoFailure ? kIo : e.code() == lagom::ErrorCode::GridTooLarge ? kGrid
                                                                                                      : kValidation;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kValidation;
  }
}
