// Search-speed driver — TEST / BASELINE INFRASTRUCTURE.
//
// Times tune(start=min) with the simulator ProfileFn on the reference's own
// sample workloads (BASELINE config 1: gen allreduce-pair, fsdp(4,7),
// tp(3,5), ep(2,11), fsdp(32,1); reference README.md:60,70 and SURVEY.md
// Appendix A.5), default params, budget 500, best of `reps` runs on one
// thread. Compiled twice: against the product (build/tune_speed) and against
// the reference build (oracle/_ref/tune_speed_ref, namespace lagom_ref), so
// bench.py's cpu_baseline leg can put the reference CPU tuner's speed next to
// the product's on the same host. Prints one JSON object.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "lagom/tuner.hpp"
#include "lagom/workloads.hpp"

using namespace lagom;

int main(int argc, char** argv) {
  const int reps = argc > 1 ? std::atoi(argv[1]) : 7;
  const SubspaceParams params = SubspaceParams::defaults();
  struct Case {
    const char* name;
    Workload w;
  };
  const std::vector<Case> cases = {{"allreduce-pair", gen_allreduce_pair()},
                                   {"fsdp(4,7)", gen_fsdp(4, 7)},
                                   {"tp(3,5)", gen_tp_domino(3, 5)},
                                   {"ep(2,11)", gen_ep_dualbatch(2, 11)},
                                   {"fsdp(32,1)", gen_fsdp(32, 1)}};
  std::printf("{");
  bool first = true;
  for (const Case& c : cases) {
    std::vector<CommConfig> init;
    for (const CommOp& op : c.w.comm_ops)
      init.push_back(minimum_config(select_subspace(op, c.w.gpu, params), bounds_for(op, c.w.gpu)));
    const ProfileFn f = make_sim_profiler(c.w, params);
    double best = 1e300;
    int calls = 0;
    double z = 0.0;
    for (int k = 0; k < reps; ++k) {
      const auto t0 = std::chrono::steady_clock::now();
      const TuneResult r = tune(c.w, init, f, 500);
      const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      if (us < best) best = us;
      calls = r.profile_calls;
      z = r.final_profile.makespan;
    }
    std::printf("%s\"%s\": {\"us\": %.3f, \"calls\": %d, \"us_per_call\": %.4f, \"final_Z\": \"%a\"}", first ? "" : ", ",
                c.name, best, calls, best / (calls > 0 ? calls : 1), z);
    first = false;
  }
  std::printf("}\n");
  return 0;
}
