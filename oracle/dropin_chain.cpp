// Test infrastructure (never product code): the per-step frontier API --
// min_energy_schedule, get_next_schedule, discretize (frontier.hpp:73-161)
// -- driven in a chain, printed as JSON lines.  Compiled twice by
// oracle/Makefile: against the UNMODIFIED reference headers
// (oracle/_ref/dropin_chain_ref) and against the B200 drop-in
// include/perseus_b200/perseus/frontier.hpp + the product library
// (oracle/_ref/dropin_chain_b200).  tests/test_gpu_dropin.py requires the two
// outputs to be identical (timing lines aside) and reports both timings.
//
//   dropin_chain <spec> <steps> [tau]   spec: config:K (G9) | diamond
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <string>
#include <vector>

#include "perseus/dag.hpp"
#include "perseus/frontier.hpp"
#include "g9.hpp"

using namespace perseus;

namespace {

struct Fnv {
  std::uint64_t h = 1469598103934665603ull;
  void add(std::int64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= static_cast<std::uint64_t>(v >> (8 * i)) & 0xff;
      h *= 1099511628211ull;
    }
  }
};

std::uint64_t hash_of(const EnergySchedule& s) {
  Fnv f;
  for (auto v : s.planned_t) f.add(v);
  for (auto v : s.planned_e) f.add(v);
  for (auto v : s.freq_mhz) f.add(v);
  for (auto v : s.realized_t) f.add(v);
  for (auto v : s.realized_e) f.add(v);
  return f.h;
}

void instance(const std::string& spec, NodeDag& dag, CostModel& model) {
  ProfileSet set;
  if (spec == "diamond") {
    std::vector<Computation> comps{{0, 0, 0, Kind::Forward}, {1, 1, 0, Kind::Forward}, {2, 2, 0, Kind::Forward},
                                   {3, 3, 0, Kind::Forward}, {4, 4, 0, Kind::Forward}};
    dag = finalize_custom_dag(comps, {{0, 1}, {1, 2}, {0, 3}, {4, 2}});
    set.p_blocking_watts = kDefaultBlockingWatts;
    auto two = [](int stage, Quanta t0, Millijoules e0, Quanta t1, Millijoules e1) {
      return FrequencyProfile{ClassKey{stage, Kind::Forward},
                              {ProfilePoint{1400, t0, e0}, ProfilePoint{1000, t1, e1}}};
    };
    set.profiles.push_back(two(0, 1000, 4000, 3000, 1000));
    set.profiles.push_back(two(1, 1000, 625, 3000, 400));
    set.profiles.push_back(two(2, 1000, 4000, 3000, 1000));
    set.profiles.push_back(two(3, 4000, 625, 6000, 400));
    set.profiles.push_back(two(4, 4000, 625, 6000, 400));
  } else {
    pb_g9::Params p = pb_g9::named_config(1);
    if (spec.rfind("config:", 0) == 0) p = pb_g9::named_config(std::stoi(spec.substr(7)));
    dag = build_1f1b(p.stages, p.microbatches);
    set.p_blocking_watts = 75.0;
    const auto bases = pb_g9::stage_bases(p);
    for (int s = 0; s < p.stages; ++s)
      for (int k = 0; k < 2; ++k) {
        FrequencyProfile fp;
        fp.key = ClassKey{s, k == 0 ? Kind::Forward : Kind::Backward};
        for (const auto& pt : pb_g9::stage_profile(bases[s], k == 1))
          fp.points.push_back(ProfilePoint{pt.freq_mhz, pt.time, pt.energy});
        set.profiles.push_back(fp);
      }
  }
  model = CostModel::build(set, kDefaultQuantumUs);
}

void print_schedule(const char* what, int k, const EnergySchedule& s) {
  std::printf("{\"what\":\"%s\",\"k\":%d,\"t_planned\":%" PRId64 ",\"t_realized\":%" PRId64
              ",\"eff_planned\":%.17g,\"eff_realized\":%.17g,\"hash\":\"%016" PRIx64 "\"}\n",
              what, k, static_cast<std::int64_t>(s.t_planned), static_cast<std::int64_t>(s.t_realized),
              s.eff_planned_mj, s.eff_realized_mj, hash_of(s));
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: dropin_chain <spec> <steps> [tau]\n");
    return 2;
  }
  const std::string spec = argv[1];
  const int steps = std::stoi(argv[2]);
  const Quanta tau = argc > 3 ? std::stoll(argv[3]) : 1000;
  NodeDag dag;
  CostModel model;
  instance(spec, dag, model);
  const auto t0 = std::chrono::steady_clock::now();
  EnergySchedule s = min_energy_schedule(dag, model);
  print_schedule("seed", 0, s);
  int k = 0;
  double step_s = 0, disc_s = 0;
  for (; k < steps; ++k) {
    StepInfo info;
    const auto a = std::chrono::steady_clock::now();
    auto next = get_next_schedule(dag, s, model, tau, &info);
    const auto b = std::chrono::steady_clock::now();
    step_s += std::chrono::duration<double>(b - a).count();
    if (!next) {
      std::printf("{\"what\":\"stop\",\"k\":%d}\n", k + 1);
      break;
    }
    std::string ids;
    for (int c : info.sped_up) ids += (ids.empty() ? "" : ",") + std::to_string(c);
    ids += "|";
    for (int c : info.slowed_down) ids += std::to_string(c) + ",";
    std::printf("{\"what\":\"step\",\"k\":%d,\"cut\":%" PRId64 ",\"ids\":\"%s\"}\n", k + 1,
                static_cast<std::int64_t>(info.cut_cost), ids.c_str());
    print_schedule("next", k + 1, *next);
    const auto c = std::chrono::steady_clock::now();
    const EnergySchedule d = discretize(*next, dag, model);
    disc_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - c).count();
    print_schedule("discretized", k + 1, d);
    s = std::move(*next);
  }
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"what\":\"timing\",\"steps\":%d,\"wall_s\":%.6f,\"get_next_s\":%.6f,\"discretize_s\":%.6f}\n", k,
              wall, step_s, disc_s);
  return 0;
}
