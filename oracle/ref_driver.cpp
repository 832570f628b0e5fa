// Test infrastructure (NOT product code): drives the UNMODIFIED reference
// headers under /root/reference/proj/include through their public API and
// dumps results as JSON lines.  Built by oracle/Makefile into oracle/_ref/
// (git-ignored) while /root/reference is present; the prebuilt binary
// travels to the GPU box, where it is the `--impl reference` CPU arm of
// bench.py and the generator of tests/golden/ fixtures.
//
// Modes
//   walk <spec>...           frontier walk per instance (discover_frontier
//                            loop restated with StepInfo, frontier.hpp:166-189)
//   walkprefix <K> <spec>... the same walk stopped after K steps
//                            (reason "max_steps" when T_min is not reached)
//   flow <seed> <count> <max_nodes> <max_cap>
//                            testutil::random_flow_graph corpus through
//                            max_flow_lower_bounds + min_cut_from_flow
//   slack <seed> <count>     random DAGs through annotate_slack
//   bench <threads> <spec>...  wall-time of discover_frontier over a thread
//                            pool (one instance per task, LPT order given)
//   fit <spec>               CostModel curves (bit patterns) of an instance
//   budget <s> <threads> <spec>...   walks bounded by seconds per instance
//   capped <k> <threads> <spec>...   walks bounded by k steps per instance
//   artifacts <quantum> <spec>...
//                            frontier.csv + schedule_<k>.json bytes
//                            (serde.hpp frontier_csv / schedule_json dump(2))
//                            for the first, middle and last schedules
//   brute <spec>...          brute_force_frontier (oracle.hpp:47-114) points
//   rule5 <first> <count> [maxn]  r5 specs whose walk hits SURVEY §7 rule 5
//   getnext <tau> (<spec> <t0,t1,...>)...  get_next_schedule from a caller
//                            schedule (planned times anywhere)
//   savings <P> <factors,...> <spec>...
//                            straggler_savings (baselines.hpp:162-188) on the
//                            reference frontier: rows + the looked-up point
//
// Instance specs
//   g9:N:M:B:imbalance:seed:straggler:phi     SURVEY §8d generator
//   config:K[:phi]                            named configs 1-4
//   batch:I                                   config-5 instance I
//   diamond | lone:ft:fe:st:se                test_frontier.cpp:23-58
//   grid:seed:stages:micro[:maxpts]           testutil::grid_profiles walk
//   r5:seed[:maxn]                            random custom DAG (rule-5 search)
//   cubic:seed:stages:micro                   testutil::cubic_profiles walk
#include <atomic>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "helpers.hpp"  // reference tests: generators + independent oracles
#include "perseus/frontier.hpp"
#include "perseus/serde.hpp"
#include "g9.hpp"

using namespace perseus;

namespace {

struct Instance {
  std::string spec;
  NodeDag dag;
  ProfileSet set;
  CostModel model;
  Quanta tau = 1000;
};

std::vector<std::string> split(const std::string& s, char d) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, d)) out.push_back(tok);
  return out;
}

ProfileSet g9_profiles(const pb_g9::Params& p) {
  ProfileSet set;
  set.p_blocking_watts = 75.0;
  const auto bases = pb_g9::stage_bases(p);
  for (int s = 0; s < p.stages; ++s) {
    for (int k = 0; k < 2; ++k) {
      FrequencyProfile fp;
      fp.key = ClassKey{s, k == 0 ? Kind::Forward : Kind::Backward};
      for (const auto& pt : pb_g9::stage_profile(bases[s], k == 1))
        fp.points.push_back(ProfilePoint{pt.freq_mhz, pt.time, pt.energy});
      set.profiles.push_back(fp);
    }
  }
  return set;
}

Instance make_instance(const std::string& spec) {
  Instance in;
  in.spec = spec;
  const auto t = split(spec, ':');
  auto g9 = [&](const pb_g9::Params& p) {
    in.dag = build_1f1b(p.stages, p.microbatches);
    in.set = g9_profiles(p);
  };
  if (t[0] == "g9") {
    pb_g9::Params p;
    p.stages = std::stoi(t[1]);
    p.microbatches = std::stoi(t[2]);
    p.base = std::stoi(t[3]);
    p.imbalance = std::stod(t[4]);
    p.seed = static_cast<std::uint32_t>(std::stoul(t[5]));
    p.straggler_stage = std::stoi(t[6]);
    p.phi = std::stod(t[7]);
    g9(p);
  } else if (t[0] == "config") {
    g9(pb_g9::named_config(std::stoi(t[1]), t.size() > 2 ? std::stod(t[2]) : 1.0));
  } else if (t[0] == "batch") {
    g9(pb_g9::batch_instance(std::stoi(t[1])));
  } else if (t[0] == "diamond") {
    std::vector<Computation> comps{{0, 0, 0, Kind::Forward}, {1, 1, 0, Kind::Forward},
                                   {2, 2, 0, Kind::Forward}, {3, 3, 0, Kind::Forward},
                                   {4, 4, 0, Kind::Forward}};
    in.dag = finalize_custom_dag(comps, {{0, 1}, {1, 2}, {0, 3}, {4, 2}});
    in.set.p_blocking_watts = kDefaultBlockingWatts;
    auto two = [](int stage, Quanta t0, Millijoules e0, Quanta t1, Millijoules e1) {
      return FrequencyProfile{ClassKey{stage, Kind::Forward},
                              {ProfilePoint{1400, t0, e0}, ProfilePoint{1000, t1, e1}}};
    };
    in.set.profiles.push_back(two(0, 1000, 4000, 3000, 1000));
    in.set.profiles.push_back(two(1, 1000, 625, 3000, 400));
    in.set.profiles.push_back(two(2, 1000, 4000, 3000, 1000));
    in.set.profiles.push_back(two(3, 4000, 625, 6000, 400));
    in.set.profiles.push_back(two(4, 4000, 625, 6000, 400));
  } else if (t[0] == "lone") {
    std::vector<Computation> comps{{0, 0, 0, Kind::Forward}};
    in.dag = finalize_custom_dag(comps, {});
    in.set.p_blocking_watts = kDefaultBlockingWatts;
    in.set.profiles.push_back(
        {ClassKey{0, Kind::Forward},
         {ProfilePoint{1400, std::stoll(t[1]), std::stoll(t[2])},
          ProfilePoint{1000, std::stoll(t[3]), std::stoll(t[4])}}});
    if (t.size() > 5) in.tau = std::stoll(t[5]);
  } else if (t[0] == "grid") {
    std::mt19937 rng(static_cast<std::uint32_t>(std::stoul(t[1])));
    const int stages = std::stoi(t[2]), micro = std::stoi(t[3]);
    const int maxpts = t.size() > 4 ? std::stoi(t[4]) : 4;
    in.dag = build_1f1b(stages, micro);
    in.set = testutil::grid_profiles(rng, stages, 1000, maxpts, true);
  } else if (t[0] == "cubic") {
    std::mt19937 rng(static_cast<std::uint32_t>(std::stoul(t[1])));
    const int stages = std::stoi(t[2]), micro = std::stoi(t[3]);
    std::uniform_real_distribution<double> scale(0.8, 1.3);
    std::vector<double> fs(stages), bs(stages);
    for (int s = 0; s < stages; ++s) {
      fs[s] = scale(rng);
      bs[s] = 2.0 * scale(rng);
    }
    in.dag = build_1f1b(stages, micro);
    in.set = testutil::cubic_profiles(stages, {1400, 1300, 1200, 1100, 1000, 900}, 4.0e6, fs, bs);
  } else if (t[0] == "r5") {
    // small random custom DAG for the rule-5 search (mode_rule5): every
    // computation its own class, ~1/3 constant (one Pareto point), the rest
    // grid profiles with 2-4 points on tau multiples
    std::mt19937 rng(static_cast<std::uint32_t>(std::stoul(t[1])));
    const int n = std::uniform_int_distribution<int>(3, t.size() > 2 ? std::stoi(t[2]) : 8)(rng);
    std::vector<Computation> comps;
    for (int i = 0; i < n; ++i) comps.push_back(Computation{i, i, 0, Kind::Forward});
    std::vector<std::pair<int, int>> edges;
    std::uniform_real_distribution<double> coin(0, 1);
    for (int u = 0; u < n; ++u)
      for (int v = u + 1; v < n; ++v)
        if (coin(rng) < 0.4) edges.emplace_back(u, v);
    in.dag = finalize_custom_dag(comps, edges);
    in.set.p_blocking_watts = kDefaultBlockingWatts;
    for (int i = 0; i < n; ++i) {
      if (coin(rng) < 0.35) {
        const Quanta b = std::uniform_int_distribution<int>(1, 9)(rng) * 1000;
        in.set.profiles.push_back(  // dominated slow point: Pareto set collapses to one point
            {ClassKey{i, Kind::Forward}, {ProfilePoint{1400, b, 3000}, ProfilePoint{1200, b + 1000, 3500}}});
      } else {
        in.set.profiles.push_back(testutil::grid_profile(rng, ClassKey{i, Kind::Forward}, 1000, 4, false));
      }
    }
  } else {
    std::fprintf(stderr, "unknown spec %s\n", spec.c_str());
    std::exit(2);
  }
  in.model = CostModel::build(in.set, kDefaultQuantumUs);
  return in;
}

// FNV-1a over int64 words; the tests recompute it from our expansion.
struct Fnv {
  std::uint64_t h = 1469598103934665603ull;
  void add(std::int64_t v) {
    std::uint64_t u = static_cast<std::uint64_t>(v);
    for (int i = 0; i < 8; ++i) {
      h ^= (u >> (8 * i)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
};

std::uint64_t schedule_hash(const EnergySchedule& s) {
  Fnv f;
  for (auto v : s.planned_t) f.add(v);
  for (auto v : s.planned_e) f.add(v);
  for (auto v : s.freq_mhz) f.add(v);
  for (auto v : s.realized_t) f.add(v);
  for (auto v : s.realized_e) f.add(v);
  return f.h;
}

template <class T>
void put_list(std::string& o, const std::vector<T>& v) {
  o += '[';
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) o += ',';
    o += std::to_string(v[i]);
  }
  o += ']';
}

std::string dbl(double d) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", d);
  return buf;
}

std::string instance_json(const Instance& in) {
  std::string o = "{\"n\":" + std::to_string(in.dag.computations.size());
  o += ",\"tau\":" + std::to_string(in.tau);
  o += ",\"blocking_watts\":" + dbl(in.model.blocking.watts);
  o += ",\"quantum_us\":" + std::to_string(in.model.quantum_us);
  o += ",\"comps\":[";
  for (size_t i = 0; i < in.dag.computations.size(); ++i) {
    const auto& c = in.dag.computations[i];
    if (i) o += ',';
    o += "[" + std::to_string(c.stage) + "," + std::to_string(static_cast<int>(c.kind)) + "," +
         std::to_string(c.microbatch.value_or(-1)) + "]";
  }
  o += "],\"edges\":[";
  for (size_t i = 0; i < in.dag.edges.size(); ++i) {
    if (i) o += ',';
    o += "[" + std::to_string(in.dag.edges[i].first) + "," + std::to_string(in.dag.edges[i].second) + "]";
  }
  o += "],\"profiles\":[";
  for (size_t i = 0; i < in.set.profiles.size(); ++i) {
    const auto& p = in.set.profiles[i];
    if (i) o += ',';
    o += "{\"stage\":" + std::to_string(p.key.stage) + ",\"kind\":" +
         std::to_string(static_cast<int>(p.key.kind)) + ",\"points\":[";
    for (size_t j = 0; j < p.points.size(); ++j) {
      if (j) o += ',';
      o += "[" + std::to_string(p.points[j].freq_mhz) + "," + std::to_string(p.points[j].time) +
           "," + std::to_string(p.points[j].energy) + "]";
    }
    o += "]}";
  }
  o += "]}";
  return o;
}

std::string curves_json(const CostModel& m) {
  std::string o = "[";
  bool first = true;
  for (const auto& [key, cm] : m.classes) {
    if (!first) o += ',';
    first = false;
    o += "{\"stage\":" + std::to_string(key.stage) + ",\"kind\":" +
         std::to_string(static_cast<int>(key.kind)) + ",\"constant\":" +
         (cm.is_constant ? "true" : "false") + ",\"pareto\":[";
    for (size_t j = 0; j < cm.pareto.size(); ++j) {
      if (j) o += ',';
      o += "[" + std::to_string(cm.pareto[j].freq_mhz) + "," + std::to_string(cm.pareto[j].time) +
           "," + std::to_string(cm.pareto[j].energy) + "]";
    }
    o += "]";
    if (cm.curve) {
      std::uint64_t a, b, c;
      std::memcpy(&a, &cm.curve->a, 8);
      std::memcpy(&b, &cm.curve->b, 8);
      std::memcpy(&c, &cm.curve->c, 8);
      char buf[160];
      std::snprintf(buf, sizeof buf, ",\"curve_bits\":[\"%016" PRIx64 "\",\"%016" PRIx64 "\",\"%016" PRIx64 "\"]",
                    a, b, c);
      o += buf;
      o += ",\"t_min\":" + std::to_string(cm.curve->t_min) + ",\"t_max\":" + std::to_string(cm.curve->t_max);
    }
    o += "}";
  }
  o += "]";
  return o;
}

// discover_frontier (frontier.hpp:166-189) restated step by step so that
// StepInfo and the terminal reason are observable; cross-checked against
// discover_frontier itself for small instances (check=true).
std::string walk_json(const Instance& in, bool full, bool check, long long max_steps = -1) {
  const auto t0 = std::chrono::steady_clock::now();
  const AllMaxAssignment am = all_max_assignment(in.dag, in.model);
  const Quanta t_min = simulate(in.dag, am.durations).iteration_time;
  EnergySchedule cur = min_energy_schedule(in.dag, in.model);
  const Quanta t_star = cur.t_planned;
  std::vector<EnergySchedule> pts;
  pts.push_back(discretize(cur, in.dag, in.model));
  std::vector<StepInfo> infos;
  std::vector<Quanta> step_sizes;
  std::string reason = "at_t_min";
  while (cur.t_planned > t_min) {
    if (max_steps >= 0 && static_cast<long long>(infos.size()) >= max_steps) {
      reason = "max_steps";
      break;
    }
    const Quanta step = std::min<Quanta>(in.tau, cur.t_planned - t_min);
    StepInfo info;
    auto next = get_next_schedule(in.dag, cur, in.model, step, &info);
    if (!next) {
      const EdgeDag e = to_edge_centric(in.dag);
      const SlackAnnotation sl = annotate_slack(e, cur.planned_t);
      const FlowGraph g = build_capacity_dag(critical_subdag(e, sl), cur.planned_t, in.model, step);
      reason = max_flow_lower_bounds(g).has_value() ? "infinite_cut" : "infeasible";
      break;
    }
    if (next->t_planned >= cur.t_planned) {
      reason = "no_progress";
      break;
    }
    cur = std::move(*next);
    cur.schedule_id = static_cast<int>(pts.size());
    pts.push_back(discretize(cur, in.dag, in.model));
    infos.push_back(std::move(info));
    step_sizes.push_back(step);
  }
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (check) {
    const Frontier f = discover_frontier(in.dag, in.model, in.tau);
    bool ok = f.t_min == t_min && f.t_star == t_star && f.schedules.size() == pts.size();
    for (size_t k = 0; ok && k < pts.size(); ++k)
      ok = schedule_hash(f.schedules[k]) == schedule_hash(pts[k]) &&
           f.schedules[k].t_planned == pts[k].t_planned &&
           f.schedules[k].t_realized == pts[k].t_realized &&
           f.schedules[k].eff_planned_mj == pts[k].eff_planned_mj &&
           f.schedules[k].eff_realized_mj == pts[k].eff_realized_mj;
    if (!ok) {
      std::fprintf(stderr, "restated walk disagrees with discover_frontier on %s\n", in.spec.c_str());
      std::exit(3);
    }
  }
  std::string o = "{\"spec\":\"" + in.spec + "\",\"instance\":" + instance_json(in);
  o += ",\"curves\":" + curves_json(in.model);
  o += ",\"t_min\":" + std::to_string(t_min) + ",\"t_star\":" + std::to_string(t_star);
  o += ",\"steps\":" + std::to_string(infos.size()) + ",\"reason\":\"" + reason + "\"";
  o += ",\"wall_s\":" + dbl(wall);
  std::vector<Quanta> tp, tr;
  std::vector<Millijoules> spe, sre;
  std::vector<std::string> hashes;
  o += ",\"eff_planned\":[";
  for (size_t k = 0; k < pts.size(); ++k) {
    if (k) o += ',';
    o += dbl(pts[k].eff_planned_mj);
  }
  o += "],\"eff_realized\":[";
  for (size_t k = 0; k < pts.size(); ++k) {
    if (k) o += ',';
    o += dbl(pts[k].eff_realized_mj);
  }
  o += "]";
  for (const auto& s : pts) {
    tp.push_back(s.t_planned);
    tr.push_back(s.t_realized);
    Millijoules a = 0, b = 0;
    for (auto v : s.planned_e) a += v;
    for (auto v : s.realized_e) b += v;
    spe.push_back(a);
    sre.push_back(b);
    char buf[32];
    std::snprintf(buf, sizeof buf, "\"%016" PRIx64 "\"", schedule_hash(s));
    hashes.push_back(buf);
  }
  o += ",\"t_planned\":";
  put_list(o, tp);
  o += ",\"t_realized\":";
  put_list(o, tr);
  o += ",\"sum_planned_e\":";
  put_list(o, spe);
  o += ",\"sum_realized_e\":";
  put_list(o, sre);
  o += ",\"hash\":[";
  for (size_t k = 0; k < hashes.size(); ++k) {
    if (k) o += ',';
    o += hashes[k];
  }
  o += "],\"step_size\":";
  put_list(o, step_sizes);
  o += ",\"cut_cost\":[";
  for (size_t k = 0; k < infos.size(); ++k) {
    if (k) o += ',';
    o += std::to_string(infos[k].cut_cost);
  }
  o += "],\"sped\":[";
  for (size_t k = 0; k < infos.size(); ++k) {
    if (k) o += ',';
    put_list(o, infos[k].sped_up);
  }
  o += "],\"slowed\":[";
  for (size_t k = 0; k < infos.size(); ++k) {
    if (k) o += ',';
    put_list(o, infos[k].slowed_down);
  }
  o += "]";
  if (full) {
    o += ",\"seed_planned_t\":";
    put_list(o, pts[0].planned_t);
    o += ",\"final_planned_t\":";
    put_list(o, pts.back().planned_t);
    o += ",\"final_freq\":";
    put_list(o, pts.back().freq_mhz);
  }
  o += "}";
  return o;
}

std::string flow_graph_json(const FlowGraph& g) {
  std::string o = "{\"nodes\":" + std::to_string(g.node_count) + ",\"source\":" +
                  std::to_string(g.source) + ",\"sink\":" + std::to_string(g.sink) + ",\"edges\":[";
  for (size_t i = 0; i < g.edges.size(); ++i) {
    const auto& e = g.edges[i];
    if (i) o += ',';
    o += "[" + std::to_string(e.tail) + "," + std::to_string(e.head) + "," + std::to_string(e.lower) +
         "," + std::to_string(e.upper) + "," + (e.infinite ? "1" : "0") + "]";
  }
  o += "]}";
  return o;
}

int mode_flow(int argc, char** argv) {
  const std::uint32_t seed = static_cast<std::uint32_t>(std::stoul(argv[2]));
  const int count = std::stoi(argv[3]);
  const int max_nodes = std::stoi(argv[4]);
  const std::int64_t max_cap = std::stoll(argv[5]);
  std::mt19937 rng(seed);
  for (int i = 0; i < count; ++i) {
    const FlowGraph g = testutil::random_flow_graph(rng, max_nodes, max_cap);
    std::string o = "{\"graph\":" + flow_graph_json(g);
    std::string status;
    try {
      const auto f = max_flow_lower_bounds(g);
      if (!f) {
        o += ",\"feasible\":false";
      } else {
        const CutResult c = min_cut_from_flow(g, *f);
        o += ",\"feasible\":true,\"value\":" + std::to_string(f->value) + ",\"sentinel\":" +
             std::to_string(g.infinity_sentinel()) + ",\"cost\":" + std::to_string(c.cost) +
             ",\"source_side\":";
        std::vector<int> ss(c.source_side.begin(), c.source_side.end());
        put_list(o, ss);
        o += ",\"speed_up\":";
        put_list(o, c.speed_up);
        o += ",\"slow_down\":";
        put_list(o, c.slow_down);
      }
    } catch (const std::exception& ex) {
      o += ",\"error\":\"" + std::string(ex.what()) + "\"";
    }
    o += "}";
    std::printf("%s\n", o.c_str());
  }
  (void)argc;
  return 0;
}

// Same generator as test_dag.cpp:27-45 (restated: it lives in an anonymous
// namespace of the Catch2 test file, which cannot be built here).
NodeDag random_custom_dag(std::mt19937& rng, int max_comps = 9) {
  const int n = std::uniform_int_distribution<int>(2, max_comps)(rng);
  std::vector<Computation> comps;
  for (int i = 0; i < n; ++i) comps.push_back(Computation{i, i % 3, std::nullopt, Kind::Constant});
  std::vector<std::pair<int, int>> edges;
  std::uniform_real_distribution<double> coin(0, 1);
  for (int u = 0; u < n; ++u)
    for (int v = u + 1; v < n; ++v)
      if (coin(rng) < 0.35) edges.emplace_back(u, v);
  return finalize_custom_dag(std::move(comps), std::move(edges));
}

int mode_slack(int argc, char** argv) {
  const std::uint32_t seed = static_cast<std::uint32_t>(std::stoul(argv[2]));
  const int count = std::stoi(argv[3]);
  std::mt19937 rng(seed);
  for (int trial = 0; trial < count; ++trial) {
    NodeDag dag = trial % 4 == 0 ? build_1f1b(1 + trial % 4, 1 + trial % 5) : random_custom_dag(rng, 24);
    std::uniform_int_distribution<Quanta> d(0, 9);
    Durations dur(dag.computations.size());
    for (auto& v : dur) v = d(rng);
    const EdgeDag e = to_edge_centric(dag);
    const SlackAnnotation ann = annotate_slack(e, dur);
    std::string o = "{\"n\":" + std::to_string(dag.computations.size()) + ",\"edges\":[";
    for (size_t i = 0; i < dag.edges.size(); ++i) {
      if (i) o += ',';
      o += "[" + std::to_string(dag.edges[i].first) + "," + std::to_string(dag.edges[i].second) + "]";
    }
    o += "],\"durations\":";
    put_list(o, dur);
    o += ",\"makespan\":" + std::to_string(ann.makespan) + ",\"earliest\":";
    put_list(o, ann.earliest);
    o += ",\"latest\":";
    put_list(o, ann.latest);
    std::vector<int> crit(ann.critical.begin(), ann.critical.end());
    o += ",\"critical\":";
    put_list(o, crit);
    o += "}";
    std::printf("%s\n", o.c_str());
  }
  (void)argc;
  return 0;
}

int mode_bench(int argc, char** argv) {
  const int threads = std::max(1, std::stoi(argv[2]));
  std::vector<std::string> specs;
  for (int i = 3; i < argc; ++i) specs.push_back(argv[i]);
  std::vector<Instance> insts;
  for (const auto& s : specs) insts.push_back(make_instance(s));
  std::atomic<size_t> next{0};
  std::atomic<long long> points{0}, steps{0};
  std::vector<double> inst_s(insts.size(), 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (;;) {
        const size_t i = next.fetch_add(1);
        if (i >= insts.size()) return;
        const auto w0 = std::chrono::steady_clock::now();
        const Frontier f = discover_frontier(insts[i].dag, insts[i].model, insts[i].tau);
        inst_s[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
        points += static_cast<long long>(f.schedules.size());
        steps += f.steps;
      }
    });
  for (auto& th : pool) th.join();
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::string per;
  for (size_t i = 0; i < inst_s.size(); ++i) per += (i ? "," : "") + dbl(inst_s[i]);
  std::printf("{\"instances\":%zu,\"threads\":%d,\"points\":%lld,\"steps\":%lld,\"wall_s\":%.6f,"
              "\"instance_s\":[%s]}\n",
              insts.size(), threads, points.load(), steps.load(), wall, per.c_str());
  return 0;
}

// Time-bounded walks: every instance walks from its seed with the
// reference's public API (the discover_frontier loop, frontier.hpp:166-189)
// until it reaches T_min or its per-instance budget expires; instances run
// one per thread.  Frontier points = schedules produced (seed included).
// straggler_savings over a P-pipeline cluster for comma-separated factors.
int mode_savings(int argc, char** argv) {
  ClusterScenario sc;
  sc.pipelines = std::stoi(argv[2]);
  std::vector<double> factors;
  for (const auto& f : split(argv[3], ',')) factors.push_back(std::stod(f));
  for (int i = 4; i < argc; ++i) {
    const Instance in = make_instance(argv[i]);
    const Frontier fr = discover_frontier(in.dag, in.model, in.tau);
    const auto rows = straggler_savings(fr, in.dag, in.model, sc, factors);
    const AllMaxAssignment am = all_max_assignment(in.dag, in.model);
    const Quanta tmin = simulate(in.dag, am.durations).iteration_time;
    std::ostringstream o;
    o << "{\"spec\":\"" << argv[i] << "\",\"pipelines\":" << sc.pipelines << ",\"num_stages\":" << in.dag.num_stages
      << ",\"rows\":[";
    for (size_t k = 0; k < rows.size(); ++k) {
      const Quanta tp = std::llround(factors[k] * static_cast<double>(tmin));
      const EnergySchedule& s = lookup(fr, tp);
      char buf[256];
      std::snprintf(buf, sizeof buf, "%s{\"factor\":%.17g,\"savings_pct\":%.17g,\"savings_mj\":%.17g,\"point\":%d}",
                    k ? "," : "", rows[k].factor, rows[k].savings_pct, rows[k].savings_mj, s.schedule_id);
      o << buf;
    }
    o << "]}";
    std::printf("%s\n", o.str().c_str());
  }
  return 0;
}

int mode_artifacts(int argc, char** argv) {
  const std::int64_t q = std::stoll(argv[2]);
  for (int i = 3; i < argc; ++i) {
    const Instance in = make_instance(argv[i]);
    const Frontier fr = discover_frontier(in.dag, in.model, in.tau);
    nlohmann::ordered_json j;
    j["spec"] = argv[i];
    j["quantum"] = q;
    j["csv"] = frontier_csv(fr, q);
    const int last = static_cast<int>(fr.schedules.size()) - 1;
    nlohmann::ordered_json sj = nlohmann::ordered_json::object();
    for (int k : {0, last / 2, last}) sj[std::to_string(k)] = schedule_json(fr.schedules[k], q).dump(2) + "\n";
    j["schedules"] = sj;
    std::printf("%s\n", j.dump().c_str());
  }
  return 0;
}

int mode_brute(int argc, char** argv) {
  for (int i = 2; i < argc; ++i) {
    const Instance in = make_instance(argv[i]);
    nlohmann::ordered_json j;
    j["spec"] = argv[i];
    try {
      const ExactFrontier ex = brute_force_frontier(in.dag, in.model);
      nlohmann::ordered_json pts = nlohmann::ordered_json::array();
      for (const auto& p : ex.points) {
        std::uint64_t bitsv;
        std::memcpy(&bitsv, &p.eff_energy_mj, 8);
        pts.push_back({{"time", p.time}, {"eff_bits", std::to_string(bitsv)}, {"freq_mhz", p.freq_mhz}});
      }
      j["points"] = pts;
    } catch (const BudgetExceeded&) {
      j["budget_exceeded"] = true;
    }
    std::printf("%s\n", j.dump().c_str());
  }
  return 0;
}

// budget <seconds> <threads> <spec>...: each instance walked for at most
// that many seconds; capped <steps> <threads> <spec>...: for at most that
// many steps (a deterministic sample: the GPU arm walks the identical
// capped sample with pb_instance_desc.max_steps).
int mode_budget(int argc, char** argv, bool by_steps) {
  const double budget = by_steps ? 1e300 : std::stod(argv[2]);
  const long long max_steps = by_steps ? std::stoll(argv[2]) : -1;
  const int threads = std::max(1, std::stoi(argv[3]));
  std::vector<std::string> specs;
  for (int i = 4; i < argc; ++i) specs.push_back(argv[i]);
  std::vector<Instance> insts;
  for (const auto& s : specs) insts.push_back(make_instance(s));
  std::atomic<size_t> next{0};
  std::atomic<long long> points{0}, steps{0}, complete{0};
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (;;) {
        const size_t i = next.fetch_add(1);
        if (i >= insts.size()) return;
        const Instance& in = insts[i];
        const auto s0 = std::chrono::steady_clock::now();
        const AllMaxAssignment am = all_max_assignment(in.dag, in.model);
        const Quanta t_min = simulate(in.dag, am.durations).iteration_time;
        EnergySchedule cur = min_energy_schedule(in.dag, in.model);
        EnergySchedule first = discretize(cur, in.dag, in.model);
        long long p = 1, k = 0;
        bool done = true;
        while (cur.t_planned > t_min) {
          if ((max_steps >= 0 && k >= max_steps) ||
              std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count() > budget) {
            done = false;
            break;
          }
          const Quanta step = std::min<Quanta>(in.tau, cur.t_planned - t_min);
          auto nxt = get_next_schedule(in.dag, cur, in.model, step);
          if (!nxt || nxt->t_planned >= cur.t_planned) break;
          cur = std::move(*nxt);
          EnergySchedule d = discretize(cur, in.dag, in.model);
          ++p;
          ++k;
        }
        points += p;
        steps += k;
        if (done) ++complete;
      }
    });
  for (auto& th : pool) th.join();
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"instances\":%zu,\"threads\":%d,\"budget_s\":%.3f,\"max_steps\":%lld,\"points\":%lld,"
              "\"steps\":%lld,\"complete\":%lld,\"wall_s\":%.6f}\n",
              insts.size(), threads, by_steps ? 0.0 : budget, max_steps, points.load(), steps.load(),
              complete.load(), wall);
  (void)argc;
  return 0;
}

// get_next_schedule (frontier.hpp:90-135) from a caller schedule: planned
// times given (comma-separated, any value -- also outside a class's curve
// interval), planned energies from detail::planned_energy.
int mode_getnext(int argc, char** argv) {
  const Quanta tau = std::stoll(argv[2]);
  for (int i = 3; i + 1 < argc; i += 2) {
    const Instance in = make_instance(argv[i]);
    EnergySchedule s;
    for (const auto& tok : split(argv[i + 1], ',')) s.planned_t.push_back(std::stoll(tok));
    for (size_t c = 0; c < s.planned_t.size(); ++c)
      s.planned_e.push_back(
          detail::planned_energy(in.model.require(class_of(in.dag.computations[c])), s.planned_t[c]));
    detail::refresh_totals(in.dag, in.model, s);
    std::string o = "{\"spec\":\"" + std::string(argv[i]) + "\",\"tau\":" + std::to_string(tau) +
                    ",\"start\":";
    put_list(o, s.planned_t);
    o += ",\"start_e\":";
    put_list(o, s.planned_e);
    StepInfo info;
    const auto nx = get_next_schedule(in.dag, s, in.model, tau, &info);
    if (!nx) {
      o += ",\"next\":null}";
    } else {
      o += ",\"cut_cost\":" + std::to_string(info.cut_cost) + ",\"sped\":";
      put_list(o, info.sped_up);
      o += ",\"slowed\":";
      put_list(o, info.slowed_down);
      o += ",\"planned_t\":";
      put_list(o, nx->planned_t);
      o += ",\"planned_e\":";
      put_list(o, nx->planned_e);
      o += ",\"t_planned\":" + std::to_string(nx->t_planned) + ",\"eff_planned\":" + dbl(nx->eff_planned_mj) + "}";
    }
    std::printf("%s\n", o.c_str());
  }
  (void)argc;
  return 0;
}

// Rule-5 search (SURVEY.md §7 parity rule 5): walks r5:<seed> instances and
// reports the specs whose walk speeds up a computation through an infinite
// edge inside a cut of value < sentinel (a constant class, or a planned time
// pushed below the curve's t_min: frontier.hpp:111-116 has no bound check).
int mode_rule5(int argc, char** argv) {
  const std::uint32_t first = static_cast<std::uint32_t>(std::stoul(argv[2]));
  const int count = std::stoi(argv[3]);
  const std::string maxn = argc > 4 ? argv[4] : "8";
  for (int q = 0; q < count; ++q) {
    const std::string spec = "r5:" + std::to_string(first + q) + ":" + maxn;
    const Instance in = make_instance(spec);
    const AllMaxAssignment am = all_max_assignment(in.dag, in.model);
    const Quanta t_min = simulate(in.dag, am.durations).iteration_time;
    EnergySchedule cur = min_energy_schedule(in.dag, in.model);
    int steps = 0, events = 0, below = 0, first_step = -1;
    while (cur.t_planned > t_min && steps < 2000) {
      const Quanta step = std::min<Quanta>(in.tau, cur.t_planned - t_min);
      StepInfo info;
      auto next = get_next_schedule(in.dag, cur, in.model, step, &info);
      if (!next || next->t_planned >= cur.t_planned) break;
      for (int c : info.sped_up) {
        const auto& cm = in.model.require(class_of(in.dag.computations[c]));
        const bool ev = cm.is_constant || next->planned_t[c] < cm.curve->t_min;
        if (ev) {
          ++events;
          if (!cm.is_constant && next->planned_t[c] < cm.curve->t_min - in.tau) ++below;
          if (first_step < 0) first_step = steps;
        }
      }
      cur = std::move(*next);
      ++steps;
    }
    if (events)
      std::printf("{\"spec\":\"%s\",\"steps\":%d,\"events\":%d,\"below_tau\":%d,\"first\":%d}\n",
                  spec.c_str(), steps, events, below, first_step);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver walk|walkfull|flow|slack|bench|fit ...\n");
    return 2;
  }
  const std::string mode = argv[1];
  try {
    if (mode == "walk" || mode == "walkfull" || mode == "walkcheck") {
      for (int i = 2; i < argc; ++i) {
        const Instance in = make_instance(argv[i]);
        std::printf("%s\n", walk_json(in, mode == "walkfull", mode == "walkcheck").c_str());
        std::fflush(stdout);
      }
      return 0;
    }
    if (mode == "walkprefix") {  // walkprefix <max_steps> <spec>...: the first K steps only
      const long long k = std::stoll(argv[2]);
      for (int i = 3; i < argc; ++i) {
        const Instance in = make_instance(argv[i]);
        std::printf("%s\n", walk_json(in, false, false, k).c_str());
        std::fflush(stdout);
      }
      return 0;
    }
    if (mode == "rule5") return mode_rule5(argc, argv);
    if (mode == "getnext") return mode_getnext(argc, argv);
    if (mode == "flow") return mode_flow(argc, argv);
    if (mode == "slack") return mode_slack(argc, argv);
    if (mode == "bench") return mode_bench(argc, argv);
    if (mode == "budget") return mode_budget(argc, argv, false);
    if (mode == "capped") return mode_budget(argc, argv, true);
    if (mode == "savings") return mode_savings(argc, argv);
    if (mode == "artifacts") return mode_artifacts(argc, argv);
    if (mode == "brute") return mode_brute(argc, argv);
    if (mode == "fit") {
      for (int i = 2; i < argc; ++i) {
        const Instance in = make_instance(argv[i]);
        std::printf("{\"spec\":\"%s\",\"curves\":%s}\n", argv[i], curves_json(in.model).c_str());
      }
      return 0;
    }
  } catch (const std::exception& ex) {
    std::fprintf(stderr, "error: %s\n", ex.what());
    return 3;
  }
  std::fprintf(stderr, "unknown mode %s\n", mode.c_str());
  return 2;
}
