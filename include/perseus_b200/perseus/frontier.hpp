// perseus/frontier.hpp -- B200 drop-in for the reference planner's frontier
// API (/root/reference/proj/include/perseus/frontier.hpp:16-220).
//
// Put include/perseus_b200 BEFORE the reference include directory on the
// include path; every other perseus/*.hpp header (dag, costmodel, emulator,
// flow, units, ...) stays the reference's own.  The types and signatures are
// the reference's; the frontier walk (discover_frontier, get_next_schedule)
// runs on the GPU through the C ABI of include/perseus_b200.h, and the
// result is expanded into the same EnergySchedule / Frontier values.
// Link with paper_2312_06902_b200/_lib/libperseus_b200.so.
//
// Device: env PERSEUS_B200_DEVICE (default 0).  Errors raise the reference's
// exception classes (invalid_argument, overflow_error, logic_error,
// DegenerateFit-compatible domain_error); device failures raise
// std::runtime_error.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "perseus/costmodel.hpp"
#include "perseus/dag.hpp"
#include "perseus/emulator.hpp"
#include "perseus/flow.hpp"
#include "perseus/units.hpp"
#include "../../perseus_b200.h"

namespace perseus {

// frontier.hpp:20-33
struct EnergySchedule {
  int schedule_id = 0;
  Durations planned_t;
  std::vector<Millijoules> planned_e;
  std::vector<int> freq_mhz;  // empty before discretization
  Durations realized_t;
  std::vector<Millijoules> realized_e;
  Quanta t_planned = 0;
  Quanta t_realized = 0;
  double eff_planned_mj = 0;
  double eff_realized_mj = 0;

  bool discretized() const { return !freq_mhz.empty(); }
};

// frontier.hpp:35-40
struct Frontier {
  std::vector<EnergySchedule> schedules;  // strictly decreasing planned T, T* first
  Quanta t_min = 0;
  Quanta t_star = 0;
  int steps = 0;
};

// frontier.hpp:43-47
struct StepInfo {
  Millijoules cut_cost = 0;
  std::vector<int> sped_up;
  std::vector<int> slowed_down;
};

namespace detail {

// Sum of effective energies in index order (frontier.hpp:51-57).
inline double effective_total(const std::vector<Millijoules>& energies, const Durations& times,
                              BlockingPower blocking, std::int64_t quantum_us) {
  double acc = 0;
  const size_t n = energies.size();
  for (size_t i = 0; i < n; ++i) acc += effective_energy_mj(energies[i], times[i], blocking, quantum_us);
  return acc;
}

// Curve-relaxed energy at t; constant classes use their single point (frontier.hpp:59-62).
inline Millijoules planned_energy(const CostModel::ClassModel& cm, Quanta t) {
  return cm.is_constant ? cm.pareto.front().energy
                        : static_cast<Millijoules>(std::llround(cm.curve->eval(static_cast<double>(t))));
}

// Longest source->sink path of the node DAG (the iteration time of
// simulate(), emulator.hpp:28-55).
inline Quanta longest_path(const NodeDag& dag, const Durations& d) {
  const int n = static_cast<int>(dag.computations.size());
  if (static_cast<int>(d.size()) < n) throw std::invalid_argument("durations must cover every computation");
  for (int i = 0; i < n; ++i)
    if (d[i] < 0) throw std::invalid_argument("durations must be non-negative");
  const auto order = topo_order(dag.node_count(), dag.edges);
  std::vector<std::vector<int>> out(dag.node_count());
  for (const auto& e : dag.edges) out[e.first].push_back(e.second);
  std::vector<Quanta> start(dag.node_count(), 0);
  for (int u : order) {
    const Quanta fin = start[u] + (u < n ? d[u] : 0);
    for (int v : out[u]) start[v] = std::max(start[v], fin);
  }
  return start[dag.sink_id()];
}

inline void refresh_totals(const NodeDag& dag, const CostModel& model, EnergySchedule& s) {
  s.t_planned = longest_path(dag, s.planned_t);
  s.eff_planned_mj = effective_total(s.planned_e, s.planned_t, model.blocking, model.quantum_us);
}

// ---- B200 binding ---------------------------------------------------------

inline int b200_device() {
  const char* e = std::getenv("PERSEUS_B200_DEVICE");
  return e ? std::atoi(e) : 0;
}

[[noreturn]] inline void b200_raise(pb_status s) {
  const std::string msg = pb_last_error();
  switch (s) {
    case PB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PB_ERR_OVERFLOW: throw std::overflow_error(msg);
    case PB_ERR_LOGIC: throw std::logic_error(msg);
    case PB_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error("perseus-b200: " + msg);
  }
}

inline void b200_check(pb_status s) {
  if (s != PB_OK) b200_raise(s);
}

// Flat view of (NodeDag, CostModel) for pb_batch_add; classes are numbered in
// the CostModel's map order.
struct B200Instance {
  std::vector<int32_t> comp_class, tail, head, point_off, freq;
  std::vector<uint8_t> is_const;
  std::vector<int64_t> time, energy, trange;
  std::vector<double> curve;
  pb_instance_desc desc{};

  B200Instance(const NodeDag& dag, const CostModel& model, Quanta tau) {
    std::map<ClassKey, int32_t> index;
    point_off.push_back(0);
    for (const auto& kv : model.classes) {
      const auto& cm = kv.second;
      index.emplace(kv.first, static_cast<int32_t>(is_const.size()));
      is_const.push_back(cm.is_constant ? 1 : 0);
      for (const auto& p : cm.pareto) {
        freq.push_back(p.freq_mhz);
        time.push_back(p.time);
        energy.push_back(p.energy);
      }
      point_off.push_back(static_cast<int32_t>(time.size()));
      const bool has = !cm.is_constant && cm.curve.has_value();
      curve.push_back(has ? cm.curve->a : 0.0);
      curve.push_back(has ? cm.curve->b : 0.0);
      curve.push_back(has ? cm.curve->c : 0.0);
      trange.push_back(has ? cm.curve->t_min : 0);
      trange.push_back(has ? cm.curve->t_max : 0);
    }
    for (const auto& c : dag.computations) {
      auto it = index.find(class_of(c));
      if (it == index.end()) throw std::invalid_argument("missing profile for a computation class");
      comp_class.push_back(it->second);
    }
    for (const auto& e : dag.edges) {
      tail.push_back(e.first);
      head.push_back(e.second);
    }
    desc.n = static_cast<int32_t>(dag.computations.size());
    desc.comp_class = comp_class.data();
    desc.n_edges = static_cast<int32_t>(tail.size());
    desc.edge_tail = tail.data();
    desc.edge_head = head.data();
    desc.n_classes = static_cast<int32_t>(is_const.size());
    desc.class_is_constant = is_const.data();
    desc.class_point_off = point_off.data();
    desc.point_freq = freq.data();
    desc.point_time = time.data();
    desc.point_energy = energy.data();
    desc.class_curve = curve.data();
    desc.class_t_range = trange.data();
    desc.blocking_watts = model.blocking.watts;
    desc.quantum_us = model.quantum_us;
    desc.tau = tau;
  }
};

// RAII pb_batch handle (single-thread, like the reference's per-job rule).
struct B200Batch {
  pb_batch* h = nullptr;
  B200Batch() { b200_check(pb_batch_create(&h)); }
  ~B200Batch() { pb_batch_destroy(h); }
  B200Batch(const B200Batch&) = delete;
  B200Batch& operator=(const B200Batch&) = delete;
};

// The calling thread's persistent handle, emptied for each call: its device
// context (stream, device and pinned buffers) is reused across calls, so a
// loop of get_next_schedule calls packs and uploads one instance per call
// and allocates nothing.  Distinct threads get distinct handles (and
// streams), as the reference lets distinct jobs run concurrently.
inline pb_batch* b200_handle() {
  thread_local B200Batch b;
  b200_check(pb_batch_clear(b.h));
  return b.h;
}

// Walks instance `inst` (start schedule / step cap as set in its desc) on
// the calling thread's handle; returns the summary, raising the reference's
// exception for an error status.
inline pb_frontier_summary b200_walk(pb_batch* h, B200Instance& inst) {
  b200_check(pb_batch_add(h, &inst.desc, nullptr));
  b200_check(pb_batch_run(h, b200_device()));
  pb_frontier_summary sum;
  b200_check(pb_batch_summary(h, 0, &sum));
  if (sum.status != PB_OK) b200_raise(static_cast<pb_status>(sum.status));
  return sum;
}

// Schedules [first, first + count) of a walked instance, materialized from
// the delta log in one incremental replay (pb_batch_schedules) and appended
// to out; iteration times are the device's (pb_point).
inline void b200_schedules(const pb_batch* b, int32_t first, int32_t count, int32_t n, const pb_point* pts,
                           std::vector<EnergySchedule>& out) {
  const size_t cells = static_cast<size_t>(count) * static_cast<size_t>(n);
  std::vector<int64_t> pt(cells), pe(cells), rt(cells), re(cells);
  std::vector<int32_t> fr(cells);
  std::vector<double> ep(count), er(count);
  b200_check(pb_batch_schedules(b, 0, first, count, pt.data(), pe.data(), fr.data(), rt.data(), re.data(),
                                ep.data(), er.data()));
  for (int32_t q = 0; q < count; ++q) {
    const size_t o = static_cast<size_t>(q) * static_cast<size_t>(n);
    EnergySchedule s;
    s.schedule_id = first + q;
    s.planned_t.assign(pt.begin() + o, pt.begin() + o + n);
    s.planned_e.assign(pe.begin() + o, pe.begin() + o + n);
    s.freq_mhz.assign(fr.begin() + o, fr.begin() + o + n);
    s.realized_t.assign(rt.begin() + o, rt.begin() + o + n);
    s.realized_e.assign(re.begin() + o, re.begin() + o + n);
    s.t_planned = pts[first + q].t_planned;
    s.t_realized = pts[first + q].t_realized;
    s.eff_planned_mj = ep[q];
    s.eff_realized_mj = er[q];
    out.push_back(std::move(s));
  }
}

}  // namespace detail

// Minimum-energy seed (frontier.hpp:73-83): point 0 of a zero-step walk on
// the GPU (planned times at each class's t_max, energies from the curve
// tables, the device's longest path as T*).
inline EnergySchedule min_energy_schedule(const NodeDag& dag, const CostModel& model) {
  EnergySchedule s;
  const int32_t n = static_cast<int32_t>(dag.computations.size());
  if (n == 0) {
    detail::refresh_totals(dag, model, s);
    return s;
  }
  detail::B200Instance inst(dag, model, kDefaultTauUs);
  inst.desc.max_steps = -1;  // no step: the seed only
  pb_batch* h = detail::b200_handle();
  (void)detail::b200_walk(h, inst);
  pb_point p0;
  detail::b200_check(pb_batch_points(h, 0, &p0, 1));
  s.planned_t.resize(n);
  s.planned_e.resize(n);
  detail::b200_check(pb_batch_schedule(h, 0, 0, s.planned_t.data(), s.planned_e.data(), nullptr, nullptr,
                                       nullptr, &s.eff_planned_mj, nullptr));
  s.t_planned = p0.t_planned;
  return s;
}

// One frontier step (frontier.hpp:90-135), run on the GPU as a single-step
// walk from schedule.planned_t.  nullopt when the bounded network is
// infeasible or the minimum cut is infinite.
inline std::optional<EnergySchedule> get_next_schedule(const NodeDag& dag, const EnergySchedule& schedule,
                                                       const CostModel& model, Quanta tau,
                                                       StepInfo* info = nullptr) {
  if (tau <= 0) throw std::invalid_argument("tau must be positive");
  const int32_t n = static_cast<int32_t>(dag.computations.size());
  if (static_cast<int32_t>(schedule.planned_t.size()) != n)
    throw std::invalid_argument("durations must cover every computation");
  EnergySchedule next = schedule;
  next.freq_mhz.clear();
  next.realized_t.clear();
  next.realized_e.clear();
  StepInfo st;
  if (n == 0) {
    // an empty DAG has no edge to cut: the reference's max flow is 0 < sentinel 1
    st.cut_cost = 0;
    detail::refresh_totals(dag, model, next);
    if (info) *info = std::move(st);
    return next;
  }
  detail::B200Instance inst(dag, model, tau);
  inst.desc.start_planned_t = schedule.planned_t.data();
  inst.desc.max_steps = 1;
  pb_batch* h = detail::b200_handle();
  const pb_frontier_summary sum = detail::b200_walk(h, inst);
  if (sum.stop == PB_STOP_INFEASIBLE || sum.stop == PB_STOP_INFINITE_CUT) return std::nullopt;
  if (sum.steps != 1) throw std::logic_error("perseus-b200: single step did not run");
  pb_point pts[2];
  detail::b200_check(pb_batch_points(h, 0, pts, 2));
  std::vector<int32_t> ids(std::max(sum.n_ids, 1));
  detail::b200_check(pb_batch_deltas(h, 0, ids.data(), nullptr, static_cast<int32_t>(ids.size())));
  // the device's step: new planned times and energies of the touched
  // computations (curve tables), the new planned makespan
  std::vector<int64_t> dev_t(n), dev_e(n);
  detail::b200_check(pb_batch_schedule(h, 0, 1, dev_t.data(), dev_e.data(), nullptr, nullptr, nullptr, nullptr,
                                       nullptr));
  st.cut_cost = pts[1].cut_cost;
  for (int32_t j = 0; j < sum.n_ids; ++j) {
    const int comp = (ids[j] > 0 ? ids[j] : -ids[j]) - 1;
    (ids[j] > 0 ? st.sped_up : st.slowed_down).push_back(comp);
    next.planned_t[comp] = dev_t[comp];
    next.planned_e[comp] = dev_e[comp];
  }
  next.t_planned = pts[1].t_planned;
  // refresh_totals (frontier.hpp:64-67): untouched computations keep the
  // caller's planned_e, so the index-order sum runs over the merged vector
  next.eff_planned_mj = detail::effective_total(next.planned_e, next.planned_t, model.blocking, model.quantum_us);
  if (info) *info = std::move(st);
  return next;
}

// Snap to profiled frequencies (frontier.hpp:140-161): the last Pareto point
// (ascending time) whose time fits the planned duration, else the fastest.
// Runs on the GPU as a zero-step walk from schedule.planned_t: the device's
// choice per computation, realized durations and realized makespan.
inline EnergySchedule discretize(const EnergySchedule& schedule, const NodeDag& dag, const CostModel& model) {
  EnergySchedule out = schedule;
  out.freq_mhz.clear();
  out.realized_t.clear();
  out.realized_e.clear();
  const int32_t n = static_cast<int32_t>(dag.computations.size());
  if (n == 0) {
    out.t_realized = detail::longest_path(dag, out.realized_t);
    out.eff_realized_mj = 0;
    return out;
  }
  if (static_cast<int32_t>(schedule.planned_t.size()) < n)
    throw std::invalid_argument("durations must cover every computation");
  detail::B200Instance inst(dag, model, kDefaultTauUs);
  inst.desc.start_planned_t = schedule.planned_t.data();
  inst.desc.max_steps = -1;  // no step: discretize the start schedule only
  pb_batch* h = detail::b200_handle();
  (void)detail::b200_walk(h, inst);
  pb_point p0;
  detail::b200_check(pb_batch_points(h, 0, &p0, 1));
  out.freq_mhz.resize(n);
  out.realized_t.resize(n);
  out.realized_e.resize(n);
  detail::b200_check(pb_batch_schedule(h, 0, 0, nullptr, nullptr, out.freq_mhz.data(), out.realized_t.data(),
                                       out.realized_e.data(), nullptr, &out.eff_realized_mj));
  out.t_realized = p0.t_realized;
  return out;
}

// The whole frontier from T* down to T_min (frontier.hpp:166-189): one walk
// on the GPU, every point expanded from the delta log and discretized.
inline Frontier discover_frontier(const NodeDag& dag, const CostModel& model, Quanta tau = kDefaultTauUs) {
  if (tau <= 0) throw std::invalid_argument("tau must be positive");
  Frontier f;
  const int32_t n = static_cast<int32_t>(dag.computations.size());
  if (n == 0) {
    // nothing to walk: T_min = T* and the frontier is the seed alone
    for (const auto& c : dag.computations) (void)model.require(class_of(c));
    EnergySchedule s = min_energy_schedule(dag, model);
    f.t_min = f.t_star = s.t_planned;
    f.schedules.push_back(discretize(s, dag, model));
    return f;
  }
  detail::B200Instance inst(dag, model, tau);
  pb_batch* h = detail::b200_handle();
  const pb_frontier_summary sum = detail::b200_walk(h, inst);
  f.t_min = sum.t_min;
  f.t_star = sum.t_star;
  f.steps = sum.steps;
  std::vector<pb_point> pts(sum.steps + 1);
  detail::b200_check(pb_batch_points(h, 0, pts.data(), sum.steps + 1));
  f.schedules.reserve(sum.steps + 1);
  // expand the delta log in chunks of ~16 MB of schedule data
  const int32_t chunk = static_cast<int32_t>(std::max<int64_t>(1, (int64_t{1} << 24) / (36 * int64_t{n})));
  for (int32_t k = 0; k <= sum.steps; k += chunk)
    detail::b200_schedules(h, k, std::min(chunk, sum.steps + 1 - k), n, pts.data(), f.schedules);
  return f;
}

// All-max reference schedule (frontier.hpp:193-207).
inline EnergySchedule all_max_schedule(const NodeDag& dag, const CostModel& model) {
  const AllMaxAssignment am = all_max_assignment(dag, model);
  EnergySchedule s;
  s.schedule_id = -1;
  s.planned_t = am.durations;
  s.realized_t = am.durations;
  s.planned_e = am.energies;
  s.realized_e = am.energies;
  s.freq_mhz = am.freqs_mhz;
  s.t_planned = detail::longest_path(dag, am.durations);
  s.t_realized = s.t_planned;
  s.eff_planned_mj = detail::effective_total(am.energies, am.durations, model.blocking, model.quantum_us);
  s.eff_realized_mj = s.eff_planned_mj;
  return s;
}

// Frontier point for a straggler iteration time (frontier.hpp:212-220): the
// first schedule (decreasing planned T) with t_planned <= min(T*, T').
inline const EnergySchedule& lookup(const Frontier& frontier, Quanta straggler_time) {
  if (frontier.schedules.empty()) throw std::logic_error("frontier is empty");
  const Quanta target = std::min(frontier.t_star, straggler_time);
  size_t lo = 0, hi = frontier.schedules.size();
  while (lo < hi) {
    const size_t mid = lo + (hi - lo) / 2;
    if (frontier.schedules[mid].t_planned > target)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo == frontier.schedules.size() ? frontier.schedules.back() : frontier.schedules[lo];
}

}  // namespace perseus
