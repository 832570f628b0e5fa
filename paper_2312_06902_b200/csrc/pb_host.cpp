// Host side of the C ABI (include/perseus_b200.h): cost-model fitting,
// instance packing into flat device layouts, curve tables, LPT ordering,
// device memory, launches and result access.  Compiled with g++
// -ffp-contract=off so that pareto/fit/table arithmetic reproduces the
// reference's libm results bit for bit (SURVEY.md §7 hard part 1).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "g9.hpp"
#include "pb_internal.h"
#include "perseus_b200.h"

namespace {

thread_local std::string g_last_error;

pb_status fail(pb_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ----------------------------------------------------------- owned instance

struct HostInst {
  int32_t n = 0;
  std::vector<int32_t> comp_class, edge_tail, edge_head;
  std::vector<uint8_t> cls_const;
  std::vector<int32_t> cls_pt_off, pt_freq;
  std::vector<int64_t> pt_time, pt_energy, cls_trange;
  std::vector<double> cls_curve;
  double watts = 75.0;
  int64_t quantum = 1, tau = 1000;
  std::vector<int64_t> start;  // empty = min-energy seed
  int32_t max_steps = 0;
  // derived by validate_and_derive(): the static device layout (pb_internal.h)
  int32_t n_levels = 0;
  std::vector<int32_t> lvl_off, orig, inv, icls;
  std::vector<uint8_t> cflag;
  std::vector<int32_t> ilev, snk;  // level of each internal id; ids with an edge to the sink (ascending)
  std::vector<int32_t> pin_off, pin, pout_off, pout;
  std::vector<pb::int4h> frow, brow;
  std::vector<pb::int2h> dep_nd;  // network order (sorted by head, tail)
  std::vector<int32_t> dep_orig;  // network dependency index -> caller's edge index
  pb::NetLayout net;
  std::vector<int64_t> istart;  // start schedule in internal order
  int64_t t_min_est = 0, t_star_est = 0, est_steps = 0, work = 0;
  uint64_t gen = 0;  // pb_batch::derived_gen this instance was derived under (pb_batch_add), 0 = other
};

// Longest path on the node DAG with the given durations (internal order;
// host estimate used only to size output buffers and order work; the device
// computes its own).
int64_t host_makespan(const HostInst& h, const std::vector<int64_t>& dur) {
  std::vector<int64_t> fin(h.n, 0);
  int64_t ms = 0;
  for (int32_t i = 0; i < h.n; ++i) {
    int64_t m = 0;
    for (int32_t j = h.pin_off[i]; j < h.pin_off[i + 1]; ++j) m = std::max(m, fin[h.pin[j]]);
    fin[i] = m + dur[i];
    if (h.cflag[i] & 2) ms = std::max(ms, fin[i]);
  }
  return ms;
}

}  // namespace

namespace pb {
// Position-indexed incidence of an edge list (tail[k] -> head[k], k < E):
// per node the list of its arcs; entry p = {other end, twin position,
// other's list range}; epos[k] = {position at tail, position at head}.
void build_net(int32_t V, const std::vector<int32_t>& tail, const std::vector<int32_t>& head,
               NetLayout& out, int32_t pairs) {
  const int32_t E = static_cast<int32_t>(tail.size());
  if (2 * static_cast<int64_t>(E) > kTwinMask) throw std::length_error("flow network too large for 26-bit positions");
  out.inc_off.assign(V + 1, 0);
  for (int32_t k = 0; k < E; ++k) {
    ++out.inc_off[tail[k] + 1];
    ++out.inc_off[head[k] + 1];
  }
  for (int32_t v = 0; v < V; ++v) out.inc_off[v + 1] += out.inc_off[v];
  out.epos.assign(E, int2h{0, 0});
  // edges are placed in index order, so computation edge i (< pairs) is the
  // first entry of both nodes 2i and 2i+1
  std::vector<int32_t> fill(out.inc_off.begin(), out.inc_off.end() - 1);
  for (int32_t k = 0; k < E; ++k) {
    out.epos[k].x = fill[tail[k]]++;
    out.epos[k].y = fill[head[k]]++;
  }
  auto pdeg = [&](int32_t b) {
    if (b >= 2 * pairs) return kNoPartner;
    const int32_t d = out.inc_off[(b ^ 1) + 1] - out.inc_off[b ^ 1];
    return d < kNoPartner ? d : kNoPartner;
  };
  out.ient.assign(out.inc_off[V], IEnt{0, 0, 0, 0});
  for (int32_t k = 0; k < E; ++k) {
    const int32_t a = tail[k], b = head[k], pa = out.epos[k].x, pb = out.epos[k].y;
    const int32_t flag = k < pairs ? kCompArc : 0;
    out.ient[pa] = IEnt{b, pb | flag | (pdeg(b) << kPdegShift), out.inc_off[b], out.inc_off[b + 1]};
    out.ient[pb] = IEnt{a, pa | flag | (pdeg(a) << kPdegShift), out.inc_off[a], out.inc_off[a + 1]};
  }
}
}  // namespace pb

namespace {

// Validation mirrors the reference's throws; derived arrays are the static
// device layout (level-major computations, row records, incidence).
pb_status derive_start(HostInst& h);

// Estimated device time of a walk (ns), for the LPT order, the cooperative
// head and the device split only (never for results).  A step's cost is
// latency-bound and grows with the DAG's width (BFS levels and the sweep's
// levels carry ~width arcs / computations, several rounds each) and its size
// (the capacity pass scans every edge): per step ~ 79 ns x width + 0.0223 ns
// x E - 226 ns (us units in the fit; least squares over the 4096 config-5
// walks on one B200, Spearman 0.976 vs 0.958 for E x steps).  PB_WORK_MODEL=0
// restores E x steps.
int64_t walk_work(const HostInst& h) {
  const int64_t E = h.n + static_cast<int64_t>(h.edge_tail.size()) + 1;
  static const bool edges_only = [] {
    const char* e = std::getenv("PB_WORK_MODEL");
    return e && std::atoi(e) == 0;
  }();
  if (edges_only) return E * h.est_steps;
  const double width = static_cast<double>(h.n) / std::max(1, h.n_levels);
  const double per_step = std::max(10.0, 79.0 * width + 0.0223 * static_cast<double>(E) - 226.0);
  return static_cast<int64_t>(per_step * 1000.0) * h.est_steps;
}

pb_status validate_and_derive(HostInst& h) {
  const int32_t n = h.n, ne = static_cast<int32_t>(h.edge_tail.size());
  const int32_t nc = static_cast<int32_t>(h.cls_const.size());
  if (n < 1) return fail(PB_ERR_INVALID_ARGUMENT, "dag needs at least one computation");
  if (h.tau <= 0) return fail(PB_ERR_INVALID_ARGUMENT, "tau must be positive");
  if (h.quantum <= 0) return fail(PB_ERR_INVALID_ARGUMENT, "quantum must be positive");
  if (n > (1 << 28)) return fail(PB_ERR_UNSUPPORTED, "too many computations");
  for (int32_t c = 0; c < nc; ++c) {
    const int32_t np = h.cls_pt_off[c + 1] - h.cls_pt_off[c];
    if (np < 1) return fail(PB_ERR_INVALID_ARGUMENT, "profile has no points");
    if (np > 255) return fail(PB_ERR_INVALID_ARGUMENT, "more than 255 Pareto points in a class");
    for (int32_t p = h.cls_pt_off[c]; p < h.cls_pt_off[c + 1]; ++p)
      if (h.pt_time[p] < 0) return fail(PB_ERR_INVALID_ARGUMENT, "durations must be non-negative");
    if (!h.cls_const[c] && h.cls_trange[2 * c] > h.cls_trange[2 * c + 1])
      return fail(PB_ERR_INVALID_ARGUMENT, "curve interval is empty");
  }
  for (int32_t i = 0; i < n; ++i)
    if (h.comp_class[i] < 0 || h.comp_class[i] >= nc)
      return fail(PB_ERR_INVALID_ARGUMENT, "missing profile for a computation class");
  for (int32_t j = 0; j < ne; ++j) {
    const int32_t u = h.edge_tail[j], v = h.edge_head[j];
    if (u < 0 || u > n + 1 || v < 0 || v > n + 1 || u == n + 1 || v == n || u == v)
      return fail(PB_ERR_INVALID_ARGUMENT, "edge references unknown computation");
  }
  if (!h.start.empty()) {
    if (static_cast<int32_t>(h.start.size()) != n)
      return fail(PB_ERR_INVALID_ARGUMENT, "durations must cover every computation");
    for (int64_t t : h.start)
      if (t < 0) return fail(PB_ERR_INVALID_ARGUMENT, "durations must be non-negative");
  }
  // Kahn over the full node set (dag.hpp:64-86) for cycle detection, levels
  // over computations = longest hop distance from any root.
  std::vector<int32_t> indeg(n + 2, 0);
  std::vector<std::vector<int32_t>> succ(n + 2);
  for (int32_t j = 0; j < ne; ++j) {
    succ[h.edge_tail[j]].push_back(h.edge_head[j]);
    ++indeg[h.edge_head[j]];
  }
  std::vector<int32_t> order, level(n + 2, 0);
  order.reserve(n + 2);
  for (int32_t v = 0; v < n + 2; ++v)
    if (indeg[v] == 0) order.push_back(v);
  for (size_t q = 0; q < order.size(); ++q) {
    const int32_t u = order[q];
    for (int32_t v : succ[u]) {
      if (u < n) level[v] = std::max(level[v], level[u] + 1);
      if (--indeg[v] == 0) order.push_back(v);
    }
  }
  if (static_cast<int32_t>(order.size()) != n + 2)
    return fail(PB_ERR_INVALID_ARGUMENT, "dependency graph contains a cycle");
  int32_t L = 0;
  for (int32_t i = 0; i < n; ++i) L = std::max(L, level[i] + 1);
  h.n_levels = L;
  h.lvl_off.assign(L + 1, 0);
  for (int32_t i = 0; i < n; ++i) ++h.lvl_off[level[i] + 1];
  for (int32_t l = 0; l < L; ++l) h.lvl_off[l + 1] += h.lvl_off[l];
  // level-major renumbering (stable in caller order inside a level)
  h.orig.assign(n, 0);
  h.inv.assign(n, 0);
  {
    std::vector<int32_t> fill(h.lvl_off.begin(), h.lvl_off.end() - 1);
    for (int32_t i = 0; i < n; ++i) {
      h.inv[i] = fill[level[i]]++;
      h.orig[h.inv[i]] = i;
    }
  }
  auto in_id = [&](int32_t x) { return x < n ? h.inv[x] : x; };
  h.icls.assign(n, 0);
  for (int32_t i = 0; i < n; ++i) h.icls[h.inv[i]] = h.comp_class[i];
  h.cflag.assign(n, 0);
  h.dep_nd.assign(ne, pb::int2h{0, 0});
  std::vector<std::vector<int32_t>> pv(n), sv(n);
  for (int32_t j = 0; j < ne; ++j) {
    const int32_t u = in_id(h.edge_tail[j]), v = in_id(h.edge_head[j]);
    h.dep_nd[j] = pb::int2h{u, v};
    if (v == n + 1 && u < n) h.cflag[u] |= 2;
    if (u == n && v < n) h.cflag[v] |= 1;
    if (u < n && v < n) {
      pv[v].push_back(u);
      sv[u].push_back(v);
    }
  }
  if (n >= (1 << 24)) return fail(PB_ERR_UNSUPPORTED, "more than 2^24 computations");
  // level of each internal id (level-major order)
  std::vector<int32_t>& ilev = h.ilev;
  ilev.assign(n, 0);
  for (int32_t l = 0; l < L; ++l)
    for (int32_t i = h.lvl_off[l]; i < h.lvl_off[l + 1]; ++i) ilev[i] = l;
  h.snk.clear();
  for (int32_t i = 0; i < n; ++i)
    if (h.cflag[i] & 2) h.snk.push_back(i);
  // sweep ring slot of neighbour u seen from i (pb_internal.h kRingLevels)
  auto ring = [&](int32_t i, int32_t u) {
    const int32_t gap = std::abs(ilev[i] - ilev[u]);
    const int32_t idx = u - h.lvl_off[ilev[u]];
    if (gap < 1 || gap >= pb::kRingLevels || idx >= 16) return u | (pb::kRingNone << 24);
    return u | (((ilev[u] % pb::kRingLevels) * 16 + idx) << 24);
  };
  auto csr = [&](std::vector<std::vector<int32_t>>& lists, std::vector<int32_t>& off,
                 std::vector<int32_t>& idx, std::vector<pb::int4h>& row, bool with_sink) {
    off.assign(n + 1, 0);
    idx.clear();
    row.assign(n, pb::int4h{0, -1, -1, -1});
    for (int32_t i = 0; i < n; ++i) {
      const auto& l = lists[i];
      const int32_t c = static_cast<int32_t>(l.size());
      row[i].x = std::min(c, 0xffff) | (with_sink && (h.cflag[i] & 2) ? (1 << 16) : 0);
      if (c > 0) row[i].y = ring(i, l[0]);
      if (c > 1) row[i].z = ring(i, l[1]);
      if (c > 2) row[i].w = ring(i, l[2]);
      idx.insert(idx.end(), l.begin(), l.end());
      off[i + 1] = static_cast<int32_t>(idx.size());
    }
  };
  csr(pv, h.pin_off, h.pin, h.frow, true);
  csr(sv, h.pout_off, h.pout, h.brow, false);
  // edge-centric network (dag.hpp:209-224) + return arc, internal ids
  const int32_t V = 2 * n + 2;
  std::vector<int32_t> et(n + ne + 1), eh(n + ne + 1);
  for (int32_t i = 0; i < n; ++i) {
    et[i] = 2 * i;
    eh[i] = 2 * i + 1;
  }
  for (int32_t j = 0; j < ne; ++j) {
    const int32_t u = h.dep_nd[j].x, v = h.dep_nd[j].y;
    et[n + j] = u == n ? 2 * n : 2 * u + 1;
    eh[n + j] = v == n + 1 ? 2 * n + 1 : 2 * v;
  }
  et[n + ne] = 2 * n + 1;
  eh[n + ne] = 2 * n;
  pb::build_net(V, et, eh, h.net, n);
  // network order of the dependency edges: by (head, tail) in internal ids,
  // so that the per-step criticality gathers (build_caps) walk memory
  // sequentially.  Only edge-indexed arrays are permuted: the incidence
  // lists (arc order, hence BFS discovery order) stay as built.
  {
    std::vector<int32_t> ord(ne);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
      return std::make_pair(h.dep_nd[x].y, h.dep_nd[x].x) < std::make_pair(h.dep_nd[y].y, h.dep_nd[y].x);
    });
    std::vector<pb::int2h> nd(ne), ep(ne);
    for (int32_t j = 0; j < ne; ++j) {
      nd[j] = h.dep_nd[ord[j]];
      ep[j] = h.net.epos[n + ord[j]];
    }
    h.dep_nd = std::move(nd);
    for (int32_t j = 0; j < ne; ++j) h.net.epos[n + j] = ep[j];
    h.dep_orig = std::move(ord);
  }
  return derive_start(h);
}

// The start-schedule-dependent part of validate_and_derive: the start in
// internal order and the sizing estimates (T_min, T*, steps, work).
pb_status derive_start(HostInst& h) {
  const int32_t n = h.n;
  h.istart.clear();
  if (!h.start.empty()) {
    h.istart.assign(n, 0);
    for (int32_t i = 0; i < n; ++i) h.istart[h.inv[i]] = h.start[i];
  }
  // sizing estimates
  std::vector<int64_t> fast(n), seed(n);
  for (int32_t i = 0; i < n; ++i) {
    const int32_t c = h.icls[i];
    fast[i] = h.pt_time[h.cls_pt_off[c]];
    seed[i] = h.start.empty() ? (h.cls_const[c] ? fast[i] : h.cls_trange[2 * c + 1]) : h.istart[i];
  }
  h.t_min_est = host_makespan(h, fast);
  h.t_star_est = host_makespan(h, seed);
  if (!h.start.empty()) {
    h.est_steps = std::max<int64_t>(1, h.max_steps);
  } else {
    const int64_t gap = std::max<int64_t>(0, h.t_star_est - h.t_min_est);
    h.est_steps = gap / h.tau + 2;
    if (h.max_steps > 0) h.est_steps = std::min<int64_t>(h.est_steps, h.max_steps);
  }
  h.work = walk_work(h);
  return PB_OK;
}

// ------------------------------------------------------------------- blobs

struct Blob {
  std::vector<char> bytes;
  size_t put(const void* p, size_t n) {
    const size_t at = (bytes.size() + 255) / 256 * 256;
    bytes.resize(at + n);
    if (n && p) std::memcpy(bytes.data() + at, p, n);
    return at;
  }
  template <class T>
  size_t put(const std::vector<T>& v) {
    return put(v.data(), v.size() * sizeof(T));
  }
};

struct int2h_pair {
  int32_t a, b;
};

struct CurveKey {
  uint64_t a, b, c;
  int64_t lo, hi;
  bool operator<(const CurveKey& o) const {
    return std::tie(a, b, c, lo, hi) < std::tie(o.a, o.b, o.c, o.lo, o.hi);
  }
};

uint64_t bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}

// Cooperative (wide) walk plan, see choose_wide().
struct WidePlan {
  int32_t n = 0, ctas = 0, warps = 4;
};

struct DeviceRun {
  int device = -1;
  char* d_static = nullptr;
  size_t wide_static_begin = 0, wide_static_end = 0;
  char* d_out = nullptr;
  char* d_ws = nullptr;
  pb::DevInst* d_insts = nullptr;
  int32_t* d_order = nullptr;
  int32_t* d_counter = nullptr;
  pb::RunCounters* d_counters = nullptr;
  int32_t* d_pool_ids = nullptr;
  uint8_t* d_pool_choice = nullptr;
  unsigned long long* d_pool_cursor = nullptr;
  long long pool_cap = 0;
  size_t out_bytes = 0;
  int32_t slots = 0;
  pb::WsLayout ws{};
  // allocated capacities (buffers are reused across runs while they fit)
  size_t cap_static = 0, cap_out = 0, cap_ws = 0, cap_insts = 0, cap_order = 0;
  long long cap_pool = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // walk launch
  cudaEvent_t ex0 = nullptr, ex1 = nullptr;  // H2D / D2H copies
  WidePlan wide;
  int32_t smem_ctas = 0, smem_region = 0;  // > 0: every walk runs in walk_kernel_smem
  char* h_out = nullptr;  // pinned
  char* d_carry = nullptr;  // warm-start state of a get-next chain (pb_internal.h CarryHdr)
  size_t cap_carry = 0;
  void release() {
    if (device < 0) return;
    cudaSetDevice(device);
    cudaFree(d_static);
    cudaFree(d_out);
    cudaFree(d_ws);
    cudaFree(d_insts);
    cudaFree(d_order);
    cudaFree(d_counter);
    cudaFree(d_counters);
    cudaFree(d_pool_ids);
    cudaFree(d_pool_choice);
    cudaFree(d_pool_cursor);
    cudaFree(d_carry);
    if (h_out) cudaFreeHost(h_out);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ex0) cudaEventDestroy(ex0);
    if (ex1) cudaEventDestroy(ex1);
    if (stream) cudaStreamDestroy(stream);
    *this = DeviceRun{};
  }
};

}  // namespace

struct pb_batch {
  std::vector<HostInst> insts;
  // packed host-side view (tables kept for host expansion)
  std::vector<double> tables;
  std::vector<std::vector<int64_t>> cls_tab;  // per instance per class: table offset of E(t_min)
  std::vector<std::pair<int64_t, int64_t>> tab_margin;  // per instance: table extent below t_min / above t_max
  // outputs (host copies)
  std::vector<size_t> out_points, out_summary;
  std::vector<int32_t> cap_points;
  std::vector<char> out;  // host results of a multi-device run (stitched)
  const char* outp = nullptr;  // host results: R.h_out (pinned) or out.data()
  std::vector<int32_t> pool_ids;  // delta pool (used prefix)
  std::vector<uint8_t> pool_choice;
  std::vector<long long> pool_base;  // per instance: offset of its id_begin values
  long long pool_cap = 0;
  bool have_results = false;
  DeviceRun run;
  pb_run_stats stats{};
  int64_t prof[pb::kPrSlots] = {};
  HostInst derived;  // last instance derived by pb_batch_add (kept across pb_batch_clear)
  uint64_t derived_gen = 0;  // bumped whenever `derived` is replaced
  // get-next chain (one instance, the drop-in's loop of get_next_schedule):
  // the device carry buffer holds the flow state the last walk ended in,
  // valid for the start schedule carry_start (caller order) of derived_gen
  bool carry_valid = false;
  uint64_t carry_gen = 0;
  int64_t carry_tau = 0;
  std::vector<int64_t> carry_start;
  char* h_static = nullptr;  // pinned staging of the packed static blob (reused)
  size_t h_static_cap = 0;
  // E(t) = a exp(b t) + c per curve over a contiguous range [lo, lo + size),
  // grown on demand (costmodel.hpp:47: same expression and libm)
  struct CurveCache {
    int64_t lo = 0;
    std::vector<double> v;
  };
  std::map<std::array<uint64_t, 3>, CurveCache> curve_cache;
  size_t curve_cache_values = 0;
  static std::array<uint64_t, 3> curve_id(double a, double b, double c) {
    uint64_t x, y, z;
    std::memcpy(&x, &a, 8);
    std::memcpy(&y, &b, 8);
    std::memcpy(&z, &c, 8);
    return {x, y, z};
  }
  int64_t curve_lo(double a, double b, double c) const { return curve_cache.at(curve_id(a, b, c)).lo; }
  const std::vector<double>& curve_values(double a, double b, double c, int64_t lo, int64_t hi) {
    if (curve_cache_values > (size_t{1} << 26)) {  // bound the cache (~512 MB)
      curve_cache.clear();
      curve_cache_values = 0;
    }
    auto eval = [&](int64_t t) { return a * std::exp(b * static_cast<double>(t)) + c; };
    auto ins = curve_cache.emplace(curve_id(a, b, c), CurveCache{});
    CurveCache& cc = ins.first->second;
    if (ins.second || cc.v.empty()) {
      cc.lo = lo;
      cc.v.resize(hi - lo + 1);
      for (int64_t t = lo; t <= hi; ++t) cc.v[t - lo] = eval(t);
      curve_cache_values += cc.v.size();
      return cc.v;
    }
    const int64_t clo = cc.lo, chi = cc.lo + static_cast<int64_t>(cc.v.size()) - 1;
    if (lo < clo) {
      std::vector<double> head(clo - lo);
      for (int64_t t = lo; t < clo; ++t) head[t - lo] = eval(t);
      cc.v.insert(cc.v.begin(), head.begin(), head.end());
      cc.lo = lo;
      curve_cache_values += head.size();
    }
    if (hi > chi) {
      const size_t old = cc.v.size();
      cc.v.resize(old + (hi - chi));
      for (int64_t t = chi + 1; t <= hi; ++t) cc.v[t - cc.lo] = eval(t);
      curve_cache_values += hi - chi;
    }
    return cc.v;
  }
  ~pb_batch() {
    run.release();
    if (h_static) cudaFreeHost(h_static);
  }
};

namespace {

// Packs all instances; returns host blobs and per-instance DevInst with
// offsets (converted to device pointers once the blob is uploaded).
struct Packed {
  long long pool_cap = 0;
  size_t stat_bytes = 0;  // packed static blob (tables first), in pb_batch::h_static
  std::vector<pb::DevInst> dev;
  std::vector<std::array<size_t, 32>> offs;
  size_t out_bytes = 0;
  int64_t max_n = 1, max_v = 1, max_e = 1;
  std::vector<int32_t> order;
};

enum OffIdx {
  O_ORIG, O_CLASS, O_CFLAG, O_LVLOFF, O_FROW, O_BROW, O_PINOFF, O_PIN, O_POUTOFF, O_POUT, O_DEPND,
  O_INCOFF, O_IENT, O_EPOS, O_DEPORIG, O_CCONST, O_CTMIN, O_CTMAX, O_CTAB, O_CPOFF, O_PTIME, O_PENERGY,
  O_START, O_CURVE, O_CREC, O_POINTS, O_SUMMARY, O_ILEV, O_SNK, O_COUNT
};

void put_static(Blob& blob, const HostInst& h, std::array<size_t, 32>& o) {
  o[O_ORIG] = blob.put(h.orig);
  o[O_CLASS] = blob.put(h.icls);
  o[O_CFLAG] = blob.put(h.cflag);
  o[O_LVLOFF] = blob.put(h.lvl_off);
  o[O_FROW] = blob.put(h.frow);
  o[O_BROW] = blob.put(h.brow);
  o[O_PINOFF] = blob.put(h.pin_off);
  o[O_PIN] = blob.put(h.pin);
  o[O_POUTOFF] = blob.put(h.pout_off);
  o[O_POUT] = blob.put(h.pout);
  o[O_DEPND] = blob.put(h.dep_nd);
  o[O_INCOFF] = blob.put(h.net.inc_off);
  o[O_IENT] = blob.put(h.net.ient);
  o[O_EPOS] = blob.put(h.net.epos);
  o[O_DEPORIG] = blob.put(h.dep_orig);
  o[O_ILEV] = blob.put(h.ilev);
  o[O_SNK] = blob.put(h.snk);
}

void fill_shape(pb::DevInst& d, const HostInst& h) {
  d.n = h.n;
  d.ne = static_cast<int32_t>(h.edge_tail.size());
  d.n_levels = h.n_levels;
  d.V = 2 * h.n + 2;
  d.E = h.n + d.ne + 1;
  d.ret_pt = h.net.epos[d.E - 1].x;
  d.ret_ph = h.net.epos[d.E - 1].y;
  d.n_snk = static_cast<int32_t>(h.snk.size());
}

// Every static section of instance k in blob order: f(slot, data, bytes).
// With fill = false only the sizes are needed (data may be null).
template <class F>
void instance_sections(const pb_batch* b, size_t k, bool fill, F&& f) {
  const HostInst& h = b->insts[k];
  auto vec = [&](int slot, const auto& v) { f(slot, static_cast<const void*>(v.data()), v.size() * sizeof(v[0])); };
  vec(O_ORIG, h.orig);
  vec(O_CLASS, h.icls);
  vec(O_CFLAG, h.cflag);
  vec(O_LVLOFF, h.lvl_off);
  vec(O_FROW, h.frow);
  vec(O_BROW, h.brow);
  vec(O_PINOFF, h.pin_off);
  vec(O_PIN, h.pin);
  vec(O_POUTOFF, h.pout_off);
  vec(O_POUT, h.pout);
  vec(O_DEPND, h.dep_nd);
  vec(O_INCOFF, h.net.inc_off);
  vec(O_IENT, h.net.ient);
  vec(O_EPOS, h.net.epos);
  vec(O_DEPORIG, h.dep_orig);
  vec(O_ILEV, h.ilev);
  vec(O_SNK, h.snk);
  vec(O_CCONST, h.cls_const);
  const size_t nc = h.cls_const.size();
  std::vector<int64_t> tmin, tmax;
  std::vector<pb::CompRec> rec;
  if (fill) {
    tmin.resize(nc);
    tmax.resize(nc);
    for (size_t c = 0; c < nc; ++c) {
      tmin[c] = h.cls_trange[2 * c];
      tmax[c] = h.cls_trange[2 * c + 1];
    }
    rec.resize(h.n);
    for (int32_t i = 0; i < h.n; ++i) {
      const int32_t c = h.icls[i];
      const bool cst = h.cls_const[c] != 0;
      rec[i] = pb::CompRec{cst ? 0 : h.cls_trange[2 * c], cst ? 0 : h.cls_trange[2 * c + 1],
                           cst ? -1 : b->cls_tab[k][c], h.net.epos[i].x, h.net.epos[i].y};
    }
  }
  f(O_CTMIN, tmin.data(), sizeof(int64_t) * nc);
  f(O_CTMAX, tmax.data(), sizeof(int64_t) * nc);
  vec(O_CTAB, b->cls_tab[k]);
  vec(O_CPOFF, h.cls_pt_off);
  vec(O_PTIME, h.pt_time);
  vec(O_PENERGY, h.pt_energy);
  if (!h.istart.empty()) vec(O_START, h.istart);
  vec(O_CURVE, h.cls_curve);
  f(O_CREC, rec.data(), sizeof(pb::CompRec) * static_cast<size_t>(h.n));
}

void pack(pb_batch* b, Packed& P, std::vector<int32_t>& cap_points, double cap_scale) {
  const size_t N = b->insts.size();
  // curve tables, deduplicated by (a, b, c, t_min, t_max) bit patterns
  // A discover walk only evaluates curves inside [t_min, t_max]: speed-ups
  // cross finite S->T edges (can_speed: t - tau >= t_min) and slow-downs are
  // bounded by t_max (frontier.hpp:117-125).  The cut of a feasible network
  // never holds an infinite S->T edge below the sentinel ("Rule
  // 5"), so frontier.hpp:111-116's unchecked speed-up cannot leave the range
  // either.  A get-next start schedule may lie anywhere: its tables are
  // widened to cover every start time +- tau.
  b->tab_margin.assign(N, {0, 0});
  for (size_t k = 0; k < N; ++k) {
    const HostInst& h = b->insts[k];
    if (h.start.empty()) continue;
    int64_t mlo = 0, mhi = 0;
    for (int32_t i = 0; i < h.n; ++i) {
      const int32_t c = h.comp_class[i];
      if (h.cls_const[c]) continue;
      mlo = std::max(mlo, h.cls_trange[2 * c] - (h.start[i] - h.tau));
      mhi = std::max(mhi, h.start[i] + h.tau - h.cls_trange[2 * c + 1]);
    }
    b->tab_margin[k] = {mlo, mhi};
  }
  std::map<CurveKey, int64_t> table_of;
  b->tables.clear();
  b->cls_tab.assign(N, {});
  for (size_t k = 0; k < N; ++k) {
    const HostInst& h = b->insts[k];
    const size_t nc = h.cls_const.size();
    b->cls_tab[k].assign(nc, 0);
    for (size_t c = 0; c < nc; ++c) {
      if (h.cls_const[c]) continue;
      const double a = h.cls_curve[3 * c], bb = h.cls_curve[3 * c + 1], cc = h.cls_curve[3 * c + 2];
      const int64_t lo = h.cls_trange[2 * c], hi = h.cls_trange[2 * c + 1];
      const int64_t tlo = lo - b->tab_margin[k].first, thi = hi + b->tab_margin[k].second;
      const CurveKey key{bits(a), bits(bb), bits(cc), tlo, thi};
      auto it = table_of.find(key);
      if (it == table_of.end()) {
        const int64_t at = static_cast<int64_t>(b->tables.size());
        const int64_t span = thi - tlo + 1;
        if (span > (int64_t{1} << 27)) throw std::length_error("curve interval too long to tabulate");
        b->tables.resize(b->tables.size() + span);
        // ExpCurve::eval (costmodel.hpp:47), same expression and libm; values
        // persist in the handle's curve cache across runs and pb_batch_clear
        // (a get_next_schedule chain re-tabulates only the newly reached times)
        const std::vector<double>& v = b->curve_values(a, bb, cc, tlo, thi);
        std::memcpy(b->tables.data() + at, v.data() + (tlo - b->curve_lo(a, bb, cc)), sizeof(double) * span);
        it = table_of.emplace(key, at).first;
      }
      b->cls_tab[k][c] = it->second + (lo - tlo);  // offset of E(t_min)
    }
  }
  P.dev.assign(N, pb::DevInst{});
  P.offs.assign(N, {});
  cap_points.assign(N, 0);
  long long pool = 0;
  size_t out = 0;
  auto out_take = [&](size_t bytes) {
    const size_t at = (out + 255) / 256 * 256;
    out = at + bytes;
    return at;
  };
  // LPT: largest estimated work first
  P.order.resize(N);
  std::iota(P.order.begin(), P.order.end(), 0);
  std::stable_sort(P.order.begin(), P.order.end(), [&](int32_t x, int32_t y) {
    return b->insts[x].work > b->insts[y].work;
  });
  // layout pass: section offsets of every instance (tables at offset 0),
  // instances in LPT order so the head walks' static data is contiguous
  size_t off = b->tables.size() * sizeof(double);
  for (size_t q = 0; q < N; ++q) {
    const size_t k = static_cast<size_t>(P.order[q]);
    auto& o = P.offs[k];
    o[O_START] = SIZE_MAX;
    instance_sections(b, k, false, [&](int slot, const void*, size_t bytes) {
      off = (off + 255) / 256 * 256;
      o[slot] = off;
      off += bytes;
    });
  }
  P.stat_bytes = std::max<size_t>(off, 256);
  if (b->h_static_cap < P.stat_bytes) {
    if (b->h_static) cudaFreeHost(b->h_static);
    b->h_static = nullptr;
    b->h_static_cap = 0;
    ck(cudaMallocHost(&b->h_static, P.stat_bytes + P.stat_bytes / 4), "malloc pinned static");
    b->h_static_cap = P.stat_bytes + P.stat_bytes / 4;
  }
  std::memcpy(b->h_static, b->tables.data(), b->tables.size() * sizeof(double));
  // fill pass: instances copied in parallel straight into pinned memory
  {
    // threads only for batches worth it (a single instance -- the drop-in's
    // per-call path -- is copied inline: thread start-up would dominate)
    const unsigned nt = std::max(1u, std::min<unsigned>({std::thread::hardware_concurrency(), 16u,
                                                          static_cast<unsigned>((N + 15) / 16)}));
    auto fill = [&](unsigned t) {
      for (size_t k = t; k < N; k += nt)
        instance_sections(b, k, true, [&](int slot, const void* p, size_t bytes) {
          if (bytes) std::memcpy(b->h_static + P.offs[k][slot], p, bytes);
        });
    };
    if (nt == 1) {
      fill(0);
    } else {
      std::vector<std::thread> pool_t;
      for (unsigned t = 0; t < nt; ++t) pool_t.emplace_back(fill, t);
      for (auto& th : pool_t) th.join();
    }
  }
  for (size_t k = 0; k < N; ++k) {
    const HostInst& h = b->insts[k];
    auto& o = P.offs[k];
    const int64_t est = static_cast<int64_t>(static_cast<double>(h.est_steps) * cap_scale);
    cap_points[k] = static_cast<int32_t>(std::min<int64_t>(est + 8, INT32_MAX / 2));
    pool += est * 12 + 2 * int64_t{h.n} + 64;
    o[O_POINTS] = out_take(sizeof(pb_point) * cap_points[k]);
    o[O_SUMMARY] = out_take(sizeof(pb_frontier_summary));
    pb::DevInst& d = P.dev[k];
    fill_shape(d, h);
    d.mode = h.start.empty() ? pb::kModeDiscover : pb::kModeGetNext;
    d.max_steps = h.start.empty() ? h.max_steps : (h.max_steps == 0 ? 1 : h.max_steps);
    d.cap_points = cap_points[k];
    d.tau = h.tau;
    d.tab_mlo = b->tab_margin[k].first;
    d.tab_mhi = b->tab_margin[k].second;
    d.watts = h.watts;
    d.quantum = h.quantum;
    P.max_n = std::max<int64_t>(P.max_n, d.n);
    P.max_v = std::max<int64_t>(P.max_v, d.V);
    P.max_e = std::max<int64_t>(P.max_e, d.E);
  }
  P.out_bytes = out;
  P.pool_cap = std::min<long long>(pool, (1ll << 31) - 1);
  b->cap_points = cap_points;
  b->pool_cap = P.pool_cap;
  b->out_points.assign(N, 0);
  b->out_summary.assign(N, 0);
  b->pool_base.assign(N, 0);
  for (size_t k = 0; k < N; ++k) {
    b->out_points[k] = P.offs[k][O_POINTS];
    b->out_summary[k] = P.offs[k][O_SUMMARY];
  }
}

template <class T>
T* dptr(char* base, size_t off) {
  return off == SIZE_MAX ? nullptr : reinterpret_cast<T*>(base + off);
}

void bind_static(pb::DevInst& d, char* base, const std::array<size_t, 32>& o) {
  d.orig = dptr<int32_t>(base, o[O_ORIG]);
  d.comp_class = dptr<int32_t>(base, o[O_CLASS]);
  d.cflag = dptr<uint8_t>(base, o[O_CFLAG]);
  d.lvl_off = dptr<int32_t>(base, o[O_LVLOFF]);
  d.frow = dptr<int4>(base, o[O_FROW]);
  d.brow = dptr<int4>(base, o[O_BROW]);
  d.pin_off = dptr<int32_t>(base, o[O_PINOFF]);
  d.pin = dptr<int32_t>(base, o[O_PIN]);
  d.pout_off = dptr<int32_t>(base, o[O_POUTOFF]);
  d.pout = dptr<int32_t>(base, o[O_POUT]);
  d.dep_nd = dptr<int2>(base, o[O_DEPND]);
  d.inc_off = dptr<int32_t>(base, o[O_INCOFF]);
  d.ient = dptr<pb::IEnt>(base, o[O_IENT]);
  d.epos = dptr<int2>(base, o[O_EPOS]);
  d.dep_orig = dptr<int32_t>(base, o[O_DEPORIG]);
  d.ilev = dptr<int32_t>(base, o[O_ILEV]);
  d.snk = dptr<int32_t>(base, o[O_SNK]);
}

void bind_device(Packed& P, char* d_static, char* d_out, size_t tables_off) {
  for (size_t k = 0; k < P.dev.size(); ++k) {
    auto& o = P.offs[k];
    pb::DevInst& d = P.dev[k];
    bind_static(d, d_static, o);
    d.cls_const = dptr<uint8_t>(d_static, o[O_CCONST]);
    d.cls_tmin = dptr<int64_t>(d_static, o[O_CTMIN]);
    d.cls_tmax = dptr<int64_t>(d_static, o[O_CTMAX]);
    d.cls_tab = dptr<int64_t>(d_static, o[O_CTAB]);
    d.cls_pt_off = dptr<int32_t>(d_static, o[O_CPOFF]);
    d.pt_time = dptr<int64_t>(d_static, o[O_PTIME]);
    d.pt_energy = dptr<int64_t>(d_static, o[O_PENERGY]);
    d.tables = dptr<double>(d_static, tables_off);
    d.start_planned_t = dptr<int64_t>(d_static, o[O_START]);
    d.cls_curve = dptr<double>(d_static, o[O_CURVE]);
    d.crec = dptr<pb::CompRec>(d_static, o[O_CREC]);
    d.points = dptr<pb_point>(d_out, o[O_POINTS]);
    d.summary = dptr<pb_frontier_summary>(d_out, o[O_SUMMARY]);
  }
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

// Cooperative (wide) walks, pb_internal.h launch_walks: the LPT head.
// PB_WIDE = number of instances (default: those whose estimated work is at
// least PB_WIDE_PERMILLE of the largest, only for batches that fill the
// device), PB_WIDE_CTAS = concurrent wide walks, PB_WIDE_WARPS = warps each.
// DAGs whose BFS levels are wide enough for two warps to pay off.
bool wide_dag(const HostInst& h) { return h.n >= 11 * std::max(1, h.n_levels); }

WidePlan choose_wide(const pb_batch* b, const std::vector<int32_t>& order, int sms, int per_sm) {
  WidePlan w;
  const int64_t N = static_cast<int64_t>(order.size());
  w.warps = std::max(2, std::min(4, env_int("PB_WIDE_WARPS", 2)));
  int n = env_int("PB_WIDE", -1);
  const int ctas = env_int("PB_WIDE_CTAS", 128);
  if (n < 0 && N > 0) {
    n = 0;
    // Walker load: the estimated walker time left after a full wave of
    // cooperative CTAs, in units of the longest walk on all walker slots
    // (each cooperative CTA costs its SM one 4-warp walker block).
    const double top = static_cast<double>(b->insts[order[0]].work);
    const int64_t head = std::min<int64_t>(ctas, N);
    double rest = 0;
    for (int64_t k = head; k < N; ++k) rest += static_cast<double>(b->insts[order[k]].work);
    const double slots = std::max<double>(1.0, double(sms) * per_sm - 4.0 * std::min(head, int64_t{sms}));
    const double load = top > 0 ? rest / (slots * top) : 0.0;
    if (load <= 0.5) {
      // walkers have slack (a strong-scaling shard, a small batch): a full
      // wave of cooperative walks.  Measured on LPT shards of the 4096 batch
      // (DESIGN.md): 1/8 shard 8.79 -> 6.52-6.73 s, 1/4 9.72 -> 7.31 s, 1/2
      // 8.55 -> 7.83 s
      n = static_cast<int>(head);
    } else {
      // walkers saturated (the 4096 batch: load 0.72): only the walks with
      // >= 87.5% of the largest estimated time (54 walks).  With the anchor
      // chase (walkers 9% faster): 8.89-9.00 s vs 9.37-9.52 (80%), 9.21-9.29
      // (82.5%), 9.00 (85%), 9.07-9.10 (90%)
      const int permille = env_int("PB_WIDE_PERMILLE", 875);
      while (permille > 0 && n < N && static_cast<double>(b->insts[order[n]].work) * 1000.0 >= permille * top) ++n;
    }
    // a batch of (near-)equal walks: unless every walk gets a cooperative
    // CTA, the walker walks still take as long as before, so cooperative CTAs
    // only cost walker slots (config 4 x 296: 4.68 s with 128 vs 4.53 s
    // without; config 1 x 4096: 0.29 s with a cooperative head vs 0.05 s)
    if (N > ctas && static_cast<double>(b->insts[order[N - 1]].work) * 1000.0 >= 825.0 * top) n = 0;
    // only wide DAGs walk faster on two warps (width n / levels >= 11; on
    // 6-8-wide DAGs the cooperative discovery order needs 2-4x the augmenting
    // paths): the head ends at the first narrow walk
    int wide_ok = 0;
    while (wide_ok < n && wide_dag(b->insts[order[wide_ok]])) ++wide_ok;
    n = wide_ok;
  }
  // the head is at most one wave of cooperative CTAs (a batch of equal walks
  // would otherwise queue every walk behind them)
  if (env_int("PB_WIDE", -1) < 0) n = std::min(n, ctas);
  w.n = static_cast<int32_t>(std::min<int64_t>(n, N));
  w.ctas = w.n > 0 ? std::max(1, std::min(ctas, w.n)) : 0;
  return w;
}

// Walker warps: what is left of the device after the wide CTAs (4-warp
// blocks, like the walker's).
int32_t device_slots(int device, int64_t n_walk, const pb::WsLayout& ws, const WidePlan& w) {
  int sms = 0;
  ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "sm count");
  const int per_sm = std::max(1, env_int("PB_WARPS_PER_SM", pb::walk_slots_per_sm(ws)));
  const int64_t wide_warps = int64_t{w.ctas} * w.warps;
  return static_cast<int32_t>(
      std::max<int64_t>(std::min<int64_t>(n_walk, int64_t{sms} * per_sm - wide_warps), std::min<int64_t>(n_walk, 4)));
}

// Device allocation owned by one call: freed on every exit path, including
// the CudaError thrown by a later ck().
template <class T>
struct DevBuf {
  T* p = nullptr;
  DevBuf(size_t count, const char* what) {
    ck(cudaMalloc(reinterpret_cast<void**>(&p), sizeof(T) * std::max<size_t>(count, 1)), what);
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// (Re)allocates a device buffer only when the current one is too small.
template <class T>
void ensure_device(T*& ptr, size_t& cap, size_t bytes, const char* what) {
  bytes = std::max<size_t>(bytes, 256);
  if (ptr && cap >= bytes) return;
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
  ck(cudaMalloc(reinterpret_cast<void**>(&ptr), bytes), what);
  cap = bytes;
}

// Packs the batch (host, parallel, into pinned staging) and uploads it.
// Device buffers, pinned buffers, streams and events persist across runs on
// the same device and are only grown.
pb_status prepare_impl(pb_batch* b, int32_t device, double cap_scale) {
  DeviceRun& R = b->run;
  if (R.device >= 0 && R.device != device) {
    R.release();
    b->carry_valid = false;
  }
  b->have_results = false;
  const size_t N = b->insts.size();
  if (N == 0) return PB_OK;
  ck(cudaSetDevice(device), "cudaSetDevice");
  if (R.device < 0) {
    R.device = device;
    ck(cudaStreamCreateWithFlags(&R.stream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&R.ev0), "event");
    ck(cudaEventCreate(&R.ev1), "event");
    ck(cudaEventCreate(&R.ex0), "event");
    ck(cudaEventCreate(&R.ex1), "event");
    ck(cudaMalloc(&R.d_counter, 3 * sizeof(int32_t)), "malloc counter");
    ck(cudaMalloc(&R.d_counters, sizeof(pb::RunCounters)), "malloc counters");
    ck(cudaMalloc(&R.d_pool_cursor, sizeof(unsigned long long)), "malloc cursor");
  }
  Packed P;
  std::vector<int32_t> capp;
  const auto pack_t0 = std::chrono::steady_clock::now();
  pack(b, P, capp, cap_scale);
  const double pack_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - pack_t0).count();
  const size_t tables_off = 0;  // tables are the first section of the blob
  cudaEvent_t h0 = R.ex0, h1 = R.ex1;
  ensure_device(R.d_static, R.cap_static, P.stat_bytes, "malloc static");
  R.out_bytes = std::max<size_t>(P.out_bytes, 256);
  if (R.cap_out < R.out_bytes) {
    if (R.d_out) cudaFree(R.d_out);
    if (R.h_out) cudaFreeHost(R.h_out);
    R.d_out = nullptr;
    R.h_out = nullptr;
    R.cap_out = 0;
    const size_t want = R.out_bytes + R.out_bytes / 4;
    ck(cudaMalloc(&R.d_out, want), "malloc out");
    ck(cudaMallocHost(&R.h_out, want), "malloc pinned out");
    R.cap_out = want;
  }
  bind_device(P, R.d_static, R.d_out, tables_off);
  // get-next chain warm start: a single get-next walk of the handle's derived
  // instance carries its flow state to the next call; it resumes when its
  // start schedule is exactly where the last one ended
  if (N == 1 && !b->insts[0].start.empty() && b->insts[0].max_steps >= 0 && !std::getenv("PB_NO_CARRY")) {
    const HostInst& h = b->insts[0];
    pb::DevInst& d = P.dev[0];
    ensure_device(R.d_carry, R.cap_carry, pb::carry_bytes(h.n, d.E), "malloc carry");
    d.carry = R.d_carry;
    d.resume = b->carry_valid && h.gen != 0 && b->carry_gen == h.gen && b->carry_tau == h.tau &&
               b->carry_start == h.start;
  }
  R.ws = pb::make_ws_layout(P.max_n, P.max_v, P.max_e);
  {
    int sms = 0;
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "sm count");
    R.wide = choose_wide(b, P.order, sms, std::max(1, pb::walk_slots_per_sm(R.ws)));
    // Shared-memory-resident walks (walk_kernel_smem) whenever every walk of
    // the batch gets its own CTA at once (PB_SMEM: -1 auto, 0 off, 1 force):
    // one warp per SM-resident region instead of a warp of a 12-warp walker SM
    R.smem_ctas = 0;
    R.smem_region = 0;
    // (an explicit PB_WIDE request keeps the cooperative kernel; PB_SMEM_REGION
    // caps the region, e.g. to test partial placement)
    const int mode = env_int("PB_SMEM", std::getenv("PB_WIDE") ? 0 : -1);
    if (mode != 0) {
      int64_t fmax = 0;
      for (const pb::DevInst& d : P.dev)
        fmax = std::max(fmax, pb::smem_footprint(d.n, d.V, d.E, d.ne, d.n_levels, d.n_snk));
      if (const int cap_region = env_int("PB_SMEM_REGION", -1); cap_region >= 0)
        fmax = std::min<int64_t>(fmax, cap_region);
      int32_t region = 0, per = 0;
      if (pb::smem_walk_plan(R.ws, fmax, &region, &per) != 0) throw CudaError("smem walk plan");
      const int64_t cap = int64_t{sms} * per;
      // Wide DAGs that do not fit the region walk faster on the cooperative
      // kernel (2 warps split every BFS level): measured alone, width
      // n / levels >= 11 gains 13-19% (config 4 936 -> 757 us/step, 16x256
      // 1,065 -> 911), width 6-8 loses 2-3x (its discovery order finds many
      // more augmenting paths), DESIGN.md.  A batch made only of such walks,
      // one CTA each, goes cooperative instead.
      bool all_wide = mode != 1 && static_cast<int64_t>(N) <= std::min<int64_t>(sms, 128);
      for (size_t k = 0; all_wide && k < N; ++k) {
        const pb::DevInst& d = P.dev[k];
        all_wide = static_cast<double>(d.n) >= 11.0 * std::max(1, d.n_levels) &&
                   pb::smem_footprint(d.n, d.V, d.E, d.ne, d.n_levels, d.n_snk) > region;
      }
      if (all_wide) {
        R.wide.n = static_cast<int32_t>(N);
        R.wide.ctas = static_cast<int32_t>(N);
      } else if (per > 0 && (mode == 1 || static_cast<int64_t>(N) <= cap)) {
        R.smem_ctas = static_cast<int32_t>(std::min<int64_t>(static_cast<int64_t>(N), cap));
        R.smem_region = region;
        R.wide = WidePlan{};
      }
    }
  }
  // static bytes of the cooperative head walks (contiguous: LPT layout)
  R.wide_static_begin = N ? P.offs[P.order[0]][O_ORIG] : 0;
  R.wide_static_end = R.wide.n < static_cast<int32_t>(N) ? P.offs[P.order[R.wide.n]][O_ORIG] : P.stat_bytes;
  R.slots = R.smem_ctas > 0 ? R.smem_ctas : device_slots(device, static_cast<int64_t>(N) - R.wide.n, R.ws, R.wide);
  ensure_device(R.d_ws, R.cap_ws, static_cast<size_t>(R.ws.stride) * (R.slots + R.wide.ctas), "malloc workspace");
  ensure_device(R.d_insts, R.cap_insts, sizeof(pb::DevInst) * N, "malloc insts");
  ensure_device(R.d_order, R.cap_order, sizeof(int32_t) * N, "malloc order");
  R.pool_cap = P.pool_cap;
  if (R.cap_pool < std::max<long long>(R.pool_cap, 1)) {
    if (R.d_pool_ids) cudaFree(R.d_pool_ids);
    if (R.d_pool_choice) cudaFree(R.d_pool_choice);
    R.d_pool_ids = nullptr;
    R.d_pool_choice = nullptr;
    R.cap_pool = 0;
    const long long want = std::max<long long>(R.pool_cap, 1);
    ck(cudaMalloc(&R.d_pool_ids, sizeof(int32_t) * want), "malloc pool");
    ck(cudaMalloc(&R.d_pool_choice, want), "malloc pool");
    R.cap_pool = want;
  }
  ck(cudaEventRecord(h0, R.stream), "record");
  ck(cudaMemcpyAsync(R.d_static, b->h_static, P.stat_bytes, cudaMemcpyHostToDevice, R.stream), "H2D static");
  ck(cudaMemcpyAsync(R.d_insts, P.dev.data(), sizeof(pb::DevInst) * N, cudaMemcpyHostToDevice, R.stream),
     "H2D insts");
  ck(cudaMemcpyAsync(R.d_order, P.order.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, R.stream),
     "H2D order");
  ck(cudaEventRecord(h1, R.stream), "record");
  ck(cudaStreamSynchronize(R.stream), "sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, h0, h1);
  b->stats = pb_run_stats{};
  b->stats.h2d_ms = ms;
  b->stats.pack_ms = pack_ms;
  b->stats.warm_starts = N == 1 && P.dev[0].resume ? 1 : 0;
  b->stats.h2d_bytes = static_cast<int64_t>(P.stat_bytes + sizeof(pb::DevInst) * N + sizeof(int32_t) * N);
  return PB_OK;
}

pb_status launch_impl(pb_batch* b, double* kernel_ms) {
  DeviceRun& R = b->run;
  const size_t N = b->insts.size();
  if (N == 0) {
    if (kernel_ms) *kernel_ms = 0;
    return PB_OK;
  }
  if (R.device < 0) return fail(PB_ERR_LOGIC, "batch not prepared");
  ck(cudaSetDevice(R.device), "cudaSetDevice");
  ck(cudaMemsetAsync(R.d_counter, 0, 3 * sizeof(int32_t), R.stream), "memset");
  ck(cudaMemsetAsync(R.d_counters, 0, sizeof(pb::RunCounters), R.stream), "memset");
  ck(cudaMemsetAsync(R.d_pool_cursor, 0, sizeof(unsigned long long), R.stream), "memset");
  pb::DeltaPool pool{R.d_pool_ids, R.d_pool_choice, R.d_pool_cursor, R.pool_cap};
  if (const int mb = env_int("PB_L2_PERSIST_MB", 0); mb > 0 && R.wide.ctas > 0) {
    int max_persist = 0, max_win = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, R.device);
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, R.device);
    const size_t persist = std::min<size_t>(static_cast<size_t>(mb) << 20, static_cast<size_t>(max_persist));
    ck(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist), "persisting L2");
    cudaStreamAttrValue a{};
    const bool stat = std::getenv("PB_L2_STATIC") != nullptr;  // the head walks' static data instead
    a.accessPolicyWindow.base_ptr = stat ? R.d_static + R.wide_static_begin : R.d_ws;
    a.accessPolicyWindow.num_bytes =
        std::min<size_t>(stat ? R.wide_static_end - R.wide_static_begin
                              : static_cast<size_t>(R.wide.ctas) * R.ws.stride,
                         static_cast<size_t>(max_win));
    a.accessPolicyWindow.hitRatio =
        std::min(1.0f, static_cast<float>(persist) / static_cast<float>(a.accessPolicyWindow.num_bytes));
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ck(cudaStreamSetAttribute(R.stream, cudaStreamAttributeAccessPolicyWindow, &a), "L2 window");
    if (std::getenv("PB_L2_VERBOSE"))
      std::fprintf(stderr, "L2 persist %zu of max %d, window %zu (max %d), hit %.2f\n", persist, max_persist,
                   a.accessPolicyWindow.num_bytes, max_win, a.accessPolicyWindow.hitRatio);
  }
  ck(cudaEventRecord(R.ev0, R.stream), "record");
  const int rc = R.smem_ctas > 0
                     ? pb::launch_walks_smem(R.d_insts, static_cast<int32_t>(N), R.d_order, R.d_counter, R.d_ws,
                                             R.ws, R.smem_region, R.smem_ctas, R.d_counters, pool, R.stream)
                     : pb::launch_walks(R.d_insts, static_cast<int32_t>(N), R.d_order, R.d_counter, R.d_ws, R.ws,
                                        R.slots, R.d_counters, pool, R.wide.n, R.wide.ctas, R.wide.warps, R.stream);
  if (rc != 0) throw CudaError(std::string("walk launch: ") + cudaGetErrorString(static_cast<cudaError_t>(rc)));
  ck(cudaEventRecord(R.ev1, R.stream), "record");
  ck(cudaStreamSynchronize(R.stream), "walk kernel");
  float ms = 0;
  cudaEventElapsedTime(&ms, R.ev0, R.ev1);
  pb::RunCounters rcnt{};
  ck(cudaMemcpy(&rcnt, R.d_counters, sizeof rcnt, cudaMemcpyDeviceToHost), "D2H counters");
  b->stats.kernel_ms = ms;
  b->stats.arc_scans = static_cast<int64_t>(rcnt.arc_scans);
  b->stats.node_updates = static_cast<int64_t>(rcnt.node_updates);
  b->stats.rounds = static_cast<int64_t>(rcnt.rounds);
  b->stats.comp_visits = static_cast<int64_t>(rcnt.comp_visits);
  for (int q = 0; q < pb::kPrSlots; ++q) b->prof[q] = static_cast<int64_t>(rcnt.prof[q]);
  b->stats.smem_walks = R.smem_ctas > 0 ? static_cast<int64_t>(N) : 0;
  b->stats.wide_walks = R.smem_ctas > 0 ? 0 : R.wide.n;
  b->stats.smem_region = R.smem_ctas > 0 ? R.smem_region : 0;
  b->stats.kernel_launches +=
      R.smem_ctas > 0 ? 1 : (R.wide.n > 0 ? 1 : 0) + (static_cast<int32_t>(N) > R.wide.n ? 1 : 0);
  if (kernel_ms) *kernel_ms = ms;
  return PB_OK;
}

pb_status fetch_impl(pb_batch* b) {
  DeviceRun& R = b->run;
  if (b->insts.empty()) {
    b->have_results = true;
    return PB_OK;
  }
  ck(cudaSetDevice(R.device), "cudaSetDevice");
  cudaEvent_t e0 = R.ex0, e1 = R.ex1;
  ck(cudaEventRecord(e0, R.stream), "record");
  ck(cudaMemcpyAsync(R.h_out, R.d_out, R.out_bytes, cudaMemcpyDeviceToHost, R.stream), "D2H out");
  unsigned long long used = 0;
  ck(cudaMemcpyAsync(&used, R.d_pool_cursor, sizeof used, cudaMemcpyDeviceToHost, R.stream), "D2H cursor");
  ck(cudaStreamSynchronize(R.stream), "sync");
  const long long nused = std::min<long long>(static_cast<long long>(used), R.pool_cap);
  b->pool_ids.resize(nused);
  b->pool_choice.resize(nused);
  if (nused) {
    ck(cudaMemcpyAsync(b->pool_ids.data(), R.d_pool_ids, sizeof(int32_t) * nused, cudaMemcpyDeviceToHost,
                       R.stream),
       "D2H pool");
    ck(cudaMemcpyAsync(b->pool_choice.data(), R.d_pool_choice, nused, cudaMemcpyDeviceToHost, R.stream),
       "D2H pool");
  }
  ck(cudaEventRecord(e1, R.stream), "record");
  ck(cudaStreamSynchronize(R.stream), "sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  b->outp = R.h_out;  // results stay in the pinned buffer until the next run
  b->stats.d2h_ms = ms;
  b->stats.d2h_bytes = static_cast<int64_t>(R.out_bytes + 5 * nused + sizeof used);
  b->have_results = true;
  return PB_OK;
}

const pb_frontier_summary& summary_of(const pb_batch* b, int32_t k) {
  return *reinterpret_cast<const pb_frontier_summary*>(b->outp + b->out_summary[k]);
}

bool any_log_full(const pb_batch* b) {
  for (size_t k = 0; k < b->insts.size(); ++k)
    if (summary_of(b, static_cast<int32_t>(k)).status == pb::kStatusLogFull) return true;
  return false;
}

template <class F>
pb_status guarded(F&& f) {
  try {
    return f();
  } catch (const CudaError& e) {
    return fail(PB_ERR_CUDA, e.what());
  } catch (const std::length_error& e) {
    return fail(PB_ERR_UNSUPPORTED, e.what());
  } catch (const std::bad_alloc&) {
    return fail(PB_ERR_CUDA, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(PB_ERR_LOGIC, e.what());
  }
}

}  // namespace

// ===================================================================== ABI

extern "C" {

const char* pb_last_error(void) { return g_last_error.c_str(); }
const char* pb_version(void) { return "perseus-b200 0.1 (sm_100a)"; }

// pareto_filter, costmodel.hpp:70-81
int32_t pb_pareto_filter(int32_t n, const int32_t* freq, const int64_t* time, const int64_t* energy,
                         int32_t* out_freq, int64_t* out_time, int64_t* out_energy) {
  struct P {
    int32_t f;
    int64_t t, e;
  };
  std::vector<P> pts(n);
  for (int32_t i = 0; i < n; ++i) pts[i] = {freq[i], time[i], energy[i]};
  std::stable_sort(pts.begin(), pts.end(), [](const P& x, const P& y) {
    if (x.t != y.t) return x.t < y.t;
    if (x.e != y.e) return x.e < y.e;
    return x.f > y.f;
  });
  int32_t k = 0;
  for (const P& p : pts)
    if (k == 0 || p.e < out_energy[k - 1]) {
      out_freq[k] = p.f;
      out_time[k] = p.t;
      out_energy[k] = p.e;
      ++k;
    }
  return k;
}

// fit_exp, costmodel.hpp:87-149: 64-point c grid, log-linear least squares.
pb_status pb_fit_exp(int32_t n, const int64_t* time, const int64_t* energy, double* out) {
  if (n < 2) return fail(PB_ERR_INVALID_ARGUMENT, "fit needs at least two points");
  std::vector<std::pair<int64_t, int64_t>> pts(n);
  for (int32_t i = 0; i < n; ++i) pts[i] = {time[i], energy[i]};
  std::stable_sort(pts.begin(), pts.end(),
                   [](const auto& x, const auto& y) { return x.first < y.first; });
  for (int32_t i = 0; i + 1 < n; ++i)
    if (pts[i].first == pts[i + 1].first) return fail(PB_ERR_INVALID_ARGUMENT, "fit needs distinct times");
  const double e_min = static_cast<double>(pts.back().second);
  const double e_max = static_cast<double>(pts.front().second);
  if (e_min == e_max) return fail(PB_ERR_DOMAIN, "all energies equal; treat the class as constant");
  if (e_min > e_max) return fail(PB_ERR_INVALID_ARGUMENT, "fit expects energy decreasing with time");
  if (n == 2) {
    const double t1 = static_cast<double>(pts[0].first), t2 = static_cast<double>(pts[1].first);
    const double e1 = static_cast<double>(pts[0].second), e2 = static_cast<double>(pts[1].second);
    const double b = std::log(e2 / e1) / (t2 - t1);
    out[0] = e1 * std::exp(-b * t1);
    out[1] = b;
    out[2] = 0.0;
    out[3] = 0.0;
    return PB_OK;
  }
  double lowest = e_min;
  for (const auto& p : pts) lowest = std::min(lowest, static_cast<double>(p.second));
  double best = -1.0;
  for (int j = 0; j < 64; ++j) {
    const double c = static_cast<double>(j) * (0.999 * lowest) / 63.0;
    double st = 0, sy = 0, stt = 0, sty = 0;
    for (const auto& p : pts) {
      const double t = static_cast<double>(p.first);
      const double y = std::log(static_cast<double>(p.second) - c);
      st += t;
      sy += y;
      stt += t * t;
      sty += t * y;
    }
    const double dn = static_cast<double>(n);
    const double slope = (dn * sty - st * sy) / (dn * stt - st * st);
    const double intercept = (sy - slope * st) / dn;
    const double a = std::exp(intercept);
    double sq = 0;
    for (const auto& p : pts) {
      const double r = a * std::exp(slope * static_cast<double>(p.first)) + c - static_cast<double>(p.second);
      sq += r * r;
    }
    const double rmse = std::sqrt(sq / dn);
    if (best < 0 || rmse < best) {
      best = rmse;
      out[0] = a;
      out[1] = slope;
      out[2] = c;
      out[3] = rmse;
    }
  }
  if (out[1] >= 0) return fail(PB_ERR_DOMAIN, "fitted exponent is not decreasing");
  return PB_OK;
}

pb_status pb_batch_create(pb_batch** out) {
  if (!out) return fail(PB_ERR_INVALID_ARGUMENT, "null handle");
  *out = new pb_batch();
  return PB_OK;
}

void pb_batch_destroy(pb_batch* b) { delete b; }

pb_status pb_batch_clear(pb_batch* b) {
  if (!b) return fail(PB_ERR_INVALID_ARGUMENT, "null handle");
  // drop the instances and results; keep the device context (stream, device
  // and pinned buffers), which the next run reuses while it fits
  b->insts.clear();
  b->tables.clear();
  b->cls_tab.clear();
  b->tab_margin.clear();
  b->out_points.clear();
  b->out_summary.clear();
  b->cap_points.clear();
  b->out.clear();
  b->outp = nullptr;
  b->pool_ids.clear();
  b->pool_choice.clear();
  b->pool_base.clear();
  b->pool_cap = 0;
  b->have_results = false;
  b->stats = pb_run_stats{};
  return PB_OK;
}

int32_t pb_batch_size(const pb_batch* b) { return b ? static_cast<int32_t>(b->insts.size()) : 0; }

pb_status pb_batch_add(pb_batch* b, const pb_instance_desc* d, int32_t* out_index) {
  if (!b || !d) return fail(PB_ERR_INVALID_ARGUMENT, "null argument");
  if (d->n < 0 || d->n_edges < 0 || d->n_classes < 0)
    return fail(PB_ERR_INVALID_ARGUMENT, "negative size");
  HostInst h;
  h.n = d->n;
  h.comp_class.assign(d->comp_class, d->comp_class + d->n);
  h.edge_tail.assign(d->edge_tail, d->edge_tail + d->n_edges);
  h.edge_head.assign(d->edge_head, d->edge_head + d->n_edges);
  h.cls_const.assign(d->class_is_constant, d->class_is_constant + d->n_classes);
  h.cls_pt_off.assign(d->class_point_off, d->class_point_off + d->n_classes + 1);
  const int32_t np = h.cls_pt_off.empty() ? 0 : h.cls_pt_off.back();
  if (!h.cls_pt_off.empty() && h.cls_pt_off.front() != 0)
    return fail(PB_ERR_INVALID_ARGUMENT, "class point offsets must start at 0");
  h.pt_freq.assign(d->point_freq, d->point_freq + np);
  h.pt_time.assign(d->point_time, d->point_time + np);
  h.pt_energy.assign(d->point_energy, d->point_energy + np);
  h.cls_curve.assign(d->class_curve, d->class_curve + 3 * d->n_classes);
  h.cls_trange.assign(d->class_t_range, d->class_t_range + 2 * d->n_classes);
  h.watts = d->blocking_watts;
  h.quantum = d->quantum_us;
  h.tau = d->tau;
  h.max_steps = d->max_steps;
  // Same DAG and cost model as the handle's last derived instance (a
  // get_next_schedule chain through the drop-in): reuse its derived layout,
  // redo only the start-dependent part
  const HostInst& c = b->derived;
  if (c.n == h.n && c.n > 0 && c.tau == h.tau && c.quantum == h.quantum && c.watts == h.watts &&
      c.comp_class == h.comp_class && c.edge_tail == h.edge_tail && c.edge_head == h.edge_head &&
      c.cls_const == h.cls_const && c.cls_pt_off == h.cls_pt_off && c.pt_freq == h.pt_freq &&
      c.pt_time == h.pt_time && c.pt_energy == h.pt_energy && c.cls_trange == h.cls_trange &&
      std::memcmp(c.cls_curve.data(), h.cls_curve.data(), sizeof(double) * h.cls_curve.size()) == 0) {
    HostInst r = c;
    if (d->start_planned_t) r.start.assign(d->start_planned_t, d->start_planned_t + d->n);
    r.max_steps = d->max_steps;
    if (!r.start.empty())
      for (int64_t t : r.start)
        if (t < 0) return fail(PB_ERR_INVALID_ARGUMENT, "durations must be non-negative");
    const pb_status s = derive_start(r);
    if (s != PB_OK) return s;
    b->insts.push_back(std::move(r));
  } else {
    if (d->start_planned_t) h.start.assign(d->start_planned_t, d->start_planned_t + d->n);
    const pb_status s = validate_and_derive(h);
    if (s != PB_OK) return s;
    ++b->derived_gen;
    h.gen = b->derived_gen;
    b->derived = h;
    b->derived.start.clear();
    b->derived.istart.clear();
    b->insts.push_back(std::move(h));
  }
  b->have_results = false;
  if (out_index) *out_index = static_cast<int32_t>(b->insts.size()) - 1;
  return PB_OK;
}

pb_status pb_batch_prepare(pb_batch* b, int32_t device) {
  if (!b) return fail(PB_ERR_INVALID_ARGUMENT, "null handle");
  return guarded([&] { return prepare_impl(b, device, 1.0); });
}

pb_status pb_batch_launch(pb_batch* b, double* kernel_ms) {
  if (!b) return fail(PB_ERR_INVALID_ARGUMENT, "null handle");
  return guarded([&] { return launch_impl(b, kernel_ms); });
}

pb_status pb_batch_fetch(pb_batch* b) {
  if (!b) return fail(PB_ERR_INVALID_ARGUMENT, "null handle");
  return guarded([&] { return fetch_impl(b); });
}

namespace {
// After a run: a single get-next walk that took its steps left its flow
// state in the carry buffer (run_walk); remember the schedule it ended in.
// Anything else (another instance, a zero-step walk, a stop) leaves the
// carry as it was or invalidates it.
void note_carry(pb_batch* b) {
  if (b->insts.size() != 1 || b->insts[0].start.empty() || b->insts[0].max_steps < 0) {
    if (b->insts.size() != 1 || b->insts[0].start.empty()) b->carry_valid = false;
    return;
  }
  const HostInst& h = b->insts[0];
  pb_frontier_summary s;
  pb_batch_summary(b, 0, &s);
  if (s.status != PB_OK || s.stop != PB_STOP_STEP_LIMIT || s.steps < 1 || !b->run.d_carry ||
      std::getenv("PB_NO_CARRY")) {
    b->carry_valid = false;
    return;
  }
  std::vector<int64_t> pt(h.n);
  pb_batch_schedule(b, 0, s.steps, pt.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  b->carry_start = std::move(pt);
  b->carry_tau = h.tau;
  b->carry_gen = h.gen;
  b->carry_valid = h.gen != 0;
}
}  // namespace

pb_status pb_batch_run(pb_batch* b, int32_t device) {
  if (!b) return fail(PB_ERR_INVALID_ARGUMENT, "null handle");
  return guarded([&] {
    double scale = 1.0;
    static const bool trace = std::getenv("PB_TRACE") != nullptr;
    for (int attempt = 0; attempt < 6; ++attempt) {
      const auto t0 = std::chrono::steady_clock::now();
      pb_status s = prepare_impl(b, device, scale);
      if (s != PB_OK) return s;
      const auto t1 = std::chrono::steady_clock::now();
      s = launch_impl(b, nullptr);
      if (s != PB_OK) return s;
      const auto t2 = std::chrono::steady_clock::now();
      s = fetch_impl(b);
      if (s != PB_OK) return s;
      if (trace) {
        const auto t3 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto z) { return std::chrono::duration<double, std::milli>(z - a).count(); };
        std::fprintf(stderr, "pb_batch_run: %zu walks, prepare %.3f ms (pack %.3f, H2D %.3f), launch %.3f ms "
                     "(kernel %.3f), fetch %.3f ms, attempt %d\n", b->insts.size(), ms(t0, t1), b->stats.pack_ms,
                     b->stats.h2d_ms, ms(t1, t2), b->stats.kernel_ms, ms(t2, t3), attempt);
      }
      if (!any_log_full(b)) {
        note_carry(b);
        return PB_OK;
      }
      scale *= 4.0;  // rare: a walk took more steps than (T* - T_min) / tau
    }
    return fail(PB_ERR_LOGIC, "delta log kept overflowing");
  });
}

pb_status pb_batch_run_multi(pb_batch* b, int32_t n_devices, const int32_t* devices) {
  if (!b || n_devices < 1 || !devices) return fail(PB_ERR_INVALID_ARGUMENT, "bad device list");
  if (n_devices == 1) return pb_batch_run(b, devices[0]);
  return guarded([&]() -> pb_status {
    // LPT over devices by estimated work; one sub-batch and host thread each.
    const size_t N = b->insts.size();
    std::vector<size_t> idx(N);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(),
                     [&](size_t x, size_t y) { return b->insts[x].work > b->insts[y].work; });
    std::vector<int64_t> load(n_devices, 0);
    std::vector<std::vector<size_t>> part(n_devices);
    for (size_t k : idx) {
      const int d = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
      load[d] += b->insts[k].work;
      part[d].push_back(k);
    }
    std::vector<pb_batch> subs(n_devices);
    std::vector<pb_status> st(n_devices, PB_OK);
    std::vector<std::string> msg(n_devices);  // g_last_error is thread_local: carry it back
    std::vector<std::thread> th;
    for (int d = 0; d < n_devices; ++d) {
      for (size_t k : part[d]) subs[d].insts.push_back(b->insts[k]);
      th.emplace_back([&, d] {
        st[d] = pb_batch_run(&subs[d], devices[d]);
        if (st[d] != PB_OK) msg[d] = g_last_error;
      });
    }
    for (auto& t : th) t.join();
    for (int d = 0; d < n_devices; ++d)
      if (st[d] != PB_OK) return fail(st[d], "device " + std::to_string(devices[d]) + ": " + msg[d]);
    // stitch results back in the original order
    b->run.release();
    b->carry_valid = false;
    std::vector<char> out;
    b->out_points.assign(N, 0);
    b->out_summary.assign(N, 0);
    b->pool_base.assign(N, 0);
    b->cap_points.assign(N, 0);
    b->pool_ids.clear();
    b->pool_choice.clear();
    b->cls_tab.assign(N, {});
    b->tables.clear();
    b->stats = pb_run_stats{};
    for (int d = 0; d < n_devices; ++d) {
      const pb_batch& s = subs[d];
      // the sub-batch's results live in its pinned buffer (fetch_impl), valid
      // while `subs` is alive: copy them, keeping 256 B alignment
      const size_t base = (out.size() + 255) / 256 * 256;
      const long long pbase = static_cast<long long>(b->pool_ids.size());
      out.resize(base);
      if (!s.insts.empty()) out.insert(out.end(), s.outp, s.outp + s.run.out_bytes);
      b->pool_ids.insert(b->pool_ids.end(), s.pool_ids.begin(), s.pool_ids.end());
      b->pool_choice.insert(b->pool_choice.end(), s.pool_choice.begin(), s.pool_choice.end());
      const int64_t tbase = static_cast<int64_t>(b->tables.size());
      b->tables.insert(b->tables.end(), s.tables.begin(), s.tables.end());
      for (size_t q = 0; q < part[d].size(); ++q) {
        const size_t k = part[d][q];
        b->out_points[k] = base + s.out_points[q];
        b->out_summary[k] = base + s.out_summary[q];
        b->pool_base[k] = pbase + s.pool_base[q];
        b->cap_points[k] = s.cap_points[q];
        b->cls_tab[k] = s.cls_tab[q];
        for (auto& t : b->cls_tab[k]) t += tbase;
      }
      b->stats.kernel_ms = std::max(b->stats.kernel_ms, s.stats.kernel_ms);
      b->stats.h2d_bytes += s.stats.h2d_bytes;
      b->stats.d2h_bytes += s.stats.d2h_bytes;
      b->stats.arc_scans += s.stats.arc_scans;
      b->stats.node_updates += s.stats.node_updates;
      b->stats.rounds += s.stats.rounds;
      b->stats.comp_visits += s.stats.comp_visits;
      b->stats.kernel_launches += s.stats.kernel_launches;
      b->stats.smem_walks += s.stats.smem_walks;
      b->stats.wide_walks += s.stats.wide_walks;
      b->stats.smem_region = std::max(b->stats.smem_region, s.stats.smem_region);
    }
    b->out = std::move(out);
    b->outp = b->out.data();
    b->have_results = true;
    return PB_OK;
  });
}

pb_status pb_batch_summary(const pb_batch* b, int32_t k, pb_frontier_summary* out) {
  if (!b || !out || k < 0 || k >= static_cast<int32_t>(b->insts.size()))
    return fail(PB_ERR_INVALID_ARGUMENT, "bad instance index");
  if (!b->have_results) return fail(PB_ERR_LOGIC, "batch has not been run");
  *out = summary_of(b, k);
  return PB_OK;
}

pb_status pb_batch_points(const pb_batch* b, int32_t k, pb_point* out, int32_t capacity) {
  pb_frontier_summary s;
  pb_status st = pb_batch_summary(b, k, &s);
  if (st != PB_OK) return st;
  const int32_t np = s.steps + 1;
  if (capacity < np) return fail(PB_ERR_INVALID_ARGUMENT, "points buffer too small");
  std::memcpy(out, b->outp + b->out_points[k], sizeof(pb_point) * np);
  // id_begin: pool offsets on the device -> offsets into pb_batch_deltas()
  int32_t acc = 0;
  for (int32_t q = 1; q < np; ++q) {
    out[q].id_begin = acc;
    acc += out[q].n_sped + out[q].n_slowed;
  }
  return PB_OK;
}

pb_status pb_batch_deltas(const pb_batch* b, int32_t k, int32_t* ids, uint8_t* choice,
                          int32_t capacity) {
  pb_frontier_summary s;
  pb_status st = pb_batch_summary(b, k, &s);
  if (st != PB_OK) return st;
  if (capacity < s.n_ids) return fail(PB_ERR_INVALID_ARGUMENT, "delta buffer too small");
  const pb_point* pts = reinterpret_cast<const pb_point*>(b->outp + b->out_points[k]);
  int32_t j = 0;
  for (int32_t q = 1; q <= s.steps; ++q) {
    const long long at = b->pool_base[k] + pts[q].id_begin;
    const int32_t cnt = pts[q].n_sped + pts[q].n_slowed;
    for (int32_t r = 0; r < cnt; ++r, ++j) {
      if (ids) ids[j] = b->pool_ids[at + r];
      if (choice) choice[j] = b->pool_choice[at + r];
    }
  }
  return PB_OK;
}

// 64-bit digest of one walk's outputs: summary, every point's scalars (not
// the device pool offsets, which depend on the order of concurrent
// reservations) and the delta records in step order.
pb_status pb_batch_digest(const pb_batch* b, int32_t k, uint64_t* out) {
  pb_frontier_summary s;
  const pb_status st = pb_batch_summary(b, k, &s);
  if (st != PB_OK) return st;
  if (!out) return fail(PB_ERR_INVALID_ARGUMENT, "null argument");
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    h ^= v;
    h *= 1099511628211ull;
    h ^= h >> 29;
  };
  for (int64_t v : {s.t_min, s.t_star, int64_t{s.steps}, int64_t{s.stop}, int64_t{s.status}, int64_t{s.n_ids}})
    mix(static_cast<uint64_t>(v));
  const pb_point* pts = reinterpret_cast<const pb_point*>(b->outp + b->out_points[k]);
  const int32_t np = s.status == PB_OK ? s.steps + 1 : 0;
  for (int32_t q = 0; q < np; ++q) {
    const pb_point& p = pts[q];
    for (int64_t v : {p.t_planned, p.t_realized, p.sum_planned_e, p.sum_planned_t, p.sum_realized_e,
                      p.sum_realized_t, p.cut_cost, p.step_size, int64_t{p.n_sped}, int64_t{p.n_slowed}})
      mix(static_cast<uint64_t>(v));
    if (q == 0) continue;
    const long long at = b->pool_base[k] + p.id_begin;
    for (int32_t r = 0; r < p.n_sped + p.n_slowed; ++r)
      mix((static_cast<uint64_t>(static_cast<uint32_t>(b->pool_ids[at + r])) << 8) | b->pool_choice[at + r]);
  }
  *out = h;
  return PB_OK;
}

}  // extern "C"

namespace {

// Replays instance k's delta log point by point (caller ids) and
// materializes EnergySchedule fields (frontier.hpp:20-33) at any point.
struct Replay {
  const pb_batch* b;
  int32_t k;
  const HostInst& h;
  const pb_point* pts;
  const int32_t* ids;
  const uint8_t* cho;
  std::vector<int64_t> pt;
  std::vector<int32_t> ch;
  int32_t at = 0;

  Replay(const pb_batch* bb, int32_t kk)
      : b(bb), k(kk), h(bb->insts[kk]),
        pts(reinterpret_cast<const pb_point*>(bb->outp + bb->out_points[kk])),
        ids(bb->pool_ids.data() + bb->pool_base[kk]), cho(bb->pool_choice.data() + bb->pool_base[kk]) {
    const int32_t n = h.n;
    pt.resize(n);
    ch.resize(n);
    for (int32_t i = 0; i < n; ++i) {
      const int32_t c = h.comp_class[i];
      pt[i] = !h.start.empty() ? h.start[i] : (h.cls_const[c] ? h.pt_time[h.cls_pt_off[c]] : h.cls_trange[2 * c + 1]);
      int32_t chosen = 0;  // discretize (frontier.hpp:146-156)
      for (int32_t p = h.cls_pt_off[c]; p < h.cls_pt_off[c + 1]; ++p)
        if (h.pt_time[p] <= pt[i]) chosen = p - h.cls_pt_off[c];
      ch[i] = chosen;
    }
  }
  void advance_to(int32_t which) {
    for (; at < which; ++at) {
      const pb_point& p = pts[at + 1];
      const int32_t cnt = p.n_sped + p.n_slowed;
      for (int32_t j = p.id_begin; j < p.id_begin + cnt; ++j) {
        const int32_t x = ids[j];
        const int32_t i = (x > 0 ? x : -x) - 1;
        pt[i] += x > 0 ? -p.step_size : p.step_size;
        ch[i] = cho[j];
      }
    }
  }
  int64_t planned_energy(int32_t i) const {  // frontier.hpp:59-62
    const int32_t c = h.comp_class[i];
    if (h.cls_const[c]) return h.pt_energy[h.cls_pt_off[c]];
    const int64_t lo = h.cls_trange[2 * c], hi = h.cls_trange[2 * c + 1], t = pt[i];
    const double v = (t >= lo && t <= hi) ? b->tables[b->cls_tab[k][c] + (t - lo)]
                                          : h.cls_curve[3 * c] * std::exp(h.cls_curve[3 * c + 1] * static_cast<double>(t)) +
                                                h.cls_curve[3 * c + 2];
    return static_cast<int64_t>(std::llround(v));
  }
  // effective_total (frontier.hpp:51-57; units.hpp:38-48), index order
  void totals(double& effp, double& effr) const {
    effp = 0;
    effr = 0;
    for (int32_t i = 0; i < h.n; ++i) {
      const int32_t p = h.cls_pt_off[h.comp_class[i]] + ch[i];
      effp += static_cast<double>(planned_energy(i)) -
              h.watts * static_cast<double>(pt[i]) * static_cast<double>(h.quantum) * 1e-3;
      effr += static_cast<double>(h.pt_energy[p]) -
              h.watts * static_cast<double>(h.pt_time[p]) * static_cast<double>(h.quantum) * 1e-3;
    }
  }
};

pb_status check_index(const pb_batch* b, int32_t k, int32_t which) {
  pb_frontier_summary s;
  const pb_status st = pb_batch_summary(b, k, &s);
  if (st != PB_OK) return st;
  if (which < 0 || which > s.steps) return fail(PB_ERR_INVALID_ARGUMENT, "schedule index out of range");
  return PB_OK;
}

// nlohmann::json's number layout for a double (shortest round-trip digits;
// fixed notation for decimal exponents in (-4, 15], else d.ddde+XX; ".0" on
// integral values), as serde.hpp's dump() writes round3 values.
std::string json_double(double v) {
  if (v == 0) return std::signbit(v) ? "-0.0" : "0.0";
  char sci[64];
  const auto r = std::to_chars(sci, sci + sizeof sci, v, std::chars_format::scientific);
  std::string t(sci, r.ptr);
  std::string out;
  if (t[0] == '-') {
    out = "-";
    t = t.substr(1);
  }
  const size_t epos = t.find('e');
  std::string digits = t.substr(0, epos);
  const int e10 = std::stoi(t.substr(epos + 1));
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int len = static_cast<int>(digits.size());
  const int n = e10 + 1;  // position of the decimal point
  if (len <= n && n <= 15) {
    out += digits + std::string(n - len, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (len > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += eb;
  }
  return out;
}

double round3(double v) { return std::round(v * 1000.0) / 1000.0; }  // serde.hpp:30

pb_status emit(const std::string& text, char* buf, int64_t cap, int64_t* len) {
  if (len) *len = static_cast<int64_t>(text.size());
  if (buf) {
    if (cap < static_cast<int64_t>(text.size())) return fail(PB_ERR_INVALID_ARGUMENT, "output buffer too small");
    std::memcpy(buf, text.data(), text.size());
  }
  return PB_OK;
}

}  // namespace

extern "C" {

pb_status pb_batch_schedule(const pb_batch* b, int32_t k, int32_t which, int64_t* planned_t,
                            int64_t* planned_e, int32_t* freq_mhz, int64_t* realized_t,
                            int64_t* realized_e, double* eff_planned, double* eff_realized) {
  const pb_status st = check_index(b, k, which);
  if (st != PB_OK) return st;
  Replay r(b, k);
  r.advance_to(which);
  const HostInst& h = r.h;
  for (int32_t i = 0; i < h.n; ++i) {
    const int32_t p = h.cls_pt_off[h.comp_class[i]] + r.ch[i];
    if (planned_t) planned_t[i] = r.pt[i];
    if (planned_e) planned_e[i] = r.planned_energy(i);
    if (freq_mhz) freq_mhz[i] = h.pt_freq[p];
    if (realized_t) realized_t[i] = h.pt_time[p];
    if (realized_e) realized_e[i] = h.pt_energy[p];
  }
  double effp, effr;
  r.totals(effp, effr);
  if (eff_planned) *eff_planned = effp;
  if (eff_realized) *eff_realized = effr;
  return PB_OK;
}

pb_status pb_batch_schedules(const pb_batch* b, int32_t k, int32_t first, int32_t count, int64_t* planned_t,
                             int64_t* planned_e, int32_t* freq_mhz, int64_t* realized_t, int64_t* realized_e,
                             double* eff_planned, double* eff_realized) {
  if (count < 0) return fail(PB_ERR_INVALID_ARGUMENT, "negative count");
  if (count == 0) return check_index(b, k, 0);
  pb_status st = check_index(b, k, first);
  if (st == PB_OK) st = check_index(b, k, first + count - 1);
  if (st != PB_OK) return st;
  Replay r(b, k);  // one incremental replay for the whole range
  const HostInst& h = r.h;
  const size_t n = static_cast<size_t>(h.n);
  for (int32_t q = 0; q < count; ++q) {
    r.advance_to(first + q);
    const size_t o = static_cast<size_t>(q) * n;
    for (int32_t i = 0; i < h.n; ++i) {
      const int32_t p = h.cls_pt_off[h.comp_class[i]] + r.ch[i];
      if (planned_t) planned_t[o + i] = r.pt[i];
      if (planned_e) planned_e[o + i] = r.planned_energy(i);
      if (freq_mhz) freq_mhz[o + i] = h.pt_freq[p];
      if (realized_t) realized_t[o + i] = h.pt_time[p];
      if (realized_e) realized_e[o + i] = h.pt_energy[p];
    }
    if (eff_planned || eff_realized) {
      double effp, effr;
      r.totals(effp, effr);
      if (eff_planned) eff_planned[q] = effp;
      if (eff_realized) eff_realized[q] = effr;
    }
  }
  return PB_OK;
}

pb_status pb_batch_frontier_csv(const pb_batch* b, int32_t k, int64_t quantum_us, char* buf, int64_t cap,
                                int64_t* len) {
  const pb_status st = check_index(b, k, 0);
  if (st != PB_OK) return st;
  pb_frontier_summary s;
  pb_batch_summary(b, k, &s);
  Replay r(b, k);
  std::string out = "t_planned_us,t_realized_us,energy_planned_mj,energy_realized_mj,schedule_id\n";
  char line[160];
  for (int32_t q = 0; q <= s.steps; ++q) {
    r.advance_to(q);
    double effp, effr;
    r.totals(effp, effr);
    std::snprintf(line, sizeof line, "%lld,%lld,%.3f,%.3f,%d\n",
                  static_cast<long long>(r.pts[q].t_planned * quantum_us),
                  static_cast<long long>(r.pts[q].t_realized * quantum_us), effp, effr, q);
    out += line;
  }
  return emit(out, buf, cap, len);
}

pb_status pb_batch_schedule_json(const pb_batch* b, int32_t k, int32_t which, int64_t quantum_us, char* buf,
                                 int64_t cap, int64_t* len) {
  const pb_status st = check_index(b, k, which);
  if (st != PB_OK) return st;
  Replay r(b, k);
  r.advance_to(which);
  double effp, effr;
  r.totals(effp, effr);
  const HostInst& h = r.h;
  std::string o;
  o.reserve(64 + 200 * static_cast<size_t>(h.n));
  auto i64 = [](int64_t v) { return std::to_string(v); };
  o += "{\n  \"schedule_id\": " + std::to_string(which) + ",\n";
  o += "  \"t_planned_us\": " + i64(r.pts[which].t_planned * quantum_us) + ",\n";
  o += "  \"eff_planned_mj\": " + json_double(round3(effp)) + ",\n";
  o += "  \"t_realized_us\": " + i64(r.pts[which].t_realized * quantum_us) + ",\n";
  o += "  \"eff_realized_mj\": " + json_double(round3(effr)) + ",\n";
  o += "  \"computations\": [";
  for (int32_t i = 0; i < h.n; ++i) {
    const int32_t p = h.cls_pt_off[h.comp_class[i]] + r.ch[i];
    o += i ? ",\n    {\n" : "\n    {\n";
    o += "      \"id\": " + std::to_string(i) + ",\n";
    o += "      \"freq_mhz\": " + std::to_string(h.pt_freq[p]) + ",\n";
    o += "      \"t_planned_us\": " + i64(r.pt[i] * quantum_us) + ",\n";
    o += "      \"e_planned_mj\": " + i64(r.planned_energy(i)) + ",\n";
    o += "      \"t_realized_us\": " + i64(h.pt_time[p] * quantum_us) + ",\n";
    o += "      \"e_realized_mj\": " + i64(h.pt_energy[p]) + "\n    }";
  }
  o += h.n ? "\n  ]\n}\n" : "]\n}\n";
  return emit(o, buf, cap, len);
}

pb_status pb_batch_profile(const pb_batch* b, int64_t* out, int32_t n) {
  if (!b || !out) return fail(PB_ERR_INVALID_ARGUMENT, "null argument");
  for (int32_t q = 0; q < n && q < pb::kPrSlots; ++q) out[q] = b->prof[q];
  return PB_OK;
}

pb_status pb_batch_stats(const pb_batch* b, pb_run_stats* out) {
  if (!b || !out) return fail(PB_ERR_INVALID_ARGUMENT, "null argument");
  *out = b->stats;
  return PB_OK;
}

// ------------------------------------------------------- straggler sweep

pb_status pb_batch_straggler(pb_batch* b, int32_t n_factors, const double* factors, int32_t pipelines,
                             const int32_t* num_stages, pb_savings_row* out) {
  if (!b || n_factors < 0 || (n_factors && (!factors || !out)) || !num_stages)
    return fail(PB_ERR_INVALID_ARGUMENT, "null argument");
  if (pipelines < 1) return fail(PB_ERR_INVALID_ARGUMENT, "need at least one pipeline");
  for (int32_t j = 0; j < n_factors; ++j)
    if (!(factors[j] >= 1.0)) return fail(PB_ERR_INVALID_ARGUMENT, "straggler factor must be >= 1");
  if (!b->have_results || b->run.device < 0)
    return fail(PB_ERR_LOGIC, "pb_batch_run the batch on one device first");
  const int32_t N = static_cast<int32_t>(b->insts.size());
  if (N == 0 || n_factors == 0) return PB_OK;
  return guarded([&]() -> pb_status {
    DeviceRun& R = b->run;
    ck(cudaSetDevice(R.device), "cudaSetDevice");
    std::vector<pb::DevStraggler> jobs(N);
    for (int32_t k = 0; k < N; ++k) {
      const HostInst& h = b->insts[k];
      pb::DevStraggler& J = jobs[k];
      J.points = reinterpret_cast<const pb_point*>(R.d_out + b->out_points[k]);
      J.summary = reinterpret_cast<const pb_frontier_summary*>(R.d_out + b->out_summary[k]);
      J.am_energy = 0;
      J.am_time = 0;
      for (int32_t i = 0; i < h.n; ++i) {  // all_max_assignment (emulator.hpp:140-149)
        const int32_t p0 = h.cls_pt_off[h.comp_class[i]];
        J.am_energy += h.pt_energy[p0];
        J.am_time += h.pt_time[p0];
      }
      J.watts = h.watts;
      J.quantum = h.quantum;
      J.stages = num_stages[k];
      J.pad = 0;
      if (num_stages[k] < 1) return fail(PB_ERR_INVALID_ARGUMENT, "num_stages must be positive");
    }
    const size_t rows = static_cast<size_t>(N) * n_factors;
    DevBuf<pb::DevStraggler> d_jobs(N, "malloc straggler jobs");
    DevBuf<double> d_f(n_factors, "malloc factors");
    DevBuf<pb_savings_row> d_out(rows, "malloc savings rows");
    ck(cudaMemcpyAsync(d_jobs.p, jobs.data(), sizeof(pb::DevStraggler) * N, cudaMemcpyHostToDevice, R.stream), "H2D");
    ck(cudaMemcpyAsync(d_f.p, factors, sizeof(double) * n_factors, cudaMemcpyHostToDevice, R.stream), "H2D");
    const int rc = pb::launch_straggler(d_jobs.p, N, d_f.p, n_factors, pipelines, d_out.p, R.stream);
    if (rc) throw CudaError(cudaGetErrorString(static_cast<cudaError_t>(rc)));
    ck(cudaMemcpyAsync(out, d_out.p, sizeof(pb_savings_row) * rows, cudaMemcpyDeviceToHost, R.stream), "D2H");
    ck(cudaStreamSynchronize(R.stream), "straggler kernel");
    return PB_OK;
  });
}

// ------------------------------------------------------- exhaustive oracle

pb_status pb_batch_brute_force(pb_batch* b, int32_t k, double budget, int32_t device, pb_exact_point* points,
                               int32_t* freq_mhz, int32_t capacity, int32_t* count) {
  if (!b || !count || k < 0 || k >= static_cast<int32_t>(b->insts.size()))
    return fail(PB_ERR_INVALID_ARGUMENT, "bad instance index");
  const HostInst& h = b->insts[k];
  const int32_t n = h.n;
  // mixed radix over caller ids, last computation fastest (oracle.hpp:53-66)
  double combos = 1;
  std::vector<int32_t> radix(n), poff(n);
  for (int32_t j = 0; j < n; ++j) {
    const int32_t c = h.comp_class[j];
    poff[j] = h.cls_pt_off[c];
    radix[j] = h.cls_pt_off[c + 1] - h.cls_pt_off[c];
    combos *= radix[j];
    if (combos > budget) return fail(PB_ERR_BUDGET, "assignment space exceeds the enumeration budget");
  }
  if (n > 64) return fail(PB_ERR_UNSUPPORTED, "brute force supports at most 64 computations");
  std::vector<int64_t> stride(n, 1);
  for (int32_t j = n - 2; j >= 0; --j) stride[j] = stride[j + 1] * radix[j + 1];
  // iteration-time range: all fastest .. all slowest (points ascending in time)
  std::vector<int64_t> lo(n), hi(n);
  for (int32_t i = 0; i < n; ++i) {
    const int32_t j = h.orig[i];
    lo[i] = h.pt_time[poff[j]];
    hi[i] = h.pt_time[poff[j] + radix[j] - 1];
  }
  const int64_t t_lo = host_makespan(h, lo), t_hi = host_makespan(h, hi);
  const int64_t slots = t_hi - t_lo + 1;
  if (slots > (int64_t{1} << 25)) return fail(PB_ERR_UNSUPPORTED, "iteration-time range too wide to tabulate");
  return guarded([&]() -> pb_status {
    ck(cudaSetDevice(device), "cudaSetDevice");
    Blob blob;
    const size_t o_orig = blob.put(h.orig), o_pinoff = blob.put(h.pin_off), o_pin = blob.put(h.pin),
                 o_cflag = blob.put(h.cflag), o_stride = blob.put(stride), o_radix = blob.put(radix),
                 o_poff = blob.put(poff), o_pt = blob.put(h.pt_time), o_pe = blob.put(h.pt_energy);
    char* d_blob = nullptr;
    unsigned long long *d_e = nullptr, *d_c = nullptr;
    pb::DevBrute* d_job = nullptr;
    ck(cudaMalloc(&d_blob, std::max<size_t>(blob.bytes.size(), 256)), "malloc");
    ck(cudaMalloc(&d_e, sizeof(unsigned long long) * slots), "malloc");
    ck(cudaMalloc(&d_c, sizeof(unsigned long long) * slots), "malloc");
    ck(cudaMalloc(&d_job, sizeof(pb::DevBrute)), "malloc");
    ck(cudaMemcpy(d_blob, blob.bytes.data(), blob.bytes.size(), cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemset(d_e, 0xff, sizeof(unsigned long long) * slots), "memset");
    ck(cudaMemset(d_c, 0xff, sizeof(unsigned long long) * slots), "memset");
    pb::DevBrute J{};
    J.n = n;
    J.combos = static_cast<int64_t>(combos);
    J.t_lo = t_lo;
    J.slots = slots;
    J.watts = h.watts;
    J.quantum = h.quantum;
    J.orig = dptr<int32_t>(d_blob, o_orig);
    J.pin_off = dptr<int32_t>(d_blob, o_pinoff);
    J.pin = dptr<int32_t>(d_blob, o_pin);
    J.cflag = dptr<uint8_t>(d_blob, o_cflag);
    J.stride = dptr<int64_t>(d_blob, o_stride);
    J.radix = dptr<int32_t>(d_blob, o_radix);
    J.poff = dptr<int32_t>(d_blob, o_poff);
    J.pt_time = dptr<int64_t>(d_blob, o_pt);
    J.pt_energy = dptr<int64_t>(d_blob, o_pe);
    J.best_e = d_e;
    J.best_code = d_c;
    ck(cudaMemcpy(d_job, &J, sizeof J, cudaMemcpyHostToDevice), "H2D");
    for (int pass = 0; pass < 2; ++pass) {
      const int rc = pb::launch_brute(d_job, J, pass, nullptr);
      if (rc) throw CudaError(cudaGetErrorString(static_cast<cudaError_t>(rc)));
    }
    ck(cudaDeviceSynchronize(), "brute kernel");
    std::vector<unsigned long long> be(slots), bc(slots);
    ck(cudaMemcpy(be.data(), d_e, sizeof(unsigned long long) * slots, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(bc.data(), d_c, sizeof(unsigned long long) * slots, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(d_blob);
    cudaFree(d_e);
    cudaFree(d_c);
    cudaFree(d_job);
    // ascending time, strictly decreasing energy (oracle.hpp:96-112)
    int32_t cnt = 0;
    bool have = false;
    double best = 0;
    for (int64_t s = 0; s < slots; ++s) {
      if (bc[s] == ~0ull) continue;
      const unsigned long long key = be[s];
      const unsigned long long u = (key >> 63) ? (key & ~0x8000000000000000ull) : ~key;
      double e;
      std::memcpy(&e, &u, 8);
      if (have && e >= best) continue;
      best = e;
      have = true;
      if (cnt < capacity && points) {
        points[cnt] = pb_exact_point{t_lo + s, e, static_cast<int64_t>(bc[s])};
        if (freq_mhz) {
          int64_t c = static_cast<int64_t>(bc[s]);
          for (int32_t j = 0; j < n; ++j) {
            const int32_t d = static_cast<int32_t>(c / stride[j]);
            c %= stride[j];
            freq_mhz[static_cast<size_t>(cnt) * n + j] = h.pt_freq[poff[j] + d];
          }
        }
      }
      ++cnt;
    }
    *count = cnt;
    return cnt <= capacity || !points ? PB_OK : fail(PB_ERR_INVALID_ARGUMENT, "points buffer too small");
  });
}

// ------------------------------------------------------- component kernels

pb_status pb_annotate_slack_batch(int32_t device, int32_t count, const int32_t* n, const int32_t* ne,
                                  const int32_t* edge_tail, const int32_t* edge_head,
                                  const int64_t* durations, int64_t* earliest, int64_t* latest,
                                  uint8_t* critical, int64_t* makespan) {
  return guarded([&]() -> pb_status {
    if (count <= 0) return PB_OK;
    std::vector<HostInst> hs(count);
    size_t eo = 0, dofs = 0;
    for (int32_t g = 0; g < count; ++g) {
      HostInst& h = hs[g];
      h.n = n[g];
      h.edge_tail.assign(edge_tail + eo, edge_tail + eo + ne[g]);
      h.edge_head.assign(edge_head + eo, edge_head + eo + ne[g]);
      eo += ne[g];
      // one constant class so that validation passes; durations come separately
      h.comp_class.assign(h.n, 0);
      h.cls_const = {1};
      h.cls_pt_off = {0, 1};
      h.pt_freq = {1};
      h.pt_time = {0};
      h.pt_energy = {1};
      h.cls_curve = {0, 0, 0};
      h.cls_trange = {0, 0};
      for (int32_t i = 0; i < h.n; ++i)
        if (durations[dofs + i] < 0) return fail(PB_ERR_INVALID_ARGUMENT, "durations must be non-negative");
      dofs += h.n;
      const pb_status s = validate_and_derive(h);
      if (s != PB_OK) return s;
    }
    ck(cudaSetDevice(device), "cudaSetDevice");
    Blob blob;
    std::vector<std::array<size_t, 32>> off(count);
    size_t out_e = 0, out_c = 0;
    std::vector<size_t> o_e(count), o_c(count), o_d(count);
    int64_t max_n = 1, max_v = 1, max_e = 1;
    dofs = 0;
    for (int32_t g = 0; g < count; ++g) {
      const HostInst& h = hs[g];
      put_static(blob, h, off[g]);
      o_d[g] = blob.put(durations + dofs, sizeof(int64_t) * h.n);
      dofs += h.n;
      o_e[g] = out_e;
      out_e += 2 * h.n + 2;
      o_c[g] = out_c;
      out_c += h.n + h.edge_tail.size();
      max_n = std::max<int64_t>(max_n, h.n);
      max_v = std::max<int64_t>(max_v, 2 * int64_t{h.n} + 2);
      max_e = std::max<int64_t>(max_e, h.n + static_cast<int64_t>(h.edge_tail.size()) + 1);
    }
    char *d_blob = nullptr, *d_ws = nullptr;
    int64_t *d_e = nullptr, *d_l = nullptr, *d_ms = nullptr;
    uint8_t* d_c = nullptr;
    pb::DevInst* d_insts = nullptr;
    pb::SlackOut* d_outs = nullptr;
    const pb::WsLayout ws = pb::make_ws_layout(max_n, max_v, max_e);
    const int32_t slots = std::min<int32_t>(count, 1024);
    ck(cudaMalloc(&d_blob, std::max<size_t>(blob.bytes.size(), 256)), "malloc");
    ck(cudaMalloc(&d_e, sizeof(int64_t) * out_e), "malloc");
    ck(cudaMalloc(&d_l, sizeof(int64_t) * out_e), "malloc");
    ck(cudaMalloc(&d_c, std::max<size_t>(out_c, 1)), "malloc");
    ck(cudaMalloc(&d_ms, sizeof(int64_t) * count), "malloc");
    ck(cudaMalloc(&d_ws, static_cast<size_t>(ws.stride) * slots), "malloc");
    ck(cudaMalloc(&d_insts, sizeof(pb::DevInst) * count), "malloc");
    ck(cudaMalloc(&d_outs, sizeof(pb::SlackOut) * count), "malloc");
    ck(cudaMemcpy(d_blob, blob.bytes.data(), blob.bytes.size(), cudaMemcpyHostToDevice), "H2D");
    std::vector<pb::DevInst> di(count);
    std::vector<pb::SlackOut> so(count);
    for (int32_t g = 0; g < count; ++g) {
      const HostInst& h = hs[g];
      pb::DevInst& d = di[g];
      fill_shape(d, h);
      bind_static(d, d_blob, off[g]);
      so[g].dur = dptr<int64_t>(d_blob, o_d[g]);
      so[g].earliest = d_e + o_e[g];
      so[g].latest = d_l + o_e[g];
      so[g].critical = d_c + o_c[g];
    }
    ck(cudaMemcpy(d_insts, di.data(), sizeof(pb::DevInst) * count, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(d_outs, so.data(), sizeof(pb::SlackOut) * count, cudaMemcpyHostToDevice), "H2D");
    const int rc = pb::launch_slack_jobs(d_insts, d_outs, d_ms, count, d_ws, ws, slots, nullptr);
    if (rc) throw CudaError(cudaGetErrorString(static_cast<cudaError_t>(rc)));
    ck(cudaDeviceSynchronize(), "slack kernel");
    ck(cudaMemcpy(earliest, d_e, sizeof(int64_t) * out_e, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(latest, d_l, sizeof(int64_t) * out_e, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(critical, d_c, out_c, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(makespan, d_ms, sizeof(int64_t) * count, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(d_blob);
    cudaFree(d_e);
    cudaFree(d_l);
    cudaFree(d_c);
    cudaFree(d_ms);
    cudaFree(d_ws);
    cudaFree(d_insts);
    cudaFree(d_outs);
    return PB_OK;
  });
}

pb_status pb_flow_min_cut_batch(int32_t device, int32_t count, const int32_t* nodes,
                                const int32_t* source, const int32_t* sink, const int32_t* m,
                                const int32_t* tail, const int32_t* head, const int64_t* lower,
                                const int64_t* upper, const uint8_t* infinite, int32_t* status,
                                uint8_t* feasible, int64_t* value, int64_t* sentinel,
                                int64_t* cost, uint8_t* source_side, int8_t* cut_dir) {
  return guarded([&]() -> pb_status {
    if (count <= 0) return PB_OK;
    // validation mirrors FlowGraph (flow.hpp:34-50, 71-77)
    size_t eo = 0, no = 0;
    for (int32_t g = 0; g < count; ++g) {
      if (nodes[g] < 2) return fail(PB_ERR_INVALID_ARGUMENT, "flow graph needs at least two nodes");
      if (source[g] == sink[g] || source[g] < 0 || sink[g] < 0 || source[g] >= nodes[g] || sink[g] >= nodes[g])
        return fail(PB_ERR_INVALID_ARGUMENT, "invalid source/sink");
      for (int32_t e = 0; e < m[g]; ++e) {
        const size_t k = eo + e;
        if (tail[k] < 0 || head[k] < 0 || tail[k] >= nodes[g] || head[k] >= nodes[g])
          return fail(PB_ERR_INVALID_ARGUMENT, "edge endpoint out of range");
        if (tail[k] == head[k]) return fail(PB_ERR_INVALID_ARGUMENT, "self-loops not allowed");
        if (lower[k] < 0) return fail(PB_ERR_INVALID_ARGUMENT, "negative lower bound");
        if (!infinite[k] && upper[k] < lower[k]) return fail(PB_ERR_INVALID_ARGUMENT, "upper bound below lower bound");
      }
      eo += m[g];
      no += nodes[g];
    }
    ck(cudaSetDevice(device), "cudaSetDevice");
    Blob blob;
    std::vector<std::array<size_t, 8>> off(count);
    std::vector<int2h_pair> rets(count);
    int64_t max_v = 2, max_e = 1;
    eo = 0;
    for (int32_t g = 0; g < count; ++g) {
      const int32_t V = nodes[g], M = m[g];
      std::vector<int32_t> t(tail + eo, tail + eo + M), h(head + eo, head + eo + M);
      t.push_back(sink[g]);
      h.push_back(source[g]);
      pb::NetLayout net;
      pb::build_net(V, t, h, net);
      rets[g] = {net.epos[M].x, net.epos[M].y};
      t.pop_back();
      h.pop_back();
      off[g][0] = blob.put(net.inc_off);
      off[g][1] = blob.put(net.ient);
      off[g][2] = blob.put(t);
      off[g][3] = blob.put(h);
      off[g][4] = blob.put(lower + eo, sizeof(int64_t) * M);
      off[g][5] = blob.put(upper + eo, sizeof(int64_t) * M);
      off[g][6] = blob.put(infinite + eo, M);
      off[g][7] = blob.put(net.epos);
      max_v = std::max<int64_t>(max_v, V);
      max_e = std::max<int64_t>(max_e, M + 1);
      eo += M;
    }
    const size_t E = eo, NV = no;
    char *d_blob = nullptr, *d_ws = nullptr, *d_out = nullptr;
    pb::DevFlowJob* d_jobs = nullptr;
    // outputs: status, feasible, value, sentinel, cost, side, cut_dir
    Blob outl;
    const size_t o_st = outl.put(nullptr, 4 * count), o_fe = outl.put(nullptr, count),
                 o_va = outl.put(nullptr, 8 * count), o_se = outl.put(nullptr, 8 * count),
                 o_co = outl.put(nullptr, 8 * count), o_si = outl.put(nullptr, std::max<size_t>(NV, 1)),
                 o_cd = outl.put(nullptr, std::max<size_t>(E, 1));
    const pb::WsLayout ws = pb::make_ws_layout(1, max_v, max_e);
    const int32_t slots = std::min<int32_t>(count, 1024);
    ck(cudaMalloc(&d_blob, std::max<size_t>(blob.bytes.size(), 256)), "malloc");
    ck(cudaMalloc(&d_out, outl.bytes.size()), "malloc");
    ck(cudaMemset(d_out, 0, outl.bytes.size()), "memset");
    ck(cudaMalloc(&d_ws, static_cast<size_t>(ws.stride) * slots), "malloc");
    ck(cudaMalloc(&d_jobs, sizeof(pb::DevFlowJob) * count), "malloc");
    ck(cudaMemcpy(d_blob, blob.bytes.data(), blob.bytes.size(), cudaMemcpyHostToDevice), "H2D");
    std::vector<pb::DevFlowJob> jobs(count);
    eo = 0;
    no = 0;
    for (int32_t g = 0; g < count; ++g) {
      pb::DevFlowJob& j = jobs[g];
      j.nodes = nodes[g];
      j.source = source[g];
      j.sink = sink[g];
      j.m = m[g];
      j.inc_off = dptr<int32_t>(d_blob, off[g][0]);
      j.ient = dptr<pb::IEnt>(d_blob, off[g][1]);
      j.epos = dptr<int2>(d_blob, off[g][7]);
      j.ret_pt = rets[g].a;
      j.ret_ph = rets[g].b;
      j.tail = dptr<int32_t>(d_blob, off[g][2]);
      j.head = dptr<int32_t>(d_blob, off[g][3]);
      j.lower = dptr<int64_t>(d_blob, off[g][4]);
      j.upper = dptr<int64_t>(d_blob, off[g][5]);
      j.inf = dptr<uint8_t>(d_blob, off[g][6]);
      j.status = reinterpret_cast<int32_t*>(d_out + o_st);
      j.feasible = reinterpret_cast<uint8_t*>(d_out + o_fe);
      j.value = reinterpret_cast<int64_t*>(d_out + o_va);
      j.sentinel = reinterpret_cast<int64_t*>(d_out + o_se);
      j.cost = reinterpret_cast<int64_t*>(d_out + o_co);
      j.side = reinterpret_cast<uint8_t*>(d_out + o_si) + no;
      j.cut_dir = reinterpret_cast<int8_t*>(d_out + o_cd) + eo;
      eo += m[g];
      no += nodes[g];
    }
    ck(cudaMemcpy(d_jobs, jobs.data(), sizeof(pb::DevFlowJob) * count, cudaMemcpyHostToDevice), "H2D");
    const int rc = pb::launch_flow_jobs(d_jobs, count, d_ws, ws, slots, nullptr);
    if (rc) throw CudaError(cudaGetErrorString(static_cast<cudaError_t>(rc)));
    ck(cudaDeviceSynchronize(), "flow kernel");
    std::vector<char> host(outl.bytes.size());
    ck(cudaMemcpy(host.data(), d_out, host.size(), cudaMemcpyDeviceToHost), "D2H");
    std::memcpy(status, host.data() + o_st, 4 * count);
    std::memcpy(feasible, host.data() + o_fe, count);
    std::memcpy(value, host.data() + o_va, 8 * count);
    std::memcpy(sentinel, host.data() + o_se, 8 * count);
    std::memcpy(cost, host.data() + o_co, 8 * count);
    std::memcpy(source_side, host.data() + o_si, NV);
    std::memcpy(cut_dir, host.data() + o_cd, E);
    cudaFree(d_blob);
    cudaFree(d_out);
    cudaFree(d_ws);
    cudaFree(d_jobs);
    return PB_OK;
  });
}

// ------------------------------------------------------------------- G9

pb_status pb_g9_stage_bases(int32_t stages, int32_t base, double imbalance, uint32_t seed,
                            int32_t straggler_stage, double phi, int32_t* out_bases) {
  if (stages < 1) return fail(PB_ERR_INVALID_ARGUMENT, "pipeline needs at least one stage");
  pb_g9::Params p;
  p.stages = stages;
  p.base = base;
  p.imbalance = imbalance;
  p.seed = seed;
  p.straggler_stage = straggler_stage;
  p.phi = phi;
  const auto b = pb_g9::stage_bases(p);
  std::copy(b.begin(), b.end(), out_bases);
  return PB_OK;
}

pb_status pb_g9_batch_params(int32_t i, int32_t* stages, int32_t* microbatches, double* imbalance,
                             double* phi, int32_t* straggler, uint32_t* seed) {
  const pb_g9::Params p = pb_g9::batch_instance(i);
  *stages = p.stages;
  *microbatches = p.microbatches;
  *imbalance = p.imbalance;
  *phi = p.phi;
  *straggler = p.straggler_stage;
  *seed = p.seed;
  return PB_OK;
}

pb_status pb_batch_add_g9(pb_batch* b, int32_t stages, int32_t microbatches, int32_t base,
                          double imbalance, uint32_t seed, int32_t straggler_stage, double phi,
                          int64_t tau, int32_t* out_index) {
  if (!b) return fail(PB_ERR_INVALID_ARGUMENT, "null handle");
  if (stages < 1) return fail(PB_ERR_INVALID_ARGUMENT, "pipeline needs at least one stage");
  if (microbatches < 1) return fail(PB_ERR_INVALID_ARGUMENT, "pipeline needs at least one microbatch");
  pb_g9::Params p;
  p.stages = stages;
  p.microbatches = microbatches;
  p.base = base;
  p.imbalance = imbalance;
  p.seed = seed;
  p.straggler_stage = straggler_stage;
  p.phi = phi;
  const auto bases = pb_g9::stage_bases(p);
  // build_pipeline (dag.hpp:112-143), 1F1B stage streams (dag.hpp:91-103):
  // ids stage-major in stream order; kind 0 forward, 1 backward.
  const int32_t N = stages, M = microbatches, n = 2 * N * M;
  std::vector<int32_t> comp_class(n), fid(N * M), bid(N * M);
  std::vector<std::vector<int32_t>> order(N);
  int32_t id = 0;
  for (int32_t s = 0; s < N; ++s) {
    const int32_t warm = std::min(M, N - s);
    int32_t f = 0, bw = 0;
    auto emit = [&](int kind, int32_t m) {
      comp_class[id] = 2 * s + kind;  // classes sorted by (stage, kind)
      (kind == 0 ? fid : bid)[s * M + m] = id;
      order[s].push_back(id++);
    };
    for (; f < warm; ++f) emit(0, f);
    while (f < M) {
      emit(1, bw++);
      emit(0, f++);
    }
    while (bw < M) emit(1, bw++);
  }
  std::vector<int32_t> et, eh;
  for (int32_t s = 0; s < N; ++s)
    for (size_t i = 0; i + 1 < order[s].size(); ++i) {
      et.push_back(order[s][i]);
      eh.push_back(order[s][i + 1]);
    }
  for (int32_t s = 0; s + 1 < N; ++s)
    for (int32_t m = 0; m < M; ++m) {
      et.push_back(fid[s * M + m]);
      eh.push_back(fid[(s + 1) * M + m]);
      et.push_back(bid[(s + 1) * M + m]);
      eh.push_back(bid[s * M + m]);
    }
  for (int32_t s = 0; s < N; ++s) {
    et.push_back(n);
    eh.push_back(order[s].front());
    et.push_back(order[s].back());
    eh.push_back(n + 1);
  }
  // CostModel::build (costmodel.hpp:215-238) over the 2N G9 classes
  std::vector<uint8_t> cconst(2 * N, 0);
  std::vector<int32_t> poff{0}, pf;
  std::vector<int64_t> pt, pe, trange(4 * N);
  std::vector<double> curve(6 * N);
  for (int32_t s = 0; s < N; ++s)
    for (int kind = 0; kind < 2; ++kind) {
      const auto raw = pb_g9::stage_profile(bases[s], kind == 1, pb_g9::kTau);
      const int32_t c = 2 * s + kind;
      std::vector<int32_t> f(raw.size()), of(raw.size());
      std::vector<int64_t> t(raw.size()), e(raw.size()), ot(raw.size()), oe(raw.size());
      for (size_t j = 0; j < raw.size(); ++j) {
        f[j] = raw[j].freq_mhz;
        t[j] = raw[j].time;
        e[j] = raw[j].energy;
      }
      const int32_t k = pb_pareto_filter(static_cast<int32_t>(raw.size()), f.data(), t.data(), e.data(),
                                         of.data(), ot.data(), oe.data());
      double abcr[4] = {0, 0, 0, 0};
      if (k == 1 || pb_fit_exp(k, ot.data(), oe.data(), abcr) != PB_OK) {
        cconst[c] = 1;
        pf.push_back(of[0]);
        pt.push_back(ot[0]);
        pe.push_back(oe[0]);
      } else {
        for (int32_t j = 0; j < k; ++j) {
          pf.push_back(of[j]);
          pt.push_back(ot[j]);
          pe.push_back(oe[j]);
        }
        curve[3 * c] = abcr[0];
        curve[3 * c + 1] = abcr[1];
        curve[3 * c + 2] = abcr[2];
        trange[2 * c] = ot[0];
        trange[2 * c + 1] = ot[k - 1];
      }
      poff.push_back(static_cast<int32_t>(pt.size()));
    }
  pb_instance_desc d{};
  d.n = n;
  d.comp_class = comp_class.data();
  d.n_edges = static_cast<int32_t>(et.size());
  d.edge_tail = et.data();
  d.edge_head = eh.data();
  d.n_classes = 2 * N;
  d.class_is_constant = cconst.data();
  d.class_point_off = poff.data();
  d.point_freq = pf.data();
  d.point_time = pt.data();
  d.point_energy = pe.data();
  d.class_curve = curve.data();
  d.class_t_range = trange.data();
  d.blocking_watts = 75.0;
  d.quantum_us = 1;
  d.tau = tau;
  d.start_planned_t = nullptr;
  d.max_steps = 0;
  return pb_batch_add(b, &d, out_index);
}

// Config-5 instances idx[0..count) built on all host threads (batched
// CostModel::build + DAG derivation), appended in list
// order.
pb_status pb_batch_add_g9_indices(pb_batch* b, const int32_t* idx, int32_t count, int64_t tau, int32_t threads) {
  if (!b || count < 0 || (count > 0 && !idx)) return fail(PB_ERR_INVALID_ARGUMENT, "bad argument");
  for (int32_t q = 0; q < count; ++q)
    if (idx[q] < 0) return fail(PB_ERR_INVALID_ARGUMENT, "negative instance index");
  if (count == 0) return PB_OK;
  const int32_t nt = std::max(1, std::min<int32_t>(threads > 0 ? threads : static_cast<int32_t>(std::thread::hardware_concurrency()), count));
  std::vector<pb_batch> parts(nt);
  std::vector<pb_status> st(nt, PB_OK);
  std::vector<std::string> err(nt);
  std::vector<std::thread> pool;
  const int32_t chunk = (count + nt - 1) / nt;
  for (int32_t t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      for (int32_t q = t * chunk; q < std::min(count, (t + 1) * chunk); ++q) {
        const pb_g9::Params p = pb_g9::batch_instance(idx[q]);
        st[t] = pb_batch_add_g9(&parts[t], p.stages, p.microbatches, p.base, p.imbalance, p.seed, p.straggler_stage,
                                p.phi, tau, nullptr);
        if (st[t] != PB_OK) {
          err[t] = g_last_error;
          return;
        }
      }
    });
  for (auto& th : pool) th.join();
  for (int32_t t = 0; t < nt; ++t)
    if (st[t] != PB_OK) return fail(st[t], err[t]);
  for (auto& part : parts)
    for (auto& h : part.insts) b->insts.push_back(std::move(h));
  b->have_results = false;
  return PB_OK;
}

pb_status pb_batch_set_max_steps(pb_batch* b, int32_t max_steps) {
  if (!b) return fail(PB_ERR_INVALID_ARGUMENT, "null handle");
  if (max_steps < -1) return fail(PB_ERR_INVALID_ARGUMENT, "max_steps must be >= -1");
  for (auto& h : b->insts) {
    h.max_steps = max_steps;
    if (h.start.empty()) {  // sizing estimate as in validate_and_derive
      h.est_steps = std::max<int64_t>(0, h.t_star_est - h.t_min_est) / h.tau + 2;
      if (max_steps > 0) h.est_steps = std::min<int64_t>(h.est_steps, max_steps);
    } else {
      h.est_steps = std::max<int64_t>(1, max_steps);
    }
    h.work = walk_work(h);
  }
  b->have_results = false;
  return PB_OK;
}

pb_status pb_batch_add_g9_batch(pb_batch* b, int32_t first, int32_t count, int64_t tau, int32_t threads) {
  if (!b || first < 0 || count < 0) return fail(PB_ERR_INVALID_ARGUMENT, "bad argument");
  std::vector<int32_t> idx(count);
  std::iota(idx.begin(), idx.end(), first);
  return pb_batch_add_g9_indices(b, idx.data(), count, tau, threads);
}

pb_status pb_g9_profile(int32_t b, int32_t backward, int64_t tau, int32_t* freq, int64_t* time,
                        int64_t* energy) {
  const auto pts = pb_g9::stage_profile(b, backward != 0, tau);
  for (size_t j = 0; j < pts.size(); ++j) {
    freq[j] = pts[j].freq_mhz;
    time[j] = pts[j].time;
    energy[j] = pts[j].energy;
  }
  return PB_OK;
}

}  // extern "C"
