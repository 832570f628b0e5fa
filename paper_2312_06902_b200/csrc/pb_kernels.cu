// sm_100a kernels of the B200-native Perseus frontier generator.
//
// One WARP walks one instance's whole frontier (frontier.hpp:166-189) inside
// a single persistent launch: warps pull instances (LPT order) from a global
// counter, so thousands of walks are in flight and no host round trip
// happens per step.  All synchronization is __syncwarp, appends are ballot
// compactions, deduplication is __match_any_sync + a stamp.  Per step:
//
//   K2  longest path over static node-DAG levels (annotate_slack,
//       dag.hpp:233-286; simulate, emulator.hpp:28-55): pull-based,
//       deterministic;
//   K3  fused critical mask + Eq. 7 capacities (build_capacity_dag,
//       flow.hpp:285-317) from host-tabulated curve values, with the
//       reference's int128 overflow checks (flow.hpp:58-68, 196-197);
//   K4  max flow with lower bounds, WARM-STARTED: the flow of the previous
//       step is kept, clamped into the new bounds (edges leaving the critical
//       sub-DAG drop to 0, new ones start at their lower bound), and the
//       resulting node imbalances are repaired by multi-source BFS
//       augmentation in the circulation network with the return arc
//       sink->source (phase A = the feasibility test of flow.hpp:172-203);
//       phase B then augments source->sink along BFS-shortest residual
//       paths (flow.hpp:205-228).  Steps change few capacities, so a step
//       needs ~1-4 BFS instead of a from-scratch max flow;
//   K5  the last phase-B BFS (sink unreachable) visits exactly the source
//       side of the minimal minimum cut (min_cut_from_flow, flow.hpp:234-262);
//       tau update with the reference's skip rules (frontier.hpp:111-131),
//       discretize (frontier.hpp:140-161), realized longest path,
//       append-only delta log.
//
// Only the unique minimal min cut and the two verdicts (feasible, value >=
// sentinel) feed the outputs, so the flow itself is free to differ from the
// reference's Edmonds-Karp flow (SURVEY.md §7 parity rule 1).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "pb_internal.h"

namespace pb {
namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int kBlock = 32 * kWarpsPerBlock;
constexpr unsigned kFull = 0xffffffffu;
constexpr long long kHuge = LLONG_MAX / 4;  // return-arc capacity (never binding)
typedef __int128 i128;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }

__device__ __forceinline__ long long wsum(long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ long long wmax(long long v) {
  for (int o = 16; o; o >>= 1) {
    const long long u = __shfl_xor_sync(kFull, v, o);
    v = u > v ? u : v;
  }
  return v;
}
__device__ __forceinline__ long long wmin(long long v) {
  for (int o = 16; o; o >>= 1) {
    const long long u = __shfl_xor_sync(kFull, v, o);
    v = u < v ? u : v;
  }
  return v;
}
__device__ __forceinline__ int wmaxi(int v) { return __reduce_max_sync(kFull, v); }
__device__ __forceinline__ i128 wsum128(i128 v) {
  for (int o = 16; o; o >>= 1) {
    unsigned long long lo = static_cast<unsigned long long>(v);
    unsigned long long hi = static_cast<unsigned long long>(v >> 64);
    lo = __shfl_xor_sync(kFull, lo, o);
    hi = __shfl_xor_sync(kFull, hi, o);
    v += static_cast<i128>((static_cast<unsigned __int128>(hi) << 64) | lo);
  }
  return v;
}

// Ballot compaction: every lane of the (converged) warp calls it; lanes with
// pred append val at list[count ...]; count stays warp-uniform.
__device__ __forceinline__ void wappend(bool pred, int val, int32_t* list, int& count) {
  const unsigned m = __ballot_sync(kFull, pred);
  if (pred) list[count + __popc(m & lanemask_lt())] = val;
  count += __popc(m);
}

__device__ __forceinline__ void red_add(int64_t* p, long long d) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(d));
}

struct Counters {
  unsigned long long arc_scans = 0, node_updates = 0, rounds = 0, comp_visits = 0;
  unsigned long long prof[kPrSlots] = {};
  __device__ void add(int slot, long long v) {
    if (lane_id() == 0) prof[slot] += static_cast<unsigned long long>(v);
  }
};

__device__ __forceinline__ long long now() { return clock64(); }

// Flow-network view of one warp's workspace.  Edge ids: graph edges, then the
// return arc `ret` (sink -> source, capacity kHuge, enabled in phase A only);
// f[ret] is the circulation's s->t value R.
struct Net {
  int V, E, src, snk, ret;
  const int32_t* inc_off;
  const int32_t* inc;  // (edge << 1) | dir, dir = 1 when the node is the head
  const int32_t* tail;
  const int32_t* head;
  int64_t* lo;
  int64_t* up;  // finite upper bound (ignored when inf)
  int64_t* f;   // absolute flow, persistent across steps
  uint8_t* inf;
  uint8_t* crit;  // edge present in the current network
  int64_t* bal;   // inflow - outflow (phase-A imbalance)
  int32_t* vis;   // BFS stamp
  int32_t* par;   // BFS parent code (edge << 1) | backward
  int32_t* mk;    // list dedup stamp
  int32_t* f0;
  int32_t* f1;
  int32_t* touch;
  int32_t* exl;
  long long sentinel;
  int stamp, mstamp;
  bool ret_on;
};

__device__ __forceinline__ long long upres(const Net& N, int ed) {
  return ed == N.ret ? kHuge : (N.inf[ed] ? N.sentinel : N.up[ed]);
}
// Residual capacity of traversing incidence entry a away from its node:
// forward (node is tail) = upper - f, backward (node is head) = f - lower.
__device__ __forceinline__ long long residual_from(const Net& N, int a) {
  const int ed = a >> 1;
  if (ed == N.ret ? !N.ret_on : !N.crit[ed]) return 0;
  return (a & 1) ? N.f[ed] - N.lo[ed] : upres(N, ed) - N.f[ed];
}
__device__ __forceinline__ int other_end(const Net& N, int a) {
  const int ed = a >> 1;
  return (a & 1) ? N.tail[ed] : N.head[ed];
}

// Level-synchronous BFS over residual arcs from `nsrc` sources in N.f0.
// phaseA: targets are nodes with bal < 0; phaseB: the sink.  Stops at the
// first level that reaches a target and returns it (-1: none reachable; then
// the stamp N.stamp marks exactly the residual-reachable set).
__device__ int bfs(Net& N, int nsrc, bool phaseA, Counters& C) {
  const int ln = lane_id();
  const long long t0 = now();
  ++N.stamp;
  const int stamp = N.stamp;
  for (int i = ln; i < nsrc; i += 32) {
    const int v = N.f0[i];
    N.vis[v] = stamp;
    N.par[v] = -1;
  }
  __syncwarp();
  int cnt = nsrc;
  int32_t* F = N.f0;
  int32_t* G = N.f1;
  int found = -1;
  while (cnt > 0 && found < 0) {
    C.add(kPrBfsLevels, 1);
    int nc = 0;
    for (int base = 0; base < cnt; base += 32) {
      const int i = base + ln;
      const bool valid = i < cnt;
      const int w = valid ? F[i] : 0;
      const int off = valid ? N.inc_off[w] : 0;
      const int deg = valid ? N.inc_off[w + 1] - off : 0;
      const int md = wmaxi(deg);
      if (valid) C.arc_scans += deg;
      for (int j = 0; j < md; ++j) {
        bool cand = false;
        int u = 0, a = 0;
        if (j < deg) {
          a = N.inc[off + j];
          if (residual_from(N, a) > 0) {
            u = other_end(N, a);
            cand = N.vis[u] != stamp;
          }
        }
        const unsigned peers = __match_any_sync(kFull, cand ? u : -1 - ln);
        const bool lead = cand && (__ffs(peers) - 1) == ln;
        bool hit = false;
        if (lead) {
          N.vis[u] = stamp;
          N.par[u] = ((a >> 1) << 1) | (a & 1);
          ++C.node_updates;
          hit = phaseA ? N.bal[u] < 0 : u == N.snk;
        }
        const unsigned h = __ballot_sync(kFull, hit);
        if (h && found < 0) found = __shfl_sync(kFull, u, __ffs(h) - 1);
        wappend(lead, u, G, nc);
        __syncwarp();
      }
    }
    cnt = nc;
    int32_t* t = F;
    F = G;
    G = t;
  }
  __syncwarp();
  C.add(kPrBfs, now() - t0);
  return found;
}

// Augments along the BFS parent chain ending at `tgt` (lane 0; the path is a
// pointer chase).  Phase A: amount = min(residuals, bal[src], -bal[tgt]) and
// the balances move; phase B: amount = min(residuals) and R grows.
__device__ void augment(Net& N, int tgt, bool phaseA, Counters& C) {
  const long long t0 = now();
  if (lane_id() == 0) {
    long long d = phaseA ? -N.bal[tgt] : LLONG_MAX;
    int v = tgt, hops = 0;
    while (N.par[v] != -1) {
      const int code = N.par[v];
      const int ed = code >> 1;
      const long long r = (code & 1) ? N.f[ed] - N.lo[ed] : upres(N, ed) - N.f[ed];
      d = r < d ? r : d;
      v = (code & 1) ? N.head[ed] : N.tail[ed];
      ++hops;
    }
    if (phaseA) d = N.bal[v] < d ? N.bal[v] : d;
    const int src = v;
    v = tgt;
    while (N.par[v] != -1) {
      const int code = N.par[v];
      const int ed = code >> 1;
      N.f[ed] += (code & 1) ? -d : d;
      v = (code & 1) ? N.head[ed] : N.tail[ed];
    }
    if (phaseA) {
      N.bal[src] -= d;
      N.bal[tgt] += d;
    } else {
      N.f[N.ret] += d;
    }
    C.prof[kPrPaths] += 1;
    C.prof[kPrPathHops] += hops;
    C.node_updates += 2 * hops;
  }
  __syncwarp();
  C.add(kPrAugment, now() - t0);
}

// Phase A: repairs the imbalances of the nodes in N.touch (ntouch entries,
// duplicates allowed) in the circulation network (return arc enabled).
// Returns false when some excess cannot reach any deficit: the bounded
// network is infeasible (max_flow_lower_bounds returns nullopt).
__device__ bool repair(Net& N, int ntouch, Counters& C) {
  const int ln = lane_id();
  // distinct touched nodes with excess
  ++N.mstamp;
  int nex = 0;
  for (int base = 0; base < ntouch; base += 32) {
    const int i = base + ln;
    const bool valid = i < ntouch;
    const int v = valid ? N.touch[i] : 0;
    const unsigned peers = __match_any_sync(kFull, valid ? v : -1 - ln);
    bool take = valid && (__ffs(peers) - 1) == ln && N.mk[v] != N.mstamp;
    if (take) N.mk[v] = N.mstamp;
    take = take && N.bal[v] > 0;
    wappend(take, v, N.exl, nex);
    __syncwarp();
  }
  if (nex == 0) return true;
  C.add(kPrImbalanced, nex);
  const long long t0 = now();
  N.ret_on = true;
  bool ok = true;
  for (;;) {
    int ns = 0;
    for (int base = 0; base < nex; base += 32) {
      const int i = base + ln;
      const int v = i < nex ? N.exl[i] : 0;
      wappend(i < nex && N.bal[v] > 0, v, N.f0, ns);
    }
    __syncwarp();
    if (ns == 0) break;
    for (int i = ln; i < ns; i += 32) N.exl[i] = N.f0[i];
    nex = ns;
    __syncwarp();
    C.add(kPrBfsA, 1);
    const int tgt = bfs(N, ns, true, C);
    if (tgt < 0) {
      ok = false;
      break;
    }
    augment(N, tgt, true, C);
  }
  N.ret_on = false;
  C.add(kPrPhaseA, now() - t0);
  return ok;
}

// Phase B: source->sink augmentation until the sink is unreachable; the
// last BFS stamp then marks the minimal min cut's source side.
__device__ void maximize(Net& N, Counters& C) {
  const long long t0 = now();
  for (;;) {
    if (lane_id() == 0) N.f0[0] = N.src;
    __syncwarp();
    C.add(kPrBfsB, 1);
    const int tgt = bfs(N, 1, false, C);
    if (tgt < 0) break;
    augment(N, tgt, false, C);
  }
  C.add(kPrPhaseB, now() - t0);
}

// Records a flow change on edge ed: imbalance at both ends, both touched.
__device__ __forceinline__ void flow_change(Net& N, int ed, long long delta) {
  red_add(&N.bal[N.head[ed]], delta);
  red_add(&N.bal[N.tail[ed]], -delta);
}

// ------------------------------------------------------------------ walk

struct Walk {
  int64_t* planned;
  int64_t* estart;
  int64_t* lend;
  int64_t* rstart;
  int64_t* rdur;
  int64_t* pdur;
  uint8_t* choice;
  int32_t* delta;
};

// Level-synchronous longest path on the node DAG (simulate,
// emulator.hpp:28-55; forward half of annotate_slack, dag.hpp:266-271).
// start[i] = max over predecessors (start[u] + dur[u]); returns makespan.
__device__ long long forward_pass(const DevInst& I, const int64_t* dur, int64_t* start, Counters& C) {
  const int ln = lane_id();
  const long long t0 = now();
  C.add(kPrLpLevels, I.n_levels);
  for (int L = 0; L < I.n_levels; ++L) {
    const int b = I.lvl_off[L], e = I.lvl_off[L + 1];
    for (int q = b + ln; q < e; q += 32) {
      const int i = I.lvl_comps[q];
      long long m = 0;
      for (int j = I.in_off[i]; j < I.in_off[i + 1]; ++j) {
        const int u = I.dep_tail[I.in_dep[j]];
        if (u < I.n) {
          const long long c = start[u] + dur[u];
          if (c > m) m = c;
        }
      }
      start[i] = m;
      ++C.comp_visits;
    }
    __syncwarp();
  }
  long long ms = 0;
  for (int q = ln; q < I.n_snk; q += 32) {
    const int u = I.dep_tail[I.snk_dep[q]];
    if (u < I.n) {
      const long long c = start[u] + dur[u];
      if (c > ms) ms = c;
    }
  }
  ms = wmax(ms);
  C.add(kPrLp, now() - t0);
  return ms;
}

// Backward half of annotate_slack (dag.hpp:272-277): lend[i] = latest time
// of node 2i+1 = min over successors (lend[v] - dur[v]), makespan at the sink.
__device__ void backward_pass(const DevInst& I, const int64_t* dur, int64_t* lend, long long ms,
                              Counters& C) {
  const int ln = lane_id();
  const long long t0 = now();
  C.add(kPrLpLevels, I.n_levels);
  for (int L = I.n_levels - 1; L >= 0; --L) {
    const int b = I.lvl_off[L], e = I.lvl_off[L + 1];
    for (int q = b + ln; q < e; q += 32) {
      const int i = I.lvl_comps[q];
      long long m = ms;
      for (int j = I.out_off[i]; j < I.out_off[i + 1]; ++j) {
        const int v = I.dep_head[I.out_dep[j]];
        if (v < I.n) {
          const long long c = lend[v] - dur[v];
          if (c < m) m = c;
        }
      }
      lend[i] = m;
      ++C.comp_visits;
    }
    __syncwarp();
  }
  C.add(kPrLp, now() - t0);
}

__device__ __forceinline__ int discretize_choice(const DevInst& I, int c, long long t) {
  // last Pareto point with time <= planned, else the fastest (frontier.hpp:146-156)
  const int p0 = I.cls_pt_off[c], p1 = I.cls_pt_off[c + 1];
  int chosen = 0;
  for (int p = p0; p < p1; ++p)
    if (I.pt_time[p] <= t) chosen = p - p0;
  return chosen;
}

// ExpCurve::eval (costmodel.hpp:47) from the host table (bit-identical to the
// reference's libm values); outside [t_min, t_max] -- reachable only from a
// caller-supplied start schedule or the infinite-edge cut case (SURVEY.md §7
// parity rule 5) -- the device evaluates the curve itself and counts it.
__device__ __forceinline__ double table_at(const DevInst& I, int c, long long t, int* extrap) {
  if (t >= I.cls_tmin[c] && t <= I.cls_tmax[c]) return I.tables[I.cls_tab[c] + (t - I.cls_tmin[c])];
  ++*extrap;
  return I.cls_curve[3 * c] * exp(I.cls_curve[3 * c + 1] * static_cast<double>(t)) + I.cls_curve[3 * c + 2];
}

// planned_energy (frontier.hpp:59-62).
__device__ __forceinline__ long long table_energy(const DevInst& I, int c, long long t, int* extrap) {
  if (I.cls_const[c]) return I.pt_energy[I.cls_pt_off[c]];
  return llround(table_at(I, c, t, extrap));
}

__device__ void write_point(const DevInst& I, int k, long long tp, long long tr, long long spe,
                            long long spt, long long sre, long long srt, long long cut,
                            long long step, int id_begin, int ns, int nl) {
  pb_point p;
  p.t_planned = tp;
  p.t_realized = tr;
  p.sum_planned_e = spe;
  p.sum_planned_t = spt;
  p.sum_realized_e = sre;
  p.sum_realized_t = srt;
  p.cut_cost = cut;
  p.step_size = step;
  p.id_begin = id_begin;
  p.n_sped = ns;
  p.n_slowed = nl;
  p.pad = 0;
  I.points[k] = p;
}

__device__ void reset_net(Net& N) {
  const int ln = lane_id();
  for (int e = ln; e < N.E; e += 32) {
    N.f[e] = 0;
    N.lo[e] = 0;
    N.up[e] = 0;
    N.inf[e] = 0;
    N.crit[e] = 0;
  }
  for (int v = ln; v < N.V; v += 32) {
    N.bal[v] = 0;
    N.vis[v] = 0;
    N.mk[v] = 0;
  }
  N.stamp = 0;
  N.mstamp = 0;
  N.ret_on = false;
  N.sentinel = 0;
  __syncwarp();
}

// Clamps every infinite critical edge's flow to the new sentinel (only
// needed when the sentinel shrank below a carried flow; checked by caller).
__device__ void clamp_infinite(Net& N, int nedges, int& ntouch) {
  const int ln = lane_id();
  for (int base = 0; base < nedges; base += 32) {
    const int k = base + ln;
    bool ch = false;
    if (k < nedges && N.crit[k] && N.inf[k] && N.f[k] > N.sentinel) {
      flow_change(N, k, N.sentinel - N.f[k]);
      N.f[k] = N.sentinel;
      ch = true;
    }
    wappend(ch, ch ? N.tail[k] : 0, N.touch, ntouch);
    wappend(ch, ch ? N.head[k] : 0, N.touch, ntouch);
  }
  __syncwarp();
}

__device__ void run_walk(const DevInst& I, Net& N, Walk& W, const DeltaPool& pool, Counters& C) {
  const int ln = lane_id();
  const int n = I.n;
  N.V = 2 * n + 2;
  N.src = 2 * n;
  N.snk = 2 * n + 1;
  N.ret = n + I.ne;
  N.E = n + I.ne + 1;
  N.inc_off = I.inc_off;
  N.inc = I.inc;
  N.tail = I.ec_tail;
  N.head = I.ec_head;
  reset_net(N);

  int bad = 0;
  long long spe = 0, spt = 0, sre = 0, srt = 0;
  for (int i = ln; i < n; i += 32) {
    const int c = I.comp_class[i];
    long long t;
    if (I.mode == kModeGetNext)
      t = I.start_planned_t[i];
    else
      t = I.cls_const[c] ? I.pt_time[I.cls_pt_off[c]] : I.cls_tmax[c];
    W.planned[i] = t;
    const int ch = discretize_choice(I, c, t);
    W.choice[i] = static_cast<uint8_t>(ch);
    W.rdur[i] = I.pt_time[I.cls_pt_off[c] + ch];
    W.pdur[i] = I.pt_time[I.cls_pt_off[c]];  // all-max durations (emulator.hpp:140-149)
    spe += table_energy(I, c, t, &bad);
    spt += t;
    sre += I.pt_energy[I.cls_pt_off[c] + ch];
    srt += W.rdur[i];
  }
  __syncwarp();
  spe = wsum(spe);
  spt = wsum(spt);
  sre = wsum(sre);
  srt = wsum(srt);

  const long long t_walk0 = now();
  int detail = 0;
  const long long t_min = forward_pass(I, W.pdur, W.estart, C);
  long long t_cur = forward_pass(I, W.planned, W.estart, C);
  long long t_real = forward_pass(I, W.rdur, W.rstart, C);
  const long long t_star = t_cur;
  if (ln == 0) write_point(I, 0, t_cur, t_real, spe, spt, sre, srt, 0, 0, 0, 0, 0);
  int steps = 0;
  long long n_ids = 0;
  int status = PB_OK;
  int stop = PB_STOP_AT_TMIN;
  const int nedges = n + I.ne;

  for (;;) {
    long long step;
    if (I.mode == kModeDiscover) {
      if (!(t_cur > t_min)) {
        stop = PB_STOP_AT_TMIN;
        break;
      }
      step = I.tau < t_cur - t_min ? I.tau : t_cur - t_min;
    } else {
      step = I.tau;
    }
    if (I.max_steps != 0 && steps >= (I.max_steps < 0 ? 0 : I.max_steps)) {
      stop = PB_STOP_STEP_LIMIT;
      break;
    }
    if (steps + 2 > I.cap_points) {
      status = kStatusLogFull;
      break;
    }
    // ---- K2 backward pass (latest) on the current planned durations
    backward_pass(I, W.planned, W.lend, t_cur, C);
    // ---- K3 critical mask + capacities; carried flow clamped into the new bounds
    const long long tcap = now();
    C.add(kPrSteps, 1);
    i128 suml = 0, sumu = 0;
    long long ninf = 0, max_inf_f = 0;
    int ntouch = 0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + ln;
      bool ch = false;
      if (i < n) {
        const int c = I.comp_class[i];
        const long long t = W.planned[i];
        const bool crit = W.estart[i] + t == W.lend[i];
        long long l = 0, u = 0;
        uint8_t inf = 1;
        if (crit && !I.cls_const[c]) {
          const long long tmin = I.cls_tmin[c], tmax = I.cls_tmax[c];
          const bool can_speed = t - step >= tmin;
          const bool can_slow = t + step <= tmax;
          const double et = (can_speed || can_slow) ? table_at(I, c, t, &bad) : 0.0;
          if (can_slow) {
            const long long r = llround(et - table_at(I, c, t + step, &bad));
            l = r > 0 ? r : 0;
          }
          if (can_speed) {
            const long long r = llround(table_at(I, c, t - step, &bad) - et);
            u = r > l ? r : l;
            inf = 0;
          }
        }
        const long long fo = N.f[i];
        long long fn = 0;
        if (crit) {
          fn = fo < l ? l : fo;
          if (!inf && fn > u) fn = u;
          suml += l;
          if (!inf)
            sumu += u;
          else {
            ++ninf;
            max_inf_f = fn > max_inf_f ? fn : max_inf_f;
          }
        }
        N.lo[i] = l;
        N.up[i] = u;
        N.inf[i] = inf;
        N.crit[i] = crit;
        if (fn != fo) {
          N.f[i] = fn;
          flow_change(N, i, fn - fo);
          ch = true;
        }
      }
      wappend(ch, 2 * i, N.touch, ntouch);
      wappend(ch, 2 * i + 1, N.touch, ntouch);
    }
    for (int base = 0; base < I.ne; base += 32) {
      const int j = base + ln;
      bool ch = false;
      const int k = n + j;
      if (j < I.ne) {
        const int u = I.dep_tail[j], v = I.dep_head[j];
        long long te, he;
        bool tc, hc;
        if (u == n) {
          te = 0;
          tc = true;  // latest[source] == 0 whenever a critical head exists
        } else {
          te = W.estart[u] + W.planned[u];
          tc = te == W.lend[u];
        }
        if (v == n + 1) {
          he = t_cur;
          hc = true;
        } else {
          he = W.estart[v];
          hc = W.estart[v] + W.planned[v] == W.lend[v];
        }
        const bool crit = tc && hc && te == he;
        N.crit[k] = crit;
        N.lo[k] = 0;
        N.inf[k] = 1;
        const long long fo = N.f[k];
        if (crit) {
          ++ninf;
          max_inf_f = fo > max_inf_f ? fo : max_inf_f;
        } else if (fo != 0) {
          N.f[k] = 0;
          flow_change(N, k, -fo);
          ch = true;
        }
      }
      wappend(ch, ch ? N.tail[k] : 0, N.touch, ntouch);
      wappend(ch, ch ? N.head[k] : 0, N.touch, ntouch);
    }
    suml = wsum128(suml);
    sumu = wsum128(sumu);
    ninf = wsum(ninf);
    max_inf_f = wmax(max_inf_f);
    // infinity_sentinel (flow.hpp:58-68) and the aux total (flow.hpp:196-197)
    const i128 sent128 = suml + sumu + 1;
    if (sent128 > static_cast<i128>(LLONG_MAX / 4)) {
      status = PB_ERR_OVERFLOW;
      break;
    }
    N.sentinel = static_cast<long long>(sent128);
    const i128 aux = sumu + static_cast<i128>(ninf) * N.sentinel + suml;
    if (aux + 1 > static_cast<i128>(LLONG_MAX / 2)) {
      status = PB_ERR_OVERFLOW;
      break;
    }
    __syncwarp();
    if (max_inf_f > N.sentinel) clamp_infinite(N, nedges, ntouch);
    C.add(kPrCap, now() - tcap);
    // ---- K4 warm-started max flow with lower bounds
    if (!repair(N, ntouch, C)) {
      stop = PB_STOP_INFEASIBLE;
      break;
    }
    maximize(N, C);
    if (N.f[N.ret] >= N.sentinel) {
      stop = PB_STOP_INFINITE_CUT;
      break;
    }
    // ---- K5 minimal min cut = the last BFS's visited set
    const long long tupd = now();
    const int side_stamp = N.stamp;
    long long cost = 0;
    int nd = 0;
    for (int base = 0; base < nedges; base += 32) {
      const int k = base + ln;
      int rec = 0;
      if (k < nedges && N.crit[k]) {
        const bool a = N.vis[N.tail[k]] == side_stamp, b = N.vis[N.head[k]] == side_stamp;
        if (a && !b) {
          cost += N.inf[k] ? N.sentinel : N.up[k];
          if (k < n) rec = k + 1;
        } else if (!a && b) {
          cost -= N.lo[k];
          if (k < n) {
            const int c = I.comp_class[k];
            if (!I.cls_const[c] && W.planned[k] + step <= I.cls_tmax[c]) rec = -(k + 1);
          }
        }
      }
      wappend(rec != 0, rec, W.delta, nd);
    }
    cost = wsum(cost);
    __syncwarp();
    // reserve a contiguous range of the batch delta pool
    unsigned long long at = 0;
    if (ln == 0 && nd) at = atomicAdd(pool.cursor, static_cast<unsigned long long>(nd));
    at = __shfl_sync(kFull, at, 0);
    if (static_cast<long long>(at) + nd > pool.cap) {
      status = kStatusLogFull;
      break;
    }
    // order: sped ascending, then slowed ascending (frontier.hpp:111-125)
    int ns_loc = 0;
    long long dpe = 0, dpt = 0, dre = 0, drt = 0;
    for (int q = ln; q < nd; q += 32) {
      const int x = W.delta[q];
      const long long kx = x > 0 ? x : (1ll << 40) - x;
      int rank = 0;
      for (int r = 0; r < nd; ++r) {
        const int y = W.delta[r];
        const long long ky = y > 0 ? y : (1ll << 40) - y;
        rank += ky < kx;
      }
      const int i = (x > 0 ? x : -x) - 1;
      const int c = I.comp_class[i];
      const long long told = W.planned[i];
      const long long tnew = x > 0 ? told - step : told + step;
      const long long eold = table_energy(I, c, told, &bad);
      const long long enew = table_energy(I, c, tnew, &bad);
      const int chold = W.choice[i];
      const int chnew = discretize_choice(I, c, tnew);
      const int p0 = I.cls_pt_off[c];
      dpe += enew - eold;
      dpt += tnew - told;
      dre += I.pt_energy[p0 + chnew] - I.pt_energy[p0 + chold];
      drt += I.pt_time[p0 + chnew] - I.pt_time[p0 + chold];
      ns_loc += x > 0;
      pool.ids[at + rank] = x;
      pool.choice[at + rank] = static_cast<uint8_t>(chnew);
    }
    __syncwarp();
    for (int q = ln; q < nd; q += 32) {
      const int x = W.delta[q];
      const int i = (x > 0 ? x : -x) - 1;
      const int c = I.comp_class[i];
      const long long tnew = x > 0 ? W.planned[i] - step : W.planned[i] + step;
      W.planned[i] = tnew;
      const int ch = discretize_choice(I, c, tnew);
      W.choice[i] = static_cast<uint8_t>(ch);
      W.rdur[i] = I.pt_time[I.cls_pt_off[c] + ch];
    }
    __syncwarp();
    const int ns = static_cast<int>(wsum(ns_loc));
    dpe = wsum(dpe);
    dpt = wsum(dpt);
    dre = wsum(dre);
    drt = wsum(drt);
    C.add(kPrUpdate, now() - tupd);
    // refresh_totals (frontier.hpp:64-67): new planned makespan
    const long long t_new = forward_pass(I, W.planned, W.estart, C);
    if (I.mode == kModeDiscover && t_new >= t_cur) {
      stop = PB_STOP_NO_PROGRESS;
      break;
    }
    t_cur = t_new;
    spe += dpe;
    spt += dpt;
    sre += dre;
    srt += drt;
    // discretize (frontier.hpp:157): realized makespan
    t_real = forward_pass(I, W.rdur, W.rstart, C);
    ++steps;
    if (ln == 0)
      write_point(I, steps, t_cur, t_real, spe, spt, sre, srt, cost, step, static_cast<int>(at), ns, nd - ns);
    n_ids += nd;
  }
  __syncwarp();
  const long long n_extrap = wsum(bad);
  C.add(kPrWalk, now() - t_walk0);
  if (ln == 0) {
    pb_frontier_summary s;
    s.t_min = t_min;
    s.t_star = t_star;
    s.steps = steps;
    s.stop = stop;
    s.status = status;
    s.n_ids = static_cast<int32_t>(n_ids);
    s.n_extrapolated = static_cast<int32_t>(n_extrap);
    s.pad = detail;
    *I.summary = s;
  }
  __syncwarp();
}

struct WsPtrs {
  Net N;
  Walk W;
};

__device__ WsPtrs bind_ws(char* base, const WsLayout& L) {
  WsPtrs p;
  p.N.lo = reinterpret_cast<int64_t*>(base + L.off_lo);
  p.N.up = reinterpret_cast<int64_t*>(base + L.off_up);
  p.N.f = reinterpret_cast<int64_t*>(base + L.off_f);
  p.N.inf = reinterpret_cast<uint8_t*>(base + L.off_inf);
  p.N.crit = reinterpret_cast<uint8_t*>(base + L.off_crit);
  p.N.bal = reinterpret_cast<int64_t*>(base + L.off_bal);
  p.N.vis = reinterpret_cast<int32_t*>(base + L.off_vis);
  p.N.par = reinterpret_cast<int32_t*>(base + L.off_par);
  p.N.mk = reinterpret_cast<int32_t*>(base + L.off_mk);
  p.N.f0 = reinterpret_cast<int32_t*>(base + L.off_f0);
  p.N.f1 = reinterpret_cast<int32_t*>(base + L.off_f1);
  p.N.touch = reinterpret_cast<int32_t*>(base + L.off_touch);
  p.N.exl = reinterpret_cast<int32_t*>(base + L.off_exl);
  p.W.planned = reinterpret_cast<int64_t*>(base + L.off_planned);
  p.W.estart = reinterpret_cast<int64_t*>(base + L.off_estart);
  p.W.lend = reinterpret_cast<int64_t*>(base + L.off_lend);
  p.W.rstart = reinterpret_cast<int64_t*>(base + L.off_rstart);
  p.W.rdur = reinterpret_cast<int64_t*>(base + L.off_rdur);
  p.W.pdur = reinterpret_cast<int64_t*>(base + L.off_pdur);
  p.W.choice = reinterpret_cast<uint8_t*>(base + L.off_choice);
  p.W.delta = reinterpret_cast<int32_t*>(base + L.off_delta);
  return p;
}

__device__ void flush_counters(const Counters& C, RunCounters* out) {
  if (!out) return;
  const unsigned long long a = wsum(static_cast<long long>(C.arc_scans));
  const unsigned long long u = wsum(static_cast<long long>(C.node_updates));
  const unsigned long long v = wsum(static_cast<long long>(C.comp_visits));
  if (lane_id() == 0) {
    atomicAdd(&out->arc_scans, a);
    atomicAdd(&out->node_updates, u);
    atomicAdd(&out->comp_visits, v);
    atomicAdd(&out->rounds, C.prof[kPrBfsLevels]);
    for (int q = 0; q < kPrSlots; ++q) atomicAdd(&out->prof[q], C.prof[q]);
  }
}

__device__ __forceinline__ int warp_slot() {
  return blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
}

__global__ void __launch_bounds__(kBlock) walk_kernel(const DevInst* insts, int n_inst,
                                                      const int32_t* order, int32_t* counter,
                                                      char* ws_base, WsLayout L, int slots,
                                                      RunCounters* ctr, DeltaPool pool) {
  const int slot = warp_slot();
  if (slot >= slots) return;
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(slot) * L.stride, L);
  Counters C;
  for (;;) {
    int k = 0;
    if (lane_id() == 0) k = atomicAdd(counter, 1);
    k = __shfl_sync(kFull, k, 0);
    if (k >= n_inst) break;
    run_walk(insts[order[k]], P.N, P.W, pool, C);
  }
  flush_counters(C, ctr);
}

// ------------------------------------------------------------ flow jobs

// max_flow_lower_bounds + min_cut_from_flow on an arbitrary FlowGraph with
// the same machinery from the all-lower-bound start (f = l everywhere).
__global__ void __launch_bounds__(kBlock) flow_kernel(const DevFlowJob* jobs, int count,
                                                      char* ws_base, WsLayout L, int slots) {
  const int slot = warp_slot();
  if (slot >= slots) return;
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(slot) * L.stride, L);
  Net& N = P.N;
  Counters C;
  const int ln = lane_id();
  for (int g = slot; g < count; g += slots) {
    const DevFlowJob& J = jobs[g];
    N.V = J.nodes;
    N.src = J.source;
    N.snk = J.sink;
    N.ret = J.m;
    N.E = J.m + 1;
    N.inc_off = J.inc_off;
    N.inc = J.inc;
    N.tail = J.tail;
    N.head = J.head;
    reset_net(N);
    i128 suml = 0, sumu = 0;
    long long ninf = 0;
    int ntouch = 0;
    for (int base = 0; base < J.m; base += 32) {
      const int e = base + ln;
      bool ch = false;
      if (e < J.m) {
        N.lo[e] = J.lower[e];
        N.up[e] = J.upper[e];
        N.inf[e] = J.inf[e];
        N.crit[e] = 1;
        suml += J.lower[e];
        if (!J.inf[e])
          sumu += J.upper[e];
        else
          ++ninf;
        if (J.lower[e] > 0) {
          N.f[e] = J.lower[e];
          flow_change(N, e, J.lower[e]);
          ch = true;
        }
      }
      wappend(ch, ch ? J.tail[e] : 0, N.touch, ntouch);
      wappend(ch, ch ? J.head[e] : 0, N.touch, ntouch);
    }
    suml = wsum128(suml);
    sumu = wsum128(sumu);
    ninf = wsum(ninf);
    const i128 sent128 = suml + sumu + 1;
    int status = PB_OK;
    i128 aux = 0;
    if (sent128 > static_cast<i128>(LLONG_MAX / 4)) {
      status = PB_ERR_OVERFLOW;
    } else {
      N.sentinel = static_cast<long long>(sent128);
      aux = sumu + static_cast<i128>(ninf) * N.sentinel + suml;
      if (aux + 1 > static_cast<i128>(LLONG_MAX / 2)) status = PB_ERR_OVERFLOW;
    }
    __syncwarp();
    if (status != PB_OK) {
      if (ln == 0) {
        J.status[g] = status;
        J.feasible[g] = 0;
      }
      __syncwarp();
      continue;
    }
    if (!repair(N, ntouch, C)) {
      if (ln == 0) {
        J.status[g] = PB_OK;
        J.feasible[g] = 0;
        J.sentinel[g] = N.sentinel;
      }
      __syncwarp();
      continue;
    }
    maximize(N, C);
    const int side_stamp = N.stamp;
    long long cost = 0;
    for (int e = ln; e < J.m; e += 32) {
      const bool a = N.vis[N.tail[e]] == side_stamp, b = N.vis[N.head[e]] == side_stamp;
      int8_t dir = 0;
      if (a && !b) {
        cost += J.inf[e] ? N.sentinel : J.upper[e];
        dir = 1;
      } else if (!a && b) {
        cost -= J.lower[e];
        dir = -1;
      }
      J.cut_dir[e] = dir;
    }
    for (int v = ln; v < N.V; v += 32) J.side[v] = N.vis[v] == side_stamp ? 1 : 0;
    cost = wsum(cost);
    if (ln == 0) {
      J.status[g] = N.vis[N.snk] == side_stamp ? PB_ERR_LOGIC : PB_OK;
      J.feasible[g] = 1;
      J.value[g] = N.f[N.ret];
      J.sentinel[g] = N.sentinel;
      J.cost[g] = cost;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------ slack jobs

__global__ void __launch_bounds__(kBlock) slack_kernel(const DevInst* insts, const SlackOut* outs,
                                                       int64_t* makespan, int count, char* ws_base,
                                                       WsLayout L, int slots) {
  const int slot = warp_slot();
  if (slot >= slots) return;
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(slot) * L.stride, L);
  Counters C;
  const int ln = lane_id();
  for (int g = slot; g < count; g += slots) {
    const DevInst& I = insts[g];
    const SlackOut& O = outs[g];
    const int n = I.n;
    const long long ms = forward_pass(I, O.dur, P.W.estart, C);
    backward_pass(I, O.dur, P.W.lend, ms, C);
    // latest of the source node: min over source out-edges of latest[2v]
    long long ls = ms;
    for (int j = ln; j < I.ne; j += 32)
      if (I.dep_tail[j] == n && I.dep_head[j] < n) {
        const int v = I.dep_head[j];
        const long long c = P.W.lend[v] - O.dur[v];
        if (c < ls) ls = c;
      }
    ls = wmin(ls);
    for (int i = ln; i < n; i += 32) {
      O.earliest[2 * i] = P.W.estart[i];
      O.earliest[2 * i + 1] = P.W.estart[i] + O.dur[i];
      O.latest[2 * i + 1] = P.W.lend[i];
      O.latest[2 * i] = P.W.lend[i] - O.dur[i];
      O.critical[i] = P.W.estart[i] + O.dur[i] == P.W.lend[i];
    }
    if (ln == 0) {
      O.earliest[2 * n] = 0;
      O.latest[2 * n] = ls;
      O.earliest[2 * n + 1] = ms;
      O.latest[2 * n + 1] = ms;
      makespan[g] = ms;
    }
    for (int j = ln; j < I.ne; j += 32) {
      const int u = I.dep_tail[j], v = I.dep_head[j];
      long long te, tl, he, hl;
      if (u == n) {
        te = 0;
        tl = ls;
      } else {
        te = P.W.estart[u] + O.dur[u];
        tl = P.W.lend[u];
      }
      if (v == n + 1) {
        he = ms;
        hl = ms;
      } else {
        he = P.W.estart[v];
        hl = P.W.lend[v] - O.dur[v];
      }
      O.critical[n + j] = te == tl && he == hl && te == he;
    }
    __syncwarp();
  }
}

int blocks_for(int slots) { return (slots + kWarpsPerBlock - 1) / kWarpsPerBlock; }

}  // namespace

int walk_slots_per_sm() {
  int blocks = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, walk_kernel, kBlock, 0);
  return blocks * kWarpsPerBlock;
}

int launch_walks(const DevInst* d_insts, int32_t n_inst, const int32_t* d_order, int32_t* d_counter,
                 char* d_ws, const WsLayout& ws, int32_t slots, RunCounters* d_counters,
                 DeltaPool pool, void* stream) {
  walk_kernel<<<blocks_for(slots), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      d_insts, n_inst, d_order, d_counter, d_ws, ws, slots, d_counters, pool);
  return static_cast<int>(cudaGetLastError());
}

int launch_flow_jobs(const DevFlowJob* d_jobs, int32_t count, char* d_ws, const WsLayout& ws,
                     int32_t slots, void* stream) {
  flow_kernel<<<blocks_for(slots), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(d_jobs, count, d_ws,
                                                                                   ws, slots);
  return static_cast<int>(cudaGetLastError());
}

int launch_slack_jobs(const DevInst* d_insts, const SlackOut* d_outs, int64_t* d_makespan,
                      int32_t count, char* d_ws, const WsLayout& ws, int32_t slots, void* stream) {
  slack_kernel<<<blocks_for(slots), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      d_insts, d_outs, d_makespan, count, d_ws, ws, slots);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace pb
