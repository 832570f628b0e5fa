// sm_100a kernels of the B200-native Perseus frontier generator.
//
// One WARP walks one instance's whole frontier (frontier.hpp:166-189) inside
// a single persistent launch: warps pull instances (LPT order) from a global
// counter, so thousands of walks are in flight and no host round trip
// happens per step.  The graphs are deep and narrow (<= ~2N nodes per level,
// SURVEY.md §7 hard part 7), so a warp covers a level; all synchronization
// is __syncwarp, all appends are ballot compactions, and deduplication is
// __match_any_sync + a round stamp (no global atomics with return values on
// the critical path).  Per step:
//
//   K2  longest path over static node-DAG levels (annotate_slack,
//       dag.hpp:233-286; simulate, emulator.hpp:28-55): pull-based,
//       deterministic;
//   K3  fused critical mask + Eq. 7 capacities (build_capacity_dag,
//       flow.hpp:285-317) from host-tabulated curve values, with the
//       reference's int128 overflow checks (flow.hpp:58-68, 196-197);
//   K4  push-relabel max flow with lower bounds: phase A = feasibility
//       circulation with netted demands (flow.hpp:172-203), phase B =
//       source->sink max preflow on the same residual arrays
//       (flow.hpp:205-228), global relabel by backward BFS;
//   K5  minimal min cut = residual reachability from {s} U {excess nodes}
//       (min_cut_from_flow's source side, flow.hpp:234-278), tau update with
//       the reference's skip rules (frontier.hpp:111-131), discretize
//       (frontier.hpp:140-161), realized longest path, append-only delta log.
//
// Only the unique minimal min cut and the two verdicts (feasible, value >=
// sentinel) feed the outputs, so the flow algorithm is free to differ from
// the reference's Edmonds-Karp (SURVEY.md §7 parity rule 1).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "pb_internal.h"

namespace pb {
namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int kBlock = 32 * kWarpsPerBlock;
constexpr unsigned kFull = 0xffffffffu;
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

__device__ __forceinline__ long long ldcg(const int64_t* p) { return __ldcg(p); }
__device__ __forceinline__ void red_add(int64_t* p, long long d) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(d));
}

struct Counters {
  unsigned long long arc_scans = 0, node_updates = 0, rounds = 0, comp_visits = 0;
  unsigned long long prof[kPrSlots] = {};
  __device__ void add(int slot, long long v) {
    if (lane_id() == 0) prof[slot] += static_cast<unsigned long long>(v);
  }
  __device__ void maxv(int slot, long long v) {
    if (lane_id() == 0 && static_cast<unsigned long long>(v) > prof[slot]) prof[slot] = v;
  }
};

__device__ __forceinline__ long long now() { return clock64(); }

// Flow-network view of one warp's workspace.
struct Net {
  int V, E, src, snk, ret;  // E counts graph edges + the return arc (index ret)
  const int32_t* inc_off;
  const int32_t* inc;  // (edge << 1) | dir, dir = 1 when the node is the head
  const int32_t* tail;
  const int32_t* head;
  int64_t* lower;
  int64_t* cap;   // resolved upper - lower (0 for absent edges)
  int64_t* flow;  // f - lower
  uint8_t* einf;
  uint8_t* ecrit;
  int64_t* excess;
  int64_t* tres;  // phase-A residual to the super sink t'
  int32_t* height;
  int32_t* mark;
  uint8_t* nr;
  int32_t* side;
  int32_t* list0;
  int32_t* list1;
  int32_t* bfs0;
  int32_t* bfs1;
  int32_t* dead;
  int32_t* dem;  // nodes with a super-sink arc (phase A)
  int32_t* tgt;  // push targets of one round (with duplicates)
  // warp-uniform bookkeeping
  int n_dead, n_dem, stamp, flag;
};

__device__ __forceinline__ long long residual_out(const Net& N, int a) {
  const int ed = a >> 1;
  return (a & 1) ? N.flow[ed] : N.cap[ed] - N.flow[ed];
}
__device__ __forceinline__ int other_end(const Net& N, int a) {
  const int ed = a >> 1;
  return (a & 1) ? N.tail[ed] : N.head[ed];
}

// Global relabel: exact residual distances to the sink (phase B) or to the
// super sink t' (phase A; distance 1 for nodes with tres > 0).  Unreached
// nodes get H.  Heights only grow, so labels stay valid.
__device__ void global_relabel(Net& N, bool phaseA, int H, Counters& C) {
  const int ln = lane_id();
  const long long t0 = now();
  C.add(kPrGrCalls, 1);
  for (int v = ln; v < N.V; v += 32) N.height[v] = H;
  __syncwarp();
  int cnt = 0;
  if (phaseA) {
    for (int base = 0; base < N.n_dem; base += 32) {
      const int i = base + ln;
      const int v = i < N.n_dem ? N.dem[i] : 0;
      const bool ok = i < N.n_dem && N.tres[v] > 0;
      if (ok) N.height[v] = 1;
      wappend(ok, v, N.bfs0, cnt);
    }
  } else {
    if (ln == 0) {
      N.height[N.snk] = 0;
      N.bfs0[0] = N.snk;
    }
    cnt = 1;
  }
  __syncwarp();
  int32_t* F = N.bfs0;
  int32_t* G = N.bfs1;
  int level = phaseA ? 1 : 0;
  while (cnt > 0) {
    C.add(kPrGrLevels, 1);
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
        int u = 0;
        if (j < deg) {
          const int a = N.inc[off + j];
          const int ed = a >> 1;
          u = (a & 1) ? N.tail[ed] : N.head[ed];
          // arc u -> w: forward of ed when w is the head, backward otherwise
          const long long r = (a & 1) ? N.cap[ed] - N.flow[ed] : N.flow[ed];
          cand = r > 0 && N.height[u] == H && (phaseA || u != N.src);
        }
        // one writer per distinct u among the lanes of this instruction
        const unsigned peers = __match_any_sync(kFull, cand ? u : -1 - ln);
        const bool lead = cand && (__ffs(peers) - 1) == ln;
        if (lead) N.height[u] = level + 1;
        wappend(lead, u, G, nc);
        __syncwarp();
      }
    }
    __syncwarp();
    cnt = nc;
    ++level;
    int32_t* t = F;
    F = G;
    G = t;
  }
  C.add(kPrGr, now() - t0);
}

// Keeps list entries with excess and height < H.  Phase A: excess stranded
// at H means the circulation is infeasible (N.flag).  Phase B: stranded
// excess goes to the dead list (it seeds the cut BFS).
__device__ int filter_active(Net& N, bool phaseA, int H, const int32_t* from, int cnt, int32_t* to) {
  const int ln = lane_id();
  int out = 0;
  for (int base = 0; base < cnt; base += 32) {
    const int i = base + ln;
    const int v = i < cnt ? from[i] : 0;
    const bool has = i < cnt && ldcg(&N.excess[v]) > 0;
    const bool live = has && N.height[v] < H;
    const bool stuck = has && !live;
    if (phaseA) {
      if (__any_sync(kFull, stuck)) N.flag = 1;
    } else {
      wappend(stuck, v, N.dead, N.n_dead);
    }
    wappend(live, v, to, out);
  }
  __syncwarp();
  return out;
}

// Dedups the round's push targets (+ nodes keeping excess) into the next
// worklist: __match_any_sync elects one lane per node within a chunk, the
// round stamp filters repeats across chunks.
__device__ int build_next(Net& N, int ntgt, int32_t* nxt) {
  const int ln = lane_id();
  ++N.stamp;
  const int stamp = N.stamp;
  int cnt = 0;
  for (int base = 0; base < ntgt; base += 32) {
    const int i = base + ln;
    const bool valid = i < ntgt;
    const int w = valid ? N.tgt[i] : 0;
    const unsigned peers = __match_any_sync(kFull, valid ? w : -1 - ln);
    bool fresh = valid && (__ffs(peers) - 1) == ln && N.mark[w] != stamp;
    if (fresh) N.mark[w] = stamp;
    wappend(fresh, w, nxt, cnt);
    __syncwarp();
  }
  return cnt;
}

// Synchronous push-relabel rounds.  Push sub-phase: every active node pushes
// along admissible arcs (h(v) == h(w) + 1) against a fixed height snapshot,
// so each arc has one writer per sub-phase; excess arrives by integer REDs
// (order-independent).  Relabel sub-phase: nodes left with excess take
// 1 + min residual-neighbour height (valid under concurrent relabels because
// heights only increase).  Returns 0 when no active node is left, 1 if
// phase A proves infeasibility, 2 if the round watchdog fires (a bug guard
// that turns a would-be hang into a PB_ERR_LOGIC status).
__device__ int push_relabel(Net& N, bool phaseA, int H, int cnt, Counters& C) {
  const int ln = lane_id();
  int32_t* cur = N.list0;
  int32_t* nxt = N.list1;
  long long relabels_since = 0;
  const long long gr_threshold = N.V > 64 ? N.V : 64;
  const long long max_rounds = 64ll * N.V + 100000;
  long long rounds = 0;
  while (cnt > 0) {
    C.add(phaseA ? kPrRoundsA : kPrRoundsB, 1);
    ++C.rounds;
    if (++rounds > max_rounds) return 2;
    C.maxv(kPrMaxRounds, rounds);
    // ---- push
    int ntgt = 0;
    for (int base = 0; base < cnt; base += 32) {
      const int i = base + ln;
      const bool valid = i < cnt;
      const int v = valid ? cur[i] : 0;
      const int hv = valid ? N.height[v] : H;
      long long e = valid ? ldcg(&N.excess[v]) : 0;
      const bool act = valid && e > 0 && hv < H;
      long long pushed = 0;
      if (phaseA && act && hv == 1) {
        const long long tr = N.tres[v];
        if (tr > 0) {
          const long long d = e < tr ? e : tr;
          N.tres[v] = tr - d;
          e -= d;
          pushed += d;
          ++C.node_updates;
        }
      }
      const int off = act ? N.inc_off[v] : 0;
      const int deg = act ? N.inc_off[v + 1] - off : 0;
      const int md = wmaxi(deg);
      for (int j = 0; j < md; ++j) {
        bool push = false;
        int w = 0;
        if (j < deg && e > 0) {
          const int a = N.inc[off + j];
          ++C.arc_scans;
          w = other_end(N, a);
          if (N.height[w] == hv - 1) {
            const long long r = residual_out(N, a);
            if (r > 0) {
              const long long d = e < r ? e : r;
              N.flow[a >> 1] += (a & 1) ? -d : d;
              e -= d;
              pushed += d;
              red_add(&N.excess[w], d);
              ++C.node_updates;
              push = phaseA || (w != N.snk && w != N.src);
            }
          }
        }
        wappend(push, w, N.tgt, ntgt);
      }
      if (pushed) red_add(&N.excess[v], -pushed);
      if (act && e > 0) N.nr[v] = 1;
    }
    __syncwarp();
    // ---- relabel
    int relabeled = 0;
    bool stuck_any = false;
    for (int base = 0; base < cnt; base += 32) {
      const int i = base + ln;
      const bool valid = i < cnt;
      const int v = valid ? cur[i] : 0;
      const bool rl = valid && N.nr[v];
      const int off = rl ? N.inc_off[v] : 0;
      const int deg = rl ? N.inc_off[v + 1] - off : 0;
      const int md = wmaxi(deg);
      int mh = INT_MAX;
      if (rl && phaseA && N.tres[v] > 0) mh = 0;
      for (int j = 0; j < md; ++j) {
        if (j < deg) {
          const int a = N.inc[off + j];
          if (residual_out(N, a) > 0) {
            const int hw = N.height[other_end(N, a)];
            mh = hw < mh ? hw : mh;
          }
        }
      }
      if (rl) {
        C.arc_scans += deg;
        N.nr[v] = 0;
        N.height[v] = (mh == INT_MAX || mh + 1 >= H) ? H : mh + 1;
        ++C.node_updates;
      }
      relabeled += __popc(__ballot_sync(kFull, rl));
      __syncwarp();
      const bool has = valid && ldcg(&N.excess[v]) > 0;
      const bool live = has && N.height[v] < H;
      const bool stuck = has && !live;
      wappend(live, v, N.tgt, ntgt);
      if (phaseA) {
        stuck_any |= __any_sync(kFull, stuck);
      } else {
        wappend(stuck, v, N.dead, N.n_dead);
      }
    }
    __syncwarp();
    if (stuck_any) return 1;
    cnt = build_next(N, ntgt, nxt);
    relabels_since += relabeled;
    int32_t* t = cur;
    cur = nxt;
    nxt = t;
    if (cnt > 0 && relabels_since >= gr_threshold) {
      relabels_since = 0;
      global_relabel(N, phaseA, H, C);
      N.flag = 0;
      cnt = filter_active(N, phaseA, H, cur, cnt, nxt);
      if (phaseA && N.flag) return 1;
      t = cur;
      cur = nxt;
      nxt = t;
    }
  }
  return 0;
}

// Reachability from {source} U dead-list (excess) nodes over residual arcs:
// the source side of the minimal minimum cut (flow.hpp:234-262).
__device__ void cut_bfs(Net& N, Counters& C) {
  const int ln = lane_id();
  const long long t0 = now();
  for (int v = ln; v < N.V; v += 32) N.side[v] = 0;
  __syncwarp();
  int cnt = 0;
  if (ln == 0) {
    N.side[N.src] = 1;
    N.bfs0[0] = N.src;
  }
  cnt = 1;
  __syncwarp();
  for (int base = 0; base < N.n_dead; base += 32) {
    const int i = base + ln;
    const int v = i < N.n_dead ? N.dead[i] : 0;
    bool ok = i < N.n_dead && v != N.snk && v != N.src && ldcg(&N.excess[v]) > 0;
    const unsigned peers = __match_any_sync(kFull, ok ? v : -1 - ln);
    ok = ok && (__ffs(peers) - 1) == ln && N.side[v] == 0;
    if (ok) N.side[v] = 1;
    wappend(ok, v, N.bfs0, cnt);
    __syncwarp();
  }
  int32_t* F = N.bfs0;
  int32_t* G = N.bfs1;
  while (cnt > 0) {
    C.add(kPrCutLevels, 1);
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
        int u = 0;
        if (j < deg) {
          const int a = N.inc[off + j];
          if (residual_out(N, a) > 0) {
            u = other_end(N, a);
            cand = N.side[u] == 0;
          }
        }
        const unsigned peers = __match_any_sync(kFull, cand ? u : -1 - ln);
        const bool lead = cand && (__ffs(peers) - 1) == ln;
        if (lead) N.side[u] = 1;
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
  C.add(kPrCut, now() - t0);
}

// Phase A (feasibility) + phase B (max preflow) + value, on a network whose
// lower/cap/einf/ecrit/flow(=0) arrays are set, demand list N.dem (nodes with
// tres > 0) and the initial phase-A worklist in list0 (n_init entries).
// Excess and tres must be zero elsewhere.  Returns 0 ok, 1 infeasible,
// 2 watchdog.  *value = net flow into the sink.
__device__ int solve_flow(Net& N, long long return_cap, int n_init, long long* value, Counters& C,
                          int* detail) {
  const int ln = lane_id();
  long long t0 = now();
  if (N.n_dem > 0 || n_init > 0) {
    if (ln == 0) {
      N.cap[N.ret] = return_cap;
      N.flow[N.ret] = 0;
    }
    __syncwarp();
    const int HA = N.V + 2;
    global_relabel(N, true, HA, C);
    N.flag = 0;
    int cnt = filter_active(N, true, HA, N.list0, n_init, N.list1);
    if (N.flag) return 1;
    for (int i = ln; i < cnt; i += 32) N.list0[i] = N.list1[i];
    __syncwarp();
    const int rc = push_relabel(N, true, HA, cnt, C);
    if (rc == 2) *detail = 1;
    if (rc) return rc;
  }
  C.add(kPrPhaseA, now() - t0);
  t0 = now();
  // ---- phase B: drop the return arc, saturate every residual arc out of s
  if (ln == 0) {
    N.cap[N.ret] = 0;
    N.flow[N.ret] = 0;
  }
  N.n_dead = 0;
  __syncwarp();
  const int HB = N.V;
  int cnt = 0;
  {
    const int off = N.inc_off[N.src], deg = N.inc_off[N.src + 1] - off;
    for (int base = 0; base < deg; base += 32) {
      const int j = base + ln;
      bool ok = false;
      int w = 0;
      if (j < deg) {
        const int a = N.inc[off + j];
        const long long r = residual_out(N, a);
        if (r > 0) {
          w = other_end(N, a);
          N.flow[a >> 1] += (a & 1) ? -r : r;
          red_add(&N.excess[w], r);
          ok = w != N.snk && w != N.src;
        }
      }
      wappend(ok, w, N.tgt, cnt);
    }
  }
  __syncwarp();
  cnt = build_next(N, cnt, N.list1);
  global_relabel(N, false, HB, C);
  if (ln == 0) N.height[N.src] = HB;
  __syncwarp();
  cnt = filter_active(N, false, HB, N.list1, cnt, N.list0);
  if (push_relabel(N, false, HB, cnt, C)) {
    *detail = 2;
    return 2;
  }
  C.add(kPrPhaseB, now() - t0);
  // value = net flow into the sink over graph edges
  long long vloc = 0;
  {
    const int off = N.inc_off[N.snk], deg = N.inc_off[N.snk + 1] - off;
    for (int j = ln; j < deg; j += 32) {
      const int a = N.inc[off + j];
      const int ed = a >> 1;
      if (ed == N.ret || !N.ecrit[ed]) continue;
      const long long f = N.lower[ed] + N.flow[ed];
      vloc += (a & 1) ? f : -f;
    }
  }
  *value = wsum(vloc);
  return 0;
}

// Restores excess == 0 everywhere after phase B (dead nodes, sink).
__device__ void clear_excess(Net& N) {
  const int ln = lane_id();
  for (int i = ln; i < N.n_dead; i += 32) N.excess[N.dead[i]] = 0;
  if (ln == 0) {
    N.excess[N.snk] = 0;
    N.excess[N.src] = 0;
  }
  __syncwarp();
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
  N.stamp = 1;
  N.n_dead = 0;
  N.n_dem = 0;
  N.flag = 0;

  // ---- reset workspace for this instance
  for (int v = ln; v < N.V; v += 32) {
    N.excess[v] = 0;
    N.tres[v] = 0;
    N.mark[v] = 0;
    N.nr[v] = 0;
    N.height[v] = 0;
  }
  for (int e = ln; e < N.E; e += 32) {
    N.flow[e] = 0;
    N.cap[e] = 0;
    N.lower[e] = 0;
    N.ecrit[e] = 0;
    N.einf[e] = 0;
  }
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
    // ---- K3 critical mask + capacities
    const long long tcap = now();
    C.add(kPrSteps, 1);
    i128 suml = 0, sumu = 0;
    long long ninf = 0;
    int n_init = 0;
    N.n_dem = 0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + ln;
      const bool valid = i < n;
      long long l = 0, capv = 0;
      uint8_t inf = 1;
      bool crit = false;
      if (valid) {
        const int c = I.comp_class[i];
        const long long t = W.planned[i];
        crit = W.estart[i] + t == W.lend[i];
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
            capv = (r > l ? r : l) - l;
            inf = 0;
          }
        }
        N.ecrit[i] = crit;
        N.lower[i] = crit ? l : 0;
        N.einf[i] = inf;
        N.cap[i] = crit ? capv : 0;
        N.flow[i] = 0;
        if (crit) {
          suml += l;
          if (!inf)
            sumu += l + capv;
          else
            ++ninf;
        }
        if (crit && l > 0) {
          N.tres[2 * i] = l;
          N.excess[2 * i + 1] = l;
        }
      }
      const bool dem = valid && crit && l > 0;
      wappend(dem, 2 * i, N.dem, N.n_dem);
      wappend(dem, 2 * i + 1, N.list0, n_init);
    }
    for (int j = ln; j < I.ne; j += 32) {
      const int u = I.dep_tail[j], v = I.dep_head[j];
      const int k = n + j;
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
      N.ecrit[k] = crit;
      N.lower[k] = 0;
      N.einf[k] = 1;
      N.cap[k] = 0;
      N.flow[k] = 0;
      if (crit) ++ninf;
    }
    if (ln == 0) {
      N.ecrit[N.ret] = 0;
      N.lower[N.ret] = 0;
      N.einf[N.ret] = 0;
      N.cap[N.ret] = 0;
      N.flow[N.ret] = 0;
    }
    suml = wsum128(suml);
    sumu = wsum128(sumu);
    ninf = wsum(ninf);
    // infinity_sentinel (flow.hpp:58-68) and the aux total (flow.hpp:196-197)
    const i128 sent128 = suml + sumu + 1;
    if (sent128 > static_cast<i128>(LLONG_MAX / 4)) {
      status = PB_ERR_OVERFLOW;
      break;
    }
    const long long sentinel = static_cast<long long>(sent128);
    const i128 aux = sumu + static_cast<i128>(ninf) * sentinel + suml;
    if (aux + 1 > static_cast<i128>(LLONG_MAX / 2)) {
      status = PB_ERR_OVERFLOW;
      break;
    }
    __syncwarp();
    for (int k = ln; k < n + I.ne; k += 32)
      if (N.ecrit[k] && N.einf[k]) N.cap[k] = sentinel - N.lower[k];
    __syncwarp();
    C.add(kPrCap, now() - tcap);
    // ---- K4 max flow with lower bounds
    long long value = 0;
    const int frc = solve_flow(N, static_cast<long long>(aux + 1), n_init, &value, C, &detail);
    if (frc == 2) {
      status = PB_ERR_LOGIC;
      break;
    }
    if (frc) {
      stop = PB_STOP_INFEASIBLE;
      break;
    }
    if (value >= sentinel) {
      clear_excess(N);
      stop = PB_STOP_INFINITE_CUT;
      break;
    }
    // ---- K5 minimal min cut
    cut_bfs(N, C);
    if (N.side[N.snk]) {
      detail = 3;
      status = PB_ERR_LOGIC;
      break;
    }
    const long long tupd = now();
    clear_excess(N);
    long long cost = 0;
    int nd = 0;
    for (int base = 0; base < n + I.ne; base += 32) {
      const int k = base + ln;
      int rec = 0;
      if (k < n + I.ne && N.ecrit[k]) {
        const int a = N.side[N.tail[k]], b = N.side[N.head[k]];
        if (a && !b) {
          cost += N.einf[k] ? sentinel : N.lower[k] + N.cap[k];
          if (k < n) rec = k + 1;
        } else if (!a && b) {
          cost -= N.lower[k];
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
  p.N.excess = reinterpret_cast<int64_t*>(base + L.off_excess);
  p.N.tres = reinterpret_cast<int64_t*>(base + L.off_tres);
  p.N.height = reinterpret_cast<int32_t*>(base + L.off_height);
  p.N.mark = reinterpret_cast<int32_t*>(base + L.off_mark);
  p.N.nr = reinterpret_cast<uint8_t*>(base + L.off_nr);
  p.N.side = reinterpret_cast<int32_t*>(base + L.off_side);
  p.N.lower = reinterpret_cast<int64_t*>(base + L.off_lower);
  p.N.cap = reinterpret_cast<int64_t*>(base + L.off_cap);
  p.N.flow = reinterpret_cast<int64_t*>(base + L.off_flow);
  p.N.einf = reinterpret_cast<uint8_t*>(base + L.off_einf);
  p.N.ecrit = reinterpret_cast<uint8_t*>(base + L.off_ecrit);
  p.N.list0 = reinterpret_cast<int32_t*>(base + L.off_list0);
  p.N.list1 = reinterpret_cast<int32_t*>(base + L.off_list1);
  p.N.bfs0 = reinterpret_cast<int32_t*>(base + L.off_bfs0);
  p.N.bfs1 = reinterpret_cast<int32_t*>(base + L.off_bfs1);
  p.N.dead = reinterpret_cast<int32_t*>(base + L.off_dead);
  p.N.dem = reinterpret_cast<int32_t*>(base + L.off_dem);
  p.N.tgt = reinterpret_cast<int32_t*>(base + L.off_tgt);
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
    atomicAdd(&out->rounds, C.rounds);
    for (int q = 0; q < kPrSlots; ++q) {
      if (q == kPrMaxRounds)
        atomicMax(&out->prof[q], C.prof[q]);
      else
        atomicAdd(&out->prof[q], C.prof[q]);
    }
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
    N.stamp = 1;
    N.n_dead = 0;
    N.n_dem = 0;
    N.flag = 0;
    for (int v = ln; v < N.V; v += 32) {
      N.excess[v] = 0;
      N.tres[v] = 0;
      N.mark[v] = 0;
      N.nr[v] = 0;
      N.height[v] = 0;
    }
    i128 suml = 0, sumu = 0;
    long long ninf = 0;
    for (int e = ln; e < J.m; e += 32) {
      N.lower[e] = J.lower[e];
      N.einf[e] = J.inf[e];
      N.ecrit[e] = 1;
      N.flow[e] = 0;
      suml += J.lower[e];
      if (!J.inf[e])
        sumu += J.upper[e];
      else
        ++ninf;
    }
    if (ln == 0) {
      N.lower[N.ret] = 0;
      N.einf[N.ret] = 0;
      N.ecrit[N.ret] = 0;
      N.flow[N.ret] = 0;
      N.cap[N.ret] = 0;
    }
    suml = wsum128(suml);
    sumu = wsum128(sumu);
    ninf = wsum(ninf);
    const i128 sent128 = suml + sumu + 1;
    int status = PB_OK;
    long long sentinel = 0;
    i128 aux = 0;
    if (sent128 > static_cast<i128>(LLONG_MAX / 4)) {
      status = PB_ERR_OVERFLOW;
    } else {
      sentinel = static_cast<long long>(sent128);
      // aux arcs: sum (resolved upper - lower) + sum lower_in + sum lower_out
      aux = sumu + static_cast<i128>(ninf) * sentinel + suml;
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
    for (int e = ln; e < J.m; e += 32) N.cap[e] = (J.inf[e] ? sentinel : J.upper[e]) - J.lower[e];
    __syncwarp();
    // netted demands per node
    int n_init = 0;
    for (int base = 0; base < N.V; base += 32) {
      const int v = base + ln;
      long long d = 0;
      if (v < N.V)
        for (int j = N.inc_off[v]; j < N.inc_off[v + 1]; ++j) {
          const int a = N.inc[j];
          const int ed = a >> 1;
          if (ed == N.ret) continue;
          d += (a & 1) ? N.lower[ed] : -N.lower[ed];
        }
      if (d > 0) N.excess[v] = d;
      if (d < 0) N.tres[v] = -d;
      wappend(d > 0, v, N.list0, n_init);
      wappend(d < 0, v, N.dem, N.n_dem);
    }
    __syncwarp();
    long long value = 0;
    int detail = 0;
    const int frc = solve_flow(N, static_cast<long long>(aux + 1), n_init, &value, C, &detail);
    if (frc) {
      for (int v = ln; v < N.V; v += 32) {
        N.excess[v] = 0;
        N.tres[v] = 0;
      }
      if (ln == 0) {
        J.status[g] = frc == 2 ? PB_ERR_LOGIC : PB_OK;
        J.feasible[g] = 0;
        J.sentinel[g] = sentinel;
      }
      __syncwarp();
      continue;
    }
    cut_bfs(N, C);
    long long cost = 0;
    for (int e = ln; e < J.m; e += 32) {
      const int a = N.side[N.tail[e]], b = N.side[N.head[e]];
      int8_t dir = 0;
      if (a && !b) {
        cost += J.inf[e] ? sentinel : J.upper[e];
        dir = 1;
      } else if (!a && b) {
        cost -= J.lower[e];
        dir = -1;
      }
      J.cut_dir[e] = dir;
    }
    for (int v = ln; v < N.V; v += 32) J.side[v] = static_cast<uint8_t>(N.side[v]);
    cost = wsum(cost);
    if (ln == 0) {
      J.status[g] = N.side[N.snk] ? PB_ERR_LOGIC : PB_OK;
      J.feasible[g] = 1;
      J.value[g] = value;
      J.sentinel[g] = sentinel;
      J.cost[g] = cost;
    }
    clear_excess(N);
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
