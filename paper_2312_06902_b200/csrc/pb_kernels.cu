// sm_100a kernels of the B200-native Perseus frontier generator.
//
// One CTA walks one instance's whole frontier (frontier.hpp:166-189) in a
// single persistent launch: no host round trip per step.  Per step:
//
//   K2  longest path over the static node-DAG levels (annotate_slack,
//       dag.hpp:233-286, and simulate, emulator.hpp:28-55): pull-based,
//       deterministic, no atomics;
//   K3  fused critical mask + Eq. 7 capacities (build_capacity_dag,
//       flow.hpp:285-317) from host-tabulated curve values E_c[t], with the
//       reference's int128 overflow checks (flow.hpp:58-68, 196-197);
//   K4  push-relabel max flow with lower bounds: phase A is the feasibility
//       circulation (flow.hpp:172-203) with netted demands, phase B the
//       source->sink max preflow on the same residual arrays
//       (flow.hpp:205-228); periodic global relabel by backward BFS;
//   K5  minimal min cut = residual reachability from {s} U {excess nodes}
//       (equal to min_cut_from_flow's source side, flow.hpp:234-278),
//       tau update with the reference's skip rules (frontier.hpp:111-131),
//       discretize (frontier.hpp:140-161), realized longest path, and an
//       append-only delta log instead of full schedules.
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

constexpr int kBlock = 128;
constexpr int kWarps = kBlock / 32;
constexpr unsigned kFull = 0xffffffffu;
typedef __int128 i128;

struct Sh {
  int n_next, n_dead, n_dem, n_bfs, flag, relabels, stamp, n_delta;
  int status, stop, inst, pad;
  long long red[kWarps];
  unsigned long long red_lo[kWarps];
  long long red_hi[kWarps];
  long long b[8];
};

__device__ __forceinline__ long long ld_vol(const int64_t* p) {
  return *reinterpret_cast<const volatile long long*>(p);
}

__device__ __forceinline__ unsigned long long as_ull(long long v) {
  return static_cast<unsigned long long>(v);
}

template <class Op>
__device__ long long block_reduce(long long v, Sh& sh, Op op, long long ident) {
  for (int o = 16; o; o >>= 1) v = op(v, static_cast<long long>(__shfl_xor_sync(kFull, as_ull(v), o)));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh.red[warp] = v;
  __syncthreads();
  long long r = ident;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) r = op(r, sh.red[w]);
  __syncthreads();
  return r;
}

struct OpSum {
  __device__ long long operator()(long long a, long long b) const { return a + b; }
};
struct OpMax {
  __device__ long long operator()(long long a, long long b) const { return a > b ? a : b; }
};
struct OpMin {
  __device__ long long operator()(long long a, long long b) const { return a < b ? a : b; }
};

__device__ i128 block_sum128(i128 v, Sh& sh) {
  for (int o = 16; o; o >>= 1) {
    unsigned long long lo = static_cast<unsigned long long>(v);
    unsigned long long hi = static_cast<unsigned long long>(v >> 64);
    lo = __shfl_xor_sync(kFull, lo, o);
    hi = __shfl_xor_sync(kFull, hi, o);
    v += static_cast<i128>((static_cast<unsigned __int128>(hi) << 64) | lo);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sh.red_lo[warp] = static_cast<unsigned long long>(v);
    sh.red_hi[warp] = static_cast<long long>(v >> 64);
  }
  __syncthreads();
  i128 r = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w)
    r += static_cast<i128>((static_cast<unsigned __int128>(static_cast<unsigned long long>(sh.red_hi[w])) << 64) |
                           sh.red_lo[w]);
  __syncthreads();
  return r;
}

// Flow-network view of one CTA's workspace.
struct Net {
  int V, E, src, snk, ret;  // E counts graph edges + the return arc (index ret)
  const int32_t* inc_off;
  const int32_t* inc;
  const int32_t* tail;
  const int32_t* head;
  int64_t* lower;
  int64_t* cap;  // resolved upper - lower (0 for absent edges)
  int64_t* flow; // f - lower
  uint8_t* einf;
  uint8_t* ecrit;
  int64_t* excess;
  int64_t* tres;  // phase A residual to the super sink t'
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
};

struct Counters {
  unsigned long long arc_scans = 0, node_updates = 0, rounds = 0, comp_visits = 0;
};

// Residual capacity of incidence entry a seen from its own node.
__device__ __forceinline__ long long residual_out(const Net& N, int a) {
  const int ed = a >> 1;
  return (a & 1) ? N.flow[ed] : N.cap[ed] - N.flow[ed];
}
__device__ __forceinline__ int other_end(const Net& N, int a) {
  const int ed = a >> 1;
  return (a & 1) ? N.tail[ed] : N.head[ed];
}

// Global relabel: exact residual distances to the sink (phase B) or to the
// super sink t' (phase A, distance 1 for nodes with tres > 0).  Unreached
// nodes get H.  Heights only grow, so labels stay valid.
__device__ void global_relabel(const Net& N, Sh& sh, bool phaseA, int H, Counters& C) {
  const int tid = threadIdx.x;
  for (int v = tid; v < N.V; v += kBlock) N.height[v] = H;
  if (tid == 0) sh.n_bfs = 0;
  __syncthreads();
  if (phaseA) {
    const int nd = sh.n_dem;
    for (int i = tid; i < nd; i += kBlock) {
      const int v = N.dem[i];
      if (N.tres[v] > 0) {
        N.height[v] = 1;
        N.bfs0[atomicAdd(&sh.n_bfs, 1)] = v;
      }
    }
  } else if (tid == 0) {
    N.height[N.snk] = 0;
    N.bfs0[0] = N.snk;
    sh.n_bfs = 1;
  }
  __syncthreads();
  int cnt = sh.n_bfs;
  int32_t* F = N.bfs0;
  int32_t* G = N.bfs1;
  while (cnt > 0) {
    __syncthreads();
    if (tid == 0) sh.n_bfs = 0;
    __syncthreads();
    for (int i = tid; i < cnt; i += kBlock) {
      const int w = F[i];
      const int hw = N.height[w];
      const int e0 = N.inc_off[w], e1 = N.inc_off[w + 1];
      C.arc_scans += static_cast<unsigned long long>(e1 - e0);
      for (int j = e0; j < e1; ++j) {
        const int a = N.inc[j];
        const int ed = a >> 1;
        const int u = (a & 1) ? N.tail[ed] : N.head[ed];
        // arc u -> w: forward of ed when w is the head, backward otherwise
        const long long r = (a & 1) ? N.cap[ed] - N.flow[ed] : N.flow[ed];
        if (r > 0 && N.height[u] == H && (phaseA || u != N.src)) {
          if (atomicCAS(&N.height[u], H, hw + 1) == H) {
            G[atomicAdd(&sh.n_bfs, 1)] = u;
            ++C.node_updates;
          }
        }
      }
    }
    __syncthreads();
    cnt = sh.n_bfs;
    int32_t* t = F;
    F = G;
    G = t;
  }
  __syncthreads();
}

// Keeps list entries with excess and height < H.  Phase A: excess stranded
// at H means the circulation is infeasible (sets sh.flag).  Phase B:
// stranded excess is recorded in the dead list (it seeds the cut BFS).
__device__ int filter_active(const Net& N, Sh& sh, bool phaseA, int H, int32_t* from, int cnt,
                             int32_t* to) {
  const int tid = threadIdx.x;
  if (tid == 0) sh.n_next = 0;
  __syncthreads();
  for (int i = tid; i < cnt; i += kBlock) {
    const int v = from[i];
    if (N.excess[v] <= 0) continue;
    if (N.height[v] < H) {
      to[atomicAdd(&sh.n_next, 1)] = v;
    } else if (phaseA) {
      sh.flag = 1;
    } else {
      N.dead[atomicAdd(&sh.n_dead, 1)] = v;
    }
  }
  __syncthreads();
  return sh.n_next;
}

// Synchronous push-relabel rounds.  Push sub-phase: every active node pushes
// along admissible arcs (h(v) == h(w) + 1) against a fixed height snapshot,
// so each arc has a single writer per sub-phase; excess arrives by integer
// atomics (order-independent).  Relabel sub-phase: nodes left with excess
// take 1 + min neighbour height (valid under concurrent relabels because
// heights only increase).  Returns 0 when no active node is left, 1 if
// phase A proves infeasibility, 2 if the round watchdog fires (a bug guard:
// it turns a would-be GPU hang into a PB_ERR_LOGIC status).
__device__ int push_relabel(const Net& N, Sh& sh, bool phaseA, int H, int cnt, Counters& C) {
  const int tid = threadIdx.x;
  int32_t* cur = N.list0;
  int32_t* nxt = N.list1;
  int relabels_since = 0;
  const int gr_threshold = N.V > 64 ? N.V : 64;
  const long long max_rounds = 64ll * N.V + 100000;
  long long rounds = 0;
  while (cnt > 0) {
    if (++rounds > max_rounds) return 2;
    if (tid == 0) {
      sh.n_next = 0;
      sh.relabels = 0;
      ++sh.stamp;
    }
    __syncthreads();
    const int stamp = sh.stamp;
    ++C.rounds;
    // ---- push
    for (int i = tid; i < cnt; i += kBlock) {
      const int v = cur[i];
      const int hv = N.height[v];
      long long e = ld_vol(&N.excess[v]);
      if (e <= 0 || hv >= H) continue;
      long long pushed = 0;
      if (phaseA && hv == 1) {
        const long long tr = N.tres[v];
        if (tr > 0) {
          const long long d = e < tr ? e : tr;
          N.tres[v] = tr - d;
          e -= d;
          pushed += d;
          ++C.node_updates;
        }
      }
      const int e0 = N.inc_off[v], e1 = N.inc_off[v + 1];
      for (int j = e0; j < e1 && e > 0; ++j) {
        const int a = N.inc[j];
        ++C.arc_scans;
        const int w = other_end(N, a);
        if (N.height[w] != hv - 1) continue;
        const long long r = residual_out(N, a);
        if (r <= 0) continue;
        const long long d = e < r ? e : r;
        N.flow[a >> 1] += (a & 1) ? -d : d;
        e -= d;
        pushed += d;
        atomicAdd(reinterpret_cast<unsigned long long*>(&N.excess[w]), as_ull(d));
        ++C.node_updates;
        const bool terminal = !phaseA && (w == N.snk || w == N.src);
        if (!terminal && atomicMax(&N.mark[w], stamp) < stamp) nxt[atomicAdd(&sh.n_next, 1)] = w;
      }
      if (pushed) atomicAdd(reinterpret_cast<unsigned long long*>(&N.excess[v]), as_ull(-pushed));
      if (e > 0) N.nr[v] = 1;
    }
    __syncthreads();
    // ---- relabel
    int local_relabels = 0;
    for (int i = tid; i < cnt; i += kBlock) {
      const int v = cur[i];
      if (N.nr[v]) {
        N.nr[v] = 0;
        int mh = INT_MAX;
        if (phaseA && N.tres[v] > 0) mh = 0;
        const int e0 = N.inc_off[v], e1 = N.inc_off[v + 1];
        C.arc_scans += static_cast<unsigned long long>(e1 - e0);
        for (int j = e0; j < e1; ++j) {
          const int a = N.inc[j];
          if (residual_out(N, a) > 0) {
            const int hw = N.height[other_end(N, a)];
            if (hw < mh) mh = hw;
          }
        }
        const int nh = (mh == INT_MAX || mh + 1 >= H) ? H : mh + 1;
        N.height[v] = nh;
        ++local_relabels;
        ++C.node_updates;
      }
      if (N.excess[v] > 0) {
        if (N.height[v] < H) {
          if (atomicMax(&N.mark[v], stamp) < stamp) nxt[atomicAdd(&sh.n_next, 1)] = v;
        } else if (phaseA) {
          sh.flag = 1;
        } else if (atomicMax(&N.mark[v], stamp) < stamp) {
          N.dead[atomicAdd(&sh.n_dead, 1)] = v;
        }
      }
    }
    if (local_relabels) atomicAdd(&sh.relabels, local_relabels);
    __syncthreads();
    if (phaseA && sh.flag) return 1;
    cnt = sh.n_next;
    relabels_since += sh.relabels;
    int32_t* t = cur;
    cur = nxt;
    nxt = t;
    if (cnt > 0 && relabels_since >= gr_threshold) {
      relabels_since = 0;
      global_relabel(N, sh, phaseA, H, C);
      cnt = filter_active(N, sh, phaseA, H, cur, cnt, nxt);
      if (phaseA && sh.flag) return 1;
      t = cur;
      cur = nxt;
      nxt = t;
    }
  }
  return 0;
}

// Reachability from {source} U dead-list (excess) nodes over residual arcs:
// the source side of the minimal minimum cut (flow.hpp:234-262).
__device__ void cut_bfs(const Net& N, Sh& sh, Counters& C) {
  const int tid = threadIdx.x;
  for (int v = tid; v < N.V; v += kBlock) N.side[v] = 0;
  if (tid == 0) sh.n_bfs = 0;
  __syncthreads();
  if (tid == 0) {
    N.side[N.src] = 1;
    N.bfs0[atomicAdd(&sh.n_bfs, 1)] = N.src;
  }
  __syncthreads();
  const int nd = sh.n_dead;
  for (int i = tid; i < nd; i += kBlock) {
    const int v = N.dead[i];
    if (v != N.snk && N.excess[v] > 0 && atomicExch(&N.side[v], 1) == 0)
      N.bfs0[atomicAdd(&sh.n_bfs, 1)] = v;
  }
  __syncthreads();
  int cnt = sh.n_bfs;
  int32_t* F = N.bfs0;
  int32_t* G = N.bfs1;
  while (cnt > 0) {
    __syncthreads();
    if (tid == 0) sh.n_bfs = 0;
    __syncthreads();
    for (int i = tid; i < cnt; i += kBlock) {
      const int w = F[i];
      const int e0 = N.inc_off[w], e1 = N.inc_off[w + 1];
      C.arc_scans += static_cast<unsigned long long>(e1 - e0);
      for (int j = e0; j < e1; ++j) {
        const int a = N.inc[j];
        if (residual_out(N, a) > 0) {
          const int u = other_end(N, a);
          if (N.side[u] == 0 && atomicExch(&N.side[u], 1) == 0) G[atomicAdd(&sh.n_bfs, 1)] = u;
        }
      }
    }
    __syncthreads();
    cnt = sh.n_bfs;
    int32_t* t = F;
    F = G;
    G = t;
  }
  __syncthreads();
}

// Phase A (feasibility) + phase B (max preflow) + value, on a network whose
// lower/cap/einf/ecrit/flow(=0) arrays and demand list are set up, with the
// return arc (index ret) carrying return_cap in phase A.  Excess and tres
// must be zero on entry (restored on exit except for dead/sink excess,
// which the caller clears through clear_excess).
// Returns 0 ok, 1 infeasible, 2 watchdog.  *value = net flow into the sink.
__device__ int solve_flow(const Net& N, Sh& sh, long long return_cap, long long* value,
                          Counters& C) {
  const int tid = threadIdx.x;
  // ---- phase A: demands d(v) = lower_in - lower_out, excess d+ / tres d-
  if (sh.n_dem > 0) {
    if (tid == 0) {
      N.cap[N.ret] = return_cap;
      N.flow[N.ret] = 0;
      sh.n_next = 0;
      sh.flag = 0;
    }
    __syncthreads();
    const int HA = N.V + 2;
    // initial worklist: nodes with positive excess were placed by the caller
    // in list0 (count in sh.n_next).
    global_relabel(N, sh, true, HA, C);
    int cnt = filter_active(N, sh, true, HA, N.list0, sh.b[7], N.list1);
    if (sh.flag) return 1;
    // filter_active wrote into list1; move to list0 for push_relabel
    for (int i = tid; i < cnt; i += kBlock) N.list0[i] = N.list1[i];
    __syncthreads();
    const int rc = push_relabel(N, sh, true, HA, cnt, C);
    if (rc) return rc;
    // all excess delivered: tres are zero, excess zero
  }
  // ---- phase B
  if (tid == 0) {
    N.cap[N.ret] = 0;
    N.flow[N.ret] = 0;
    sh.n_next = 0;
    sh.n_dead = 0;
  }
  __syncthreads();
  const int HB = N.V;
  // saturate every residual arc out of the source
  if (tid == 0) {
    const int e0 = N.inc_off[N.src], e1 = N.inc_off[N.src + 1];
    for (int j = e0; j < e1; ++j) {
      const int a = N.inc[j];
      const long long r = residual_out(N, a);
      if (r <= 0) continue;
      const int w = other_end(N, a);
      N.flow[a >> 1] += (a & 1) ? -r : r;
      N.excess[w] += r;
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int e0 = N.inc_off[N.src], e1 = N.inc_off[N.src + 1];
    for (int j = e0; j < e1; ++j) {
      const int w = other_end(N, N.inc[j]);
      if (w != N.snk && w != N.src && N.excess[w] > 0) {
        // dedup parallel arcs to the same neighbour
        bool seen = false;
        for (int q = 0; q < sh.n_next; ++q)
          if (N.list0[q] == w) { seen = true; break; }
        if (!seen) N.list0[sh.n_next++] = w;
      }
    }
  }
  __syncthreads();
  global_relabel(N, sh, false, HB, C);
  if (tid == 0) N.height[N.src] = HB;
  __syncthreads();
  int cnt = filter_active(N, sh, false, HB, N.list0, sh.n_next, N.list1);
  for (int i = tid; i < cnt; i += kBlock) N.list0[i] = N.list1[i];
  __syncthreads();
  if (push_relabel(N, sh, false, HB, cnt, C)) return 2;
  // value = net flow into the sink over graph edges
  long long vloc = 0;
  {
    const int e0 = N.inc_off[N.snk], e1 = N.inc_off[N.snk + 1];
    for (int j = e0 + tid; j < e1; j += kBlock) {
      const int a = N.inc[j];
      const int ed = a >> 1;
      if (ed == N.ret || !N.ecrit[ed]) continue;
      const long long f = N.lower[ed] + N.flow[ed];
      vloc += (a & 1) ? f : -f;
    }
  }
  *value = block_reduce(vloc, sh, OpSum(), 0);
  return 0;
}

__device__ void clear_excess(const Net& N, Sh& sh) {
  const int tid = threadIdx.x;
  const int nd = sh.n_dead;
  for (int i = tid; i < nd; i += kBlock) N.excess[N.dead[i]] = 0;
  if (tid == 0) {
    N.excess[N.snk] = 0;
    N.excess[N.src] = 0;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ walk

struct Walk {
  const DevInst* I;
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
__device__ long long forward_pass(const DevInst& I, const int64_t* dur, int64_t* start, Sh& sh,
                                  Counters& C) {
  const int tid = threadIdx.x;
  for (int L = 0; L < I.n_levels; ++L) {
    const int b = I.lvl_off[L], e = I.lvl_off[L + 1];
    for (int q = b + tid; q < e; q += kBlock) {
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
    __syncthreads();
  }
  long long ms = 0;
  for (int q = tid; q < I.n_snk; q += kBlock) {
    const int u = I.dep_tail[I.snk_dep[q]];
    if (u < I.n) {
      const long long c = start[u] + dur[u];
      if (c > ms) ms = c;
    }
  }
  return block_reduce(ms, sh, OpMax(), 0);
}

// Backward half of annotate_slack (dag.hpp:272-277): lend[i] = latest time
// of node 2i+1 = min over successors (lend[v] - dur[v]), makespan at the sink.
__device__ void backward_pass(const DevInst& I, const int64_t* dur, int64_t* lend, long long ms,
                              Counters& C) {
  const int tid = threadIdx.x;
  for (int L = I.n_levels - 1; L >= 0; --L) {
    const int b = I.lvl_off[L], e = I.lvl_off[L + 1];
    for (int q = b + tid; q < e; q += kBlock) {
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
    __syncthreads();
  }
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

__device__ void run_walk(const DevInst& I, Net& N, Walk& W, Sh& sh, Counters& C) {
  const int tid = threadIdx.x;
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

  // ---- reset workspace for this instance
  for (int v = tid; v < N.V; v += kBlock) {
    N.excess[v] = 0;
    N.tres[v] = 0;
    N.mark[v] = 0;
    N.nr[v] = 0;
    N.height[v] = 0;
  }
  for (int e = tid; e < N.E; e += kBlock) {
    N.flow[e] = 0;
    N.cap[e] = 0;
    N.lower[e] = 0;
    N.ecrit[e] = 0;
    N.einf[e] = 0;
  }
  int bad = 0;
  long long spe = 0, spt = 0, sre = 0, srt = 0;
  for (int i = tid; i < n; i += kBlock) {
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
  if (tid == 0) {
    sh.stamp = 1;
    sh.status = PB_OK;
    sh.stop = PB_STOP_AT_TMIN;
    sh.flag = 0;
  }
  __syncthreads();
  spe = block_reduce(spe, sh, OpSum(), 0);
  spt = block_reduce(spt, sh, OpSum(), 0);
  sre = block_reduce(sre, sh, OpSum(), 0);
  srt = block_reduce(srt, sh, OpSum(), 0);

  const long long t_min = forward_pass(I, W.pdur, W.estart, sh, C);
  long long t_cur = forward_pass(I, W.planned, W.estart, sh, C);
  long long t_real = forward_pass(I, W.rdur, W.rstart, sh, C);
  const long long t_star = t_cur;
  if (tid == 0) write_point(I, 0, t_cur, t_real, spe, spt, sre, srt, 0, 0, 0, 0, 0);
  int steps = 0;
  int id_total = 0;
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
    // latest time of the edge-centric source node (dag.hpp:272-277)
    // ---- K3 critical mask + capacities
    if (tid == 0) {
      sh.n_dem = 0;
      sh.b[7] = 0;
    }
    __syncthreads();
    i128 suml = 0, sumu = 0;
    long long ninf = 0;
    for (int i = tid; i < n; i += kBlock) {
      const int c = I.comp_class[i];
      const long long t = W.planned[i];
      const bool crit = W.estart[i] + t == W.lend[i];
      long long l = 0, capv = 0;
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
        if (l > 0) {
          N.dem[atomicAdd(&sh.n_dem, 1)] = 2 * i;
          N.tres[2 * i] = l;
          N.excess[2 * i + 1] = l;
          N.list0[atomicAdd(reinterpret_cast<unsigned long long*>(&sh.b[7]), 1ull)] = 2 * i + 1;
        }
      }
    }
    // latest[source] = min over source out-edges of latest[2v] (or makespan)
    for (int j = tid; j < I.ne; j += kBlock) {
      const int u = I.dep_tail[j], v = I.dep_head[j];
      const int k = n + j;
      long long te, he;
      bool tc, hc;
      if (u == n) {
        te = 0;
        tc = true;  // resolved below via src_latest check
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
    if (tid == 0) {
      N.ecrit[N.ret] = 0;
      N.lower[N.ret] = 0;
      N.einf[N.ret] = 0;
      N.cap[N.ret] = 0;
      N.flow[N.ret] = 0;
    }
    suml = block_sum128(suml, sh);
    sumu = block_sum128(sumu, sh);
    ninf = block_reduce(ninf, sh, OpSum(), 0);
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
    for (int k = tid; k < n + I.ne; k += kBlock)
      if (N.ecrit[k] && N.einf[k]) N.cap[k] = sentinel - N.lower[k];
    __syncthreads();
    // ---- K4 max flow with lower bounds
    long long value = 0;
    const int frc = solve_flow(N, sh, static_cast<long long>(aux + 1), &value, C);
    if (frc == 2) {
      status = PB_ERR_LOGIC;
      break;
    }
    if (frc) {
      stop = PB_STOP_INFEASIBLE;
      break;
    }
    if (value >= sentinel) {
      clear_excess(N, sh);
      stop = PB_STOP_INFINITE_CUT;
      break;
    }
    // ---- K5 minimal min cut
    cut_bfs(N, sh, C);
    if (N.side[N.snk]) {
      status = PB_ERR_LOGIC;
      break;
    }
    clear_excess(N, sh);
    if (tid == 0) sh.n_delta = 0;
    __syncthreads();
    long long cost = 0;
    for (int k = tid; k < n + I.ne; k += kBlock) {
      if (!N.ecrit[k]) continue;
      const int a = N.side[N.tail[k]], b = N.side[N.head[k]];
      if (a && !b) {
        cost += N.einf[k] ? sentinel : N.lower[k] + N.cap[k];
        if (k < n) W.delta[atomicAdd(&sh.n_delta, 1)] = k + 1;
      } else if (!a && b) {
        cost -= N.lower[k];
        if (k < n) {
          const int c = I.comp_class[k];
          if (!I.cls_const[c] && W.planned[k] + step <= I.cls_tmax[c])
            W.delta[atomicAdd(&sh.n_delta, 1)] = -(k + 1);
        }
      }
    }
    cost = block_reduce(cost, sh, OpSum(), 0);
    const int nd = sh.n_delta;
    if (id_total + nd > I.cap_ids) {
      status = kStatusLogFull;
      break;
    }
    // order: sped ascending, then slowed ascending (frontier.hpp:111-125)
    int ns_loc = 0;
    long long dpe = 0, dpt = 0, dre = 0, drt = 0;
    for (int q = tid; q < nd; q += kBlock) {
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
      I.ids[id_total + rank] = x;
      I.choice[id_total + rank] = static_cast<uint8_t>(chnew);
    }
    // all reads of planned/choice for the deltas happen before the writes
    __syncthreads();
    for (int q = tid; q < nd; q += kBlock) {
      const int x = W.delta[q];
      const int i = (x > 0 ? x : -x) - 1;
      const int c = I.comp_class[i];
      const long long tnew = x > 0 ? W.planned[i] - step : W.planned[i] + step;
      W.planned[i] = tnew;
      const int ch = discretize_choice(I, c, tnew);
      W.choice[i] = static_cast<uint8_t>(ch);
      W.rdur[i] = I.pt_time[I.cls_pt_off[c] + ch];
    }
    const int ns = static_cast<int>(block_reduce(ns_loc, sh, OpSum(), 0));
    dpe = block_reduce(dpe, sh, OpSum(), 0);
    dpt = block_reduce(dpt, sh, OpSum(), 0);
    dre = block_reduce(dre, sh, OpSum(), 0);
    drt = block_reduce(drt, sh, OpSum(), 0);
    // refresh_totals (frontier.hpp:64-67): new planned makespan
    const long long t_new = forward_pass(I, W.planned, W.estart, sh, C);
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
    t_real = forward_pass(I, W.rdur, W.rstart, sh, C);
    ++steps;
    if (tid == 0) write_point(I, steps, t_cur, t_real, spe, spt, sre, srt, cost, step, id_total, ns, nd - ns);
    id_total += nd;
  }
  const long long n_extrap = block_reduce(bad, sh, OpSum(), 0);
  if (tid == 0) {
    pb_frontier_summary s;
    s.n_extrapolated = static_cast<int32_t>(n_extrap);
    s.t_min = t_min;
    s.t_star = t_star;
    s.steps = steps;
    s.stop = stop;
    s.status = status;
    s.n_ids = id_total;
    s.pad = 0;
    *I.summary = s;
  }
  __syncthreads();
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
  atomicAdd(&out->arc_scans, C.arc_scans);
  atomicAdd(&out->node_updates, C.node_updates);
  if (threadIdx.x == 0) atomicAdd(&out->rounds, C.rounds);
  atomicAdd(&out->comp_visits, C.comp_visits);
}

__global__ void __launch_bounds__(kBlock) walk_kernel(const DevInst* insts, int n_inst,
                                                      const int32_t* order, int32_t* counter,
                                                      char* ws_base, WsLayout L,
                                                      RunCounters* ctr) {
  __shared__ Sh sh;
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(blockIdx.x) * L.stride, L);
  Counters C;
  for (;;) {
    if (threadIdx.x == 0) sh.inst = atomicAdd(counter, 1);
    __syncthreads();
    const int k = sh.inst;
    __syncthreads();
    if (k >= n_inst) break;
    P.W.I = &insts[order[k]];
    run_walk(insts[order[k]], P.N, P.W, sh, C);
  }
  flush_counters(C, ctr);
}

// ------------------------------------------------------------ flow jobs

__global__ void __launch_bounds__(kBlock) flow_kernel(const DevFlowJob* jobs, int count,
                                                      char* ws_base, WsLayout L) {
  __shared__ Sh sh;
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(blockIdx.x) * L.stride, L);
  Net& N = P.N;
  Counters C;
  const int tid = threadIdx.x;
  for (int g = blockIdx.x; g < count; g += gridDim.x) {
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
    for (int v = tid; v < N.V; v += kBlock) {
      N.excess[v] = 0;
      N.tres[v] = 0;
      N.mark[v] = 0;
      N.nr[v] = 0;
      N.height[v] = 0;
    }
    if (tid == 0) {
      sh.stamp = 1;
      sh.n_dem = 0;
      sh.b[7] = 0;
      sh.flag = 0;
    }
    i128 suml = 0, sumu = 0;
    long long ninf = 0;
    for (int e = tid; e < J.m; e += kBlock) {
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
    if (tid == 0) {
      N.lower[N.ret] = 0;
      N.einf[N.ret] = 0;
      N.ecrit[N.ret] = 0;
      N.flow[N.ret] = 0;
      N.cap[N.ret] = 0;
    }
    suml = block_sum128(suml, sh);
    sumu = block_sum128(sumu, sh);
    ninf = block_reduce(ninf, sh, OpSum(), 0);
    const i128 sent128 = suml + sumu + 1;
    int status = PB_OK;
    long long sentinel = 0;
    i128 aux = 0;
    if (sent128 > static_cast<i128>(LLONG_MAX / 4)) {
      status = PB_ERR_OVERFLOW;
    } else {
      sentinel = static_cast<long long>(sent128);
      // aux arcs: sum (resolved upper - lower) + sum lower_in + sum lower_out
      aux = sumu + static_cast<i128>(ninf) * sentinel - suml + 2 * suml;
      if (aux + 1 > static_cast<i128>(LLONG_MAX / 2)) status = PB_ERR_OVERFLOW;
    }
    if (status != PB_OK) {
      if (tid == 0) {
        J.status[g] = status;
        J.feasible[g] = 0;
      }
      __syncthreads();
      continue;
    }
    for (int e = tid; e < J.m; e += kBlock)
      N.cap[e] = (J.inf[e] ? sentinel : J.upper[e]) - J.lower[e];
    __syncthreads();
    // netted demands per node
    for (int v = tid; v < N.V; v += kBlock) {
      long long d = 0;
      for (int j = N.inc_off[v]; j < N.inc_off[v + 1]; ++j) {
        const int a = N.inc[j];
        const int ed = a >> 1;
        if (ed == N.ret) continue;
        d += (a & 1) ? N.lower[ed] : -N.lower[ed];
      }
      if (d > 0) {
        N.excess[v] = d;
        N.list0[atomicAdd(reinterpret_cast<unsigned long long*>(&sh.b[7]), 1ull)] = v;
      } else if (d < 0) {
        N.tres[v] = -d;
        N.dem[atomicAdd(&sh.n_dem, 1)] = v;
      }
    }
    __syncthreads();
    long long value = 0;
    const int frc = solve_flow(N, sh, static_cast<long long>(aux + 1), &value, C);
    if (frc) {
      // reset phase-A state for the next job
      for (int v = tid; v < N.V; v += kBlock) {
        N.excess[v] = 0;
        N.tres[v] = 0;
      }
      if (tid == 0) {
        J.status[g] = frc == 2 ? PB_ERR_LOGIC : PB_OK;
        J.feasible[g] = 0;
        J.sentinel[g] = sentinel;
      }
      __syncthreads();
      continue;
    }
    cut_bfs(N, sh, C);
    long long cost = 0;
    for (int e = tid; e < J.m; e += kBlock) {
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
    for (int v = tid; v < N.V; v += kBlock) J.side[v] = static_cast<uint8_t>(N.side[v]);
    cost = block_reduce(cost, sh, OpSum(), 0);
    if (tid == 0) {
      J.status[g] = N.side[N.snk] ? PB_ERR_LOGIC : PB_OK;
      J.feasible[g] = 1;
      J.value[g] = value;
      J.sentinel[g] = sentinel;
      J.cost[g] = cost;
    }
    clear_excess(N, sh);
  }
}

// ------------------------------------------------------------ slack jobs

__global__ void __launch_bounds__(kBlock) slack_kernel(const DevInst* insts, const SlackOut* outs,
                                                       int64_t* makespan, int count,
                                                       char* ws_base, WsLayout L) {
  __shared__ Sh sh;
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(blockIdx.x) * L.stride, L);
  Counters C;
  const int tid = threadIdx.x;
  for (int g = blockIdx.x; g < count; g += gridDim.x) {
    const DevInst& I = insts[g];
    const SlackOut& O = outs[g];
    const int n = I.n;
    const long long ms = forward_pass(I, O.dur, P.W.estart, sh, C);
    backward_pass(I, O.dur, P.W.lend, ms, C);
    // latest of the source node: min over source out-edges of latest[2v]
    long long ls = ms;
    for (int j = tid; j < I.ne; j += kBlock)
      if (I.dep_tail[j] == n && I.dep_head[j] < n) {
        const int v = I.dep_head[j];
        const long long c = P.W.lend[v] - O.dur[v];
        if (c < ls) ls = c;
      }
    ls = block_reduce(ls, sh, OpMin(), ms);
    for (int i = tid; i < n; i += kBlock) {
      O.earliest[2 * i] = P.W.estart[i];
      O.earliest[2 * i + 1] = P.W.estart[i] + O.dur[i];
      O.latest[2 * i + 1] = P.W.lend[i];
      O.latest[2 * i] = P.W.lend[i] - O.dur[i];
      O.critical[i] = P.W.estart[i] + O.dur[i] == P.W.lend[i];
    }
    if (tid == 0) {
      O.earliest[2 * n] = 0;
      O.latest[2 * n] = ls;
      O.earliest[2 * n + 1] = ms;
      O.latest[2 * n + 1] = ms;
      makespan[g] = ms;
    }
    for (int j = tid; j < I.ne; j += kBlock) {
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
    __syncthreads();
  }
}

}  // namespace

int walk_slots_per_sm() {
  int blocks = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, walk_kernel, kBlock, 0);
  return blocks;
}

int launch_walks(const DevInst* d_insts, int32_t n_inst, const int32_t* d_order, int32_t* d_counter,
                 char* d_ws, const WsLayout& ws, int32_t slots, RunCounters* d_counters,
                 void* stream) {
  walk_kernel<<<slots, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      d_insts, n_inst, d_order, d_counter, d_ws, ws, d_counters);
  return static_cast<int>(cudaGetLastError());
}

int launch_flow_jobs(const DevFlowJob* d_jobs, int32_t count, char* d_ws, const WsLayout& ws,
                     int32_t slots, void* stream) {
  flow_kernel<<<slots, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(d_jobs, count, d_ws, ws);
  return static_cast<int>(cudaGetLastError());
}

int launch_slack_jobs(const DevInst* d_insts, const SlackOut* d_outs, int64_t* d_makespan,
                      int32_t count, char* d_ws, const WsLayout& ws, int32_t slots, void* stream) {
  slack_kernel<<<slots, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(d_insts, d_outs, d_makespan,
                                                                         count, d_ws, ws);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace pb
