// sm_100a kernels of the B200-native Perseus frontier generator.
//
// One WARP walks one instance's whole frontier (frontier.hpp:166-189) inside
// a single persistent launch (walk_kernel): warps pull instances (LPT order)
// from a global counter, so thousands of walks are in flight and no host
// round trip happens per step.  Synchronization is __syncwarp only; appends
// are ballot compactions.  The LPT head (the walks that bound the batch)
// runs in walk_kernel_wide: 2 warps per walk, every BFS level split across
// them (named barriers).  Batches whose walks all get a CTA at once (single
// instances: the drop-in's calls) run in walk_kernel_smem: one warp per CTA,
// the walk's arrays placed in the CTA's shared memory as far as they fit,
// compiled as a latency variant (run_walk<true>).  Per step:
//
//   K2  ONE fused longest-path sweep over the level-major computation order:
//       lanes 0-15 run the forward pass (planned AND realized finish times,
//       simulate, emulator.hpp:28-55; earliest, dag.hpp:266-271), lanes 16-31
//       the backward pass (tail lengths; latest = makespan - tail,
//       dag.hpp:272-277).  Static per-level data is software-pipelined one
//       level ahead, so a level waits on one dependent load;
//   K3  fused critical mask + Eq. 7 capacities (build_capacity_dag,
//       flow.hpp:285-317) from host-tabulated curve values, with the
//       reference's int128 overflow checks (flow.hpp:58-68, 196-197).  Flows
//       persist across steps (warm start) and are clamped into the new
//       bounds; infinite edges store -(f + 1) so the sentinel can change
//       without touching them;
//   K4  max flow with lower bounds: the clamp imbalances are repaired by
//       multi-source BFS augmentation in the circulation network with the
//       return arc sink->source (phase A = the feasibility test of
//       flow.hpp:172-203), then source->sink BFS augmentation (phase B,
//       flow.hpp:205-228).  A BFS level loads {ient[p], resid[p]} for its
//       arcs in parallel; the visited set is a shared-memory bitset; a node
//       reached with a positive computation-arc residual brings its partner
//       node into the same level (pok bitset), halving BFS depth;
//   K5  the last phase-B BFS (sink unreachable) marks exactly the source
//       side of the minimal minimum cut (min_cut_from_flow, flow.hpp:234-262);
//       tau update with the reference's skip rules (frontier.hpp:111-131),
//       discretize (frontier.hpp:140-161), append-only delta log.
//
// Also here: the component kernels behind pb_flow_min_cut_batch and
// pb_annotate_slack_batch, the straggler sweep (pb_batch_straggler) and the
// exhaustive oracle (pb_batch_brute_force).
//
// Only the unique minimal min cut and the two verdicts (feasible, value >=
// sentinel) feed the outputs, so the flow itself is free to differ from the
// reference's Edmonds-Karp flow (SURVEY.md §7 parity rule 1).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstdint>
#include <map>
#include <tuple>
#include <type_traits>

#include "pb_internal.h"

namespace pb {
namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int kBlock = 32 * kWarpsPerBlock;
#ifndef PB_MIN_BLOCKS
#define PB_MIN_BLOCKS 3
#endif
constexpr int kMinBlocks = PB_MIN_BLOCKS;  // walker blocks per SM the register budget must allow
#ifndef PB_LANE_GROUP_LOG2
#define PB_LANE_GROUP_LOG2 -1
#endif
constexpr int kLaneGroupLog2 = PB_LANE_GROUP_LOG2;  // >= 0 forces lanes per frontier node (experiments)
constexpr unsigned kFull = 0xffffffffu;
constexpr long long kHuge = LLONG_MAX / 4;  // return-arc capacity (never binding)
constexpr int kMaxEnds = 32;               // phase-B path ends kept per BFS
#ifndef PB_WALKER_PAR
#define PB_WALKER_PAR 1
#endif
constexpr bool kWalkerPar = PB_WALKER_PAR;  // walkers chase a compact parent array, not the log
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

__device__ __forceinline__ void red_add(long long* p, long long d) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(d));
}

__device__ __forceinline__ long long now() { return clock64(); }
// L1 prefetch of the line holding p (global); no value returned, never faults.
// Generic form: a prefetch of a shared-memory address (the shared-memory-
// resident walk, walk_kernel_smem) performs no operation.
#ifndef PB_PF_BFS
#define PB_PF_BFS 1
#endif
#ifndef PB_PF_SWEEP
#define PB_PF_SWEEP 1
#endif
__device__ __forceinline__ void pf_l1(const void* p) { asm volatile("prefetch.L1 [%0];" ::"l"(p)); }

// Cooperative (head) walks' BFS loads carry an L2 evict-last policy
// (createpolicy + L2::cache_hint; global memory only): their lines are the
// last the walkers' traffic displaces.
#ifndef PB_HEAD_EVICT_LAST
#define PB_HEAD_EVICT_LAST 1
#endif
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int4 ld_i4_hint(const void* a, unsigned long long pol) {
  int4 v;
  asm volatile("ld.global.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ long long ld_s64_hint(const long long* a, unsigned long long pol) {
  long long v;
  asm volatile("ld.global.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void pf_bfs(const void* p) {
  if (PB_PF_BFS) pf_l1(p);
}
__device__ __forceinline__ void pf_sweep(const void* p) {
  if (PB_PF_SWEEP) pf_l1(p);
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Work counters: per-lane in registers (flushed once per warp), phase
// profile in shared memory (lane 0 only).
struct Counters {
  unsigned arc_scans = 0, node_updates = 0, comp_visits = 0;
  unsigned long long* prof = nullptr;
  __device__ void add(int slot, long long v) {
    if (lane_id() == 0) prof[slot] += static_cast<unsigned long long>(v);
  }
};

// Effective residual of a raw position value: >= 0 is a plain residual;
// < 0 encodes the forward side of an infinite edge carrying f = -raw - 1,
// whose residual is sentinel - f.  Augmentation arithmetic (raw -= d,
// twin += d) is the same for both encodings.
__device__ __forceinline__ long long eff_res(long long raw, long long S) {
  return raw >= 0 ? raw : S + 1 + raw;
}

// Flow-network view of one warp's workspace.
struct Net {
  int V, src, snk, ret_pt, ret_ph, nbitw, fstride;
  const int32_t* inc_off;
  const IEnt* ient;
  long long* resid;
  long long* bal;
  int4* lg;        // BFS log: {arc into the node, arc before it or -1, parent log index, node}
  int32_t* lvl_start;  // first log index of each BFS level of the last BFS
  int32_t* path_log;   // per path arc: its log entry (>= 0) or -1 - tail entry (arc into the sink)
  int last_nlog, last_levels;  // extent of the last BFS (for restarts)
  int32_t* node_li;    // [V] log index of each node marked by the last BFS
  bool prev_valid;     // the bitset / log / levels still describe the last
                       // step's final BFS (reach(s) of its max flow)
  int4* fglob;     // frontier overflow, 2 buffers of fstride entries
  uint32_t s_bits;  // smem (shared-window address) visited bitset
  uint32_t s_pok;   // smem bitset: node x < 2n whose computation arc to x ^ 1 has residual > 0
  uint32_t s_fs;    // smem frontier, 2 buffers of kFrontCap int4 entries
  uint32_t s_ring;  // smem longest-path rings (forward, backward)
  int2* ends;       // smem: phase-B arcs into the sink {position, parent log index}
  int32_t* path;
  int32_t* touch;
  int32_t* exl;
  long long S;  // infinity sentinel of the current network
  long long R;  // flow on the return arc = s->t value
  struct CoopCtl* ctl;  // cooperative BFS (nw > 1 warps of one CTA), else null
  int nw;
  int32_t* par;    // parent log index of every log entry (-1: seed): shared memory on
                   // cooperative / shared-memory-resident walks, else a compact global array
  int par_cap;     // entries par holds (0: none, chase the 16 B log entries)
  // Path-chase anchors (global parent arrays only; off when par is in shared
  // memory, where a hop is cheap): up[li] = par[par_cap + li] = the log index
  // of li's ancestor at the nearest BFS level below li's that is a multiple
  // of kAnc (-1 for a seed).  A frontier entry's .x carries what its
  // children store.
  bool anc;
};
#ifndef PB_ANCHORS
#define PB_ANCHORS 1
#endif
#ifndef PB_ANC_GUARD
#define PB_ANC_GUARD 1
#endif
constexpr int kAnc = 32;  // anchor level spacing (power of two)

constexpr int kCtlBytes = 256;  // shared memory reserved for CoopCtl
// Control block of a cooperative walk CTA (shared memory): warp 0 drives the
// walk and posts each BFS as a job; helper warps join it.
struct CoopCtl {
  int cmd;   // 0 exit, 1 BFS phase B, 2 BFS phase A, 3 capacity-pass dependency edges,
             // 4 capacity-pass criticality (crit_pass)
  int nsrc;
  int start;  // restart level (-1: fresh BFS from the seeds)
  long long S;
  const DevInst* inst;
  int nc[3];                 // next-level sizes, rotating by level
  unsigned long long found;  // phase A: (log index << 32) | node, ~0 = none
  unsigned long long snk_li; // phase B: log index of the sink's discovery, ~0 = none
  // cmd 3 (capacity pass, dependency edges): inputs and per-warp results
  long long ms;
  int ntouch;       // shared touch-list length (cmd 4: heavy-list length)
  int step, kfrom;  // cmd 4: step size changed, first computation with a new finish
  int prev_valid, last_levels;
  int part_jc[4];
  long long part_dinf[4];
  // Termination is decided per level from log indices (< the level's log
  // end), never from state a faster warp may already be changing in the
  // next level -- otherwise warps could leave the level loop at different
  // levels and deadlock on the barriers.
};

__device__ __forceinline__ void bar_sync(int id, int nthreads) {
  // non-aligned form: threads of a warp may arrive from diverged paths
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Explicit shared-memory accessors (the smem base travels in a struct, so
// plain pointers would compile to generic LD/ST).
__device__ __forceinline__ int4 lds128(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, int4 v) {
  asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void atoms_and(uint32_t a, uint32_t m) {
  asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a), "r"(m) : "memory");
}
// Static incidence entry as one 16 B load (generic: the incidence may be
// staged in shared memory, walk_kernel_smem).
__device__ __forceinline__ int4 ldg_ient(const IEnt* p) { return *reinterpret_cast<const int4*>(p); }
__device__ __forceinline__ uint32_t atoms_or(uint32_t a, uint32_t m) {
  uint32_t old;
  asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(m) : "memory");
  return old;
}

__device__ __forceinline__ int4 fread(const Net& N, int buf, int k) {
  return k < kFrontCap ? lds128(N.s_fs + 16u * (buf * kFrontCap + k))
                       : N.fglob[static_cast<size_t>(buf) * N.fstride + k];
}
__device__ __forceinline__ void fwrite(const Net& N, int buf, int k, int4 v) {
  if (k < kFrontCap)
    sts128(N.s_fs + 16u * (buf * kFrontCap + k), v);
  else
    N.fglob[static_cast<size_t>(buf) * N.fstride + k] = v;
}

__device__ __forceinline__ void clear_bits(Net& N) {
  for (int w = lane_id(); w < N.nbitw; w += 32) sts32(N.s_bits + 4u * w, 0u);
  __syncwarp();
}
// true when this call set the bit
__device__ __forceinline__ bool test_and_set(Net& N, int u) {
  const uint32_t m = 1u << (u & 31);
  return (atoms_or(N.s_bits + 4u * (u >> 5), m) & m) == 0;
}
__device__ __forceinline__ void pok_set(Net& N, int x) { atoms_or(N.s_pok + 4u * (x >> 5), 1u << (x & 31)); }
__device__ __forceinline__ void pok_clear(Net& N, int x) { atoms_and(N.s_pok + 4u * (x >> 5), ~(1u << (x & 31))); }
__device__ __forceinline__ bool bit_of(const Net& N, int u) {
  return (lds32(N.s_bits + 4u * (u >> 5)) >> (u & 31)) & 1u;
}

// Seeds frontier slot k (buffer 0) and log entry k with node v.
__device__ __forceinline__ void seed(Net& N, int k, int v) {
  fwrite(N, 0, k, make_int4(k, N.inc_off[v], N.inc_off[v + 1], k));  // .x: children's anchor (level 0)
  N.lg[k] = make_int4(-1 - v, -1, -1, v);
  if (k < N.par_cap) N.par[k] = -1;
  if (N.anc) N.par[N.par_cap + k] = -1;
  N.node_li[v] = k;
}

// Phase B: the arcs of frontier buffer buf (cnt entries) that enter the sink
// with positive residual -> N.ends (at most kMaxEnds).
__device__ int collect_ends(Net& N, int buf, int cnt) {
  const int ln = lane_id();
  const long long negS = -N.S;
  int nend = 0;
  for (int base = 0; base < cnt; base += 32) {
    const int slot = base + ln;
    int4 fe = make_int4(0, 0, 0, 0);
    if (slot < cnt) fe = fread(N, buf, slot);
    const int rounds = wmaxi(fe.z - fe.y);
    for (int r = 0; r < rounds; ++r) {
      const int p = fe.y + r;
      bool end = false;
      if (p < fe.z && ldg_ient(N.ient + p).x == N.snk) {
        const long long w = N.resid[p];
        end = w != 0 && w >= negS;
      }
      const unsigned m = __ballot_sync(kFull, end);
      const int k = nend + __popc(m & lanemask_lt());
      if (end && k < kMaxEnds) N.ends[k] = make_int2(p, fe.w);
      nend += __popc(m);
    }
  }
  __syncwarp();
  return nend > kMaxEnds ? kMaxEnds : nend;
}

// Level-synchronous BFS over residual arcs from the nsrc seeded sources
// (already marked).  g = 1, 2 or 4 lanes share a frontier node and take its
// arcs round-robin; per arc one {ient, resid} load pair, one unconditional
// shared atomic test-and-set (mask 0 for non-arcs) and one ballot.  The
// frontier lives in shared memory (spilling to global past kFrontCap).
// Phase A (kA): targets are nodes with bal < 0; stops after the level that
// reaches one and returns its log index (tgt = node).  Phase B: stops after
// the level that marks the sink (one shared load per level) and returns the
// number of that level's arcs into the sink, recorded in N.ends (0 = sink
// unreachable; the bitset then marks exactly the residual-reachable set).
// Level-synchronous BFS over residual arcs from the nsrc seeded sources
// (already marked).  g = 1, 2 or 4 lanes share a frontier node and take its
// arcs round-robin; per arc one {ient, resid} load pair, one unconditional
// shared atomic test-and-set (mask 0 for non-arcs), the partner shortcut and
// one ballot.  The frontier lives in shared memory (spilling to global past
// kFrontCap).  kCoop: the nw warps of the CTA split every level (next-level
// slots from a shared counter, one named barrier per level); warp wi.
// Phase A (kA): targets are nodes with bal < 0; stops after the level that
// reaches one and returns its log index (tgt = node).  Phase B: stops after
// the level that marks the sink (one shared load per level) and returns the
// number of that level's arcs into the sink, recorded in N.ends (0 = sink
// unreachable; the bitset then marks exactly the residual-reachable set).
template <bool kA, bool kCoop, bool kLat = false>
__device__ int bfs_core(Net& N, int nsrc, int& tgt, Counters& C, int wi, int start) {
  const int ln = lane_id();
#ifndef PB_WALKER_BFS_EL
#define PB_WALKER_BFS_EL 0
#endif
  // evict-last BFS loads: cooperative walks, and (PB_WALKER_BFS_EL) global-memory walkers
  constexpr bool kHint = PB_HEAD_EVICT_LAST && (kCoop || (PB_WALKER_BFS_EL && !kLat));
  const unsigned long long pol = kHint ? policy_evict_last() : 0ull;
  const unsigned lt = lanemask_lt();
  const int nw = kCoop ? N.nw : 1;
  const long long t0 = now();
  const long long negS = -N.S;  // raw residual r is positive iff r != 0 && r >= -S
  int cnt = nsrc, cur = 0, nlog = nsrc, found = -1, levels = 0, prev = 0;
  if (start >= 0) {
    // restart: levels <= start are kept from the last BFS, frontier buffer 0
    // holds level `start` (prepare_restart)
    levels = start;
    nlog = N.lvl_start[start + 1];
    cnt = nlog - N.lvl_start[start];
  } else if (wi == 0 && ln == 0) {
    N.lvl_start[0] = 0;
    N.lvl_start[1] = nsrc;
  }
  const int levels0 = levels;
  unsigned arcs = 0, upd = 0;
  tgt = -1;
  const uint32_t snk_word = N.s_bits + 4u * (N.snk >> 5), snk_mask = 1u << (N.snk & 31);
  while (cnt > 0) {
    const int per = kCoop ? (cnt + nw - 1) / nw : cnt;
    const int lg2 = kLaneGroupLog2 >= 0 ? kLaneGroupLog2 : (per <= 8 ? 2 : (per <= 16 ? 1 : 0));
    const int g = 1 << lg2;
    const int sub = ln & (g - 1);
    const int nxt = cur ^ 1;
    const uint32_t fcur = N.s_fs + 16u * kFrontCap * cur, fnxt = N.s_fs + 16u * kFrontCap * nxt;
    int4* gcur = N.fglob + static_cast<size_t>(cur) * N.fstride;
    int4* gnxt = N.fglob + static_cast<size_t>(nxt) * N.fstride;
    int* ncp = kCoop ? &N.ctl->nc[levels % 3] : nullptr;  // reset for `levels` done by the poster
    if (kCoop && wi == 0 && ln == 0) N.ctl->nc[(levels + 1) % 3] = 0;
    ++levels;
    const bool anc_lvl = (levels & (kAnc - 1)) == 0;  // this level's discoveries are anchors
    int nc = 0;
    for (int base = wi * (32 >> lg2); base < cnt; base += nw * (32 >> lg2)) {
      const int slot = base + (ln >> lg2);
      int4 fe = make_int4(0, 0, 0, 0);
      if (slot < cnt) fe = slot < kFrontCap ? lds128(fcur + 16u * slot) : gcur[slot];
      int p = fe.y + sub;
      const int mine = fe.z > p ? (fe.z - p + g - 1) >> lg2 : 0;
      const int rounds = wmaxi(mine);
      arcs += mine;
      // software pipeline: round r + 1's {ient, resid} pair is issued before
      // round r is processed (nothing in a BFS writes resid), so a node's
      // arcs cost about one dependent round trip instead of one per round.
      // kLat (shared-memory-resident walks, 255 registers): two register
      // buffers, so a new load never waits on the registers of the one in
      // flight; walkers keep one (register budget, measured)
      int4 ea = make_int4(0, 0, 0, 0), eb = ea;  // {other, packed twin, other_off, other_end}
      long long wa = 0, wb = 0;
      if (p < fe.z) {
        if (kHint) {
          ea = ld_i4_hint(N.ient + p, pol);
          wa = ld_s64_hint(N.resid + p, pol);
        } else {
          ea = ldg_ient(N.ient + p);
          wa = N.resid[p];
        }
      }
      auto round = [&](const int4 e, const long long w, const int p) {
        const bool v = p < fe.z;
        const bool ok = v && w != 0 && w >= negS;  // e, w are stale past this lane's arcs
        const uint32_t m = ok ? 1u << (e.x & 31) : 0u;
        const uint32_t pw = lds32(N.s_pok + 4u * (e.x >> 5));  // issued beside the atomic
        const uint32_t o = atoms_or(N.s_bits + 4u * (e.x >> 5), m);
        const bool c = ok && (o & m) == 0;
        // partner shortcut: a new node y = e.x whose computation arc (first in
        // its list, position e.z) has residual also reaches z = y ^ 1 in this
        // level; z's list is adjacent to y's (pd = its degree)
        const int pd = static_cast<int>(static_cast<unsigned>(e.y) >> kPdegShift);
        bool cz = false;
        if (c && pd != kNoPartner && ((pw >> (e.x & 31)) & 1u)) cz = test_and_set(N, e.x ^ 1);
        const unsigned bm = __ballot_sync(kFull, c);
        const unsigned bz = __ballot_sync(kFull, cz);
        int b0 = nc;
        if (kCoop) {
          const int t = __popc(bm) + __popc(bz);
          if (ln == 0 && t) b0 = atomicAdd(ncp, t);
          b0 = __shfl_sync(kFull, b0, 0);
        }
        const int pos = b0 + __popc(bm & lt);
        const int posz = b0 + __popc(bm) + __popc(bz & lt);
        int hitli = -1, hitnode = -1;
        if (c) {
          const int li = nlog + pos;
          N.lg[li] = make_int4(p, -1, fe.w, e.x);
          if (li < N.par_cap) N.par[li] = fe.w;
          if (N.anc) N.par[N.par_cap + li] = fe.x;
          N.node_li[e.x] = li;
          if (kCoop && !kA && e.x == N.snk) atomicMin(&N.ctl->snk_li, static_cast<unsigned long long>(li));
          const int4 ent = make_int4(anc_lvl ? li : fe.x, e.z, e.w, li);
          // the next level reads this node's arcs: start their DRAM->L1 fill now
          pf_bfs(N.ient + e.z);
          pf_bfs(N.resid + e.z);
          if (pos < kFrontCap)
            sts128(fnxt + 16u * pos, ent);
          else
            gnxt[pos] = ent;
          if (kA && N.bal[e.x] < 0) {
            hitli = li;
            hitnode = e.x;
          }
        }
        if (cz) {
          const int z = e.x ^ 1;
          const int zo = (e.x & 1) ? e.z - pd : e.w;
          const int ze = (e.x & 1) ? e.z : e.w + pd;
          const int lz = nlog + posz;
          N.lg[lz] = make_int4(e.z, p, fe.w, z);  // y's computation arc, the arc into y, y's parent
          if (lz < N.par_cap) N.par[lz] = fe.w;
          if (N.anc) N.par[N.par_cap + lz] = fe.x;
          N.node_li[z] = lz;
          const int4 ent = make_int4(anc_lvl ? lz : fe.x, zo, ze, lz);
          pf_bfs(N.ient + zo);
          pf_bfs(N.resid + zo);
          if (posz < kFrontCap)
            sts128(fnxt + 16u * posz, ent);
          else
            gnxt[posz] = ent;
          if (kA && hitli < 0 && N.bal[z] < 0) {
            hitli = lz;
            hitnode = z;
          }
        }
        if (kA) {
          const unsigned h = __ballot_sync(kFull, hitli >= 0);
          if (h) {
            const int hl = __ffs(h) - 1;
            const int fl = __shfl_sync(kFull, hitli, hl);
            const int fn = __shfl_sync(kFull, hitnode, hl);
            if (kCoop) {
              if (ln == 0)
                atomicMin(&N.ctl->found, (static_cast<unsigned long long>(fl) << 32) | static_cast<unsigned>(fn));
            } else if (found < 0) {
              found = fl;
              tgt = fn;
            }
          }
        }
        if (!kCoop) nc += __popc(bm) + __popc(bz);
        upd += c + cz;
      };
      if (kLat) {
        for (int r = 0; r < rounds; r += 2, p += 2 * g) {
          if (p + g < fe.z) {
            eb = ldg_ient(N.ient + p + g);
            wb = N.resid[p + g];
          }
          round(ea, wa, p);
          if (r + 1 >= rounds) break;
          if (p + 2 * g < fe.z) {
            ea = ldg_ient(N.ient + p + 2 * g);
            wa = N.resid[p + 2 * g];
          }
          round(eb, wb, p + g);
        }
      } else {
        for (int r = 0; r < rounds; ++r, p += g) {
          const int4 e = ea;
          const long long w = wa;
          if (p + g < fe.z) {
            if (kHint) {
              ea = ld_i4_hint(N.ient + p + g, pol);
              wa = ld_s64_hint(N.resid + p + g, pol);
            } else {
              ea = ldg_ient(N.ient + p + g);
              wa = N.resid[p + g];
            }
          }
          round(e, w, p);
        }
      }
    }
    if (kCoop) {
      bar_sync(1, 32 * nw);
      nc = *reinterpret_cast<volatile int*>(ncp);
    } else {
      __syncwarp();
    }
    nlog += nc;
    if (wi == 0 && ln == 0) N.lvl_start[levels + 1] = nlog;  // levels was incremented: next level's end
    prev = cnt;
    cnt = nc;
    cur = nxt;
    bool done;
    if (kA) {
      if (kCoop) {
        const unsigned long long f = *reinterpret_cast<volatile unsigned long long*>(&N.ctl->found);
        if (f != ~0ull && static_cast<int>(f >> 32) < nlog) {  // a hit of THIS level
          found = static_cast<int>(f >> 32);
          tgt = static_cast<int>(f & 0xffffffffu);
        }
      }
      done = found >= 0;
    } else if (kCoop) {
      done = *reinterpret_cast<volatile unsigned long long*>(&N.ctl->snk_li) < static_cast<unsigned long long>(nlog);
    } else {
      done = (lds32(snk_word) & snk_mask) != 0;
    }
    if (done) break;
  }
  if (kCoop) bar_sync(2, 32 * nw);  // every warp is past its last read of shared state
  N.last_nlog = nlog;
  N.last_levels = levels;
  C.arc_scans += arcs;
  C.node_updates += upd;
  C.add(kPrBfsLevels, levels - levels0);
  int ret = found;
  if (!kA) ret = (wi == 0 && (lds32(snk_word) & snk_mask)) ? collect_ends(N, cur ^ 1, prev) : 0;
  C.add(kPrBfs, now() - t0);
  return ret;
}

// Restart after an augmentation (maximize): every node at BFS level <= j
// keeps an unsaturated tree path from the source and no new residual arc
// leaves that set (the augmentation only adds arcs back along its path), so
// a fresh BFS would repeat levels 0..j exactly.  Un-mark the nodes logged
// after level j and reload level j into frontier buffer 0.
__device__ void prepare_restart(Net& N, int j) {
  const int ln = lane_id();
  const int b = N.lvl_start[j], e = N.lvl_start[j + 1];
  for (int i = e + ln; i < N.last_nlog; i += 32) {
    const int v = N.lg[i].w;
    atoms_and(N.s_bits + 4u * (v >> 5), ~(1u << (v & 31)));
  }
  const bool alvl = (j & (kAnc - 1)) == 0;
  for (int i = b + ln; i < e; i += 32) {
    const int v = N.lg[i].w;
    const int a = alvl ? i : (N.anc ? N.par[N.par_cap + i] : 0);
    fwrite(N, 0, i - b, make_int4(a, N.inc_off[v], N.inc_off[v + 1], i));
  }
  __syncwarp();
}

// BFS entry for the walk driver (warp 0): solo, or posted to the CTA's
// helper warps (walk_kernel_wide) and run cooperatively.  start >= 0
// restarts from that level of the last BFS (prepare_restart).
template <bool kA, bool kLat = false>
__device__ int bfs(Net& N, int nsrc, int& tgt, Counters& C, int start = -1) {
  if (start >= 0) prepare_restart(N, start);
  if (N.nw <= 1) return bfs_core<kA, false, kLat>(N, nsrc, tgt, C, 0, start);
  if (lane_id() == 0) {
    CoopCtl* k = N.ctl;
    k->cmd = kA ? 2 : 1;
    k->nsrc = nsrc;
    k->start = start;
    k->S = N.S;
    k->nc[start >= 0 ? start % 3 : 0] = 0;
    k->found = ~0ull;
    k->snk_li = ~0ull;
  }
  __syncwarp();
  bar_sync(1, 32 * N.nw);  // release the helpers
  return bfs_core<kA, true>(N, nsrc, tgt, C, 0, start);
}

// BFS level of log index i in the last BFS (largest L with lvl_start[L] <= i).
__device__ __forceinline__ int level_of(const Net& N, int i) {
  int lo = 0, hi = N.last_levels + 1;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (N.lvl_start[mid] <= i)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Pushes flow along a chain: position `first` (if >= 0), then the logged
// parent links from log index `idx`, for at most `cap` units and, in phase A,
// at most the excess bal[src] of the chain's source.  Lane 0 chases the
// parent links only (one dependent load per hop); the warp then takes the
// bottleneck over the chain's residuals in parallel and updates both sides
// of every arc.  Returns the amount pushed (0 = chain blocked).
__device__ long long push_chain(Net& N, int first, int idx, long long cap, bool phaseA, int& src,
                                Counters& C, int* restart = nullptr) {
  const int ln = lane_id();
  int k = 0, s = -1;
  if (ln == 0 && first >= 0) {
    N.path_log[k] = -1 - idx;  // arc into the sink: its tail is entry idx
    N.path[k++] = first;
  }
  if (N.par_cap > 0) {
    // Cooperative walk: lane 0 follows the parent links in shared memory,
    // collecting the path's log entries (scratch: frontier buffer 1, dead
    // between BFSs); the warp then reads the entries together.
    int* ent = reinterpret_cast<int*>(N.fglob + N.fstride);
    int m = 0;
    if (N.anc) {
      // Global parent array: lane 0 follows the anchors (one hop per kAnc
      // levels) down to the seed; then lane j walks segment j (anchor j to
      // anchor j + 1) through the parent links, all segments at once.  A
      // segment between two anchors spans exactly kAnc levels, one log entry
      // each; the first one (from idx) is shorter.  Chase order does not
      // matter to the callers (bottleneck, update and restart level are
      // order-free), so ent = [seed, segments 1.., segment 0].
      int* cpt = ent + 2 * N.fstride;
      int K = 0;
      if (ln == 0) {
        for (int x = idx; x >= 0; x = N.par[N.par_cap + x]) cpt[K++] = x;
      }
      K = __shfl_sync(kFull, K, 0);
      __syncwarp();
      int len0 = 0;
      for (int j = ln; j < K - 1; j += 32) {
        int x = cpt[j];
        const int stop = cpt[j + 1];
        const int o = j == 0 ? 1 + (K - 2) * kAnc : 1 + (j - 1) * kAnc;
        int t = 0;
        while (x != stop && t < kAnc) {
          ent[o + t++] = x;
          x = N.par[x];
        }
        // a segment that does not span its levels exactly means a broken log: fail loudly
        if (PB_ANC_GUARD && (x != stop || (j > 0 && t != kAnc))) __trap();
        if (j == 0) len0 = t;
      }
      if (ln == 0) ent[0] = cpt[K - 1];
      len0 = __shfl_sync(kFull, len0, 0);
      m = K >= 2 ? 1 + (K - 2) * kAnc + len0 : 1;
    } else if (ln == 0) {
      for (int x = idx; x >= 0; x = N.par[x]) ent[m++] = x;
    }
    m = __shfl_sync(kFull, m, 0);
    k = __shfl_sync(kFull, k, 0);
    __syncwarp();
    // the last entry is the seed (its log x = -1 - source); the others carry
    // one arc, or two through a shortcut, in chase order
    for (int base = 0; base < m; base += 32) {
      const int q = base + ln;
      int4 l = make_int4(0, -1, 0, 0);
      int x = 0;
      if (q < m) {
        x = ent[q];
        l = N.lg[x];
      }
      const bool arc = q < m && l.x >= 0;
      if (q < m && l.x < 0) s = -1 - l.x;
      const bool two = arc && l.y >= 0;
      const unsigned ba = __ballot_sync(kFull, arc), b2 = __ballot_sync(kFull, two);
      const int at = k + __popc(ba & lanemask_lt()) + __popc(b2 & lanemask_lt());
      if (arc) {
        N.path_log[at] = x;
        N.path[at] = l.x;
        if (two) {
          N.path_log[at + 1] = x;
          N.path[at + 1] = l.y;
        }
      }
      k += __popc(ba) + __popc(b2);
    }
    s = static_cast<int>(wmaxi(s));
  } else if (ln == 0) {
    for (;;) {
      const int4 l = N.lg[idx];
      if (l.x < 0) {
        s = -1 - l.x;
        break;
      }
      N.path_log[k] = idx;
      N.path[k++] = l.x;
      if (l.y >= 0) {  // shortcut entry: two arcs per hop
        N.path_log[k] = idx;
        N.path[k++] = l.y;
      }
      idx = l.z;
    }
  }
  k = __shfl_sync(kFull, k, 0);
  src = __shfl_sync(kFull, s, 0);
  __syncwarp();
  long long d = cap;
  for (int q = ln; q < k; q += 32) {
    const long long r = eff_res(N.resid[N.path[q]], N.S);
    d = r < d ? r : d;
  }
  if (phaseA && ln == 0) {
    const long long ex = N.bal[src];
    d = ex < d ? ex : d;
  }
  d = wmin(d);
  C.add(kPrPathHops, k);
  if (ln == 0) C.node_updates += 2 * k;
  if (d <= 0) return 0;
  int jmin = INT_MAX;
  for (int q = ln; q < k; q += 32) {
    const int p = N.path[q];
    const int4 e = ldg_ient(N.ient + p);
    const long long nv = N.resid[p] - d;
    N.resid[p] = nv;
    N.resid[e.y & kTwinMask] += d;
    const bool sat = eff_res(nv, N.S) <= 0;
    if (e.y & kCompArc) {
      // computation arc owner -> e.x (owner = e.x ^ 1): keep the shortcut bits exact
      if (sat) pok_clear(N, e.x ^ 1);
      pok_set(N, e.x);
    }
    if (restart && sat) {
      // a saturated arc logged at level L (entered a node of level L) leaves
      // levels <= L - 1 intact; the arc into the sink leaves its tail's level
      const int pl = N.path_log[q];
      const int j = pl >= 0 ? level_of(N, pl) - 1 : level_of(N, -1 - pl);
      jmin = j < jmin ? j : jmin;
    }
  }
  if (restart) {
    jmin = static_cast<int>(wmin(jmin));
    *restart = jmin < *restart ? jmin : *restart;
  }
  __syncwarp();
  C.add(kPrPaths, 1);
  return d;
}

// Phase A augmentation to the deficit node tgt (log index found): amount =
// min(residuals, bal[src], -bal[tgt]); the balances move.
__device__ void augment_a(Net& N, int found, int tgt, Counters& C) {
  const long long t0 = now();
  int src = -1;
  const long long d = push_chain(N, -1, found, -N.bal[tgt], true, src, C);
  if (d > 0 && lane_id() == 0) {
    N.bal[src] -= d;
    N.bal[tgt] += d;
  }
  __syncwarp();
  C.add(kPrAugment, now() - t0);
}

// Phase B augmentation along every recorded end arc into the sink (paths of
// one BFS level graph; each is re-checked against the current residuals).
// Returns the level the next BFS can restart from (-1: none).
__device__ int augment_b(Net& N, int nend, Counters& C) {
  const long long t0 = now();
  int restart = INT_MAX;
  for (int k = 0; k < nend; ++k) {
    const int2 en = N.ends[k];
    int src;
    N.R += push_chain(N, en.x, en.y, LLONG_MAX, false, src, C, &restart);
  }
  C.add(kPrAugment, now() - t0);
#ifdef PB_NO_RESTART
  return -1;
#else
  return restart == INT_MAX || restart < 0 ? -1 : restart;
#endif
}

// Phase A: repairs the imbalances of the nodes in N.touch (ntouch entries,
// duplicates allowed) in the circulation network (return arc enabled).
// Returns false when some excess cannot reach any deficit: the bounded
// network is infeasible (max_flow_lower_bounds returns nullopt).
template <bool kLat = false>
__device__ bool repair(Net& N, int ntouch, Counters& C) {
  const int ln = lane_id();
  if (ntouch == 0) return true;  // nothing moved: keep the last BFS state
  N.prev_valid = false;          // the dedup below (and any phase-A BFS) reuses the bitset
  clear_bits(N);
  int nex = 0;
  for (int base = 0; base < ntouch; base += 32) {
    const int i = base + ln;
    bool take = false;
    int v = 0;
    if (i < ntouch) {
      v = N.touch[i];
      take = test_and_set(N, v) && N.bal[v] > 0;
    }
    wappend(take, v, N.exl, nex);
  }
  __syncwarp();
  if (nex == 0) return true;
  C.add(kPrImbalanced, nex);
  const long long t0 = now();
  if (ln == 0) {
    N.resid[N.ret_pt] = kHuge - N.R;
    N.resid[N.ret_ph] = N.R;
  }
  __syncwarp();
  bool ok = true;
  for (;;) {
    clear_bits(N);
    int ns = 0;
    for (int base = 0; base < nex; base += 32) {
      const int i = base + ln;
      const int v = i < nex ? N.exl[i] : 0;
      const bool pred = i < nex && N.bal[v] > 0;
      const unsigned m = __ballot_sync(kFull, pred);
      if (pred) {
        const int k = ns + __popc(m & lanemask_lt());
        N.exl[k] = v;
        test_and_set(N, v);
        seed(N, k, v);
      }
      ns += __popc(m);
    }
    __syncwarp();
    if (ns == 0) break;
    nex = ns;
    C.add(kPrBfsA, 1);
    int tgt;
    const int found = bfs<true, kLat>(N, ns, tgt, C);
    if (found < 0) {
      ok = false;
      break;
    }
    augment_a(N, found, tgt, C);
  }
  __syncwarp();
  N.R = N.resid[N.ret_ph];
  __syncwarp();
  if (ln == 0) {
    N.resid[N.ret_pt] = 0;
    N.resid[N.ret_ph] = 0;
  }
  __syncwarp();
  C.add(kPrPhaseA, now() - t0);
  return ok;
}

// Phase B: source->sink augmentation until the sink is unreachable; the
// bitset then marks the minimal min cut's source side.
// first_restart >= 0: the first BFS resumes the last step's final BFS from
// that level (build_caps found no residual change below it).
template <bool kLat = false>
__device__ void maximize(Net& N, Counters& C, int first_restart = -1) {
  const long long t0 = now();
  int restart = N.prev_valid ? first_restart : -1;
  for (;;) {
    if (restart < 0) {
      clear_bits(N);
      if (lane_id() == 0) {
        test_and_set(N, N.src);
        seed(N, 0, N.src);
      }
      __syncwarp();
    }
    C.add(kPrBfsB, 1);
    int tgt;
    const int nend = bfs<false, kLat>(N, 1, tgt, C, restart);
    if (nend <= 0) break;
    restart = augment_b(N, nend, C);
  }
  N.prev_valid = true;  // the final BFS is complete: reach(s) with its levels
  C.add(kPrPhaseB, now() - t0);
}

// ------------------------------------------------------------------ walk

struct Walk {
  long long* durp;   // planned durations
  long long* durr;   // realized (discretized) durations
  long long* fin;    // planned finish
  long long* finr;   // realized finish (the sweep and the realized makespan only)
  long long* tl;     // planned duration + longest tail to the sink
  longlong2* cap;    // {lower, upper; -1 = infinite} of critical computation edges
  uint8_t* ecrit;    // [E] edge in the current critical network
  longlong2* key;    // [n] {critical ? finish : -1, critical ? start : -2} (build_caps):
                     // a dependency edge u -> v is critical iff key[u].x == key[v].y
  uint8_t* dirty;    // [n] duration changed since the capacity was built
  uint8_t* choice;
  int32_t* delta;
};

__device__ __forceinline__ void sts_ll2(uint32_t a, long long x, long long y) {
  asm volatile("st.shared.v2.s64 [%0], {%1, %2};" ::"r"(a), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ longlong2 lds_ll2(uint32_t a) {
  longlong2 v;
  asm volatile("ld.shared.v2.s64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a) : "memory");
  return v;
}
// Fused longest path over the level-major order (K2).  Forward lanes (0-15)
// compute fin[i] = max over predecessors of fin + (dp[i], dr[i]); backward
// lanes (16-31, when `back`) compute tl[i].x = dp[i] + max over successors
// tl.x.  The forward pass covers levels lf..L-1 and the backward pass levels
// lb..0, one level of each per iteration: a walk step changes durations only
// at the computations it sped up or slowed down, so fin is unchanged below
// the lowest of their levels and tl above the highest (lf = 0, lb = L - 1 is
// the full sweep).  The per-level static data (row records, level bounds) and
// the durations are loaded one iteration ahead.
template <bool kLat = false>
__device__ void sweep(const DevInst& I, const long long* dp, const long long* dr, long long* fin,
                      long long* finr, long long* tl, bool back, long long& msp, long long& msr, uint32_t s_ring,
                      Counters& C, int lf = 0, int lb = INT_MAX) {
  const int ln = lane_id();
  const long long t0 = now();
  const bool fwd = ln < 16;
  const int s = ln & 15;
  const int L = I.n_levels;
  if (lb > L - 1) lb = L - 1;
  if (!back) lb = -1;
  const int nf = L - lf, nb = lb + 1;
  const int cnt_me = fwd ? nf : nb;  // levels of this half
  const int iters = max(nf, nb);
  const int4* row = fwd ? I.frow : I.brow;
  const int32_t* noff = fwd ? I.pin_off : I.pout_off;
  const int32_t* nb_ = fwd ? I.pin : I.pout;
  // this half's values: {planned, realized} finish (forward) or the tail
  // length (backward; its realized half is unused)
  auto vload = [&](int m) -> longlong2 { return fwd ? make_longlong2(fin[m], finr[m]) : make_longlong2(tl[m], 0); };
  auto vstore = [&](int i, long long a, long long c) {
    if (fwd) {
      fin[i] = a;
      finr[i] = c;
    } else {
      tl[i] = a;
    }
  };
  const uint32_t ring = (fwd ? s_ring : s_ring + 16u * kRingLevels * 16);
  long long mp = 0, mr = 0;
  C.add(kPrLpLevels, iters);
  auto lev_of = [&](int k) { return fwd ? lf + k : lb - k; };
  // the levels just outside the swept range keep their values: reload their
  // ring slots (row records name ring slots up to kRingLevels - 1 levels away)
  if (fwd ? lf > 0 : (back && lb < L - 1)) {
    for (int d = 1; d < kRingLevels; ++d) {
      const int lev = fwd ? lf - d : lb + d;
      if (lev < 0 || lev >= L || cnt_me <= 0) continue;
      const int b = I.lvl_off[lev], e = I.lvl_off[lev + 1];
      if (b + s < e) {
        const longlong2 v = vload(b + s);
        sts_ll2(ring + 16u * ((lev % kRingLevels) * 16 + s), v.x, v.y);
      }
    }
  }
  int b0 = 0, e0 = 0, b1 = 0, e1 = 0;
  if (cnt_me > 0) {
    b0 = I.lvl_off[lev_of(0)];
    e0 = I.lvl_off[lev_of(0) + 1];
  }
  if (cnt_me > 1) {
    b1 = I.lvl_off[lev_of(1)];
    e1 = I.lvl_off[lev_of(1) + 1];
  }
  int4 r0 = make_int4(0, 0, 0, 0);
  long long dp0 = 0, dr0 = 0;
  if (b0 + s < e0) {
    r0 = row[b0 + s];
    dp0 = dp[b0 + s];
    dr0 = fwd ? dr[b0 + s] : 0;
  }
  int pf = fwd ? b0 : e0;  // next row not yet prefetched (this half's direction)
  __syncwarp();
  for (int k = 0; k < iters; ++k) {
    // issue the loads of the next iterations
    int b2 = 0, e2 = 0;
    if (k + 2 < cnt_me) {
      b2 = I.lvl_off[lev_of(k + 2)];
      e2 = I.lvl_off[lev_of(k + 2) + 1];
    }
    int4 r1 = make_int4(0, 0, 0, 0);
    long long dp1 = 0, dr1 = 0;
    if (b1 + s < e1) {
      r1 = row[b1 + s];
      dp1 = dp[b1 + s];
      dr1 = fwd ? dr[b1 + s] : 0;
    }
    const int i0 = b0 + s;
    if (i0 < e0) {
      const int cnt = r0.x & 0xffff;
      long long x = 0, y = 0;
      // ring reads first (shared memory only); the rare far neighbours
      // (global memory) are folded in by a separate, normally skipped block
      const unsigned q0 = static_cast<unsigned>(r0.y) >> 24, q1 = static_cast<unsigned>(r0.z) >> 24,
                     q2 = static_cast<unsigned>(r0.w) >> 24;
      const bool g0 = cnt > 0 && q0 == kRingNone, g1 = cnt > 1 && q1 == kRingNone, g2 = cnt > 2 && q2 == kRingNone;
      longlong2 v0 = make_longlong2(0, 0), v1 = v0, v2 = v0;
      if (cnt > 0 && !g0) v0 = lds_ll2(ring + 16u * q0);
      if (cnt > 1 && !g1) v1 = lds_ll2(ring + 16u * q1);
      if (cnt > 2 && !g2) v2 = lds_ll2(ring + 16u * q2);
      x = max(max(v0.x, v1.x), max(v2.x, x));
      y = max(max(v0.y, v1.y), max(v2.y, y));
      if (g0 | g1 | g2) {
        const int m = g0 ? r0.y : (g1 ? r0.z : r0.w);
        const longlong2 v = vload(m & 0xffffff);
        x = max(x, v.x);
        y = max(y, v.y);
        if (g0 && g1) {
          const longlong2 w = vload(r0.z & 0xffffff);
          x = max(x, w.x);
          y = max(y, w.y);
        }
        if (g2 && (g0 || g1)) {
          const longlong2 w = vload(r0.w & 0xffffff);
          x = max(x, w.x);
          y = max(y, w.y);
        }
      }
      if (cnt > 3)
        for (int j = noff[i0] + 3; j < noff[i0 + 1]; ++j) {
          const longlong2 v = vload(nb_[j]);
          x = max(x, v.x);
          y = max(y, v.y);
        }
      const long long a = x + dp0, c = fwd ? y + dr0 : 0;
      vstore(i0, a, c);
      sts_ll2(ring + 16u * ((lev_of(k) % kRingLevels) * 16 + s), a, c);
      if (fwd && (r0.x >> 16)) {
        mp = max(mp, a);
        mr = max(mr, c);
      }
      ++C.comp_visits;
      // levels wider than 16: the remaining computations, plain CSR
      for (int i = i0 + 16; i < e0; i += 16) {
        long long xx = 0, yy = 0;
        for (int j = noff[i]; j < noff[i + 1]; ++j) {
          const longlong2 v = vload(nb_[j]);
          xx = max(xx, v.x);
          yy = max(yy, v.y);
        }
        const long long aa = xx + dp[i], cc = fwd ? yy + dr[i] : 0;
        vstore(i, aa, cc);
        if (fwd && (row[i].x >> 16)) {
          mp = max(mp, aa);
          mr = max(mr, cc);
        }
        ++C.comp_visits;
      }
    }
    // each row / duration line prefetched once, ~64 computations ahead
    // (level-major order: the sweep consumes them contiguously)
    if (!kLat && k < cnt_me) {  // (shared-memory walks: nothing to prefetch)
      if (fwd) {
        const int want = min(b0 + 64, I.n);
        if (pf < want) {
          const int r = pf + 8 * s;
          if (r < want) {
            pf_sweep(row + r);
            pf_sweep(dp + r);
            pf_sweep(dr + r);
          }
          pf = min(want, pf + 128);
        }
      } else {
        const int want = max(b0 - 64, 0);
        if (pf > want) {
          const int r = pf - 8 * (s + 1);
          if (r >= want) {
            pf_sweep(row + r);
            pf_sweep(dp + r);
          }
          pf = max(want, pf - 128);
        }
      }
    }
    __syncwarp();
    b0 = b1;
    e0 = e1;
    b1 = b2;
    e1 = e2;
    r0 = r1;
    dp0 = dp1;
    dr0 = dr1;
  }
  // sink computations below the forward range keep their finish times
  if (lf > 0) {
    const int lim = lf < L ? I.lvl_off[lf] : I.n;
    for (int j = ln; j < I.n_snk; j += 32) {
      const int i = I.snk[j];
      if (i >= lim) break;
      mp = max(mp, fin[i]);
      mr = max(mr, finr[i]);
    }
  }
  msp = wmax(mp);
  msr = wmax(mr);
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
// reference's libm values).  The table covers every time a walk can evaluate
// (pack(): [t_min, t_max] for a discover walk, widened around a get-next
// start schedule), so a miss cannot happen; if it ever did, the miss is
// counted and the walk ends with PB_ERR_UNSUPPORTED -- the device never
// substitutes its own exp for glibc's.
__device__ __forceinline__ double table_at(const DevInst& I, int c, long long t, int* miss) {
  const long long t0 = I.cls_tmin[c];
  if (t >= t0 - I.tab_mlo && t <= I.cls_tmax[c] + I.tab_mhi) return I.tables[I.cls_tab[c] + (t - t0)];
  ++*miss;
  return 0.0;
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

__device__ __forceinline__ int ec_tail_of(int n, int u) { return u == n ? 2 * n : 2 * u + 1; }
__device__ __forceinline__ int ec_head_of(int n, int v) { return v == n + 1 ? 2 * n + 1 : 2 * v; }

// Curve value at t for a computation record (table_at).
__device__ __forceinline__ double table_rec(const DevInst& I, const CompRec& rc, long long t, int* miss) {
  if (t >= rc.tmin - I.tab_mlo && t <= rc.tmax + I.tab_mhi) return I.tables[rc.tab + (t - rc.tmin)];
  ++*miss;
  return 0.0;
}

// Totals of the critical network (flow.hpp:58-68, 196-197), maintained
// incrementally across the steps of a walk: sum of lower bounds, sum of
// finite upper bounds, number of infinite edges.
struct CapSums {
  i128 suml, sumu;
  long long ninf;
};

#ifndef PB_CAP_KU
#define PB_CAP_KU 4  // blocks of 32 * PB_CAP_KU computations per round
#endif
#ifndef PB_DEP_KU
#define PB_DEP_KU 4  // blocks of 32 * PB_DEP_KU dependency edges per round
#endif
#ifndef PB_DEP_PIPE
#define PB_DEP_PIPE 1
#endif
#ifndef PB_DEP_PF_OC
#define PB_DEP_PF_OC 1
#endif

// Dependency edges of build_caps (always infinite, lower bound 0): only
// criticality changes matter.  Warp wi of nw takes every nw-th block of
// 32 * kU edges; kCoop appends to the touch list through the CTA's shared
// counter (N.ctl->ntouch) instead of the warp-local count.
template <bool kCoop>
__device__ void dep_edges(const DevInst& I, Net& N, Walk& W, long long ms, int wi, int& ntouch,
                          long long& dinf, int& jc) {
  const int ln = lane_id();
  const int n = I.n;
  const int nw = kCoop ? N.nw : 1;
  constexpr int kU = PB_DEP_KU;
  auto touch_level = [&](int node) {
    if (N.prev_valid && bit_of(N, node)) {
      const int l = level_of(N, N.node_li[node]) - 1;
      jc = l < jc ? l : jc;
    }
  };
  // kPipe: the next block's endpoint ids are loaded one block ahead (static
  // data), so a block waits on one dependent round trip (its gathers), not two
  constexpr bool kPipe = PB_DEP_PIPE == 1 || (PB_DEP_PIPE == 2 && kCoop);
  int2 nuv[kU];
  if (kPipe) {
#pragma unroll
    for (int q = 0; q < kU; ++q) nuv[q] = I.dep_nd[min(32 * kU * wi + 32 * q + ln, I.ne - 1)];
  }
  for (int base = 32 * kU * wi; base < I.ne; base += 32 * kU * nw) {
    int2 uv[kU];
    bool oc[kU], tc[kU], hc[kU];
    long long tk[kU], hk[kU], hd[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int jr = base + 32 * q + ln, j = min(jr, I.ne - 1);
      uv[q] = kPipe ? nuv[q] : I.dep_nd[j];
      // predicated, not clamped: the owner of the last edge may rewrite it below
      oc[q] = jr < I.ne ? W.ecrit[n + j] : 0;
    }
    if (kPipe && base + 32 * kU * nw < I.ne) {
#pragma unroll
      for (int q = 0; q < kU; ++q) nuv[q] = I.dep_nd[min(base + 32 * kU * nw + 32 * q + ln, I.ne - 1)];
      // and the next block's criticality flags (32 * kU bytes, at most two
      // lines) into L1, without holding registers
      if (PB_DEP_PF_OC && ln < 2)
        pf_l1(W.ecrit + n + min(base + 32 * kU * nw + (ln ? 32 * kU - 1 : 0), I.ne - 1));
    }
    // endpoint loads, branch-free (index 0 stands in for the source / sink).
    // kCoop: one 16 B key per endpoint (the source "finishes" at 0, the sink
    // "starts" at the makespan); walkers: criticality flags + times (fewer
    // registers; the key stores cost the walkers more than the gathers save)
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const bool ts = uv[q].x == n, hs = uv[q].y == n + 1;
      const int tu = ts ? 0 : uv[q].x, hv = hs ? 0 : uv[q].y;
      if (kCoop) {
        const long long kt = W.key[tu].x, kh = W.key[hv].y;
        tk[q] = ts ? 0 : kt;
        hk[q] = hs ? ms : kh;
      } else {
        // every load unconditional: all 5 x kU requests in flight together
        const bool tcr = W.ecrit[tu], hcr = W.ecrit[hv];
        const long long tf = W.fin[tu], hf = W.fin[hv], hdd = W.durp[hv];
        tc[q] = ts || tcr;
        hc[q] = hs || hcr;
        tk[q] = ts ? 0 : tf;
        hk[q] = hs ? ms : hf;
        hd[q] = hs ? 0 : hdd;
      }
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int j = base + 32 * q + ln;
      bool ch = false;
      int et = 0, eh = 0;
      if (j < I.ne) {
        // kCoop: both critical (keys >= 0) and tight
        const bool crit = kCoop ? tk[q] == hk[q] : tc[q] && hc[q] && tk[q] == hk[q] - hd[q];
        if (crit != oc[q]) {
          const int2 ps = I.epos[n + j];
          W.ecrit[n + j] = crit;
          touch_level(ec_tail_of(n, uv[q].x));
          touch_level(ec_head_of(n, uv[q].y));
          if (crit) {
            ++dinf;
            N.resid[ps.y] = 0;
            N.resid[ps.x] = -1;  // infinite forward side carrying f = 0
          } else {
            --dinf;
            const long long fo = N.resid[ps.y];
            N.resid[ps.y] = 0;
            N.resid[ps.x] = 0;
            if (fo != 0) {
              et = ec_tail_of(n, uv[q].x);
              eh = ec_head_of(n, uv[q].y);
              red_add(&N.bal[eh], -fo);
              red_add(&N.bal[et], fo);
              ch = true;
            }
          }
        }
      }
      if (kCoop) {
        // shared append: both endpoints of each changed edge, adjacent
        const unsigned bm = __ballot_sync(kFull, ch);
        int at = 0;
        if (ln == 0 && bm) at = atomicAdd(&N.ctl->ntouch, 2 * __popc(bm));
        at = __shfl_sync(kFull, at, 0) + 2 * __popc(bm & lanemask_lt());
        if (ch) {
          N.touch[at] = et;
          N.touch[at + 1] = eh;
        }
      } else {
        wappend(ch, et, N.touch, ntouch);
        wappend(ch, eh, N.touch, ntouch);
      }
    }
  }
}

// K3: critical mask + Eq. 7 capacities + warm-start clamp.  Only "heavy"
// edges are rebuilt: those whose criticality changed, and critical
// computations whose duration (dirty) or the step size changed; every other
// critical edge keeps its bounds and flow.  Returns PB_OK or
// PB_ERR_OVERFLOW; ntouch = nodes whose balance moved.
// Stage 1 of build_caps: criticality of every computation; the heavy ones
// (criticality changed, or critical with a new duration / step size) are
// appended to W.delta.  kCoop: warp wi of nw takes every nw-th block and
// appends through the CTA's shared counter (N.ctl->ntouch); the dependency
// keys are written only for cooperative walks (dep_edges<true>).
template <bool kCoop>
__device__ void crit_pass(const DevInst& I, Net& N, Walk& W, long long ms, bool step_changed, int kfrom, int wi,
                          int& nh) {
  const int ln = lane_id();
  const int n = I.n;
  const int nw = kCoop ? N.nw : 1;
  constexpr int kU = PB_CAP_KU;
  for (int base = 32 * kU * wi; base < n; base += 32 * kU * nw) {
    long long t[kU], fx[kU], tx[kU];
    bool oc[kU];
    uint8_t dt[kU];
    // branch-free, clamped loads: all 5 x kU requests are in flight together
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int ir = base + 32 * q + ln, i = min(ir, n - 1);
      t[q] = W.durp[i];
      fx[q] = W.fin[i];
      tx[q] = W.tl[i];
      oc[q] = W.ecrit[i];
      dt[q] = ir < n ? W.dirty[i] : 0;  // predicated: the owner clears it below
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int i = base + 32 * q + ln;
      bool heavy = false;
      if (i < n) {
        const bool crit = fx[q] + tx[q] - t[q] == ms;
        heavy = crit != oc[q] || (crit && (dt[q] || step_changed));
        if (kCoop && (crit != oc[q] || (i >= kfrom && (crit || kfrom == 0))))
          W.key[i] = make_longlong2(crit ? fx[q] : -1, crit ? fx[q] - t[q] : -2);
        if (dt[q]) W.dirty[i] = 0;
      }
      if (kCoop) {
        const unsigned bm = __ballot_sync(kFull, heavy);
        int at = 0;
        if (ln == 0 && bm) at = atomicAdd(&N.ctl->ntouch, __popc(bm));
        at = __shfl_sync(kFull, at, 0) + __popc(bm & lanemask_lt());
        if (heavy) W.delta[at] = i;
      } else {
        wappend(heavy, i, W.delta, nh);
      }
    }
  }
}

// kfrom: the first computation whose planned finish or duration may have
// changed since the last call (0 on a walk's first call): dependency keys
// below it change only with the criticality.
__device__ int build_caps(const DevInst& I, Net& N, Walk& W, long long step, bool step_changed,
                          long long ms, CapSums& T, int& ntouch, int* extrap, Counters& C, int& jprev,
                          int kfrom, bool all_pok = false) {
  const int ln = lane_id();
  const int n = I.n;
  // Level (in the last step's final BFS) below which no residual changes:
  // every rebuilt edge's endpoints that BFS reached bound it (restart rule
  // of maximize: a changed arc out of a level-L node leaves levels <= L-1).
  int jc = INT_MAX;
  auto touch_level = [&](int node) {
    if (N.prev_valid && bit_of(N, node)) {
      const int l = level_of(N, N.node_li[node]) - 1;
      jc = l < jc ? l : jc;
    }
  };
  const long long t0 = now();
  C.add(kPrSteps, 1);
  ntouch = 0;
  i128 dl = 0, du = 0;
  long long dinf = 0;
  // stage 1: criticality of every computation, heavy ones compacted into W.delta
  int nh = 0;
  if (N.nw > 1) {
    // cooperative walk: every warp takes every nw-th block
    if (ln == 0) {
      CoopCtl* k = N.ctl;
      k->cmd = 4;
      k->ms = ms;
      k->step = step_changed ? 1 : 0;
      k->kfrom = kfrom;
      k->ntouch = 0;  // heavy-list counter
    }
    __syncwarp();
    bar_sync(1, 32 * N.nw);  // release the helpers
    crit_pass<true>(I, N, W, ms, step_changed, kfrom, 0, nh);
    bar_sync(2, 32 * N.nw);  // every warp's blocks are done
    nh = *reinterpret_cast<volatile int*>(&N.ctl->ntouch);
  } else {
    crit_pass<false>(I, N, W, ms, step_changed, kfrom, 0, nh);
  }
  __syncwarp();
  // stage 2: heavy computations, one per lane
  for (int base = 0; base < nh; base += 32) {
    const int k = base + ln;
    bool ch = false;
    int i = 0;
    if (k < nh) {
      i = W.delta[k];
      const long long t = W.durp[i];
      const bool crit = W.fin[i] + W.tl[i] - t == ms;
      const bool oc = W.ecrit[i];
      const CompRec rc = I.crec[i];
      long long fo = 0;
      if (oc) {
        const longlong2 cp = W.cap[i];
        fo = cp.x + N.resid[rc.ph];
        dl -= cp.x;
        if (cp.y >= 0)
          du -= cp.y;
        else
          --dinf;
      }
      long long l = 0, u = 0;
      bool inf = true;
      if (crit && rc.tab >= 0) {
        const bool can_speed = t - step >= rc.tmin;
        const bool can_slow = t + step <= rc.tmax;
        const double et = (can_speed || can_slow) ? table_rec(I, rc, t, extrap) : 0.0;
        if (can_slow) {
          const long long r = llround(et - table_rec(I, rc, t + step, extrap));
          l = r > 0 ? r : 0;
        }
        if (can_speed) {
          const long long r = llround(table_rec(I, rc, t - step, extrap) - et);
          u = r > l ? r : l;
          inf = false;
        }
      }
      long long fn = 0;
      if (crit) {
        fn = fo < l ? l : fo;
        if (!inf && fn > u) fn = u;
        dl += l;
        if (!inf)
          du += u;
        else
          ++dinf;
      }
      N.resid[rc.pt] = crit ? (inf ? -(fn + 1) : u - fn) : 0;
      N.resid[rc.ph] = crit ? fn - l : 0;
      W.cap[i] = make_longlong2(l, inf ? -1 : u);
      W.ecrit[i] = crit;
      touch_level(2 * i);
      touch_level(2 * i + 1);
      if (fn != fo) {
        red_add(&N.bal[2 * i + 1], fn - fo);
        red_add(&N.bal[2 * i], fo - fn);
        ch = true;
      }
    }
    wappend(ch, 2 * i, N.touch, ntouch);
    wappend(ch, 2 * i + 1, N.touch, ntouch);
  }
  __syncwarp();
  // dependency edges (always infinite, lower bound 0): only criticality changes matter
  if (N.nw > 1) {
    // cooperative walk: the helper warps take every nw-th block of edges
    if (ln == 0) {
      CoopCtl* k = N.ctl;
      k->cmd = 3;
      k->ms = ms;
      k->ntouch = ntouch;
      k->prev_valid = N.prev_valid;
      k->last_levels = N.last_levels;
    }
    __syncwarp();
    bar_sync(1, 32 * N.nw);  // release the helpers
    dep_edges<true>(I, N, W, ms, 0, ntouch, dinf, jc);
    bar_sync(2, 32 * N.nw);  // every warp's edges are done
    ntouch = *reinterpret_cast<volatile int*>(&N.ctl->ntouch);
    for (int w = 1; w < N.nw; ++w) {
      dinf += ln == 0 ? *reinterpret_cast<volatile long long*>(&N.ctl->part_dinf[w]) : 0;
      const int j = *reinterpret_cast<volatile int*>(&N.ctl->part_jc[w]);
      jc = j < jc ? j : jc;
    }
  } else {
    dep_edges<false>(I, N, W, ms, 0, ntouch, dinf, jc);
  }
  T.suml += wsum128(dl);
  T.sumu += wsum128(du);
  T.ninf += wsum(dinf);
  // infinity_sentinel (flow.hpp:58-68) and the aux total (flow.hpp:196-197)
  const i128 sent128 = T.suml + T.sumu + 1;
  if (sent128 > static_cast<i128>(LLONG_MAX / 4)) return PB_ERR_OVERFLOW;
  N.S = static_cast<long long>(sent128);
  const i128 aux = T.sumu + static_cast<i128>(T.ninf) * N.S + T.suml;
  if (aux + 1 > static_cast<i128>(LLONG_MAX / 2)) return PB_ERR_OVERFLOW;
  __syncwarp();
  // The carried flow is an s-t flow of value R on a DAG, so no edge carries
  // more than R: infinite edges need clamping only when R exceeds the new
  // sentinel.
  if (N.R > N.S) {
    N.prev_valid = false;
    const int nedges = n + I.ne;
    for (int base = 0; base < nedges; base += 32) {
      const int k = base + ln;
      bool ch = false;
      int a = 0, b = 0;
      if (k < nedges && W.ecrit[k]) {
        const bool inf = k >= n || W.cap[k].y < 0;
        const int2 ps = I.epos[k];
        const long long f = -N.resid[ps.x] - 1;
        if (inf && f > N.S) {
          const long long lo = k < n ? W.cap[k].x : 0;
          N.resid[ps.x] = -(N.S + 1);
          N.resid[ps.y] = N.S - lo;
          if (k < n) {
            a = 2 * k;
            b = 2 * k + 1;
          } else {
            const int2 uv = I.dep_nd[k - n];
            a = ec_tail_of(n, uv.x);
            b = ec_head_of(n, uv.y);
          }
          red_add(&N.bal[b], N.S - f);
          red_add(&N.bal[a], f - N.S);
          ch = true;
        }
      }
      wappend(ch, a, N.touch, ntouch);
      wappend(ch, b, N.touch, ntouch);
    }
  }
  __syncwarp();
  jc = static_cast<int>(wmin(jc));
  jprev = !N.prev_valid ? -1 : (jc == INT_MAX ? N.last_levels - 1 : jc);
  // shortcut bits of the rebuilt computation arcs (exact now that S is known);
  // when a carried flow may reach the sentinel, rebuild them all
  const bool all = N.R >= N.S || all_pok;
  const int cnt = all ? n : nh;
  for (int k = ln; k < cnt; k += 32) {
    const int i = all ? k : W.delta[k];
    const CompRec rc = I.crec[i];
    const bool fwd = W.ecrit[i] && eff_res(N.resid[rc.pt], N.S) > 0;
    const bool bwd = W.ecrit[i] && N.resid[rc.ph] > 0;
    if (fwd) pok_set(N, 2 * i); else pok_clear(N, 2 * i);
    if (bwd) pok_set(N, 2 * i + 1); else pok_clear(N, 2 * i + 1);
  }
  __syncwarp();
  C.add(kPrCap, now() - t0);
  return PB_OK;
}

template <bool kLat = false>
__device__ void run_walk(const DevInst& I, Net& N, Walk& W, const DeltaPool& pool, Counters& C) {
  const int ln = lane_id();
  const unsigned long long g0 = gtimer();
  const int n = I.n;
  N.V = I.V;
  N.src = 2 * n;
  N.snk = 2 * n + 1;
  N.ret_pt = I.ret_pt;
  N.ret_ph = I.ret_ph;
  N.nbitw = (I.V + 31) >> 5;
  N.inc_off = I.inc_off;
  N.ient = I.ient;
  N.S = 0;
  N.R = 0;
  N.prev_valid = false;
  // a get-next chain resumes the flow state its last call ended in
  // (DevInst::carry): residuals, critical set, bounds, dirty flags, totals
  const bool resume = I.resume != 0 && I.carry != nullptr;
  const CarryHdr* ch = reinterpret_cast<const CarryHdr*>(I.carry);
  const long long* c_resid = resume ? reinterpret_cast<const long long*>(I.carry + 64) : nullptr;
  const longlong2* c_cap = resume ? reinterpret_cast<const longlong2*>(I.carry + 64 + 16 * I.E) : nullptr;
  const uint8_t* c_ecrit = resume ? reinterpret_cast<const uint8_t*>(I.carry + 64 + 16 * I.E + 16 * n) : nullptr;
  for (int p = ln; p < 2 * I.E; p += 32) N.resid[p] = resume ? c_resid[p] : 0;
  for (int v = ln; v < I.V; v += 32) N.bal[v] = 0;
  for (int e = ln; e < I.E; e += 32) W.ecrit[e] = resume ? c_ecrit[e] : 0;
  for (int i = ln; i < n; i += 32) W.dirty[i] = resume ? c_ecrit[I.E + i] : 0;
  if (resume)
    for (int i = ln; i < n; i += 32) W.cap[i] = c_cap[i];
  for (int w = ln; w < N.nbitw; w += 32) sts32(N.s_pok + 4u * w, 0u);

  int bad = 0;
  long long spe = 0, spt = 0, sre = 0, srt = 0;
  // all-max durations (emulator.hpp:140-149) first, for T_min
  for (int i = ln; i < n; i += 32) W.durr[i] = I.pt_time[I.cls_pt_off[I.comp_class[i]]];
  __syncwarp();
  long long t_min, unused;
  sweep<kLat>(I, W.durr, W.durr, W.fin, W.finr, W.tl, false, t_min, unused, N.s_ring, C);
  for (int i = ln; i < n; i += 32) {
    const int c = I.comp_class[i];
    long long t;
    if (I.mode == kModeGetNext)
      t = I.start_planned_t[i];
    else
      t = I.cls_const[c] ? I.pt_time[I.cls_pt_off[c]] : I.cls_tmax[c];
    W.durp[i] = t;
    const int ch = discretize_choice(I, c, t);
    W.choice[i] = static_cast<uint8_t>(ch);
    W.durr[i] = I.pt_time[I.cls_pt_off[c] + ch];
    spe += table_energy(I, c, t, &bad);
    spt += t;
    sre += I.pt_energy[I.cls_pt_off[c] + ch];
    srt += W.durr[i];
  }
  __syncwarp();
  spe = wsum(spe);
  spt = wsum(spt);
  sre = wsum(sre);
  srt = wsum(srt);

  const long long t_walk0 = now();
  long long t_cur, t_real;
  sweep<kLat>(I, W.durp, W.durr, W.fin, W.finr, W.tl, true, t_cur, t_real, N.s_ring, C);
  const long long t_star = t_cur;
  if (ln == 0) write_point(I, 0, t_cur, t_real, spe, spt, sre, srt, 0, 0, 0, 0, 0);
  int steps = 0;
  long long n_ids = 0;
  // a curve evaluation outside the host tables ends the walk (table_at)
  int status = __any_sync(kFull, bad != 0) ? PB_ERR_UNSUPPORTED : PB_OK;
  int stop = PB_STOP_AT_TMIN;
  long long prev_step = -1;
  CapSums sums{0, 0, 0};
  bool all_pok = false;  // rebuild every partner-ok bit in the first capacity pass
  if (resume) {
    sums.suml = static_cast<i128>((static_cast<unsigned __int128>(static_cast<uint64_t>(ch->suml_hi)) << 64) |
                                  static_cast<uint64_t>(ch->suml_lo));
    sums.sumu = static_cast<i128>((static_cast<unsigned __int128>(static_cast<uint64_t>(ch->sumu_hi)) << 64) |
                                  static_cast<uint64_t>(ch->sumu_lo));
    sums.ninf = ch->ninf;
    N.R = ch->R;
    prev_step = ch->prev_step;
    all_pok = true;
  }

  int kfrom = 0;  // build_caps: every dependency key is written on the first step
  while (status == PB_OK) {
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
    // ---- K3 critical network + capacities, carried flow clamped into the new bounds
    int ntouch = 0;
    const bool step_changed = step != prev_step;
    prev_step = step;
    int jprev = -1;
    const int cs = build_caps(I, N, W, step, step_changed, t_cur, sums, ntouch, &bad, C, jprev, kfrom, all_pok);
    all_pok = false;
    if (cs != PB_OK || __any_sync(kFull, bad != 0)) {
      status = cs != PB_OK ? cs : PB_ERR_UNSUPPORTED;
      break;
    }
    // ---- K4 warm-started max flow with lower bounds
    if (!repair<kLat>(N, ntouch, C)) {
      stop = PB_STOP_INFEASIBLE;
      break;
    }
    maximize<kLat>(N, C, jprev);
    if (N.R >= N.S) {
      stop = PB_STOP_INFINITE_CUT;
      break;
    }
    // ---- K5 minimal min cut = the last BFS's visited set.  A computation
    // edge 2i -> 2i+1 crosses iff its two bits in the bitset word differ;
    // its cost equals the max-flow value R (strong duality).
    const long long tupd = now();
    const long long cost = N.R;
    int nd = 0;
    const int ncw = (2 * n + 31) >> 5;
    for (int base = 0; base < ncw; base += 32) {
      const int w = base + ln;
      uint32_t word = 0, x = 0;
      if (w < ncw) {
        word = lds32(N.s_bits + 4u * w);
        x = (word ^ (word >> 1)) & 0x55555555u;
        const int lim = 2 * n - 32 * w;  // bits from lim on are the source / sink
        if (lim < 32) x &= (1u << lim) - 1u;
      }
      while (__ballot_sync(kFull, x != 0)) {
        int rec = 0;
        if (x) {
          const int b = __ffs(x) - 1;
          x &= x - 1;
          const int i = (32 * w + b) >> 1;
          if (W.ecrit[i]) {
            if ((word >> b) & 1u) {
              rec = i + 1;  // start in S, end in T: speed up
            } else {
              const CompRec rc = I.crec[i];  // T -> S: slow down (frontier.hpp:117-125)
              if (rc.tab >= 0 && W.durp[i] + step <= rc.tmax) rec = -(i + 1);
            }
          }
        }
        wappend(rec != 0, rec, W.delta, nd);
      }
    }
    __syncwarp();
    // reserve a contiguous range of the batch delta pool
    unsigned long long at = 0;
    if (ln == 0 && nd) at = atomicAdd(pool.cursor, static_cast<unsigned long long>(nd));
    at = __shfl_sync(kFull, at, 0);
    if (static_cast<long long>(at) + nd > pool.cap) {
      status = kStatusLogFull;
      break;
    }
    // order: sped ascending, then slowed ascending, by caller id (frontier.hpp:111-125)
    int ns_loc = 0;
    long long dpe = 0, dpt = 0, dre = 0, drt = 0;
    for (int q = ln; q < nd; q += 32) {
      const int x = W.delta[q];
      const int i = (x > 0 ? x : -x) - 1;
      const int oi = I.orig[i];
      const long long kx = x > 0 ? oi : (1ll << 40) + oi;
      int rank = 0;
      for (int r = 0; r < nd; ++r) {
        const int y = W.delta[r];
        const int oj = I.orig[(y > 0 ? y : -y) - 1];
        const long long ky = y > 0 ? oj : (1ll << 40) + oj;
        rank += ky < kx;
      }
      const int c = I.comp_class[i];
      const long long told = W.durp[i];
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
      pool.ids[at + rank] = x > 0 ? oi + 1 : -(oi + 1);
      pool.choice[at + rank] = static_cast<uint8_t>(chnew);
    }
    __syncwarp();
    int imin = INT_MAX, imax = -1;
    for (int q = ln; q < nd; q += 32) {
      const int x = W.delta[q];
      const int i = (x > 0 ? x : -x) - 1;
      const int c = I.comp_class[i];
      const long long tnew = x > 0 ? W.durp[i] - step : W.durp[i] + step;
      W.durp[i] = tnew;
      const int ch = discretize_choice(I, c, tnew);
      W.choice[i] = static_cast<uint8_t>(ch);
      W.durr[i] = I.pt_time[I.cls_pt_off[c] + ch];
      W.dirty[i] = 1;
      imin = min(imin, i);
      imax = max(imax, i);
    }
    imin = __reduce_min_sync(kFull, imin);
    imax = __reduce_max_sync(kFull, imax);
    if (__any_sync(kFull, bad != 0)) {
      status = PB_ERR_UNSUPPORTED;
      break;
    }
    const int ns = static_cast<int>(wsum(ns_loc));
    dpe = wsum(dpe);
    dpt = wsum(dpt);
    dre = wsum(dre);
    drt = wsum(drt);
    C.add(kPrUpdate, now() - tupd);
    // refresh_totals (frontier.hpp:64-67) + discretize (frontier.hpp:157):
    // planned and realized makespans and the next step's tails, one sweep
    long long t_new;
    // computation ids are level-major: levels below imin's keep fin, above imax's keep tl
    const int lf = nd ? I.ilev[imin] : I.n_levels, lb = nd ? I.ilev[imax] : -1;
    kfrom = nd ? imin : I.n;
    sweep<kLat>(I, W.durp, W.durr, W.fin, W.finr, W.tl, true, t_new, t_real, N.s_ring, C, lf, lb);
    if (I.mode == kModeDiscover && t_new >= t_cur) {
      stop = PB_STOP_NO_PROGRESS;
      break;
    }
    t_cur = t_new;
    spe += dpe;
    spt += dpt;
    sre += dre;
    srt += drt;
    ++steps;
    if (ln == 0)
      write_point(I, steps, t_cur, t_real, spe, spt, sre, srt, cost, step, static_cast<int>(at), ns, nd - ns);
    n_ids += nd;
  }
  __syncwarp();
  // a get-next walk that took its steps leaves its flow state for the next
  // call of the chain (DevInst::carry)
  if (I.carry != nullptr && I.mode == kModeGetNext && status == PB_OK && stop == PB_STOP_STEP_LIMIT && steps > 0) {
    long long* o_resid = reinterpret_cast<long long*>(I.carry + 64);
    longlong2* o_cap = reinterpret_cast<longlong2*>(I.carry + 64 + 16 * I.E);
    uint8_t* o_ecrit = reinterpret_cast<uint8_t*>(I.carry + 64 + 16 * I.E + 16 * n);
    for (int p = ln; p < 2 * I.E; p += 32) o_resid[p] = N.resid[p];
    for (int i = ln; i < n; i += 32) o_cap[i] = W.cap[i];
    for (int e = ln; e < I.E; e += 32) o_ecrit[e] = W.ecrit[e];
    for (int i = ln; i < n; i += 32) o_ecrit[I.E + i] = W.dirty[i];
    if (ln == 0) {
      CarryHdr h;
      h.suml_lo = static_cast<int64_t>(static_cast<uint64_t>(static_cast<unsigned __int128>(sums.suml)));
      h.suml_hi = static_cast<int64_t>(static_cast<uint64_t>(static_cast<unsigned __int128>(sums.suml) >> 64));
      h.sumu_lo = static_cast<int64_t>(static_cast<uint64_t>(static_cast<unsigned __int128>(sums.sumu)));
      h.sumu_hi = static_cast<int64_t>(static_cast<uint64_t>(static_cast<unsigned __int128>(sums.sumu) >> 64));
      h.ninf = sums.ninf;
      h.R = N.R;
      h.prev_step = prev_step;
      h.valid = 1;
      *reinterpret_cast<CarryHdr*>(I.carry) = h;
    }
    __syncwarp();
  }
  const long long n_miss = wsum(bad);
  C.add(kPrWalk, now() - t_walk0);
  if (ln == 0) {
    pb_frontier_summary s;
    s.t_min = t_min;
    s.t_star = t_star;
    s.steps = steps;
    s.stop = stop;
    s.status = status;
    s.n_ids = static_cast<int32_t>(n_ids);
    s.n_table_misses = static_cast<int32_t>(n_miss);
    s.walk_us = static_cast<int32_t>((gtimer() - g0) / 1000);
    s.warps = N.nw;
    s.start_us = static_cast<int32_t>((g0 / 1000) & 0x7fffffffull);
    *I.summary = s;
  }
  __syncwarp();
}

struct WsPtrs {
  Net N;
  Walk W;
};

__device__ WsPtrs bind_ws(char* base, const WsLayout& L, char* smem) {
  WsPtrs p;
  p.N.resid = reinterpret_cast<long long*>(base + L.off_resid);
  p.N.bal = reinterpret_cast<long long*>(base + L.off_bal);
  p.N.lg = reinterpret_cast<int4*>(base + L.off_log);
  p.N.fglob = reinterpret_cast<int4*>(base + L.off_front);
  p.N.par = reinterpret_cast<int32_t*>(base + L.off_par);
  p.N.par_cap = kWalkerPar ? static_cast<int>(L.max_v) : 0;
  p.N.anc = kWalkerPar && PB_ANCHORS;
  p.N.fstride = static_cast<int>(L.max_v);
  p.N.path = reinterpret_cast<int32_t*>(base + L.off_path);
  p.N.path_log = reinterpret_cast<int32_t*>(base + L.off_pathlog);
  p.N.lvl_start = reinterpret_cast<int32_t*>(base + L.off_lvlstart);
  p.N.last_nlog = 0;
  p.N.last_levels = 0;
  p.N.node_li = reinterpret_cast<int32_t*>(base + L.off_nodeli);
  p.N.prev_valid = false;
  p.N.touch = reinterpret_cast<int32_t*>(base + L.off_touch);
  p.N.exl = reinterpret_cast<int32_t*>(base + L.off_exl);
  p.W.durp = reinterpret_cast<long long*>(base + L.off_durp);
  p.W.durr = reinterpret_cast<long long*>(base + L.off_durr);
  p.W.fin = reinterpret_cast<long long*>(base + L.off_fin);
  p.W.finr = reinterpret_cast<long long*>(base + L.off_fin + 8 * L.max_n);
  p.W.tl = reinterpret_cast<long long*>(base + L.off_hl);
  p.W.cap = reinterpret_cast<longlong2*>(base + L.off_cap);
  p.W.ecrit = reinterpret_cast<uint8_t*>(base + L.off_ecrit);
  p.W.key = reinterpret_cast<longlong2*>(base + L.off_key);
  p.W.dirty = reinterpret_cast<uint8_t*>(base + L.off_ccrit);
  p.W.choice = reinterpret_cast<uint8_t*>(base + L.off_choice);
  p.W.delta = reinterpret_cast<int32_t*>(base + L.off_delta);
  // shared memory: path ends, frontier (16 B aligned), visited bitset,
  // partner-ok bitset, longest-path rings
  p.N.ends = reinterpret_cast<int2*>(smem);
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  p.N.s_fs = sa + 8 * kMaxEnds;
  p.N.s_bits = sa + 8 * kMaxEnds + 16 * 2 * kFrontCap;
  p.N.s_pok = p.N.s_bits + static_cast<uint32_t>((4 * ((L.max_v + 31) / 32) + 15) / 16 * 16);
  p.N.s_ring = p.N.s_pok + static_cast<uint32_t>((4 * ((L.max_v + 31) / 32) + 15) / 16 * 16);
  p.N.ctl = nullptr;
  p.N.nw = 1;
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

__device__ __forceinline__ int warp_in_block() { return threadIdx.x >> 5; }
__device__ __forceinline__ int warp_slot() { return blockIdx.x * kWarpsPerBlock + warp_in_block(); }

// Per-warp shared memory: [profile 16 x u64][frontier + bitset].
extern __shared__ __align__(16) char g_smem[];

__device__ __forceinline__ char* my_smem(const WsLayout& L, unsigned long long** prof) {
  const int per = 128 + 8 * kMaxEnds + L.smem_bytes;
  char* base = g_smem + warp_in_block() * per;
  *prof = reinterpret_cast<unsigned long long*>(base);
  if (lane_id() < kPrSlots) (*prof)[lane_id()] = 0;
  __syncwarp();
  return base + 128;
}

__global__ void __launch_bounds__(kBlock, kMinBlocks) walk_kernel(const DevInst* insts, int n_inst,
                                                      const int32_t* order, int32_t* counter,
                                                      char* ws_base, WsLayout L, int slots,
                                                      RunCounters* ctr, DeltaPool pool, int n_wide,
                                                      int ws_first) {
  const int slot = warp_slot();
  if (slot >= slots) return;
  Counters C;
  char* sm = my_smem(L, &C.prof);
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(ws_first + slot) * L.stride, L, sm);
  for (;;) {
    int k = 0;
    if (lane_id() == 0) k = n_wide + atomicAdd(counter, 1);
    k = __shfl_sync(kFull, k, 0);
    if (k >= n_inst) break;
    run_walk(insts[order[k]], P.N, P.W, pool, C);
  }
  flush_counters(C, ctr);
}

// Cooperative walks for the longest instances (their walk time bounds the
// batch): a CTA of nw warps per walk.  Warp 0 drives run_walk; every BFS is
// posted to the CTA's control block and expanded by all nw warps
// (bfs_core<., true>); the other phases stay on warp 0.  The walk's shared
// structures (frontier, bitsets, path ends) are warp 0's region.
// The cooperative kernel runs 64-thread CTAs beside at most 2 walker blocks
// (the walkers' 168 registers x 128 threads x 3 blocks fill the register
// file), so it may use up to 255 registers at no occupancy cost: measured on
// the 4096 batch, every walk gets faster (sum of walk times -11%, batch
// 10.7 -> 10.1 s)
#ifndef PB_WIDE_MIN_BLOCKS
#define PB_WIDE_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(kBlock, PB_WIDE_MIN_BLOCKS) walk_kernel_wide(const DevInst* insts, int n_wide,
                                                           const int32_t* order, int32_t* counter,
                                                           char* ws_base, WsLayout L, RunCounters* ctr,
                                                           DeltaPool pool) {
  // this CTA is resident: the walker grid (programmatic dependent launch on
  // the same stream) may start once every cooperative CTA got here, so the
  // persistent walkers can never take the SMs the cooperative CTAs need
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int nw = blockDim.x >> 5;
  const int wi = warp_in_block();
  Counters C;
  (void)my_smem(L, &C.prof);  // this warp's profile slots
  const int per = 128 + 8 * kMaxEnds + L.smem_bytes;
  CoopCtl* ctl = reinterpret_cast<CoopCtl*>(g_smem + nw * per);
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(blockIdx.x) * L.stride, L, g_smem + 128);
  P.N.ctl = ctl;
  P.N.nw = nw;
  if (L.wide_par > 0) {  // else the global parent array of bind_ws (or the log)
    P.N.par = reinterpret_cast<int32_t*>(g_smem + nw * per + kCtlBytes);
    P.N.par_cap = L.wide_par;
    P.N.anc = false;
  }
  if (wi == 0) {
    for (;;) {
      int k = 0;
      if (lane_id() == 0) k = atomicAdd(counter + 1, 1);
      k = __shfl_sync(kFull, k, 0);
      if (k >= n_wide) break;
      const DevInst& I = insts[order[k]];
      if (lane_id() == 0) ctl->inst = &I;
      run_walk(I, P.N, P.W, pool, C);
    }
    if (lane_id() == 0) ctl->cmd = 0;
    __syncwarp();
    bar_sync(1, 32 * nw);  // release the helpers to exit
  } else {
    for (;;) {
      bar_sync(1, 32 * nw);
      const int cmd = *reinterpret_cast<volatile int*>(&ctl->cmd);
      if (cmd == 0) break;
      const DevInst* I = *reinterpret_cast<const DevInst* volatile*>(&ctl->inst);
      Net& N = P.N;
      if (cmd == 4) {
        // capacity pass, stage 1: this warp's blocks of computations
        int unused = 0;
        crit_pass<true>(*I, N, P.W, *reinterpret_cast<volatile long long*>(&ctl->ms),
                        *reinterpret_cast<volatile int*>(&ctl->step) != 0,
                        *reinterpret_cast<volatile int*>(&ctl->kfrom), wi, unused);
        bar_sync(2, 32 * nw);
        continue;
      }
      if (cmd == 3) {
        // capacity pass: this warp's blocks of dependency edges
        N.prev_valid = *reinterpret_cast<volatile int*>(&ctl->prev_valid) != 0;
        N.last_levels = *reinterpret_cast<volatile int*>(&ctl->last_levels);
        long long dinf = 0;
        int jc = INT_MAX, unused = 0;
        dep_edges<true>(*I, N, P.W, *reinterpret_cast<volatile long long*>(&ctl->ms), wi, unused, dinf, jc);
        dinf = wsum(dinf);
        jc = static_cast<int>(wmin(jc));
        if (lane_id() == 0) {
          ctl->part_dinf[wi] = dinf;
          ctl->part_jc[wi] = jc;
        }
        bar_sync(2, 32 * nw);
        continue;
      }
      N.ient = I->ient;
      N.snk = 2 * I->n + 1;
      N.S = *reinterpret_cast<volatile long long*>(&ctl->S);
      const int nsrc = *reinterpret_cast<volatile int*>(&ctl->nsrc);
      const int start = *reinterpret_cast<volatile int*>(&ctl->start);
      int tgt;
      if (cmd == 2)
        bfs_core<true, true>(N, nsrc, tgt, C, wi, start);
      else
        bfs_core<false, true>(N, nsrc, tgt, C, wi, start);
    }
  }
  flush_counters(C, ctr);
}

// ------------------------------------------- shared-memory-resident walks
//
// Small instances (and single walks, whose latency is what a caller of
// discover_frontier sees) run from shared memory: the CTA's region holds a
// copy of the instance record and, greedily in order of accesses per byte,
// the walk's residuals, BFS log and static network (incidence entries, row
// records, capacity records), then its longest-path state.  An array that
// does not fit stays in global memory, so every instance can run here; the
// walk code is unchanged (generic addressing).  Curve tables, outputs and
// the cold lists (frontier overflow, touch / path lists) stay global.

// 16 B-granular copy global -> shared (sources are 256 B aligned in the
// static blob, whose sections are padded to 256 B, so the rounded-up tail
// stays inside the blob).
__device__ __forceinline__ void copy16(void* dst, const void* src, size_t bytes) {
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  const size_t n = (bytes + 15) / 16;
  for (size_t q = lane_id(); q < n; q += 32) d[q] = s[q];
}

// Places the walk's arrays into [region, region + cap): workspace arrays are
// re-pointed (P), static arrays copied and re-pointed in the shared copy S of
// the instance record.  Every lane computes the same layout.
__device__ void bind_smem(DevInst& S, WsPtrs& P, char* region, size_t cap) {
  char* cur = region;
  char* const end = region + cap;
  auto take = [&](size_t bytes) -> char* {
    bytes = (bytes + 15) & ~static_cast<size_t>(15);
    if (cur + bytes > end) return nullptr;
    char* r = cur;
    cur += bytes;
    return r;
  };
  auto ws = [&](auto*& ptr, size_t bytes) {
    if (char* r = take(bytes)) ptr = reinterpret_cast<std::remove_reference_t<decltype(ptr)>>(r);
  };
  auto st = [&](auto*& ptr, size_t bytes) {
    if (char* r = take(bytes)) {
      const void* src = ptr;
      copy16(r, src, bytes);
      __syncwarp();
      ptr = reinterpret_cast<std::remove_reference_t<decltype(ptr)>>(r);
    }
  };
  const size_t n = S.n, V = S.V, E = S.E, ne = S.ne;
  // BFS: {incidence, residual} per arc, log + node index per discovery
  ws(P.N.resid, 16 * E);
  st(S.ient, 32 * E);
  st(S.inc_off, 4 * (V + 1));
  ws(P.N.lg, 16 * V);
  {
    const int32_t* par0 = P.N.par;
    ws(P.N.par, 4 * V);
    if (P.N.par != par0) P.N.anc = false;  // shared-memory parents: plain chase
  }
  ws(P.N.node_li, 4 * V);
  ws(P.N.lvl_start, 4 * (V + 2));
  // longest-path sweep + capacity pass
  st(S.lvl_off, 4 * (S.n_levels + 1));
  ws(P.W.durp, 8 * n);
  ws(P.W.fin, 8 * n);
  ws(P.W.tl, 8 * n);
  ws(P.W.finr, 8 * n);
  st(S.frow, 16 * n);
  st(S.brow, 16 * n);
  ws(P.W.durr, 8 * n);
  ws(P.W.ecrit, E);
  ws(P.W.dirty, n);
  st(S.crec, 32 * n);
  ws(P.W.cap, 16 * n);
  ws(P.W.key, 16 * n);
  st(S.dep_nd, 8 * ne);
  st(S.epos, 8 * E);
  ws(P.N.bal, 8 * V);
  ws(P.W.choice, n);
  st(S.ilev, 4 * n);
  st(S.snk, 4 * static_cast<size_t>(S.n_snk));
  st(S.comp_class, 4 * n);
  __syncwarp();
}

__global__ void __launch_bounds__(32, 1) walk_kernel_smem(const DevInst* insts, int n_inst, const int32_t* order,
                                                          int32_t* counter, char* ws_base, WsLayout L,
                                                          int region, RunCounters* ctr, DeltaPool pool) {
  Counters C;
  char* sm = my_smem(L, &C.prof);
  const int per = 128 + 8 * kMaxEnds + L.smem_bytes;
  DevInst* S = reinterpret_cast<DevInst*>(g_smem + per);
  char* reg = g_smem + per + ((sizeof(DevInst) + 15) & ~static_cast<size_t>(15));
  const WsPtrs G = bind_ws(ws_base + static_cast<size_t>(blockIdx.x) * L.stride, L, sm);
  static_assert(sizeof(DevInst) % 8 == 0, "DevInst copy granularity");
  for (;;) {
    int k = 0;
    if (lane_id() == 0) k = atomicAdd(counter + 2, 1);
    k = __shfl_sync(kFull, k, 0);
    if (k >= n_inst) break;
    const long long* src = reinterpret_cast<const long long*>(&insts[order[k]]);
    long long* dst = reinterpret_cast<long long*>(S);
    for (int q = lane_id(); q < static_cast<int>(sizeof(DevInst) / 8); q += 32) dst[q] = src[q];
    __syncwarp();
    WsPtrs P = G;
    bind_smem(*S, P, reg, static_cast<size_t>(region));
    run_walk<true>(*S, P.N, P.W, pool, C);
    __syncwarp();
  }
  flush_counters(C, ctr);
}

// ------------------------------------------------------- straggler sweep

// blocking_energy_mj (units.hpp:38-41)
__device__ __forceinline__ double blocking_mj(double w, long long t, long long q) {
  return w * static_cast<double>(t) * static_cast<double>(q) * 1e-3;
}

// energy_report(...).total_mj (emulator.hpp:77-112): computation energy +
// per-stage blocking over the iteration + per-stage straggler wait.
__device__ __forceinline__ double report_total(double w, long long q, int stages, long long e_sum, long long t,
                                               long long busy_sum, long long t_prime) {
  return static_cast<double>(e_sum) + blocking_mj(w, static_cast<long long>(stages) * t - busy_sum, q) +
         static_cast<double>(stages) * blocking_mj(w, t_prime - t, q);
}

// One thread per (instance, factor): straggler_savings (baselines.hpp:162-188).
__global__ void straggler_kernel(const DevStraggler* jobs, int n_inst, const double* factors, int n_factors,
                                 int pipelines, pb_savings_row* out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_inst * n_factors) return;
  const int k = g / n_factors, j = g - k * n_factors;
  const DevStraggler J = jobs[k];
  const pb_frontier_summary sm = *J.summary;
  const double f = factors[j];
  const long long tp = llround(f * static_cast<double>(sm.t_min));
  pb_savings_row r;
  r.factor = f;
  r.status = PB_OK;
  r.all_max_mj = report_total(J.watts, J.quantum, J.stages, J.am_energy, sm.t_min, J.am_time, tp);
  // lookup (frontier.hpp:212-220): first point, in decreasing planned time,
  // with t_planned <= min(T*, T'); the last point if none
  const long long target = sm.t_star < tp ? sm.t_star : tp;
  int lo = 0, hi = sm.steps + 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (J.points[mid].t_planned > target)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo > sm.steps) lo = sm.steps;
  const pb_point p = J.points[lo];
  r.point = lo;
  if (tp < p.t_realized) r.status = PB_ERR_INVALID_ARGUMENT;
  r.tuned_mj = report_total(J.watts, J.quantum, J.stages, p.sum_realized_e, p.t_realized, p.sum_realized_t, tp);
  r.savings_mj = static_cast<double>(pipelines - 1) * (r.all_max_mj - r.tuned_mj);
  r.savings_pct = 100.0 * r.savings_mj / (static_cast<double>(pipelines) * r.all_max_mj);
  out[g] = r;
}

// ------------------------------------------------------- exhaustive oracle

constexpr int kBruteMaxN = 64;

// Order-preserving unsigned key of a double (no NaNs here).
__device__ __forceinline__ unsigned long long dkey(double d) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(d));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// One thread per assignment code (oracle.hpp:47-114): iteration time via the
// longest path in internal (topological) order, effective energy summed in
// caller index order with explicit round-to-nearest ops (no FMA: the
// reference's host arithmetic).  Pass 0: best energy per time; pass 1: the
// smallest code reaching it.
__global__ void brute_kernel(const DevBrute* jp, int pass) {
  const DevBrute J = *jp;
  for (long long code = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; code < J.combos;
       code += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long t[kBruteMaxN];
    double eff = 0;
    for (int j = 0; j < J.n; ++j) {
      const int d = static_cast<int>((code / J.stride[j]) % J.radix[j]);
      const long long tj = J.pt_time[J.poff[j] + d];
      const long long ej = J.pt_energy[J.poff[j] + d];
      t[j] = tj;
      // effective_energy_mj (units.hpp:45-48): e - W * t * q * 1e-3
      const double blk = __dmul_rn(__dmul_rn(__dmul_rn(J.watts, static_cast<double>(tj)), static_cast<double>(J.quantum)), 1e-3);
      eff = __dadd_rn(eff, __dsub_rn(static_cast<double>(ej), blk));
    }
    long long fin[kBruteMaxN];
    long long ms = 0;
    for (int i = 0; i < J.n; ++i) {
      long long st = 0;
      for (int q = J.pin_off[i]; q < J.pin_off[i + 1]; ++q) st = max(st, fin[J.pin[q]]);
      fin[i] = st + t[J.orig[i]];
      if (J.cflag[i] & 2) ms = max(ms, fin[i]);
    }
    const long long slot = ms - J.t_lo;
    if (slot < 0 || slot >= J.slots) continue;  // cannot happen: t_lo / slots bound every path
    const unsigned long long k = dkey(eff);
    if (pass == 0)
      atomicMin(&J.best_e[slot], k);
    else if (J.best_e[slot] == k)
      atomicMin(&J.best_code[slot], static_cast<unsigned long long>(code));
  }
}

// ------------------------------------------------------------ flow jobs

// max_flow_lower_bounds + min_cut_from_flow on an arbitrary FlowGraph with
// the same machinery from the all-lower-bound start (f = l everywhere).
__global__ void __launch_bounds__(kBlock) flow_kernel(const DevFlowJob* jobs, int count,
                                                      char* ws_base, WsLayout L, int slots) {
  const int slot = warp_slot();
  if (slot >= slots) return;
  Counters C;
  char* sm = my_smem(L, &C.prof);
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(slot) * L.stride, L, sm);
  Net& N = P.N;
  const int ln = lane_id();
  for (int g = slot; g < count; g += slots) {
    const DevFlowJob& J = jobs[g];
    N.V = J.nodes;
    N.src = J.source;
    N.snk = J.sink;
    N.ret_pt = J.ret_pt;
    N.ret_ph = J.ret_ph;
    N.nbitw = (J.nodes + 31) >> 5;
    N.inc_off = J.inc_off;
    N.ient = J.ient;
    N.R = 0;
    for (int p = ln; p < 2 * (J.m + 1); p += 32) N.resid[p] = 0;
    for (int v = ln; v < J.nodes; v += 32) N.bal[v] = 0;
    __syncwarp();
    i128 suml = 0, sumu = 0;
    long long ninf = 0;
    int ntouch = 0;
    for (int base = 0; base < J.m; base += 32) {
      const int e = base + ln;
      bool ch = false;
      int a = 0, b = 0;
      if (e < J.m) {
        const long long l = J.lower[e];
        const int2 ps = J.epos[e];
        N.resid[ps.x] = J.inf[e] ? -(l + 1) : J.upper[e] - l;
        N.resid[ps.y] = 0;
        suml += l;
        if (!J.inf[e])
          sumu += J.upper[e];
        else
          ++ninf;
        if (l > 0) {
          a = J.tail[e];
          b = J.head[e];
          red_add(&N.bal[b], l);
          red_add(&N.bal[a], -l);
          ch = true;
        }
      }
      wappend(ch, a, N.touch, ntouch);
      wappend(ch, b, N.touch, ntouch);
    }
    suml = wsum128(suml);
    sumu = wsum128(sumu);
    ninf = wsum(ninf);
    const i128 sent128 = suml + sumu + 1;
    int status = PB_OK;
    if (sent128 > static_cast<i128>(LLONG_MAX / 4)) {
      status = PB_ERR_OVERFLOW;
    } else {
      N.S = static_cast<long long>(sent128);
      const i128 aux = sumu + static_cast<i128>(ninf) * N.S + suml;
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
        J.sentinel[g] = N.S;
      }
      __syncwarp();
      continue;
    }
    maximize(N, C);
    long long cost = 0;
    for (int e = ln; e < J.m; e += 32) {
      const bool a = bit_of(N, J.tail[e]), b = bit_of(N, J.head[e]);
      int8_t dir = 0;
      if (a && !b) {
        cost += J.inf[e] ? N.S : J.upper[e];
        dir = 1;
      } else if (!a && b) {
        cost -= J.lower[e];
        dir = -1;
      }
      J.cut_dir[e] = dir;
    }
    for (int v = ln; v < N.V; v += 32) J.side[v] = bit_of(N, v) ? 1 : 0;
    cost = wsum(cost);
    if (ln == 0) {
      J.status[g] = bit_of(N, N.snk) ? PB_ERR_LOGIC : PB_OK;
      J.feasible[g] = 1;
      J.value[g] = N.R;
      J.sentinel[g] = N.S;
      J.cost[g] = cost;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------ slack jobs

// annotate_slack (dag.hpp:233-286) through the fused sweep; outputs in the
// caller's ids.
__global__ void __launch_bounds__(kBlock) slack_kernel(const DevInst* insts, const SlackOut* outs,
                                                       int64_t* makespan, int count, char* ws_base,
                                                       WsLayout L, int slots) {
  const int slot = warp_slot();
  if (slot >= slots) return;
  Counters C;
  char* sm = my_smem(L, &C.prof);
  WsPtrs P = bind_ws(ws_base + static_cast<size_t>(slot) * L.stride, L, sm);
  Walk& W = P.W;
  const int ln = lane_id();
  for (int g = slot; g < count; g += slots) {
    const DevInst& I = insts[g];
    const SlackOut& O = outs[g];
    const int n = I.n;
    for (int i = ln; i < n; i += 32) W.durp[i] = O.dur[I.orig[i]];
    __syncwarp();
    long long ms, unused;
    sweep(I, W.durp, W.durp, W.fin, W.finr, W.tl, true, ms, unused, P.N.s_ring, C);
    __syncwarp();
    // latest of the source node: min over its successors' latest start
    long long ls = ms;
    for (int j = ln; j < I.ne; j += 32) {
      const int2 uv = I.dep_nd[j];
      if (uv.x == n && uv.y < n) {
        const long long c = ms - W.tl[uv.y];
        if (c < ls) ls = c;
      }
    }
    ls = wmin(ls);
    for (int i = ln; i < n; i += 32) {
      const int o = I.orig[i];
      const long long d = W.durp[i], f = W.fin[i], h = W.tl[i];
      O.earliest[2 * o] = f - d;
      O.earliest[2 * o + 1] = f;
      O.latest[2 * o + 1] = ms - (h - d);
      O.latest[2 * o] = ms - h;
      O.critical[o] = f + h - d == ms;
    }
    if (ln == 0) {
      O.earliest[2 * n] = 0;
      O.latest[2 * n] = ls;
      O.earliest[2 * n + 1] = ms;
      O.latest[2 * n + 1] = ms;
      makespan[g] = ms;
    }
    for (int j = ln; j < I.ne; j += 32) {
      const int2 uv = I.dep_nd[j];
      long long te, tl, he, hl;
      if (uv.x == n) {
        te = 0;
        tl = ls;
      } else {
        te = W.fin[uv.x];
        tl = ms - (W.tl[uv.x] - W.durp[uv.x]);
      }
      if (uv.y == n + 1) {
        he = ms;
        hl = ms;
      } else {
        he = W.fin[uv.y] - W.durp[uv.y];
        hl = ms - W.tl[uv.y];
      }
      O.critical[n + I.dep_orig[j]] = te == tl && he == hl && te == he;
    }
    __syncwarp();
  }
}

int blocks_for(int slots) { return (slots + kWarpsPerBlock - 1) / kWarpsPerBlock; }
size_t block_smem(const WsLayout& L) {
  return static_cast<size_t>(kWarpsPerBlock) * (128 + 8 * kMaxEnds + L.smem_bytes);
}

template <class K>
void set_smem(K kernel, size_t bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (const char* e = std::getenv("PB_CARVEOUT"))
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e));
}

}  // namespace

// Occupancy answers depend only on (device, shared-memory bytes): cached,
// so a stream of small runs (the drop-in's per-call path) queries once.
template <class K>
int cached_blocks(K kernel, int which, int threads, size_t sm) {
  static thread_local std::map<std::tuple<int, int, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, which, sm);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  set_smem(kernel, sm);
  int blocks = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, threads, sm);
  cache.emplace(key, blocks);
  return blocks;
}

int walk_slots_per_sm(const WsLayout& ws) {
  return cached_blocks(walk_kernel, 0, kBlock, block_smem(ws)) * kWarpsPerBlock;
}

// d_counter[0] = walker queue cursor, d_counter[1] = wide queue cursor.
int launch_walks(const DevInst* d_insts, int32_t n_inst, const int32_t* d_order, int32_t* d_counter,
                 char* d_ws, const WsLayout& ws, int32_t slots, RunCounters* d_counters,
                 DeltaPool pool, int32_t n_wide, int32_t wide_ctas, int32_t wide_warps, void* stream) {
  if (n_wide > 0 && wide_ctas > 0) {
    static_assert(sizeof(CoopCtl) <= kCtlBytes, "CoopCtl outgrew its shared-memory block");
    size_t sm = static_cast<size_t>(wide_warps) * (128 + 8 * kMaxEnds + ws.smem_bytes) + kCtlBytes;
    // shared parent links for the augment chase, when every log entry fits
    WsLayout wl = ws;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t par = 4 * static_cast<size_t>(ws.max_v);
    wl.wide_par = sm + par <= static_cast<size_t>(optin) && !std::getenv("PB_WIDE_NO_SHARED_PARENTS")
                      ? static_cast<int32_t>(ws.max_v)
                      : 0;
    if (wl.wide_par) sm += par;
    set_smem(walk_kernel_wide, sm);
    walk_kernel_wide<<<wide_ctas, 32 * wide_warps, sm, static_cast<cudaStream_t>(stream)>>>(
        d_insts, n_wide, d_order, d_counter, d_ws, wl, d_counters, pool);
  }
  if (n_inst > n_wide) {
    const size_t sm = block_smem(ws);
    set_smem(walk_kernel, sm);
    // same stream as the cooperative kernel, programmatic dependent launch:
    // the walkers start as soon as every cooperative CTA is resident (they
    // share only the pre-zeroed queue counters, no data)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(blocks_for(slots)));
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = n_wide > 0 && wide_ctas > 0 ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, walk_kernel, d_insts, n_inst, d_order, d_counter, d_ws, ws,
                                             slots, d_counters, pool, n_wide, wide_ctas);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return static_cast<int>(cudaGetLastError());
}

int smem_walk_plan(const WsLayout& ws, int64_t footprint, int32_t* region, int32_t* ctas_per_sm) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int64_t base = 128 + 8 * kMaxEnds + ws.smem_bytes + ((sizeof(DevInst) + 15) & ~static_cast<size_t>(15));
  const int64_t r = std::max<int64_t>(0, std::min<int64_t>(align_up(footprint, 16), optin - base));
  const size_t sm = static_cast<size_t>(base + r);
  *region = static_cast<int32_t>(r);
  *ctas_per_sm = cached_blocks(walk_kernel_smem, 1, 32, sm);
  return static_cast<int>(cudaGetLastError());
}

int launch_walks_smem(const DevInst* d_insts, int32_t n_inst, const int32_t* d_order, int32_t* d_counter,
                      char* d_ws, const WsLayout& ws, int32_t region, int32_t ctas, RunCounters* d_counters,
                      DeltaPool pool, void* stream) {
  const size_t sm = 128 + 8 * kMaxEnds + ws.smem_bytes + ((sizeof(DevInst) + 15) & ~static_cast<size_t>(15)) +
                    static_cast<size_t>(region);
  set_smem(walk_kernel_smem, sm);
  walk_kernel_smem<<<ctas, 32, sm, static_cast<cudaStream_t>(stream)>>>(d_insts, n_inst, d_order, d_counter, d_ws,
                                                                        ws, region, d_counters, pool);
  return static_cast<int>(cudaGetLastError());
}

int launch_straggler(const DevStraggler* d_jobs, int32_t n_inst, const double* d_factors, int32_t n_factors,
                     int32_t pipelines, pb_savings_row* d_out, void* stream) {
  const int total = n_inst * n_factors;
  straggler_kernel<<<(total + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(d_jobs, n_inst, d_factors,
                                                                                      n_factors, pipelines, d_out);
  return static_cast<int>(cudaGetLastError());
}

int launch_brute(const DevBrute* d_job, const DevBrute& host_job, int pass, void* stream) {
  const long long blocks = std::min<long long>((host_job.combos + 255) / 256, 148LL * 64);
  brute_kernel<<<static_cast<int>(std::max<long long>(blocks, 1)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_job, pass);
  return static_cast<int>(cudaGetLastError());
}

int launch_flow_jobs(const DevFlowJob* d_jobs, int32_t count, char* d_ws, const WsLayout& ws,
                     int32_t slots, void* stream) {
  const size_t sm = block_smem(ws);
  set_smem(flow_kernel, sm);
  flow_kernel<<<blocks_for(slots), kBlock, sm, static_cast<cudaStream_t>(stream)>>>(d_jobs, count, d_ws,
                                                                                    ws, slots);
  return static_cast<int>(cudaGetLastError());
}

int launch_slack_jobs(const DevInst* d_insts, const SlackOut* d_outs, int64_t* d_makespan,
                      int32_t count, char* d_ws, const WsLayout& ws, int32_t slots, void* stream) {
  const size_t sm = block_smem(ws);
  set_smem(slack_kernel, sm);
  slack_kernel<<<blocks_for(slots), kBlock, sm, static_cast<cudaStream_t>(stream)>>>(
      d_insts, d_outs, d_makespan, count, d_ws, ws, slots);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace pb
