// Internal layout shared by the host packer (pb_host.cpp) and the sm_100a
// kernels (pb_kernels.cu).  Not part of the public ABI.
//
// Design rule: every per-level step of the walk (one BFS level, one
// longest-path level) must wait on at most ONE dependent global load.  Hence
//   * computations are renumbered level-major (Kahn depth), so a level is a
//     contiguous id range and static per-level data can be prefetched;
//   * the flow network is stored by incidence POSITION: entry p of node x's
//     list carries {other end, twin position, other's list range}, and the
//     residual of traversing p away from x lives at resid[p].  A BFS level
//     therefore loads {ient[p], resid[p]} in parallel and nothing else;
//   * the visited set, the frontier and the last longest-path levels live in
//     shared memory.
#pragma once

#include <cstdint>
#include <vector>

#include "perseus_b200.h"

namespace pb {

// Walk modes.
enum : int32_t { kModeDiscover = 0, kModeGetNext = 1 };

// Internal per-instance status beyond pb_status.
enum : int32_t { kStatusLogFull = 100 };

// Incidence entry (16 B, one LDG.128): the arc leaving the owning node.
// `twin` packs the position of the same edge in other's list (bits 0-25),
// a computation-arc flag (bit 26) and the degree of other's partner node
// other ^ 1 (bits 27-31; kNoPartner = no shortcut).  Computation arcs are
// the FIRST entry of both of their nodes' lists.
struct alignas(16) IEnt {
  int32_t other;      // node at the other end
  int32_t twin;       // packed, see above
  int32_t other_off;  // other's list = [other_off, other_end)
  int32_t other_end;
};
constexpr int32_t kTwinMask = (1 << 26) - 1;
constexpr int32_t kCompArc = 1 << 26;
constexpr int kPdegShift = 27;
constexpr int kNoPartner = 31;

// Per-computation static record for the capacity build (32 B): the class's
// curve interval, its table offset (tab < 0: constant class) and the
// computation edge's two incidence positions.
struct CompRec {
  int64_t tmin, tmax, tab;
  int32_t pt, ph;
};

// Host mirrors of the int2 / int4 layouts (no CUDA headers needed).
struct int2h {
  int32_t x, y;
};
struct int4h {
  int32_t x, y, z, w;
};

// Host-built position-indexed incidence (pb_host.cpp build_net).
struct NetLayout {
  std::vector<int32_t> inc_off;
  std::vector<IEnt> ient;
  std::vector<int2h> epos;
};
// pairs = n for an edge-centric walk network (nodes 2i, 2i+1 joined by
// computation edge i, i < n), 0 for a generic flow graph (no shortcut).
void build_net(int32_t V, const std::vector<int32_t>& tail, const std::vector<int32_t>& head,
               NetLayout& out, int32_t pairs = 0);

// One packed instance: every pointer is a DEVICE address into the batch blob
// (static data) or the output blob.
//
// Internal ids: computation i (0..n-1) in level-major order, orig[i] is the
// caller's id; node-DAG virtual source n, sink n+1.  Edge-centric network
// (dag.hpp:209-224): computation i -> nodes 2i (start), 2i+1 (end), source
// 2n, sink 2n+1; edge i = computation edge 2i -> 2i+1, edge n+j = dependency
// j (network order, sorted by head then tail; dep_orig maps back to the
// caller's edge index), edge n+ne = phase-A return arc sink -> source
// (flow.hpp:196-200).
struct DevInst {
  int32_t n, ne, n_levels, mode;
  int32_t max_steps, cap_points, V, E;  // E includes the return arc
  int32_t ret_pt, ret_ph, n_snk, pad1;  // return-arc positions (sink side, source side); |snk|
  int64_t tau;
  double watts;
  int64_t quantum;
  // curve tables cover [t_min - tab_mlo, t_max + tab_mhi] per class (0, 0 for
  // a discover walk, whose planned times never leave [t_min, t_max]; a
  // get-next start schedule widens them, pack())
  int64_t tab_mlo, tab_mhi;
  // node DAG (internal ids)
  const int32_t* orig;        // [n]
  const int32_t* comp_class;  // [n]
  const uint8_t* cflag;       // [n] bit 1: has an edge to the sink
  const int32_t* lvl_off;     // [n_levels + 1]
  const int32_t* ilev;        // [n] level of each computation
  const int32_t* snk;         // [n_snk] computations with an edge to the sink, ascending
  const int4* frow;           // [n] {count | has-sink << 16, first 3 predecessors (u | ring slot << 24)}
  const int4* brow;           // [n] {count, first 3 successors (same packing)}
  const int32_t* pin_off;     // [n + 1] computation predecessors
  const int32_t* pin;
  const int32_t* pout_off;    // [n + 1] computation successors
  const int32_t* pout;
  const int2* dep_nd;         // [ne] node-DAG endpoints (n = source, n + 1 = sink), network order
  const int32_t* dep_orig;    // [ne] network dependency index -> caller's edge index
  // edge-centric flow network
  const int32_t* inc_off;     // [V + 1]
  const IEnt* ient;           // [2E]
  const int2* epos;           // [E] {position at tail, position at head}
  const CompRec* crec;        // [n]
  // cost model
  const uint8_t* cls_const;   // [classes]
  const int64_t* cls_tmin;    // [classes] curve t_min (table origin)
  const int64_t* cls_tmax;    // [classes]
  const int64_t* cls_tab;     // [classes] offset of E(t_min) in tables
  const int32_t* cls_pt_off;  // [classes + 1]
  const int64_t* pt_time;
  const int64_t* pt_energy;
  const double* tables;           // E(t) = a exp(b t) + c for t in [t_min - tab_mlo, t_max + tab_mhi]
  const double* cls_curve;        // [3 * classes] a, b, c (host expansion only)
  const int64_t* start_planned_t; // get-next mode only (internal order)
  // Warm start of a get-next chain (pb_host.cpp prepare_impl): the flow
  // state a single-instance get-next walk leaves in `carry` (CarryHdr +
  // resid[2E] + cap[n] + ecrit[E] + dirty[n]); resume = 1 when this walk's
  // start schedule is exactly the state the last one ended in.
  char* carry;
  int32_t resume, pad2;
  // outputs; delta records go to the batch-wide pool (DeltaPool)
  pb_point* points;             // [cap_points]
  pb_frontier_summary* summary; // [1]
};

// Header of the warm-start carry buffer (DevInst::carry), 64 B; the arrays
// follow at 64 (resid), 64 + 16E (cap), 64 + 16E + 16n (ecrit, dirty).
struct CarryHdr {
  int64_t suml_lo, suml_hi, sumu_lo, sumu_hi;  // CapSums (int128 halves)
  int64_t ninf, R, prev_step, valid;
};
inline size_t carry_bytes(int64_t n, int64_t E) { return 64 + 16 * E + 16 * n + E + n + 64; }

// Batch-wide append-only delta log: each step reserves a contiguous range
// with one atomicAdd, so only the used prefix is copied back.
struct DeltaPool {
  int32_t* ids;      // +(c + 1) sped up, -(c + 1) slowed down (caller ids)
  uint8_t* choice;   // new Pareto index of that computation
  unsigned long long* cursor;
  long long cap;
};

// Profile slots (pb_batch_profile): cycles per phase (warp lane 0, summed over
// warps) and counts.
enum : int {
  kPrLp = 0, kPrCap, kPrPhaseA, kPrPhaseB, kPrBfs, kPrAugment, kPrUpdate, kPrWalk,
  kPrBfsA, kPrBfsB, kPrBfsLevels, kPrPaths, kPrPathHops, kPrSteps, kPrImbalanced, kPrLpLevels,
  kPrSlots
};

// Shared memory per walker warp: ping-pong BFS frontier, visited and
// partner-ok bitsets, longest-path rings (layout in pb_kernels.cu bind_ws).
constexpr int kFrontCap = 128;  // frontier entries per buffer kept in smem
// Longest-path sweep: values of the last kRingLevels levels (<= 16 per level)
// also live in a shared-memory ring per direction; a row-record neighbour is
// u | slot << 24 with slot = ring slot, or kRingNone to read global memory.
constexpr int kRingLevels = 4;
constexpr int kRingNone = 255;

// Per-warp global workspace; arrays sized for the largest instance of a batch.
// The flow (encoded in resid) persists across the steps of a walk.
struct WsLayout {
  int64_t max_n, max_v, max_e;
  int64_t off_resid;                   // int64 [2E] residual by position
  int64_t off_bal;                     // int64 [V] phase-A imbalance
  int64_t off_log;                     // int4  [V] BFS log {arc, arc before or -1, parent, node}
  int64_t off_front;                   // int4  [2V] frontier overflow (ping-pong)
  int64_t off_ecrit;                   // u8    [E] edge critical in the current network
  int64_t off_durp, off_durr;          // int64 [n]
  int64_t off_hl;                      // int64 [n] planned duration + tail
  int64_t off_fin;                     // int64 [n] planned finish, then int64 [max_n] realized finish
  int64_t off_cap;                     // int64x2 [n] {lower, upper (-1 = infinite)}
  int64_t off_key;                     // int64x2 [n] dependency-edge criticality keys (build_caps)
  int64_t off_ccrit, off_choice;       // u8 [n] (off_ccrit: dirty flags)
  int64_t off_touch, off_exl, off_delta, off_path;  // int32 lists
  int64_t off_pathlog;                 // int32 [V] log entry of each path arc (BFS restart)
  int64_t off_lvlstart;                // int32 [V + 2] first log index of each BFS level
  int64_t off_nodeli;                  // int32 [V] log index of each node in the last BFS
  int64_t off_par;                     // int32 [V] parent log index of each log entry, then
                                       // int32 [V] nearest anchor above it (path chase)
  int64_t stride;
  int32_t smem_bytes;  // dynamic shared memory per warp
  int32_t wide_par = 0;  // cooperative kernel: shared parent links for max_v log entries (0: none)
};

struct RunCounters {
  unsigned long long arc_scans;
  unsigned long long node_updates;
  unsigned long long rounds;
  unsigned long long comp_visits;
  unsigned long long prof[kPrSlots];
};

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

inline WsLayout make_ws_layout(int64_t max_n, int64_t max_v, int64_t max_e) {
  WsLayout L{};
  L.max_n = max_n;
  L.max_v = max_v;
  L.max_e = max_e;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L.off_resid = take(8 * 2 * max_e);
  L.off_bal = take(8 * max_v);
  L.off_log = take(16 * max_v);
  L.off_front = take(16 * 2 * max_v);
  L.off_ecrit = take(max_e);
  L.off_durp = take(8 * max_n);
  L.off_durr = take(8 * max_n);
  L.off_hl = take(8 * max_n);
  L.off_fin = take(16 * max_n);
  L.off_cap = take(16 * max_n);
  L.off_key = take(16 * max_n);
  L.off_ccrit = take(max_n);
  L.off_choice = take(max_n);
  L.off_touch = take(4 * 2 * max_e);
  L.off_exl = take(4 * max_v);
  L.off_delta = take(4 * max_n);
  L.off_path = take(4 * max_v);
  L.off_pathlog = take(4 * max_v);
  L.off_lvlstart = take(4 * (max_v + 2));
  L.off_nodeli = take(4 * max_v);
  L.off_par = take(8 * max_v);
  L.stride = o;
  const int64_t bitwords = (max_v + 31) / 32;
  // frontier, visited bitset, partner-ok bitset, sweep rings (fwd, bwd)
  L.smem_bytes = static_cast<int32_t>(16 * 2 * kFrontCap + 2 * align_up(4 * bitwords, 16) +
                                      2 * kRingLevels * 16 * 16);
  return L;
}

// Generic flow-graph job for pb_flow_min_cut_batch: the same device max-flow
// code on an arbitrary FlowGraph (flow.hpp:22-80).  Edge m = return arc.
struct DevFlowJob {
  int32_t nodes, source, sink, m;
  int32_t ret_pt, ret_ph, pad0, pad1;
  const int32_t* inc_off;  // [nodes + 1]
  const IEnt* ient;        // [2(m + 1)]
  const int2* epos;        // [m + 1]
  const int32_t* tail;     // [m]
  const int32_t* head;
  const int64_t* lower;    // [m]
  const int64_t* upper;    // [m]
  const uint8_t* inf;      // [m]
  // outputs
  int32_t* status;
  uint8_t* feasible;
  int64_t* value;
  int64_t* sentinel;
  int64_t* cost;
  uint8_t* side;   // [nodes]
  int8_t* cut_dir; // [m]
};

// annotate_slack job outputs (per DAG, caller ids).
struct SlackOut {
  const int64_t* dur;  // [n] caller order
  int64_t* earliest;
  int64_t* latest;
  uint8_t* critical;
};

// Straggler-sweep job of one instance (pb_batch_straggler).
struct DevStraggler {
  const pb_point* points;
  const pb_frontier_summary* summary;
  int64_t am_energy, am_time;  // all-max sums of energy (mJ) and duration (quanta)
  double watts;
  int64_t quantum;
  int32_t stages, pad;
};
int launch_straggler(const DevStraggler* d_jobs, int32_t n_inst, const double* d_factors, int32_t n_factors,
                     int32_t pipelines, pb_savings_row* d_out, void* stream);

// Exhaustive enumeration job (pb_batch_brute_force): internal-order
// topology + per-computation digit decoding (caller order for the energy sum).
struct DevBrute {
  int32_t n, pad;
  int64_t combos;
  int64_t t_lo;             // smallest possible iteration time (table origin)
  int64_t slots;            // table size
  double watts;
  int64_t quantum;
  const int32_t* orig;      // [n] internal -> caller id
  const int32_t* pin_off;   // [n + 1] internal predecessor CSR
  const int32_t* pin;
  const uint8_t* cflag;     // [n] bit 1: edge to the sink
  const int64_t* stride;    // [n] caller order
  const int32_t* radix;     // [n] caller order: Pareto points of the class
  const int32_t* poff;      // [n] caller order: first point of the class
  const int64_t* pt_time;
  const int64_t* pt_energy;
  unsigned long long* best_e;     // [slots] order-preserving key of the best energy
  unsigned long long* best_code;  // [slots]
};
int launch_brute(const DevBrute* d_job, const DevBrute& host_job, int pass, void* stream);

// Host-side launchers (pb_kernels.cu).  slots = number of walker warps (one
// workspace each).
// The first n_wide instances of the LPT order (the longest walks, which
// bound the batch) run in walk_kernel_wide: wide_ctas CTAs of wide_warps
// warps, one walk per CTA, every BFS expanded by all its warps; the rest run
// in the persistent walker kernel (`slots` warps, one walk each).
// Workspace slots: [0, wide_ctas) wide CTAs, [wide_ctas, +slots) walkers.
int launch_walks(const DevInst* d_insts, int32_t n_inst, const int32_t* d_order, int32_t* d_counter,
                 char* d_ws, const WsLayout& ws, int32_t slots, RunCounters* d_counters,
                 DeltaPool pool, int32_t n_wide, int32_t wide_ctas, int32_t wide_warps, void* stream);
int walk_slots_per_sm(const WsLayout& ws);
// Shared-memory-resident walks (walk_kernel_smem): one warp per CTA, each
// CTA's region (bytes) holds as much of its walk's hot data as fits.
// smem_walk_plan sizes the region for the largest footprint (smem_footprint)
// and reports how many such CTAs fit per SM; the kernel pulls instances from
// queue cursor d_counter[2].
int smem_walk_plan(const WsLayout& ws, int64_t footprint, int32_t* region, int32_t* ctas_per_sm);
int launch_walks_smem(const DevInst* d_insts, int32_t n_inst, const int32_t* d_order, int32_t* d_counter,
                      char* d_ws, const WsLayout& ws, int32_t region, int32_t ctas, RunCounters* d_counters,
                      DeltaPool pool, void* stream);
// Bytes a walk needs to be fully shared-memory resident (bind_smem's arrays,
// 16 B aligned each).
inline int64_t smem_footprint(int64_t n, int64_t V, int64_t E, int64_t ne, int64_t levels, int64_t nsnk) {
  const int64_t a[] = {16 * E, 32 * E, 4 * (V + 1), 16 * V, 4 * V, 4 * V, 4 * (V + 2), 4 * (levels + 1), 8 * n, 16 * n,
                       16 * n, 8 * n, 16 * n, 8 * n, E, n, 32 * n, 16 * n, 16 * n, 8 * ne, 8 * E, 8 * V, n, 4 * n,
                       4 * nsnk, 4 * n};
  int64_t t = 0;
  for (int64_t x : a) t += align_up(x, 16);
  return t;
}
int launch_flow_jobs(const DevFlowJob* d_jobs, int32_t count, char* d_ws, const WsLayout& ws,
                     int32_t slots, void* stream);
int launch_slack_jobs(const DevInst* d_insts, const SlackOut* d_outs, int64_t* d_makespan,
                      int32_t count, char* d_ws, const WsLayout& ws, int32_t slots, void* stream);

}  // namespace pb
