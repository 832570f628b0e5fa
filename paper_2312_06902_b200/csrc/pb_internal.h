// Internal layout shared by the host packer (pb_host.cpp) and the sm_100a
// kernels (pb_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cstdint>

#include "perseus_b200.h"

namespace pb {

// Walk modes.
enum : int32_t { kModeDiscover = 0, kModeGetNext = 1 };

// Internal per-instance status beyond pb_status.
enum : int32_t { kStatusLogFull = 100 };

// One packed instance: every pointer is a DEVICE address into the batch blob
// (static data) or the output blob.  Node-DAG ids: computations 0..n-1,
// virtual source n, sink n+1.  Edge-centric ids (dag.hpp:209-224):
// computation i -> edge i from node 2i to 2i+1; dependency j -> edge n+j;
// edge n+ne is the phase-A return arc sink->source (flow.hpp:196-200).
struct DevInst {
  int32_t n, ne, n_levels, mode;
  int32_t max_steps, cap_points, cap_ids, pad0;
  int64_t tau;
  double watts;
  int64_t quantum;
  // node DAG
  const int32_t* comp_class;  // [n]
  const int32_t* lvl_off;     // [n_levels + 1]
  const int32_t* lvl_comps;   // [n], topological levels (Kahn depth)
  const int32_t* in_off;      // [n + 1]
  const int32_t* in_dep;      // dependency ids j with head == comp
  const int32_t* out_off;     // [n + 1]
  const int32_t* out_dep;     // dependency ids j with tail == comp
  const int32_t* snk_dep;     // dependency ids j with head == sink
  int32_t n_snk, pad1;
  const int32_t* dep_tail;  // [ne] node-DAG ids
  const int32_t* dep_head;  // [ne]
  // edge-centric incidence (flow network), V = 2n + 2 nodes, E = n + ne + 1
  const int32_t* inc_off;  // [V + 1]
  const int32_t* inc;      // (edge << 1) | dir, dir = 1 when the node is the head
  const int32_t* ec_tail;  // [E]
  const int32_t* ec_head;  // [E]
  // cost model
  const uint8_t* cls_const;   // [classes]
  const int64_t* cls_tmin;    // [classes] curve t_min (table origin)
  const int64_t* cls_tmax;    // [classes]
  const int64_t* cls_tab;     // [classes] offset of E(t_min) in tables
  const int32_t* cls_pt_off;  // [classes + 1]
  const int64_t* pt_time;
  const int64_t* pt_energy;
  const double* tables;           // E(t) = a exp(b t) + c for t in [t_min, t_max]
  const double* cls_curve;        // [3 * classes] a, b, c (extrapolation only)
  const int64_t* start_planned_t; // get-next mode only
  // outputs; delta records go to the batch-wide pool (DeltaPool)
  pb_point* points;             // [cap_points]
  pb_frontier_summary* summary; // [1]
};

// Batch-wide append-only delta log: each step reserves a contiguous range
// with one atomicAdd, so only the used prefix is copied back.
struct DeltaPool {
  int32_t* ids;      // +(c + 1) sped up, -(c + 1) slowed down
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

// Per-warp workspace slot; arrays sized for the largest instance of a batch.
// The flow f[] persists across the steps of a walk (warm start).
struct WsLayout {
  int64_t max_n, max_v, max_e;
  int64_t off_lo, off_up, off_f, off_inf, off_crit;      // per edge
  int64_t off_bal, off_vis, off_par, off_mk;             // per node
  int64_t off_planned, off_estart, off_lend, off_rstart, off_rdur, off_pdur, off_choice;  // per comp
  int64_t off_f0, off_f1, off_touch, off_exl, off_delta;  // lists
  int64_t stride;
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
  L.off_lo = take(8 * max_e);
  L.off_up = take(8 * max_e);
  L.off_f = take(8 * max_e);
  L.off_inf = take(max_e);
  L.off_crit = take(max_e);
  L.off_bal = take(8 * max_v);
  L.off_vis = take(4 * max_v);
  L.off_par = take(4 * max_v);
  L.off_mk = take(4 * max_v);
  L.off_planned = take(8 * max_n);
  L.off_estart = take(8 * max_n);
  L.off_lend = take(8 * max_n);
  L.off_rstart = take(8 * max_n);
  L.off_rdur = take(8 * max_n);
  L.off_pdur = take(8 * max_n);
  L.off_choice = take(max_n);
  L.off_f0 = take(4 * max_v);
  L.off_f1 = take(4 * max_v);
  L.off_touch = take(4 * 2 * max_e);
  L.off_exl = take(4 * max_v);
  L.off_delta = take(4 * max_n);
  L.stride = o;
  return L;
}

// Generic flow-graph job for pb_flow_min_cut_batch: the same push-relabel
// device code on an arbitrary FlowGraph (flow.hpp:22-80).
struct DevFlowJob {
  int32_t nodes, source, sink, m;
  const int32_t* inc_off;  // [nodes + 1]
  const int32_t* inc;      // (edge << 1) | dir
  const int32_t* tail;     // [m + 1], edge m = return arc sink -> source
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

// Host-side launchers (pb_kernels.cu).
// slots = number of walker warps (one workspace each).
int launch_walks(const DevInst* d_insts, int32_t n_inst, const int32_t* d_order, int32_t* d_counter,
                 char* d_ws, const WsLayout& ws, int32_t slots, RunCounters* d_counters,
                 DeltaPool pool, void* stream);
int walk_slots_per_sm();
int launch_flow_jobs(const DevFlowJob* d_jobs, int32_t count, char* d_ws, const WsLayout& ws,
                     int32_t slots, void* stream);
// annotate_slack job outputs (per DAG).
struct SlackOut {
  const int64_t* dur;
  int64_t* earliest;
  int64_t* latest;
  uint8_t* critical;
};
int launch_slack_jobs(const DevInst* d_insts, const SlackOut* d_outs, int64_t* d_makespan,
                      int32_t count, char* d_ws, const WsLayout& ws, int32_t slots, void* stream);

}  // namespace pb
