/*
 * perseus_b200.h -- C ABI of the B200-native Perseus frontier generator.
 *
 * This is the drop-in boundary for the reference planner's hot path
 * (/root/reference/proj/include/perseus/frontier.hpp:166-189,
 * perseus::discover_frontier and the get_next_schedule / discretize /
 * min_energy_schedule / all_max_schedule / lookup family it is built on).
 * The reference has no C ABI; its callers bind the C++ API (CLI
 * run_optimize, tools/perseus.cpp:58-59; service characterize,
 * service.hpp:260-261).  include/perseus_b200/frontier.hpp re-exposes the
 * exact C++ signatures on top of this ABI, and INTEGRATION.md shows the
 * binding a maintainer adds.
 *
 * Plain pointers and sizes only.  A pb_batch handle is single-thread (same
 * rule as SPEC.md:292); distinct handles may be used from distinct threads.
 * Every entry point returns a pb_status; pb_last_error() gives the message of
 * the last failure on the calling thread.
 */
#ifndef PERSEUS_B200_H_
#define PERSEUS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto the reference's exception classes
 * (SURVEY.md §8b "Errors"). */
typedef enum {
  PB_OK = 0,
  PB_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (frontier.hpp:94,168; costmodel.hpp:209-213) */
  PB_ERR_OVERFLOW = 2,         /* std::overflow_error (flow.hpp:65-66,196-197) */
  PB_ERR_LOGIC = 3,            /* std::logic_error (flow.hpp:265; frontier.hpp:213) */
  PB_ERR_DOMAIN = 4,           /* DegenerateFit, std::domain_error (costmodel.hpp:50-52) */
  PB_ERR_CUDA = 5,             /* device failure (no reference counterpart) */
  PB_ERR_UNSUPPORTED = 6,      /* input outside what the device layout supports
                                  (a curve interval too long to tabulate, or a
                                  curve value outside the host tables) */
  PB_ERR_BUDGET = 7            /* BudgetExceeded (oracle.hpp:17-19): assignment
                                  space above the enumeration budget */
} pb_status;

/* Why a frontier walk ended (frontier.hpp:178-187). */
typedef enum {
  PB_STOP_AT_TMIN = 0,      /* loop condition t_planned > T_min failed */
  PB_STOP_INFEASIBLE = 1,   /* max_flow_lower_bounds returned nullopt */
  PB_STOP_INFINITE_CUT = 2, /* flow value >= infinity sentinel */
  PB_STOP_NO_PROGRESS = 3,  /* next t_planned >= current */
  PB_STOP_STEP_LIMIT = 4    /* max_steps reached (single-step mode) */
} pb_stop_reason;

/* Kinds, perseus::Kind (dag.hpp:18). */
enum { PB_KIND_FORWARD = 0, PB_KIND_BACKWARD = 1, PB_KIND_CONSTANT = 2 };

/*
 * One frontier-walk instance = (NodeDag, CostModel, tau).
 *
 * DAG (dag.hpp:50-58): computations 0..n-1; dependency edges (edge_tail[k],
 * edge_head[k]) may name the virtual source n and sink n+1; the edge list is
 * the NodeDag's (build_pipeline / finalize_custom_dag output).
 *
 * Cost model (costmodel.hpp:194-239), one entry per class c:
 *   class_is_constant[c]            CostModel::ClassModel::is_constant
 *   class_point_off[c..c+1]         Pareto points, ascending time
 *   point_freq/time/energy          ProfilePoint fields
 *   class_curve[3c..3c+2]           ExpCurve a, b, c (ignored if constant)
 *   class_t_range[2c..2c+1]         ExpCurve t_min, t_max
 * comp_class[i] selects the class of computation i.
 */
typedef struct {
  int32_t n;
  const int32_t* comp_class;
  int32_t n_edges;
  const int32_t* edge_tail;
  const int32_t* edge_head;
  int32_t n_classes;
  const uint8_t* class_is_constant;
  const int32_t* class_point_off; /* n_classes + 1 */
  const int32_t* point_freq;
  const int64_t* point_time;
  const int64_t* point_energy;
  const double* class_curve;    /* 3 * n_classes */
  const int64_t* class_t_range; /* 2 * n_classes */
  double blocking_watts;        /* BlockingPower::watts (units.hpp:19-21) */
  int64_t quantum_us;           /* CostModel::quantum_us */
  int64_t tau;                  /* planning step (frontier.hpp:167) */
  /* Optional start schedule (NULL = min_energy_schedule, frontier.hpp:73-83)
   * and step cap (0 = unbounded, > 0 = at most that many steps, -1 = no step:
   * only the discretized start point).  With start_planned_t set the walk
   * is a chain of get_next_schedule(tau) calls (frontier.hpp:90-135): no
   * clipping to T_min and no progress check; max_steps 0 means 1 there. */
  const int64_t* start_planned_t;
  int32_t max_steps;
} pb_instance_desc;

typedef struct pb_batch pb_batch;

/* Per-walk summary (Frontier, frontier.hpp:35-40). */
typedef struct {
  int64_t t_min;  /* all-max iteration time */
  int64_t t_star; /* minimum-energy iteration time */
  int32_t steps;  /* Frontier::steps */
  int32_t stop;   /* pb_stop_reason */
  int32_t status; /* pb_status of this instance */
  int32_t n_ids;  /* total delta records */
  /* curve evaluations that fell outside the host-built E_c[t] tables.  The
   * tables cover every time a walk can evaluate, so
   * this is 0; if it were not, status is PB_ERR_UNSUPPORTED -- the device
   * never substitutes its own exp for the reference's libm
   * (costmodel.hpp:47). */
  int32_t n_table_misses;
  /* device time of this walk (microseconds, %globaltimer); diagnostics */
  int32_t walk_us;
  /* warps that walked it: 1 = a walker warp, > 1 = a cooperative CTA */
  int32_t warps;
  /* walk start (microseconds of %globaltimer, low 31 bits); diagnostics:
   * start_us - min over the batch = when the walk began in the launch */
  int32_t start_us;
} pb_frontier_summary;

/* Per-point scalars; point 0 is the T* seed, point k>0 follows step k. */
typedef struct {
  int64_t t_planned;
  int64_t t_realized;
  int64_t sum_planned_e; /* sum of planned_e (mJ) */
  int64_t sum_planned_t; /* sum of planned_t (quanta) */
  int64_t sum_realized_e;
  int64_t sum_realized_t;
  int64_t cut_cost;  /* StepInfo::cut_cost of the step that produced it (0 for seed) */
  int64_t step_size; /* the tau used for that step */
  int32_t id_begin;  /* first delta record of that step */
  int32_t n_sped;    /* StepInfo::sped_up.size() */
  int32_t n_slowed;  /* StepInfo::slowed_down.size() */
  int32_t pad;
} pb_point;

const char* pb_last_error(void);
const char* pb_version(void);

/* ---- cost model (costmodel.hpp:70-149), native host code -------------- */
/* pareto_filter: returns the kept count (<= n) written to out_*. */
int32_t pb_pareto_filter(int32_t n, const int32_t* freq, const int64_t* time, const int64_t* energy,
                         int32_t* out_freq, int64_t* out_time, int64_t* out_energy);
/* fit_exp on Pareto points (ascending time): writes a, b, c, rmse. */
pb_status pb_fit_exp(int32_t n, const int64_t* time, const int64_t* energy, double* out_abcr);

/* ---- batched frontier walks ------------------------------------------- */
pb_status pb_batch_create(pb_batch** out);
/* Appends one instance (copied); *out_index receives its position. */
pb_status pb_batch_add(pb_batch* b, const pb_instance_desc* desc, int32_t* out_index);
/* Runs every instance on one CUDA device (the calling rank's):
 * pb_batch_prepare + pb_batch_launch + pb_batch_fetch. */
pb_status pb_batch_run(pb_batch* b, int32_t device);
/* Split form, so that a caller can time the device walk alone with inputs
 * already resident in HBM: prepare packs and uploads (H2D), launch runs the
 * walk kernel to completion (re-runnable), fetch copies results back (D2H). */
pb_status pb_batch_prepare(pb_batch* b, int32_t device);
pb_status pb_batch_launch(pb_batch* b, double* kernel_ms);
pb_status pb_batch_fetch(pb_batch* b);
/* Number of instances, and the estimated work (edges x steps) of one. */
int32_t pb_batch_size(const pb_batch* b);
/* Runs the batch sharded (LPT) over n_devices devices, one host thread each. */
pb_status pb_batch_run_multi(pb_batch* b, int32_t n_devices, const int32_t* devices);
pb_status pb_batch_summary(const pb_batch* b, int32_t index, pb_frontier_summary* out);
/* Copies points [0, steps] of instance `index` (steps + 1 entries). */
pb_status pb_batch_points(const pb_batch* b, int32_t index, pb_point* out, int32_t capacity);
/* Copies the delta records: ids[j] = +(c + 1) for a sped-up computation c,
 * -(c + 1) for a slowed-down one; choice[j] = its new Pareto index. */
pb_status pb_batch_deltas(const pb_batch* b, int32_t index, int32_t* ids, uint8_t* choice,
                          int32_t capacity);
/* 64-bit digest of instance `index`'s results (summary, point scalars,
 * delta records in step order; not the device pool offsets): equal digests
 * across launches = deterministic output. */
pb_status pb_batch_digest(const pb_batch* b, int32_t index, uint64_t* out);
/* Materializes schedule k of instance `index` (EnergySchedule fields,
 * frontier.hpp:20-33); any pointer may be NULL.  eff_* are summed in index
 * order exactly as detail::effective_total (frontier.hpp:51-57). */
pb_status pb_batch_schedule(const pb_batch* b, int32_t index, int32_t k, int64_t* planned_t,
                            int64_t* planned_e, int32_t* freq_mhz, int64_t* realized_t,
                            int64_t* realized_e, double* eff_planned, double* eff_realized);
/* Schedules first .. first + count - 1 of instance `index` in ONE
 * incremental replay of the delta log (the whole Frontier of
 * discover_frontier, frontier.hpp:166-189, without pb_batch_schedule's
 * replay from point 0 per call): row q of each n-wide array (caller
 * computation order) is schedule first + q; any pointer may be NULL. */
pb_status pb_batch_schedules(const pb_batch* b, int32_t index, int32_t first, int32_t count,
                             int64_t* planned_t, int64_t* planned_e, int32_t* freq_mhz, int64_t* realized_t,
                             int64_t* realized_e, double* eff_planned, double* eff_realized);
/* Optimizer artifacts from the delta log, byte-identical to the reference
 * writer (serde.hpp:250-257 frontier_csv; write_frontier_artifacts,
 * serde.hpp:304-316: schedule_json(s).dump(2) + "\n").  *len receives the
 * byte count; bytes are written when buf != NULL and cap >= *len. */
pb_status pb_batch_frontier_csv(const pb_batch* b, int32_t index, int64_t quantum_us, char* buf,
                                int64_t cap, int64_t* len);
pb_status pb_batch_schedule_json(const pb_batch* b, int32_t index, int32_t k, int64_t quantum_us,
                                 char* buf, int64_t cap, int64_t* len);
/* Device-side timing/counters of the last run: kernel ms and work counters
 * (arc scans, node updates, BFS levels), and which walk kernels ran. */
typedef struct {
  double kernel_ms;
  double h2d_ms;
  double d2h_ms;
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int64_t arc_scans;
  int64_t node_updates;
  int64_t rounds; /* BFS levels (max-flow augmenting-path searches) */
  int64_t kernel_launches;
  int64_t comp_visits; /* longest-path node visits */
  int64_t smem_walks;   /* instances walked shared-memory resident (walk_kernel_smem) */
  int64_t wide_walks;   /* instances walked by cooperative multi-warp CTAs */
  int64_t smem_region;  /* bytes of shared memory per resident walk (0: none) */
  double pack_ms;       /* host packing of the static blob (pb_batch_prepare / run) */
  int64_t warm_starts;  /* walks that resumed the flow state of the handle's last get-next walk */
} pb_run_stats;
pb_status pb_batch_stats(const pb_batch* b, pb_run_stats* out);
/* Raw per-phase profile of the last launch (cycles summed over walks, then
 * counts), n <= 16 slots (pb_internal.h kPr*): cycles in the longest-path
 * sweep, the capacity pass, max-flow phase A (feasibility repair), phase B
 * (s->t augmentation), all BFS, all augmentations, the cut/tau update, the
 * whole walk; then counts: phase-A BFS, phase-B BFS, BFS levels, augmenting
 * paths, path arcs, steps, imbalanced nodes repaired, sweep levels. */
pb_status pb_batch_profile(const pb_batch* b, int64_t* out, int32_t n);
/* Drops every instance and result but keeps the handle's device context
 * (stream, device and pinned buffers, curve values, the last derived DAG
 * layout) for the next add/run: a persistent per-thread handle serves
 * repeated single-instance calls (the drop-in's get_next_schedule) without
 * re-allocating.  A single-instance get-next run (start_planned_t set,
 * max_steps >= 0) whose start schedule is exactly where the handle's last
 * such run ended resumes that run's flow state on the device (warm start;
 * results identical to a cold start, PB_NO_CARRY disables it). */
pb_status pb_batch_clear(pb_batch* b);
void pb_batch_destroy(pb_batch* b);

/* ---- straggler sweep on the device-resident frontiers -- */
/* Savings over a cluster of `pipelines` identical pipelines when one
 * straggles to T' = llround(factor * T_min): the P-1 healthy pipelines move
 * from all-max to lookup(frontier, T') (straggler_savings, baselines.hpp:
 * 162-188; lookup, frontier.hpp:212-220; Eq. 3 energy_report,
 * emulator.hpp:77-112 with the blocking power and quantum of the instance).
 * One device thread per (instance, factor) on the frontier points of the
 * last single-device pb_batch_run.  Energies agree with the reference to
 * 1e-9 relative (the per-stage blocking terms are summed as one product). */
typedef struct {
  double factor;
  double savings_pct;
  double savings_mj;
  double all_max_mj; /* energy_report(all-max).total_mj */
  double tuned_mj;   /* energy_report(frontier point).total_mj */
  int32_t point;     /* index of the looked-up frontier point */
  int32_t status;    /* PB_OK, or PB_ERR_INVALID_ARGUMENT when T' is shorter
                        than that point's realized iteration (emulator.hpp:85) */
} pb_savings_row;
/* out[k * n_factors + j] for instance k and factors[j]; num_stages[k] is
 * NodeDag::num_stages of instance k. */
pb_status pb_batch_straggler(pb_batch* b, int32_t n_factors, const double* factors, int32_t pipelines,
                             const int32_t* num_stages, pb_savings_row* out);

/* ---- exhaustive oracle on the GPU -------------------- */
/* brute_force_frontier (oracle.hpp:47-114) for instance `index`: every
 * assignment of per-computation Pareto points enumerated on the device (one
 * thread per assignment code; longest path + effective energy summed in
 * index order exactly as simulate / detail::effective_total), the cheapest
 * (first-enumerated on ties) per distinct iteration time kept, then the
 * ascending-time, strictly-decreasing-energy frontier.  code = the
 * reference's mixed-radix assignment code (last computation fastest).
 * freq_mhz (optional) receives capacity x n frequencies, caller order. */
typedef struct {
  int64_t time;
  double eff_energy_mj;
  int64_t code;
} pb_exact_point;
pb_status pb_batch_brute_force(pb_batch* b, int32_t index, double combination_budget, int32_t device,
                               pb_exact_point* points, int32_t* freq_mhz, int32_t capacity,
                               int32_t* count);

/* ---- component kernels, exposed for parity tests ----------------------- */
/* annotate_slack (dag.hpp:233-286) for a batch of DAGs on one device.
 * Per DAG g: n[g] computations, ne[g] node-DAG edges; arrays concatenated;
 * outputs per edge-centric node (2n+2) and edge (n + ne). */
pb_status pb_annotate_slack_batch(int32_t device, int32_t count, const int32_t* n,
                                  const int32_t* ne, const int32_t* edge_tail,
                                  const int32_t* edge_head, const int64_t* durations,
                                  int64_t* earliest, int64_t* latest, uint8_t* critical,
                                  int64_t* makespan);
/* max_flow_lower_bounds + min_cut_from_flow (flow.hpp:167-278) for a batch of
 * FlowGraphs.  Per graph g: nodes[g], source[g], sink[g], m[g] edges.
 * Outputs: status[g] (pb_status), feasible[g], value[g], sentinel[g],
 * cost[g], source_side (per node), cut_dir (per edge: 1 speed-up S->T,
 * -1 slow-down T->S, 0 otherwise). */
pb_status pb_flow_min_cut_batch(int32_t device, int32_t count, const int32_t* nodes,
                                const int32_t* source, const int32_t* sink, const int32_t* m,
                                const int32_t* tail, const int32_t* head, const int64_t* lower,
                                const int64_t* upper, const uint8_t* infinite, int32_t* status,
                                uint8_t* feasible, int64_t* value, int64_t* sentinel,
                                int64_t* cost, uint8_t* source_side, int8_t* cut_dir);

/* ---- synthetic G9 workload, for bench and tests --------- */
/* Stage bases b_s (tau units) for the generator parameters. */
pb_status pb_g9_stage_bases(int32_t stages, int32_t base, double imbalance, uint32_t seed,
                            int32_t straggler_stage, double phi, int32_t* out_bases);
/* Config-5 batch instance i: N, M, imbalance, phi, straggler, seed. */
pb_status pb_g9_batch_params(int32_t i, int32_t* stages, int32_t* microbatches,
                             double* imbalance, double* phi, int32_t* straggler,
                             uint32_t* seed);
/* Appends a complete G9 instance (1F1B DAG, build_pipeline dag.hpp:112-143;
 * G9 profiles; CostModel::build with pareto_filter + fit_exp) to a batch. */
pb_status pb_batch_add_g9(pb_batch* b, int32_t stages, int32_t microbatches, int32_t base,
                          double imbalance, uint32_t seed, int32_t straggler_stage, double phi,
                          int64_t tau, int32_t* out_index);
/* Config-5 instances [first, first + count) built in parallel on `threads`
 * host threads (0 = all), appended in index order. */
pb_status pb_batch_add_g9_batch(pb_batch* b, int32_t first, int32_t count, int64_t tau, int32_t threads);
/* Config-5 instances idx[0..count) (any order, repeats allowed), built in
 * parallel, appended in list order (an LPT shard of the batch). */
pb_status pb_batch_add_g9_indices(pb_batch* b, const int32_t* idx, int32_t count, int64_t tau, int32_t threads);
/* Sets pb_instance_desc.max_steps of every instance already added (a capped
 * sample: each walk stops after that many steps). */
pb_status pb_batch_set_max_steps(pb_batch* b, int32_t max_steps);
/* The 9 (freq, time, energy) points of a stage base (descending frequency). */
pb_status pb_g9_profile(int32_t b, int32_t backward, int64_t tau, int32_t* freq, int64_t* time,
                        int64_t* energy);

#ifdef __cplusplus
}
#endif

#endif /* PERSEUS_B200_H_ */
