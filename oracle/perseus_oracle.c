/*
 * perseus_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the reference CPU planner's frontier path
 * (/root/reference/proj/include/perseus/{dag,costmodel,flow,frontier,emulator}.hpp),
 * used only as the checker by tests/, __graft_entry__.smoke() and the
 * `cpu_baseline` leg of bench.py.  The product (paper_2312_06902_b200/) never
 * links, imports or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * reference's own golden vectors (test_frontier.cpp, test_flow.cpp) and
 * against fixtures produced by the reference itself (oracle/_ref/ref_driver,
 * tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_INVALID 1  /* std::invalid_argument */
#define OR_OVERFLOW 2 /* std::overflow_error   */
#define OR_LOGIC 3    /* std::logic_error      */
#define OR_CAPACITY 4 /* output buffer too small */
#define OR_DEGENERATE 5 /* DegenerateFit (costmodel.hpp:50-52) */

/* stop reasons of the walk */
#define OR_STOP_AT_TMIN 0
#define OR_STOP_INFEASIBLE 1
#define OR_STOP_INFINITE_CUT 2
#define OR_STOP_NO_PROGRESS 3

typedef __int128 i128;

/* ---------------------------------------------------------------- costmodel */

/* pareto_filter, costmodel.hpp:70-81: sort by (time asc, energy asc, freq
 * desc) and keep strictly decreasing energies. */
typedef struct { int32_t freq; int64_t time; int64_t energy; } or_point;

static int cmp_point(const void* a, const void* b) {
  const or_point* x = (const or_point*)a;
  const or_point* y = (const or_point*)b;
  if (x->time != y->time) return x->time < y->time ? -1 : 1;
  if (x->energy != y->energy) return x->energy < y->energy ? -1 : 1;
  if (x->freq != y->freq) return x->freq > y->freq ? -1 : 1;
  return 0;
}

int or_pareto_filter(int npts, const int32_t* freq, const int64_t* time, const int64_t* energy,
                     int32_t* out_freq, int64_t* out_time, int64_t* out_energy) {
  or_point* p = (or_point*)malloc(sizeof(or_point) * (size_t)(npts > 0 ? npts : 1));
  for (int i = 0; i < npts; ++i) {
    p[i].freq = freq[i];
    p[i].time = time[i];
    p[i].energy = energy[i];
  }
  qsort(p, (size_t)npts, sizeof(or_point), cmp_point);
  int k = 0;
  for (int i = 0; i < npts; ++i) {
    if (k == 0 || p[i].energy < out_energy[k - 1]) {
      out_freq[k] = p[i].freq;
      out_time[k] = p[i].time;
      out_energy[k] = p[i].energy;
      ++k;
    }
  }
  free(p);
  return k;
}

/* fit_exp, costmodel.hpp:87-149 (input already ascending time, distinct). */
int or_fit_exp(int n, const int64_t* time, const int64_t* energy, double* abc) {
  if (n < 2) return OR_INVALID;
  for (int i = 0; i + 1 < n; ++i)
    if (time[i] == time[i + 1]) return OR_INVALID;
  const double e_min = (double)energy[n - 1];
  const double e_max = (double)energy[0];
  if (e_min == e_max) return OR_DEGENERATE;
  if (e_min > e_max) return OR_INVALID;
  if (n == 2) {
    const double t1 = (double)time[0], t2 = (double)time[1];
    const double e1 = (double)energy[0], e2 = (double)energy[1];
    const double b = log(e2 / e1) / (t2 - t1);
    abc[0] = e1 * exp(-b * t1);
    abc[1] = b;
    abc[2] = 0.0;
    return OR_OK;
  }
  double lowest = e_min;
  for (int i = 0; i < n; ++i)
    if ((double)energy[i] < lowest) lowest = (double)energy[i];
  double best = -1.0;
  for (int j = 0; j < 64; ++j) {
    const double c = (double)j * (0.999 * lowest) / 63.0;
    double st = 0, sy = 0, stt = 0, sty = 0;
    for (int i = 0; i < n; ++i) {
      const double t = (double)time[i];
      const double y = log((double)energy[i] - c);
      st += t;
      sy += y;
      stt += t * t;
      sty += t * y;
    }
    const double dn = (double)n;
    const double slope = (dn * sty - st * sy) / (dn * stt - st * st);
    const double intercept = (sy - slope * st) / dn;
    const double a = exp(intercept);
    double sq = 0;
    for (int i = 0; i < n; ++i) {
      const double r = a * exp(slope * (double)time[i]) + c - (double)energy[i];
      sq += r * r;
    }
    const double rmse = sqrt(sq / dn);
    if (best < 0 || rmse < best) {
      best = rmse;
      abc[0] = a;
      abc[1] = slope;
      abc[2] = c;
    }
  }
  if (abc[1] >= 0) return OR_DEGENERATE;
  return OR_OK;
}

/* ---------------------------------------------------------------- instance */

typedef struct {
  int n;                 /* computations */
  const int32_t* cls;    /* class per computation */
  int ne;                /* node-DAG edges (source = n, sink = n + 1) */
  const int32_t* et;
  const int32_t* eh;
  int ncls;
  const uint8_t* is_const;
  const int32_t* pt_off; /* ncls + 1 offsets into the Pareto arrays */
  const int32_t* pt_freq;
  const int64_t* pt_time;
  const int64_t* pt_energy;
  const double* curve;    /* 3 per class: a, b, c */
  const int64_t* t_range; /* 2 per class: t_min, t_max */
  double watts;
  int64_t quantum;
} or_instance;

static double eval_curve(const or_instance* I, int c, double t) {
  /* ExpCurve::eval, costmodel.hpp:47 */
  return I->curve[3 * c] * exp(I->curve[3 * c + 1] * t) + I->curve[3 * c + 2];
}

static int64_t planned_energy(const or_instance* I, int c, int64_t t) {
  /* frontier.hpp:59-62 */
  if (I->is_const[c]) return I->pt_energy[I->pt_off[c]];
  return (int64_t)llround(eval_curve(I, c, (double)t));
}

static double effective_total(const int64_t* e, const int64_t* t, int n, double watts, int64_t q) {
  /* frontier.hpp:51-57 with units.hpp:38-48 */
  double total = 0;
  for (int i = 0; i < n; ++i) total += (double)e[i] - watts * (double)t[i] * (double)q * 1e-3;
  return total;
}

/* Kahn order with a FIFO queue, dag.hpp:64-86 (ties resolved by node id). */
static int topo_order(int nn, int m, const int32_t* tail, const int32_t* head, int32_t* order) {
  int32_t* indeg = (int32_t*)calloc((size_t)nn, sizeof(int32_t));
  int32_t* off = (int32_t*)calloc((size_t)nn + 1, sizeof(int32_t));
  int32_t* adj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  for (int k = 0; k < m; ++k) {
    ++off[tail[k] + 1];
    ++indeg[head[k]];
  }
  for (int v = 0; v < nn; ++v) off[v + 1] += off[v];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)nn);
  memcpy(fill, off, sizeof(int32_t) * (size_t)nn);
  for (int k = 0; k < m; ++k) adj[fill[tail[k]]++] = head[k];
  int qh = 0, qt = 0;
  for (int v = 0; v < nn; ++v)
    if (indeg[v] == 0) order[qt++] = v;
  while (qh < qt) {
    const int u = order[qh++];
    for (int j = off[u]; j < off[u + 1]; ++j)
      if (--indeg[adj[j]] == 0) order[qt++] = adj[j];
  }
  free(indeg);
  free(off);
  free(adj);
  free(fill);
  return qt == nn ? OR_OK : OR_INVALID;
}

/* simulate, emulator.hpp:28-55: longest path on the node DAG. */
int or_simulate(const or_instance* I, const int64_t* dur, int64_t* makespan, int64_t* start) {
  const int n = I->n, nn = n + 2;
  for (int i = 0; i < n; ++i)
    if (dur[i] < 0) return OR_INVALID;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)nn);
  if (topo_order(nn, I->ne, I->et, I->eh, order) != OR_OK) {
    free(order);
    return OR_INVALID;
  }
  int64_t* begin = (int64_t*)calloc((size_t)nn, sizeof(int64_t));
  /* successor lists in insertion order */
  int32_t* off = (int32_t*)calloc((size_t)nn + 1, sizeof(int32_t));
  int32_t* adj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(I->ne > 0 ? I->ne : 1));
  for (int k = 0; k < I->ne; ++k) ++off[I->et[k] + 1];
  for (int v = 0; v < nn; ++v) off[v + 1] += off[v];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)nn);
  memcpy(fill, off, sizeof(int32_t) * (size_t)nn);
  for (int k = 0; k < I->ne; ++k) adj[fill[I->et[k]]++] = I->eh[k];
  for (int o = 0; o < nn; ++o) {
    const int u = order[o];
    const int64_t du = u < n ? dur[u] : 0;
    for (int j = off[u]; j < off[u + 1]; ++j) {
      const int v = adj[j];
      if (begin[u] + du > begin[v]) begin[v] = begin[u] + du;
    }
  }
  *makespan = begin[n + 1];
  if (start) memcpy(start, begin, sizeof(int64_t) * (size_t)n);
  free(order);
  free(begin);
  free(off);
  free(adj);
  free(fill);
  return OR_OK;
}

/* -------------------------------------------------------------- edge-centric */

typedef struct {
  int nn, source, sink, m;
  int32_t* tail;
  int32_t* head;
  int32_t* comp; /* -1 for dependency connectors */
} or_edag;

/* to_edge_centric, dag.hpp:209-224 */
static void edge_centric(const or_instance* I, or_edag* E) {
  const int n = I->n;
  E->nn = 2 * n + 2;
  E->source = 2 * n;
  E->sink = 2 * n + 1;
  E->m = n + I->ne;
  E->tail = (int32_t*)malloc(sizeof(int32_t) * (size_t)E->m);
  E->head = (int32_t*)malloc(sizeof(int32_t) * (size_t)E->m);
  E->comp = (int32_t*)malloc(sizeof(int32_t) * (size_t)E->m);
  for (int i = 0; i < n; ++i) {
    E->tail[i] = 2 * i;
    E->head[i] = 2 * i + 1;
    E->comp[i] = i;
  }
  for (int k = 0; k < I->ne; ++k) {
    const int u = I->et[k], v = I->eh[k];
    E->tail[n + k] = (u == n) ? E->source : 2 * u + 1;
    E->head[n + k] = (v == n + 1) ? E->sink : 2 * v;
    E->comp[n + k] = -1;
  }
}

static void free_edag(or_edag* E) {
  free(E->tail);
  free(E->head);
  free(E->comp);
}

/* annotate_slack, dag.hpp:233-286 */
static int annotate_slack(const or_edag* E, const int64_t* dur, int n, int64_t* earliest,
                          int64_t* latest, uint8_t* critical, int64_t* makespan) {
  for (int i = 0; i < n; ++i)
    if (dur[i] < 0) return OR_INVALID;
  const int nn = E->nn;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)nn);
  if (topo_order(nn, E->m, E->tail, E->head, order) != OR_OK) {
    free(order);
    return OR_INVALID;
  }
  int32_t* off = (int32_t*)calloc((size_t)nn + 1, sizeof(int32_t));
  int32_t* adj = (int32_t*)malloc(sizeof(int32_t) * (size_t)E->m);
  for (int k = 0; k < E->m; ++k) ++off[E->tail[k] + 1];
  for (int v = 0; v < nn; ++v) off[v + 1] += off[v];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)nn);
  memcpy(fill, off, sizeof(int32_t) * (size_t)nn);
  for (int k = 0; k < E->m; ++k) adj[fill[E->tail[k]]++] = k;
#define DUR(k) (E->comp[k] >= 0 ? dur[E->comp[k]] : 0)
  for (int v = 0; v < nn; ++v) earliest[v] = 0;
  for (int o = 0; o < nn; ++o) {
    const int u = order[o];
    for (int j = off[u]; j < off[u + 1]; ++j) {
      const int k = adj[j];
      const int64_t c = earliest[u] + DUR(k);
      if (c > earliest[E->head[k]]) earliest[E->head[k]] = c;
    }
  }
  const int64_t ms = earliest[E->sink];
  for (int v = 0; v < nn; ++v) latest[v] = ms;
  for (int o = nn - 1; o >= 0; --o) {
    const int u = order[o];
    for (int j = off[u]; j < off[u + 1]; ++j) {
      const int k = adj[j];
      const int64_t c = latest[E->head[k]] - DUR(k);
      if (c < latest[u]) latest[u] = c;
    }
  }
  for (int k = 0; k < E->m; ++k) {
    const int t = E->tail[k], h = E->head[k];
    critical[k] = earliest[t] == latest[t] && earliest[h] == latest[h] &&
                  earliest[t] + DUR(k) == earliest[h];
  }
#undef DUR
  *makespan = ms;
  free(order);
  free(off);
  free(adj);
  free(fill);
  return OR_OK;
}

int or_annotate_slack(int n, int ne, const int32_t* et, const int32_t* eh, const int64_t* dur,
                      int64_t* earliest, int64_t* latest, uint8_t* critical, int64_t* makespan) {
  or_instance I;
  memset(&I, 0, sizeof I);
  I.n = n;
  I.ne = ne;
  I.et = et;
  I.eh = eh;
  or_edag E;
  edge_centric(&I, &E);
  const int rc = annotate_slack(&E, dur, n, earliest, latest, critical, makespan);
  free_edag(&E);
  return rc;
}

/* ---------------------------------------------------------------- flow */

typedef struct {
  int nn, s, t, m;
  const int32_t* tail;
  const int32_t* head;
  const int64_t* lower;
  const int64_t* upper;
  const uint8_t* inf;
} or_flowgraph;

/* infinity_sentinel, flow.hpp:58-68 */
static int sentinel_of(const or_flowgraph* g, int64_t* out) {
  i128 sum = 0;
  for (int i = 0; i < g->m; ++i) {
    sum += g->lower[i];
    if (!g->inf[i]) sum += g->upper[i];
  }
  sum += 1;
  if (sum > (i128)(INT64_MAX / 4)) return OR_OVERFLOW;
  *out = (int64_t)sum;
  return OR_OK;
}

/* ResidualNet, flow.hpp:99-158: paired arcs, adjacency in insertion order. */
typedef struct {
  int nn, na, cap_arcs;
  int32_t* heads;
  int64_t* caps;
  int32_t* from; /* tail per arc, to build adjacency */
  int32_t* off;
  int32_t* adj;
} or_resnet;

static void rn_init(or_resnet* r, int nn, int max_pairs) {
  r->nn = nn;
  r->na = 0;
  r->cap_arcs = 2 * max_pairs;
  r->heads = (int32_t*)malloc(sizeof(int32_t) * (size_t)r->cap_arcs);
  r->caps = (int64_t*)malloc(sizeof(int64_t) * (size_t)r->cap_arcs);
  r->from = (int32_t*)malloc(sizeof(int32_t) * (size_t)r->cap_arcs);
  r->off = NULL;
  r->adj = NULL;
}

static int rn_add(or_resnet* r, int from, int to, int64_t cf, int64_t cb) {
  const int id = r->na;
  r->heads[id] = to;
  r->caps[id] = cf;
  r->from[id] = from;
  r->heads[id + 1] = from;
  r->caps[id + 1] = cb;
  r->from[id + 1] = to;
  r->na += 2;
  return id;
}

static void rn_finish(or_resnet* r) {
  r->off = (int32_t*)calloc((size_t)r->nn + 1, sizeof(int32_t));
  r->adj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(r->na > 0 ? r->na : 1));
  for (int a = 0; a < r->na; ++a) ++r->off[r->from[a] + 1];
  for (int v = 0; v < r->nn; ++v) r->off[v + 1] += r->off[v];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)r->nn);
  memcpy(fill, r->off, sizeof(int32_t) * (size_t)r->nn);
  for (int a = 0; a < r->na; ++a) r->adj[fill[r->from[a]]++] = a;
  free(fill);
}

static void rn_free(or_resnet* r) {
  free(r->heads);
  free(r->caps);
  free(r->from);
  free(r->off);
  free(r->adj);
}

/* ResidualNet::run, flow.hpp:117-152: Edmonds-Karp, BFS in arc order. */
static int64_t rn_run(or_resnet* r, int s, int t, int* paths) {
  int64_t total = 0;
  int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)r->nn);
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (size_t)r->nn);
  for (;;) {
    for (int v = 0; v < r->nn; ++v) parent[v] = -1;
    parent[s] = -2;
    int qh = 0, qt = 0;
    queue[qt++] = s;
    while (qh < qt && parent[t] == -1) {
      const int v = queue[qh++];
      for (int j = r->off[v]; j < r->off[v + 1]; ++j) {
        const int a = r->adj[j];
        const int w = r->heads[a];
        if (r->caps[a] > 0 && parent[w] == -1) {
          parent[w] = a;
          queue[qt++] = w;
        }
      }
    }
    if (parent[t] == -1) break;
    int64_t b = INT64_MAX;
    for (int v = t; v != s;) {
      const int a = parent[v];
      if (r->caps[a] < b) b = r->caps[a];
      v = r->heads[a ^ 1];
    }
    for (int v = t; v != s;) {
      const int a = parent[v];
      r->caps[a] -= b;
      r->caps[a ^ 1] += b;
      v = r->heads[a ^ 1];
    }
    total += b;
    if (paths) ++*paths;
  }
  free(parent);
  free(queue);
  return total;
}

/* max_flow_lower_bounds, flow.hpp:167-229.  Returns OR_OK with *feasible. */
static int max_flow_lb(const or_flowgraph* g, int* feasible, int64_t* flow, int64_t* value) {
  int64_t sentinel;
  int rc = sentinel_of(g, &sentinel);
  if (rc) return rc;
  const int n = g->nn, ss = n, st = n + 1;
  or_resnet aux;
  rn_init(&aux, n + 2, g->m + 2 * n + 1);
  int32_t* earc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->m > 0 ? g->m : 1));
  int64_t* lin = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  int64_t* lout = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  i128 aux_total = 0;
  for (int i = 0; i < g->m; ++i) {
    const int64_t up = g->inf[i] ? sentinel : g->upper[i];
    const int64_t slack = up - g->lower[i];
    earc[i] = rn_add(&aux, g->tail[i], g->head[i], slack, 0);
    lin[g->head[i]] += g->lower[i];
    lout[g->tail[i]] += g->lower[i];
    aux_total += slack;
  }
  int64_t lower_total = 0;
  for (int v = 0; v < n; ++v) {
    if (lin[v] > 0) {
      rn_add(&aux, ss, v, lin[v], 0);
      lower_total += lin[v];
      aux_total += lin[v];
    }
    if (lout[v] > 0) {
      rn_add(&aux, v, st, lout[v], 0);
      aux_total += lout[v];
    }
  }
  if (aux_total + 1 > (i128)(INT64_MAX / 2)) {
    rn_free(&aux);
    free(earc);
    free(lin);
    free(lout);
    return OR_OVERFLOW;
  }
  const int64_t ret_cap = (int64_t)aux_total + 1;
  const int ret_arc = rn_add(&aux, g->t, g->s, ret_cap, 0);
  rn_finish(&aux);
  int paths = 0;
  const int64_t sat = rn_run(&aux, ss, st, &paths);
  if (sat != lower_total) {
    *feasible = 0;
    rn_free(&aux);
    free(earc);
    free(lin);
    free(lout);
    return OR_OK;
  }
  *feasible = 1;
  int64_t* base = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->m > 0 ? g->m : 1));
  for (int i = 0; i < g->m; ++i) {
    const int64_t up = g->inf[i] ? sentinel : g->upper[i];
    const int64_t slack = up - g->lower[i];
    base[i] = g->lower[i] + (slack - aux.caps[earc[i]]);
  }
  const int64_t base_value = ret_cap - aux.caps[ret_arc];
  or_resnet net;
  rn_init(&net, n, g->m);
  int32_t* arc2 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->m > 0 ? g->m : 1));
  for (int i = 0; i < g->m; ++i) {
    const int64_t up = g->inf[i] ? sentinel : g->upper[i];
    arc2[i] = rn_add(&net, g->tail[i], g->head[i], up - base[i], base[i] - g->lower[i]);
  }
  rn_finish(&net);
  const int64_t extra = rn_run(&net, g->s, g->t, &paths);
  for (int i = 0; i < g->m; ++i) flow[i] = g->lower[i] + net.caps[arc2[i] ^ 1];
  *value = base_value + extra;
  rn_free(&aux);
  rn_free(&net);
  free(earc);
  free(lin);
  free(lout);
  free(base);
  free(arc2);
  return OR_OK;
}

/* min_cut_from_flow, flow.hpp:234-278.  speed/slow lists in edge order. */
static int min_cut(const or_flowgraph* g, const int64_t* flow, uint8_t* side, int32_t* speed,
                   int* nspeed, int32_t* slow, int* nslow, int64_t* cost) {
  int64_t sentinel;
  int rc = sentinel_of(g, &sentinel);
  if (rc) return rc;
  const int nn = g->nn;
  /* incidence lists in edge order: (edge, forward) tail side then head side */
  int32_t* off = (int32_t*)calloc((size_t)nn + 1, sizeof(int32_t));
  int32_t* inc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * g->m + 1));
  for (int i = 0; i < g->m; ++i) {
    ++off[g->tail[i] + 1];
    ++off[g->head[i] + 1];
  }
  for (int v = 0; v < nn; ++v) off[v + 1] += off[v];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)nn);
  memcpy(fill, off, sizeof(int32_t) * (size_t)nn);
  for (int i = 0; i < g->m; ++i) {
    inc[fill[g->tail[i]]++] = 2 * i;     /* forward */
    inc[fill[g->head[i]]++] = 2 * i + 1; /* backward */
  }
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (size_t)nn);
  for (int v = 0; v < nn; ++v) side[v] = 0;
  side[g->s] = 1;
  int qh = 0, qt = 0;
  queue[qt++] = g->s;
  while (qh < qt) {
    const int v = queue[qh++];
    for (int j = off[v]; j < off[v + 1]; ++j) {
      const int e = inc[j] >> 1, fwd = !(inc[j] & 1);
      const int other = fwd ? g->head[e] : g->tail[e];
      if (side[other]) continue;
      const int64_t up = g->inf[e] ? sentinel : g->upper[e];
      const int ok = fwd ? (flow[e] < up) : (flow[e] > g->lower[e]);
      if (ok) {
        side[other] = 1;
        queue[qt++] = other;
      }
    }
  }
  free(off);
  free(inc);
  free(fill);
  free(queue);
  if (side[g->t]) return OR_LOGIC;
  int64_t c = 0;
  int ns = 0, nl = 0;
  for (int i = 0; i < g->m; ++i) {
    const int ts = side[g->tail[i]], hs = side[g->head[i]];
    if (ts && !hs) {
      if (speed) speed[ns] = i;
      ++ns;
      c += g->inf[i] ? sentinel : g->upper[i];
    } else if (!ts && hs) {
      if (slow) slow[nl] = i;
      ++nl;
      c -= g->lower[i];
    }
  }
  *nspeed = ns;
  *nslow = nl;
  *cost = c;
  return OR_OK;
}

/* Flat entry for the flow corpus tests: max_flow_lower_bounds followed by
 * min_cut_from_flow.  *feasible = 0 means nullopt. */
int or_flow_min_cut(int nn, int s, int t, int m, const int32_t* tail, const int32_t* head,
                    const int64_t* lower, const int64_t* upper, const uint8_t* inf, int* feasible,
                    int64_t* value, int64_t* sentinel, uint8_t* side, int32_t* speed, int* nspeed,
                    int32_t* slow, int* nslow, int64_t* cost) {
  or_flowgraph g = {nn, s, t, m, tail, head, lower, upper, inf};
  int rc = sentinel_of(&g, sentinel);
  if (rc) return rc;
  int64_t* flow = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  rc = max_flow_lb(&g, feasible, flow, value);
  if (rc == OR_OK && *feasible) rc = min_cut(&g, flow, side, speed, nspeed, slow, nslow, cost);
  free(flow);
  return rc;
}

/* ---------------------------------------------------------------- frontier */

typedef struct {
  int64_t* planned_t;
  int64_t* planned_e;
  int64_t t_planned;
  double eff_planned;
} or_sched;

static int refresh_totals(const or_instance* I, or_sched* s) {
  /* frontier.hpp:64-67 */
  int rc = or_simulate(I, s->planned_t, &s->t_planned, NULL);
  if (rc) return rc;
  s->eff_planned = effective_total(s->planned_e, s->planned_t, I->n, I->watts, I->quantum);
  return OR_OK;
}

typedef struct {
  int64_t t_realized;
  double eff_realized;
  uint64_t hash;
  int64_t sum_planned_e, sum_realized_e;
} or_point_out;

static void fnv_add(uint64_t* h, int64_t v) {
  uint64_t u = (uint64_t)v;
  for (int i = 0; i < 8; ++i) {
    *h ^= (u >> (8 * i)) & 0xffu;
    *h *= 1099511628211ull;
  }
}

/* discretize, frontier.hpp:140-161 (+ the schedule hash of ref_driver.cpp). */
static int discretize(const or_instance* I, const or_sched* s, or_point_out* out, int32_t* freq_out,
                      int64_t* rt_out) {
  const int n = I->n;
  int32_t* fr = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int64_t* rt = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* re = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    const int c = I->cls[i];
    int chosen = I->pt_off[c];
    for (int p = I->pt_off[c]; p < I->pt_off[c + 1]; ++p)
      if (I->pt_time[p] <= s->planned_t[i]) chosen = p;
    fr[i] = I->pt_freq[chosen];
    rt[i] = I->pt_time[chosen];
    re[i] = I->pt_energy[chosen];
  }
  int rc = or_simulate(I, rt, &out->t_realized, NULL);
  out->eff_realized = effective_total(re, rt, n, I->watts, I->quantum);
  uint64_t h = 1469598103934665603ull;
  int64_t spe = 0, sre = 0;
  for (int i = 0; i < n; ++i) fnv_add(&h, s->planned_t[i]);
  for (int i = 0; i < n; ++i) {
    fnv_add(&h, s->planned_e[i]);
    spe += s->planned_e[i];
  }
  for (int i = 0; i < n; ++i) fnv_add(&h, fr[i]);
  for (int i = 0; i < n; ++i) fnv_add(&h, rt[i]);
  for (int i = 0; i < n; ++i) {
    fnv_add(&h, re[i]);
    sre += re[i];
  }
  out->hash = h;
  out->sum_planned_e = spe;
  out->sum_realized_e = sre;
  if (freq_out) memcpy(freq_out, fr, sizeof(int32_t) * (size_t)n);
  if (rt_out) memcpy(rt_out, rt, sizeof(int64_t) * (size_t)n);
  free(fr);
  free(rt);
  free(re);
  return rc;
}

/* get_next_schedule, frontier.hpp:90-135.  *stop != 0 means nullopt. */
static int get_next(const or_instance* I, const or_edag* E, const or_sched* cur, int64_t tau,
                    or_sched* next, int* stop, int64_t* cut_cost, int32_t* sped, int* nsped,
                    int32_t* slowed, int* nslowed) {
  const int n = I->n;
  if (tau <= 0) return OR_INVALID;
  int64_t* earliest = (int64_t*)malloc(sizeof(int64_t) * (size_t)E->nn);
  int64_t* latest = (int64_t*)malloc(sizeof(int64_t) * (size_t)E->nn);
  uint8_t* crit = (uint8_t*)malloc((size_t)E->m);
  int64_t ms;
  int rc = annotate_slack(E, cur->planned_t, n, earliest, latest, crit, &ms);
  if (rc) goto out0;
  /* critical_subdag (dag.hpp:290-299) + build_capacity_dag (flow.hpp:285-317) */
  int m = 0;
  for (int k = 0; k < E->m; ++k) m += crit[k] != 0;
  int32_t* tl = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
  int32_t* hd = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
  int32_t* cp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
  int64_t* lo = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t* up = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  uint8_t* inf = (uint8_t*)malloc((size_t)(m + 1));
  int j = 0;
  for (int k = 0; k < E->m; ++k) {
    if (!crit[k]) continue;
    tl[j] = E->tail[k];
    hd[j] = E->head[k];
    cp[j] = E->comp[k];
    lo[j] = 0;
    up[j] = 0;
    inf[j] = 1;
    const int comp = E->comp[k];
    if (comp >= 0 && !I->is_const[I->cls[comp]]) {
      const int c = I->cls[comp];
      const int64_t t = cur->planned_t[comp];
      const int can_speed = t - tau >= I->t_range[2 * c];
      const int can_slow = t + tau <= I->t_range[2 * c + 1];
      int64_t l = 0;
      if (can_slow) {
        const double em = eval_curve(I, c, (double)t) - eval_curve(I, c, (double)(t + tau));
        const int64_t r = (int64_t)llround(em);
        l = r > 0 ? r : 0;
      }
      lo[j] = l;
      if (can_speed) {
        const double ep = eval_curve(I, c, (double)(t - tau)) - eval_curve(I, c, (double)t);
        const int64_t r = (int64_t)llround(ep);
        up[j] = r > l ? r : l;
        inf[j] = 0;
      }
    }
    ++j;
  }
  or_flowgraph g = {E->nn, E->source, E->sink, m, tl, hd, lo, up, inf};
  int64_t* flow = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int feasible = 0;
  int64_t value = 0, sentinel = 0;
  rc = sentinel_of(&g, &sentinel);
  if (rc) goto out1;
  rc = max_flow_lb(&g, &feasible, flow, &value);
  if (rc) goto out1;
  if (!feasible) {
    *stop = OR_STOP_INFEASIBLE;
    goto out1;
  }
  if (value >= sentinel) {
    *stop = OR_STOP_INFINITE_CUT;
    goto out1;
  }
  {
    uint8_t* side = (uint8_t*)malloc((size_t)E->nn);
    int32_t* sp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
    int32_t* sl = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
    int nsp = 0, nsl = 0;
    int64_t cost = 0;
    rc = min_cut(&g, flow, side, sp, &nsp, sl, &nsl, &cost);
    if (rc == OR_OK) {
      *stop = 0;
      memcpy(next->planned_t, cur->planned_t, sizeof(int64_t) * (size_t)n);
      memcpy(next->planned_e, cur->planned_e, sizeof(int64_t) * (size_t)n);
      *cut_cost = cost;
      *nsped = 0;
      *nslowed = 0;
      for (int q = 0; q < nsp; ++q) {
        const int comp = cp[sp[q]];
        if (comp < 0) continue;
        next->planned_t[comp] -= tau;
        sped[(*nsped)++] = comp;
      }
      for (int q = 0; q < nsl; ++q) {
        const int comp = cp[sl[q]];
        if (comp < 0) continue;
        const int c = I->cls[comp];
        if (I->is_const[c]) continue;
        if (next->planned_t[comp] + tau > I->t_range[2 * c + 1]) continue;
        next->planned_t[comp] += tau;
        slowed[(*nslowed)++] = comp;
      }
      for (int q = 0; q < *nsped; ++q)
        next->planned_e[sped[q]] = planned_energy(I, I->cls[sped[q]], next->planned_t[sped[q]]);
      for (int q = 0; q < *nslowed; ++q)
        next->planned_e[slowed[q]] =
            planned_energy(I, I->cls[slowed[q]], next->planned_t[slowed[q]]);
      rc = refresh_totals(I, next);
    }
    free(side);
    free(sp);
    free(sl);
  }
out1:
  free(tl);
  free(hd);
  free(cp);
  free(lo);
  free(up);
  free(inf);
  free(flow);
out0:
  free(earliest);
  free(latest);
  free(crit);
  return rc;
}

/* Results of one walk.  Arrays sized by the caller (max_points points,
 * max_ids sped/slowed ids); *needed reports the sizes actually required. */
typedef struct {
  int64_t t_min, t_star;
  int32_t steps, stop;
  int64_t* t_planned;   /* [points] */
  int64_t* t_realized;  /* [points] */
  double* eff_planned;  /* [points] */
  double* eff_realized; /* [points] */
  int64_t* sum_planned_e;
  int64_t* sum_realized_e;
  uint64_t* hash;       /* [points] */
  int64_t* cut_cost;    /* [steps] */
  int64_t* step_size;   /* [steps] */
  int32_t* id_off;      /* [steps + 1] offsets into ids */
  int32_t* ids;         /* sped ids as +(c + 1), slowed as -(c + 1) */
  int64_t* final_planned_t; /* [n] */
  int32_t* final_freq;      /* [n] */
} or_walk_out;

/* discover_frontier, frontier.hpp:166-189 (+ all_max_assignment,
 * emulator.hpp:140-149, and min_energy_schedule, frontier.hpp:73-83). */
int or_discover_frontier(const or_instance* I, int64_t tau, int max_points, int max_ids,
                         or_walk_out* out, int* needed_points, int* needed_ids) {
  const int n = I->n;
  if (tau <= 0) return OR_INVALID;
  int64_t* amax = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int i = 0; i < n; ++i) amax[i] = I->pt_time[I->pt_off[I->cls[i]]];
  int rc = or_simulate(I, amax, &out->t_min, NULL);
  free(amax);
  if (rc) return rc;
  or_sched cur, nxt;
  cur.planned_t = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  cur.planned_e = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  nxt.planned_t = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  nxt.planned_e = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    const int c = I->cls[i];
    const int64_t t = I->is_const[c] ? I->pt_time[I->pt_off[c]] : I->t_range[2 * c + 1];
    cur.planned_t[i] = t;
    cur.planned_e[i] = planned_energy(I, c, t);
  }
  rc = refresh_totals(I, &cur);
  or_edag E;
  edge_centric(I, &E);
  int32_t* sped = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* slowed = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* freq = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int np = 0, nid = 0;
  out->t_star = cur.t_planned;
  out->stop = OR_STOP_AT_TMIN;
  or_point_out po;
#define EMIT_POINT(S)                                                       \
  do {                                                                      \
    rc = discretize(I, &(S), &po, freq, NULL);                              \
    if (np < max_points) {                                                  \
      out->t_planned[np] = (S).t_planned;                                   \
      out->t_realized[np] = po.t_realized;                                  \
      out->eff_planned[np] = (S).eff_planned;                               \
      out->eff_realized[np] = po.eff_realized;                              \
      out->sum_planned_e[np] = po.sum_planned_e;                            \
      out->sum_realized_e[np] = po.sum_realized_e;                          \
      out->hash[np] = po.hash;                                              \
    }                                                                       \
    ++np;                                                                   \
  } while (0)
  if (rc == OR_OK) EMIT_POINT(cur);
  int steps = 0;
  if (max_points > 0) out->id_off[0] = 0;
  while (rc == OR_OK && cur.t_planned > out->t_min) {
    const int64_t step = tau < cur.t_planned - out->t_min ? tau : cur.t_planned - out->t_min;
    int stop = 0, ns = 0, nl = 0;
    int64_t cost = 0;
    rc = get_next(I, &E, &cur, step, &nxt, &stop, &cost, sped, &ns, slowed, &nl);
    if (rc) break;
    if (stop) {
      out->stop = stop;
      break;
    }
    if (nxt.t_planned >= cur.t_planned) {
      out->stop = OR_STOP_NO_PROGRESS;
      break;
    }
    or_sched tmp = cur;
    cur = nxt;
    nxt = tmp;
    if (steps < max_points - 1) {
      out->cut_cost[steps] = cost;
      out->step_size[steps] = step;
    }
    for (int q = 0; q < ns; ++q, ++nid)
      if (nid < max_ids) out->ids[nid] = sped[q] + 1;
    for (int q = 0; q < nl; ++q, ++nid)
      if (nid < max_ids) out->ids[nid] = -(slowed[q] + 1);
    ++steps;
    if (steps < max_points) out->id_off[steps] = nid;
    EMIT_POINT(cur);
  }
#undef EMIT_POINT
  out->steps = steps;
  if (out->final_planned_t) memcpy(out->final_planned_t, cur.planned_t, sizeof(int64_t) * (size_t)n);
  if (out->final_freq) memcpy(out->final_freq, freq, sizeof(int32_t) * (size_t)n);
  *needed_points = np;
  *needed_ids = nid;
  free(cur.planned_t);
  free(cur.planned_e);
  free(nxt.planned_t);
  free(nxt.planned_e);
  free(sped);
  free(slowed);
  free(freq);
  free_edag(&E);
  if (rc == OR_OK && (np > max_points || nid > max_ids)) return OR_CAPACITY;
  return rc;
}

/* lookup, frontier.hpp:212-220: index of the first point whose planned time
 * is <= min(t_star, straggler) (planned times strictly decrease). */
int or_lookup(int npoints, const int64_t* t_planned, int64_t t_star, int64_t straggler) {
  if (npoints <= 0) return -1;
  const int64_t target = t_star < straggler ? t_star : straggler;
  int lo = 0, hi = npoints;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (t_planned[mid] > target)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo == npoints ? npoints - 1 : lo;
}
