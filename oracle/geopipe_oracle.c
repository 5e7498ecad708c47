/* geopipe_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU oracle (checker).
 *
 * Plain-C restatement of the reference hot path (see geopipe_oracle.h). The
 * restatement favours clarity over speed: it regenerates every cell and every
 * task like the reference does, so it is only used on test-sized inputs and
 * as the "port" CPU baseline. Compiled with -ffp-contract=off so every double
 * expression rounds like the reference's x86-64 -O2 build.
 */
#include "geopipe_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */

static _Thread_local char g_err[512];
static _Thread_local int g_rc;

static void fail(int rc, const char* fmt, ...) {
  if (g_rc != GPB_OK) return; /* keep the first failure */
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  g_rc = rc;
}

const char* orc_last_error(void) { return g_err; }

static void reset_err(void) {
  g_err[0] = 0;
  g_rc = GPB_OK;
}

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz ? sz : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory\n");
    abort();
  }
  return p;
}

/* -------------------------------------------------------------- base.h */

/* ms_to_ns = llround(ms * 1e6) (base.h:15-17). */
static int64_t ms_to_ns(double ms) { return (int64_t)llround(ms * 1e6); }
/* ns_to_ms (base.h:19). */
static double ns_to_ms(int64_t ns) { return (double)ns / 1e6; }

/* ReservationList (base.h:63-124): sorted, non-overlapping intervals. */
typedef struct {
  int64_t* s;
  int64_t* e;
  int n, cap;
} resv_t;

static void resv_free(resv_t* r) {
  free(r->s);
  free(r->e);
  memset(r, 0, sizeof *r);
}

/* free_at (base.h:65-72) */
static int resv_free_at(const resv_t* r, int64_t start, int64_t end) {
  if (start >= end) return 1;
  for (int i = 0; i < r->n; ++i) {
    if (r->s[i] >= end) break;
    if (r->s[i] < end && start < r->e[i]) return 0;
  }
  return 1;
}

/* earliest_fit (base.h:75-84) */
static int64_t resv_earliest_fit(const resv_t* r, int64_t lo, int64_t len) {
  if (len <= 0) return lo;
  int64_t t = lo;
  for (int i = 0; i < r->n; ++i) {
    if (r->e[i] <= t) continue;
    if (r->s[i] >= t + len) break;
    t = r->e[i];
  }
  return t;
}

/* latest_fit (base.h:88-99) */
static int64_t resv_latest_fit(const resv_t* r, int64_t lo, int64_t hi,
                               int64_t len) {
  if (hi < lo) return lo - 1;
  if (len <= 0) return hi;
  int64_t t = hi;
  for (int i = r->n - 1; i >= 0; --i) {
    if (r->s[i] >= t + len) continue;
    if (r->e[i] <= t) break;
    t = r->s[i] - len;
    if (t < lo) return lo - 1;
  }
  return t >= lo ? t : lo - 1;
}

/* reserve (base.h:101-106): insert before the first start >= start. */
static void resv_reserve(resv_t* r, int64_t start, int64_t end) {
  if (start >= end) return;
  if (r->n == r->cap) {
    r->cap = r->cap ? 2 * r->cap : 16;
    r->s = realloc(r->s, sizeof(int64_t) * r->cap);
    r->e = realloc(r->e, sizeof(int64_t) * r->cap);
  }
  int i = 0;
  while (i < r->n && r->s[i] < start) ++i;
  memmove(r->s + i + 1, r->s + i, sizeof(int64_t) * (r->n - i));
  memmove(r->e + i + 1, r->e + i, sizeof(int64_t) * (r->n - i));
  r->s[i] = start;
  r->e[i] = end;
  r->n++;
}

/* unreserve (base.h:109-118) */
static void resv_unreserve(resv_t* r, int64_t start, int64_t end) {
  if (start >= end) return;
  for (int i = 0; i < r->n; ++i) {
    if (r->s[i] == start && r->e[i] == end) {
      memmove(r->s + i, r->s + i + 1, sizeof(int64_t) * (r->n - i - 1));
      memmove(r->e + i, r->e + i + 1, sizeof(int64_t) * (r->n - i - 1));
      r->n--;
      return;
    }
  }
  fail(GPB_ERROR, "unreserve: interval not found");
}

/* ---------------------------------------------------------- comm_model */

static const double kTcpLat[4] = {10.0, 20.0, 30.0, 40.0};
/* mbps_to_bytes_per_ms (base.h:24) of Table 1 (topology.cpp:45-52) */
static const double kTcpMbps[4] = {1220.0, 600.0, 396.0, 293.0};

static int tcp_table(const gpb_topology* t, double* lat, double* bw) {
  if (t->n_tcp > 0) {
    for (int i = 0; i < t->n_tcp; ++i) {
      lat[i] = t->tcp_latency_ms[i];
      bw[i] = t->tcp_bw[i];
    }
    return t->n_tcp;
  }
  for (int i = 0; i < 4; ++i) {
    lat[i] = kTcpLat[i];
    bw[i] = kTcpMbps[i] * 125.0;
  }
  return 4;
}

/* single_tcp_bandwidth (comm_model.cpp:8-25) */
double orc_single_tcp_bandwidth(const gpb_topology* topo, double latency_ms) {
  double lat[GPB_MAX_TCP], bw[GPB_MAX_TCP];
  int n = tcp_table(topo, lat, bw);
  if (latency_ms <= lat[0]) return bw[0];
  if (latency_ms >= lat[n - 1]) return bw[n - 1] * lat[n - 1] / latency_ms;
  for (int i = 1; i < n; ++i) {
    if (latency_ms > lat[i]) continue;
    if (latency_ms == lat[i]) return bw[i];
    double f = (log(latency_ms) - log(lat[i - 1])) /
               (log(lat[i]) - log(lat[i - 1]));
    return exp(log(bw[i - 1]) + f * (log(bw[i]) - log(bw[i - 1])));
  }
  return bw[n - 1];
}

/* effective_pair_bandwidth (comm_model.cpp:27-31) */
static double effective_pair_bandwidth(const gpb_topology* topo, double lat,
                                       int n_conns) {
  double single = orc_single_tcp_bandwidth(topo, lat);
  double v = n_conns * single;
  return v < topo->pair_bw_cap ? v : topo->pair_bw_cap; /* std::min */
}

/* allreduce_time_ms (comm_model.cpp:38-41) */
static double allreduce_time_ms(double params, int ring, double bw) {
  if (ring <= 1) return 0.0;
  return 4.0 * params * (ring - 1) / (ring * bw);
}

/* activation_bytes (comm_model.cpp:43-45) */
static int64_t activation_bytes(const gpb_scenario* sc) {
  return sc->microbatch * sc->seq_len * sc->hidden * sc->bytes_per_element;
}

/* ----------------------------------------------------------- workload */

static int partition_count(const gpb_scenario* sc) {
  return (sc->num_layers + sc->layers_per_partition - 1) /
         sc->layers_per_partition; /* workload.h:22-24 */
}

static double effective_params_per_layer(const gpb_scenario* sc) {
  return sc->params_per_layer > 0
             ? sc->params_per_layer
             : 12.0 * (double)sc->hidden * (double)sc->hidden; /* :25-29 */
}

typedef struct {
  double fwd, bwd, rec;
} profile_t;

/* resolve_profile (dc_select.cpp:12-18) + from_ratio (workload.cpp:21-33) */
static profile_t resolve_profile(const gpb_topology* topo,
                                 const gpb_scenario* sc) {
  profile_t p;
  if (sc->ratio_C > 0) {
    double comm_ms = (double)activation_bytes(sc) / topo->pair_bw_cap;
    p.fwd = comm_ms / sc->ratio_C;
    p.bwd = 2.0 * p.fwd;
    p.rec = p.fwd;
  } else {
    p.fwd = sc->fwd_ms;
    p.bwd = sc->bwd_ms;
    p.rec = sc->recompute_ms;
  }
  return p;
}

/* The plan: per stage DC, GPU numbering (build_plan, workload.cpp:57-124). */
typedef struct {
  int D, C, S, tp;
  int* stage_dc;   /* [S] */
  int* gpu;        /* [D][C][S] front GPU id */
} plan_t;

static void plan_free(plan_t* p) {
  free(p->stage_dc);
  free(p->gpu);
  memset(p, 0, sizeof *p);
}

static int scenario_order(const gpb_topology* topo, const gpb_scenario* sc,
                          int* order) {
  if (sc->n_order > 0) {
    for (int i = 0; i < sc->n_order; ++i) order[i] = sc->dc_order[i];
    return sc->n_order;
  }
  /* default_dc_order (workload.cpp:47-55): stable sort by count desc */
  int n = topo->n_dc;
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 1; i < n; ++i) { /* insertion sort is stable */
    int v = order[i], j = i - 1;
    while (j >= 0 && topo->gpu_count[order[j]] < topo->gpu_count[v]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = v;
  }
  return n;
}

/* Returns 0 when infeasible (InsufficientGpus, workload.cpp:84-89). */
static int build_plan(const gpb_topology* topo, const gpb_scenario* sc, int D,
                      plan_t* out) {
  const int C = sc->pipelines_per_cell, tp = sc->tp_degree;
  const int P = partition_count(sc);
  int order[GPB_MAX_DC];
  int n_order = scenario_order(topo, sc, order);
  int blk_dc[GPB_MAX_DC], blk_first[GPB_MAX_DC], blk_count[GPB_MAX_DC];
  int nb = 0, assigned = 0;
  for (int i = 0; i < n_order; ++i) { /* :71-83 */
    if (assigned >= P) break;
    int dc = order[i];
    int capacity = topo->gpu_count[dc] / (D * C * tp);
    int take = P - assigned < capacity ? P - assigned : capacity;
    if (take > 0) {
      blk_dc[nb] = dc;
      blk_first[nb] = assigned;
      blk_count[nb] = take;
      ++nb;
      assigned += take;
    }
  }
  if (assigned < P) return 0;
  memset(out, 0, sizeof *out);
  out->D = D;
  out->C = C;
  out->S = P;
  out->tp = tp;
  out->stage_dc = xcalloc(P, sizeof(int));
  out->gpu = xcalloc((size_t)D * C * P, sizeof(int));
  for (int b = 0; b < nb; ++b)
    for (int k = 0; k < blk_count[b]; ++k) out->stage_dc[blk_first[b] + k] = blk_dc[b];
  int dc_base[GPB_MAX_DC], next_gpu[GPB_MAX_DC];
  int base = 0;
  for (int i = 0; i < topo->n_dc; ++i) {
    dc_base[i] = base;
    base += topo->gpu_count[i];
    next_gpu[i] = 0;
  }
  for (int cell = 0; cell < D; ++cell) /* :93-122 */
    for (int pipe = 0; pipe < C; ++pipe)
      for (int s = 0; s < P; ++s) {
        int dc = out->stage_dc[s];
        out->gpu[((size_t)cell * C + pipe) * P + s] = dc_base[dc] + next_gpu[dc];
        next_gpu[dc] += tp;
      }
  return 1;
}

/* ---------------------------------------------------------- scheduler */

typedef struct {
  int C, S, M;
  int64_t fwd, bwd, rec;
  int* wan;            /* [S-1] */
  int64_t* ser_spatial, *ser_pooled, *lat;
  int64_t bytes;
} geom_t;

static void geom_free(geom_t* g) {
  free(g->wan);
  free(g->ser_spatial);
  free(g->ser_pooled);
  free(g->lat);
}

/* build_geometry (scheduler.cpp:32-76) for one cell (all cells identical). */
static void build_geometry(const gpb_topology* topo, const gpb_scenario* sc,
                           const plan_t* plan, profile_t prof, geom_t* g) {
  const int64_t bytes = activation_bytes(sc);
  const int n_conns = sc->multi_conn ? sc->n_connections : 1;
  g->C = plan->C;
  g->S = plan->S;
  g->M = sc->num_microbatches;
  g->fwd = ms_to_ns(prof.fwd);
  g->bwd = ms_to_ns(prof.bwd);
  g->rec = ms_to_ns(prof.rec);
  g->bytes = bytes;
  int nb = g->S > 1 ? g->S - 1 : 0;
  g->wan = xcalloc(nb, sizeof(int));
  g->ser_spatial = xcalloc(nb, sizeof(int64_t));
  g->ser_pooled = xcalloc(nb, sizeof(int64_t));
  g->lat = xcalloc(nb, sizeof(int64_t));
  for (int s = 0; s + 1 < g->S; ++s) {
    int a = plan->stage_dc[s], b = plan->stage_dc[s + 1];
    g->wan[s] = a != b;
    if (a != b) {
      double lat = topo->latency_ms[a][b];
      double bw = effective_pair_bandwidth(topo, lat, n_conns);
      g->ser_spatial[s] = ms_to_ns(bytes / bw);
      g->ser_pooled[s] = ms_to_ns(bytes / (g->C * bw));
      g->lat[s] = ms_to_ns(lat);
    }
  }
}

static int64_t pair_dur(const geom_t* g, int recompute) {
  return recompute ? g->rec + g->bwd : g->bwd; /* scheduler.cpp:27-29 */
}

typedef struct {
  orc_task* v;
  int64_t n, cap;
} tasks_t;

static void push_task(tasks_t* t, int gpu, int cell, int pipe, int kind, int m,
                      int s, int64_t start, int64_t end) {
  if (t->n == t->cap) {
    t->cap = t->cap ? 2 * t->cap : 256;
    t->v = realloc(t->v, sizeof(orc_task) * t->cap);
  }
  orc_task* o = &t->v[t->n++];
  o->gpu = gpu;
  o->cell = cell;
  o->pipeline = pipe;
  o->kind = kind;
  o->microbatch = m;
  o->stage = s;
  o->start = start;
  o->end = end;
}

enum { K_FWD = 0, K_BWD = 1, K_REC = 2, K_AR = 3, K_PRE = 4 };

typedef struct {
  const geom_t* g;
  const plan_t* plan;
  int cell;
  tasks_t* out;
} emit_ctx;

static int gpu_of(const emit_ctx* e, int p, int s) {
  return e->plan->gpu[((size_t)e->cell * e->plan->C + p) * e->plan->S + s];
}

/* emit_pair (scheduler.cpp:94-105) */
static void emit_pair(emit_ctx* e, int p, int s, int m, int64_t t,
                      int recompute) {
  int gpu = gpu_of(e, p, s);
  if (recompute) {
    push_task(e->out, gpu, e->cell, p, K_REC, m, s, t, t + e->g->rec);
    push_task(e->out, gpu, e->cell, p, K_BWD, m, s, t + e->g->rec,
              t + e->g->rec + e->g->bwd);
  } else {
    push_task(e->out, gpu, e->cell, p, K_BWD, m, s, t, t + e->g->bwd);
  }
}

#define IDX(s, m) ((size_t)(s) * M + (m))

/* flush_pipeline (scheduler.cpp:113-171): gpipe / varuna. */
static void flush_pipeline(emit_ctx* e, int p, int reverse_drain,
                           int barrier_last_fwd, int recompute) {
  const geom_t* g = e->g;
  const int S = g->S, M = g->M;
  int64_t* gpu_free = xcalloc(S, sizeof(int64_t));
  int64_t* arr = xcalloc((size_t)S * M, sizeof(int64_t));
  int64_t* fd = xcalloc((size_t)S * M, sizeof(int64_t));
  int64_t* garr = xcalloc((size_t)S * M, sizeof(int64_t));
  int64_t* lf = xcalloc(S, sizeof(int64_t));
  int64_t* lb = xcalloc(S, sizeof(int64_t));
  for (int m = 0; m < M; ++m) {
    for (int s = 0; s < S; ++s) {
      int64_t t = arr[IDX(s, m)] > gpu_free[s] ? arr[IDX(s, m)] : gpu_free[s];
      int64_t en = t + g->fwd;
      push_task(e->out, gpu_of(e, p, s), e->cell, p, K_FWD, m, s, t, en);
      gpu_free[s] = en;
      fd[IDX(s, m)] = en;
      if (s + 1 < S) {
        if (g->wan[s]) {
          int64_t start = en > lf[s] ? en : lf[s];
          int64_t occ = start + g->ser_spatial[s];
          lf[s] = occ;
          arr[IDX(s + 1, m)] = occ + g->lat[s];
        } else {
          arr[IDX(s + 1, m)] = en;
        }
      }
    }
  }
  const int64_t barrier = barrier_last_fwd ? fd[IDX(S - 1, M - 1)] : 0;
  const int64_t dur = pair_dur(g, recompute);
  for (int s = S - 1; s >= 0; --s) {
    for (int i = 0; i < M; ++i) {
      int m = reverse_drain ? M - 1 - i : i;
      int64_t ready = (s == S - 1) ? fd[IDX(s, m)] : garr[IDX(s, m)];
      if (barrier > ready) ready = barrier;
      int64_t t = ready > gpu_free[s] ? ready : gpu_free[s];
      emit_pair(e, p, s, m, t, recompute);
      int64_t en = t + dur;
      gpu_free[s] = en;
      if (s > 0) {
        if (g->wan[s - 1]) {
          int64_t start = en > lb[s - 1] ? en : lb[s - 1];
          int64_t occ = start + g->ser_spatial[s - 1];
          lb[s - 1] = occ;
          garr[IDX(s - 1, m)] = occ + g->lat[s - 1];
        } else {
          garr[IDX(s - 1, m)] = en;
        }
      }
    }
  }
  free(gpu_free);
  free(arr);
  free(fd);
  free(garr);
  free(lf);
  free(lb);
}

/* onef1b_pipeline (scheduler.cpp:177-267) */
static void onef1b_pipeline(emit_ctx* e, int p, int recompute) {
  const geom_t* g = e->g;
  const int S = g->S, M = g->M;
  int64_t* gpu_free = xcalloc(S, sizeof(int64_t));
  int64_t* arr = xcalloc((size_t)S * M, sizeof(int64_t));
  int64_t* fd = xcalloc((size_t)S * M, sizeof(int64_t));
  int64_t* garr = xcalloc((size_t)S * M, sizeof(int64_t));
  char* has_garr = xcalloc((size_t)S * M, 1);
  int64_t* lf = xcalloc(S, sizeof(int64_t));
  int64_t* lb = xcalloc(S, sizeof(int64_t));
  for (size_t i = 0; i < (size_t)S * M; ++i) fd[i] = -1;
  /* per-stage program: kind (0 F, 1 B) and microbatch */
  int* len = xcalloc(S, sizeof(int));
  int* seq_kind = xcalloc((size_t)S * 2 * M, sizeof(int));
  int* seq_m = xcalloc((size_t)S * 2 * M, sizeof(int));
  long remaining = 0;
  for (int s = 0; s < S; ++s) {
    int w = S - s < M ? S - s : M;
    int n = 0;
    for (int m = 0; m < w; ++m) {
      seq_kind[(size_t)s * 2 * M + n] = 0;
      seq_m[(size_t)s * 2 * M + n++] = m;
    }
    int next_f = w, next_b = 0;
    while (next_b < M) {
      seq_kind[(size_t)s * 2 * M + n] = 1;
      seq_m[(size_t)s * 2 * M + n++] = next_b++;
      if (next_f < M) {
        seq_kind[(size_t)s * 2 * M + n] = 0;
        seq_m[(size_t)s * 2 * M + n++] = next_f++;
      }
    }
    len[s] = n;
    remaining += n;
  }
  int* cursor = xcalloc(S, sizeof(int));
  const int64_t dur = pair_dur(g, recompute);
  int progress = 1;
  while (remaining > 0) {
    if (!progress) {
      fail(GPB_ERROR, "1F1B generation stalled; dependency cycle");
      break;
    }
    progress = 0;
    for (int s = S - 1; s >= 0; --s) {
      while (cursor[s] < len[s]) {
        int kind = seq_kind[(size_t)s * 2 * M + cursor[s]];
        int m = seq_m[(size_t)s * 2 * M + cursor[s]];
        if (kind == 0) {
          if (s > 0 && fd[IDX(s - 1, m)] < 0) break;
          int64_t t = arr[IDX(s, m)] > gpu_free[s] ? arr[IDX(s, m)] : gpu_free[s];
          int64_t en = t + g->fwd;
          push_task(e->out, gpu_of(e, p, s), e->cell, p, K_FWD, m, s, t, en);
          gpu_free[s] = en;
          fd[IDX(s, m)] = en;
          if (s + 1 < S) {
            if (g->wan[s]) {
              int64_t start = en > lf[s] ? en : lf[s];
              int64_t occ = start + g->ser_spatial[s];
              lf[s] = occ;
              arr[IDX(s + 1, m)] = occ + g->lat[s];
            } else {
              arr[IDX(s + 1, m)] = en;
            }
          }
        } else {
          if (fd[IDX(s, m)] < 0) break;
          int64_t ready;
          if (s == S - 1) {
            ready = fd[IDX(s, m)];
          } else if (has_garr[IDX(s, m)]) {
            ready = garr[IDX(s, m)];
          } else {
            break;
          }
          int64_t t = ready > gpu_free[s] ? ready : gpu_free[s];
          emit_pair(e, p, s, m, t, recompute);
          int64_t en = t + dur;
          gpu_free[s] = en;
          if (s > 0) {
            if (g->wan[s - 1]) {
              int64_t start = en > lb[s - 1] ? en : lb[s - 1];
              int64_t occ = start + g->ser_spatial[s - 1];
              lb[s - 1] = occ;
              garr[IDX(s - 1, m)] = occ + g->lat[s - 1];
            } else {
              garr[IDX(s - 1, m)] = en;
            }
            has_garr[IDX(s - 1, m)] = 1;
          }
        }
        ++cursor[s];
        --remaining;
        progress = 1;
      }
    }
  }
  free(gpu_free);
  free(arr);
  free(fd);
  free(garr);
  free(has_garr);
  free(lf);
  free(lb);
  free(len);
  free(seq_kind);
  free(seq_m);
  free(cursor);
}

/* ------------------------------------------------------------- ATLAS */

typedef struct {
  const geom_t* g;
  int C, S, M;
  int64_t* gpu_free;  /* [C][S] */
  int64_t* arr;       /* [C][S][M] */
  int64_t* fd;        /* [C][S][M] */
  int64_t* garr;      /* [C][S][M] */
  char* has_garr;     /* [C][S][M] */
  resv_t* res_fwd;    /* [S-1] */
  resv_t* res_bwd;    /* [S-1] */
  int* drained;       /* [C][S] */
  int64_t* pair_start;/* [C][S][M] */
} atlas_t;

#define A3(p, s, m) (((size_t)(p) * cs->S + (s)) * cs->M + (m))
#define A2(p, s) ((size_t)(p) * cs->S + (s))

/* atlas_pair_start (scheduler.cpp:287-294) */
static int64_t atlas_pair_start(atlas_t* cs, int s, int64_t lo, int64_t dur) {
  const geom_t* g = cs->g;
  if (s > 0 && g->wan[s - 1]) {
    int64_t slot = resv_earliest_fit(&cs->res_bwd[s - 1], lo + dur,
                                     g->ser_pooled[s - 1]);
    return slot - dur;
  }
  return lo;
}

/* atlas_commit_pair (scheduler.cpp:298-317) */
static void atlas_commit_pair(emit_ctx* e, atlas_t* cs, int p, int s, int m,
                              int recompute, int64_t t) {
  const geom_t* g = cs->g;
  const int64_t dur = pair_dur(g, recompute);
  emit_pair(e, p, s, m, t, recompute);
  int64_t en = t + dur;
  if (en > cs->gpu_free[A2(p, s)]) cs->gpu_free[A2(p, s)] = en;
  if (s > 0) {
    if (g->wan[s - 1]) {
      int64_t occ = en + g->ser_pooled[s - 1];
      cs->garr[A3(p, s - 1, m)] = occ + g->lat[s - 1];
    } else {
      cs->garr[A3(p, s - 1, m)] = en;
    }
    cs->has_garr[A3(p, s - 1, m)] = 1;
  }
  cs->drained[A2(p, s)] += 1;
}

/* atlas_drain_step (scheduler.cpp:321-346) */
static int atlas_drain_step(emit_ctx* e, atlas_t* cs, int p, int recompute) {
  const geom_t* g = cs->g;
  const int64_t dur = pair_dur(g, recompute);
  for (int s = cs->S - 1; s >= 0; --s) {
    int m = cs->drained[A2(p, s)];
    if (m >= cs->M) continue;
    int64_t ready;
    if (s == cs->S - 1) {
      if (cs->fd[A3(p, s, m)] < 0) continue;
      ready = cs->fd[A3(p, s, m)];
    } else {
      if (!cs->has_garr[A3(p, s, m)]) continue;
      ready = cs->garr[A3(p, s, m)];
    }
    int64_t lo = ready > cs->gpu_free[A2(p, s)] ? ready : cs->gpu_free[A2(p, s)];
    int64_t t = atlas_pair_start(cs, s, lo, dur);
    if (s > 0 && g->wan[s - 1])
      resv_reserve(&cs->res_bwd[s - 1], t + dur, t + dur + g->ser_pooled[s - 1]);
    cs->pair_start[A3(p, s, m)] = t;
    atlas_commit_pair(e, cs, p, s, m, recompute, t);
    return 1;
  }
  return 0;
}

/* atlas_cell (scheduler.cpp:348-538) */
static void atlas_cell(emit_ctx* e, int recompute, int mem_limit) {
  const geom_t* g = e->g;
  atlas_t st;
  atlas_t* cs = &st;
  const int S = g->S, M = g->M, C = g->C;
  cs->g = g;
  cs->C = C;
  cs->S = S;
  cs->M = M;
  size_t n3 = (size_t)C * S * M, n2 = (size_t)C * S;
  cs->gpu_free = xcalloc(n2, sizeof(int64_t));
  cs->arr = xcalloc(n3, sizeof(int64_t));
  cs->fd = xcalloc(n3, sizeof(int64_t));
  cs->garr = xcalloc(n3, sizeof(int64_t));
  cs->has_garr = xcalloc(n3, 1);
  cs->pair_start = xcalloc(n3, sizeof(int64_t));
  for (size_t i = 0; i < n3; ++i) {
    cs->fd[i] = -1;
    cs->pair_start[i] = -1;
  }
  cs->res_fwd = xcalloc(S, sizeof(resv_t));
  cs->res_bwd = xcalloc(S, sizeof(resv_t));
  cs->drained = xcalloc(n2, sizeof(int));

  /* Forward phase (:362-431) */
  for (int p = 0; p < C && g_rc == GPB_OK; ++p) {
    for (int m = 0; m < M && g_rc == GPB_OK; ++m) {
      int blocked = 1;
      while (blocked) {
        blocked = 0;
        for (int s = 0; s < S; ++s) {
          if (m - cs->drained[A2(p, s)] >= mem_limit) {
            blocked = 1;
            break;
          }
        }
        if (blocked && !atlas_drain_step(e, cs, p, recompute)) {
          fail(GPB_ERROR, "memory cap admission stalled: no drainable backward");
          goto done;
        }
      }
      int64_t t0 = cs->gpu_free[A2(p, 0)];
      for (;;) {
        int ok = 1;
        int64_t cur = t0;
        for (int s = 0; s < S; ++s) {
          int64_t gf = cs->gpu_free[A2(p, s)];
          int64_t start = cur > gf ? cur : gf;
          int64_t en = start + g->fwd;
          if (s + 1 < S) {
            if (g->wan[s]) {
              if (!resv_free_at(&cs->res_fwd[s], en, en + g->ser_pooled[s])) {
                int64_t slot = resv_earliest_fit(&cs->res_fwd[s], en, g->ser_pooled[s]);
                t0 += slot - en;
                ok = 0;
                break;
              }
              cur = en + g->ser_pooled[s] + g->lat[s];
            } else {
              cur = en;
            }
          }
        }
        if (ok) break;
      }
      int64_t cur = t0;
      for (int s = 0; s < S; ++s) {
        int64_t gf = cs->gpu_free[A2(p, s)];
        int64_t start = cur > gf ? cur : gf;
        int64_t en = start + g->fwd;
        push_task(e->out, gpu_of(e, p, s), e->cell, p, K_FWD, m, s, start, en);
        cs->gpu_free[A2(p, s)] = en;
        cs->fd[A3(p, s, m)] = en;
        if (s + 1 < S) {
          if (g->wan[s]) {
            int64_t occ = en + g->ser_pooled[s];
            resv_reserve(&cs->res_fwd[s], en, occ);
            cs->arr[A3(p, s + 1, m)] = occ + g->lat[s];
            cur = cs->arr[A3(p, s + 1, m)];
          } else {
            cs->arr[A3(p, s + 1, m)] = en;
            cur = en;
          }
        }
      }
    }
  }

  {
    /* Drain pass 1: greedy exact-fit (:452-505) */
    const int64_t dur = pair_dur(g, recompute);
    int* first_m = xcalloc(n2, sizeof(int));
    int* next_m = xcalloc(n2, sizeof(int));
    long remaining = 0;
    for (int p = 0; p < C; ++p)
      for (int s = 0; s < S; ++s) {
        first_m[A2(p, s)] = next_m[A2(p, s)] = cs->drained[A2(p, s)];
        remaining += M - next_m[A2(p, s)];
      }
    while (remaining > 0 && g_rc == GPB_OK) {
      int bp = -1, bs = -1, bm = -1;
      int64_t bt = 0;
      for (int s = S - 1; s >= 0; --s) {
        for (int p = 0; p < C; ++p) {
          const int m = next_m[A2(p, s)];
          if (m >= M) continue;
          int64_t ready;
          if (s == S - 1) {
            ready = cs->fd[A3(p, s, m)];
          } else {
            if (!cs->has_garr[A3(p, s, m)]) continue;
            ready = cs->garr[A3(p, s, m)];
          }
          int64_t gf = cs->gpu_free[A2(p, s)];
          int64_t t = atlas_pair_start(cs, s, ready > gf ? ready : gf, dur);
          if (bp < 0 || t < bt) {
            bt = t;
            bp = p;
            bs = s;
            bm = m;
          }
        }
      }
      if (bp < 0) {
        fail(GPB_ERROR, "atlas drain: no candidate");
        break;
      }
      const int wan_grad = bs > 0 && g->wan[bs - 1];
      if (wan_grad)
        resv_reserve(&cs->res_bwd[bs - 1], bt + dur, bt + dur + g->ser_pooled[bs - 1]);
      cs->pair_start[A3(bp, bs, bm)] = bt;
      cs->gpu_free[A2(bp, bs)] = bt + dur;
      if (bs > 0) {
        cs->garr[A3(bp, bs - 1, bm)] =
            wan_grad ? bt + dur + g->ser_pooled[bs - 1] + g->lat[bs - 1] : bt + dur;
        cs->has_garr[A3(bp, bs - 1, bm)] = 1;
      }
      ++next_m[A2(bp, bs)];
      --remaining;
    }
    /* Pass 2: right-pack (:506-529) */
    for (int s = 0; s < S; ++s) {
      const int wan_grad = s > 0 && g->wan[s - 1];
      const int64_t ser = wan_grad ? g->ser_pooled[s - 1] : 0;
      for (int p = 0; p < C; ++p) {
        for (int m = M - 2; m >= first_m[A2(p, s)]; --m) {
          int64_t cur = cs->pair_start[A3(p, s, m)];
          int64_t end_max = cs->pair_start[A3(p, s, m + 1)];
          if (s > 0) {
            int64_t consumer = cs->pair_start[A3(p, s - 1, m)];
            int64_t lim = wan_grad ? consumer - g->lat[s - 1] - ser : consumer;
            if (lim < end_max) end_max = lim;
          }
          if (end_max <= cur + dur) continue;
          if (wan_grad) {
            resv_unreserve(&cs->res_bwd[s - 1], cur + dur, cur + dur + ser);
            int64_t slot = resv_latest_fit(&cs->res_bwd[s - 1], cur + dur, end_max, ser);
            cs->pair_start[A3(p, s, m)] = slot - dur;
            resv_reserve(&cs->res_bwd[s - 1], slot, slot + ser);
          } else {
            cs->pair_start[A3(p, s, m)] = end_max - dur;
          }
        }
      }
    }
    /* Pass 3: emit (:530-537) */
    for (int s = S - 1; s >= 0; --s)
      for (int p = 0; p < C; ++p)
        for (int m = first_m[A2(p, s)]; m < M; ++m)
          atlas_commit_pair(e, cs, p, s, m, recompute, cs->pair_start[A3(p, s, m)]);
    free(first_m);
    free(next_m);
  }
done:
  for (int s = 0; s < S; ++s) {
    resv_free(&cs->res_fwd[s]);
    resv_free(&cs->res_bwd[s]);
  }
  free(cs->res_fwd);
  free(cs->res_bwd);
  free(cs->gpu_free);
  free(cs->arr);
  free(cs->fd);
  free(cs->garr);
  free(cs->has_garr);
  free(cs->pair_start);
  free(cs->drained);
}

/* finalize_schedule task order (schedule.cpp:23-45) */
static int task_cmp(const void* a_, const void* b_) {
  const orc_task* a = a_;
  const orc_task* b = b_;
#define CMP(f)                \
  if (a->f != b->f) return a->f < b->f ? -1 : 1;
  CMP(cell) CMP(pipeline) CMP(stage) CMP(start) CMP(end) CMP(microbatch)
#undef CMP
  return 0;
}

/* make_schedule (scheduler.cpp:540-572) over the first `cells` cells. */
static int make_schedule(const gpb_topology* topo, const gpb_scenario* sc,
                         const plan_t* plan, int cells, tasks_t* out,
                         int64_t* makespan) {
  profile_t prof = resolve_profile(topo, sc);
  geom_t g;
  memset(&g, 0, sizeof g);
  build_geometry(topo, sc, plan, prof, &g);
  if (sc->policy == GPB_ATLAS) {
    int mem_limit = sc->mem_limit > 0 ? sc->mem_limit : g.S;
    if (mem_limit < 1) fail(GPB_CONFIG_ERROR, "mem_limit: must be >= 1");
  }
  for (int cell = 0; cell < cells && g_rc == GPB_OK; ++cell) {
    emit_ctx e = {&g, plan, cell, out};
    switch (sc->policy) {
      case GPB_GPIPE:
        for (int p = 0; p < g.C; ++p) flush_pipeline(&e, p, 1, 1, sc->recompute);
        break;
      case GPB_VARUNA:
        for (int p = 0; p < g.C; ++p) flush_pipeline(&e, p, 0, 0, sc->recompute);
        break;
      case GPB_1F1B:
        for (int p = 0; p < g.C; ++p) onef1b_pipeline(&e, p, sc->recompute);
        break;
      case GPB_ATLAS:
        atlas_cell(&e, sc->recompute, sc->mem_limit > 0 ? sc->mem_limit : g.S);
        break;
      default:
        fail(GPB_CONFIG_ERROR, "policy: unknown policy %d", sc->policy);
    }
  }
  geom_free(&g);
  qsort(out->v, out->n, sizeof(orc_task), task_cmp);
  int64_t ms = 0;
  for (int64_t i = 0; i < out->n; ++i)
    if (out->v[i].end > ms) ms = out->v[i].end;
  *makespan = ms;
  return g_rc;
}

/* ------------------------------------------------------------ metrics */

static int gpu_cmp(const void* a_, const void* b_) {
  const orc_task* a = a_;
  const orc_task* b = b_;
  if (a->gpu != b->gpu) return a->gpu < b->gpu ? -1 : 1;
  if (a->start != b->start) return a->start < b->start ? -1 : 1;
  return 0;
}

/* utilization (bubbletea.cpp:224-238) == report().mean_utilization
 * (metrics.cpp:39-54): per-GPU clipped busy, summed in GPU-id order. */
static double utilization_of(const orc_task* tasks, int64_t n, int64_t horizon) {
  if (n == 0) return 0.0;
  orc_task* v = xcalloc(n, sizeof(orc_task));
  memcpy(v, tasks, sizeof(orc_task) * n);
  qsort(v, n, sizeof(orc_task), gpu_cmp);
  double sum = 0.0;
  long count = 0;
  for (int64_t i = 0; i < n;) {
    int gpu = v[i].gpu;
    int64_t busy = 0;
    for (; i < n && v[i].gpu == gpu; ++i) {
      int64_t lo = v[i].start > 0 ? v[i].start : 0;
      int64_t hi = v[i].end < horizon ? v[i].end : horizon;
      busy += hi - lo > 0 ? hi - lo : 0;
    }
    sum += (double)busy / (double)horizon;
    ++count;
  }
  free(v);
  return sum / (double)count;
}

/* ----------------------------------------------------------- dc_select */

static int validate(const gpb_topology* topos, const gpb_scenario* sc) {
  (void)topos;
  if (sc->pipelines_per_cell < 1)
    fail(GPB_CONFIG_ERROR, "select.pipelines_per_cell: must be >= 1");
  else if (sc->tp_degree < 1)
    fail(GPB_CONFIG_ERROR, "select.tp_degree: must be >= 1");
  else if (sc->policy < 0 || sc->policy > 3)
    fail(GPB_CONFIG_ERROR, "policy: unknown policy");
  else if (sc->ratio_C <= 0 && (sc->fwd_ms <= 0 || sc->bwd_ms <= 0 || sc->recompute_ms < 0))
    fail(GPB_CONFIG_ERROR, "compute: durations must be positive");
  return g_rc;
}

int orc_select(const gpb_topology* topos, const gpb_scenario* sc, gpb_row* rows,
               int32_t cap, int32_t* n_rows, int32_t* chosen_d,
               int64_t* gpus_used) {
  reset_err();
  if (validate(topos, sc) != GPB_OK) return g_rc;
  const gpb_topology* topo = &topos[sc->topology];
  /* default_d_max (dc_select.cpp:20-25) */
  long long total = 0;
  for (int i = 0; i < topo->n_dc; ++i) total += topo->gpu_count[i];
  long long per_cell = (long long)sc->pipelines_per_cell * partition_count(sc) * sc->tp_degree;
  long long dflt = total / per_cell;
  if (dflt < 0) dflt = 0;
  int d_max = sc->d_max > 0 ? sc->d_max : (int)dflt;
  if (d_max < 1) d_max = 1;
  *n_rows = d_max;
  int chosen = 0;
  double chosen_thr = 0.0;
  for (int d = 1; d <= d_max && g_rc == GPB_OK; ++d) {
    gpb_row r;
    memset(&r, 0, sizeof r);
    r.d = d;
    r.pp_time_ms = r.allreduce_time_ms = r.total_time_ms = INFINITY;
    plan_t plan;
    if (build_plan(topo, sc, d, &plan)) {
      for (int s = 0; s < plan.S; ++s) r.partitions[plan.stage_dc[s]] += 1;
      tasks_t t = {0, 0, 0};
      int64_t ms = 0;
      make_schedule(topo, sc, &plan, d, &t, &ms);
      r.makespan_ns = ms;
      r.pp_time_ms = ns_to_ms(ms);
      r.utilization = ms > 0 ? utilization_of(t.v, t.n, ms) : 0.0;
      free(t.v);
      /* per-stage worst all-reduce (dc_select.cpp:46-60) */
      const int n = d * sc->pipelines_per_cell;
      double worst = 0.0;
      for (int s = 0; s < plan.S; ++s) {
        int begin = s * sc->layers_per_partition;
        int end = begin + sc->layers_per_partition < sc->num_layers
                      ? begin + sc->layers_per_partition
                      : sc->num_layers;
        int layers = end - begin > 0 ? end - begin : 0;
        double params = effective_params_per_layer(sc) * layers;
        double v = allreduce_time_ms(params, n, topo->intra_bw[plan.stage_dc[s]]);
        if (worst < v) worst = v;
      }
      r.allreduce_time_ms = worst;
      r.total_time_ms = r.pp_time_ms + r.allreduce_time_ms;
      r.throughput = (double)d * sc->pipelines_per_cell / r.total_time_ms;
      r.feasible = 1;
      plan_free(&plan);
      if (chosen == 0 || r.throughput > chosen_thr) { /* :110-116 */
        chosen = d;
        chosen_thr = r.throughput;
      }
    }
    if (d - 1 < cap) rows[d - 1] = r;
  }
  for (int d = 1; d <= d_max && d - 1 < cap; ++d) rows[d - 1].chosen = d == chosen;
  *chosen_d = chosen;
  *gpus_used = chosen > 0 ? (long long)chosen * sc->pipelines_per_cell *
                                partition_count(sc) * sc->tp_degree
                          : 0;
  return g_rc;
}

static int timeline(const gpb_topology* topos, const gpb_scenario* sc, int d,
                    plan_t* plan, tasks_t* t, int64_t* ms) {
  if (validate(topos, sc) != GPB_OK) return g_rc;
  const gpb_topology* topo = &topos[sc->topology];
  if (!build_plan(topo, sc, d, plan)) {
    fail(GPB_INFEASIBLE, "plan needs more GPUs than the topology");
    return g_rc;
  }
  return make_schedule(topo, sc, plan, d, t, ms);
}

int orc_timeline(const gpb_topology* topos, const gpb_scenario* sc, int32_t d,
                 orc_task* out, int64_t cap, int64_t* n, int64_t* makespan) {
  reset_err();
  plan_t plan;
  memset(&plan, 0, sizeof plan);
  tasks_t t = {0, 0, 0};
  if (timeline(topos, sc, d, &plan, &t, makespan) == GPB_OK) {
    *n = t.n;
    for (int64_t i = 0; i < t.n && i < cap; ++i) out[i] = t.v[i];
  }
  free(t.v);
  plan_free(&plan);
  return g_rc;
}

/* ----------------------------------------------------------- bubbletea */

typedef struct {
  int64_t lo, hi;
  int training;
} span_t;

typedef struct {
  span_t* v;
  int n, cap;
} spans_t;

typedef struct {
  int64_t lo, hi;
  int before_training;
} gap_t;

static void spans_insert(spans_t* sp, int at, span_t s) {
  if (sp->n == sp->cap) {
    sp->cap = sp->cap ? 2 * sp->cap : 16;
    sp->v = realloc(sp->v, sizeof(span_t) * sp->cap);
  }
  memmove(sp->v + at + 1, sp->v + at, sizeof(span_t) * (sp->n - at));
  sp->v[at] = s;
  sp->n++;
}

/* busy_by_gpu (bubbletea.cpp:20-37): GPUs indexed 0..n_gpu-1 by id. */
static spans_t* busy_by_gpu(const orc_task* tasks, int64_t n, int64_t horizon,
                            int n_gpu) {
  spans_t* busy = xcalloc(n_gpu, sizeof(spans_t));
  orc_task* v = xcalloc(n, sizeof(orc_task));
  memcpy(v, tasks, sizeof(orc_task) * n);
  qsort(v, n, sizeof(orc_task), gpu_cmp);
  for (int64_t i = 0; i < n; ++i) {
    int64_t lo = v[i].start > 0 ? v[i].start : 0;
    int64_t hi = v[i].end < horizon ? v[i].end : horizon;
    if (lo >= hi) continue;
    span_t s = {lo, hi, v[i].kind != K_PRE};
    spans_insert(&busy[v[i].gpu], busy[v[i].gpu].n, s);
  }
  free(v);
  return busy;
}

/* gaps_of (bubbletea.cpp:43-53); returns the gap count. */
static int gaps_of(const spans_t* sp, int64_t horizon, gap_t* out) {
  int n = 0;
  int64_t cursor = 0;
  for (int i = 0; i < sp->n; ++i) {
    if (sp->v[i].lo > cursor) {
      out[n].lo = cursor;
      out[n].hi = sp->v[i].lo;
      out[n].before_training = sp->v[i].training;
      ++n;
    }
    if (sp->v[i].hi > cursor) cursor = sp->v[i].hi;
  }
  if (cursor < horizon) {
    out[n].lo = cursor;
    out[n].hi = horizon;
    out[n].before_training = 0;
    ++n;
  }
  return n;
}

static int max_gpu_id(const orc_task* t, int64_t n) {
  int m = -1;
  for (int64_t i = 0; i < n; ++i)
    if (t[i].gpu > m) m = t[i].gpu;
  return m;
}

int orc_bubbles(const gpb_topology* topos, const gpb_scenario* sc, int32_t d,
                int64_t horizon, gpb_bubble* out, int64_t cap, int64_t* n_out) {
  reset_err();
  plan_t plan;
  memset(&plan, 0, sizeof plan);
  tasks_t t = {0, 0, 0};
  int64_t ms = 0;
  if (timeline(topos, sc, d, &plan, &t, &ms) == GPB_OK) {
    int64_t h = horizon > 0 ? horizon : ms;
    if (h <= 0) {
      fail(GPB_CONFIG_ERROR, "horizon: must be positive");
    } else {
      int n_gpu = max_gpu_id(t.v, t.n) + 1;
      spans_t* busy = busy_by_gpu(t.v, t.n, h, n_gpu);
      int64_t k = 0;
      for (int gpu = 0; gpu < n_gpu; ++gpu) {
        if (busy[gpu].n == 0) continue; /* only GPUs present in the map */
        gap_t* gaps = xcalloc(busy[gpu].n + 1, sizeof(gap_t));
        int ng = gaps_of(&busy[gpu], h, gaps);
        for (int i = 0; i < ng; ++i, ++k) {
          if (k < cap) {
            out[k].gpu_id = gpu;
            out[k].pad_ = 0;
            out[k].start_ns = gaps[i].lo;
            out[k].end_ns = gaps[i].hi;
          }
        }
        free(gaps);
        free(busy[gpu].v);
      }
      free(busy);
      *n_out = k;
    }
  }
  free(t.v);
  plan_free(&plan);
  return g_rc;
}

/* build_prefill_pipelines (bubbletea.cpp:88-130): pipeline pi = pipe*S+stage,
 * stage k of it = cell k's GPU. Returns layers per cell in `layers`. */
static int prefill_layers(const gpb_prefill_model* pm, int D, int* layers) {
  int base = pm->inference_layers / D, extra = pm->inference_layers % D;
  long long worst = 0;
  for (int c = 0; c < D; ++c) {
    layers[c] = base + (c < extra ? 1 : 0);
    if (layers[c] > worst) worst = layers[c];
  }
  double ppl = pm->inference_params_per_layer > 0
                   ? pm->inference_params_per_layer
                   : 12.0 * (double)pm->inference_hidden * (double)pm->inference_hidden;
  long long mem = (long long)((double)worst * ppl * pm->bytes_per_element);
  if (mem > pm->memory_budget_bytes) {
    fail(GPB_CONFIG_ERROR, "prefill.memory_budget_bytes: inference model needs %lld bytes per stage, over the budget of %lld",
         mem, (long long)pm->memory_budget_bytes);
    return 0;
  }
  return 1;
}

static uint64_t fnv_mix(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xffu;
    h *= 1099511628211ull;
  }
  return h;
}

static int i64_cmp(const void* a_, const void* b_) {
  int64_t a = *(const int64_t*)a_, b = *(const int64_t*)b_;
  return a < b ? -1 : (a > b ? 1 : 0);
}

int orc_pack_prefills(const gpb_topology* topos, const gpb_scenario* sc,
                      int32_t d, const gpb_request* reqs, int64_t n_req,
                      const gpb_prefill_model* pm, int64_t horizon,
                      gpb_pack_summary* sum, gpb_placement* pl) {
  reset_err();
  plan_t plan;
  memset(&plan, 0, sizeof plan);
  tasks_t t = {0, 0, 0};
  int64_t ms = 0;
  if (timeline(topos, sc, d, &plan, &t, &ms) != GPB_OK) goto out;
  const int64_t h = horizon > 0 ? horizon : ms;
  if (h <= 0) {
    fail(GPB_CONFIG_ERROR, "horizon: must be positive");
    goto out;
  }
  const int D = plan.D, C = plan.C, S = plan.S;
  int* layers = xcalloc(D, sizeof(int));
  if (!prefill_layers(pm, D, layers)) {
    free(layers);
    goto out;
  }
  int total_layers = 0;
  for (int c = 0; c < D; ++c) total_layers += layers[c];
  const int n_gpu = max_gpu_id(t.v, t.n) + 1;
  spans_t* busy = busy_by_gpu(t.v, t.n, h, n_gpu);
  const int64_t guard = ms_to_ns(pm->guard_ms);
  int64_t* dur = xcalloc(D, sizeof(int64_t));
  int64_t* off = xcalloc(D, sizeof(int64_t));
  gap_t** stage_gaps = xcalloc(D, sizeof(gap_t*));
  int* stage_ng = xcalloc(D, sizeof(int));
  int64_t accepted = 0, rejected = 0;
  uint64_t hash = 1469598103934665603ull;
  /* prefill busy per GPU for the after-utilization */
  for (int64_t r = 0; r < n_req && g_rc == GPB_OK; ++r) {
    const gpb_request* req = &reqs[r];
    if (req->tokens < 1 || req->tokens > pm->max_tokens) { /* :68-76 */
      fail(GPB_CONFIG_ERROR, "request.tokens: must be in [1, %d]", pm->max_tokens);
      break;
    }
    const double dur_ms = pm->saturation_ms * (double)req->tokens / (double)pm->max_tokens;
    const double bytes = (double)(1LL * req->tokens * pm->inference_hidden * pm->bytes_per_element);
    if (pm->stage_bw <= 0) {
      fail(GPB_ERROR, "bandwidth must be positive");
      break;
    }
    const double xfer = pm->boundary_latency_ms + bytes / pm->stage_bw; /* :33-36 */
    int placed = 0;
    for (int pi = 0; pi < C * S && !placed; ++pi) {
      const int pipe = pi / S, stage = pi % S;
      const int64_t ovh = ms_to_ns(1 * xfer); /* prefill_pp_overhead_ms(act, 1) */
      int64_t cursor = 0;
      for (int k = 0; k < D; ++k) {
        dur[k] = ms_to_ns(dur_ms * layers[k] / (double)(total_layers > 1 ? total_layers : 1));
        off[k] = cursor;
        cursor += dur[k] + ovh;
      }
      const int64_t arrival = ms_to_ns(req->arrival_ms);
      long ncand = 1;
      for (int k = 0; k < D; ++k) {
        int gpu = plan.gpu[((size_t)k * C + pipe) * S + stage];
        free(stage_gaps[k]);
        stage_gaps[k] = xcalloc(busy[gpu].n + 1, sizeof(gap_t));
        stage_ng[k] = gaps_of(&busy[gpu], h, stage_gaps[k]);
        ncand += stage_ng[k];
      }
      int64_t* cand = xcalloc(ncand, sizeof(int64_t));
      long nc = 0;
      cand[nc++] = arrival;
      for (int k = 0; k < D; ++k)
        for (int i = 0; i < stage_ng[k]; ++i)
          if (stage_gaps[k][i].lo - off[k] >= arrival) cand[nc++] = stage_gaps[k][i].lo - off[k];
      qsort(cand, nc, sizeof(int64_t), i64_cmp);
      for (long ci = 0; ci < nc; ++ci) {
        if (ci > 0 && cand[ci] == cand[ci - 1]) continue; /* std::set */
        const int64_t t0 = cand[ci];
        int ok = 1;
        for (int k = 0; k < D && ok; ++k) {
          const int64_t lo = t0 + off[k], hi = lo + dur[k];
          ok = 0;
          for (int i = 0; i < stage_ng[k]; ++i) {
            const gap_t* gp = &stage_gaps[k][i];
            if (gp->lo > lo) break;
            int64_t usable_end = gp->hi - (gp->before_training ? guard : 0);
            if (lo >= gp->lo && hi <= usable_end) {
              ok = 1;
              break;
            }
          }
        }
        if (!ok) continue;
        for (int k = 0; k < D; ++k) { /* commit (:189-215) */
          const int64_t lo = t0 + off[k], hi = lo + dur[k];
          int gpu = plan.gpu[((size_t)k * C + pipe) * S + stage];
          push_task(&t, gpu, k, pi, K_PRE, req->id, k, lo, hi);
          spans_t* sp = &busy[gpu];
          int at = 0; /* upper_bound by start */
          while (at < sp->n && !(lo < sp->v[at].lo)) ++at;
          span_t nsp = {lo, hi, 0};
          spans_insert(sp, at, nsp);
        }
        double ttft = D - 1 == 0 ? 0.0 : (D - 1) * xfer;
        if (pl) {
          pl[r].start_ns = t0;
          pl[r].ttft_overhead_ms = ttft;
          pl[r].accepted = 1;
          pl[r].pipeline = pi;
        }
        hash = fnv_mix(hash, (uint64_t)(int64_t)req->id);
        hash = fnv_mix(hash, (uint64_t)(int64_t)pi);
        hash = fnv_mix(hash, (uint64_t)t0);
        placed = 1;
        break;
      }
      free(cand);
    }
    if (placed) {
      ++accepted;
    } else {
      ++rejected;
      if (pl) {
        pl[r].start_ns = -1;
        pl[r].ttft_overhead_ms = 0;
        pl[r].accepted = 0;
        pl[r].pipeline = -1;
      }
    }
  }
  if (g_rc == GPB_OK) {
    /* training tasks are the first n_train entries; utilization over both */
    int64_t n_train = t.n - accepted * D;
    sum->utilization_before = utilization_of(t.v, n_train, h);
    sum->utilization_after = utilization_of(t.v, t.n, h);
    sum->accepted = accepted;
    sum->rejected = rejected;
    sum->horizon_ns = h;
    sum->placement_hash = hash;
  }
  for (int k = 0; k < D; ++k) free(stage_gaps[k]);
  for (int gpu = 0; gpu < n_gpu; ++gpu) free(busy[gpu].v);
  free(busy);
  free(stage_gaps);
  free(stage_ng);
  free(dur);
  free(off);
  free(layers);
out:
  free(t.v);
  plan_free(&plan);
  return g_rc;
}

/* saturating_requests (bubbletea.cpp:240-267) */
int orc_saturating_requests(const gpb_topology* topos, const gpb_scenario* sc,
                            int32_t d, const gpb_prefill_model* pm,
                            int64_t horizon, gpb_request* out, int64_t cap,
                            int64_t* n_out) {
  reset_err();
  plan_t plan;
  memset(&plan, 0, sizeof plan);
  tasks_t t = {0, 0, 0};
  int64_t ms = 0;
  if (timeline(topos, sc, d, &plan, &t, &ms) != GPB_OK) goto out;
  const int64_t h = horizon > 0 ? horizon : ms;
  int* layers = xcalloc(plan.D, sizeof(int));
  if (!prefill_layers(pm, plan.D, layers)) {
    free(layers);
    goto out;
  }
  free(layers);
  const int n_gpu = max_gpu_id(t.v, t.n) + 1;
  spans_t* busy = busy_by_gpu(t.v, t.n, h, n_gpu);
  int64_t n = 0;
  int next_id = 0;
  for (int pi = 0; pi < plan.C * plan.S; ++pi) {
    const int pipe = pi / plan.S, stage = pi % plan.S;
    int gpu = plan.gpu[((size_t)0 * plan.C + pipe) * plan.S + stage];
    gap_t* gaps = xcalloc(busy[gpu].n + 1, sizeof(gap_t));
    int ng = gaps_of(&busy[gpu], h, gaps);
    for (int i = 0; i < ng; ++i) {
      int64_t cursor = gaps[i].lo;
      while (cursor < gaps[i].hi) {
        double gap_ms = ns_to_ms(gaps[i].hi - cursor);
        int tokens = (int)(gap_ms * pm->max_tokens / pm->saturation_ms);
        if (tokens > pm->max_tokens) tokens = pm->max_tokens;
        while (tokens >= 1 &&
               cursor + ms_to_ns(pm->saturation_ms * (double)tokens / (double)pm->max_tokens) > gaps[i].hi)
          tokens -= 1;
        if (tokens < 1) break;
        if (n < cap) {
          out[n].id = next_id;
          out[n].tokens = tokens;
          out[n].arrival_ms = ns_to_ms(cursor);
        }
        ++n;
        ++next_id;
        cursor += ms_to_ns(pm->saturation_ms * (double)tokens / (double)pm->max_tokens);
      }
    }
    free(gaps);
  }
  for (int gpu = 0; gpu < n_gpu; ++gpu) free(busy[gpu].v);
  free(busy);
  *n_out = n;
out:
  free(t.v);
  plan_free(&plan);
  return g_rc;
}
