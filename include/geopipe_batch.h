/* geopipe_batch.h — C ABI of the B200 plan-evaluation hot path.
 *
 * This is the thin, plain-pointer boundary between the host planner (C++,
 * libgeopipe_b200.so) and the sm_100a kernels. It batches what the reference
 * evaluates one call at a time:
 *
 *   reference (C++ API, /root/reference/proj/src)        this ABI
 *   ---------------------------------------------------   -----------------------------
 *   select(const SelectionInput&)  dc_select.h:57,        gpb_load + gpb_evaluate
 *     body dc_select.cpp:99-123 (D sweep, argmax)           (+ gpb_fetch_rows / _scenarios)
 *   whatif(const std::vector<WhatIfScenario>&)            same, many scenarios per call
 *     dc_select.h:72, body dc_select.cpp:125-134
 *   evaluate_d (dc_select.cpp:27-66)                      one gpb_row
 *   schedule_for_policy (scheduler.h:56-61) makespan      gpb_row.makespan_ns
 *   report()/utilization() (metrics.cpp:39-54,            gpb_row.utilization
 *     bubbletea.cpp:224-238)
 *   extract_bubbles (bubbletea.h:81, .cpp:43-66)          gpb_bubbles
 *   build_prefill_pipelines + schedule_prefills           gpb_pack_prefills
 *     (bubbletea.h:93-104, .cpp:88-222)
 *
 * The session-level C ABI of the reference (geopipe.h:26-60, 17 gp_*
 * functions) is kept verbatim in include/geopipe.h and is implemented on top
 * of this layer.
 *
 * Conventions (same as geopipe.h:19-22 / capi.cpp:19-39):
 *   return GPB_OK 0, GPB_ERROR 1 (internal / CUDA / I/O), GPB_CONFIG_ERROR 2
 *   (malformed input), GPB_INFEASIBLE 3; never throws across the ABI; the
 *   message of the last failing call is gpb_last_error(). Input buffers are
 *   borrowed for the duration of the call; output buffers are caller-owned.
 *   A context is bound to one CUDA device and is not thread-safe: use one
 *   context per thread (geopipe.h:9).
 *
 * Units: times are integer nanoseconds (base.h:13) or double milliseconds;
 * bandwidths are bytes/ms (base.h:23-24); byte counts are int64.
 */
#ifndef GEOPIPE_BATCH_H_
#define GEOPIPE_BATCH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPB_OK 0
#define GPB_ERROR 1
#define GPB_CONFIG_ERROR 2
#define GPB_INFEASIBLE 3

#define GPB_MAX_DC 8  /* datacenters per topology */
#define GPB_MAX_TCP 8 /* single-TCP calibration points (topology.h:18-22) */

/* Pipeline policies (scheduler.cpp:540-572). */
#define GPB_GPIPE 0
#define GPB_1F1B 1
#define GPB_VARUNA 2
#define GPB_ATLAS 3

/* ClusterTopology (topology.h:12-40), DCs in config order. */
typedef struct gpb_topology {
  int32_t n_dc;
  int32_t gpu_count[GPB_MAX_DC];
  double intra_bw[GPB_MAX_DC];                     /* bytes/ms */
  double latency_ms[GPB_MAX_DC][GPB_MAX_DC];       /* one-way, symmetric */
  double pair_bw_cap;                              /* bytes/ms */
  int32_t n_tcp;                                   /* 0 => Table 1 default */
  int32_t pad_;
  double tcp_latency_ms[GPB_MAX_TCP];
  double tcp_bw[GPB_MAX_TCP];                      /* bytes/ms */
} gpb_topology;

/* One selection problem = SelectionInput (dc_select.h:18-30) with its
 * ModelSpec (workload.h:12-33), ComputeProfile (workload.h:39-52) and
 * SchedulerOptions (scheduler.h:11-16) flattened. */
typedef struct gpb_scenario {
  int32_t topology;            /* index into the topology array */
  int32_t policy;              /* GPB_GPIPE .. GPB_ATLAS */
  int32_t num_layers;
  int32_t layers_per_partition;
  int32_t num_microbatches;    /* M */
  int32_t bytes_per_element;
  int64_t hidden;
  int64_t seq_len;
  int64_t microbatch;          /* sequences per microbatch (B) */
  double params_per_layer;     /* 0 => 12 H^2 */
  double fwd_ms, bwd_ms, recompute_ms;
  double ratio_C;              /* > 0 => ComputeProfile::from_ratio */
  int32_t pipelines_per_cell;  /* C */
  int32_t tp_degree;
  int32_t d_max;               /* 0 => total_gpus / (C * P * tp) */
  int32_t n_order;             /* 0 => default_dc_order */
  int32_t dc_order[GPB_MAX_DC];/* topology DC indices, walk order */
  int32_t recompute;
  int32_t multi_conn;
  int32_t n_connections;       /* used when multi_conn (default 32) */
  int32_t mem_limit;           /* ATLAS cap; 0 => number of stages */
} gpb_scenario;

/* SelectionRow (dc_select.h:32-40) + mean utilization of the iteration
 * timeline (metrics.cpp:39-54, horizon = makespan). */
typedef struct gpb_row {
  double pp_time_ms;           /* +inf when infeasible */
  double allreduce_time_ms;    /* +inf when infeasible */
  double total_time_ms;        /* +inf when infeasible */
  double throughput;           /* D*C/total; 0 when infeasible */
  double utilization;          /* 0 when infeasible */
  int64_t makespan_ns;         /* 0 when infeasible */
  int32_t scenario;
  int32_t d;
  int32_t feasible;
  int32_t chosen;              /* row.d == report.chosen_d */
  int16_t partitions[GPB_MAX_DC]; /* per topology DC: partitions hosted */
} gpb_row;

/* SelectionReport (dc_select.h:42-46) per scenario. */
typedef struct gpb_scenario_result {
  int64_t first_row;           /* index of D=1 row in the row table */
  int64_t gpus_used;
  int32_t n_rows;              /* d_max */
  int32_t chosen_d;            /* 0 when no feasible row */
} gpb_scenario_result;

/* Best plan of a batch: key = (throughput desc, row index asc). */
typedef struct gpb_best {
  double throughput;
  int64_t row;                 /* global row index, -1 when none */
} gpb_best;

/* Bubble (bubbletea.h:13-17). */
typedef struct gpb_bubble {
  int32_t gpu_id;
  int32_t pad_;
  int64_t start_ns;
  int64_t end_ns;
} gpb_bubble;

/* PrefillRequest (bubbletea.h:19-24), model_id implied "default". */
typedef struct gpb_request {
  int32_t id;
  int32_t tokens;
  double arrival_ms;
} gpb_request;

/* PrefillModel (bubbletea.h:38-58). */
typedef struct gpb_prefill_model {
  double saturation_ms;        /* 300 */
  int32_t max_tokens;          /* 8192 */
  int32_t inference_layers;    /* 8 */
  double stage_bw;             /* bytes/ms, 25e6 */
  double boundary_latency_ms;  /* 0 */
  double guard_ms;             /* 0 */
  int64_t memory_budget_bytes; /* 1 GiB */
  int64_t inference_hidden;    /* 1024 */
  double inference_params_per_layer; /* 0 => 12 H^2 */
  int32_t bytes_per_element;   /* 2 */
  int32_t pad_;
} gpb_prefill_model;

/* One request's outcome (PrefillPlacement / PrefillRejection,
 * bubbletea.h:60-71). */
typedef struct gpb_placement {
  int64_t start_ns;            /* stage-0 start; -1 when rejected */
  double ttft_overhead_ms;
  int32_t accepted;
  int32_t pipeline;            /* (pipe * S + stage), -1 when rejected */
} gpb_placement;

/* Per-plan packing summary (bubbletea_metrics_csv, export.cpp:264-274). */
typedef struct gpb_pack_summary {
  double utilization_before;
  double utilization_after;
  int64_t accepted;
  int64_t rejected;
  int64_t horizon_ns;
  uint64_t placement_hash;     /* FNV-1a over (id, pipeline, start_ns) of accepted */
} gpb_pack_summary;

typedef struct gpb_ctx gpb_ctx;

/* Context bound to CUDA device `device` (one per thread). NULL on failure. */
gpb_ctx* gpb_create(int device);
void gpb_destroy(gpb_ctx* ctx);
const char* gpb_last_error(gpb_ctx* ctx);

/* Host-side comm model: single_tcp_bandwidth (comm_model.cpp:8-25) with the
 * host libm, exposed for tests. */
double gpb_single_tcp_bandwidth(const gpb_topology* topo, double latency_ms);

/* Validate and upload a plan space: every scenario expands into its D rows
 * (D = 1..d_max; dc_select.cpp:99-104). Inputs are host pointers, copied to
 * HBM with one H2D per table. *n_rows receives the total row count. */
int gpb_load(gpb_ctx* ctx, const gpb_topology* topos, int32_t n_topo,
             const gpb_scenario* scens, int32_t n_scen, int64_t* n_rows);

/* Evaluate every loaded row on the device and select per scenario and
 * globally. Asynchronous on the context stream unless `sync` is nonzero. */
int gpb_evaluate(gpb_ctx* ctx, int32_t sync);

/* Copy results back (synchronizes). NULL outputs are skipped. */
int gpb_fetch_rows(gpb_ctx* ctx, gpb_row* rows, int64_t n_rows);
int gpb_fetch_scenarios(gpb_ctx* ctx, gpb_scenario_result* out, int32_t n_scen);
int gpb_fetch_best(gpb_ctx* ctx, gpb_best* out);

/* Launch on an external stream (e.g. the caller's framework stream);
 * NULL restores the context's own stream. */
int gpb_set_stream(gpb_ctx* ctx, void* cuda_stream);

/* Device address of the batch's gpb_best record (for an NCCL all-gather of
 * per-GPU winners). */
void* gpb_device_best(gpb_ctx* ctx);

/* Asynchronous device-to-device copy of the gpb_best record (16 bytes) to
 * `dst` on the launch stream (feeds an NCCL all-gather without a host
 * round trip). */
int gpb_copy_best(gpb_ctx* ctx, void* dst);

/* Bubbles of one row's iteration timeline (run(), engine.cpp:452-460) over
 * [0, horizon_ns) (horizon_ns <= 0 => makespan), sorted (gpu, start) like
 * extract_bubbles (bubbletea.cpp:56-66). Writes at most `cap` entries;
 * *n_out receives the full count. */
int gpb_bubbles(gpb_ctx* ctx, int64_t row, int64_t horizon_ns,
                gpb_bubble* out, int64_t cap, int64_t* n_out);

/* Raw iteration timeline of one row's cell 0 (all D cells are identical):
 * forward end times and pair (recompute+backward) start times, laid out
 * [pipeline][stage][microbatch] with Ce = C pipelines for atlas and 1
 * otherwise (spatial policies schedule every pipeline identically).
 * dims receives {Ce, S, M, D}; arrays are written when cap >= Ce*S*M. */
int gpb_timeline_arrays(gpb_ctx* ctx, int64_t row, int64_t* fe, int64_t* ps,
                        int64_t cap, int32_t* dims, int64_t* makespan);

/* BubbleTea: pack one request trace (sorted by arrival, FCFS) into the
 * bubbles of each listed row, independently per row (schedule_prefills,
 * bubbletea.cpp:132-222). horizon_ns <= 0 => each row's makespan.
 * `placements` (nullable) receives n_rows_sel x n_req entries, row-major. */
int gpb_pack_prefills(gpb_ctx* ctx, const int64_t* rows, int32_t n_rows_sel,
                      const gpb_request* reqs, int64_t n_req,
                      const gpb_prefill_model* pm, int64_t horizon_ns,
                      gpb_pack_summary* summaries, gpb_placement* placements);

/* Include each stage's all-reduce tail (append_allreduce,
 * scheduler.cpp:613-650; the simulate.allreduce option) in the timelines
 * behind gpb_bubbles and gpb_pack_prefills. Default off. */
int gpb_set_allreduce_tail(gpb_ctx* ctx, int32_t enable);

/* saturating_requests (bubbletea.cpp:240-267) on the device: every prefill
 * pipeline's head GPU's bubbles of one row's timeline (horizon_ns <= 0 =>
 * makespan) filled with back-to-back requests of the largest fitting token
 * count, in build_prefill_pipelines order. Writes the requests when
 * cap >= *n_out (the full count). */
int gpb_saturating_requests(gpb_ctx* ctx, int64_t row, const gpb_prefill_model* pm,
                            int64_t horizon_ns, gpb_request* out, int64_t cap,
                            int64_t* n_out);

/* On-device structural check of one row's iteration timeline (cell 0), the
 * reference's validate_timeline (tests/support/validate.h:77-256): *check =
 * 0 valid, 1 incomplete, 2 overlapping tasks on a GPU, 3 overlapping
 * transfers on a link lane, 4 forward before its activation arrives, 5
 * recompute/backward before its gradient (or forward) arrives, 6 makespan
 * is not the last task end; *where = (pipeline << 48 | stage << 32 |
 * microbatch) of the first failure. fe / ps (nullable) replace the device's
 * own timeline with caller arrays in gpb_timeline_arrays' layout. */
int gpb_validate_timeline(gpb_ctx* ctx, int64_t row, const int64_t* fe, const int64_t* ps,
                          int32_t* check, int64_t* where);

/* append_allreduce (scheduler.cpp:613-650) of one row computed on the device:
 * per stage s < *n_stages, the start (last backward end over every replica)
 * and duration of its all-reduce task; written when cap >= *n_stages. */
int gpb_allreduce_tail(gpb_ctx* ctx, int64_t row, int64_t* start_ns, int64_t* dur_ns,
                       int32_t cap, int32_t* n_stages);

/* Deterministic request sources on the host (bubbletea.cpp:269-284). */
int gpb_synthetic_requests(int32_t count, uint32_t seed, double horizon_ms,
                           const gpb_prefill_model* pm, gpb_request* out);

/* Device time of the last gpb_evaluate / gpb_pack_prefills, per kernel
 * family, from CUDA events on the context stream (ms). */
typedef struct gpb_timing {
  float evaluate_ms;           /* whole gpb_evaluate launch sequence */
  float timing_kernels_ms;     /* schedule-timing kernels only */
  float select_ms;             /* selection kernels */
  float pack_ms;               /* last gpb_pack_prefills */
  float policy_ms[4];          /* timing kernels per policy (GPB_GPIPE..) */
  int32_t launches;            /* kernels launched by the last call */
  int32_t pad_;
  int64_t h2d_bytes;           /* bytes uploaded by the last gpb_load */
  int64_t d2h_bytes;           /* bytes fetched since the last gpb_load */
} gpb_timing;
int gpb_get_timing(gpb_ctx* ctx, gpb_timing* out);

/* On-device issue-rate microbenchmark used as the roofline denominator:
 * max-plus ops (one max or one add = 1 op) in independent register chains
 * over every SM; kind 0 = int64 (the kernels' representation), 1 = FP64
 * holding exact integers (DADD/DMNMX), 2 = int32. Returns Gop/s. */
int gpb_microbench(gpb_ctx* ctx, int32_t kind, double* gops);

/* Per-bucket timing events in gpb_evaluate (default on: gpb_get_timing's
 * policy_ms and gpb_bucket_infos' times need them; off saves ~2 event
 * records per bucket of host launch time). */
int gpb_set_bucket_timing(gpb_ctx* ctx, int32_t enable);

/* Profiling: record each row's clock64 cost in the evaluation kernels. */
int gpb_set_profile(gpb_ctx* ctx, int32_t enable);
int gpb_fetch_row_cycles(gpb_ctx* ctx, int64_t* out, int64_t n);

/* Profiling: the last gpb_evaluate's row buckets (one kernel launch each, on
 * concurrent streams) with their shapes and device times. Writes
 * min(n, cap) records; *n = number of buckets. */
typedef struct gpb_bucket_info {
  int32_t policy, B, rows, max_s, max_c, max_m, stream, pad_;
  float start_ms;              /* launch-stream fork -> bucket start */
  float ms;                    /* bucket kernel duration */
  double algo_ops;             /* algorithmic max-plus ops of its feasible rows */
} gpb_bucket_info;
int gpb_bucket_infos(gpb_ctx* ctx, gpb_bucket_info* out, int32_t cap, int32_t* n);

/* ---------------------------------------------------------------------
 * One plan space over several GPUs of one box (the batch
 * behind whatif(), dc_select.cpp:125-134, as run_whatif calls it,
 * runner.cpp:112-122). Whole scenarios are dealt to the devices by estimated
 * cost (longest first onto the least-loaded device); each device's context
 * is driven from its own host thread; the per-device winners (16 bytes) are
 * exchanged with one ncclAllGather over NVLink (NCCL opened at run time).
 * Rows, scenario results and the winner come back in the order of the whole
 * space and equal a single-device evaluation bit for bit.
 * --------------------------------------------------------------------- */
typedef struct gpb_group gpb_group;

/* Contexts on `devices[0..n_dev)` (n_dev <= 0: every visible device). A
 * device listed twice gets two contexts (the winners then go through the
 * host instead of NCCL). NULL on failure. */
gpb_group* gpb_group_create(int32_t n_dev, const int32_t* devices);
void gpb_group_destroy(gpb_group* g);
const char* gpb_group_last_error(gpb_group* g);
int32_t gpb_group_size(gpb_group* g);
int gpb_group_load(gpb_group* g, const gpb_topology* topos, int32_t n_topo,
                   const gpb_scenario* scens, int32_t n_scen, int64_t* n_rows);
/* Evaluate every shard and all-gather the per-device winners (async). */
int gpb_group_evaluate(gpb_group* g);
int gpb_group_fetch_rows(gpb_group* g, gpb_row* rows, int64_t n_rows);
int gpb_group_fetch_scenarios(gpb_group* g, gpb_scenario_result* out, int32_t n_scen);
int gpb_group_fetch_best(gpb_group* g, gpb_best* out);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* GEOPIPE_BATCH_H_ */
