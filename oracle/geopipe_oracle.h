/* geopipe_oracle.h — TEST INFRASTRUCTURE ONLY: the CPU oracle (checker).
 *
 * A plain-C restatement of the reference's plan-evaluation hot path
 * (/root/reference/proj/src). Each function cites the reference lines it
 * follows. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load liboracle.so; the product (libgeopipe_b200.so) never does.
 *
 * Pinned by: the reference's golden vectors (test_scheduler.cpp:53-258,
 * test_engine.cpp:87-99, test_comm_model.cpp:24-115, acceptance.cpp) in
 * tests/test_oracle_kat.py, and by differential runs against the compiled
 * reference (oracle/_ref/libgeopipe_ref.so) in tests/test_oracle_vs_ref.py,
 * whose outputs are also frozen into tests/golden/ for the GPU box.
 */
#ifndef GEOPIPE_ORACLE_H_
#define GEOPIPE_ORACLE_H_

#include <stdint.h>

#include "../include/geopipe_batch.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Task record; kind follows TaskKind (schedule.h:10):
 * 0 Forward, 1 Backward, 2 Recompute, 3 AllReduce, 4 Prefill. */
typedef struct orc_task {
  int32_t gpu, cell, pipeline, kind, microbatch, stage;
  int64_t start, end;
} orc_task;

const char* orc_last_error(void);

double orc_single_tcp_bandwidth(const gpb_topology* topo, double latency_ms);

/* select() for one scenario (dc_select.cpp:99-123), rows extended with
 * makespan_ns and the report() utilization of each feasible row's timeline. */
int orc_select(const gpb_topology* topos, const gpb_scenario* sc, gpb_row* rows,
               int32_t cap, int32_t* n_rows, int32_t* chosen_d,
               int64_t* gpus_used);

/* Full iteration timeline of one (scenario, D) row: all D cells, sorted by
 * finalize_schedule's key (schedule.cpp:23-45). Replay-equivalent (see
 * DESIGN.md "replay"). */
int orc_timeline(const gpb_topology* topos, const gpb_scenario* sc, int32_t d,
                 orc_task* out, int64_t cap, int64_t* n, int64_t* makespan);

/* extract_bubbles over that timeline (bubbletea.cpp:56-66). */
int orc_bubbles(const gpb_topology* topos, const gpb_scenario* sc, int32_t d,
                int64_t horizon, gpb_bubble* out, int64_t cap, int64_t* n);

/* schedule_prefills over that timeline (bubbletea.cpp:132-222). */
int orc_pack_prefills(const gpb_topology* topos, const gpb_scenario* sc,
                      int32_t d, const gpb_request* reqs, int64_t n_req,
                      const gpb_prefill_model* pm, int64_t horizon,
                      gpb_pack_summary* sum, gpb_placement* pl);

/* saturating_requests (bubbletea.cpp:240-267). */
int orc_saturating_requests(const gpb_topology* topos, const gpb_scenario* sc,
                            int32_t d, const gpb_prefill_model* pm,
                            int64_t horizon, gpb_request* out, int64_t cap,
                            int64_t* n);

#ifdef __cplusplus
}
#endif

#endif
