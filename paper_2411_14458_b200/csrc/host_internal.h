// host_internal.h — the batch context behind the opaque gpb_ctx handle.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/geopipe_batch.h"
#include "atlas_layout.h"
#include "device_common.cuh"

namespace gpb {

struct Buf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

// The device exposes CUDA_DEVICE_MAX_CONNECTIONS (default 8) hardware work
// queues; more streams alias onto them and serialize unrelated buckets.
constexpr size_t kSideStreams = 8;

struct Bucket {
  int policy = 0;
  int B = 1;            // stages per lane = ceil(S / 32)
  int32_t offset = 0;   // into the work list
  int32_t count = 0;
  int max_m = 0;
  int max_cs = 0;
  int max_cm = 0;
  long long max_csm = 0;
  int max_c = 0, max_s = 0, max_nw = 0;
  long long max_slice = 0;  // atlas_seq buckets: per-thread scratch slice (int64)
  double est = 0;   // estimated bucket makespan (same units as cost)
  double cost = 0;  // estimated cost of the bucket's heaviest row
  int stream = 0;   // side stream it ran on
  bool heavy = false;  // ATLAS rows near the heaviest estimate (launched first)
  int gw = 32;         // flush rows per warp = 32 / gw (flush_group_kernel when < 32)
  // its scenarios (every row of a scenario lands in one bucket): selected on
  // the bucket's stream as soon as its kernel ends
  int32_t scen_off = 0, scen_cnt = 0;
  int32_t sel_grid = 0, sel_off = 0;  // select blocks and their block_best slots
};

// Launch shape of one ATLAS kernel (evaluation or timeline variant) over
// `count` rows whose largest C, S, M, WAN count and C*S*M are given.
struct AtlasPlan {
  AtlasLayout L;
  int wpc = 0, grid = 0;
  long long scratch_per_warp = 0;  // int64 per warp of global scratch: queues + lists
  long long scratch_big_off = 0;   // int64 offset of the lists (when not in shared memory)
};
struct Ctx {
  int device = 0;
  int num_sms = 148;
  int smem_optin = 227 * 1024;
  cudaStream_t stream = nullptr;     // active launch stream
  cudaStream_t own_stream = nullptr; // the context's own stream
  int64_t d2h_bytes = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  cudaEvent_t pack_ev0 = nullptr, pack_ev1 = nullptr;  // gpb_pack_prefills / microbench
  cudaEvent_t switch_ev = nullptr;                     // gpb_set_stream ordering
  std::string last_error;

  bool loaded = false;
  int64_t n_rows = 0;
  int32_t n_scen = 0, n_topo = 0;
  size_t h2d_bytes = 0;
  std::vector<Bucket> buckets;
  // host view of the loaded tables (in the pinned staging they were uploaded
  // from; valid until the next gpb_load)
  const DevScen* dev_scens_host = nullptr;
  const DevTopo* dev_topos_host = nullptr;
  std::vector<int32_t> bscen_host;  // bucket scenario lists (Bucket::scen_off / scen_cnt)
  // scenario of a row: the last scenario whose first row is <= row
  int32_t scen_of_row(int64_t row) const {
    int32_t lo = 0, hi = n_scen;  // first scenario with first_row > row
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (dev_scens_host[mid].first_row <= row) lo = mid + 1; else hi = mid;
    }
    return lo - 1;
  }

  // device tables
  Buf b_topos, b_scens, b_row_scen, b_work, b_rows, b_results, b_cursors, b_best, b_bscen;
  int32_t sel_blocks = 0;  // select blocks over all buckets
  // One-lane WAN drain greedy from this many stages up (measured: S = 80
  // rows 0.75 vs 0.80 ms, S = 16 rows 108 K vs 88 K drain cycles);
  // GPB_DRAIN_LANE overrides per evaluate, 0 = never.
  int32_t drain_lane = 32;
  // heavy ATLAS bucket's CTAs reserve a whole SM's shared memory (no other
  // bucket's CTAs with shared memory co-reside with the critical rows);
  // set per evaluate (GPB_HEAVY_EXCL, default on for small spaces)
  int32_t heavy_excl = 0;
  Buf b_scratch, b_cycles;
  bool profile_rows = false;
  // timeline / bubbletea buffers
  Buf b_tl_rows, b_tl_spans, b_tl_nspan, b_tl_scratch, b_gaps, b_ngaps, b_reqs, b_pl,
      b_sum, b_pack_scratch, b_pack_misc, b_sufmin, b_pack_stats, b_pack_memo;

  std::vector<cudaEvent_t> bucket_ev;      // [buckets + 1] bucket start (+ fork)
  std::vector<cudaEvent_t> bucket_ev_end;  // [buckets]
  std::vector<cudaStream_t> side;          // concurrent bucket streams
  std::vector<cudaEvent_t> side_done;
  Buf b_placements, b_ar;
  std::vector<long long> sufmin_host;  // pack: suffix-min arrivals (pinned by the call)
  std::vector<int32_t> pack_order;     // pack: CTA -> slot launch order
  std::vector<long long> pack_est;     // pack: per-slot cost estimate
  cudaStream_t pack_side = nullptr;    // pack: the heavy plans' launch
  cudaEvent_t pack_fork = nullptr, pack_join = nullptr;
  bool pack_allreduce = false;  // include the all-reduce tail in timelines
  bool pack_warm = false;       // pack kernels launched once (module loaded)
  // last build_timelines() outputs (device pointers into the buffers above)
  long long *tl_glo = nullptr, *tl_ghi = nullptr, *tl_gsum = nullptr, *tl_hz = nullptr;
  unsigned char* tl_gfl = nullptr;
  longlong2* tl_gpk = nullptr;  // packed copy of the gap lists (pack kernel)
  long long* tl_ar = nullptr;   // all-reduce tail: durations [n_ar], then starts [n_ar]
  int *tl_gcnt = nullptr, *tl_ghas = nullptr;
  void* tl_slots_dev = nullptr;
  bool timing_valid = false;
  bool bucket_timing = true;         // record per-bucket events in evaluate
  bool bucket_timing_valid = false;  // ... and the last evaluate did
  // evaluate launch sequence: prepared once per loaded space, replayed as a graph
  bool eval_ready = false;
  size_t n_side = 0;
  cudaEvent_t fork_ev = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t graph_stream = nullptr;
  std::vector<long long> graph_key;  // what the captured graph baked in
  void drop_graph();
  std::vector<AtlasPlan> aplan;  // per bucket (ATLAS only)
  std::vector<size_t> scr_off;    // per bucket offset into b_scratch (int64)
  int last_launches = 0;
  float pack_ms = 0.f;
  // pinned staging of the uploaded tables (async H2D; reused once the
  // previous upload has left it: upload_ev)
  void* stage = nullptr;  // row tables
  size_t stage_bytes = 0;
  void* stage_ts = nullptr;  // topology + scenario tables
  size_t stage_ts_bytes = 0;
  cudaEvent_t upload_ev = nullptr;
  bool upload_pending = false;

  std::vector<Buf*> all_bufs() {
    return {&b_topos, &b_scens, &b_row_scen, &b_work, &b_bscen, &b_rows, &b_results, &b_cursors,
            &b_best, &b_scratch, &b_cycles, &b_tl_rows, &b_tl_spans, &b_tl_nspan, &b_tl_scratch,
            &b_gaps, &b_ngaps, &b_reqs, &b_pl, &b_sum, &b_pack_scratch, &b_pack_misc, &b_sufmin, &b_pack_stats, &b_pack_memo,
            &b_placements, &b_ar};
  }

  void set_error(const char* fmt, ...);
  int cuda_fail(cudaError_t e, const char* what);
  void* dev_buf(Buf& b, size_t bytes);
  int check_error_flag();
  ~Ctx();
};

int plan_atlas(Ctx& c, int B, bool timeline, int C, int S, int M, int nw, long long max_csm,
               long long count, AtlasPlan& P);

int row_wan_boundaries(const Ctx& c, int64_t row);

// Validate + flatten a plan space on the host (multi-threaded for large
// spaces); row_scen (nullable) receives the row -> scenario table.
int flatten_space(const gpb_topology* topos, int32_t n_topo, const gpb_scenario* scens,
                  int32_t n_scen, DevTopo* dt, DevScen* ds, std::vector<int32_t>* row_scen,
                  int64_t& n_rows, std::string& err);

}  // namespace gpb
