// host.cu — host side of the batch C ABI (include/geopipe_batch.h).
//
// Validates and flattens plan spaces into HBM tables, buckets rows by
// (policy, stages-per-lane) so each kernel instantiation sees uniform
// register shapes, launches the evaluation/selection kernels on the
// context's stream and times them with CUDA events. Host-only arithmetic is
// limited to what the reference itself evaluates once per scenario with
// libm (single_tcp_bandwidth, comm_model.cpp:8-25) or exact basic operations
// (from_ratio, workload.cpp:21-33); every per-row quantity is computed on the
// device.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "../../include/geopipe_batch.h"
#include "device_common.cuh"
#include "host_internal.h"
#include "kernels.h"

using namespace gpb;

namespace {

const double kTcpLat[4] = {10.0, 20.0, 30.0, 40.0};
const double kTcpMbps[4] = {1220.0, 600.0, 396.0, 293.0};  // topology.cpp:45-52

struct ConfigErr {
  std::string msg;
};

}  // namespace

// single_tcp_bandwidth (comm_model.cpp:8-25), host libm.
extern "C" double gpb_single_tcp_bandwidth(const gpb_topology* t, double latency_ms) {
  double lat[GPB_MAX_TCP], bw[GPB_MAX_TCP];
  int n;
  if (t->n_tcp > 0) {
    n = t->n_tcp;
    for (int i = 0; i < n; ++i) {
      lat[i] = t->tcp_latency_ms[i];
      bw[i] = t->tcp_bw[i];
    }
  } else {
    n = 4;
    for (int i = 0; i < 4; ++i) {
      lat[i] = kTcpLat[i];
      bw[i] = kTcpMbps[i] * 125.0;  // mbps_to_bytes_per_ms (base.h:24)
    }
  }
  if (latency_ms <= lat[0]) return bw[0];
  if (latency_ms >= lat[n - 1]) return bw[n - 1] * lat[n - 1] / latency_ms;
  for (int i = 1; i < n; ++i) {
    if (latency_ms > lat[i]) continue;
    if (latency_ms == lat[i]) return bw[i];
    double f = (std::log(latency_ms) - std::log(lat[i - 1])) /
               (std::log(lat[i]) - std::log(lat[i - 1]));
    return std::exp(std::log(bw[i - 1]) + f * (std::log(bw[i]) - std::log(bw[i - 1])));
  }
  return bw[n - 1];
}

extern "C" double gpb_repeated_sum_host(double u, long long G) { return repeated_sum(u, G); }

namespace gpb {

void Ctx::set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  last_error = buf;
}

int Ctx::cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return GPB_ERROR;
}

void* Ctx::dev_buf(Buf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.bytes < bytes) {
    if (b.ptr) cudaFree(b.ptr);
    b.ptr = nullptr;
    b.bytes = 0;
    if (cudaMalloc(&b.ptr, bytes) != cudaSuccess) return nullptr;
    b.bytes = bytes;
  }
  return b.ptr;
}

Ctx::~Ctx() {
  for (Buf* b : all_bufs()) {
    if (b->ptr) cudaFree(b->ptr);
  }
  drop_graph();
  if (upload_ev) {
    cudaEventSynchronize(upload_ev);
    cudaEventDestroy(upload_ev);
  }
  if (stage) cudaFreeHost(stage);
  if (stage_ts) cudaFreeHost(stage_ts);
  if (pack_side) cudaStreamDestroy(pack_side);
  if (pack_fork) cudaEventDestroy(pack_fork);
  if (pack_join) cudaEventDestroy(pack_join);
  if (fork_ev) cudaEventDestroy(fork_ev);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (ev2) cudaEventDestroy(ev2);
  if (ev3) cudaEventDestroy(ev3);
  if (pack_ev0) cudaEventDestroy(pack_ev0);
  if (pack_ev1) cudaEventDestroy(pack_ev1);
  if (switch_ev) cudaEventDestroy(switch_ev);
  for (cudaEvent_t e : bucket_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : bucket_ev_end) cudaEventDestroy(e);
  for (cudaEvent_t e : side_done) cudaEventDestroy(e);
  for (cudaStream_t s2 : side) cudaStreamDestroy(s2);
  if (own_stream) cudaStreamDestroy(own_stream);
}

// ------------------------------------------------------------ validation

static void validate_topology(const gpb_topology& t, int idx) {
  const auto p = [idx] { return "topologies[" + std::to_string(idx) + "]"; };  // errors only
  if (t.n_dc < 1 || t.n_dc > GPB_MAX_DC)
    throw ConfigErr{p() + ".n_dc: must be in [1, 8]"};
  for (int i = 0; i < t.n_dc; ++i) {
    if (t.gpu_count[i] < 0) throw ConfigErr{p() + ".gpu_count: must be >= 0"};
    if (!(t.intra_bw[i] > 0)) throw ConfigErr{p() + ".intra_bw: must be > 0"};
    for (int j = 0; j < t.n_dc; ++j)
      if (!(t.latency_ms[i][j] >= 0))
        throw ConfigErr{p() + ".latency_ms: must be >= 0"};
  }
  if (!(t.pair_bw_cap > 0)) throw ConfigErr{p() + ".pair_bw_cap: must be > 0"};
  if (t.n_tcp < 0 || t.n_tcp > GPB_MAX_TCP)
    throw ConfigErr{p() + ".n_tcp: must be in [0, 8]"};
  for (int i = 0; i < t.n_tcp; ++i) {  // validate_tcp_table (topology.cpp:56-76)
    if (t.tcp_latency_ms[i] <= 0 || t.tcp_bw[i] <= 0)
      throw ConfigErr{"wan.tcp_table: latency and bandwidth must be positive"};
    if (i > 0 && t.tcp_latency_ms[i] <= t.tcp_latency_ms[i - 1])
      throw ConfigErr{"wan.tcp_table: latencies must be strictly increasing"};
    if (i > 0 && t.tcp_bw[i] >= t.tcp_bw[i - 1])
      throw ConfigErr{"wan.tcp_table: bandwidths must be strictly decreasing"};
  }
}

static std::string P_(int i) { return "scenarios[" + std::to_string(i) + "]"; }

static int64_t act_bytes(const gpb_scenario& s) {
  return s.microbatch * s.seq_len * s.hidden * (int64_t)s.bytes_per_element;
}

static void validate_scenario(const gpb_scenario& s, int idx, int n_topo,
                              const gpb_topology* topos) {
  const auto P = [idx] { return P_(idx); };  // built only for an error message
  if (s.topology < 0 || s.topology >= n_topo) throw ConfigErr{P() + ".topology: out of range"};
  const gpb_topology& t = topos[s.topology];
  if (s.policy < 0 || s.policy > 3)
    throw ConfigErr{"policy: must be one of gpipe, 1f1b, varuna, atlas"};
  if (s.pipelines_per_cell < 1) throw ConfigErr{"select.pipelines_per_cell: must be >= 1"};
  if (s.tp_degree < 1) throw ConfigErr{"select.tp_degree: must be >= 1"};
  if (s.num_layers < 1) throw ConfigErr{"model.num_layers: must be >= 1"};
  if (s.layers_per_partition < 1) throw ConfigErr{"model.layers_per_partition: must be >= 1"};
  if (s.num_microbatches < 1) throw ConfigErr{"model.num_microbatches: must be >= 1"};
  if (s.num_microbatches > 65535)
    throw ConfigErr{P() + ": more than 65535 microbatches is outside the kernel envelope"};
  if (s.bytes_per_element < 1 || s.hidden < 1 || s.seq_len < 1 || s.microbatch < 1)
    throw ConfigErr{"model: dimensions must be >= 1"};
  if (s.params_per_layer < 0) throw ConfigErr{"model.params_per_layer: must be >= 0"};
  if (s.ratio_C > 0) {
  } else if (s.ratio_C < 0) {
    throw ConfigErr{"compute.ratio_C: must be > 0"};
  } else if (!(s.fwd_ms > 0) || !(s.bwd_ms > 0) || s.recompute_ms < 0) {
    throw ConfigErr{"compute: durations must be positive"};  // workload.cpp:11-13
  }
  if (s.d_max < 0) throw ConfigErr{"select.d_max: must be >= 1"};
  if (s.n_order < 0 || s.n_order > GPB_MAX_DC) throw ConfigErr{P() + ".n_order: out of range"};
  unsigned seen = 0;
  for (int i = 0; i < s.n_order; ++i) {
    const int dc = s.dc_order[i];
    if (dc < 0 || dc >= t.n_dc) throw ConfigErr{"datacenters: unknown datacenter id"};
    if (seen & (1u << dc))
      throw ConfigErr{P() + ".dc_order: duplicate datacenter (unsupported, see DESIGN.md)"};
    seen |= 1u << dc;
  }
  if (s.mem_limit < 0) throw ConfigErr{"mem_limit: must be >= 1"};
  if (s.multi_conn && s.n_connections < 1)
    throw ConfigErr{"simulate.n_connections: must be >= 1"};
  const int S = (s.num_layers + s.layers_per_partition - 1) / s.layers_per_partition;
  if (S > 256)
    throw ConfigErr{P() + ": more than 256 pipeline stages is outside the kernel envelope"};
  if (act_bytes(s) <= 0) throw ConfigErr{"model: activation size overflow"};
}


// One scenario: validate (config.cpp / dc_select.cpp rules) and resolve it
// into its DevScen (profile, order, d_max). Throws ConfigErr.
static void flatten_scenario(const gpb_scenario& s, int i, int n_topo, const gpb_topology* topos,
                             DevScen& d) {
  validate_scenario(s, i, n_topo, topos);
  const gpb_topology& t = topos[s.topology];
  std::memset(&d, 0, sizeof d);
  d.topo = s.topology;
  d.policy = s.policy;
  d.S = (s.num_layers + s.layers_per_partition - 1) / s.layers_per_partition;
  d.M = s.num_microbatches;
  d.C = s.pipelines_per_cell;
  d.tp = s.tp_degree;
  d.L = s.num_layers;
  d.lpp = s.layers_per_partition;
  d.recompute = s.recompute ? 1 : 0;
  d.mem_limit = s.mem_limit > 0 ? s.mem_limit : d.S;  // scheduler.cpp:561
  d.n_conns = s.multi_conn ? s.n_connections : 1;
  d.bytes = act_bytes(s);
  d.ppl = s.params_per_layer > 0 ? s.params_per_layer
                                 : 12.0 * (double)s.hidden * (double)s.hidden;
  if (s.ratio_C > 0) {  // from_ratio (workload.cpp:21-33)
    const double comm_ms = (double)d.bytes / t.pair_bw_cap;
    d.fwd_ms = comm_ms / s.ratio_C;
    d.bwd_ms = 2.0 * d.fwd_ms;
    d.rec_ms = d.fwd_ms;
  } else {
    d.fwd_ms = s.fwd_ms;
    d.bwd_ms = s.bwd_ms;
    d.rec_ms = s.recompute_ms;
  }
  if (d.policy == GPB_ATLAS) {
    // the per-stage drain decomposition needs a positive pair duration
    const long long dur = (long long)std::llround(d.bwd_ms * 1e6) +
                          (d.recompute ? (long long)std::llround(d.rec_ms * 1e6) : 0);
    if (dur <= 0)
      throw ConfigErr{P_(i) + ": atlas pair duration rounds to 0 ns (outside the envelope)"};
    // one lane per pipeline in the per-stage drain greedy
    if (d.C > 32)
      throw ConfigErr{P_(i) + ": atlas with more than 32 pipelines per cell is outside the "
                              "kernel envelope"};
  }
  int order[GPB_MAX_DC];
  int n_order = s.n_order;
  if (n_order > 0) {
    for (int k = 0; k < n_order; ++k) order[k] = s.dc_order[k];
  } else {  // default_dc_order (workload.cpp:47-55): stable, count desc
    n_order = t.n_dc;
    for (int k = 0; k < n_order; ++k) order[k] = k;
    std::stable_sort(order, order + n_order,
                     [&](int a, int b) { return t.gpu_count[a] > t.gpu_count[b]; });
  }
  d.n_order = n_order;
  for (int k = 0; k < n_order; ++k) d.order[k] = (int8_t)order[k];
  long long total = 0;
  for (int k = 0; k < t.n_dc; ++k) total += t.gpu_count[k];
  const long long per_cell = (long long)d.C * d.S * d.tp;
  const int dflt = (int)std::max<long long>(0, total / per_cell);  // dc_select.cpp:20-25
  const int d_max = std::max(1, s.d_max > 0 ? s.d_max : dflt);
  d.n_rows = d_max;
}

}  // namespace gpb

namespace gpb {

// Run fn(lo, hi) over [0, n) in contiguous chunks on up to 16 host threads
// (one chunk when n is small).
template <typename Fn>
static void parallel_chunks(int64_t n, int64_t min_chunk, Fn fn) {
  const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nt = std::max<int64_t>(1, std::min<int64_t>({16, hw, n / std::max<int64_t>(1, min_chunk)}));
  if (nt <= 1) {
    fn(0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] { fn(n * t / nt, n * (t + 1) / nt, (int)t); });
  for (auto& x : th) x.join();
}

// Validate a plan space and flatten it into the device tables (DevTopo /
// DevScen with resolved profile, order, d_max and first row; optionally the
// row -> scenario table). Multi-threaded over topologies and scenarios for
// large spaces; the error reported is the first one in input order
// (topologies, then scenarios), as a sequential pass would find it.
int flatten_space(const gpb_topology* topos, int32_t n_topo, const gpb_scenario* scens,
                  int32_t n_scen, DevTopo* dt, DevScen* ds, std::vector<int32_t>* row_scen,
                  int64_t& n_rows, std::string& err) {
  if (n_scen < 0 || n_topo < 0 || (n_scen > 0 && (!topos || !scens))) {
    err = "null input";
    return GPB_CONFIG_ERROR;
  }
  constexpr int kMaxThreads = 16;
  // first error per chunk: (input index, message); topologies before scenarios
  std::vector<std::pair<int64_t, std::string>> errs(kMaxThreads, {-1, ""});
  auto first_error = [&]() -> const std::string* {
    const std::pair<int64_t, std::string>* best = nullptr;
    for (const auto& e : errs)
      if (e.first >= 0 && (!best || e.first < best->first)) best = &e;
    return best ? &best->second : nullptr;
  };
  parallel_chunks(n_topo, 2048, [&](int64_t lo, int64_t hi, int tid) {
    // single_tcp_bandwidth (libm log/exp) per distinct latency of the default
    // calibration table: plan spaces repeat a handful of WAN latencies
    std::vector<std::pair<double, double>> tcp_memo;
    auto single_bw = [&](const gpb_topology& t, double lat) {
      if (t.n_tcp > 0) return gpb_single_tcp_bandwidth(&t, lat);
      for (const auto& kv : tcp_memo)
        if (kv.first == lat) return kv.second;
      const double v = gpb_single_tcp_bandwidth(&t, lat);
      tcp_memo.emplace_back(lat, v);
      return v;
    };
    for (int64_t i = lo; i < hi; ++i) {
      try {
        validate_topology(topos[i], (int)i);
      } catch (const ConfigErr& e) {
        errs[tid] = {i, e.msg};
        return;
      }
      const gpb_topology& t = topos[i];
      DevTopo& d = dt[i];
      std::memset(&d, 0, sizeof d);
      d.n_dc = t.n_dc;
      int base = 0;
      for (int a = 0; a < t.n_dc; ++a) {
        d.gpu_count[a] = t.gpu_count[a];
        d.dc_base[a] = base;
        base += t.gpu_count[a];
        d.intra_bw[a] = t.intra_bw[a];
        for (int b = 0; b < t.n_dc; ++b) {
          // latency_between (topology.cpp:21-30): symmetric by unordered pair
          const double lat = a == b ? 0.0 : t.latency_ms[std::min(a, b)][std::max(a, b)];
          d.lat_ms[a][b] = lat;
          d.single_bw[a][b] = single_bw(t, lat);
        }
      }
      d.pair_cap = t.pair_bw_cap;
    }
  });
  if (const std::string* e = first_error()) {
    err = *e;
    return GPB_CONFIG_ERROR;
  }
  parallel_chunks(n_scen, 4096, [&](int64_t lo, int64_t hi, int tid) {
    for (int64_t i = lo; i < hi; ++i) {
      try {
        flatten_scenario(scens[i], (int)i, n_topo, topos, ds[i]);
      } catch (const ConfigErr& e) {
        errs[tid] = {n_topo + i, e.msg};
        return;
      }
    }
  });
  if (const std::string* e = first_error()) {
    err = *e;
    return GPB_CONFIG_ERROR;
  }
  int64_t row = 0;
  for (int i = 0; i < n_scen; ++i) {
    ds[i].first_row = row;
    row += ds[i].n_rows;
    if (row > (int64_t)1 << 31) {
      err = "plan space exceeds 2^31 rows";
      return GPB_CONFIG_ERROR;
    }
  }
  n_rows = row;
  if (row_scen) {
    row_scen->resize(row);
    int32_t* rs = row_scen->data();
    parallel_chunks(n_scen, 8192, [&](int64_t lo, int64_t hi, int) {
      for (int64_t i = lo; i < hi; ++i)
        std::fill(rs + ds[i].first_row, rs + ds[i].first_row + ds[i].n_rows, (int32_t)i);
    });
  }
  return GPB_OK;
}

}  // namespace gpb

// --------------------------------------------------------------- API

extern "C" {

gpb_ctx* gpb_create(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  Ctx* c = new Ctx();
  c->device = device;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  c->num_sms = prop.multiProcessorCount;
  c->smem_optin = (int)prop.sharedMemPerBlockOptin;
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
      cudaEventCreate(&c->ev2) != cudaSuccess || cudaEventCreate(&c->ev3) != cudaSuccess ||
      cudaEventCreate(&c->pack_ev0) != cudaSuccess || cudaEventCreate(&c->pack_ev1) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->switch_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return nullptr;
  }
  c->stream = c->own_stream;
  return reinterpret_cast<gpb_ctx*>(c);
}

void gpb_destroy(gpb_ctx* ctx) { delete reinterpret_cast<Ctx*>(ctx); }

const char* gpb_last_error(gpb_ctx* ctx) {
  return ctx ? reinterpret_cast<Ctx*>(ctx)->last_error.c_str() : "";
}

// GPB_NO_GROUP_FLUSH=1: one warp per flush row (A/B switch)
static const bool kNoGroupFlush = std::getenv("GPB_NO_GROUP_FLUSH") != nullptr;
// spaces with fewer rows keep one warp per flush row (GPB_GROUP_FLUSH_MIN_ROWS
// overrides, read at every load: tests force the grouped kernel)
// one-thread ATLAS rows: per-thread slice bound (int64 elements, 256 KB)
constexpr long long kSeqMaxSlice = 32768;
// heavy ATLAS rows with 2..4 pipelines (S <= 32) can run one CTA per row, one
// warp per pipeline (atlas_wave_kernel): GPB_ATLAS_WAVE=1 for heavy rows, =2
// for every such ATLAS row (tests). Off by default: on config 2's critical
// row (S=16, C=4, M=64) pipeline p's microbatches sit far later in simulated
// time than p-1's (the pooled links are saturated by the earlier pipelines),
// so p trails p-1 by ~40-60 microbatches of work and the staircase of
// frontier waits leaves little concurrency: 0.96 M cycles on the wave vs
// 1.03 M on one warp (profiles/r02_summary.md), within run-to-run noise of
// the step.
static int atlas_wave_mode() {
  const char* e = std::getenv("GPB_ATLAS_WAVE");
  return e ? std::atoi(e) : 0;
}
static int atlas_seq_mode() {
  const char* e = std::getenv("GPB_ATLAS_SEQ");
  return e ? std::atoi(e) : 1;
}
// The 4-blocks-per-SM ATLAS instantiation (kernels_atlas.cu OCC4) for spaces
// large enough to be throughput-bound: measured config 5 (10^7 rows) 207 ->
// 193 ms, but its N=8 shard (1.25*10^6 rows, bound by its slowest warp rows)
// 50.6 -> 60.8 ms and small spaces' critical rows ~15 % slower.
static int64_t occ4_min_rows() {
  const char* e = std::getenv("GPB_OCC4_MIN_ROWS");
  return e ? std::atoll(e) : 2000000;
}
static int64_t group_flush_min_rows() {
  const char* e = std::getenv("GPB_GROUP_FLUSH_MIN_ROWS");
  return e ? std::atoll(e) : 200000;
}

static bool same_shapes(const std::vector<Bucket>& a, const std::vector<Bucket>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    const Bucket &x = a[i], &y = b[i];
    if (x.policy != y.policy || x.B != y.B || x.offset != y.offset || x.count != y.count ||
        x.max_m != y.max_m || x.max_cs != y.max_cs || x.max_cm != y.max_cm ||
        x.max_csm != y.max_csm || x.max_c != y.max_c || x.max_s != y.max_s ||
        x.max_nw != y.max_nw || x.heavy != y.heavy || x.gw != y.gw ||
        x.max_slice != y.max_slice)
      return false;
  }
  return true;
}

int gpb_load(gpb_ctx* ctx_, const gpb_topology* topos, int32_t n_topo,
             const gpb_scenario* scens, int32_t n_scen, int64_t* n_rows_out) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  c.last_error.clear();
  c.loaded = false;
  if (cudaSetDevice(c.device) != cudaSuccess) return c.cuda_fail(cudaGetLastError(), "set device");
  if (n_scen < 0 || n_topo < 0 || (n_scen > 0 && (!topos || !scens))) {
    c.set_error("null input");
    return GPB_CONFIG_ERROR;
  }
  // GPB_DEBUG_LOAD=1: host time of each load stage on stderr
  static const bool dbg = std::getenv("GPB_DEBUG_LOAD") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t_prev = now();
  auto lap = [&](const char* what) {
    if (!dbg) return;
    const auto t = now();
    std::fprintf(stderr, "gpb_load %-10s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t_prev).count());
    t_prev = t;
  };
  // The topology and scenario tables are flattened straight into pinned
  // staging (already resident: no page faults on 10^5-scenario spaces, no
  // copy before the H2D); they stay the host view of the loaded space.
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t sz_t = sizeof(DevTopo) * std::max(n_topo, 1),
               sz_s = sizeof(DevScen) * std::max(n_scen, 1);
  if (c.upload_pending) {  // the previous upload must have left the staging buffers
    cudaEventSynchronize(c.upload_ev);
    c.upload_pending = false;
  }
  if (c.stage_ts_bytes < al(sz_t) + al(sz_s)) {
    if (c.stage_ts) cudaFreeHost(c.stage_ts);
    c.stage_ts = nullptr;
    c.stage_ts_bytes = 0;
    if (cudaMallocHost(&c.stage_ts, al(sz_t) + al(sz_s)) != cudaSuccess)
      return c.cuda_fail(cudaErrorMemoryAllocation, "pinned staging");
    c.stage_ts_bytes = al(sz_t) + al(sz_s);
  }
  DevTopo* dt = (DevTopo*)c.stage_ts;
  DevScen* ds = (DevScen*)((unsigned char*)c.stage_ts + al(sz_t));
  int64_t n_rows = 0;
  {
    const int rc = flatten_space(topos, n_topo, scens, n_scen, dt, ds, nullptr, n_rows,
                                 c.last_error);
    if (rc != GPB_OK) return rc;
  }
  lap("flatten");

  // Buckets: (policy, B = ceil(S/32)); within a bucket scenarios are dealt
  // in decreasing estimated cost so the persistent warps finish together.
  const std::vector<Bucket> prev_buckets = c.eval_ready ? c.buckets : std::vector<Bucket>();
  c.buckets.clear();
  // One bucket (one kernel) per (policy, B): rows of every shape share the
  // persistent warps, heaviest first. Estimated row cost in clock cycles
  // (fitted to profiled config-2 rows): ATLAS ~ C*M*(2000*C + 250*S) (list
  // unions over C pipelines + per-pair work), the flush/1F1B wavefronts
  // ~ 20*M*S.
  // ATLAS rows within 30% of the heaviest estimate form their own "heavy"
  // bucket, launched first (few warps, the critical path); the short
  // flush/1F1B buckets follow, then the bulk ATLAS rows fill the GPU.
  static const double kFlushK = [] {
    const char* e = std::getenv("GPB_FLUSH_COST");
    return e ? std::atof(e) : 20.0;
  }();
  auto cost = [&](int i) {
    const DevScen& d = ds[i];
    return d.policy == GPB_ATLAS ? (double)d.C * d.M * (2000.0 * d.C + 250.0 * d.S)
                                 : kFlushK * (d.policy == GPB_1F1B ? 1.5 : 1.0) * d.M * d.S;
  };
  double max_atlas = 0;
  for (int i = 0; i < n_scen; ++i)
    if (ds[i].policy == GPB_ATLAS) max_atlas = std::max(max_atlas, cost(i));
  // in large (throughput-bound) spaces, gpipe/varuna/1f1b rows of shallow
  // pipelines (S <= 8 / 16) get their own buckets with several rows per warp
  // (flush_group_kernel, onef1b_group_kernel); small spaces are bound by their longest row and
  // keep fewer buckets (measured: config 2 0.59 -> 0.63 ms with the split,
  // config 5 387 -> 369 ms)
  const int64_t group_min = group_flush_min_rows();
  // ... and ATLAS rows of shallow pipelines (S <= 16) outside the heavy
  // bucket run one per thread (atlas_seq_kernel); GPB_ATLAS_SEQ=0 disables,
  // =2 also takes heavy rows (tests)
  const int seq_mode = atlas_seq_mode();
  // A row on one thread takes ~10-16x its warp-kernel time (measured: the
  // slowest config-3 / config-5 thread rows, S = 14, C = 4, M = 64 / 256,
  // 49 M / 126 M cycles against 3 M / 12 M estimated), and the seq buckets
  // start their heaviest rows first, so in a plan-space shard the slowest
  // thread rows set the step (config 5 at N = 8: the S <= 16 thread bucket
  // ran 78.5 ms, every other bucket ended by 45 ms). Rows whose estimated
  // cost exceeds the space's total cost / (8 warps x SMs x GPB_SEQ_RATIO)
  // stay on a warp. Measured (tools/space_shard_rows.py, one GPU per shard):
  // ratio 25 keeps configs 3 and 5 at N = 1 unchanged (26 / 205 ms) and
  // takes config 3's N = 4 shard 19.2 -> 11.5 ms and config 5's N = 8 shard
  // 75.7 -> 50.6 ms; larger ratios move more rows (config 5 N = 8: 32 ms at
  // 300) but slow config 3 at N = 1 (26 -> 31 ms, its warp bucket
  // saturates). 0 disables the cut.
  static const double kSeqRatio = [] {
    const char* e = std::getenv("GPB_SEQ_RATIO");
    return e ? std::atof(e) : 25.0;
  }();
  double space_cost = 0;
  for (int i = 0; i < n_scen; ++i) space_cost += cost(i) * ds[i].n_rows;
  const double seq_cost_max =
      kSeqRatio > 0 ? space_cost / (8.0 * std::max(1, c.num_sms) * kSeqRatio) : 1e300;
  auto seq_ok = [&](const DevScen& d, bool heavy, double row_cost) {
    return seq_mode > 0 && n_rows >= group_min && d.S <= 16 && d.C <= 8 &&
           (!heavy || seq_mode == 2) && (seq_mode == 2 || row_cost <= seq_cost_max) &&
           atlas_seq_slice(d.C, d.S, d.M, d.n_order - 1, d.mem_limit) <= kSeqMaxSlice;
  };
  const int wave_mode = atlas_wave_mode();
  auto wave_ok = [&](const DevScen& d, bool heavy) {
    return wave_mode > 0 && (heavy || wave_mode == 2) && d.S <= 32 && d.C >= 2 &&
           d.C <= kWaveMaxPipes;
  };
  auto gw_of = [&](const DevScen& d, bool heavy, double row_cost) {
    // ATLAS: 32 = one warp per row, 4 / 8 / 16 = one thread per row with
    // stage loops unrolled to that bound (atlas_seq_kernel<SMAX>), 0 = one
    // CTA per row with one warp per pipeline (atlas_wave_kernel)
    if (d.policy == GPB_ATLAS) {
      if (wave_ok(d, heavy)) return 0;
      return seq_ok(d, heavy, row_cost) ? (d.S <= 4 ? 4 : d.S <= 8 ? 8 : 16) : 32;
    }
    if (kNoGroupFlush || n_rows < group_min) return 32;
    const int gw = d.S <= 8 ? 8 : (d.S <= 16 ? 16 : 32);
    // the per-row last-stage buffer (M entries per row) must fit the block
    return (size_t)(kEvalThreads / gw) * d.M * 8 <= 160 * 1024 ? gw : 32;
  };
  const int heavy_b = [] {
    const char* e = std::getenv("GPB_HEAVY_B");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  std::map<std::tuple<int, int, int, int>, std::vector<int>> by_key;
  for (int i = 0; i < n_scen; ++i) {
    int heavy = ds[i].policy == GPB_ATLAS && cost(i) >= 0.3 * max_atlas;
    const int gw = gw_of(ds[i], heavy != 0, cost(i));
    if (ds[i].policy == GPB_ATLAS && gw > 0 && gw < 32) heavy = 0;
    if (ds[i].policy == GPB_ATLAS && gw == 0) heavy = 1;
    int B = (ds[i].S + 31) / 32;
    if (heavy && gw == 32) B = std::max(B, std::min(8, heavy_b));
    by_key[{ds[i].policy, B, heavy, gw}].push_back(i);
  }
  std::vector<int32_t> bscen;
  bscen.reserve(n_scen);
  std::vector<int64_t> bscen_row;  // work-list offset of each bscen entry's first row
  bscen_row.reserve(n_scen);
  int64_t n_work = 0;
  for (auto& [key, list] : by_key) {
    std::stable_sort(list.begin(), list.end(), [&](int a, int b) { return cost(a) > cost(b); });
    Bucket b;
    b.policy = std::get<0>(key);
    b.B = std::get<1>(key);
    b.heavy = std::get<2>(key) != 0;
    b.gw = std::get<3>(key);
    b.offset = (int32_t)n_work;
    double total = 0;
    for (int i : list) {
      total += cost(i) * ds[i].n_rows;
      bscen_row.push_back(n_work);
      n_work += ds[i].n_rows;
      b.max_m = std::max(b.max_m, ds[i].M);
      b.max_cs = std::max(b.max_cs, ds[i].C * ds[i].S);
      b.max_cm = std::max(b.max_cm, ds[i].C * ds[i].M);
      b.max_csm = std::max(b.max_csm, (long long)ds[i].C * ds[i].S * ds[i].M);
      b.max_c = std::max(b.max_c, ds[i].C);
      b.max_s = std::max(b.max_s, ds[i].S);
      b.max_nw = std::max(b.max_nw, ds[i].n_order - 1);
      if (b.policy == GPB_ATLAS && b.gw > 0 && b.gw < 32)
        b.max_slice = std::max(b.max_slice, atlas_seq_slice(ds[i].C, ds[i].S, ds[i].M,
                                                            ds[i].n_order - 1, ds[i].mem_limit));
    }
    b.count = (int32_t)(n_work - b.offset);
    b.scen_off = (int32_t)bscen.size();
    b.scen_cnt = (int32_t)list.size();
    for (int i : list) bscen.push_back(i);
    b.cost = cost(list.front());
    // makespan estimate: the longest row, or the whole bucket spread over
    // ~8 resident warps per SM
    b.est = std::max(b.cost, total / (8.0 * std::max(1, c.num_sms)));
    c.buckets.push_back(b);
  }
  // launch order: heavy ATLAS, flush/1F1B, bulk ATLAS; heaviest first within
  auto rank = [](const Bucket& b) { return b.policy != GPB_ATLAS ? 1 : (b.heavy ? 0 : 2); };
  std::stable_sort(c.buckets.begin(), c.buckets.end(), [&](const Bucket& x, const Bucket& y) {
    return rank(x) != rank(y) ? rank(x) < rank(y) : x.cost > y.cost;
  });
  c.sel_blocks = 0;
  for (Bucket& b : c.buckets) {
    b.sel_grid = b.count > 0 ? std::max(1, std::min(256, (b.scen_cnt + 3) / 4)) : 0;
    b.sel_off = c.sel_blocks;
    c.sel_blocks += b.sel_grid;
  }

  lap("buckets");
  // Upload: the tables are written straight into one pinned staging buffer
  // (the per-row tables by several host threads) and copied asynchronously
  // on the launch stream (evaluate is ordered after them).
  cudaStream_t st = c.stream;
  const size_t sz_r = sizeof(int32_t) * n_rows, sz_w = sizeof(int32_t) * n_work,
               sz_b = sizeof(int32_t) * bscen.size();
  const size_t stage_need = al(sz_r) + al(sz_w) + al(sz_b);
  if (c.stage_bytes < stage_need) {
    if (c.stage) cudaFreeHost(c.stage);
    c.stage = nullptr;
    c.stage_bytes = 0;
    if (cudaMallocHost(&c.stage, stage_need) != cudaSuccess)
      return c.cuda_fail(cudaErrorMemoryAllocation, "pinned staging");
    c.stage_bytes = stage_need;
  }
  if (!c.upload_ev && cudaEventCreateWithFlags(&c.upload_ev, cudaEventDisableTiming) != cudaSuccess)
    return c.cuda_fail(cudaGetLastError(), "event");
  const unsigned char* st_t = (const unsigned char*)dt;
  const unsigned char* st_s = (const unsigned char*)ds;
  int32_t* st_r = (int32_t*)c.stage;
  int32_t* st_w = (int32_t*)((unsigned char*)st_r + al(sz_r));
  int32_t* st_b = (int32_t*)((unsigned char*)st_w + al(sz_w));
  std::memcpy(st_b, bscen.data(), sz_b);
  // row -> scenario and the bucket work lists (rows of each bucket scenario
  // in D order), one contiguous range of scenarios per host thread
  parallel_chunks(n_scen, 8192, [&](int64_t lo, int64_t hi, int) {
    for (int64_t i = lo; i < hi; ++i)
      std::fill(st_r + ds[i].first_row, st_r + ds[i].first_row + ds[i].n_rows, (int32_t)i);
    for (int64_t j = lo; j < hi; ++j) {
      const DevScen& d = ds[bscen[j]];
      int32_t* w = st_w + bscen_row[j];
      for (int k = 0; k < d.n_rows; ++k) w[k] = (int32_t)(d.first_row + k);
    }
  });
  lap("fill");
  auto up = [&](Buf& b, const void* src, size_t bytes) -> bool {
    void* p = c.dev_buf(b, bytes);
    if (!p) return false;
    if (bytes == 0) return true;
    return cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, st) == cudaSuccess;
  };
  if (!up(c.b_topos, st_t, sz_t) || !up(c.b_scens, st_s, sz_s) ||
      !up(c.b_row_scen, st_r, sz_r) || !up(c.b_work, st_w, sz_w) ||
      !up(c.b_bscen, st_b, sz_b) ||
      !c.dev_buf(c.b_rows, sizeof(gpb_row) * std::max<int64_t>(n_rows, 1)) ||
      !c.dev_buf(c.b_results, sizeof(gpb_scenario_result) * std::max(n_scen, 1)) ||
      !c.dev_buf(c.b_cursors, sizeof(int32_t) * (c.buckets.size() + 1)) ||
      !c.dev_buf(c.b_best, sizeof(gpb_best) * (2 + (size_t)c.sel_blocks))) {
    return c.cuda_fail(cudaGetLastError(), "upload");
  }
  cudaEventRecord(c.upload_ev, st);
  c.upload_pending = true;
  lap("upload");
  c.d2h_bytes = 0;
  c.h2d_bytes = sz_t + sz_s + sz_r + sz_w + sz_b;
  c.n_rows = n_rows;
  c.n_scen = n_scen;
  c.n_topo = n_topo;
  c.dev_scens_host = ds;
  c.dev_topos_host = dt;
  c.bscen_host = std::move(bscen);
  lap("keep");
  // the launch sequence (ATLAS shapes, scratch, stream assignment) depends
  // only on the buckets' shapes: reuse it when a reload has the same ones.
  // A captured graph (GPB_GRAPH) also bakes in each bucket's select split and
  // every table pointer; gpb_evaluate replays it only while that
  // fingerprint is unchanged (graph_key), else re-captures.
  if (!same_shapes(prev_buckets, c.buckets)) {
    c.eval_ready = false;
  } else {
    for (size_t i = 0; i < c.buckets.size(); ++i) c.buckets[i].stream = prev_buckets[i].stream;
  }
  c.loaded = true;
  if (n_rows_out) *n_rows_out = n_rows;
  return GPB_OK;
}

// The evaluate launch sequence (timing events, cursor reset, bucket kernels
// forked onto side streams, join, selection) on stream `st`. `cap` marks a
// stream capture: timing events become external event nodes of the graph.
static int record_evaluate(Ctx& c, cudaStream_t st, bool cap) {
  auto rec = [&](cudaEvent_t ev, cudaStream_t s2) {
    return cap ? cudaEventRecordWithFlags(ev, s2, cudaEventRecordExternal)
               : cudaEventRecord(ev, s2);
  };
  int32_t* cursors = (int32_t*)c.b_cursors.ptr;
  int32_t* err_flag = cursors + c.buckets.size();
  rec(c.ev0, st);
  cudaMemsetAsync(cursors, 0, sizeof(int32_t) * (c.buckets.size() + 1), st);
  int launches = 0;
  const int grid_eval = c.num_sms * 8;
  const size_t n_side = c.n_side;
  cudaEventRecord(c.fork_ev, st);  // fork point (dependency only)
  for (size_t k = 0; k < n_side; ++k) cudaStreamWaitEvent(c.side[k], c.fork_ev, 0);
  const bool bt = c.bucket_timing;  // per-bucket events (profiling, roofline)
  if (bt) rec(c.bucket_ev[c.buckets.size()], st);
  for (size_t bi = 0; bi < c.buckets.size(); ++bi) {
    const Bucket& b = c.buckets[bi];
    cudaStream_t ss = c.side[b.stream];
    if (bt) rec(c.bucket_ev[bi], ss);
    if (b.count == 0) {
      if (bt) rec(c.bucket_ev_end[bi], ss);
      continue;
    }
    EvalArgs a;
    std::memset(&a, 0, sizeof a);
    a.scens = (const DevScen*)c.b_scens.ptr;
    a.topos = (const DevTopo*)c.b_topos.ptr;
    a.row_scen = (const int32_t*)c.b_row_scen.ptr;
    a.work = (const int32_t*)c.b_work.ptr + b.offset;
    a.n_work = b.count;
    a.cursor = cursors + bi;
    a.rows = (gpb_row*)c.b_rows.ptr;
    a.error_flag = err_flag;
    a.row_cycles = c.profile_rows ? (long long*)c.b_cycles.ptr : nullptr;
    a.row_phase = a.row_cycles ? a.row_cycles + c.n_rows : nullptr;
    a.drain_lane = c.drain_lane;
    a.occ4 = b.B == 1 && c.n_rows >= occ4_min_rows();
    const int grid = std::min(grid_eval, (b.count + 3) / 4);
    cudaError_t e;
    if (b.policy == GPB_GPIPE || b.policy == GPB_VARUNA) {
      a.smem_m = b.max_m;
      e = b.gw < 32 ? launch_flush_group(b.gw, b.policy == GPB_GPIPE, a,
                                         std::min(grid_eval, (b.count + 4 * (32 / b.gw) - 1) /
                                                                 (4 * (32 / b.gw))), ss)
                    : launch_flush(b.B, b.policy == GPB_GPIPE, a, grid, ss);
    } else if (b.policy == GPB_1F1B) {
      e = b.gw < 32 ? launch_onef1b_group(b.gw, a,
                                          std::min(grid_eval, (b.count + 4 * (32 / b.gw) - 1) /
                                                                  (4 * (32 / b.gw))), ss)
                    : launch_onef1b(b.B, a, grid, ss);
    } else {
      const AtlasPlan& P = c.aplan[bi];
      a.lay = P.L;
      a.scratch_per_warp = P.scratch_per_warp;
      a.scratch_big_off = P.scratch_big_off;
      a.scratch = P.scratch_per_warp > 0 ? (long long*)c.b_scratch.ptr + c.scr_off[bi] : nullptr;
      if (b.heavy && b.gw == 32 && c.heavy_excl) a.smem_floor = c.smem_optin;
      e = b.gw == 0   ? launch_atlas_wave(a, P.grid, P.wpc, ss)
          : b.gw < 32 ? launch_atlas_seq(b.gw, a, P.grid, ss)
                      : launch_atlas(b.B, a, P.grid, P.wpc, ss);
    }
    if (e != cudaSuccess) return c.cuda_fail(e, "eval launch");
    if (bt) rec(c.bucket_ev_end[bi], ss);
    ++launches;
    // select() over the bucket's scenarios (dc_select.cpp:99-123), on its stream
    SelectArgs sa;
    sa.scens = (const DevScen*)c.b_scens.ptr;
    sa.scen_list = (const int32_t*)c.b_bscen.ptr + b.scen_off;
    sa.n_scen = b.scen_cnt;
    sa.rows = (gpb_row*)c.b_rows.ptr;
    sa.results = (gpb_scenario_result*)c.b_results.ptr;
    sa.block_best = (gpb_best*)c.b_best.ptr + 1 + b.sel_off;
    sa.best = (gpb_best*)c.b_best.ptr;
    if ((e = launch_select_part(sa, b.sel_grid, ss)) != cudaSuccess)
      return c.cuda_fail(e, "select launch");
    ++launches;
  }
  for (size_t k = 0; k < n_side; ++k) {  // join
    cudaEventRecord(c.side_done[k], c.side[k]);
    cudaStreamWaitEvent(st, c.side_done[k], 0);
  }
  rec(c.ev1, st);
  cudaError_t e = launch_best_reduce((gpb_best*)c.b_best.ptr + 1, c.sel_blocks,
                                     (gpb_best*)c.b_best.ptr, st);
  if (e != cudaSuccess) return c.cuda_fail(e, "select launch");
  launches += 1;
  rec(c.ev2, st);
  c.last_launches = launches + 1;  // + the cursor memset
  return GPB_OK;
}

// Everything the launch sequence needs, once per loaded space: events, side
// streams, ATLAS launch shapes, scratch, stream assignment (LPT).
static int prepare_evaluate(Ctx& c) {
  auto mk = [&](std::vector<cudaEvent_t>& v, size_t n, unsigned flags) -> bool {
    while (v.size() < n) {
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, flags) != cudaSuccess) return false;
      v.push_back(e);
    }
    return true;
  };
  if (!mk(c.bucket_ev, c.buckets.size() + 1, cudaEventDefault) ||
      !mk(c.bucket_ev_end, c.buckets.size(), cudaEventDefault))
    return c.cuda_fail(cudaGetLastError(), "event");
  if (!c.fork_ev && cudaEventCreateWithFlags(&c.fork_ev, cudaEventDisableTiming) != cudaSuccess)
    return c.cuda_fail(cudaGetLastError(), "event");
  // buckets run concurrently on side streams forked from the launch stream
  size_t max_side = kSideStreams;
  if (const char* e = std::getenv("GPB_SIDE_STREAMS")) max_side = std::max(1, std::atoi(e));
  c.n_side = std::max<size_t>(1, std::min<size_t>(max_side, c.buckets.size()));
  // Side stream 0 carries the bucket with the longest row (below) and runs at
  // the highest priority, so the critical rows' CTAs are dispatched first
  // when the buckets co-run; graph replays keep it (per-node priorities).
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  const char* penv = std::getenv("GPB_PRIO");
  if (penv && penv[0] == '0') prio_hi = prio_lo;
  while (c.side.size() < c.n_side) {
    cudaStream_t s2;
    cudaEvent_t e2;
    if (cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking,
                                     c.side.empty() ? prio_hi : prio_lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&e2, cudaEventDisableTiming) != cudaSuccess)
      return c.cuda_fail(cudaGetLastError(), "side streams");
    c.side.push_back(s2);
    c.side_done.push_back(e2);
  }
  for (const Bucket& b : c.buckets)
    if ((b.policy == GPB_GPIPE || b.policy == GPB_VARUNA) &&
        (int)((size_t)(kEvalThreads / 32) * b.max_m * 8) > c.smem_optin) {
      c.set_error("num_microbatches too large for the flush kernel's shared buffer");
      return GPB_CONFIG_ERROR;
    }
  // ATLAS launch shapes: the global scratch of every concurrently running
  // bucket is carved from one allocation
  c.aplan.assign(c.buckets.size(), AtlasPlan());
  c.scr_off.assign(c.buckets.size(), 0);
  size_t scr_total = 0;
  for (size_t bi = 0; bi < c.buckets.size(); ++bi) {
    const Bucket& b = c.buckets[bi];
    if (b.policy != GPB_ATLAS || b.count == 0) continue;
    if (b.gw == 0) {  // one CTA per row, one warp per pipeline
      AtlasPlan& P = c.aplan[bi];
      const int rc = plan_atlas(c, 1, false, b.max_c, b.max_s, b.max_m, b.max_nw, b.max_csm, 1, P);
      if (rc != GPB_OK) return rc;
      if (atlas_wave_smem(P.L) > c.smem_optin) {
        c.set_error("atlas wave plan too large for the shared-memory slice");
        return GPB_CONFIG_ERROR;
      }
      P.wpc = b.max_c;
      const int per_sm = std::max(1, atlas_wave_blocks_per_sm(P.wpc, atlas_wave_smem(P.L)));
      P.grid = std::max(1, std::min(b.count, c.num_sms * per_sm));
      c.scr_off[bi] = scr_total;
      scr_total += (size_t)P.scratch_per_warp * P.grid;
      continue;
    }
    if (b.gw < 32) {  // one thread per row: a per-thread slice
      AtlasPlan& P = c.aplan[bi];
      const long long slice = b.max_slice;
      P.wpc = kEvalThreads / 32;
      long long per_sm = std::max(1, atlas_seq_blocks_per_sm(b.gw));
      if (const char* e = std::getenv("GPB_SEQ_PER_SM")) per_sm = std::max(1, std::atoi(e));
      long long grid = std::min<long long>((long long)c.num_sms * per_sm,
                                           (b.count + kEvalThreads - 1) / kEvalThreads);
      // scratch bound: 12 GiB per bucket (rows beyond the resident ones reuse it)
      while (grid > c.num_sms && grid * kEvalThreads * slice * 8 > (12LL << 30)) grid -= c.num_sms;
      P.grid = (int)std::max(1LL, grid);
      P.scratch_per_warp = 32 * slice;
      P.scratch_big_off = 0;
      c.scr_off[bi] = scr_total;
      scr_total += (size_t)P.scratch_per_warp * P.grid * P.wpc;
      continue;
    }
    const int rc = plan_atlas(c, b.B, false, b.max_c, b.max_s, b.max_m, b.max_nw, b.max_csm,
                              b.count, c.aplan[bi]);
    if (rc != GPB_OK) return rc;
    if (!b.heavy) {
      // small (latency-bound) spaces: the bulk ATLAS rows keep one CTA per
      // SM so the flush/1F1B buckets launched beside them find room at once
      // (config 2: 0.551 -> 0.521 ms; their last kernel ended at 0.53 ms
      // behind two bulk CTAs per SM, now at 0.44 ms)
      const char* e = std::getenv("GPB_BULK_PER_SM");
      const int cap = e ? std::atoi(e) : (c.n_rows < group_flush_min_rows() ? 1 : 0);
      if (cap > 0) c.aplan[bi].grid = std::max(1, std::min(c.aplan[bi].grid, c.num_sms * cap));
    }
    if (std::getenv("GPB_DEBUG_PLAN"))
      std::fprintf(stderr, "atlas bucket %zu B=%d rows=%d C=%d S=%d M=%d nw=%d csm=%lld cap=%lld "
                   "total=%zu big_in_smem=%d wpc=%d grid=%d spw=%lld\n", bi, b.B, b.count,
                   b.max_c, b.max_s, b.max_m, b.max_nw, b.max_csm, c.aplan[bi].L.garr_cap,
                   c.aplan[bi].L.total, (int)c.aplan[bi].L.big_in_smem, c.aplan[bi].wpc,
                   c.aplan[bi].grid, c.aplan[bi].scratch_per_warp);
    c.scr_off[bi] = scr_total;
    scr_total += (size_t)c.aplan[bi].scratch_per_warp * c.aplan[bi].grid * c.aplan[bi].wpc;
  }
  if (scr_total > 0 && !c.dev_buf(c.b_scratch, sizeof(long long) * scr_total))
    return c.cuda_fail(cudaErrorMemoryAllocation, "atlas scratch");
  if (c.profile_rows && !c.dev_buf(c.b_cycles, 136 * (size_t)c.n_rows))
    return c.cuda_fail(cudaErrorMemoryAllocation, "row profile");
  {  // streams: longest estimate first onto the least loaded stream (LPT)
    std::vector<size_t> ord(c.buckets.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(),
                     [&](size_t x, size_t y) { return c.buckets[x].est > c.buckets[y].est; });
    std::vector<double> load(c.n_side, 0.0);
    for (size_t i : ord) {
      const size_t si = std::min_element(load.begin(), load.end()) - load.begin();
      load[si] += c.buckets[i].est;
      c.buckets[i].stream = (int)si;
    }
    // the bucket with the longest row (the step's critical path) goes to
    // side stream 0, the high-priority one
    size_t crit = 0;
    for (size_t i = 1; i < c.buckets.size(); ++i)
      if (c.buckets[i].cost > c.buckets[crit].cost) crit = i;
    const int cs = c.buckets.empty() ? 0 : c.buckets[crit].stream;
    for (Bucket& b : c.buckets)
      b.stream = b.stream == cs ? 0 : (b.stream == 0 ? cs : b.stream);
  }
  c.eval_ready = true;
  return GPB_OK;
}

void Ctx::drop_graph() {
  if (graph_exec) cudaGraphExecDestroy(graph_exec);
  graph_exec = nullptr;
  graph_stream = nullptr;
}

int gpb_evaluate(gpb_ctx* ctx_, int32_t sync) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  c.last_error.clear();
  if (!c.loaded) {
    c.set_error("no plan space loaded");
    return GPB_CONFIG_ERROR;
  }
  cudaSetDevice(c.device);
  cudaStream_t st = c.stream;
  if (!c.eval_ready) {
    c.drop_graph();
    const int rc = prepare_evaluate(c);
    if (rc != GPB_OK) return rc;
  }
  // The launch sequence is captured into a CUDA graph and replayed while
  // everything it baked in is unchanged: the stream, the buckets' launch
  // parameters (shapes, offsets, select splits, streams) and every device
  // pointer (a reload may reallocate a table). Measured on config 2: the
  // host launch cost per step drops 0.155 -> 0.022 ms and the two-session
  // e2e step 0.69 -> 0.56 ms; the replayed step itself is ~2 % slower on the
  // device (0.563 vs 0.549 ms). GPB_GRAPH=0 launches directly.
  const char* genv = std::getenv("GPB_GRAPH");
  const bool use_graph = !(genv && genv[0] == '0');
  const char* dl = std::getenv("GPB_DRAIN_LANE");
  c.drain_lane = dl ? std::atoi(dl) : 32;
  // small (latency-bound) spaces: the heavy ATLAS CTAs get whole SMs
  // (config 2: heavy bucket 0.511 -> 0.489 ms); saturated spaces keep the
  // SMs shared (config 5 with it: 204 -> 237 ms)
  const char* hx = std::getenv("GPB_HEAVY_EXCL");
  c.heavy_excl = hx ? std::atoi(hx) : (c.n_rows < group_flush_min_rows() ? 1 : 0);
  if (!use_graph) {
    const int rc = record_evaluate(c, st, false);
    if (rc != GPB_OK) return rc;
  } else {
    std::vector<long long> key;
    for (Buf* b : c.all_bufs()) key.push_back((long long)(uintptr_t)b->ptr);
    key.push_back((long long)(uintptr_t)st);
    key.push_back(c.bucket_timing);
    key.push_back(c.profile_rows);
    key.push_back(c.sel_blocks);
    key.push_back(c.drain_lane);
    key.push_back(c.heavy_excl);
    for (const Bucket& b : c.buckets)
      for (long long v : {(long long)b.policy, (long long)b.B, (long long)b.offset,
                          (long long)b.count, (long long)b.gw, (long long)b.stream,
                          (long long)b.scen_off, (long long)b.scen_cnt, (long long)b.sel_grid,
                          (long long)b.sel_off, (long long)b.max_m})
        key.push_back(v);
    for (size_t i = 0; i < c.aplan.size(); ++i)
      key.push_back(c.aplan[i].grid * 1000003LL + c.aplan[i].wpc + (long long)c.scr_off[i]);
    if (!c.graph_exec || key != c.graph_key) {
      c.drop_graph();
      cudaGraph_t g = nullptr;
      if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        return c.cuda_fail(cudaGetLastError(), "graph capture");
      const int rc = record_evaluate(c, st, true);
      const cudaError_t ce = cudaStreamEndCapture(st, &g);
      if (rc != GPB_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (ce != cudaSuccess) return c.cuda_fail(ce, "graph capture");
      const cudaError_t ie =
          cudaGraphInstantiate(&c.graph_exec, g, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) {
        c.graph_exec = nullptr;
        return c.cuda_fail(ie, "graph instantiate");
      }
      c.graph_stream = st;
      c.graph_key = key;
    }
    const cudaError_t e = cudaGraphLaunch(c.graph_exec, st);
    if (e != cudaSuccess) return c.cuda_fail(e, "graph launch");
  }
  c.timing_valid = true;
  c.bucket_timing_valid = c.bucket_timing;
  if (sync) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return c.cuda_fail(e, "evaluate");
    return c.check_error_flag();
  }
  return GPB_OK;
}

int gpb_fetch_rows(gpb_ctx* ctx_, gpb_row* rows, int64_t n) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  if (!c.loaded) {
    c.set_error("no plan space loaded");
    return GPB_CONFIG_ERROR;
  }
  cudaSetDevice(c.device);
  if (rows && n > 0) {
    n = std::min(n, c.n_rows);
    cudaError_t e = cudaMemcpyAsync(rows, c.b_rows.ptr, sizeof(gpb_row) * n,
                                    cudaMemcpyDeviceToHost, c.stream);
    c.d2h_bytes += (int64_t)sizeof(gpb_row) * n;
    if (e != cudaSuccess) return c.cuda_fail(e, "fetch rows");
  }
  cudaError_t e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) return c.cuda_fail(e, "fetch rows");
  return c.check_error_flag();
}

int gpb_fetch_scenarios(gpb_ctx* ctx_, gpb_scenario_result* out, int32_t n) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  cudaSetDevice(c.device);
  if (out && n > 0) {
    n = std::min(n, c.n_scen);
    cudaError_t e = cudaMemcpyAsync(out, c.b_results.ptr, sizeof(gpb_scenario_result) * n,
                                    cudaMemcpyDeviceToHost, c.stream);
    if (e != cudaSuccess) return c.cuda_fail(e, "fetch scenarios");
  }
  cudaError_t e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) return c.cuda_fail(e, "fetch scenarios");
  return c.check_error_flag();
}

int gpb_fetch_best(gpb_ctx* ctx_, gpb_best* out) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  cudaSetDevice(c.device);
  cudaError_t e = cudaMemcpyAsync(out, c.b_best.ptr, sizeof(gpb_best), cudaMemcpyDeviceToHost,
                                  c.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) return c.cuda_fail(e, "fetch best");
  return c.check_error_flag();
}

int gpb_copy_best(gpb_ctx* ctx_, void* dst) {
  if (!ctx_ || !dst) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  cudaError_t e = cudaMemcpyAsync(dst, c.b_best.ptr, sizeof(gpb_best), cudaMemcpyDeviceToDevice,
                                  c.stream);
  return e == cudaSuccess ? GPB_OK : c.cuda_fail(e, "copy best");
}

int gpb_set_stream(gpb_ctx* ctx_, void* s) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  cudaStream_t ns = s ? (cudaStream_t)s : c.own_stream;
  // work on the new stream is ordered after everything already enqueued on
  // the old one (uploads, an evaluate or pack still running), so fetches on
  // the new stream and the next load's H2D never overtake it
  if (ns != c.stream) {
    cudaSetDevice(c.device);
    if (cudaEventRecord(c.switch_ev, c.stream) != cudaSuccess ||
        cudaStreamWaitEvent(ns, c.switch_ev, 0) != cudaSuccess)
      return c.cuda_fail(cudaGetLastError(), "set stream");
  }
  c.stream = ns;
  return GPB_OK;  // the evaluate graph is re-captured for a new stream
}

int gpb_bucket_infos(gpb_ctx* ctx_, gpb_bucket_info* out, int32_t cap, int32_t* n) {
  if (!ctx_ || !n || (cap > 0 && !out)) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  *n = (int32_t)c.buckets.size();
  if (c.timing_valid) cudaEventSynchronize(c.ev2);
  for (int32_t bi = 0; bi < std::min<int32_t>(cap, *n); ++bi) {
    const Bucket& b = c.buckets[bi];
    gpb_bucket_info& o = out[bi];
    std::memset(&o, 0, sizeof o);
    o.policy = b.policy;
    o.B = b.B;
    o.rows = b.count;
    o.max_s = b.max_s;
    o.max_c = b.max_c;
    o.max_m = b.max_m;
    o.stream = b.stream;
    // algorithmic max-plus ops of the bucket's feasible rows
    double ops = 0;
    for (int32_t j = 0; j < b.scen_cnt; ++j) {
      const DevScen& d = c.dev_scens_host[c.bscen_host[b.scen_off + j]];
      for (int32_t k = 0; k < d.n_rows; ++k) {
        const int W = row_wan_boundaries(c, d.first_row + k);
        if (W < 0) continue;
        const double SM = (double)d.S * d.M, WM = (double)W * d.M;
        ops += d.policy == GPB_ATLAS ? d.C * (4 * SM + 6 * WM)
                                     : (d.policy == GPB_1F1B ? 4 * SM : 5 * SM) + 6 * WM;
      }
    }
    o.algo_ops = ops;
    if (c.timing_valid && c.bucket_timing_valid) {
      cudaEventElapsedTime(&o.start_ms, c.bucket_ev[c.buckets.size()], c.bucket_ev[bi]);
      cudaEventElapsedTime(&o.ms, c.bucket_ev[bi], c.bucket_ev_end[bi]);
    }
  }
  return GPB_OK;
}

void* gpb_device_best(gpb_ctx* ctx_) {
  if (!ctx_) return nullptr;
  return reinterpret_cast<Ctx*>(ctx_)->b_best.ptr;
}

int gpb_set_bucket_timing(gpb_ctx* ctx_, int32_t enable) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  if (c.bucket_timing != (enable != 0)) c.drop_graph();
  c.bucket_timing = enable != 0;
  return GPB_OK;
}

int gpb_get_timing(gpb_ctx* ctx_, gpb_timing* out) {
  if (!ctx_ || !out) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  std::memset(out, 0, sizeof *out);
  if (c.timing_valid) {
    cudaEventSynchronize(c.ev2);
    cudaEventElapsedTime(&out->evaluate_ms, c.ev0, c.ev2);
    cudaEventElapsedTime(&out->timing_kernels_ms, c.ev0, c.ev1);
    cudaEventElapsedTime(&out->select_ms, c.ev1, c.ev2);
    for (size_t bi = 0; c.bucket_timing_valid && bi < c.buckets.size(); ++bi) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c.bucket_ev[bi], c.bucket_ev_end[bi]);
      out->policy_ms[c.buckets[bi].policy] += ms;
    }
  }
  out->pack_ms = c.pack_ms;
  out->launches = c.last_launches;
  out->h2d_bytes = (int64_t)c.h2d_bytes;
  out->d2h_bytes = c.d2h_bytes;
  return GPB_OK;
}

}  // extern "C"

namespace gpb {
int Ctx::check_error_flag() {
  int32_t flag = 0;
  int32_t* cursors = (int32_t*)b_cursors.ptr;
  if (!cursors) return GPB_OK;
  cudaMemcpyAsync(&flag, cursors + buckets.size(), sizeof flag, cudaMemcpyDeviceToHost, stream);
  cudaStreamSynchronize(stream);
  if (flag) {
    set_error("kernel invariant failure (see rows with feasible == -1)");
    return GPB_ERROR;
  }
  return GPB_OK;
}
}  // namespace gpb

extern "C" int gpb_microbench(gpb_ctx* ctx_, int32_t kind, double* gops) {
  if (!ctx_ || !gops) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  if (kind < 0 || kind > 2) {
    c.set_error("unknown microbenchmark kind");
    return GPB_CONFIG_ERROR;
  }
  cudaSetDevice(c.device);
  void* out = c.dev_buf(c.b_pack_misc, 64);
  const int grid = c.num_sms * 8, iters = 4096;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(c.pack_ev0, c.stream);
    cudaError_t e = launch_maxplus_bench(kind, (long long*)out, grid, iters, c.stream);
    if (e != cudaSuccess) return c.cuda_fail(e, "microbench");
    cudaEventRecord(c.pack_ev1, c.stream);
    cudaEventSynchronize(c.pack_ev1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c.pack_ev0, c.pack_ev1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double ops = (double)grid * 256 * iters * 8 * 2;
  *gops = ops / (best * 1e-3) / 1e9;
  return GPB_OK;
}

extern "C" int gpb_set_profile(gpb_ctx* ctx_, int32_t enable) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  if (c.profile_rows != (enable != 0)) c.eval_ready = false;
  c.profile_rows = enable != 0;
  return GPB_OK;
}

extern "C" int gpb_fetch_row_cycles(gpb_ctx* ctx_, int64_t* out, int64_t n) {
  if (!ctx_ || !out) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  if (!c.profile_rows || !c.b_cycles.ptr) {
    c.set_error("row profiling not enabled");
    return GPB_CONFIG_ERROR;
  }
  cudaSetDevice(c.device);
  // out: n row costs followed by n x 16 atlas phase counters (when n == 17 * rows)
  const int64_t rows = c.n_rows;
  n = std::min(n, 17 * rows);
  cudaError_t e = cudaMemcpyAsync(out, c.b_cycles.ptr, 8 * (size_t)n, cudaMemcpyDeviceToHost,
                                  c.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
  return e == cudaSuccess ? GPB_OK : c.cuda_fail(e, "fetch row cycles");
}

namespace gpb {

// ATLAS launch shape. The per-warp shared slice holds the reservation lists,
// the per-pipeline stage state and the last-stage forward ends; the gradient
// queues [C][S][M] go to a per-warp global scratch (L1/L2-resident). Measured
// on config 2: global queues with 12 warps/SM beat shared-memory queues at
// 4-8 warps/SM both for the bucket makespan and for the longest row (the
// stage-strided queue accesses conflict on shared-memory banks).
// GPB_ATLAS_GARR_SMEM=<warps per SM> keeps queues that fit in shared memory
// at that occupancy (experiments).
int plan_atlas(Ctx& c, int B, bool timeline, int C, int S, int M, int nw, long long max_csm,
               long long count, AtlasPlan& P) {
  const size_t sm_budget = 220 * 1024;
  AtlasLayout& L = P.L;
  L.C = C;
  L.S = S;
  L.M = M;
  L.nw = nw;
  L.garr_cap = 0;
  L.compute();
  if (const char* t = std::getenv("GPB_ATLAS_GARR_SMEM")) {
    const long long target = std::max(1, std::atoi(t));
    const long long room = ((long long)(sm_budget / target) - (long long)L.total) / 8;
    L.garr_cap = std::max(0LL, std::min(max_csm, room));
    L.compute();
  }
  P.wpc = (int)std::min<size_t>(4, (size_t)c.smem_optin / L.total);
  if (P.wpc < 1) {  // lists too large for the slice: they go to the global scratch
    L.big_in_smem = false;
    L.garr_cap = 0;
    L.compute();
    P.wpc = (int)std::min<size_t>(4, (size_t)c.smem_optin / L.total);
  }
  if (P.wpc < 1) {
    c.set_error("atlas plan too large for the shared-memory slice");
    return GPB_CONFIG_ERROR;
  }
  const size_t smem = (size_t)P.wpc * L.total;
  int per_sm = atlas_blocks_per_sm(B, timeline, P.wpc, smem,
                                   B == 1 && !timeline && c.n_rows >= occ4_min_rows());
  per_sm = std::max(1, std::min(per_sm, (int)(sm_budget / smem)));
  P.grid = (int)std::max(1LL, std::min<long long>((long long)c.num_sms * per_sm,
                                                  (count + P.wpc - 1) / P.wpc));
  P.scratch_big_off = L.garr_cap < max_csm ? max_csm : 0;
  P.scratch_per_warp = P.scratch_big_off + (L.big_in_smem ? 0 : (long long)(L.big_total / 8));
  return GPB_OK;
}

}  // namespace gpb
