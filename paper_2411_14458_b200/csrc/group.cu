// group.cpp — one plan space sharded over several B200s of one box
// (include/geopipe_batch.h, gpb_group_*).
//
// The reference evaluates a whatif() space on one CPU thread
// (dc_select.cpp:125-134, called from run_whatif, runner.cpp:112-122). Plans
// are independent, so the group deals whole scenarios to the
// devices — longest estimated cost first onto the least-loaded device (LPT,
// the bucket cost model of host.cu), select()'s per-scenario argmax stays
// local — and drives each device's batch context from its own host thread
// (a context is single-threaded, geopipe.h:9). The only exchange is one
// ncclAllGather of the 16-byte per-device winners over NVLink; every device
// then holds all of them, and the global winner is keyed (throughput desc,
// global row asc): exactly the first maximum of one whatif() over the whole
// space. NCCL is opened at run time (dlopen), so the library has no link
// dependency on it and shares whichever libnccl the process already loaded.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/geopipe_batch.h"
#include "host_internal.h"

using namespace gpb;

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;

  bool open(std::string& err) {
    if (h) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      err = "libnccl.so.2 not found (needed to exchange winners between devices)";
      return false;
    }
    comm_init_all = (decltype(comm_init_all))dlsym(h, "ncclCommInitAll");
    all_gather = (decltype(all_gather))dlsym(h, "ncclAllGather");
    group_start = (decltype(group_start))dlsym(h, "ncclGroupStart");
    group_end = (decltype(group_end))dlsym(h, "ncclGroupEnd");
    comm_destroy = (decltype(comm_destroy))dlsym(h, "ncclCommDestroy");
    error_string = (decltype(error_string))dlsym(h, "ncclGetErrorString");
    if (!comm_init_all || !all_gather || !group_start || !group_end || !comm_destroy ||
        !error_string) {
      err = "libnccl.so.2 lacks the collective entry points";
      return false;
    }
    return true;
  }
};

Nccl& nccl() {
  static Nccl n;
  return n;
}

// Estimated cycles of one row (the bucket cost model of host.cu's gpb_load).
double row_cost(const DevScen& d) {
  return d.policy == GPB_ATLAS ? (double)d.C * d.M * (2000.0 * d.C + 250.0 * d.S)
                               : 20.0 * d.M * d.S;
}

}  // namespace

struct gpb_group {
  std::vector<int> devices;
  std::vector<gpb_ctx*> ctx;
  std::vector<ncclComm_t> comms;   // empty when devices repeat (no NCCL)
  std::vector<void*> gathered;     // per device: n_dev gpb_best records
  std::string last_error;
  // loaded space
  bool loaded = false;
  int64_t n_rows = 0;
  int32_t n_scen = 0;
  std::vector<std::vector<int32_t>> shard;      // per device: global scenario ids (space order)
  std::vector<std::vector<int64_t>> row_map;    // per device: local row -> global row (run starts)
  std::vector<int64_t> first_row;               // global first row per scenario
  std::vector<int32_t> rows_of;                 // d_max per scenario
  std::vector<int64_t> dev_rows;                // rows per device
  std::vector<std::vector<gpb_scenario>> dev_scens;
  std::vector<void*> staging;                   // pinned, per device
  std::vector<size_t> staging_bytes;
  bool evaluated = false;

  int fail(int rc, const std::string& msg) {
    last_error = msg;
    return rc;
  }
};

namespace {

// Run fn(k) for every device on its own host thread; the first failing rc
// (device order) wins, its message goes to the group.
template <typename Fn>
int on_devices(gpb_group& g, Fn fn) {
  const size_t n = g.ctx.size();
  std::vector<int> rc(n, GPB_OK);
  std::vector<std::string> msg(n);
  if (n == 1) {
    rc[0] = fn(0, msg[0]);
  } else {
    std::vector<std::thread> th;
    for (size_t k = 0; k < n; ++k) th.emplace_back([&, k] { rc[k] = fn((int)k, msg[k]); });
    for (auto& t : th) t.join();
  }
  for (size_t k = 0; k < n; ++k)
    if (rc[k] != GPB_OK) return g.fail(rc[k], msg[k]);
  return GPB_OK;
}

bool distinct(const std::vector<int>& v) {
  std::vector<int> s = v;
  std::sort(s.begin(), s.end());
  return std::adjacent_find(s.begin(), s.end()) == s.end();
}

}  // namespace

extern "C" {

gpb_group* gpb_group_create(int32_t n_dev, const int32_t* devices) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) return nullptr;
  gpb_group* g = new gpb_group();
  if (n_dev <= 0) {
    for (int d = 0; d < count; ++d) g->devices.push_back(d);
  } else {
    for (int k = 0; k < n_dev; ++k) {
      if (!devices || devices[k] < 0 || devices[k] >= count) {
        delete g;
        return nullptr;
      }
      g->devices.push_back(devices[k]);
    }
  }
  for (int d : g->devices) {
    gpb_ctx* c = gpb_create(d);
    if (!c) {
      gpb_group_destroy(g);
      return nullptr;
    }
    g->ctx.push_back(c);
  }
  const size_t n = g->devices.size();
  g->gathered.assign(n, nullptr);
  for (size_t k = 0; k < n; ++k) {
    cudaSetDevice(g->devices[k]);
    if (cudaMalloc(&g->gathered[k], sizeof(gpb_best) * n) != cudaSuccess) {
      gpb_group_destroy(g);
      return nullptr;
    }
  }
  // the winner exchange: one NCCL communicator per device (single process,
  // ncclCommInitAll); devices listed twice (tests) exchange through the host
  if (n > 1 && distinct(g->devices)) {
    std::string err;
    if (!nccl().open(err)) {
      gpb_group_destroy(g);
      return nullptr;
    }
    g->comms.assign(n, nullptr);
    if (nccl().comm_init_all(g->comms.data(), (int)n, g->devices.data()) != ncclSuccess) {
      g->comms.clear();
      gpb_group_destroy(g);
      return nullptr;
    }
  }
  g->staging.assign(n, nullptr);
  g->staging_bytes.assign(n, 0);
  return g;
}

void gpb_group_destroy(gpb_group* g) {
  if (!g) return;
  for (ncclComm_t c : g->comms)
    if (c) nccl().comm_destroy(c);
  for (size_t k = 0; k < g->gathered.size(); ++k)
    if (g->gathered[k]) {
      cudaSetDevice(g->devices[k]);
      cudaFree(g->gathered[k]);
    }
  for (void* p : g->staging)
    if (p) cudaFreeHost(p);
  for (gpb_ctx* c : g->ctx) gpb_destroy(c);
  delete g;
}

const char* gpb_group_last_error(gpb_group* g) { return g ? g->last_error.c_str() : ""; }

int32_t gpb_group_size(gpb_group* g) { return g ? (int32_t)g->ctx.size() : 0; }

int gpb_group_load(gpb_group* g, const gpb_topology* topos, int32_t n_topo,
                   const gpb_scenario* scens, int32_t n_scen, int64_t* n_rows_out) {
  if (!g) return GPB_ERROR;
  g->last_error.clear();
  g->loaded = g->evaluated = false;
  // validate the whole space once (same messages as a single-device load)
  std::vector<DevTopo> dt(std::max(n_topo, 1));
  std::vector<DevScen> ds(std::max(n_scen, 1));
  int64_t n_rows = 0;
  int rc = flatten_space(topos, n_topo, scens, n_scen, dt.data(), ds.data(), nullptr, n_rows,
                         g->last_error);
  if (rc != GPB_OK) return rc;
  const size_t n = g->ctx.size();
  // LPT over the devices by estimated cost, each shard in space order
  std::vector<int32_t> order(n_scen);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return row_cost(ds[a]) * ds[a].n_rows > row_cost(ds[b]) * ds[b].n_rows;
  });
  std::vector<double> load(n, 0.0);
  g->shard.assign(n, {});
  for (int32_t i : order) {
    const size_t k = std::min_element(load.begin(), load.end()) - load.begin();
    load[k] += row_cost(ds[i]) * ds[i].n_rows;
    g->shard[k].push_back(i);
  }
  g->first_row.assign(n_scen, 0);
  g->rows_of.assign(n_scen, 0);
  for (int32_t i = 0; i < n_scen; ++i) {
    g->first_row[i] = ds[i].first_row;
    g->rows_of[i] = ds[i].n_rows;
  }
  g->dev_scens.assign(n, {});
  g->dev_rows.assign(n, 0);
  for (size_t k = 0; k < n; ++k) {
    std::sort(g->shard[k].begin(), g->shard[k].end());
    for (int32_t i : g->shard[k]) g->dev_scens[k].push_back(scens[i]);
  }
  rc = on_devices(*g, [&](int k, std::string& msg) {
    int64_t nr = 0;
    const int r = gpb_load(g->ctx[k], topos, n_topo, g->dev_scens[k].data(),
                           (int32_t)g->dev_scens[k].size(), &nr);
    if (r != GPB_OK) msg = gpb_last_error(g->ctx[k]);
    g->dev_rows[k] = nr;
    return r;
  });
  if (rc != GPB_OK) return rc;
  g->n_rows = n_rows;
  g->n_scen = n_scen;
  g->loaded = true;
  if (n_rows_out) *n_rows_out = n_rows;
  return GPB_OK;
}

int gpb_group_evaluate(gpb_group* g) {
  if (!g) return GPB_ERROR;
  if (!g->loaded) return g->fail(GPB_CONFIG_ERROR, "no plan space loaded");
  int rc = on_devices(*g, [&](int k, std::string& msg) {
    const int r = gpb_evaluate(g->ctx[k], 0);
    if (r != GPB_OK) msg = gpb_last_error(g->ctx[k]);
    return r;
  });
  if (rc != GPB_OK) return rc;
  if (!g->comms.empty()) {
    // all-gather the 16-byte winners on each device's launch stream
    Nccl& N = nccl();
    N.group_start();
    for (size_t k = 0; k < g->ctx.size(); ++k) {
      Ctx& c = *reinterpret_cast<Ctx*>(g->ctx[k]);
      cudaSetDevice(c.device);
      const ncclResult_t r = N.all_gather(c.b_best.ptr, g->gathered[k], 2, ncclInt64,
                                          g->comms[k], c.stream);
      if (r != ncclSuccess) {
        N.group_end();
        return g->fail(GPB_ERROR, std::string("ncclAllGather: ") + N.error_string(r));
      }
    }
    const ncclResult_t r = N.group_end();
    if (r != ncclSuccess)
      return g->fail(GPB_ERROR, std::string("ncclGroupEnd: ") + N.error_string(r));
  }
  g->evaluated = true;
  return GPB_OK;
}

int gpb_group_fetch_rows(gpb_group* g, gpb_row* rows, int64_t n) {
  if (!g) return GPB_ERROR;
  if (!g->loaded) return g->fail(GPB_CONFIG_ERROR, "no plan space loaded");
  return on_devices(*g, [&](int k, std::string& msg) {
    const size_t bytes = sizeof(gpb_row) * std::max<int64_t>(1, g->dev_rows[k]);
    if (g->staging_bytes[k] < bytes) {
      if (g->staging[k]) cudaFreeHost(g->staging[k]);
      cudaSetDevice(g->devices[k]);
      if (cudaMallocHost(&g->staging[k], bytes) != cudaSuccess) {
        g->staging[k] = nullptr;
        g->staging_bytes[k] = 0;
        msg = "pinned staging";
        return GPB_ERROR;
      }
      g->staging_bytes[k] = bytes;
    }
    gpb_row* st = (gpb_row*)g->staging[k];
    const int r = gpb_fetch_rows(g->ctx[k], st, g->dev_rows[k]);
    if (r != GPB_OK) {
      msg = gpb_last_error(g->ctx[k]);
      return r;
    }
    // scatter each scenario's run of rows to its place in the space
    int64_t local = 0;
    for (int32_t gi : g->shard[k]) {
      const int64_t at = g->first_row[gi], cnt = g->rows_of[gi];
      for (int64_t j = 0; j < cnt; ++j) {
        if (at + j < n) {
          rows[at + j] = st[local + j];
          rows[at + j].scenario = gi;
        }
      }
      local += cnt;
    }
    return GPB_OK;
  });
}

int gpb_group_fetch_scenarios(gpb_group* g, gpb_scenario_result* out, int32_t n) {
  if (!g) return GPB_ERROR;
  if (!g->loaded) return g->fail(GPB_CONFIG_ERROR, "no plan space loaded");
  return on_devices(*g, [&](int k, std::string& msg) {
    std::vector<gpb_scenario_result> loc(std::max<size_t>(1, g->shard[k].size()));
    const int r = gpb_fetch_scenarios(g->ctx[k], loc.data(), (int32_t)g->shard[k].size());
    if (r != GPB_OK) {
      msg = gpb_last_error(g->ctx[k]);
      return r;
    }
    for (size_t j = 0; j < g->shard[k].size(); ++j) {
      const int32_t gi = g->shard[k][j];
      if (gi < n) {
        out[gi] = loc[j];
        out[gi].first_row = g->first_row[gi];
      }
    }
    return GPB_OK;
  });
}

int gpb_group_fetch_best(gpb_group* g, gpb_best* out) {
  if (!g || !out) return GPB_ERROR;
  if (!g->evaluated) return g->fail(GPB_CONFIG_ERROR, "no evaluation");
  const size_t n = g->ctx.size();
  std::vector<gpb_best> rec(n);
  if (!g->comms.empty()) {
    // every device holds every winner after the all-gather: read device 0's
    Ctx& c = *reinterpret_cast<Ctx*>(g->ctx[0]);
    cudaSetDevice(c.device);
    if (cudaMemcpyAsync(rec.data(), g->gathered[0], sizeof(gpb_best) * n,
                        cudaMemcpyDeviceToHost, c.stream) != cudaSuccess ||
        cudaStreamSynchronize(c.stream) != cudaSuccess)
      return g->fail(GPB_ERROR, "fetch gathered winners");
    for (size_t k = 1; k < n; ++k) {  // the other devices' streams must be done too
      Ctx& ck = *reinterpret_cast<Ctx*>(g->ctx[k]);
      cudaSetDevice(ck.device);
      if (cudaStreamSynchronize(ck.stream) != cudaSuccess)
        return g->fail(GPB_ERROR, "evaluate");
    }
  } else {
    for (size_t k = 0; k < n; ++k)
      if (gpb_fetch_best(g->ctx[k], &rec[k]) != GPB_OK)
        return g->fail(GPB_ERROR, gpb_last_error(g->ctx[k]));
  }
  // local row -> global row, then (throughput desc, global row asc)
  gpb_best best{0.0, -1};
  for (size_t k = 0; k < n; ++k) {
    if (rec[k].row < 0) continue;
    int64_t local = rec[k].row, grow = -1;
    for (int32_t gi : g->shard[k]) {
      if (local < g->rows_of[gi]) {
        grow = g->first_row[gi] + local;
        break;
      }
      local -= g->rows_of[gi];
    }
    if (grow < 0) return g->fail(GPB_ERROR, "winner row out of range");
    if (best.row < 0 || rec[k].throughput > best.throughput ||
        (rec[k].throughput == best.throughput && grow < best.row))
      best = {rec[k].throughput, grow};
  }
  *out = best;
  return GPB_OK;
}

}  // extern "C"
