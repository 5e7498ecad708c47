// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A C entry layer over the *unmodified* reference C++ API, compiled against
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libgeopipe_ref.so.
// It converts the batch ABI's plain structs (include/geopipe_batch.h) into the
// reference's own types and calls its public functions:
//   select()            dc_select.cpp:99-123
//   schedule_for_policy scheduler.cpp:604-611, run() engine.cpp:452-460
//   report()            metrics.cpp:32-81, utilization() bubbletea.cpp:224-238
//   extract_bubbles()   bubbletea.cpp:56-66
//   build_prefill_pipelines / schedule_prefills  bubbletea.cpp:88-222
//   synthetic_requests / saturating_requests     bubbletea.cpp:240-284
// Only tests/, __graft_entry__.smoke() and bench.py's reference leg load it.
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "bubbletea.h"
#include "comm_model.h"
#include "dc_select.h"
#include "engine.h"
#include "metrics.h"
#include "scheduler.h"
#include "topology.h"
#include "workload.h"

#include "../include/geopipe_batch.h"

using namespace geopipe;

namespace {

const char* kPolicies[4] = {"gpipe", "1f1b", "varuna", "atlas"};

std::string dc_name(int i) { return "dc" + std::to_string(i); }

ClusterTopology to_topo(const gpb_topology& t) {
  ClusterTopology topo;
  for (int i = 0; i < t.n_dc; ++i) {
    Datacenter d;
    d.id = dc_name(i);
    d.gpu_count = t.gpu_count[i];
    d.intra_bw = t.intra_bw[i];
    topo.datacenters.push_back(d);
  }
  for (int i = 0; i < t.n_dc; ++i)
    for (int j = i + 1; j < t.n_dc; ++j)
      topo.wan.latency_ms[{dc_name(i), dc_name(j)}] = t.latency_ms[i][j];
  topo.wan.pair_bw_cap = t.pair_bw_cap;
  if (t.n_tcp > 0) {
    for (int k = 0; k < t.n_tcp; ++k)
      topo.wan.tcp_table.push_back({t.tcp_latency_ms[k], t.tcp_bw[k]});
  } else {
    topo.wan.tcp_table = default_tcp_table();
  }
  return topo;
}

ModelSpec to_model(const gpb_scenario& s) {
  ModelSpec m;
  m.num_layers = s.num_layers;
  m.hidden = s.hidden;
  m.seq_len = s.seq_len;
  m.microbatch = s.microbatch;
  m.num_microbatches = s.num_microbatches;
  m.params_per_layer = s.params_per_layer;
  m.bytes_per_element = s.bytes_per_element;
  m.layers_per_partition = s.layers_per_partition;
  return m;
}

SelectionInput to_input(const gpb_topology* topos, const gpb_scenario& s) {
  SelectionInput in;
  in.topo = to_topo(topos[s.topology]);
  in.model = to_model(s);
  if (s.ratio_C > 0) {
    in.profile.ratio_C = s.ratio_C;
  } else {
    in.profile = ComputeProfile::explicit_durations(s.fwd_ms, s.bwd_ms,
                                                    s.recompute_ms);
  }
  in.pipelines_per_cell = s.pipelines_per_cell;
  in.tp_degree = s.tp_degree;
  if (s.d_max > 0) in.d_max = s.d_max;
  for (int k = 0; k < s.n_order; ++k)
    in.dc_order.push_back(dc_name(s.dc_order[k]));
  in.policy = kPolicies[s.policy];
  in.sched.recompute = s.recompute != 0;
  in.sched.multi_conn = s.multi_conn != 0;
  in.sched.n_connections = s.n_connections;
  if (s.mem_limit > 0) in.sched.mem_limit = s.mem_limit;
  return in;
}

ComputeProfile resolved_profile(const SelectionInput& in) {
  if (in.profile.ratio_C.has_value())
    return ComputeProfile::from_ratio(*in.profile.ratio_C, in.model,
                                      in.topo.wan);
  return in.profile;
}

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  g_err.clear();
  try {
    fn();
    return GPB_OK;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return GPB_CONFIG_ERROR;
  } catch (const InsufficientGpus& e) {
    g_err = e.what();
    return GPB_INFEASIBLE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GPB_ERROR;
  }
}

struct RefTask {
  int32_t gpu, cell, pipeline, kind, microbatch, stage;
  int64_t start, end;
};

Timeline timeline_of(const gpb_topology* topos, const gpb_scenario& s, int d,
                     int replay, ParallelismPlan* plan_out,
                     SelectionInput* in_out) {
  SelectionInput in = to_input(topos, s);
  ParallelismPlan plan = build_plan(in.topo, in.model, d, in.pipelines_per_cell,
                                    in.dc_order, in.tp_degree);
  ComputeProfile prof = resolved_profile(in);
  Timeline tl;
  if (replay) {
    tl = run(plan, in.policy, in.model, prof, in.topo, in.sched, false);
  } else {
    tl = schedule_for_policy(in.policy, plan, in.model, prof, in.topo,
                             in.sched);
  }
  if (plan_out) *plan_out = plan;
  if (in_out) *in_out = in;
  return tl;
}

PrefillModel to_pm(const gpb_prefill_model* p) {
  PrefillModel pm;
  pm.saturation_ms = p->saturation_ms;
  pm.max_tokens = p->max_tokens;
  pm.stage_bw = p->stage_bw;
  pm.boundary_latency_ms = p->boundary_latency_ms;
  pm.guard_ms = p->guard_ms;
  pm.memory_budget_bytes = p->memory_budget_bytes;
  pm.inference_layers = p->inference_layers;
  pm.inference_hidden = p->inference_hidden;
  pm.inference_params_per_layer = p->inference_params_per_layer;
  pm.bytes_per_element = p->bytes_per_element;
  return pm;
}

uint64_t fnv_mix(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xffu;
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

double ref_single_tcp_bandwidth(const gpb_topology* topo, double lat) {
  ClusterTopology t = to_topo(*topo);
  return single_tcp_bandwidth(lat, t.wan);
}

// select() for one scenario; rows[d-1] filled for d = 1..n.
int ref_select(const gpb_topology* topos, const gpb_scenario* sc,
               gpb_row* rows, int32_t cap, int32_t* n_rows, int32_t* chosen_d,
               int64_t* gpus_used) {
  return guarded([&] {
    SelectionInput in = to_input(topos, *sc);
    SelectionReport rep = select(in);
    *n_rows = static_cast<int32_t>(rep.rows.size());
    *chosen_d = rep.chosen_d;
    *gpus_used = rep.gpus_used;
    for (size_t i = 0; i < rep.rows.size() && static_cast<int>(i) < cap; ++i) {
      const SelectionRow& r = rep.rows[i];
      gpb_row& o = rows[i];
      std::memset(&o, 0, sizeof o);
      o.pp_time_ms = r.pp_time_ms;
      o.allreduce_time_ms = r.allreduce_time_ms;
      o.total_time_ms = r.total_time_ms;
      o.throughput = r.throughput;
      o.d = r.d;
      o.feasible = r.feasible;
      o.chosen = r.d == rep.chosen_d;
      for (const auto& [dc, n] : r.partitions) {
        int idx = std::stoi(dc.substr(2));
        o.partitions[idx] = static_cast<int16_t>(n);
      }
    }
  });
}

// whatif() over many scenarios (used as the timed CPU baseline): returns the
// number of rows and a checksum of chosen flags.
int ref_whatif_count(const gpb_topology* topos, const gpb_scenario* scens,
                     int32_t n_scen, int64_t* n_rows, int64_t* n_chosen) {
  return guarded([&] {
    std::vector<WhatIfScenario> v;
    v.reserve(n_scen);
    for (int i = 0; i < n_scen; ++i)
      v.push_back({"s" + std::to_string(i), to_input(topos, scens[i])});
    std::vector<WhatIfRow> rows = whatif(v);
    int64_t c = 0;
    for (const auto& r : rows) c += r.chosen ? 1 : 0;
    *n_rows = static_cast<int64_t>(rows.size());
    *n_chosen = c;
  });
}

// Timeline tasks of one (scenario, D) row. replay=0: schedule_for_policy;
// replay=1: run() (engine replay, the bubbletea path).
int ref_timeline(const gpb_topology* topos, const gpb_scenario* sc, int32_t d,
                 int32_t replay, RefTask* out, int64_t cap, int64_t* n,
                 int64_t* makespan) {
  return guarded([&] {
    Timeline tl = timeline_of(topos, *sc, d, replay, nullptr, nullptr);
    *n = static_cast<int64_t>(tl.tasks.size());
    *makespan = tl.makespan;
    for (size_t i = 0; i < tl.tasks.size() && static_cast<int64_t>(i) < cap;
         ++i) {
      const ScheduledTask& t = tl.tasks[i];
      out[i] = {t.gpu_id, t.cell_id, t.pipeline_id, static_cast<int32_t>(t.kind),
                t.microbatch, t.stage, t.start, t.end};
    }
  });
}

// report() on the run() timeline: mean utilization with horizon = makespan.
int ref_utilization(const gpb_topology* topos, const gpb_scenario* sc,
                    int32_t d, int32_t replay, double* util) {
  return guarded([&] {
    Timeline tl = timeline_of(topos, *sc, d, replay, nullptr, nullptr);
    *util = report(tl).mean_utilization;
  });
}

// report() on the run() timeline of every row d = 1..n of one scenario:
// mean utilization (metrics.cpp:39-54) and makespan (schedule.cpp:42-44);
// infeasible rows (InsufficientGpus) get 0 / 0 like gpb_row.
int ref_report_rows(const gpb_topology* topos, const gpb_scenario* sc,
                    int32_t n, double* util, int64_t* makespan) {
  return guarded([&] {
    for (int d = 1; d <= n; ++d) {
      util[d - 1] = 0.0;
      makespan[d - 1] = 0;
      try {
        Timeline tl = timeline_of(topos, *sc, d, 1, nullptr, nullptr);
        util[d - 1] = report(tl).mean_utilization;
        makespan[d - 1] = tl.makespan;
      } catch (const InsufficientGpus&) {
      }
    }
  });
}

// append_allreduce (scheduler.cpp:613-650) on the schedule of row d: per
// stage the start and duration of its all-reduce task (cell 0, pipeline 0).
int ref_allreduce_tail(const gpb_topology* topos, const gpb_scenario* sc, int32_t d,
                       int64_t* start, int64_t* dur, int32_t cap, int32_t* n_stages) {
  return guarded([&] {
    SelectionInput in = to_input(topos, *sc);
    ParallelismPlan plan = build_plan(in.topo, in.model, d, in.pipelines_per_cell,
                                      in.dc_order, in.tp_degree);
    ComputeProfile prof = resolved_profile(in);
    Schedule sched = schedule_for_policy(in.policy, plan, in.model, prof, in.topo, in.sched);
    sched = append_allreduce(sched, plan, in.model, in.topo);
    const int S = plan.num_stages();
    *n_stages = S;
    for (const ScheduledTask& t : sched.tasks)
      if (t.kind == TaskKind::AllReduce && t.cell_id == 0 && t.pipeline_id == 0 &&
          t.stage < cap) {
        start[t.stage] = t.start;
        dur[t.stage] = t.end - t.start;
      }
  });
}

int ref_bubbles(const gpb_topology* topos, const gpb_scenario* sc, int32_t d,
                int64_t horizon, gpb_bubble* out, int64_t cap, int64_t* n) {
  return guarded([&] {
    Timeline tl = timeline_of(topos, *sc, d, 1, nullptr, nullptr);
    TimeNs h = horizon > 0 ? horizon : tl.makespan;
    std::vector<Bubble> b = extract_bubbles(tl, h);
    *n = static_cast<int64_t>(b.size());
    for (size_t i = 0; i < b.size() && static_cast<int64_t>(i) < cap; ++i)
      out[i] = {b[i].gpu_id, 0, b[i].start, b[i].end};
  });
}

static std::vector<PrefillRequest> to_reqs(const gpb_request* r, int64_t n) {
  std::vector<PrefillRequest> v;
  v.reserve(n);
  for (int64_t i = 0; i < n; ++i)
    v.push_back({r[i].id, r[i].arrival_ms, r[i].tokens, "default"});
  return v;
}

int ref_pack_prefills(const gpb_topology* topos, const gpb_scenario* sc,
                      int32_t d, const gpb_request* reqs, int64_t n_req,
                      const gpb_prefill_model* pmp, int64_t horizon,
                      gpb_pack_summary* sum, gpb_placement* pl) {
  return guarded([&] {
    ParallelismPlan plan;
    Timeline tl = timeline_of(topos, *sc, d, 1, &plan, nullptr);
    TimeNs h = horizon > 0 ? horizon : tl.makespan;
    PrefillModel pm = to_pm(pmp);
    auto pipes = build_prefill_pipelines(plan, pm);
    std::vector<PrefillRequest> rq = to_reqs(reqs, n_req);
    PlacementResult res = schedule_prefills(tl, rq, pipes, pm, h);
    std::map<int, const PrefillPlacement*> by_id;
    for (const auto& a : res.accepted) by_id[a.request.id] = &a;
    uint64_t hash = 1469598103934665603ull;
    for (const auto& a : res.accepted) {
      hash = fnv_mix(hash, static_cast<uint64_t>(a.request.id));
      hash = fnv_mix(hash, static_cast<uint64_t>(a.pipeline_index));
      hash = fnv_mix(hash, static_cast<uint64_t>(a.stage_intervals.front().start));
    }
    sum->utilization_before = utilization(tl, h);
    sum->utilization_after = utilization(res.augmented, h);
    sum->accepted = static_cast<int64_t>(res.accepted.size());
    sum->rejected = static_cast<int64_t>(res.rejected.size());
    sum->horizon_ns = h;
    sum->placement_hash = hash;
    if (pl) {
      // Requests are identified by position in the trace (ids may repeat).
      size_t ai = 0;
      for (int64_t i = 0; i < n_req; ++i) {
        gpb_placement& o = pl[i];
        if (ai < res.accepted.size() &&
            res.accepted[ai].request.id == reqs[i].id &&
            res.accepted[ai].request.arrival_ms == reqs[i].arrival_ms &&
            res.accepted[ai].request.tokens == reqs[i].tokens) {
          const PrefillPlacement& a = res.accepted[ai++];
          o.start_ns = a.stage_intervals.front().start;
          o.ttft_overhead_ms = a.ttft_overhead_ms;
          o.accepted = 1;
          o.pipeline = a.pipeline_index;
        } else {
          o.start_ns = -1;
          o.ttft_overhead_ms = 0;
          o.accepted = 0;
          o.pipeline = -1;
        }
      }
    }
  });
}

int ref_synthetic_requests(int32_t count, uint32_t seed, double horizon_ms,
                           const gpb_prefill_model* pmp, gpb_request* out) {
  return guarded([&] {
    auto v = synthetic_requests(count, seed, horizon_ms, to_pm(pmp));
    for (size_t i = 0; i < v.size(); ++i)
      out[i] = {v[i].id, v[i].tokens, v[i].arrival_ms};
  });
}

int ref_saturating_requests(const gpb_topology* topos, const gpb_scenario* sc,
                            int32_t d, const gpb_prefill_model* pmp,
                            int64_t horizon, gpb_request* out, int64_t cap,
                            int64_t* n) {
  return guarded([&] {
    ParallelismPlan plan;
    Timeline tl = timeline_of(topos, *sc, d, 1, &plan, nullptr);
    TimeNs h = horizon > 0 ? horizon : tl.makespan;
    PrefillModel pm = to_pm(pmp);
    auto pipes = build_prefill_pipelines(plan, pm);
    auto v = saturating_requests(tl, pipes, pm, h);
    *n = static_cast<int64_t>(v.size());
    for (size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i)
      out[i] = {v[i].id, v[i].tokens, v[i].arrival_ms};
  });
}

}  // extern "C"
