// capi_session.cpp — the session-level C ABI (include/geopipe.h), a drop-in
// for the reference's libgeopipe.so (geopipe.h:26-60, capi.cpp:64-160).
//
// Host work only: parse the JSON experiment description (config.cpp:111-330
// semantics: same keys, defaults, validation and field paths), expand
// scenarios by JSON merge-patch (config.cpp:282-312), apply overrides
// (runner.cpp:45-70), hand every plan evaluation to the batch ABI
// (include/geopipe_batch.h -> sm_100a kernels) and write the artifacts in the
// reference's byte formats (export.cpp). Timelines for simulate/trace/
// bubbletea come from the device (gpb_timeline_arrays) and are expanded here
// into task/transfer records for the exports.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include <nlohmann/json.hpp>

#include <cuda_runtime.h>

#include "../../include/geopipe.h"
#include "../../include/geopipe_batch.h"

namespace {

using nlohmann::json;

// ------------------------------------------------------------ errors

struct ConfigError : std::runtime_error {
  ConfigError(const std::string& path, const std::string& msg)
      : std::runtime_error(path.empty() ? msg : path + ": " + msg) {}
};
struct Infeasible : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Internal : std::runtime_error {
  using std::runtime_error::runtime_error;
};

long long ms_to_ns(double ms) { return std::llround(ms * 1e6); }  // base.h:15-17
double ns_to_ms(long long ns) { return static_cast<double>(ns) / 1e6; }
double gbps(double g) { return g * 125000.0; }
double mbps(double m) { return m * 125.0; }

// --------------------------------------------------------- data model

struct Dc {
  std::string id;
  int gpu_count = 0;
  double intra_bw = 0.0;
  double intra_lat = 0.0;
};

struct Topo {
  std::vector<Dc> dcs;
  std::map<std::pair<std::string, std::string>, double> lat;
  double cap = 625000.0;
  std::vector<std::pair<double, double>> tcp;

  int index(const std::string& id) const {
    for (size_t i = 0; i < dcs.size(); ++i)
      if (dcs[i].id == id) return static_cast<int>(i);
    throw ConfigError("datacenters", "unknown datacenter id " + id);
  }
  static std::pair<std::string, std::string> key(const std::string& a, const std::string& b) {
    return a <= b ? std::make_pair(a, b) : std::make_pair(b, a);
  }
  double latency(int a, int b) const {
    if (a == b) return 0.0;
    auto it = lat.find(key(dcs[a].id, dcs[b].id));
    if (it == lat.end())
      throw ConfigError("wan.latency_ms", "missing latency for pair " + dcs[a].id + "|" + dcs[b].id);
    return it->second;
  }
};

struct Model {
  int num_layers = 1;
  long long hidden = 1, seq_len = 1, microbatch = 1;
  int M = 1;
  double params_per_layer = 0.0;
  int bpe = 2;
  int lpp = 1;
  int partitions() const { return (num_layers + lpp - 1) / lpp; }
  double ppl() const {
    return params_per_layer > 0 ? params_per_layer : 12.0 * (double)hidden * (double)hidden;
  }
  long long act_bytes() const { return microbatch * seq_len * hidden * bpe; }
};

struct Profile {
  double fwd = 0, bwd = 0, rec = 0;
  double ratio = 0;  // > 0: from_ratio
};

struct Sched {
  bool recompute = true, multi_conn = true;
  int n_conns = 32;
  std::optional<int> mem_limit;
};

struct RunConfig {
  Topo topo;
  Model model;
  Profile profile;
  int dp_cells = 1, C = 1, tp = 1;
  std::vector<std::string> dc_order;
  std::string policy = "atlas";
  bool with_allreduce = false;
  std::optional<std::string> reference_policy;
  Sched sched;
  unsigned seed = 42;
  std::optional<double> horizon_ms;
  std::optional<int> select_d_max;
  int select_C = 0, select_tp = 0;
  std::vector<std::string> select_dc_order;
  std::string select_policy = "atlas";
  gpb_prefill_model prefill;
  std::optional<std::string> requests_csv;
  std::optional<int> synthetic_count;
  bool saturating = false;
};

struct Overrides {
  std::optional<std::string> policy;
  std::optional<unsigned> seed;
  std::optional<bool> multi_conn, recompute;
  std::optional<int> mem_limit;
  std::optional<double> horizon_ms;
};

const std::set<std::string>& policies() {
  static const std::set<std::string> p{"gpipe", "1f1b", "varuna", "atlas"};
  return p;
}

int policy_code(const std::string& p) {
  if (p == "gpipe") return GPB_GPIPE;
  if (p == "1f1b") return GPB_1F1B;
  if (p == "varuna") return GPB_VARUNA;
  if (p == "atlas") return GPB_ATLAS;
  throw ConfigError("policy", "unknown policy " + p);
}

// ------------------------------------------------------- config parse

long long require_int(const json& node, const std::string& path, long long min_value) {
  if (!node.is_number_integer()) throw ConfigError(path, "required integer");
  long long v = node.get<long long>();
  if (v < min_value) throw ConfigError(path, "must be >= " + std::to_string(min_value));
  return v;
}

double require_number(const json& node, const std::string& path, bool positive) {
  if (!node.is_number()) throw ConfigError(path, "required number");
  double v = node.get<double>();
  if (positive && !(v > 0)) throw ConfigError(path, "must be > 0");
  if (!positive && v < 0) throw ConfigError(path, "must be >= 0");
  return v;
}

// topology (topology.cpp:81-190 semantics)
Topo parse_topology(const json& doc) {
  Topo t;
  if (!doc.contains("datacenters") || !doc["datacenters"].is_array() || doc["datacenters"].empty())
    throw ConfigError("datacenters", "required non-empty list");
  std::set<std::string> seen;
  for (size_t i = 0; i < doc["datacenters"].size(); ++i) {
    const json& d = doc["datacenters"][i];
    const std::string path = "datacenters[" + std::to_string(i) + "]";
    Dc dc;
    if (!d.contains("id") || !d["id"].is_string()) throw ConfigError(path + ".id", "required string");
    dc.id = d["id"].get<std::string>();
    if (!seen.insert(dc.id).second)
      throw ConfigError(path + ".id", "duplicate datacenter id " + dc.id);
    if (!d.contains("gpu_count") || !d["gpu_count"].is_number_integer() ||
        d["gpu_count"].get<long long>() < 1)
      throw ConfigError(path + ".gpu_count", "required integer >= 1");
    dc.gpu_count = d["gpu_count"].get<int>();
    double intra = d.value("intra_bw_gbps", 100.0);
    if (!(intra > 0)) throw ConfigError(path + ".intra_bw_gbps", "must be > 0");
    dc.intra_bw = gbps(intra);
    dc.intra_lat = d.value("intra_latency_ms", 0.0);
    if (dc.intra_lat < 0) throw ConfigError(path + ".intra_latency_ms", "must be >= 0");
    t.dcs.push_back(dc);
  }
  const json wan = doc.value("wan", json::object());
  double cap = wan.value("pair_bw_cap_gbps", 5.0);
  if (!(cap > 0)) throw ConfigError("wan.pair_bw_cap_gbps", "must be > 0");
  t.cap = gbps(cap);
  if (wan.contains("tcp_table")) {
    if (!wan["tcp_table"].is_array())
      throw ConfigError("wan.tcp_table", "must be a list of [ms, mbps] pairs");
    for (size_t i = 0; i < wan["tcp_table"].size(); ++i) {
      const json& row = wan["tcp_table"][i];
      if (!row.is_array() || row.size() != 2 || !row[0].is_number() || !row[1].is_number())
        throw ConfigError("wan.tcp_table[" + std::to_string(i) + "]",
                          "must be a [latency_ms, mbps] pair");
      t.tcp.push_back({row[0].get<double>(), mbps(row[1].get<double>())});
    }
  } else {
    t.tcp = {{10.0, mbps(1220.0)}, {20.0, mbps(600.0)}, {30.0, mbps(396.0)}, {40.0, mbps(293.0)}};
  }
  if (t.tcp.empty()) throw ConfigError("wan.tcp_table", "tcp_table must be non-empty");
  for (size_t i = 0; i < t.tcp.size(); ++i) {
    const std::string p = "wan.tcp_table[" + std::to_string(i) + "]";
    if (t.tcp[i].first <= 0 || t.tcp[i].second <= 0)
      throw ConfigError(p, "latency and bandwidth must be positive");
    if (i > 0 && t.tcp[i].first <= t.tcp[i - 1].first)
      throw ConfigError(p, "latencies must be strictly increasing");
    if (i > 0 && t.tcp[i].second >= t.tcp[i - 1].second)
      throw ConfigError(p, "bandwidths must be strictly decreasing");
  }
  const json lat = wan.value("latency_ms", json::object());
  if (!lat.is_object()) throw ConfigError("wan.latency_ms", "must be a map of \"a|b\" -> ms");
  for (auto it = lat.begin(); it != lat.end(); ++it) {
    const std::string key = it.key();
    const auto bar = key.find('|');
    if (bar == std::string::npos)
      throw ConfigError("wan.latency_ms." + key, "key must be of the form \"a|b\"");
    const std::string a = key.substr(0, bar), b = key.substr(bar + 1);
    if (!seen.count(a) || !seen.count(b))
      throw ConfigError("wan.latency_ms." + key, "unknown datacenter in pair");
    if (!it.value().is_number())
      throw ConfigError("wan.latency_ms." + key, "latency must be a number");
    const double v = it.value().get<double>();
    if (a == b) {
      if (v != 0.0) throw ConfigError("wan.latency_ms." + key, "self latency must be zero");
      continue;
    }
    if (v < 0) throw ConfigError("wan.latency_ms." + key, "must be >= 0");
    const auto k = Topo::key(a, b);
    auto ex = t.lat.find(k);
    if (ex != t.lat.end() && ex->second != v)
      throw ConfigError("wan.latency_ms." + key, "asymmetric latency for pair " + a + "|" + b);
    t.lat[k] = v;
  }
  for (size_t i = 0; i < t.dcs.size(); ++i)
    for (size_t j = i + 1; j < t.dcs.size(); ++j) {
      const auto k = Topo::key(t.dcs[i].id, t.dcs[j].id);
      if (!t.lat.count(k))
        throw ConfigError("wan.latency_ms", "missing latency for pair " + k.first + "|" + k.second);
    }
  return t;
}

std::vector<std::string> parse_dc_order(const json& node, const std::string& path,
                                        const Topo& topo) {
  if (!node.is_array()) throw ConfigError(path, "must be a list of DC ids");
  std::vector<std::string> order;
  for (size_t i = 0; i < node.size(); ++i) {
    if (!node[i].is_string())
      throw ConfigError(path + "[" + std::to_string(i) + "]", "must be a DC id string");
    order.push_back(node[i].get<std::string>());
    topo.index(order.back());
  }
  return order;
}

// run config (config.cpp:111-258 semantics)
RunConfig parse_run_config(const json& doc) {
  RunConfig c;
  c.topo = parse_topology(doc);
  if (!doc.contains("model") || !doc["model"].is_object())
    throw ConfigError("model", "required object");
  const json& m = doc["model"];
  c.model.num_layers = (int)require_int(m.value("num_layers", json(1)), "model.num_layers", 1);
  c.model.hidden = require_int(m.value("hidden", json(1)), "model.hidden", 1);
  c.model.seq_len = require_int(m.value("seq_len", json(1)), "model.seq_len", 1);
  c.model.microbatch = require_int(m.value("microbatch", json(1)), "model.microbatch", 1);
  c.model.M = (int)require_int(m.value("num_microbatches", json(1)), "model.num_microbatches", 1);
  if (m.contains("params_per_layer"))
    c.model.params_per_layer = require_number(m["params_per_layer"], "model.params_per_layer", false);
  c.model.bpe = (int)require_int(m.value("bytes_per_element", json(2)), "model.bytes_per_element", 1);
  c.model.lpp = (int)require_int(m.value("layers_per_partition", json(1)),
                                 "model.layers_per_partition", 1);
  if (!doc.contains("compute") || !doc["compute"].is_object())
    throw ConfigError("compute", "required object");
  const json& cp = doc["compute"];
  const bool has_ratio = cp.contains("comm_compute_ratio"), has_explicit = cp.contains("fwd_ms");
  if (has_ratio == has_explicit)
    throw ConfigError("compute", "give either fwd_ms/bwd_ms/recompute_ms or comm_compute_ratio, not both");
  if (has_ratio) {
    c.profile.ratio = require_number(cp["comm_compute_ratio"], "compute.comm_compute_ratio", true);
    const double comm = (double)c.model.act_bytes() / c.topo.cap;  // from_ratio
    c.profile.fwd = comm / c.profile.ratio;
    c.profile.bwd = 2.0 * c.profile.fwd;
    c.profile.rec = c.profile.fwd;
  } else {
    c.profile.fwd = require_number(cp["fwd_ms"], "compute.fwd_ms", true);
    if (!cp.contains("bwd_ms")) throw ConfigError("compute.bwd_ms", "required");
    c.profile.bwd = require_number(cp["bwd_ms"], "compute.bwd_ms", true);
    c.profile.rec = require_number(cp.value("recompute_ms", json(c.profile.fwd)),
                                   "compute.recompute_ms", false);
    if (c.profile.fwd <= 0 || c.profile.bwd <= 0 || c.profile.rec < 0)
      throw ConfigError("compute", "durations must be positive");
  }
  const json par = doc.value("parallelism", json::object());
  if (!par.is_object()) throw ConfigError("parallelism", "must be an object");
  c.dp_cells = (int)require_int(par.value("dp_cells", json(1)), "parallelism.dp_cells", 1);
  c.C = (int)require_int(par.value("pipelines_per_cell", json(1)), "parallelism.pipelines_per_cell", 1);
  c.tp = (int)require_int(par.value("tp_degree", json(1)), "parallelism.tp_degree", 1);
  if (par.contains("dc_order")) c.dc_order = parse_dc_order(par["dc_order"], "parallelism.dc_order", c.topo);
  const json sim = doc.value("simulate", json::object());
  if (!sim.is_object()) throw ConfigError("simulate", "must be an object");
  c.policy = sim.value("policy", "atlas");
  if (!policies().count(c.policy))
    throw ConfigError("simulate.policy", "must be one of gpipe, 1f1b, varuna, atlas");
  if (sim.contains("allreduce") && !sim["allreduce"].is_boolean())
    throw ConfigError("simulate.allreduce", "must be a boolean");
  c.with_allreduce = sim.value("allreduce", false);
  if (sim.contains("reference_policy")) {
    const std::string ref = sim["reference_policy"].get<std::string>();
    if (!policies().count(ref))
      throw ConfigError("simulate.reference_policy", "must be one of gpipe, 1f1b, varuna, atlas");
    c.reference_policy = ref;
  }
  if (sim.contains("multi_conn") && !sim["multi_conn"].is_boolean())
    throw ConfigError("simulate.multi_conn", "must be a boolean");
  c.sched.multi_conn = sim.value("multi_conn", true);
  if (sim.contains("recompute") && !sim["recompute"].is_boolean())
    throw ConfigError("simulate.recompute", "must be a boolean");
  c.sched.recompute = sim.value("recompute", true);
  c.sched.n_conns = (int)require_int(sim.value("n_connections", json(32)), "simulate.n_connections", 1);
  if (sim.contains("mem_limit") && !sim["mem_limit"].is_null())
    c.sched.mem_limit = (int)require_int(sim["mem_limit"], "simulate.mem_limit", 1);
  c.seed = (unsigned)require_int(doc.value("seed", json(42)), "seed", 0);
  if (doc.contains("horizon_ms") && !doc["horizon_ms"].is_null())
    c.horizon_ms = require_number(doc["horizon_ms"], "horizon_ms", true);
  const json sel = doc.value("select", json::object());
  if (!sel.is_object()) throw ConfigError("select", "must be an object");
  if (sel.contains("d_max") && !sel["d_max"].is_null())
    c.select_d_max = (int)require_int(sel["d_max"], "select.d_max", 1);
  if (sel.contains("pipelines_per_cell"))
    c.select_C = (int)require_int(sel["pipelines_per_cell"], "select.pipelines_per_cell", 1);
  if (sel.contains("tp_degree")) c.select_tp = (int)require_int(sel["tp_degree"], "select.tp_degree", 1);
  if (sel.contains("dc_order")) c.select_dc_order = parse_dc_order(sel["dc_order"], "select.dc_order", c.topo);
  c.select_policy = sel.value("policy", "atlas");
  if (!policies().count(c.select_policy))
    throw ConfigError("select.policy", "must be one of gpipe, 1f1b, varuna, atlas");
  const json pre = doc.value("prefill", json::object());
  if (!pre.is_object()) throw ConfigError("prefill", "must be an object");
  gpb_prefill_model& p = c.prefill;
  p.saturation_ms = require_number(pre.value("saturation_ms", json(300.0)), "prefill.saturation_ms", true);
  p.max_tokens = (int)require_int(pre.value("max_tokens", json(8192)), "prefill.max_tokens", 1);
  p.stage_bw = require_number(pre.value("stage_bw_bytes_per_ms", json(25000000.0)),
                              "prefill.stage_bw_bytes_per_ms", true);
  p.boundary_latency_ms = require_number(pre.value("boundary_latency_ms", json(0.0)),
                                         "prefill.boundary_latency_ms", false);
  p.guard_ms = require_number(pre.value("guard_ms", json(0.0)), "prefill.guard_ms", false);
  p.memory_budget_bytes = require_int(pre.value("memory_budget_bytes", json(1073741824LL)),
                                      "prefill.memory_budget_bytes", 1);
  p.inference_layers = (int)require_int(pre.value("inference_layers", json(8)),
                                        "prefill.inference_layers", 1);
  p.inference_hidden = require_int(pre.value("inference_hidden", json(1024)),
                                   "prefill.inference_hidden", 1);
  p.inference_params_per_layer = 0.0;
  if (pre.contains("inference_params_per_layer"))
    p.inference_params_per_layer = require_number(pre["inference_params_per_layer"],
                                                  "prefill.inference_params_per_layer", false);
  p.bytes_per_element = (int)require_int(pre.value("bytes_per_element", json(2)),
                                         "prefill.bytes_per_element", 1);
  p.pad_ = 0;
  if (pre.contains("requests_csv")) {
    if (!pre["requests_csv"].is_string()) throw ConfigError("prefill.requests_csv", "must be a path string");
    c.requests_csv = pre["requests_csv"].get<std::string>();
  }
  if (pre.contains("synthetic")) {
    const json& syn = pre["synthetic"];
    if (!syn.is_object() || !syn.contains("count"))
      throw ConfigError("prefill.synthetic", "must be an object with a count");
    c.synthetic_count = (int)require_int(syn["count"], "prefill.synthetic.count", 0);
    if (syn.contains("seed")) c.seed = (unsigned)require_int(syn["seed"], "prefill.synthetic.seed", 0);
  }
  if (pre.contains("saturating") && !pre["saturating"].is_boolean())
    throw ConfigError("prefill.saturating", "must be a boolean");
  c.saturating = pre.value("saturating", false);
  if (c.requests_csv && (c.synthetic_count || c.saturating))
    throw ConfigError("prefill", "give only one request source");
  if (c.synthetic_count && c.saturating) throw ConfigError("prefill", "give only one request source");
  return c;
}

json parse_document(const std::string& text) {
  json doc;
  try {
    doc = json::parse(text);
  } catch (const json::parse_error& e) {
    throw ConfigError("", std::string("invalid JSON: ") + e.what());
  }
  if (!doc.is_object()) throw ConfigError("", "top level must be an object");
  return doc;
}

std::vector<std::pair<std::string, RunConfig>> expand_scenarios(const std::string& text) {
  json doc = parse_document(text);
  json base = doc;
  base.erase("scenarios");
  std::vector<std::pair<std::string, RunConfig>> out;
  if (!doc.contains("scenarios")) {
    out.emplace_back("base", parse_run_config(base));
    return out;
  }
  if (!doc["scenarios"].is_array() || doc["scenarios"].empty())
    throw ConfigError("scenarios", "must be a non-empty list");
  for (size_t i = 0; i < doc["scenarios"].size(); ++i) {
    const json& s = doc["scenarios"][i];
    const std::string path = "scenarios[" + std::to_string(i) + "]";
    if (!s.is_object()) throw ConfigError(path, "must be an object");
    std::string name = s.value("name", "s" + std::to_string(i));
    if (!s.contains("patch") || !s["patch"].is_object()) throw ConfigError(path + ".patch", "required object");
    json merged = base;
    merged.merge_patch(s["patch"]);
    try {
      out.emplace_back(name, parse_run_config(merged));
    } catch (const ConfigError& e) {
      throw ConfigError(path, e.what());
    }
  }
  return out;
}

void apply_overrides(RunConfig& c, const Overrides& o) {
  if (o.policy) {
    if (!policies().count(*o.policy)) throw ConfigError("policy", "must be one of gpipe, 1f1b, varuna, atlas");
    c.policy = *o.policy;
    c.select_policy = *o.policy;
  }
  if (o.seed) c.seed = *o.seed;
  if (o.multi_conn) c.sched.multi_conn = *o.multi_conn;
  if (o.recompute) c.sched.recompute = *o.recompute;
  if (o.mem_limit) {
    if (*o.mem_limit < 1) throw ConfigError("mem_limit", "must be >= 1");
    c.sched.mem_limit = *o.mem_limit;
  }
  if (o.horizon_ms) {
    if (!(*o.horizon_ms > 0)) throw ConfigError("horizon", "must be > 0");
    c.horizon_ms = *o.horizon_ms;
  }
}

std::string read_text_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw ConfigError("config", "cannot open " + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

void write_text_file(const std::string& path, const std::string& content) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw ConfigError("out", "cannot open " + path + " for writing");
  f << content;
  if (!f) throw ConfigError("out", "failed writing " + path);
}

std::string prepare_out_dir(const std::string& out_dir) {
  if (out_dir.empty()) throw ConfigError("out", "output directory required");
  std::error_code ec;
  std::filesystem::create_directories(out_dir, ec);
  if (ec) throw ConfigError("out", "cannot create " + out_dir + ": " + ec.message());
  return out_dir + "/";
}

// --------------------------------------------------- batch conversion

gpb_topology to_gpb(const Topo& t) {
  if (t.dcs.size() > GPB_MAX_DC)
    throw ConfigError("datacenters", "more than 8 datacenters is outside the batch envelope");
  if (t.tcp.size() > GPB_MAX_TCP)
    throw ConfigError("wan.tcp_table", "more than 8 calibration points is outside the batch envelope");
  gpb_topology g;
  std::memset(&g, 0, sizeof g);
  g.n_dc = (int)t.dcs.size();
  for (int i = 0; i < g.n_dc; ++i) {
    g.gpu_count[i] = t.dcs[i].gpu_count;
    g.intra_bw[i] = t.dcs[i].intra_bw;
    for (int j = 0; j < g.n_dc; ++j) g.latency_ms[i][j] = t.latency(i, j);
  }
  g.pair_bw_cap = t.cap;
  g.n_tcp = (int)t.tcp.size();
  for (size_t i = 0; i < t.tcp.size(); ++i) {
    g.tcp_latency_ms[i] = t.tcp[i].first;
    g.tcp_bw[i] = t.tcp[i].second;
  }
  return g;
}

gpb_scenario base_scenario(const RunConfig& c) {
  gpb_scenario s;
  std::memset(&s, 0, sizeof s);
  s.num_layers = c.model.num_layers;
  s.layers_per_partition = c.model.lpp;
  s.num_microbatches = c.model.M;
  s.bytes_per_element = c.model.bpe;
  s.hidden = c.model.hidden;
  s.seq_len = c.model.seq_len;
  s.microbatch = c.model.microbatch;
  s.params_per_layer = c.model.params_per_layer;
  s.fwd_ms = c.profile.fwd;
  s.bwd_ms = c.profile.bwd;
  s.recompute_ms = c.profile.rec;
  s.ratio_C = c.profile.ratio;
  s.recompute = c.sched.recompute;
  s.multi_conn = c.sched.multi_conn;
  s.n_connections = c.sched.n_conns;
  s.mem_limit = c.sched.mem_limit.value_or(0);
  return s;
}

void set_order(gpb_scenario& s, const Topo& t, const std::vector<std::string>& order) {
  if (order.size() > GPB_MAX_DC) throw ConfigError("dc_order", "too many datacenters");
  s.n_order = (int)order.size();
  for (size_t i = 0; i < order.size(); ++i) s.dc_order[i] = t.index(order[i]);
}

// selection_input (config.cpp:314-330)
gpb_scenario selection_scenario(const RunConfig& c, int topo_index) {
  gpb_scenario s = base_scenario(c);
  s.topology = topo_index;
  s.policy = policy_code(c.select_policy);
  s.pipelines_per_cell = c.select_C > 0 ? c.select_C : c.C;
  s.tp_degree = c.select_tp > 0 ? c.select_tp : c.tp;
  s.d_max = c.select_d_max.value_or(0);
  set_order(s, c.topo, c.select_dc_order.empty() ? c.dc_order : c.select_dc_order);
  return s;
}

// ------------------------------------------------------------ session

struct Session {
  std::string config_text;
  bool config_loaded = false;
  Overrides ov;
  std::string last_error;
  std::string selection_table;
  gpb_ctx* ctx = nullptr;

  gpb_group* group = nullptr;
  bool group_checked = false;

  gpb_ctx* device() {
    if (!ctx) {
      const char* env = std::getenv("GEOPIPE_DEVICE");
      ctx = gpb_create(env ? std::atoi(env) : 0);
      if (!ctx) throw Internal("no CUDA device available for the B200 batch path");
    }
    return ctx;
  }
  // The devices a whatif / select_dc space is sharded over (gpb_group_*):
  // GEOPIPE_DEVICES="all" or a comma list ("0,1,2,3"); unset = every visible
  // device when there is more than one. nullptr = one device (device()).
  gpb_group* devices() {
    if (group_checked) return group;
    group_checked = true;
    const char* env = std::getenv("GEOPIPE_DEVICES");
    std::vector<int32_t> list;
    if (env && std::string(env) != "all") {
      std::string cur;
      for (const char* q = env;; ++q) {
        if (*q == ',' || *q == 0) {
          if (!cur.empty()) list.push_back(std::atoi(cur.c_str()));
          cur.clear();
          if (*q == 0) break;
        } else {
          cur += *q;
        }
      }
      if (list.size() <= 1) return nullptr;
    } else {
      int n = 0;
      if (cudaGetDeviceCount(&n) != cudaSuccess || n < 2) return nullptr;
    }
    group = gpb_group_create((int32_t)list.size(), list.empty() ? nullptr : list.data());
    if (!group) throw Internal("GEOPIPE_DEVICES: could not open the device group");
    return group;
  }
  void check_group(int rc) {
    if (rc == GPB_OK) return;
    const std::string msg = gpb_group_last_error(group);
    if (rc == GPB_CONFIG_ERROR) throw ConfigError("", msg);
    if (rc == GPB_INFEASIBLE) throw Infeasible(msg);
    throw Internal(msg);
  }
  void check(int rc) {
    if (rc == GPB_OK) return;
    const std::string msg = gpb_last_error(ctx);
    if (rc == GPB_CONFIG_ERROR) throw ConfigError("", msg);
    if (rc == GPB_INFEASIBLE) throw Infeasible(msg);
    throw Internal(msg);
  }
  ~Session() {
    if (group) gpb_group_destroy(group);
    if (ctx) gpb_destroy(ctx);
  }
};

// ----------------------------------------------------------- timelines

enum Kind { kForward = 0, kBackward = 1, kRecompute = 2, kAllReduce = 3, kPrefill = 4 };

struct Task {
  int gpu, cell, pipe, kind, m, stage;
  long long start, end;
};

struct Xfer {
  int cell, pipe, m, boundary, dir;
  long long bytes, start, end, arrival;
  int pooled;
};

struct Timeline {
  std::vector<Task> tasks;
  std::vector<Xfer> xfers;
  long long makespan = 0;
};

struct PlanInfo {  // build_plan's outcome on the host (workload.cpp:57-124)
  int D = 1, C = 1, S = 1, tp = 1;
  std::vector<int> stage_dc;          // [S]
  std::vector<int> gpu;               // [D][C][S] front GPU id
};

PlanInfo host_plan(const RunConfig& c, const gpb_topology& gt, int D, int C, int tp,
                   const std::vector<std::string>& order_ids) {
  PlanInfo p;
  p.D = D;
  p.C = C;
  p.tp = tp;
  p.S = c.model.partitions();
  std::vector<int> order;
  if (!order_ids.empty()) {
    for (const auto& id : order_ids) order.push_back(c.topo.index(id));
  } else {
    for (int i = 0; i < gt.n_dc; ++i) order.push_back(i);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return gt.gpu_count[a] > gt.gpu_count[b]; });
  }
  std::vector<std::pair<int, int>> blocks;  // (dc, count)
  int assigned = 0;
  for (int dc : order) {
    if (assigned >= p.S) break;
    const int take = std::min(p.S - assigned, gt.gpu_count[dc] / (D * C * tp));
    if (take > 0) {
      blocks.push_back({dc, take});
      assigned += take;
    }
  }
  if (assigned < p.S)
    throw Infeasible("plan needs " + std::to_string(p.S) + " stages x " +
                     std::to_string(D * C * tp) + " GPUs but only " + std::to_string(assigned) +
                     " stages fit");
  for (auto [dc, cnt] : blocks)
    for (int k = 0; k < cnt; ++k) p.stage_dc.push_back(dc);
  std::vector<int> base(gt.n_dc, 0), next(gt.n_dc, 0);
  for (int i = 1; i < gt.n_dc; ++i) base[i] = base[i - 1] + gt.gpu_count[i - 1];
  p.gpu.resize((size_t)D * C * p.S);
  for (int cell = 0; cell < D; ++cell)
    for (int pipe = 0; pipe < C; ++pipe)
      for (int s = 0; s < p.S; ++s) {
        const int dc = p.stage_dc[s];
        p.gpu[((size_t)cell * C + pipe) * p.S + s] = base[dc] + next[dc];
        next[dc] += tp;
      }
  return p;
}

void finalize(Timeline& t) {  // finalize_schedule (schedule.cpp:23-45)
  std::sort(t.tasks.begin(), t.tasks.end(), [](const Task& a, const Task& b) {
    return std::tie(a.cell, a.pipe, a.stage, a.start, a.end, a.m) <
           std::tie(b.cell, b.pipe, b.stage, b.start, b.end, b.m);
  });
  std::sort(t.xfers.begin(), t.xfers.end(), [](const Xfer& a, const Xfer& b) {
    return std::tie(a.cell, a.boundary, a.dir, a.start, a.pipe, a.m) <
           std::tie(b.cell, b.boundary, b.dir, b.start, b.pipe, b.m);
  });
  long long mk = 0;
  for (const Task& x : t.tasks) mk = std::max(mk, x.end);
  t.makespan = mk;
}

// Evaluate one (policy, D) plan on the device and expand its timeline.
Timeline device_timeline(Session& se, const RunConfig& c, const std::string& policy, PlanInfo& plan) {
  gpb_ctx* ctx = se.device();
  gpb_topology gt = to_gpb(c.topo);
  gpb_scenario s = base_scenario(c);
  s.policy = policy_code(policy);
  s.pipelines_per_cell = c.C;
  s.tp_degree = c.tp;
  s.d_max = c.dp_cells;
  set_order(s, c.topo, c.dc_order);
  if (s.mem_limit == 0 && c.sched.mem_limit) s.mem_limit = *c.sched.mem_limit;
  plan = host_plan(c, gt, c.dp_cells, c.C, c.tp, c.dc_order);
  int64_t n_rows = 0;
  se.check(gpb_load(ctx, &gt, 1, &s, 1, &n_rows));
  se.check(gpb_evaluate(ctx, 1));
  const int64_t row = c.dp_cells - 1;
  int32_t dims[4];
  int64_t mk = 0;
  se.check(gpb_timeline_arrays(ctx, row, nullptr, nullptr, 0, dims, &mk));
  const int Ce = dims[0], S = dims[1], M = dims[2];
  std::vector<int64_t> fe((size_t)Ce * S * M), ps((size_t)Ce * S * M);
  se.check(gpb_timeline_arrays(ctx, row, fe.data(), ps.data(), (int64_t)fe.size(), dims, &mk));
  // geometry (scheduler.cpp:32-76), host copy for the transfer records
  const long long bytes = c.model.act_bytes();
  const int n_conns = c.sched.multi_conn ? c.sched.n_conns : 1;
  const long long f = ms_to_ns(c.profile.fwd), bw_ns = ms_to_ns(c.profile.bwd),
                  rc = ms_to_ns(c.profile.rec);
  const long long dur = c.sched.recompute ? rc + bw_ns : bw_ns;
  const int C = c.C, D = c.dp_cells, pol = s.policy;
  const bool pooled = pol == GPB_ATLAS;
  std::vector<int> wan(std::max(S - 1, 0), 0);
  std::vector<long long> ser(std::max(S - 1, 0), 0), lat(std::max(S - 1, 0), 0);
  for (int b = 0; b + 1 < S; ++b) {
    const int a = plan.stage_dc[b], z = plan.stage_dc[b + 1];
    if (a == z) continue;
    wan[b] = 1;
    const double l = c.topo.latency(a, z);
    const double single = gpb_single_tcp_bandwidth(&gt, l);
    const double bw = std::min(n_conns * single, gt.pair_bw_cap);
    ser[b] = pooled ? ms_to_ns(bytes / (C * bw)) : ms_to_ns(bytes / bw);
    lat[b] = ms_to_ns(l);
  }
  Timeline t;
  for (int cell = 0; cell < D; ++cell)
    for (int p = 0; p < C; ++p) {
      const int pe = Ce > 1 ? p : 0;
      for (int st = 0; st < S; ++st) {
        const int gpu = plan.gpu[((size_t)cell * C + p) * S + st];
        for (int m = 0; m < M; ++m) {
          const long long e = fe[((size_t)pe * S + st) * M + m];
          const long long q = ps[((size_t)pe * S + st) * M + m];
          t.tasks.push_back({gpu, cell, p, kForward, m, st, e - f, e});
          if (c.sched.recompute) {
            t.tasks.push_back({gpu, cell, p, kRecompute, m, st, q, q + rc});
            t.tasks.push_back({gpu, cell, p, kBackward, m, st, q + rc, q + rc + bw_ns});
          } else {
            t.tasks.push_back({gpu, cell, p, kBackward, m, st, q, q + bw_ns});
          }
        }
      }
      for (int b = 0; b + 1 < S; ++b) {
        if (!wan[b]) continue;
        long long link = 0;  // activation FIFO (m order)
        for (int m = 0; m < M; ++m) {
          const long long e = fe[((size_t)pe * S + b) * M + m];
          const long long st0 = pooled ? e : std::max(e, link);
          const long long occ = st0 + ser[b];
          link = occ;
          t.xfers.push_back({cell, p, m, b, 0, bytes, st0, occ, occ + lat[b], pooled ? C : 1});
        }
        link = 0;  // gradient FIFO in the drain order of stage b+1
        for (int i = 0; i < M; ++i) {
          const int m = pol == GPB_GPIPE ? M - 1 - i : i;
          const long long z = ps[((size_t)pe * S + b + 1) * M + m] + dur;
          const long long st0 = pooled ? z : std::max(z, link);
          const long long occ = st0 + ser[b];
          link = occ;
          t.xfers.push_back({cell, p, m, b, 1, bytes, st0, occ, occ + lat[b], pooled ? C : 1});
        }
      }
    }
  finalize(t);
  return t;
}

// append_allreduce (scheduler.cpp:613-650): the tail's starts and durations
// come from the device (gpb_allreduce_tail on the row device_timeline loaded)
void append_allreduce(Session& se, Timeline& t, const RunConfig& c, const PlanInfo& plan) {
  std::vector<int64_t> start(plan.S), dur(plan.S);
  int32_t n = 0;
  se.check(gpb_allreduce_tail(se.device(), c.dp_cells - 1, start.data(), dur.data(),
                              (int32_t)plan.S, &n));
  if (n != plan.S) throw Internal("all-reduce tail: stage count mismatch");
  for (int s = 0; s < plan.S; ++s)
    for (int cell = 0; cell < plan.D; ++cell)
      for (int p = 0; p < plan.C; ++p)
        t.tasks.push_back({plan.gpu[((size_t)cell * plan.C + p) * plan.S + s], cell, p, kAllReduce,
                           0, s, start[s], start[s] + dur[s]});
  finalize(t);
}

Timeline simulate(Session& se, const RunConfig& c, const std::string& policy, PlanInfo& plan) {
  Timeline t = device_timeline(se, c, policy, plan);
  if (c.with_allreduce) append_allreduce(se, t, c, plan);
  return t;  // run(): the replay reproduces the schedule (test_engine.cpp:17-32)
}

// -------------------------------------------------------------- exports

std::string fixed6(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.6f", v);
  return buf;
}

const char* kind_name(int k) {
  switch (k) {
    case kForward: return "forward";
    case kBackward: return "backward";
    case kRecompute: return "recompute";
    case kAllReduce: return "allreduce";
    case kPrefill: return "prefill";
  }
  return "unknown";
}

const char* kind_letter(int k) {
  switch (k) {
    case kForward: return "F";
    case kBackward: return "B";
    case kRecompute: return "R";
    case kAllReduce: return "AR";
    case kPrefill: return "P";
  }
  return "?";
}

const char* dir_name(int d) { return d == 0 ? "activation_fwd" : "gradient_bwd"; }

std::string chrome_trace(const Timeline& t) {
  json events = json::array();
  std::map<std::tuple<int, int, int, int>, int> link_tid;
  for (const Xfer& x : t.xfers) link_tid.emplace(std::make_tuple(x.cell, x.boundary, x.dir, x.pooled > 1 ? -1 : x.pipe), 0);
  int next_tid = 100000;
  for (auto& kv : link_tid) kv.second = next_tid++;
  std::map<int, std::set<int>> gpus;
  for (const Task& x : t.tasks) gpus[x.cell].insert(x.gpu);
  for (const auto& [cell, set] : gpus)
    for (int gpu : set)
      events.push_back({{"name", "thread_name"}, {"ph", "M"}, {"pid", cell}, {"tid", gpu},
                        {"args", {{"name", "gpu " + std::to_string(gpu)}}}});
  for (const auto& [key, tid] : link_tid) {
    auto [cell, b, dir, lane] = key;
    std::string name = std::string(dir == 0 ? "act" : "grad") + " link b" + std::to_string(b) +
                       (lane < 0 ? std::string(" pooled") : " pipeline " + std::to_string(lane));
    events.push_back({{"name", "thread_name"}, {"ph", "M"}, {"pid", cell}, {"tid", tid},
                      {"args", {{"name", name}}}});
  }
  for (const Task& x : t.tasks) {
    std::string name = kind_letter(x.kind);
    if (x.kind == kAllReduce) name += " s" + std::to_string(x.stage);
    else if (x.kind == kPrefill) name += " r" + std::to_string(x.m) + " s" + std::to_string(x.stage);
    else name += " m" + std::to_string(x.m) + " s" + std::to_string(x.stage);
    events.push_back({{"name", name}, {"cat", kind_name(x.kind)}, {"ph", "X"},
                      {"ts", static_cast<double>(x.start) / 1000.0},
                      {"dur", static_cast<double>(x.end - x.start) / 1000.0},
                      {"pid", x.cell}, {"tid", x.gpu},
                      {"args", {{"pipeline", x.pipe}, {"microbatch", x.m}, {"stage", x.stage}}}});
  }
  for (const Xfer& x : t.xfers) {
    const int tid = link_tid.at(std::make_tuple(x.cell, x.boundary, x.dir, x.pooled > 1 ? -1 : x.pipe));
    std::string name = std::string(x.dir == 0 ? "act" : "grad") + " m" + std::to_string(x.m) +
                       " b" + std::to_string(x.boundary);
    events.push_back({{"name", name}, {"cat", dir_name(x.dir)}, {"ph", "X"},
                      {"ts", static_cast<double>(x.start) / 1000.0},
                      {"dur", static_cast<double>(x.end - x.start) / 1000.0},
                      {"pid", x.cell}, {"tid", tid},
                      {"args", {{"pipeline", x.pipe}, {"microbatch", x.m}, {"boundary", x.boundary},
                                {"bytes", x.bytes}, {"pooled_pipelines", x.pooled},
                                {"arrival_ms", static_cast<double>(x.arrival) / 1e6}}}});
  }
  json doc;
  doc["traceEvents"] = std::move(events);
  doc["displayTimeUnit"] = "ms";
  return doc.dump(2) + "\n";
}

std::string schedule_csv(const Timeline& t) {
  std::string out =
      "type,gpu,cell,pipeline,kind,microbatch,stage,boundary,direction,bytes,start_ms,end_ms,"
      "arrival_ms,pooled_pipelines\n";
  for (const Task& x : t.tasks)
    out += "task," + std::to_string(x.gpu) + ',' + std::to_string(x.cell) + ',' +
           std::to_string(x.pipe) + ',' + kind_name(x.kind) + ',' + std::to_string(x.m) + ',' +
           std::to_string(x.stage) + ",,,," + fixed6(ns_to_ms(x.start)) + ',' +
           fixed6(ns_to_ms(x.end)) + ",,\n";
  for (const Xfer& x : t.xfers)
    out += "transfer,," + std::to_string(x.cell) + ',' + std::to_string(x.pipe) + ",transfer," +
           std::to_string(x.m) + ",," + std::to_string(x.boundary) + ',' + dir_name(x.dir) + ',' +
           std::to_string(x.bytes) + ',' + fixed6(ns_to_ms(x.start)) + ',' +
           fixed6(ns_to_ms(x.end)) + ',' + fixed6(ns_to_ms(x.arrival)) + ',' +
           std::to_string(x.pooled) + '\n';
  return out;
}

// report() (metrics.cpp:32-81) + metrics_csv (export.cpp:184-204)
std::string metrics_csv(const Timeline& t, const Timeline* ref, std::optional<long long> horizon) {
  const double iteration = ns_to_ms(t.makespan);
  const double thr = iteration > 0 ? 1000.0 / iteration : 0.0;
  const long long hor = horizon.value_or(t.makespan);
  std::map<int, double> per_gpu;
  double mean = 0.0, bubble = 1.0, wf[2] = {0.0, 0.0};
  if (hor > 0) {
    std::map<int, long long> busy;
    for (const Task& x : t.tasks) {
      const long long lo = std::max(x.start, 0LL), hi = std::min(x.end, hor);
      busy[x.gpu] += std::max(0LL, hi - lo);
    }
    double sum = 0.0;
    for (const auto& [gpu, ns] : busy) {
      const double u = static_cast<double>(ns) / static_cast<double>(hor);
      per_gpu[gpu] = u;
      sum += u;
    }
    if (!busy.empty()) mean = sum / busy.size();
    bubble = 1.0 - mean;
    std::map<std::tuple<int, int, int>, std::vector<std::pair<long long, long long>>> links;
    for (const Xfer& x : t.xfers) links[{x.cell, x.boundary, x.dir}].push_back({x.start, x.end});
    double frac[2] = {0.0, 0.0};
    int count[2] = {0, 0};
    for (auto& [key, ivs] : links) {
      std::sort(ivs.begin(), ivs.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      long long covered = 0, cursor = 0;
      for (const auto& iv : ivs) {
        const long long lo = std::max(std::max(iv.first, cursor), 0LL), hi = std::min(iv.second, hor);
        if (hi > lo) covered += hi - lo;
        cursor = std::max(cursor, hi);
      }
      const int dir = std::get<2>(key);
      frac[dir] += static_cast<double>(covered) / static_cast<double>(hor);
      count[dir] += 1;
    }
    for (int d = 0; d < 2; ++d)
      if (count[d] > 0) wf[d] = frac[d] / count[d];
  }
  std::string out = "metric,value\n";
  out += "makespan_ms," + fixed6(iteration) + '\n';
  out += "throughput_iters_per_s," + fixed6(thr) + '\n';
  out += "mean_utilization," + fixed6(mean) + '\n';
  out += "bubble_fraction," + fixed6(bubble) + '\n';
  out += "wan_busy_fraction_fwd," + fixed6(wf[0]) + '\n';
  out += "wan_busy_fraction_bwd," + fixed6(wf[1]) + '\n';
  if (ref) {
    if (ref->makespan <= 0) throw ConfigError("reference", "reference timeline has zero makespan");
    out += "slowdown_vs_reference," +
           fixed6(static_cast<double>(t.makespan) / static_cast<double>(ref->makespan)) + '\n';
  }
  for (const auto& [gpu, u] : per_gpu) out += "utilization_gpu_" + std::to_string(gpu) + ',' + fixed6(u) + '\n';
  return out;
}

std::string partitions_string(const std::vector<std::pair<std::string, int>>& parts) {
  std::string out;
  for (const auto& [dc, n] : parts) {
    if (!out.empty()) out += ';';
    out += dc + ':' + std::to_string(n);
  }
  return out;
}

std::vector<std::pair<std::string, int>> row_partitions(const gpb_row& r, const Topo& t) {
  std::map<std::string, int> m;  // std::map order of DC ids (dc_select.h:34)
  for (size_t i = 0; i < t.dcs.size(); ++i)
    if (r.partitions[i] > 0) m[t.dcs[i].id] = r.partitions[i];
  return {m.begin(), m.end()};
}

void append_row(std::string& out, const gpb_row& r, bool chosen, const Topo& t) {
  out += std::to_string(r.d) + ',' + (r.feasible ? '1' : '0') + ',' + fixed6(r.pp_time_ms) + ',' +
         fixed6(r.allreduce_time_ms) + ',' + fixed6(r.total_time_ms) + ',' + fixed6(r.throughput) +
         ',' + (chosen ? '1' : '0') + ',' + partitions_string(row_partitions(r, t)) + '\n';
}

// ---------------------------------------------------------- selection

struct Selection {
  std::vector<gpb_row> rows;
  int chosen_d = 0;
};

std::vector<Selection> run_selection(Session& se, const std::vector<RunConfig>& cfgs) {
  std::vector<gpb_topology> topos;
  std::vector<gpb_scenario> scens;
  for (size_t i = 0; i < cfgs.size(); ++i) {
    if (cfgs[i].select_C < 0 || cfgs[i].select_tp < 0) throw ConfigError("select", "invalid");
    topos.push_back(to_gpb(cfgs[i].topo));
    scens.push_back(selection_scenario(cfgs[i], (int)i));
  }
  int64_t n_rows = 0;
  std::vector<gpb_row> rows;
  std::vector<gpb_scenario_result> res(std::max<size_t>(1, scens.size()));
  if (gpb_group* g = se.devices()) {  // the space sharded over the devices
    se.check_group(gpb_group_load(g, topos.data(), (int32_t)topos.size(), scens.data(),
                                  (int32_t)scens.size(), &n_rows));
    se.check_group(gpb_group_evaluate(g));
    rows.resize(std::max<int64_t>(1, n_rows));
    se.check_group(gpb_group_fetch_rows(g, rows.data(), n_rows));
    se.check_group(gpb_group_fetch_scenarios(g, res.data(), (int32_t)scens.size()));
  } else {
    gpb_ctx* ctx = se.device();
    se.check(gpb_load(ctx, topos.data(), (int32_t)topos.size(), scens.data(),
                      (int32_t)scens.size(), &n_rows));
    se.check(gpb_evaluate(ctx, 1));
    rows.resize(std::max<int64_t>(1, n_rows));
    se.check(gpb_fetch_rows(ctx, rows.data(), n_rows));
    se.check(gpb_fetch_scenarios(ctx, res.data(), (int32_t)scens.size()));
  }
  std::vector<Selection> out(scens.size());
  for (size_t i = 0; i < scens.size(); ++i) {
    out[i].rows.assign(rows.begin() + res[i].first_row, rows.begin() + res[i].first_row + res[i].n_rows);
    out[i].chosen_d = res[i].chosen_d;
  }
  return out;
}

std::string selection_csv(const Selection& s, const Topo& t) {
  std::string out = "d,feasible,pp_time_ms,allreduce_time_ms,total_time_ms,throughput,chosen,partitions\n";
  for (const gpb_row& r : s.rows) append_row(out, r, r.d == s.chosen_d, t);
  return out;
}

std::string selection_table(const Selection& s, const Topo& t) {
  std::string out;
  char buf[256];
  std::snprintf(buf, sizeof buf, "%4s %9s %14s %14s %14s %12s  %s\n", "D", "feasible", "pp_ms",
                "allreduce_ms", "total_ms", "iters/s", "partitions");
  out += buf;
  for (const gpb_row& r : s.rows) {
    std::snprintf(buf, sizeof buf, "%4d %9s %14.3f %14.3f %14.3f %12.4f  %s%s\n", r.d,
                  r.feasible ? "yes" : "no", r.pp_time_ms, r.allreduce_time_ms, r.total_time_ms,
                  r.throughput, partitions_string(row_partitions(r, t)).c_str(),
                  r.d == s.chosen_d ? "  <-- chosen" : "");
    out += buf;
  }
  return out;
}

// ----------------------------------------------------------- bubbletea

struct Request {
  int id;
  double arrival_ms;
  int tokens;
};

std::vector<Request> parse_requests_csv(const std::string& text) {  // config.cpp:332-368
  std::vector<Request> out;
  std::istringstream in(text);
  std::string line;
  size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.pop_back();
    if (line.empty()) continue;
    if (line_no == 1 && line.find("id") == 0) continue;
    std::istringstream row(line);
    std::string a, b, cstr;
    if (!std::getline(row, a, ',') || !std::getline(row, b, ',') || !std::getline(row, cstr, ','))
      throw ConfigError("requests_csv:line " + std::to_string(line_no), "expected id,arrival_ms,tokens");
    try {
      out.push_back({std::stoi(a), std::stod(b), std::stoi(cstr)});
    } catch (const std::exception&) {
      throw ConfigError("requests_csv:line " + std::to_string(line_no), "expected id,arrival_ms,tokens");
    }
  }
  std::stable_sort(out.begin(), out.end(),
                   [](const Request& x, const Request& y) { return x.arrival_ms < y.arrival_ms; });
  return out;
}



// ------------------------------------------------------------ runners

void run_simulate(Session& se, const std::string& out_dir, bool trace_only) {
  RunConfig c = parse_run_config(parse_document(se.config_text));
  apply_overrides(c, se.ov);
  const std::string out = prepare_out_dir(out_dir);
  PlanInfo plan;
  Timeline t = simulate(se, c, c.policy, plan);
  if (trace_only) {
    write_text_file(out + "trace.json", chrome_trace(t));
    return;
  }
  std::optional<Timeline> ref;
  if (c.reference_policy) {
    PlanInfo p2;
    ref = simulate(se, c, *c.reference_policy, p2);
  }
  std::optional<long long> hz;
  if (c.horizon_ms) hz = ms_to_ns(*c.horizon_ms);
  write_text_file(out + "metrics.csv", metrics_csv(t, ref ? &*ref : nullptr, hz));
  write_text_file(out + "schedule.csv", schedule_csv(t));
  write_text_file(out + "trace.json", chrome_trace(t));
}

std::string run_select_dc(Session& se, const std::string& out_dir) {
  RunConfig c = parse_run_config(parse_document(se.config_text));
  apply_overrides(c, se.ov);
  const std::string out = prepare_out_dir(out_dir);
  std::vector<Selection> s = run_selection(se, {c});
  write_text_file(out + "selection.csv", selection_csv(s[0], c.topo));
  return selection_table(s[0], c.topo);
}

void run_whatif(Session& se, const std::string& out_dir) {
  auto configs = expand_scenarios(se.config_text);
  const std::string out = prepare_out_dir(out_dir);
  std::vector<RunConfig> cfgs;
  for (auto& [name, cfg] : configs) {
    apply_overrides(cfg, se.ov);
    cfgs.push_back(cfg);
  }
  std::vector<Selection> s = run_selection(se, cfgs);
  std::string csv = "scenario,d,feasible,pp_time_ms,allreduce_time_ms,total_time_ms,throughput,chosen,partitions\n";
  for (size_t i = 0; i < s.size(); ++i)
    for (const gpb_row& r : s[i].rows) {
      csv += configs[i].first + ',';
      append_row(csv, r, r.d == s[i].chosen_d, cfgs[i].topo);
    }
  write_text_file(out + "whatif.csv", csv);
}

void run_bubbletea(Session& se, const std::string& out_dir) {
  RunConfig c = parse_run_config(parse_document(se.config_text));
  apply_overrides(c, se.ov);
  const std::string out = prepare_out_dir(out_dir);
  PlanInfo plan;
  Timeline t = simulate(se, c, c.policy, plan);
  const long long horizon = c.horizon_ms ? ms_to_ns(*c.horizon_ms) : t.makespan;
  const gpb_prefill_model& pm = c.prefill;
  // the simulate plan on the device (the reference-policy run may have
  // replaced it): saturating requests and the packing run on its timeline
  gpb_ctx* ctx = se.device();
  {
    gpb_topology gt = to_gpb(c.topo);
    gpb_scenario s = base_scenario(c);
    s.policy = policy_code(c.policy);
    s.pipelines_per_cell = c.C;
    s.tp_degree = c.tp;
    s.d_max = c.dp_cells;
    set_order(s, c.topo, c.dc_order);
    int64_t n_rows = 0;
    se.check(gpb_load(ctx, &gt, 1, &s, 1, &n_rows));
    se.check(gpb_evaluate(ctx, 1));
  }
  const int64_t row = c.dp_cells - 1;
  std::vector<Request> reqs;
  if (c.requests_csv) {
    reqs = parse_requests_csv(read_text_file(*c.requests_csv));
  } else if (c.synthetic_count) {
    std::vector<gpb_request> g(std::max(1, *c.synthetic_count));
    if (gpb_synthetic_requests(*c.synthetic_count, c.seed, ns_to_ms(horizon), &pm, g.data()) != GPB_OK)
      throw ConfigError("prefill.synthetic", "invalid");
    for (int i = 0; i < *c.synthetic_count; ++i) reqs.push_back({g[i].id, g[i].arrival_ms, g[i].tokens});
  } else if (c.saturating) {
    // saturating_requests (bubbletea.cpp:240-267) on the device timeline
    se.check(gpb_set_allreduce_tail(ctx, c.with_allreduce ? 1 : 0));
    int64_t n = 0;
    int rc = gpb_saturating_requests(ctx, row, &pm, horizon, nullptr, 0, &n);
    std::vector<gpb_request> g(std::max<int64_t>(1, n));
    if (rc == GPB_OK) rc = gpb_saturating_requests(ctx, row, &pm, horizon, g.data(), n, &n);
    gpb_set_allreduce_tail(ctx, 0);
    se.check(rc);
    for (int64_t i = 0; i < n; ++i) reqs.push_back({g[i].id, g[i].arrival_ms, g[i].tokens});
  }
  std::vector<gpb_request> greq(reqs.size());
  for (size_t i = 0; i < reqs.size(); ++i) greq[i] = {reqs[i].id, reqs[i].tokens, reqs[i].arrival_ms};
  gpb_pack_summary sum;
  std::vector<gpb_placement> pl(std::max<size_t>(1, reqs.size()));
  se.check(gpb_set_allreduce_tail(ctx, c.with_allreduce ? 1 : 0));
  const int rc = gpb_pack_prefills(ctx, &row, 1, greq.data(), (int64_t)greq.size(), &pm, horizon,
                                   &sum, pl.data());
  gpb_set_allreduce_tail(ctx, 0);
  se.check(rc);
  // placements.csv (export.cpp:245-262): accepted then rejected, keyed by id
  std::map<int, std::string> rows;
  Timeline aug = t;
  const int D = plan.D, base_l = pm.inference_layers / D, extra = pm.inference_layers % D;
  int total_layers = 0;
  for (int k = 0; k < D; ++k) total_layers += base_l + (k < extra ? 1 : 0);
  for (size_t i = 0; i < reqs.size(); ++i) {
    if (!pl[i].accepted) continue;
    const Request& r = reqs[i];
    rows[r.id] = std::to_string(r.id) + ",1," + std::to_string(pl[i].pipeline) + ',' +
                 fixed6(ns_to_ms(pl[i].start_ns)) + ',' + fixed6(pl[i].ttft_overhead_ms) + ",\n";
    // prefill tasks of the augmented timeline (bubbletea.cpp:189-200)
    const double dur_ms = pm.saturation_ms * static_cast<double>(r.tokens) / static_cast<double>(pm.max_tokens);
    const double bytes = static_cast<double>(1LL * r.tokens * pm.inference_hidden * pm.bytes_per_element);
    const long long ovh = ms_to_ns(1 * (pm.boundary_latency_ms + bytes / pm.stage_bw));
    const int pipe = pl[i].pipeline / plan.S, st = pl[i].pipeline % plan.S;
    long long cursor = 0;
    for (int k = 0; k < D; ++k) {
      const int layers = base_l + (k < extra ? 1 : 0);
      const long long dk = ms_to_ns(dur_ms * layers / std::max(1, total_layers));
      const long long lo = pl[i].start_ns + cursor;
      aug.tasks.push_back({plan.gpu[((size_t)k * plan.C + pipe) * plan.S + st], k, pl[i].pipeline,
                           kPrefill, r.id, k, lo, lo + dk});
      cursor += dk + ovh;
    }
  }
  for (size_t i = 0; i < reqs.size(); ++i)
    if (!pl[i].accepted) rows[reqs[i].id] = std::to_string(reqs[i].id) + ",0,,,,NoCapacity\n";
  std::string csv = "id,accepted,pipeline,start_ms,ttft_overhead_ms,reason\n";
  for (const auto& [id, line] : rows) csv += line;
  write_text_file(out + "placements.csv", csv);
  std::string m = "metric,value\n";
  m += "utilization_before," + fixed6(sum.utilization_before) + '\n';
  m += "utilization_after," + fixed6(sum.utilization_after) + '\n';
  m += "requests," + std::to_string(reqs.size()) + '\n';
  m += "accepted," + std::to_string(sum.accepted) + '\n';
  m += "rejected," + std::to_string(sum.rejected) + '\n';
  write_text_file(out + "bubbletea_metrics.csv", m);
  finalize(aug);
  write_text_file(out + "trace.json", chrome_trace(aug));
}

}  // namespace

struct gp_session : Session {};

namespace {

// capi.cpp:19-39 error mapping
template <typename Fn>
int guarded(gp_session* s, Fn&& fn) {
  if (s == nullptr) return GP_ERROR;
  s->last_error.clear();
  try {
    fn();
    return GP_OK;
  } catch (const ConfigError& e) {
    s->last_error = e.what();
    return GP_CONFIG_ERROR;
  } catch (const Infeasible& e) {
    s->last_error = e.what();
    return GP_INFEASIBLE;
  } catch (const std::exception& e) {
    s->last_error = e.what();
    return GP_ERROR;
  } catch (...) {
    s->last_error = "unknown error";
    return GP_ERROR;
  }
}

template <typename Fn>
int run_command(gp_session* s, const char* out_dir, Fn&& fn) {
  if (s == nullptr) return GP_ERROR;
  if (!s->config_loaded) {
    s->last_error = "no config loaded";
    return GP_CONFIG_ERROR;
  }
  return guarded(s, [&] {
    if (out_dir == nullptr) throw ConfigError("out", "null output directory");
    fn(std::string(out_dir));
  });
}

}  // namespace

extern "C" {

gp_session* gp_session_create(void) {
  try {
    return new gp_session();
  } catch (...) {
    return nullptr;
  }
}

void gp_session_destroy(gp_session* s) { delete s; }

int gp_load_config_file(gp_session* s, const char* path) {
  return guarded(s, [&] {
    if (path == nullptr) throw ConfigError("config", "null path");
    s->config_text = read_text_file(path);
    s->config_loaded = true;
  });
}

int gp_load_config_text(gp_session* s, const char* text) {
  return guarded(s, [&] {
    if (text == nullptr) throw ConfigError("config", "null text");
    s->config_text = text;
    s->config_loaded = true;
  });
}

int gp_set_policy(gp_session* s, const char* policy) {
  return guarded(s, [&] {
    if (policy == nullptr) throw ConfigError("policy", "null policy");
    s->ov.policy = std::string(policy);
  });
}

int gp_set_seed(gp_session* s, unsigned seed) {
  return guarded(s, [&] { s->ov.seed = seed; });
}

int gp_set_multi_conn(gp_session* s, int enabled) {
  return guarded(s, [&] { s->ov.multi_conn = enabled != 0; });
}

int gp_set_recompute(gp_session* s, int enabled) {
  return guarded(s, [&] { s->ov.recompute = enabled != 0; });
}

int gp_set_mem_limit(gp_session* s, int microbatches) {
  return guarded(s, [&] { s->ov.mem_limit = microbatches; });
}

int gp_set_horizon_ms(gp_session* s, double horizon_ms) {
  return guarded(s, [&] { s->ov.horizon_ms = horizon_ms; });
}

int gp_run_simulate(gp_session* s, const char* out_dir) {
  return run_command(s, out_dir, [&](const std::string& out) { run_simulate(*s, out, false); });
}

int gp_run_trace(gp_session* s, const char* out_dir) {
  return run_command(s, out_dir, [&](const std::string& out) { run_simulate(*s, out, true); });
}

int gp_run_select_dc(gp_session* s, const char* out_dir) {
  return run_command(s, out_dir, [&](const std::string& out) { s->selection_table = run_select_dc(*s, out); });
}

int gp_run_whatif(gp_session* s, const char* out_dir) {
  return run_command(s, out_dir, [&](const std::string& out) { run_whatif(*s, out); });
}

int gp_run_bubbletea(gp_session* s, const char* out_dir) {
  return run_command(s, out_dir, [&](const std::string& out) { run_bubbletea(*s, out); });
}

const char* gp_last_error(gp_session* s) { return s == nullptr ? "" : s->last_error.c_str(); }

const char* gp_selection_table(gp_session* s) { return s == nullptr ? "" : s->selection_table.c_str(); }

}  // extern "C"
