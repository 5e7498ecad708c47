// device_common.cuh — shared device-side types and helpers for the sm_100a
// plan-evaluation kernels. Everything that must be bit-exact against the
// reference's double arithmetic is compiled with --fmad=false and written in
// the reference's operation order (cited per function).
#pragma once

#include <cstdint>

#include "../../include/geopipe_batch.h"

namespace gpb {

constexpr long long kInf64 = 0x7fffffffffffffffLL;

// Per-topology constants (ClusterTopology, topology.h:12-40) with the
// host-computed single-TCP curve (comm_model.cpp:8-25 uses libm log/exp, so
// it is evaluated with the host libm and uploaded as exact doubles).
struct DevTopo {
  int32_t n_dc;
  int32_t gpu_count[GPB_MAX_DC];
  int32_t dc_base[GPB_MAX_DC];          // first GPU id of each DC (build_plan)
  int32_t pad_;
  double intra_bw[GPB_MAX_DC];
  double lat_ms[GPB_MAX_DC][GPB_MAX_DC];
  double single_bw[GPB_MAX_DC][GPB_MAX_DC];
  double pair_cap;
};

// Per-scenario constants (SelectionInput, dc_select.h:18-30) in the layout
// the kernels read: 128 bytes, 16-byte aligned.
struct alignas(16) DevScen {
  int32_t topo;
  int32_t policy;
  int32_t S;            // partition_count (workload.h:22-24)
  int32_t M;
  int32_t C;
  int32_t tp;
  int32_t L;            // num_layers
  int32_t lpp;
  int32_t n_order;
  int32_t recompute;
  int32_t mem_limit;    // resolved: > 0
  int32_t n_conns;      // multi_conn ? n_connections : 1 (scheduler.cpp:39)
  int8_t order[GPB_MAX_DC];
  double fwd_ms, bwd_ms, rec_ms;   // resolved profile (dc_select.cpp:12-18)
  double ppl;                      // effective_params_per_layer
  int64_t bytes;                   // activation_bytes (comm_model.cpp:43-45)
  int64_t first_row;
  int32_t n_rows;
  int32_t pad_;
};
static_assert(sizeof(DevScen) == 112 || sizeof(DevScen) == 128, "DevScen size");

// Decoded plan geometry for one (scenario, D) row (build_plan walk,
// workload.cpp:57-89, + build_geometry, scheduler.cpp:32-76). Stages are
// grouped in nb contiguous DC blocks; boundary after block b (b < nb-1) is a
// WAN boundary.
struct Geom {
  int32_t feasible;
  int32_t drain_lane;  // min S for the one-lane WAN drain greedy (C <= 4), 0 = never; set by the caller
  int32_t S, M, C, D;
  int32_t nb;
  int32_t blk_first[GPB_MAX_DC + 1];   // blk_first[nb] == S
  int32_t blk_dc[GPB_MAX_DC];
  long long fwd, bwd, rec, dur;        // ns; dur = pair duration
  // per WAN boundary w (between block w and w+1): stage index of the
  // producing stage (blk_first[w+1]-1), serialization and latency (ns)
  long long ser_spatial[GPB_MAX_DC];
  long long ser_pooled[GPB_MAX_DC];
  long long lat[GPB_MAX_DC];
};

__device__ __forceinline__ long long imax(long long a, long long b) { return a > b ? a : b; }
__device__ __forceinline__ long long imin(long long a, long long b) { return a < b ? a : b; }

// ms_to_ns = llround(ms * 1e6) (base.h:15-17).
__device__ __forceinline__ long long ms_to_ns(double ms) { return llround(__dmul_rn(ms, 1e6)); }

// Block index of stage s (blocks are few: linear scan).
__device__ __forceinline__ int block_of(const Geom& g, int s) {
  int b = 0;
#pragma unroll 1
  while (b + 1 < g.nb && s >= g.blk_first[b + 1]) ++b;
  return b;
}

// Boundary s -> s+1 crosses DCs iff s+1 starts a block (duplicate DCs in an
// order are rejected on the host, so adjacent blocks always differ).
__device__ __forceinline__ int wan_after(const Geom& g, int s, int& w) {
  for (int b = 1; b < g.nb; ++b)
    if (g.blk_first[b] == s + 1) {
      w = b - 1;
      return 1;
    }
  return 0;
}

// build_plan's partition walk and build_geometry for cell 0 (all D cells are
// identical, so one cell stands for all; SURVEY.md §7 "redundancy removal").
__device__ inline void decode(const DevScen& sc, const DevTopo& t, int d, Geom& g) {
  g.S = sc.S;
  g.M = sc.M;
  g.C = sc.C;
  g.D = d;
  g.nb = 0;
  int assigned = 0;
  const int denom = d * sc.C * sc.tp;
  for (int i = 0; i < sc.n_order; ++i) {  // workload.cpp:71-83
    if (assigned >= sc.S) break;
    const int dc = sc.order[i];
    const int capacity = t.gpu_count[dc] / denom;
    const int take = min(sc.S - assigned, capacity);
    if (take > 0) {
      g.blk_first[g.nb] = assigned;
      g.blk_dc[g.nb] = dc;
      ++g.nb;
      assigned += take;
    }
  }
  g.blk_first[g.nb] = assigned;
  g.feasible = assigned >= sc.S;
  if (!g.feasible) return;
  g.fwd = ms_to_ns(sc.fwd_ms);  // scheduler.cpp:47-49
  g.bwd = ms_to_ns(sc.bwd_ms);
  g.rec = ms_to_ns(sc.rec_ms);
  g.dur = sc.recompute ? g.rec + g.bwd : g.bwd;  // pair_dur, :27-29
  const double bytes = (double)sc.bytes;
  for (int w = 0; w + 1 < g.nb; ++w) {  // :57-72
    const int a = g.blk_dc[w], b = g.blk_dc[w + 1];
    const double lat = t.lat_ms[a][b];
    // effective_pair_bandwidth (comm_model.cpp:27-31)
    const double multi = __dmul_rn((double)sc.n_conns, t.single_bw[a][b]);
    const double bw = multi < t.pair_cap ? multi : t.pair_cap;
    g.ser_spatial[w] = ms_to_ns(__ddiv_rn(bytes, bw));
    g.ser_pooled[w] = ms_to_ns(__ddiv_rn(bytes, __dmul_rn((double)sc.C, bw)));
    g.lat[w] = ms_to_ns(lat);
  }
}

// Exact emulation of `double s = 0; for (k < G) s += u;` — the utilization
// mean of identical per-GPU values summed in GPU-id order (metrics.cpp:47-53).
// Within one binade the rounded increment is constant after at most one
// transient step, so runs of equal increments are applied in one jump; the
// result is bit-identical to the sequential loop (verified on the host in
// tests/test_repeated_sum.py and on the device by the row parity tests).
__host__ __device__ inline double repeated_sum(double u, long long G) {
  if (G <= 0) return 0.0;
  if (!(u > 0.0) || u > 1.7e308) {
    double s = 0.0;
    for (long long k = 0; k < G; ++k) s = s + u;
    return s;
  }
  double s = 0.0, prev_s = 0.0, prev_delta = -1.0;
  long long k = 0;
  while (k < G) {
    double sn = s + u;
    double delta = sn - s;  // exact (Sterbenz: u <= s after the first step)
    ++k;
    double before = s;
    s = sn;
    if (k < G && delta == prev_delta) {
      // both increments inside one binade?
      uint64_t bs, bp, bb;
#ifdef __CUDA_ARCH__
      bs = (uint64_t)__double_as_longlong(s);
      bp = (uint64_t)__double_as_longlong(prev_s);
      bb = (uint64_t)__double_as_longlong(before);
#else
      __builtin_memcpy(&bs, &s, 8);
      __builtin_memcpy(&bp, &prev_s, 8);
      __builtin_memcpy(&bb, &before, 8);
#endif
      const int es = (int)((bs >> 52) & 0x7ff), ep = (int)((bp >> 52) & 0x7ff),
                eb = (int)((bb >> 52) & 0x7ff);
      if (es == ep && es == eb && es != 0) {
        uint64_t bu;
#ifdef __CUDA_ARCH__
        bu = (uint64_t)__double_as_longlong(u);
#else
        __builtin_memcpy(&bu, &u, 8);
#endif
        const int eu = (int)((bu >> 52) & 0x7ff);
        const uint64_t Sm = (bs & 0xfffffffffffffULL) | (1ULL << 52);
        const uint64_t Um = (bu & 0xfffffffffffffULL) | (1ULL << 52);
        const int shift = es - eu;  // >= 0 because u <= s
        const uint64_t n = shift >= 64 ? 0 : (Um >> shift);
        // delta in units of the binade's ulp: d = delta / 2^(es-1075)
        uint64_t bd;
#ifdef __CUDA_ARCH__
        bd = (uint64_t)__double_as_longlong(delta);
#else
        __builtin_memcpy(&bd, &delta, 8);
#endif
        const int ed = (int)((bd >> 52) & 0x7ff);
        const uint64_t Dm = (bd & 0xfffffffffffffULL) | (1ULL << 52);
        const int dsh = es - ed;  // delta <= s
        if (ed != 0 && dsh <= 52 && (Dm & ((1ULL << dsh) - 1)) == 0) {
          const uint64_t dq = Dm >> dsh;  // integer ulps per step
          const uint64_t lim = (1ULL << 53) - 1;
          if (dq > 0 && Sm + n <= lim) {
            long long jmax = (long long)((lim - n - Sm) / dq);
            long long J = G - k < jmax ? G - k : jmax;
            if (J > 0) {
              s = s + (double)J * delta;  // exact: stays inside the binade
              k += J;
            }
          }
        }
      }
    }
    prev_s = before;
    prev_delta = delta;
  }
  return s;
}

// Row epilogue shared by every policy (dc_select.cpp:46-64 + metrics.cpp:39-54):
// per-stage worst all-reduce, totals, throughput and mean utilization.
__device__ inline void finish_row(const DevScen& sc, const DevTopo& t, const Geom& g,
                                  long long makespan, gpb_row& r) {
  r.feasible = 1;
  r.makespan_ns = makespan;
  r.pp_time_ms = __ddiv_rn((double)makespan, 1e6);  // ns_to_ms, base.h:19
  const int n = g.D * sc.C;
  double worst = 0.0;
  for (int b = 0; b < g.nb; ++b) {
    const int s0 = g.blk_first[b], s1 = g.blk_first[b + 1];
    r.partitions[g.blk_dc[b]] = (int16_t)(s1 - s0);
    // layers of stage s: min(lpp, L - s*lpp) (dc_select.cpp:49-55); the
    // maximum over a block is attained at its first stage, and only the last
    // stage can be short, so the block's worst is the first stage's value.
    const int begin = s0 * sc.lpp;
    const int end = min(begin + sc.lpp, sc.L);
    const int layers = max(0, end - begin);
    if (n > 1) {
      const double params = __dmul_rn(sc.ppl, (double)layers);
      // allreduce_time_ms (comm_model.cpp:38-41): 4*P*(N-1) / (N*bw)
      const double v = __ddiv_rn(__dmul_rn(__dmul_rn(4.0, params), (double)(n - 1)),
                                 __dmul_rn((double)n, t.intra_bw[g.blk_dc[b]]));
      worst = worst < v ? v : worst;  // std::max(worst, v)
    }
  }
  r.allreduce_time_ms = worst;
  r.total_time_ms = __dadd_rn(r.pp_time_ms, worst);
  r.throughput = __ddiv_rn(__dmul_rn((double)g.D, (double)sc.C), r.total_time_ms);
  // Every timeline GPU (front GPU of each stage, D*C*S of them) runs M
  // forwards and M pairs inside [0, makespan).
  if (makespan > 0) {
    const long long busy = (long long)g.M * (g.fwd + g.dur);
    const double u = __ddiv_rn((double)busy, (double)makespan);
    const long long G = (long long)g.D * sc.C * g.S;
    r.utilization = __ddiv_rn(repeated_sum(u, G), (double)G);
  } else {
    r.utilization = 0.0;
  }
}

__device__ inline void infeasible_row(gpb_row& r) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  r.pp_time_ms = inf;
  r.allreduce_time_ms = inf;
  r.total_time_ms = inf;
  r.throughput = 0.0;
  r.utilization = 0.0;
  r.makespan_ns = 0;
  r.feasible = 0;
  r.chosen = 0;
  for (int i = 0; i < GPB_MAX_DC; ++i) r.partitions[i] = 0;
}

}  // namespace gpb
