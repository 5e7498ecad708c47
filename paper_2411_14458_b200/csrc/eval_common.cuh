// eval_common.cuh — warp helpers shared by the evaluation kernels.
#pragma once

#include "device_common.cuh"
#include "kernels.h"

namespace gpb {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ long long shfl_up64(long long v, int d) {
  return __shfl_up_sync(kFull, v, d);
}
__device__ __forceinline__ long long shfl_down64(long long v, int d) {
  return __shfl_down_sync(kFull, v, d);
}
__device__ __forceinline__ long long shfl_idx64(long long v, int src) {
  return __shfl_sync(kFull, v, src);
}
__device__ __forceinline__ long long warp_max64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = imax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// Pull the next work item for this warp (lane 0 bumps the cursor).
__device__ __forceinline__ int next_work(int* cursor) {
  int idx = 0;
  if ((threadIdx.x & 31) == 0) idx = atomicAdd(cursor, 1);
  return __shfl_sync(kFull, idx, 0);
}

// Row header: decode + infeasible fast path. Returns false if infeasible.
__device__ __forceinline__ bool begin_row(const EvalArgs& a, int row, Geom& g,
                                          const DevScen*& sc, const DevTopo*& tp) {
  const int si = a.row_scen[row];
  sc = &a.scens[si];
  tp = &a.topos[sc->topo];
  const int d = (int)(row - sc->first_row) + 1;
  decode(*sc, *tp, d, g);
  g.drain_lane = a.drain_lane;
  if (!g.feasible) {
    if ((threadIdx.x & 31) == 0) {
      gpb_row r;
      infeasible_row(r);
      r.scenario = si;
      r.d = d;
      a.rows[row] = r;
    }
    return false;
  }
  return true;
}

__device__ __forceinline__ void end_row(const EvalArgs& a, int row, const Geom& g,
                                        const DevScen& sc, const DevTopo& tp,
                                        long long makespan, int err, long long t_start) {
  if ((threadIdx.x & 31) == 0) {
    if (a.row_cycles) a.row_cycles[row] = clock64() - t_start;
    gpb_row r;
    infeasible_row(r);
    r.scenario = a.row_scen[row];
    r.d = g.D;
    finish_row(sc, tp, g, makespan, r);
    if (err) {
      r.feasible = -1;  // kernel-side invariant failure: host raises GPB_ERROR
      atomicExch(a.error_flag, 1);
    }
    a.rows[row] = r;
  }
}

// Per-stage boundary info for the stages a lane owns.
template <int B>
struct StageLinks {
  unsigned wanf = 0, wanb = 0;  // bit j: WAN boundary after / before stage
  long long serf[B], latf[B], serb[B], latb[B];

  __device__ __forceinline__ void load(const Geom& g, int lane, bool pooled) {
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int s = lane * B + j;
      serf[j] = latf[j] = serb[j] = latb[j] = 0;
      int w;
      if (s < g.S) {
        if (s + 1 < g.S && wan_after(g, s, w)) {
          wanf |= 1u << j;
          serf[j] = pooled ? g.ser_pooled[w] : g.ser_spatial[w];
          latf[j] = g.lat[w];
        }
        if (s > 0 && wan_after(g, s - 1, w)) {
          wanb |= 1u << j;
          serb[j] = pooled ? g.ser_pooled[w] : g.ser_spatial[w];
          latb[j] = g.lat[w];
        }
      }
    }
  }
};

}  // namespace gpb
