// kernels_eval.cu — sm_100a plan-evaluation kernels: one warp per plan row.
//
//  flush_kernel<B, GPIPE>  gpipe / varuna  (scheduler.cpp:113-171)
//      max-plus wavefront in registers: lane k owns stages [kB, kB+B); the
//      forward phase sweeps anti-diagonals (m - k) with shfl_up hand-offs,
//      the drain sweeps them back down with shfl_down.
//  onef1b_kernel<B>        1f1b (scheduler.cpp:177-267)
//      lock-step rounds: every stage executes at most one item of its fixed
//      1F1B program per round; neighbours publish their latest output and
//      progress counters by shuffle. The reference's program DAG has a unique
//      timing, and under lock-step the producer is never more than one item
//      ahead of its consumer (checked in-kernel; violation => error row).
//  atlas_kernel            atlas (scheduler.cpp:276-538)
//      forward chains via a warp max-plus scan and O(#WAN) exact-fit checks,
//      memory-cap forced drains, then the global greedy drain with a cached
//      candidate table and a three-step redux argmin per committed pair.
//
// Every kernel pulls rows from a per-bucket work list with an atomic cursor
// (persistent warps) and finishes each row with finish_row() (all-reduce,
// throughput, utilization).
#include <cuda_runtime.h>

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
                                        long long makespan, int err) {
  if ((threadIdx.x & 31) == 0) {
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

// ---------------------------------------------------------------- flush

template <int B, bool GPIPE>
__device__ long long flush_row(const Geom& g, long long* fdl) {
  const int lane = threadIdx.x & 31;
  const int S = g.S, M = g.M;
  const int K = (S - 1) / B;  // highest lane that owns a stage
  StageLinks<B> L;
  L.load(g, lane, false);
  long long gf[B], lf[B], lb[B];
#pragma unroll
  for (int j = 0; j < B; ++j) gf[j] = lf[j] = lb[j] = 0;

  // Forward: E[s][m] = max(A[s][m], E[s][m-1]) + f; link FIFO per boundary.
  long long a_in = 0;
  for (int t = 0; t < M + K; ++t) {
    const int m = t - lane;
    long long a = lane == 0 ? 0 : a_in;
    if (lane <= K && m >= 0 && m < M) {
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int s = lane * B + j;
        if (s < S) {
          const long long e = imax(a, gf[j]) + g.fwd;
          gf[j] = e;
          if (s == S - 1) fdl[m] = e;
          if ((L.wanf >> j) & 1u) {
            const long long occ = imax(e, lf[j]) + L.serf[j];
            lf[j] = occ;
            a = occ + L.latf[j];
          } else {
            a = e;
          }
        }
      }
    }
    a_in = shfl_up64(a, 1);
  }
  __syncwarp();
  const long long beta = GPIPE ? fdl[M - 1] : 0;  // barrier_last_fwd
  // Drain: stages S-1..0, microbatch order k (varuna) or M-1-k (gpipe).
  long long g_in = 0;
  for (int t = 0; t < M + K; ++t) {
    const int i = t - (K - lane);
    long long gv = g_in;
    if (lane <= K && i >= 0 && i < M) {
      const int m = GPIPE ? M - 1 - i : i;
#pragma unroll
      for (int j = B - 1; j >= 0; --j) {
        const int s = lane * B + j;
        if (s < S) {
          long long ready = s == S - 1 ? fdl[m] : gv;
          ready = imax(ready, beta);
          const long long z = imax(ready, gf[j]) + g.dur;
          gf[j] = z;
          if (s > 0) {
            if ((L.wanb >> j) & 1u) {
              const long long occ = imax(z, lb[j]) + L.serb[j];
              lb[j] = occ;
              gv = occ + L.latb[j];
            } else {
              gv = z;
            }
          }
        }
      }
    }
    g_in = shfl_down64(gv, 1);
  }
  long long mk = 0;
#pragma unroll
  for (int j = 0; j < B; ++j) mk = imax(mk, gf[j]);
  return warp_max64(mk);
}

template <int B, bool GPIPE>
__global__ void __launch_bounds__(kEvalThreads) flush_kernel(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  long long* fdl = reinterpret_cast<long long*>(smem) + (size_t)warp * a.smem_m;
  for (;;) {
    const int w = next_work(a.cursor);
    if (w >= a.n_work) break;
    const int row = a.work[w];
    Geom g;
    const DevScen* sc;
    const DevTopo* tp;
    if (!begin_row(a, row, g, sc, tp)) continue;
    const long long mk = flush_row<B, GPIPE>(g, fdl);
    end_row(a, row, g, *sc, *tp, mk, 0);
    __syncwarp();
  }
}

// ----------------------------------------------------------------- 1F1B

// Item at program counter pc of stage s (w = min(S - s, M) warm-up forwards,
// then B/F alternation, then the remaining backwards; scheduler.cpp:186-196).
__device__ __forceinline__ void onef1b_item(int pc, int w, int M, bool& fwd, int& m) {
  if (pc < w) {
    fwd = true;
    m = pc;
  } else if (pc < 2 * M - w) {
    const int j = pc - w;
    fwd = (j & 1) != 0;
    m = fwd ? w + (j >> 1) : (j >> 1);
  } else {
    fwd = false;
    m = pc - M;
  }
}

template <int B>
__device__ long long onef1b_row(const Geom& g, int& err) {
  const int lane = threadIdx.x & 31;
  const int S = g.S, M = g.M;
  StageLinks<B> L;
  L.load(g, lane, false);
  int pc[B], nF[B], nB[B];
  long long gf[B], lf[B], lb[B], outF[B], outB[B], fdo[B];
#pragma unroll
  for (int j = 0; j < B; ++j) {
    pc[j] = nF[j] = nB[j] = 0;
    gf[j] = lf[j] = lb[j] = outF[j] = outB[j] = fdo[j] = 0;
    if (lane * B + j >= S) pc[j] = 2 * M;  // no stage: done
  }
  int bad = 0;
  for (;;) {
    bool busy = false;
#pragma unroll
    for (int j = 0; j < B; ++j) busy |= pc[j] < 2 * M;
    if (!__any_sync(kFull, busy)) break;
    // Snapshots of the neighbours' state at the start of the round.
    const int lnF = __shfl_up_sync(kFull, nF[B - 1], 1);
    const long long loutF = shfl_up64(outF[B - 1], 1);
    const int rnB = __shfl_down_sync(kFull, nB[0], 1);
    const long long routB = shfl_down64(outB[0], 1);
    int snF[B], snB[B];
    long long soutF[B], soutB[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      snF[j] = nF[j];
      snB[j] = nB[j];
      soutF[j] = outF[j];
      soutB[j] = outB[j];
    }
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int s = lane * B + j;
      if (pc[j] >= 2 * M) continue;
      const int w = min(S - s, M);
      bool fwd;
      int m;
      onef1b_item(pc[j], w, M, fwd, m);
      if (fwd) {
        long long arr = 0;
        if (s > 0) {
          const int pn = j == 0 ? lnF : snF[j - 1];
          if (pn <= m) continue;              // input not produced yet
          if (pn > m + 1) bad = 1;            // mailbox depth invariant
          arr = j == 0 ? loutF : soutF[j - 1];
        }
        const long long e = imax(arr, gf[j]) + g.fwd;
        gf[j] = e;
        fdo[j] = e;
        if (s + 1 < S) {
          if ((L.wanf >> j) & 1u) {
            const long long occ = imax(e, lf[j]) + L.serf[j];
            lf[j] = occ;
            outF[j] = occ + L.latf[j];
          } else {
            outF[j] = e;
          }
        }
        nF[j] += 1;
      } else {
        long long ready;
        if (s == S - 1) {
          if (nF[j] <= m) continue;
          ready = fdo[j];  // F(S-1, m) immediately precedes B(S-1, m)
        } else {
          const int pn = j == B - 1 ? rnB : snB[j + 1];
          if (pn <= m) continue;
          if (pn > m + 1) bad = 1;
          ready = j == B - 1 ? routB : soutB[j + 1];
        }
        const long long z = imax(ready, gf[j]) + g.dur;
        gf[j] = z;
        if (s > 0) {
          if ((L.wanb >> j) & 1u) {
            const long long occ = imax(z, lb[j]) + L.serb[j];
            lb[j] = occ;
            outB[j] = occ + L.latb[j];
          } else {
            outB[j] = z;
          }
        }
        nB[j] += 1;
      }
      pc[j] += 1;
    }
  }
  long long mk = 0;
#pragma unroll
  for (int j = 0; j < B; ++j) mk = imax(mk, gf[j]);
  err = __any_sync(kFull, bad) ? 1 : 0;
  return warp_max64(mk);
}

template <int B>
__global__ void __launch_bounds__(kEvalThreads) onef1b_kernel(EvalArgs a) {
  for (;;) {
    const int w = next_work(a.cursor);
    if (w >= a.n_work) break;
    const int row = a.work[w];
    Geom g;
    const DevScen* sc;
    const DevTopo* tp;
    if (!begin_row(a, row, g, sc, tp)) continue;
    int err = 0;
    const long long mk = onef1b_row<B>(g, err);
    end_row(a, row, g, *sc, *tp, mk, err);
    __syncwarp();
  }
}

// ---------------------------------------------------------------- ATLAS

// ReservationList (base.h:63-124) over uniform-length intervals: only the
// starts are stored (sorted, non-overlapping), `len` is the boundary's pooled
// serialization time.

// first index i with st[i] + len > x (first interval ending after x)
__device__ __forceinline__ int resv_first_end_after(const long long* st, int n,
                                                    long long len, long long x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (st[mid] + len > x) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// earliest_fit (base.h:75-84)
__device__ __forceinline__ long long resv_earliest_fit(const long long* st, int n,
                                                       long long lo, long long len) {
  if (len <= 0) return lo;
  long long t = lo;
  for (int i = resv_first_end_after(st, n, len, lo); i < n; ++i) {
    if (st[i] >= t + len) break;
    t = st[i] + len;
  }
  return t;
}

// free_at (base.h:65-72)
__device__ __forceinline__ bool resv_free_at(const long long* st, int n, long long start,
                                             long long len) {
  if (len <= 0) return true;
  const int i = resv_first_end_after(st, n, len, start);
  return !(i < n && st[i] < start + len);
}

// reserve (base.h:101-106): insert before the first start >= x. Warp-wide.
__device__ __forceinline__ void resv_insert_warp(long long* st, int& n, long long x,
                                                 long long len) {
  if (len <= 0) return;
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (st[mid] < x) lo = mid + 1; else hi = mid;
  }
  for (int base = n - 1; base >= lo; base -= 32) {
    const int idx = base - lane;
    long long v = 0;
    if (idx >= lo) v = st[idx];
    __syncwarp();
    if (idx >= lo) st[idx + 1] = v;
    __syncwarp();
  }
  if (lane == 0) st[lo] = x;
  __syncwarp();
  n += 1;
}

struct AtlasScratch {
  long long* garr;   // [C][S][M]
  long long* fdl;    // [C][M]
  long long* resf;   // [nb-1][cap]
  long long* resb;   // [nb-1][cap]
  long long* ps;     // [C][S][M] pair starts (timeline variant only)
  int cap;
};

struct AtlasShared {   // pointers into this warp's shared-memory slice
  long long* wa;       // [GPB_MAX_DC] chain offset a_w of WAN producer stages
  long long* wg;       // [GPB_MAX_DC] prefix max G_w of WAN producer stages
  long long* gf;       // [C][S] gpu_free
  long long* cand;     // [C][S] cached greedy candidate start
  int* nm;             // [C][S] next_m (drained count during forwards)
  // list lengths: kept in registers, updated identically by every lane
  int nres_f[GPB_MAX_DC];
  int nres_b[GPB_MAX_DC];
};

__device__ __forceinline__ int wan_before_idx(const Geom& g, int s) {
  int w;
  return (s > 0 && wan_after(g, s - 1, w)) ? w : -1;
}

// Candidate start for pair (p, s) at its next microbatch (INF if not ready):
// atlas_pair_start(max(ready, gpu_free)) (scheduler.cpp:461-485, 287-294).
__device__ __forceinline__ long long atlas_candidate(const Geom& g, const AtlasScratch& X,
                                                     const AtlasShared& H, int p, int s) {
  const int S = g.S, M = g.M;
  const int m = H.nm[p * S + s];
  if (m >= M) return kInf64;
  long long ready;
  if (s == S - 1) {
    ready = X.fdl[(size_t)p * M + m];
  } else {
    if (H.nm[p * S + s + 1] <= m) return kInf64;  // gradient not produced
    ready = X.garr[((size_t)p * S + s) * M + m];
  }
  const long long lo = imax(ready, H.gf[p * S + s]);
  const int w = wan_before_idx(g, s);
  if (w < 0) return lo;
  const long long* st = X.resb + (size_t)w * X.cap;
  return resv_earliest_fit(st, H.nres_b[w], lo + g.dur, g.ser_pooled[w]) - g.dur;
}

// Lane-local best over the candidates of the stages this lane owns.
__device__ __forceinline__ void lane_best(const Geom& g, const AtlasShared& H, int lane,
                                          int B, long long& bt, unsigned& brank) {
  bt = kInf64;
  brank = 0xffffffffu;
  const int S = g.S, C = g.C;
  for (int j = 0; j < B; ++j) {
    const int s = lane * B + j;
    if (s >= S) break;
    for (int p = 0; p < C; ++p) {
      const long long t = H.cand[p * S + s];
      const unsigned rank = (unsigned)((S - 1 - s) * C + p);  // scan order s desc, p asc
      if (t < bt || (t == bt && rank < brank)) {
        bt = t;
        brank = rank;
      }
    }
  }
}

template <bool TIMELINE>
__device__ long long atlas_row(const Geom& g, int mem_limit, const AtlasScratch& X,
                               AtlasShared& H, int& err) {
  const int lane = threadIdx.x & 31;
  const int S = g.S, M = g.M, C = g.C;
  const int B = (S + 31) / 32;
  const long long f = g.fwd, dur = g.dur;
  for (int i = lane; i < C * S; i += 32) {
    H.gf[i] = 0;
    H.nm[i] = 0;
  }
  for (int w = 0; w < GPB_MAX_DC; ++w) H.nres_f[w] = H.nres_b[w] = 0;
  __syncwarp();
  // a_s = s*f + sum_{i<s} delta_i, delta_i = WAN ? ser_pooled + lat : 0:
  // the chain offset of stage s.
  // Lane-local prefix then warp exclusive scan.
  long long a_loc[8];  // B <= 8 enforced on the host (S <= 256)
  long long run = 0;
  for (int j = 0; j < B; ++j) {
    const int s = lane * B + j;
    a_loc[j] = run;
    if (s < S) {
      run += f;
      int w;
      if (s + 1 < S && wan_after(g, s, w)) run += g.ser_pooled[w] + g.lat[w];
    }
  }
  long long incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = shfl_up64(incl, o);
    if (lane >= o) incl += v;
  }
  const long long excl = incl - run;
  for (int j = 0; j < B; ++j) a_loc[j] += excl;

  const int nw = g.nb - 1;  // WAN boundaries (ordinal w: producer stage blk_first[w+1]-1)

  // ---------------- forward phase (scheduler.cpp:362-431)
  for (int p = 0; p < C; ++p) {
    for (int m = 0; m < M; ++m) {
      // memory-cap admission with forced drains (atlas_drain_step)
      for (;;) {
        bool blk = false;
        for (int j = 0; j < B; ++j) {
          const int s = lane * B + j;
          if (s < S && m - H.nm[p * S + s] >= mem_limit) blk = true;
        }
        if (!__any_sync(kFull, blk)) break;
        // deepest stage with a ready pair
        int my_s = -1;
        for (int j = 0; j < B; ++j) {
          const int s = lane * B + j;
          if (s >= S) break;
          const int dm = H.nm[p * S + s];
          if (dm >= M) continue;
          const bool ready = (s == S - 1) ? dm < m : H.nm[p * S + s + 1] > dm;
          if (ready) my_s = s;
        }
        const unsigned bal = __ballot_sync(kFull, my_s >= 0);
        if (bal == 0) {
          err = 1;  // DeadlockError (cannot happen)
          return 0;
        }
        const int src = 31 - __clz(bal);
        const int s = __shfl_sync(kFull, my_s, src);
        const int dm = H.nm[p * S + s];
        const long long ready = (s == S - 1) ? X.fdl[(size_t)p * M + dm]
                                             : X.garr[((size_t)p * S + s) * M + dm];
        const long long lo = imax(ready, H.gf[p * S + s]);
        const int w = wan_before_idx(g, s);
        long long t = lo;
        if (w >= 0) {
          long long* st = X.resb + (size_t)w * X.cap;
          t = resv_earliest_fit(st, H.nres_b[w], lo + dur, g.ser_pooled[w]) - dur;
          int n = H.nres_b[w];
          resv_insert_warp(st, n, t + dur, g.ser_pooled[w]);
          H.nres_b[w] = n;
        }
        if (lane == 0) {
          const long long e = t + dur;
          H.gf[p * S + s] = imax(H.gf[p * S + s], e);
          if (s > 0)
            X.garr[((size_t)p * S + s - 1) * M + dm] =
                w >= 0 ? e + g.ser_pooled[w] + g.lat[w] : e;
          if (TIMELINE) X.ps[((size_t)p * S + s) * M + dm] = t;
          H.nm[p * S + s] = dm + 1;
        }
        __syncwarp();
      }
      // chain fit: e_s(t0) = a_s + f + max(t0, G_s), G_s = max_{j<=s}(gf_j - a_j)
      long long gl[8];
      long long runmax = -kInf64;
      for (int j = 0; j < B; ++j) {
        const int s = lane * B + j;
        if (s < S) runmax = imax(runmax, H.gf[p * S + s] - a_loc[j]);
        gl[j] = runmax;
      }
      long long pre = runmax;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long v = shfl_up64(pre, o);
        if (lane >= o) pre = imax(pre, v);
      }
      long long prev = shfl_up64(pre, 1);
      if (lane == 0) prev = -kInf64;
      for (int j = 0; j < B; ++j) gl[j] = imax(gl[j], prev);
      // gather (a_w, G_w) of each WAN producer stage to every lane via smem
      for (int j = 0; j < B; ++j) {
        const int s = lane * B + j;
        if (s < S) {
          int w;
          if (s + 1 < S && wan_after(g, s, w)) {
            H.wa[w] = a_loc[j];
            H.wg[w] = gl[j];
          }
        }
      }
      __syncwarp();
      long long t0 = H.gf[p * S + 0];
      if (lane == 0) {
        for (;;) {
          bool ok = true;
          for (int w = 0; w < nw; ++w) {
            const long long e = H.wa[w] + f + imax(t0, H.wg[w]);
            const long long* st = X.resf + (size_t)w * X.cap;
            const long long len = g.ser_pooled[w];
            if (!resv_free_at(st, H.nres_f[w], e, len)) {
              const long long slot = resv_earliest_fit(st, H.nres_f[w], e, len);
              t0 += slot - e;
              ok = false;
              break;
            }
          }
          if (ok) break;
        }
      }
      t0 = __shfl_sync(kFull, t0, 0);
      // commit the chain
      for (int w = 0; w < nw; ++w) {
        const long long e = H.wa[w] + f + imax(t0, H.wg[w]);
        long long* st = X.resf + (size_t)w * X.cap;
        int n = H.nres_f[w];
        resv_insert_warp(st, n, e, g.ser_pooled[w]);
        H.nres_f[w] = n;
      }
      for (int j = 0; j < B; ++j) {
        const int s = lane * B + j;
        if (s < S) {
          const long long e = a_loc[j] + f + imax(t0, gl[j]);
          H.gf[p * S + s] = e;
          if (s == S - 1) X.fdl[(size_t)p * M + m] = e;
        }
      }
      __syncwarp();
    }
  }

  // ---------------- drain pass 1: greedy exact-fit (scheduler.cpp:452-505)
  for (int i = lane; i < C * S; i += 32) H.cand[i] = 0;
  __syncwarp();
  long long remaining = 0;
  for (int i = 0; i < C * S; ++i) remaining += M - H.nm[i];
  for (int j = 0; j < B; ++j) {
    const int s = lane * B + j;
    if (s >= S) break;
    for (int p = 0; p < C; ++p) H.cand[p * S + s] = atlas_candidate(g, X, H, p, s);
  }
  __syncwarp();
  long long lbt;
  unsigned lrank;
  lane_best(g, H, lane, B, lbt, lrank);
  while (remaining > 0) {
    // warp argmin of (t, rank): three redux.sync steps on 32-bit parts
    const unsigned hi = (unsigned)((unsigned long long)lbt >> 32);
    const unsigned mh = __reduce_min_sync(kFull, hi);
    const unsigned lo32 = hi == mh ? (unsigned)lbt : 0xffffffffu;
    const unsigned ml = __reduce_min_sync(kFull, lo32);
    const unsigned rk = (hi == mh && (unsigned)lbt == ml) ? lrank : 0xffffffffu;
    const unsigned mr = __reduce_min_sync(kFull, rk);
    const long long bt = (long long)(((unsigned long long)mh << 32) | ml);
    if (bt >= kInf64 || mr == 0xffffffffu) {
      err = 1;  // no ready candidate: cannot happen (last stage always ready)
      return 0;
    }
    const int bs = S - 1 - (int)(mr / C), bp = (int)(mr % C);
    const int bm = H.nm[bp * S + bs];
    const int w = wan_before_idx(g, bs);
    if (w >= 0) {
      long long* st = X.resb + (size_t)w * X.cap;
      int n = H.nres_b[w];
      resv_insert_warp(st, n, bt + dur, g.ser_pooled[w]);
      H.nres_b[w] = n;
    }
    if (lane == 0) {
      H.gf[bp * S + bs] = bt + dur;
      if (bs > 0)
        X.garr[((size_t)bp * S + bs - 1) * M + bm] =
            w >= 0 ? bt + dur + g.ser_pooled[w] + g.lat[w] : bt + dur;
      if (TIMELINE) X.ps[((size_t)bp * S + bs) * M + bm] = bt;
      H.nm[bp * S + bs] = bm + 1;
    }
    __syncwarp();
    // refresh the candidates that changed: stage bs (all p when its
    // gradient link is shared, else bp) and (bp, bs-1).
    const int owner = bs / B, owner2 = bs > 0 ? (bs - 1) / B : -1;
    if (lane == owner) {
      if (w >= 0) {
        for (int p = 0; p < C; ++p) H.cand[p * S + bs] = atlas_candidate(g, X, H, p, bs);
      } else {
        H.cand[bp * S + bs] = atlas_candidate(g, X, H, bp, bs);
      }
    }
    __syncwarp();
    if (lane == owner2) H.cand[bp * S + bs - 1] = atlas_candidate(g, X, H, bp, bs - 1);
    __syncwarp();
    if (lane == owner || lane == owner2) lane_best(g, H, lane, B, lbt, lrank);
    --remaining;
  }
  long long mk = 0;
  for (int i = lane; i < C * S; i += 32) mk = imax(mk, H.gf[i]);
  return warp_max64(mk);
}

__global__ void __launch_bounds__(kEvalThreads) atlas_kernel(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + warp;
  unsigned char* base = smem + (size_t)warp * a.smem_warp_bytes;
  AtlasShared H;
  H.wa = reinterpret_cast<long long*>(base);
  H.wg = H.wa + GPB_MAX_DC;
  H.gf = H.wg + GPB_MAX_DC;
  H.cand = H.gf + a.smem_cs;
  H.nm = reinterpret_cast<int*>(H.cand + a.smem_cs);
  AtlasScratch X;
  X.cap = a.res_cap;
  X.garr = a.scratch + (size_t)gwarp * a.scratch_per_warp;
  X.fdl = X.garr + a.scratch_csm;
  X.resf = X.fdl + a.scratch_cm;
  X.resb = X.resf + (size_t)(GPB_MAX_DC - 1) * a.res_cap;
  X.ps = nullptr;
  for (;;) {
    const int wk = next_work(a.cursor);
    if (wk >= a.n_work) break;
    const int row = a.work[wk];
    Geom g;
    const DevScen* sc;
    const DevTopo* tp;
    if (!begin_row(a, row, g, sc, tp)) continue;
    int err = 0;
    const long long mk = atlas_row<false>(g, sc->mem_limit, X, H, err);
    end_row(a, row, g, *sc, *tp, mk, err);
    __syncwarp();
  }
}

// -------------------------------------------------------------- select

// One warp per scenario: select()'s strict-`>` argmax over its D rows
// (dc_select.cpp:110-121), chosen flags, gpus_used, and a per-block best.
__global__ void __launch_bounds__(kEvalThreads) select_kernel(SelectArgs a) {
  __shared__ double bthr[kEvalThreads / 32];
  __shared__ long long brow[kEvalThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double best_thr = -1.0;
  long long best_row = -1;
  for (int si = blockIdx.x * (blockDim.x >> 5) + warp; si < a.n_scen;
       si += gridDim.x * (blockDim.x >> 5)) {
    const DevScen& sc = a.scens[si];
    // chunked scan: lane-local first max, then ordered warp combine
    double cthr = -1.0;
    int cd = 0;
    for (int base = 0; base < sc.n_rows; base += 32) {
      const int d = base + lane + 1;
      double thr = -1.0;
      if (d <= sc.n_rows) {
        const gpb_row& r = a.rows[sc.first_row + d - 1];
        if (r.feasible == 1) thr = r.throughput;
      }
      // reduce (thr desc, d asc) across the chunk
      double vt = thr;
      int vd = thr >= 0 ? d : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ot = __shfl_xor_sync(kFull, vt, o);
        const int od = __shfl_xor_sync(kFull, vd, o);
        if (ot > vt || (ot == vt && od < vd)) {
          vt = ot;
          vd = od;
        }
      }
      // strict '>' against rows of earlier chunks keeps the first maximum
      if (vt >= 0 && (cd == 0 || vt > cthr)) {
        cthr = vt;
        cd = vd;
      }
    }
    for (int base = 0; base < sc.n_rows; base += 32) {
      const int d = base + lane + 1;
      if (d <= sc.n_rows) a.rows[sc.first_row + d - 1].chosen = d == cd ? 1 : 0;
    }
    if (lane == 0) {
      gpb_scenario_result res;
      res.first_row = sc.first_row;
      res.n_rows = sc.n_rows;
      res.chosen_d = cd;
      res.gpus_used = cd > 0 ? (long long)cd * sc.C * sc.S * sc.tp : 0;
      a.results[si] = res;
    }
    if (cd > 0) {
      const long long row = sc.first_row + cd - 1;
      if (cthr > best_thr || (cthr == best_thr && row < best_row)) {
        best_thr = cthr;
        best_row = row;
      }
    }
  }
  if (lane == 0) {
    bthr[warp] = best_thr;
    brow[warp] = best_row;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      if (bthr[w] > bthr[0] || (bthr[w] == bthr[0] && brow[w] >= 0 &&
                                (brow[0] < 0 || brow[w] < brow[0]))) {
        bthr[0] = bthr[w];
        brow[0] = brow[w];
      }
    }
    a.block_best[blockIdx.x].throughput = bthr[0];
    a.block_best[blockIdx.x].row = brow[0];
  }
}

__global__ void best_reduce_kernel(const gpb_best* in, int n, gpb_best* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    gpb_best b;
    b.throughput = -1.0;
    b.row = -1;
    for (int i = 0; i < n; ++i) {
      if (in[i].row < 0) continue;
      if (b.row < 0 || in[i].throughput > b.throughput ||
          (in[i].throughput == b.throughput && in[i].row < b.row))
        b = in[i];
    }
    if (b.row < 0) b.throughput = 0.0;
    *out = b;
  }
}

// -------------------------------------------------------------- launchers

template <int B>
static cudaError_t launch_flush_b(bool gpipe, const EvalArgs& a, int grid, cudaStream_t st) {
  const size_t smem = (size_t)(kEvalThreads / 32) * a.smem_m * sizeof(long long);
  if (gpipe) {
    cudaFuncSetAttribute(flush_kernel<B, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    flush_kernel<B, true><<<grid, kEvalThreads, smem, st>>>(a);
  } else {
    cudaFuncSetAttribute(flush_kernel<B, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    flush_kernel<B, false><<<grid, kEvalThreads, smem, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_flush(int B, bool gpipe, const EvalArgs& a, int grid, cudaStream_t st) {
  switch (B) {
    case 1: return launch_flush_b<1>(gpipe, a, grid, st);
    case 2: return launch_flush_b<2>(gpipe, a, grid, st);
    case 3: return launch_flush_b<3>(gpipe, a, grid, st);
    case 4: return launch_flush_b<4>(gpipe, a, grid, st);
    case 5: return launch_flush_b<5>(gpipe, a, grid, st);
    case 6: return launch_flush_b<6>(gpipe, a, grid, st);
    case 7: return launch_flush_b<7>(gpipe, a, grid, st);
    case 8: return launch_flush_b<8>(gpipe, a, grid, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_onef1b(int B, const EvalArgs& a, int grid, cudaStream_t st) {
  switch (B) {
    case 1: onef1b_kernel<1><<<grid, kEvalThreads, 0, st>>>(a); break;
    case 2: onef1b_kernel<2><<<grid, kEvalThreads, 0, st>>>(a); break;
    case 3: onef1b_kernel<3><<<grid, kEvalThreads, 0, st>>>(a); break;
    case 4: onef1b_kernel<4><<<grid, kEvalThreads, 0, st>>>(a); break;
    case 5: onef1b_kernel<5><<<grid, kEvalThreads, 0, st>>>(a); break;
    case 6: onef1b_kernel<6><<<grid, kEvalThreads, 0, st>>>(a); break;
    case 7: onef1b_kernel<7><<<grid, kEvalThreads, 0, st>>>(a); break;
    case 8: onef1b_kernel<8><<<grid, kEvalThreads, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_atlas(const EvalArgs& a, int grid, cudaStream_t st) {
  const size_t smem = (size_t)(kEvalThreads / 32) * a.smem_warp_bytes;
  cudaFuncSetAttribute(atlas_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  atlas_kernel<<<grid, kEvalThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_select(const SelectArgs& a, int grid, cudaStream_t st) {
  select_kernel<<<grid, kEvalThreads, 0, st>>>(a);
  best_reduce_kernel<<<1, 32, 0, st>>>(a.block_best, grid, a.best);
  return cudaGetLastError();
}

}  // namespace gpb

// ------------------------------------------------------- microbenchmark

namespace gpb {

// Peak int64 max-plus issue rate: 8 independent chains per thread of
// x = max(x + a, y) (2 ops per update), every SM fully occupied.
__global__ void __launch_bounds__(256) maxplus_bench_kernel(long long* out, int iters,
                                                             long long a, long long y0) {
  long long x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  long long y = y0 + blockIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = imax(x[k] + a, y + k);
  }
  long long s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= x[k];
  if (s == 0x5a5a5a5a5a5a5aLL) out[0] = s;
}

cudaError_t launch_maxplus_bench(long long* out, int grid, int iters, cudaStream_t st) {
  maxplus_bench_kernel<<<grid, 256, 0, st>>>(out, iters, 3, 1LL << 40);
  return cudaGetLastError();
}

}  // namespace gpb
