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
//  atlas_kernel            atlas (scheduler.cpp:276-538), in kernels_atlas.cu
//      forward chains via a warp max-plus scan and O(#WAN) exact-fit checks,
//      memory-cap forced drains as rounds of warp suffix scans, then the
//      drain stage by stage (per-stage greedy / prefix-max scans).
//
// Every kernel pulls rows from a per-bucket work list with an atomic cursor
// (persistent warps) and finishes each row with finish_row() (all-reduce,
// throughput, utilization).
#include <cuda_runtime.h>

#include "eval_common.cuh"

namespace gpb {

// ---------------------------------------------------------------- flush

template <int B, bool GPIPE, bool TL = false>
__device__ long long flush_row(const Geom& g, long long* fdl, long long* tfe = nullptr,
                               long long* tps = nullptr) {
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
          if (TL) tfe[(size_t)s * M + m] = e;
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
          if (TL) tps[(size_t)s * M + m] = z - g.dur;
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
    const long long t_start = clock64();
    Geom g;
    const DevScen* sc;
    const DevTopo* tp;
    if (!begin_row(a, row, g, sc, tp)) continue;
    const long long mk = flush_row<B, GPIPE>(g, fdl);
    end_row(a, row, g, *sc, *tp, mk, 0, t_start);
    __syncwarp();
  }
}

// Shallow pipelines (S <= GW <= 16): 32/GW rows per warp, one group of GW
// lanes per row (lane = stage), the same wavefronts as flush_row with
// segmented shuffles. The loop bounds are the warp's maximum so every lane
// reaches every shuffle; a group past its own row's range idles.
template <bool GPIPE, int GW>
__global__ void __launch_bounds__(kEvalThreads) flush_group_kernel(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NG = 32 / GW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gi = lane / GW, s = lane % GW;  // group in the warp, stage in the row
  long long* fdl = reinterpret_cast<long long*>(smem) + ((size_t)warp * NG + gi) * a.smem_m;
  for (;;) {
    int w0 = 0;
    if (lane == 0) w0 = atomicAdd(a.cursor, NG);
    w0 = __shfl_sync(kFull, w0, 0);
    if (w0 >= a.n_work) break;
    const int wk = w0 + gi;
    const long long t_start = clock64();
    bool ok = false;
    int row = 0, si = 0;
    Geom g;
    if (wk < a.n_work) {
      row = a.work[wk];
      si = a.row_scen[row];
      const DevScen& sc = a.scens[si];
      const int d = (int)(row - sc.first_row) + 1;
      decode(sc, a.topos[sc.topo], d, g);
      ok = g.feasible;
      if (!ok && s == 0) {
        gpb_row r;
        infeasible_row(r);
        r.scenario = si;
        r.d = d;
        a.rows[row] = r;
      }
    }
    const int S = ok ? g.S : 0, M = ok ? g.M : 0;
    const int K = S > 0 ? S - 1 : 0;  // the group's last stage lane
    int T = ok ? M + K : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) T = max(T, __shfl_xor_sync(kFull, T, o));
    StageLinks<1> L;
    if (ok) L.load(g, s, false);
    long long gf = 0, lf = 0, lb = 0;
    const long long fwd = ok ? g.fwd : 0, dur = ok ? g.dur : 0;
    // forward: E[s][m] = max(A[s][m], E[s][m-1]) + f; link FIFO per boundary
    long long a_in = 0;
    for (int t = 0; t < T; ++t) {
      const int m = t - s;
      long long av = s == 0 ? 0 : a_in;
      if (ok && s <= K && m >= 0 && m < M) {
        const long long e = imax(av, gf) + fwd;
        gf = e;
        if (s == S - 1) fdl[m] = e;
        if (L.wanf & 1u) {
          const long long occ = imax(e, lf) + L.serf[0];
          lf = occ;
          av = occ + L.latf[0];
        } else {
          av = e;
        }
      }
      a_in = __shfl_up_sync(kFull, av, 1, GW);
    }
    __syncwarp();
    const long long beta = GPIPE && ok ? fdl[M - 1] : 0;  // barrier_last_fwd
    // drain: stages S-1..0, microbatch order k (varuna) or M-1-k (gpipe)
    long long g_in = 0;
    for (int t = 0; t < T; ++t) {
      const int i = t - (K - s);
      long long gv = g_in;
      if (ok && s <= K && i >= 0 && i < M) {
        const int m = GPIPE ? M - 1 - i : i;
        long long ready = s == S - 1 ? fdl[m] : gv;
        ready = imax(ready, beta);
        const long long z = imax(ready, gf) + dur;
        gf = z;
        if (s > 0) {
          if (L.wanb & 1u) {
            const long long occ = imax(z, lb) + L.serb[0];
            lb = occ;
            gv = occ + L.latb[0];
          } else {
            gv = z;
          }
        }
      }
      g_in = __shfl_down_sync(kFull, gv, 1, GW);
    }
    long long mk = ok && s < S ? gf : 0;
#pragma unroll
    for (int o = GW / 2; o > 0; o >>= 1) mk = imax(mk, __shfl_xor_sync(kFull, mk, o, GW));
    if (ok && s == 0) {
      const DevScen& sc = a.scens[si];
      if (a.row_cycles) a.row_cycles[row] = clock64() - t_start;
      gpb_row r;
      infeasible_row(r);
      r.scenario = si;
      r.d = g.D;
      finish_row(sc, a.topos[sc.topo], g, mk, r);
      a.rows[row] = r;
    }
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

template <int B, bool TL = false>
__device__ long long onef1b_row(const Geom& g, int& err, long long* tfe = nullptr,
                                long long* tps = nullptr) {
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
        if (TL) tfe[(size_t)s * M + m] = e;
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
        if (TL) tps[(size_t)s * M + m] = z - g.dur;
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

// Shallow 1F1B pipelines (S <= GW <= 16): 32/GW rows per warp, one group of
// GW lanes per row (lane = stage), onef1b_row's lock-step rounds with
// segmented shuffles; the round loop runs while any row of the warp is busy.
template <int GW>
__global__ void __launch_bounds__(kEvalThreads) onef1b_group_kernel(EvalArgs a) {
  constexpr int NG = 32 / GW;
  const int lane = threadIdx.x & 31;
  const int gi = lane / GW, s = lane % GW;
  for (;;) {
    int w0 = 0;
    if (lane == 0) w0 = atomicAdd(a.cursor, NG);
    w0 = __shfl_sync(kFull, w0, 0);
    if (w0 >= a.n_work) break;
    const int wk = w0 + gi;
    const long long t_start = clock64();
    bool ok = false;
    int row = 0, si = 0;
    Geom g;
    if (wk < a.n_work) {
      row = a.work[wk];
      si = a.row_scen[row];
      const DevScen& sc = a.scens[si];
      const int d = (int)(row - sc.first_row) + 1;
      decode(sc, a.topos[sc.topo], d, g);
      ok = g.feasible;
      if (!ok && s == 0) {
        gpb_row r;
        infeasible_row(r);
        r.scenario = si;
        r.d = d;
        a.rows[row] = r;
      }
    }
    const int S = ok ? g.S : 0, M = ok ? g.M : 0;
    StageLinks<1> L;
    if (ok) L.load(g, s, false);
    int pc = ok && s < S ? 0 : 2 * M, nF = 0, nB = 0;
    long long gf = 0, lf = 0, lb = 0, outF = 0, outB = 0, fdo = 0;
    int bad = 0;
    for (;;) {
      if (!__any_sync(kFull, pc < 2 * M)) break;
      // snapshots of the neighbours' state at the start of the round
      const int lnF = __shfl_up_sync(kFull, nF, 1, GW);
      const long long loutF = __shfl_up_sync(kFull, outF, 1, GW);
      const int rnB = __shfl_down_sync(kFull, nB, 1, GW);
      const long long routB = __shfl_down_sync(kFull, outB, 1, GW);
      if (pc >= 2 * M) continue;
      const int w = min(S - s, M);
      bool fwd;
      int m;
      onef1b_item(pc, w, M, fwd, m);
      if (fwd) {
        long long arr = 0;
        if (s > 0) {
          if (lnF <= m) continue;           // input not produced yet
          if (lnF > m + 1) bad = 1;         // mailbox depth invariant
          arr = loutF;
        }
        const long long e = imax(arr, gf) + g.fwd;
        gf = e;
        fdo = e;
        if (s + 1 < S) {
          if (L.wanf & 1u) {
            const long long occ = imax(e, lf) + L.serf[0];
            lf = occ;
            outF = occ + L.latf[0];
          } else {
            outF = e;
          }
        }
        nF += 1;
      } else {
        long long ready;
        if (s == S - 1) {
          if (nF <= m) continue;
          ready = fdo;  // F(S-1, m) immediately precedes B(S-1, m)
        } else {
          if (rnB <= m) continue;
          if (rnB > m + 1) bad = 1;
          ready = routB;
        }
        const long long z = imax(ready, gf) + g.dur;
        gf = z;
        if (s > 0) {
          if (L.wanb & 1u) {
            const long long occ = imax(z, lb) + L.serb[0];
            lb = occ;
            outB = occ + L.latb[0];
          } else {
            outB = z;
          }
        }
        nB += 1;
      }
      pc += 1;
    }
    long long mk = ok && s < S ? gf : 0;
#pragma unroll
    for (int o = GW / 2; o > 0; o >>= 1) {
      mk = imax(mk, __shfl_xor_sync(kFull, mk, o, GW));
      bad |= __shfl_xor_sync(kFull, bad, o, GW);
    }
    if (ok && s == 0) {
      const DevScen& sc = a.scens[si];
      if (a.row_cycles) a.row_cycles[row] = clock64() - t_start;
      gpb_row r;
      infeasible_row(r);
      r.scenario = si;
      r.d = g.D;
      finish_row(sc, a.topos[sc.topo], g, mk, r);
      if (bad) {
        r.feasible = -1;  // kernel-side invariant failure: host raises GPB_ERROR
        atomicExch(a.error_flag, 1);
      }
      a.rows[row] = r;
    }
    __syncwarp();
  }
}

template <int B>
__global__ void __launch_bounds__(kEvalThreads) onef1b_kernel(EvalArgs a) {
  for (;;) {
    const int w = next_work(a.cursor);
    if (w >= a.n_work) break;
    const int row = a.work[w];
    const long long t_start = clock64();
    Geom g;
    const DevScen* sc;
    const DevTopo* tp;
    if (!begin_row(a, row, g, sc, tp)) continue;
    int err = 0;
    const long long mk = onef1b_row<B>(g, err);
    end_row(a, row, g, *sc, *tp, mk, err, t_start);
    __syncwarp();
  }
}

// ------------------------------------------------------------- timeline

// Timeline variants for gpipe/1f1b/varuna: every pipeline of a cell is
// identical, so pipeline 0 stands for all of them.
template <int B, int POLICY>
__global__ void __launch_bounds__(kEvalThreads) timeline_kernel(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  long long* fdl = reinterpret_cast<long long*>(smem) + (size_t)warp * a.smem_m;
  for (;;) {
    const int w = next_work(a.cursor);
    if (w >= a.n_work) break;
    const int row = a.work[w];
    const long long t_start = clock64();
    Geom g;
    const DevScen* sc;
    const DevTopo* tp;
    if (!begin_row(a, row, g, sc, tp)) continue;
    long long* tfe = a.tl_fe + a.tl_off[w];
    long long* tps = a.tl_ps + a.tl_off[w];
    int err = 0;
    long long mk;
    if (POLICY == GPB_1F1B) {
      mk = onef1b_row<B, true>(g, err, tfe, tps);
    } else {
      mk = flush_row<B, POLICY == GPB_GPIPE, true>(g, fdl, tfe, tps);
    }
    end_row(a, row, g, *sc, *tp, mk, err, t_start);
    __syncwarp();
  }
}

template <int B>
static cudaError_t launch_timeline_b(int policy, const EvalArgs& a, int grid, cudaStream_t st) {
  const size_t smem = (size_t)(kEvalThreads / 32) * a.smem_m * sizeof(long long);
  if (policy == GPB_GPIPE) {
    cudaFuncSetAttribute(timeline_kernel<B, GPB_GPIPE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    timeline_kernel<B, GPB_GPIPE><<<grid, kEvalThreads, smem, st>>>(a);
  } else if (policy == GPB_VARUNA) {
    cudaFuncSetAttribute(timeline_kernel<B, GPB_VARUNA>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    timeline_kernel<B, GPB_VARUNA><<<grid, kEvalThreads, smem, st>>>(a);
  } else {
    timeline_kernel<B, GPB_1F1B><<<grid, kEvalThreads, 0, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_timeline(int policy, int B, const EvalArgs& a, int grid, cudaStream_t st) {
  switch (B) {
    case 1: return launch_timeline_b<1>(policy, a, grid, st);
    case 2: return launch_timeline_b<2>(policy, a, grid, st);
    case 3: return launch_timeline_b<3>(policy, a, grid, st);
    case 4: return launch_timeline_b<4>(policy, a, grid, st);
    case 5: return launch_timeline_b<5>(policy, a, grid, st);
    case 6: return launch_timeline_b<6>(policy, a, grid, st);
    case 7: return launch_timeline_b<7>(policy, a, grid, st);
    case 8: return launch_timeline_b<8>(policy, a, grid, st);
  }
  return cudaErrorInvalidValue;
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
  for (int wi = blockIdx.x * (blockDim.x >> 5) + warp; wi < a.n_scen;
       wi += gridDim.x * (blockDim.x >> 5)) {
    const int si = a.scen_list ? a.scen_list[wi] : wi;
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

// (throughput desc, row asc) over the per-block winners; one warp, lanes
// strided over the blocks, then a shuffle combine (rows < 0 are empty)
__global__ void best_reduce_kernel(const gpb_best* in, int n, gpb_best* out) {
  const int lane = threadIdx.x & 31;
  double bt = -1.0;
  long long br = -1;
  for (int i = lane; i < n; i += 32) {
    const gpb_best v = in[i];
    if (v.row < 0) continue;
    if (br < 0 || v.throughput > bt || (v.throughput == bt && v.row < br)) {
      bt = v.throughput;
      br = v.row;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ot = __shfl_xor_sync(kFull, bt, o);
    const long long orow = __shfl_xor_sync(kFull, br, o);
    if (orow >= 0 && (br < 0 || ot > bt || (ot == bt && orow < br))) {
      bt = ot;
      br = orow;
    }
  }
  if (lane == 0) {
    gpb_best b;
    b.throughput = br < 0 ? 0.0 : bt;
    b.row = br;
    *out = b;
  }
}

// -------------------------------------------------------------- launchers

template <int B>
static cudaError_t launch_flush_b(bool gpipe, const EvalArgs& a, int grid, cudaStream_t st) {
  const size_t smem = (size_t)(kEvalThreads / 32) * a.smem_m * sizeof(long long);
  // (above the default 48 KB only: the attribute call costs host time per launch)
  if (gpipe) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(flush_kernel<B, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
    flush_kernel<B, true><<<grid, kEvalThreads, smem, st>>>(a);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(flush_kernel<B, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
    flush_kernel<B, false><<<grid, kEvalThreads, smem, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_flush_group(int gw, bool gpipe, const EvalArgs& a, int grid, cudaStream_t st) {
  const size_t smem = (size_t)(kEvalThreads / gw) * a.smem_m * sizeof(long long);
  if (gw == 8) {
    if (gpipe) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(flush_group_kernel<true, 8>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      flush_group_kernel<true, 8><<<grid, kEvalThreads, smem, st>>>(a);
    } else {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(flush_group_kernel<false, 8>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      flush_group_kernel<false, 8><<<grid, kEvalThreads, smem, st>>>(a);
    }
  } else {
    if (gpipe) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(flush_group_kernel<true, 16>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      flush_group_kernel<true, 16><<<grid, kEvalThreads, smem, st>>>(a);
    } else {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(flush_group_kernel<false, 16>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      flush_group_kernel<false, 16><<<grid, kEvalThreads, smem, st>>>(a);
    }
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

cudaError_t launch_onef1b_group(int gw, const EvalArgs& a, int grid, cudaStream_t st) {
  if (gw == 8)
    onef1b_group_kernel<8><<<grid, kEvalThreads, 0, st>>>(a);
  else
    onef1b_group_kernel<16><<<grid, kEvalThreads, 0, st>>>(a);
  return cudaGetLastError();
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

cudaError_t launch_select(const SelectArgs& a, int grid, cudaStream_t st) {
  select_kernel<<<grid, kEvalThreads, 0, st>>>(a);
  best_reduce_kernel<<<1, 32, 0, st>>>(a.block_best, grid, a.best);
  return cudaGetLastError();
}

cudaError_t launch_select_part(const SelectArgs& a, int grid, cudaStream_t st) {
  select_kernel<<<grid, kEvalThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_best_reduce(const gpb_best* in, int n, gpb_best* out, cudaStream_t st) {
  best_reduce_kernel<<<1, 32, 0, st>>>(in, n, out);
  return cudaGetLastError();
}

}  // namespace gpb

// ------------------------------------------------------- microbenchmark

namespace gpb {

// Peak max-plus issue rate: 8 independent chains per thread of
// x = max(x + a, c_k) (2 ops per update), every SM fully occupied, in the
// three representations a max-plus recurrence on integer nanoseconds can use
// (SURVEY.md Appendix D): int64 (INT32-pair IADD3/IADD3.X + compare/select),
// exact-integer FP64 (DADD + DMNMX; exact while |t| < 2^53 ns) and int32
// (IADD + IMNMX; range-limited, for comparison).
template <typename T>
__device__ __forceinline__ T mp_max(T a, T b) { return a > b ? a : b; }
template <>
__device__ __forceinline__ double mp_max<double>(double a, double b) { return fmax(a, b); }

template <typename T>
__global__ void __launch_bounds__(256) maxplus_bench_kernel(long long* out, int iters, T a, T y0) {
  T x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = (T)(threadIdx.x + k);
  const T y = y0 + (T)blockIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = mp_max<T>(x[k] + a, y + (T)k);
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == (T)12345) out[0] = (long long)s;
}

// kind 0: int64, 1: FP64 (exact integers), 2: int32
cudaError_t launch_maxplus_bench(int kind, long long* out, int grid, int iters, cudaStream_t st) {
  if (kind == 1)
    maxplus_bench_kernel<double><<<grid, 256, 0, st>>>(out, iters, 3.0, 1099511627776.0);
  else if (kind == 2)
    maxplus_bench_kernel<int><<<grid, 256, 0, st>>>(out, iters, 3, 1 << 20);
  else
    maxplus_bench_kernel<long long><<<grid, 256, 0, st>>>(out, iters, 3, 1LL << 40);
  return cudaGetLastError();
}

}  // namespace gpb
