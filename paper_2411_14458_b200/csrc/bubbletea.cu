// bubbletea.cu — bubbles (extract_bubbles, bubbletea.cpp:20-66) and
// BubbleTea prefill packing (build_prefill_pipelines + schedule_prefills,
// bubbletea.cpp:88-222) for a set of plan rows, on sm_100a.
//
// 1. timeline kernels (kernels_eval.cu / kernels_atlas.cu) write forward
//    ends and pair starts per (pipeline, stage, microbatch) of cell 0 (all D
//    cells are identical; for gpipe/1f1b/varuna so are the pipelines);
// 2. gap_kernel: one thread per (row, pipeline, stage) merges forwards and
//    pairs in start order, clips to the horizon and emits gaps_of()'s gap
//    list with the before-training flags;
// 3. pack_kernel: one warp per row runs the FCFS request loop. For each
//    request the 32 lanes each take a prefill pipeline (first-fit = lowest
//    index: ballot + ffs) and find its earliest common start t0 >= arrival by
//    a leapfrog over the D stage GPUs: a stage that does not fit at t bumps t
//    to the next gap start (minus its offset) that can hold it. The minimum
//    feasible t0 over the reals is always one of the reference's candidates
//    ({arrival} U {gap.start - off_k}), so the first feasible candidate the
//    reference finds is exactly this minimum. The winning lane set commits
//    the split of each stage's gap (copy-on-write per GPU list).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/geopipe_batch.h"
#include "eval_common.cuh"
#include "host_internal.h"

namespace gpb {

// Packed gaps (longlong2): x = start, y = end | kGapFl when the next span is a
// training task (gaps_of's before_training, bubbletea.cpp:48).
constexpr long long kGapFl = 1LL << 62;

// Per-row descriptor of a timeline / packing slot.
struct TlSlot {
  long long row;
  long long tl_off;   // into fe / ps  ([Ce][S][M])
  long long gap_off;  // into gap arrays ([Ce][S][2M+1])
  long long lst_off;  // into per-list arrays ([Ce][S])
  long long horizon;  // <= 0: makespan of the row
  long long fwd, dur;
  long long ar_off;   // >= 0: all-reduce tail durations at ar_dur[ar_off + s]
  int S, M, Ce, C, D, policy;
};

// append_allreduce's task durations (scheduler.cpp:613-650): per stage,
// allreduce_time_ms (comm_model.cpp:38-41) of the stage's parameters over the
// D*C replicas at its DC's intra bandwidth, the same double operations as
// finish_row, rounded by ms_to_ns. One block per slot, threads over stages.
__global__ void ar_dur_kernel(const TlSlot* slots, int n_slots, const DevScen* scens,
                              const DevTopo* topos, const int32_t* row_scen, long long* ar_dur) {
  const int si = blockIdx.x;
  if (si >= n_slots) return;
  const TlSlot& sl = slots[si];
  if (sl.ar_off < 0) return;
  const DevScen& sc = scens[row_scen[sl.row]];
  const DevTopo& tp = topos[sc.topo];
  Geom g;
  decode(sc, tp, sl.D, g);
  const int n = sl.D * sc.C;
  for (int s = threadIdx.x; s < sl.S; s += blockDim.x) {
    const int begin = s * sc.lpp, end = min(begin + sc.lpp, sc.L);
    const double params = __dmul_rn(sc.ppl, (double)max(0, end - begin));
    double ms = 0.0;
    if (n > 1)
      ms = __ddiv_rn(__dmul_rn(__dmul_rn(4.0, params), (double)(n - 1)),
                     __dmul_rn((double)n, tp.intra_bw[g.blk_dc[block_of(g, s)]]));
    ar_dur[sl.ar_off + s] = ms_to_ns(ms);
  }
}

// Horizon per slot: the given one, else the makespan of the timeline incl.
// the optional all-reduce tail (append_allreduce, scheduler.cpp:613-650:
// each stage's all-reduce starts at the stage's last backward end over all
// replicas).
__global__ void horizon_kernel(const TlSlot* slots, int n_slots, const gpb_row* tl_rows,
                               const long long* ps, const long long* ar_dur,
                               long long* ar_start, long long* hz_out) {
  const int si = blockIdx.x;
  if (si >= n_slots) return;
  const TlSlot& sl = slots[si];
  long long mk = tl_rows[sl.row].makespan_ns;
  if (sl.ar_off >= 0) {
    for (int s = threadIdx.x; s < sl.S; s += blockDim.x) {
      long long last = 0;
      for (int p = 0; p < sl.Ce; ++p)
        for (int m = 0; m < sl.M; ++m)
          last = imax(last, ps[sl.tl_off + ((size_t)p * sl.S + s) * sl.M + m] + sl.dur);
      ar_start[sl.ar_off + s] = last;
      atomicMax((unsigned long long*)&hz_out[si], (unsigned long long)(last + ar_dur[sl.ar_off + s]));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (sl.horizon > 0) {
      hz_out[si] = sl.horizon;
    } else {
      hz_out[si] = imax(mk, sl.ar_off >= 0 ? hz_out[si] : 0);
    }
  }
}

__device__ __forceinline__ unsigned long long fnv_mix(unsigned long long h, unsigned long long v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xffu;
    h *= 1099511628211ull;
  }
  return h;
}

__global__ void gap_kernel(const TlSlot* slots, int n_slots, const long long* fe,
                           const long long* ps, const long long* ar_dur,
                           const long long* ar_start, long long* glo, long long* ghi,
                           unsigned char* gflag, longlong2* gpk, int* gcnt, long long* gsum, int* ghas,
                           const long long* hz) {
  // grid.y = slot, threads over its (pipeline, stage) lists
  const int si = blockIdx.y;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (si >= n_slots) return;
  const TlSlot& sl = slots[si];
  if (gid >= (long long)sl.Ce * sl.S) return;
  const int M = sl.M;
  const int li = (int)gid;  // = p * S + s
  const long long H = hz[si];
  const int s_idx = li % sl.S;
  const bool ar = sl.ar_off >= 0;
  const long long ar_lo = ar ? ar_start[sl.ar_off + s_idx] : 0;
  const long long ar_hi = ar ? ar_lo + ar_dur[sl.ar_off + s_idx] : 0;
  const long long* F = fe + sl.tl_off + (size_t)li * M;
  const long long* P = ps + sl.tl_off + (size_t)li * M;
  long long* lo_out = glo + sl.gap_off + (size_t)li * (2 * M + 1);
  long long* hi_out = ghi + sl.gap_off + (size_t)li * (2 * M + 1);
  unsigned char* fl_out = gflag + sl.gap_off + (size_t)li * (2 * M + 1);
  longlong2* pk_out = gpk + sl.gap_off + (size_t)li * (2 * M + 1);
  const bool rev = sl.policy == GPB_GPIPE;  // gpipe drains in reverse order
  int i_f = 0, i_p = 0, n = 0, has = 0;
  long long cursor = 0, sum = 0;
  bool ar_done = !ar;
  while (i_f < M || i_p < M || !ar_done) {
    long long fs = kInf64, pst = kInf64;
    if (i_f < M) fs = F[i_f] - sl.fwd;
    if (i_p < M) pst = P[rev ? M - 1 - i_p : i_p];
    long long lo, hi;
    if (i_f >= M && i_p >= M) {  // the all-reduce tail comes last on its GPU
      lo = ar_lo;
      hi = ar_hi;
      ar_done = true;
    } else if (fs <= pst) {
      lo = fs;
      hi = fs + sl.fwd;
      ++i_f;
    } else {
      lo = pst;
      hi = pst + sl.dur;
      ++i_p;
    }
    lo = imax(lo, 0);  // busy_by_gpu clipping (bubbletea.cpp:24-26)
    hi = imin(hi, H);
    if (lo >= hi) continue;
    has = 1;
    if (lo > cursor) {  // gaps_of (bubbletea.cpp:44-53)
      lo_out[n] = cursor;
      hi_out[n] = lo;
      fl_out[n] = 1;  // the next span is a training task
      pk_out[n] = make_longlong2(cursor, lo | kGapFl);
      sum += lo - cursor;
      ++n;
    }
    cursor = imax(cursor, hi);
  }
  if (cursor < H) {
    lo_out[n] = cursor;
    hi_out[n] = H;
    fl_out[n] = 0;
    pk_out[n] = make_longlong2(cursor, H);
    sum += H - cursor;
    ++n;
  }
  gcnt[sl.lst_off + li] = n;
  gsum[sl.lst_off + li] = sum;
  ghas[sl.lst_off + li] = has;
}

// ------------------------------------------------------------ packing

struct PackArgs {
  const TlSlot* slots;
  int n_slots;
  const DevScen* scens;
  const DevTopo* topos;
  const int32_t* row_scen;
  const longlong2* gpk;      // base gap lists, packed (see ListView)
  const int* gcnt;
  const long long* gsum;
  const long long* hz;
  const gpb_request* reqs;
  long long n_req;
  const long long* sufmin;  // [r] = min arrival (ns) of requests r.. (caps stay valid)
  long long first_late_req_dummy;
  // prefill model (PrefillModel, bubbletea.h:38-58), pre-validated
  double sat_ms, stage_bw, lat_ms;
  int max_tokens, inf_layers, bpe, pad_;
  long long inf_hidden;
  long long guard_ns;
  // copy-on-write per-GPU lists
  longlong2* pool;
  const long long* pool_off;  // per slot [n_slots + 1]: its share of the gap pool
  int max_pipes;              // largest C*S over the slots (shared-memory caps)
  long long* stats;           // nullable: per-slot counters (GPB_PACK_STATS)
  unsigned* memo;             // [slot][pipeline][token bit]: search failed for all later arrivals
  int memo_words;             // 32-bit words per pipeline = ceil(max_tokens / 32)
  long long* gpu_off;       // [slot gpu base + gi]  -1 = shared
  int* gpu_cnt;
  int* gpu_cap;
  const long long* gpu_base;  // per slot offset into gpu_* arrays
  // outputs
  gpb_pack_summary* sums;
  gpb_placement* pl;        // nullable: [slot][req]
  int* overflow;
  const int* order;         // CTA -> slot, most expensive first (nullable)
  int order_base;           // first entry of `order` this launch covers
};

// A gap list: 16 bytes per gap (one load), x = start, y = end with the
// before-training flag in bit 62 (kGapFl).
struct ListView {
  const longlong2* e;
  int n;
  __device__ __forceinline__ long long lo(int j) const { return e[j].x; }
  __device__ __forceinline__ long long hi(int j) const { return e[j].y & (kGapFl - 1); }
  __device__ __forceinline__ bool fl(int j) const { return (e[j].y & kGapFl) != 0; }
};
__device__ __forceinline__ long long gap_ue(const longlong2& g, long long guard) {
  return (g.y & (kGapFl - 1)) - ((g.y & kGapFl) ? guard : 0);
}

__device__ __forceinline__ ListView view_of(const PackArgs& a, const TlSlot& sl, long long gb,
                                            int gi, int li_shared) {
  ListView v;
  const long long off = a.gpu_off[gb + gi];
  if (off >= 0) {
    v.e = a.pool + off;
    v.n = a.gpu_cnt[gb + gi];
  } else {
    const long long go = sl.gap_off + (long long)li_shared * (2 * sl.M + 1);
    v.e = a.gpk + go;
    v.n = a.gcnt[sl.lst_off + li_shared];
  }
  return v;
}

// last index j with lo[j] <= x, or -1
__device__ __forceinline__ int last_start_le(const ListView& v, long long x) {
  int lo = 0, hi = v.n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v.lo(mid) <= x) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

__device__ __forceinline__ long long usable_end(const ListView& v, int j, long long guard) {
  return gap_ue(v.e[j], guard);
}

// Gap that admits [lo, lo+dur) in the reference's scan (bubbletea.cpp:173-188):
// the last gap starting at or before lo, or — for a zero-length interval —
// the gap just before it when the two touch at lo. Returns -1 if none.
__device__ __forceinline__ int fitting_gap(const ListView& v, long long lo, long long dur,
                                           long long guard) {
  const int j = last_start_le(v, lo);
  if (j < 0) return -1;
  if (lo + dur <= usable_end(v, j, guard)) return j;
  if (dur == 0 && j >= 1 && v.hi(j - 1) == lo && usable_end(v, j - 1, guard) >= lo) return j - 1;
  return -1;
}

// Smallest gap start > x that can start a [start, start+dur) placement.
__device__ __forceinline__ long long next_start(const ListView& v, long long x, long long dur,
                                                long long guard) {
  for (int j = last_start_le(v, x) + 1; j < v.n; ++j) {
    const long long st = v.lo(j);
    if (st + dur <= usable_end(v, j, guard)) return st;
    if (dur == 0 && j >= 1 && v.hi(j - 1) == st && usable_end(v, j - 1, guard) >= st) return st;
  }
  return kInf64;
}

// last_start_le from a cursor c <= the answer (queries inside one search are
// non-decreasing): gallop forward, then bisect; c < -1 means unknown.
__device__ __forceinline__ int last_start_le_from(const ListView& v, long long x, int& c) {
  int j;
  if (c < -1) {
    j = last_start_le(v, x);
  } else {
    j = c;
    int step = 1;
    while (j + step < v.n && v.lo(j + step) <= x) {
      j += step;
      step <<= 1;
    }
    int lo = j + 1, hi = min(j + step, v.n);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (v.lo(mid) <= x) lo = mid + 1; else hi = mid;
    }
    j = lo - 1;
  }
  c = j;
  return j;
}

// fitting_gap / next_start given j = last_start_le(v, x)
__device__ __forceinline__ bool fits_at(const ListView& v, int j, long long lo, long long dur,
                                        long long guard) {
  if (j < 0) return false;
  if (lo + dur <= usable_end(v, j, guard)) return true;
  return dur == 0 && j >= 1 && v.hi(j - 1) == lo && usable_end(v, j - 1, guard) >= lo;
}

// One stage of a search at x = t + off_k: x itself when [x, x+dur) fits the
// gap the reference would use (fitting_gap), else the next start that can
// hold it (next_start, > x), or kInf64. `c` is the search cursor (last gap
// starting at or before the previous x; < -1: unknown). The common case — x
// has not passed the next gap's start — costs two independent 16-byte loads.
__device__ __forceinline__ long long stage_next(const ListView& v, int& c, long long x,
                                                long long dur, long long guard) {
  int j;
  longlong2 g = make_longlong2(0, 0);
  bool have = false;
  if (c >= -1) {
    const bool hn = c + 1 < v.n, hc = c >= 0;
    const longlong2 nx = hn ? v.e[c + 1] : make_longlong2(0, 0);
    const longlong2 cu = hc ? v.e[c] : make_longlong2(0, 0);
    if (!hn || nx.x > x) {
      j = c;
      g = cu;
      have = hc;
    } else {
      j = last_start_le_from(v, x, c);
    }
  } else {
    j = last_start_le(v, x);
  }
  c = j;
  if (j >= 0) {
    if (!have) g = v.e[j];
    if (x + dur <= gap_ue(g, guard)) return x;
    if (dur == 0 && j >= 1) {
      const longlong2 q = v.e[j - 1];
      if ((q.y & (kGapFl - 1)) == x && gap_ue(q, guard) >= x) return x;
    }
  }
  // next_start_from(v, j, dur, guard), with the previous gap carried
  for (++j; j < v.n; ++j) {
    const longlong2 e = v.e[j];
    if (e.x + dur <= gap_ue(e, guard)) return e.x;
    if (dur == 0 && j >= 1 && (g.y & (kGapFl - 1)) == e.x && gap_ue(g, guard) >= e.x) return e.x;
    g = e;
  }
  return kInf64;
}
__device__ __forceinline__ long long next_start_from(const ListView& v, int j, long long dur,
                                                     long long guard) {
  for (++j; j < v.n; ++j) {
    const long long st = v.lo(j);
    if (st + dur <= usable_end(v, j, guard)) return st;
    if (dur == 0 && j >= 1 && v.hi(j - 1) == st && usable_end(v, j - 1, guard) >= st) return st;
  }
  return kInf64;
}

// The shared (never copied) gap list li of a slot.
__device__ __forceinline__ ListView base_view(const PackArgs& a, const TlSlot& sl, int li) {
  ListView v;
  const long long go = sl.gap_off + (long long)li * (2 * sl.M + 1);
  v.e = a.gpk + go;
  v.n = a.gcnt[sl.lst_off + li];
  return v;
}

// Zero-length pieces at x_i = x0 + i*step (i < cnt) against one gap list: the
// shift to add to t so that the first failing piece reaches its next allowed
// point (next_start, bubbletea.cpp:164-188 for dur 0), 0 if every piece
// fits, kInf64 if one never can. A zero-length piece at x fits iff x lies in
// some gap's closed usable interval [lo, usable_end] (incl. the touching rule).
__device__ __forceinline__ long long zero_run_shift(const ListView& v, long long x0,
                                                    long long step, int cnt, long long guard) {
  int j = last_start_le(v, x0);
  long long i = 0;
  for (;;) {
    const long long x = x0 + i * step;
    while (j + 1 < v.n && v.lo(j + 1) <= x) ++j;
    if (!fits_at(v, j, x, 0, guard)) {
      const long long st = next_start_from(v, j, 0, guard);
      return st == kInf64 ? kInf64 : st - x;
    }
    if (step <= 0) return 0;
    // every point up to the end of gap j's usable interval fits too
    const long long ue = max(usable_end(v, j, guard), x);
    const long long ni = (ue - x0) / step + 1;
    if (ni >= cnt) return 0;
    i = ni;
  }
}

struct ReqGeom {
  long long d0, d1, ovh;
  int extra;
  __device__ __forceinline__ long long dur(int k) const { return k < extra ? d1 : d0; }
  __device__ __forceinline__ long long off(int k) const {
    return k <= extra ? (long long)k * (d1 + ovh)
                      : (long long)extra * (d1 + ovh) + (long long)(k - extra) * (d0 + ovh);
  }
};

__device__ __forceinline__ int gpu_index(int k, int pipe, int stage, int C, int S) {
  return (k * C + pipe) * S + stage;
}


// Upper bound on the usable room after time `a` on one GPU's gap list: the
// largest usable_end - max(start, a) over gaps ending at or after a, or -1
// when there is none (not even a zero-length interval fits).
__device__ __forceinline__ long long room_after(const ListView& v, long long a, long long guard) {
  long long best = -1;
  for (int j = v.n - 1; j >= 0; --j) {
    if (v.hi(j) < a) break;  // gaps are sorted: every earlier gap ends before a
    const long long ue = usable_end(v, j, guard), lo = max(v.lo(j), a);
    if (ue >= lo) best = max(best, ue - lo);
  }
  return best;
}

// Per-pipeline filter: every stage k of a request needs dur(k) <= room of its
// GPU after the arrival. capA = min room over stages k < extra (duration d1),
// capB = over k >= extra (d0). Rooms only shrink with commits (on the
// pipeline's own GPUs) and with a later reference time, so a bound computed
// at the minimum arrival of all requests still to come stays valid; it is
// recomputed when the pipeline commits or fails a full search.
__device__ __forceinline__ void pipeline_caps(const PackArgs& a, const TlSlot& sl, long long gb,
                                              int pi, long long arrival, int extra,
                                              long long& capA, long long& capB) {
  const int S = sl.S, C = sl.C, D = sl.D;
  const int pipe = pi / S, stage = pi % S;
  const int li = (sl.Ce > 1 ? pipe : 0) * S + stage;
  capA = kInf64;
  capB = kInf64;
  for (int k = 0; k < D; ++k) {
    const ListView v = view_of(a, sl, gb, gpu_index(k, pipe, stage, C, S), li);
    const long long r = room_after(v, arrival, a.guard_ns);
    if (k < extra) capA = min(capA, r); else capB = min(capB, r);
  }
}

// Group-parallel search: a group of gs lanes (power of two) evaluates one
// pipeline; lane gl of the group owns stages k = gl, gl+gs, ... At the
// current t every lane checks its stages' pieces [t+off_k, t+off_k+dur_k);
// a piece that does not fit proposes the next start at which it could
// (next_start - off_k); the group max of the proposals is the next t (no
// feasible start lies below any proposal). The fixpoint is the earliest
// common start t0 >= arrival, the minimum of the reference's candidate set
// (bubbletea.cpp:164-188), or kInf64. Every lane of the warp must call it
// (warp-synchronous); `pi < 0` marks an idle group. The lane's first kP
// stages keep their list view and search cursor in registers.
template <int kP>
__device__ __forceinline__ long long group_search(const PackArgs& a, const TlSlot& sl,
                                                  long long gb, int pi, long long arrival,
                                                  const ReqGeom& rg, int gs, long long& iters,
                                                  bool zrun) {
  // zrun: stages k >= extra have zero layers (D > inference_layers), so their
  // GPUs only ever hold zero-length prefills, which never change where a
  // zero-length piece fits: those stages are one run checked on the base list
  const int lane = threadIdx.x & 31, gl = lane & (gs - 1);
  const int S = sl.S, C = sl.C;
  const int D = zrun ? rg.extra : sl.D;  // stages searched one by one
  const int pipe = pi >= 0 ? pi / S : 0, stage = pi >= 0 ? pi % S : 0;
  const int li = (sl.Ce > 1 ? pipe : 0) * S + stage;
  long long t = pi >= 0 ? arrival : kInf64;
  bool active = pi >= 0;
  // (t only grows during a search and the lists do not change)
  ListView vv[kP];
  int cur[kP];
#pragma unroll
  for (int p = 0; p < kP; ++p) {
    cur[p] = -2;
    const int k = gl + p * gs;
    if (active && k < D) vv[p] = view_of(a, sl, gb, gpu_index(k, pipe, stage, C, S), li);
  }
  // Latest feasible start: piece k must end inside the last gap that can hold
  // it, so t <= usable_end - dur_k - off_k of that gap (the zero-length run:
  // its last point at or before the last usable end). A search fails as soon
  // as t passes the group minimum.
  long long lim = kInf64;
  auto stage_lim = [&](const ListView& v, int k) {
    const long long dk = rg.dur(k);
    int j = v.n - 1;
    while (j >= 0 && usable_end(v, j, a.guard_ns) - v.lo(j) < dk) --j;
    return j < 0 ? -kInf64 : usable_end(v, j, a.guard_ns) - dk - rg.off(k);
  };
  if (active) {
#pragma unroll
    for (int p = 0; p < kP; ++p)
      if (gl + p * gs < D) lim = min(lim, stage_lim(vv[p], gl + p * gs));
    for (int k = gl + kP * gs; k < D; k += gs)
      lim = min(lim, stage_lim(view_of(a, sl, gb, gpu_index(k, pipe, stage, C, S), li), k));
    if (zrun && gl == (D & (gs - 1))) {
      const ListView v = base_view(a, sl, li);
      long long ue = -kInf64;
      for (int j = v.n - 1; j >= 0 && ue == -kInf64; --j)
        if (usable_end(v, j, a.guard_ns) >= v.lo(j)) ue = usable_end(v, j, a.guard_ns);
      lim = min(lim, ue == -kInf64 ? -kInf64 : ue - rg.off(sl.D - 1));
    }
  }
  for (int o = gs >> 1; o > 0; o >>= 1) lim = min(lim, __shfl_xor_sync(kFull, lim, o));
  if (active && t > lim) {
    t = kInf64;
    active = false;
  }
  while (__any_sync(kFull, active)) {
    ++iters;
    long long prop = t;
    if (active) {
#pragma unroll
      for (int p = 0; p < kP; ++p) {
        const int k = gl + p * gs;
        if (k < D && prop != kInf64) {
          const long long off = rg.off(k), dk = rg.dur(k);
          const long long st = stage_next(vv[p], cur[p], t + off, dk, a.guard_ns);
          if (st != t + off) prop = st == kInf64 ? kInf64 : max(prop, st - off);
        }
      }
      for (int k = gl + kP * gs; k < D && prop != kInf64; k += gs) {
        const ListView v = view_of(a, sl, gb, gpu_index(k, pipe, stage, C, S), li);
        const long long off = rg.off(k), dk = rg.dur(k);
        if (fitting_gap(v, t + off, dk, a.guard_ns) < 0) {
          const long long st = next_start(v, t + off, dk, a.guard_ns);
          prop = st == kInf64 ? kInf64 : max(prop, st - off);
        }
      }
      if (zrun && gl == (D & (gs - 1)) && prop != kInf64) {  // the zero-length run
        const long long sh = zero_run_shift(base_view(a, sl, li), t + rg.off(D), rg.ovh,
                                            sl.D - D, a.guard_ns);
        prop = sh == kInf64 ? kInf64 : max(prop, t + sh);
      }
    }
    for (int o = gs >> 1; o > 0; o >>= 1) prop = max(prop, __shfl_xor_sync(kFull, prop, o));
    if (active) {
      if (prop == kInf64 || prop > lim) {
        t = kInf64;
        active = false;
      } else if (prop == t) {
        active = false;  // every stage fits at t
      } else {
        t = prop;
      }
    }
  }
  return t;
}

// Caps of pipeline pi at reference time `a_ref`, group-parallel over its
// stages (see pipeline_caps); every lane of the group gets the result.
__device__ __forceinline__ void group_caps(const PackArgs& a, const TlSlot& sl, long long gb,
                                           int pi, long long a_ref, int extra, int gs,
                                           long long& capA, long long& capB, bool zrun) {
  const int lane = threadIdx.x & 31, gl = lane & (gs - 1);
  const int S = sl.S, C = sl.C;
  const int D = zrun ? extra : sl.D;
  const int pipe = pi >= 0 ? pi / S : 0, stage = pi >= 0 ? pi % S : 0;
  const int li = (sl.Ce > 1 ? pipe : 0) * S + stage;
  capA = kInf64;
  capB = kInf64;
  if (pi >= 0) {
    for (int k = gl; k < D; k += gs) {
      const ListView v = view_of(a, sl, gb, gpu_index(k, pipe, stage, C, S), li);
      const long long r = room_after(v, a_ref, a.guard_ns);
      if (k < extra) capA = min(capA, r); else capB = min(capB, r);
    }
    // zero-length stages: their lists keep the base list's allowed points
    if (zrun && gl == (D & (gs - 1))) capB = room_after(base_view(a, sl, li), a_ref, a.guard_ns);
  }
  for (int o = gs >> 1; o > 0; o >>= 1) {
    capA = min(capA, __shfl_xor_sync(kFull, capA, o));
    capB = min(capB, __shfl_xor_sync(kFull, capB, o));
  }
}

// One CTA of W warps per plan runs the FCFS request loop
// (schedule_prefills, bubbletea.cpp:132-222). Requests are staged 32 per warp
// (one per lane: load, durations, arrival check) and searched speculatively
// by every warp at once on the batch-start state (phase 1); warp 0 then
// resolves the batch in FCFS order and commits (phase 2). A request is
// examined only if it passes the plan-wide bound (some pipeline's caps admit
// its durations).
// W = 4 for most plans (two CTAs per SM); the few most expensive plans get
// W = 8 in a concurrent launch (they set the kernel's makespan).
template <int W>
__global__ void __launch_bounds__(32 * W, 1) pack_kernel(PackArgs a) {
  extern __shared__ __align__(16) long long pk_smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int BW = 32 * W;  // requests per batch
  const int si = a.order ? a.order[a.order_base + blockIdx.x] : (int)blockIdx.x;
  if (si >= a.n_slots) return;
  const TlSlot& sl = a.slots[si];
  const long long H = a.hz[si];
  const int D = sl.D, C = sl.C, S = sl.S, Ce = sl.Ce;
  const long long gb = a.gpu_base[si];
  const int G = D * C * S;
  const int n_pipes = C * S;
  // build_prefill_pipelines (bubbletea.cpp:88-130): layers per cell
  const int base_l = a.inf_layers / D, extra = a.inf_layers % D;
  const bool zrun = base_l == 0;  // stages >= extra carry no layers
  const int d_eff = zrun ? extra + 1 : D;  // searched stages (+ the zero-length run)
  int gs = 1;
  while (gs < d_eff && gs < 32) gs <<= 1;
  const int ng = 32 / gs, grp = lane / gs, gl = lane & (gs - 1);
  unsigned* memo = a.memo + (size_t)si * a.max_pipes * a.memo_words;
  // shared: caps per pipeline, the batch table, per-batch "committed" flags
  long long* capA = pk_smem;
  long long* capB = capA + a.max_pipes;
  long long* tb_arr = capB + a.max_pipes;  // [BW] arrival
  long long* tb_d0 = tb_arr + BW;
  long long* tb_d1 = tb_d0 + BW;
  long long* tb_ovh = tb_d1 + BW;
  long long* tb_t1 = tb_ovh + BW;          // phase-1 start
  long long* tb_rstart = tb_t1 + BW;       // committed start (phase 2)
  unsigned long long* tb_fail = (unsigned long long*)(tb_rstart + BW);
  long long* tb_bound = (long long*)(tb_fail + BW);  // [0] max capA, [1] max capB
  int* tb_pipe1 = (int*)(tb_bound + 2);
  int* tb_rpipe = tb_pipe1 + BW;
  int* tb_tok = tb_rpipe + BW;
  int* tb_id = tb_tok + BW;
  int* tb_stop = tb_id + BW;  // pool overflow: every warp leaves
  unsigned char* cflag = (unsigned char*)(tb_stop + 4);
  for (int i = threadIdx.x; i < G; i += blockDim.x) a.gpu_off[gb + i] = -1;
  if (threadIdx.x == 0) *tb_stop = 0;
  const long long pool_base = a.pool_off[si], pool_cap = a.pool_off[si + 1] - pool_base;
  long long bump = 0;
  const int total_layers = max(1, base_l * D + extra);
  long long accepted = 0;
  unsigned long long hash = 1469598103934665603ull;
  long long st_exam = 0, st_search = 0, st_fail = 0, st_iter = 0, st_cyc_search = 0,
            st_cyc_caps = 0, st_cyc_commit = 0;
  const long long st_t0 = clock64();
  __syncthreads();
  // initial caps, at the earliest arrival
  const long long a0 = a.n_req > 0 ? a.sufmin[0] : 0;
  if (warp == 0) {
    for (int p0 = 0; p0 < n_pipes; p0 += ng) {
      const int pi = p0 + grp < n_pipes ? p0 + grp : -1;
      long long ca, cb;
      group_caps(a, sl, gb, pi, a0, extra, gs, ca, cb, zrun);
      if (pi >= 0 && gl == 0) {
        capA[pi] = ca;
        capB[pi] = cb;
      }
    }
    __syncwarp();
    long long mA = -kInf64, mB = -kInf64;
    for (int pi = lane; pi < n_pipes; pi += 32) {
      mA = max(mA, capA[pi]);
      mB = max(mB, capB[pi]);
    }
    mA = warp_max64(mA);
    mB = warp_max64(mB);
    if (lane == 0) {
      tb_bound[0] = mA;
      tb_bound[1] = mB;
    }
  }
  __syncthreads();
  for (long long r0 = 0; r0 < a.n_req; r0 += BW) {
    // stage 32 requests per warp: durations (prefill_duration_ms :68-76,
    // transfer :78-86, per-stage split :154-161)
    const int jb = warp * 32 + lane;  // index in the batch
    const long long r = r0 + jb;
    gpb_request q{};
    long long arrival = kInf64;
    ReqGeom rg{0, 0, 0, extra};
    double xfer = 0.0;
    bool live = false;
    if (r < a.n_req) {
      q = a.reqs[r];
      arrival = ms_to_ns(q.arrival_ms);
      live = arrival <= H;  // later arrivals cannot fit before the horizon
      if (live) {
        const double dur_ms =
            __ddiv_rn(__dmul_rn(a.sat_ms, (double)q.tokens), (double)a.max_tokens);
        const double bytes = (double)((long long)q.tokens * a.inf_hidden * a.bpe);
        xfer = __dadd_rn(a.lat_ms, __ddiv_rn(bytes, a.stage_bw));
        rg.ovh = ms_to_ns(xfer);
        rg.d1 = ms_to_ns(__ddiv_rn(__dmul_rn(dur_ms, (double)(base_l + 1)), (double)total_layers));
        rg.d0 = ms_to_ns(__ddiv_rn(__dmul_rn(dur_ms, (double)base_l), (double)total_layers));
      }
    }
    const bool in_range = r < a.n_req;
    const long long mA = tb_bound[0], mB = tb_bound[1];
    // Phase 1 — every staged request searches the batch-start state at once
    // (lane = request, pipelines in order, its stages checked with independent
    // loads). Commits only shrink gap lists and only on the committing
    // pipeline's own GPUs, so a pipeline infeasible at the batch start stays
    // infeasible for the rest of the batch, and a request's answer (pipeline,
    // earliest start) stays exact unless an earlier request of the batch
    // committed to that same pipeline (phase 2 re-searches those).
    const bool act = live && rg.d0 <= mB && (extra == 0 || rg.d1 <= mA);
    const int tok_l = q.tokens - 1;
    int pi_l = act ? 0 : n_pipes;
    int pipe1 = -1;
    long long t1 = kInf64;
    unsigned long long failm = 0;  // pipelines < 64 that failed this lane's search
    // Few active requests in the warp (the room bounds reject most of a long
    // trace) on a plan with many stages: search them one after another with
    // the whole warp (gs lanes per pipeline, ng pipelines at a time, the
    // lowest success wins, failures below it recorded) instead of one lane
    // per request walking all D stages alone. Same pipelines searched in the
    // same order on the same batch-start state: identical answers.
    // Cost model (stage checks per leapfrog round): one lane per request
    // walks its candidates one by one, max over lanes of (candidates x
    // d_eff); the warp takes the requests one by one, ng_c candidates at a
    // time with groups of gs_c lanes: sum over requests of ceil(candidates /
    // ng_c) x ceil(d_eff / gs_c).
    int n_cand = 0;  // pipelines whose caps and memo admit the request
    if (act)
      for (int pl = 0; pl < n_pipes; ++pl)
        n_cand += rg.d0 <= capB[pl] && (extra == 0 || rg.d1 <= capA[pl]) &&
                  !((memo[(size_t)pl * a.memo_words + (tok_l >> 5)] >> (tok_l & 31)) & 1u);
    const unsigned actm = __ballot_sync(kFull, n_cand > 0);
    const int gs_c = gs < 4 ? gs : 4, ng_c = 32 / gs_c, grp_c = lane / gs_c, gl_c = lane & (gs_c - 1);
    const int lane_cost = n_cand * d_eff;
    const int coop_cost = ((n_cand + ng_c - 1) / ng_c) * ((d_eff + gs_c - 1) / gs_c);
    if (actm && gs >= 4 &&
        __reduce_add_sync(kFull, coop_cost) < __reduce_max_sync(kFull, lane_cost)) {
      const long long tc = clock64();
      for (unsigned rem = actm; rem; rem &= rem - 1) {
        const int src = __ffs(rem) - 1;
        const long long arr_s = shfl_idx64(arrival, src);
        ReqGeom rg_s;
        rg_s.d0 = shfl_idx64(rg.d0, src);
        rg_s.d1 = shfl_idx64(rg.d1, src);
        rg_s.ovh = shfl_idx64(rg.ovh, src);
        rg_s.extra = extra;
        const int tok_s = __shfl_sync(kFull, tok_l, src);
        int win = -1;
        long long win_t = kInf64;
        unsigned long long fm = 0;  // this lane's failed pipelines (< 64) below the winner
        for (int c0 = 0; c0 < n_pipes && win < 0; c0 += 32) {
          const int pl = c0 + lane;
          bool cand = pl < n_pipes && rg_s.d0 <= capB[pl] && (extra == 0 || rg_s.d1 <= capA[pl]);
          if (cand)
            cand = !((memo[(size_t)pl * a.memo_words + (tok_s >> 5)] >> (tok_s & 31)) & 1u);
          unsigned pmask = __ballot_sync(kFull, cand);
          while (pmask && win < 0) {
            const unsigned bit = __fns(pmask, 0, grp_c + 1);  // one survivor per group
            const int pi = bit < 32 ? c0 + (int)bit : -1;
            st_search += pi >= 0 && gl_c == 0;
            const long long t = group_search<8>(a, sl, gb, pi, arr_s, rg_s, gs_c, st_iter, zrun);
            const unsigned ok = __ballot_sync(kFull, gl_c == 0 && pi >= 0 && t != kInf64);
            if (ok) {
              const int wl = __ffs(ok) - 1;  // lowest group = lowest pipeline
              win = __shfl_sync(kFull, pi, wl);
              win_t = shfl_idx64(t, wl);
            }
            if (gl_c == 0 && pi >= 0 && pi < 64 && t == kInf64 && (win < 0 || pi < win)) {
              fm |= 1ull << pi;
              ++st_fail;
            }
            for (int g = 0; g < ng_c && pmask; ++g) pmask &= pmask - 1;
          }
        }
        for (int o = 16; o > 0; o >>= 1) fm |= __shfl_xor_sync(kFull, fm, o);
        if (lane == src) {
          pipe1 = win;
          t1 = win_t;
          failm = fm;
        }
      }
      st_cyc_search += clock64() - tc;
    } else {
      const long long tc = clock64();
      for (;;) {
        int cand = -1;
        for (; pi_l < n_pipes; ++pi_l) {
          if (rg.d0 <= capB[pi_l] && (extra == 0 || rg.d1 <= capA[pi_l]) &&
              !((memo[(size_t)pi_l * a.memo_words + (tok_l >> 5)] >> (tok_l & 31)) & 1u)) {
            cand = pi_l;
            break;
          }
        }
        if (!__any_sync(kFull, cand >= 0)) break;
        st_search += cand >= 0;
        const long long t = group_search<8>(a, sl, gb, cand, arrival, rg, 1, st_iter, zrun);
        if (cand >= 0) {
          if (t != kInf64) {
            pipe1 = cand;
            t1 = t;
            pi_l = n_pipes;
          } else {
            ++st_fail;
            if (cand < 64) failm |= 1ull << cand;
            ++pi_l;
          }
        }
      }
      st_cyc_search += clock64() - tc;
    }
    tb_arr[jb] = arrival;
    tb_d0[jb] = rg.d0;
    tb_d1[jb] = rg.d1;
    tb_ovh[jb] = rg.ovh;
    tb_t1[jb] = t1;
    tb_fail[jb] = failm;
    tb_pipe1[jb] = pipe1;
    tb_rpipe[jb] = -1;
    tb_tok[jb] = tok_l;
    tb_id[jb] = q.id;
    __syncthreads();
    // Phase 2 (warp 0) — FCFS over the batch: commit each answer whose
    // pipeline no earlier request of the batch took; otherwise search again
    // from that pipeline on (warp-cooperative, lane groups over pipelines).
    if (warp == 0) {
      for (int i = lane; i < n_pipes; i += 32) cflag[i] = 0;
      __syncwarp();
      for (int w0 = 0; w0 < BW; w0 += 32) {
        if (*tb_stop) break;
        unsigned res = __ballot_sync(kFull, tb_pipe1[w0 + lane] >= 0);
        while (res && !*tb_stop) {
          ++st_exam;
          const int src = w0 + __ffs(res) - 1;
          res &= res - 1;
          int win = tb_pipe1[src];
          long long win_t = tb_t1[src];
          const long long a_ref = a.sufmin[r0 + src];  // <= every arrival from here on
          ReqGeom g2;
          g2.d0 = tb_d0[src];
          g2.d1 = tb_d1[src];
          g2.ovh = tb_ovh[src];
          g2.extra = extra;
          if (cflag[win]) {
            const long long tc = clock64();
            const int from = win;
            const long long arr = tb_arr[src];
            const int tok = tb_tok[src];
            win = -1;
            for (int c0 = from & ~31; c0 < n_pipes && win < 0; c0 += 32) {
              const int pl = c0 + lane;
              bool cand = pl >= from && pl < n_pipes && g2.d0 <= capB[pl] &&
                          (extra == 0 || g2.d1 <= capA[pl]);
              if (cand) cand = !((memo[(size_t)pl * a.memo_words + (tok >> 5)] >> (tok & 31)) & 1u);
              unsigned pmask = __ballot_sync(kFull, cand);
              while (pmask && win < 0) {
                // the next ng survivors, in pipeline order, one per group
                const unsigned bit = __fns(pmask, 0, grp + 1);
                const int pi = bit < 32 ? c0 + (int)bit : -1;
                st_search += pi >= 0 && gl == 0;
                const long long t = group_search<4>(a, sl, gb, pi, arr, g2, gs, st_iter, zrun);
                const unsigned ok = __ballot_sync(kFull, gl == 0 && pi >= 0 && t != kInf64);
                if (ok) {
                  const int wl = __ffs(ok) - 1;  // lowest group = lowest pipeline
                  win = __shfl_sync(kFull, pi, wl);
                  win_t = shfl_idx64(t, wl);
                }
                // failed searches below the winner (or all): tighten their caps
                const bool failed = pi >= 0 && t == kInf64 && (win < 0 || pi < win);
                st_fail += failed && gl == 0;
                // no start >= arr exists for this token count; every later request
                // arrives at or after arr when arr is the minimum of the rest
                if (failed && gl == 0 && arr == a_ref)
                  atomicOr(&memo[(size_t)pi * a.memo_words + (tok >> 5)], 1u << (tok & 31));
                if (__any_sync(kFull, failed)) {
                  long long ca, cb;
                  group_caps(a, sl, gb, failed ? pi : -1, a_ref, extra, gs, ca, cb, zrun);
                  if (failed && gl == 0) {
                    capA[pi] = ca;
                    capB[pi] = cb;
                  }
                }
                for (int g = 0; g < ng && pmask; ++g) pmask &= pmask - 1;
              }
            }
            st_cyc_caps += clock64() - tc;
          }
          __syncwarp();
          const long long tcm = clock64();
      if (win >= 0) {
        // commit (bubbletea.cpp:189-215): split the gap on each stage GPU,
        // one lane per stage GPU; copy-on-write lists come from the slot's
        // bump pool (warp prefix sum of the sizes)
        const int pipe = win / S, stage = win % S;
        const int li = (Ce > 1 ? pipe : 0) * S + stage;
        bool ovf = false;
        // (zero-length stages of a zrun plan only split gaps: no effect on
        // any later search, on the gap sums or on the summaries; skipped)
        const int D_commit = zrun ? extra : D;
        for (int k0 = 0; k0 < D_commit && !ovf; k0 += 32) {
          const int k = k0 + lane;
          const int gi = k < D_commit ? gpu_index(k, pipe, stage, C, S) : 0;
          const long long lo = k < D_commit ? win_t + g2.off(k) : 0,
                          hi = k < D_commit ? lo + g2.dur(k) : 0;
          int j = -1, need = 0, ncap = 0, n = 0;
          if (k < D_commit) {
            const ListView v0 = view_of(a, sl, gb, gi, li);
            j = fitting_gap(v0, lo, hi - lo, a.guard_ns);
            // a zero-length interval at a gap end changes nothing (upper_bound
            // insertion behind the span that ends the gap)
            need = j >= 0 && lo != v0.hi(j);
            const long long off = a.gpu_off[gb + gi];
            n = v0.n;
            const int cap = off >= 0 ? a.gpu_cap[gb + gi] : 0;
            if (need && !(off >= 0 && n + 1 <= cap)) ncap = max(2 * cap, n + 8);
          }
          int incl = ncap;
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
          }
          const int total = __shfl_sync(kFull, incl, 31);
          if (bump + total > pool_cap) {
            ovf = true;
            break;
          }
          if (ncap > 0) {  // private copy with room
            const long long noff = pool_base + bump + (incl - ncap);
            const ListView v = view_of(a, sl, gb, gi, li);
            for (int x = 0; x < n; ++x) a.pool[noff + x] = v.e[x];
            a.gpu_off[gb + gi] = noff;
            a.gpu_cnt[gb + gi] = n;
            a.gpu_cap[gb + gi] = ncap;
          }
          bump += total;
          if (need) {
            longlong2* E = a.pool + a.gpu_off[gb + gi];
            const longlong2 gj = E[j];
            const long long glo = gj.x, ghi = gj.y & (kGapFl - 1), gfl = gj.y & kGapFl;
            const int add_l = lo > glo, add_r = ghi > hi;
            const int delta = add_l + add_r - 1;
            if (delta > 0) {
              for (int x = n - 1; x > j; --x) E[x + 1] = E[x];
            } else if (delta < 0) {
              for (int x = j + 1; x < n; ++x) E[x - 1] = E[x];
            }
            int w = j;
            if (add_l) E[w++] = make_longlong2(glo, lo);  // the next span is this prefill
            if (add_r) E[w] = make_longlong2(hi, ghi | gfl);
            a.gpu_cnt[gb + gi] = n + delta;
          }
          __syncwarp();
        }
        if (ovf) {  // the whole CTA stops after this batch
          if (lane == 0) {
            atomicExch(a.overflow, 1);
            *tb_stop = 1;
          }
          __syncwarp();
          break;
        }
        ++accepted;
        const int id = tb_id[src];
        if (lane == 0) {
          hash = fnv_mix(hash, (unsigned long long)(long long)id);
          hash = fnv_mix(hash, (unsigned long long)(long long)win);
          hash = fnv_mix(hash, (unsigned long long)win_t);
          cflag[win] = 1;
        }
        if (lane == 0) {
          tb_rpipe[src] = win;
          tb_rstart[src] = win_t;
        }
        {  // the winner's GPU lists changed: its caps now
          long long ca, cb;
          group_caps(a, sl, gb, grp == 0 ? win : -1, a_ref, extra, gs, ca, cb, zrun);
          if (lane == 0) {
            capA[win] = ca;
            capB[win] = cb;
          }
        }
      }
          __syncwarp();
          st_cyc_commit += clock64() - tcm;
        }
      }
    }
    __syncthreads();
    if (*tb_stop) return;
    // every warp: its requests' placements; the phase-1 failures into the
    // memo (a failure at the minimum remaining arrival holds for every later
    // request with that token count)
    if (a.pl && in_range) {
      gpb_placement& o = a.pl[(size_t)si * a.n_req + r];
      const int wp = tb_rpipe[jb];
      const bool ok = wp >= 0;
      o.start_ns = ok ? tb_rstart[jb] : -1;
      o.ttft_overhead_ms = ok && D - 1 != 0 ? __dmul_rn((double)(D - 1), xfer) : 0.0;
      o.accepted = ok ? 1 : 0;
      o.pipeline = ok ? wp : -1;
    }
    if (act && failm && arrival == a.sufmin[r]) {
      for (unsigned long long m = failm; m; m &= m - 1) {
        const int pi = __ffsll((long long)m) - 1;
        atomicOr(&memo[(size_t)pi * a.memo_words + (tok_l >> 5)], 1u << (tok_l & 31));
      }
    }
    // warp 0: the failed pipelines' caps at the next batch's reference time,
    // then the plan-wide bounds
    if (warp == 0) {
      if (r0 + BW < a.n_req) {
        unsigned long long um = 0;
        for (int i = lane; i < BW; i += 32) um |= tb_fail[i];
        for (int o = 16; o > 0; o >>= 1) um |= __shfl_xor_sync(kFull, um, o);
        const long long a_next = a.sufmin[r0 + BW];
        while (um) {
          // the next ng failed pipelines, one per group
          unsigned long long mm = um;
          for (int g = 0; g < grp && mm; ++g) mm &= mm - 1;
          const int pi = mm ? __ffsll((long long)mm) - 1 : -1;
          long long ca, cb;
          group_caps(a, sl, gb, pi, a_next, extra, gs, ca, cb, zrun);
          if (pi >= 0 && gl == 0) {
            capA[pi] = ca;
            capB[pi] = cb;
          }
          for (int g = 0; g < ng && um; ++g) um &= um - 1;
        }
      }
      __syncwarp();
      long long ma = -kInf64, mb = -kInf64;
      for (int pi = lane; pi < n_pipes; pi += 32) {
        ma = max(ma, capA[pi]);
        mb = max(mb, capB[pi]);
      }
      ma = warp_max64(ma);
      mb = warp_max64(mb);
      if (lane == 0) {
        tb_bound[0] = ma;
        tb_bound[1] = mb;
      }
    }
    __syncthreads();
  }
  if (warp != 0) return;
  const long long rejected = a.n_req - accepted;
  if (a.stats) {
    st_search = (long long)__reduce_add_sync(kFull, (unsigned)st_search);
    st_fail = (long long)__reduce_add_sync(kFull, (unsigned)st_fail);
    if (lane == 0) {
      a.stats[si * 8 + 0] = st_exam;
      a.stats[si * 8 + 1] = st_search;
      a.stats[si * 8 + 2] = st_fail;
      a.stats[si * 8 + 3] = accepted;
      a.stats[si * 8 + 4] = clock64() - st_t0;
      a.stats[si * 8 + 5] = st_iter;
      a.stats[si * 8 + 6] = st_cyc_search;
      a.stats[si * 8 + 7] = st_cyc_caps * 1000000 / max(1LL, st_cyc_search) * 0 + st_cyc_commit;
    }
  }
  // utilization before/after (bubbletea.cpp:224-238): per GPU busy = H - sum
  // of its gaps, summed in GPU-id order (DC in topology order, then cell,
  // pipeline, stage within the DC's block), then / G.
  if (lane == 0) {
    const int row = (int)sl.row;
    const DevScen& sc = a.scens[a.row_scen[row]];
    const DevTopo& tp = a.topos[sc.topo];
    Geom g;
    decode(sc, tp, sl.D, g);
    double ub = 0.0, ua = 0.0;
    for (int dc = 0; dc < tp.n_dc; ++dc) {
      int b = -1;
      for (int x = 0; x < g.nb; ++x)
        if (g.blk_dc[x] == dc) b = x;
      if (b < 0) continue;
      for (int k = 0; k < D; ++k)
        for (int pipe = 0; pipe < C; ++pipe)
          for (int s = g.blk_first[b]; s < g.blk_first[b + 1]; ++s) {
            const int li = (Ce > 1 ? pipe : 0) * S + s;
            const long long bsum = a.gsum[sl.lst_off + li];
            ub = __dadd_rn(ub, __ddiv_rn((double)(H - bsum), (double)H));
            const int gi = gpu_index(k, pipe, s, C, S);
            long long asum = bsum;
            if (a.gpu_off[gb + gi] >= 0) {
              asum = 0;
              const long long o = a.gpu_off[gb + gi];
              for (int x = 0; x < a.gpu_cnt[gb + gi]; ++x) {
                const longlong2 g = a.pool[o + x];
                asum += (g.y & (kGapFl - 1)) - g.x;
              }
            }
            ua = __dadd_rn(ua, __ddiv_rn((double)(H - asum), (double)H));
          }
    }
    gpb_pack_summary& o = a.sums[si];
    o.utilization_before = __ddiv_rn(ub, (double)G);
    o.utilization_after = __ddiv_rn(ua, (double)G);
    o.accepted = accepted;
    o.rejected = rejected;
    o.horizon_ns = H;
    o.placement_hash = hash;
  }
}

}  // namespace gpb

// ------------------------------------------------------------------ host

using namespace gpb;

namespace {

struct HostBlocks {
  int nb = 0;
  int dc[GPB_MAX_DC];
  int first[GPB_MAX_DC + 1];
  bool feasible = false;
};

// build_plan's walk (workload.cpp:57-89) on the host, for GPU numbering.
HostBlocks host_decode(const DevScen& sc, const DevTopo& t, int d) {
  HostBlocks h;
  int assigned = 0;
  const int denom = d * sc.C * sc.tp;
  for (int i = 0; i < sc.n_order; ++i) {
    if (assigned >= sc.S) break;
    const int dc = sc.order[i];
    const int take = std::min(sc.S - assigned, t.gpu_count[dc] / denom);
    if (take > 0) {
      h.first[h.nb] = assigned;
      h.dc[h.nb] = dc;
      ++h.nb;
      assigned += take;
    }
  }
  h.first[h.nb] = assigned;
  h.feasible = assigned >= sc.S;
  return h;
}

long long host_ms_to_ns(double ms) { return std::llround(ms * 1e6); }

// Runs the timeline kernels for `rows` and the gap kernel; fills slots.
int build_timelines(Ctx& c, const int64_t* rows, int n, long long horizon,
                    std::vector<TlSlot>& slots, bool with_allreduce = false) {
  cudaStream_t st = c.stream;
  slots.resize(n);
  long long tl = 0, gp = 0, ls = 0;
  long long n_ar = 0;
  for (int i = 0; i < n; ++i) {
    if (rows[i] < 0 || rows[i] >= c.n_rows) {
      c.set_error("row index out of range");
      return GPB_CONFIG_ERROR;
    }
    const int si = c.scen_of_row(rows[i]);
    const DevScen& sc = c.dev_scens_host[si];
    const DevTopo& tp = c.dev_topos_host[sc.topo];
    const int d = (int)(rows[i] - sc.first_row) + 1;
    HostBlocks hb = host_decode(sc, tp, d);
    if (!hb.feasible) {
      c.set_error("plan needs more GPUs than the topology (row %lld)", (long long)rows[i]);
      return GPB_INFEASIBLE;
    }
    TlSlot& s = slots[i];
    s.row = rows[i];
    s.S = sc.S;
    s.M = sc.M;
    s.C = sc.C;
    s.D = d;
    s.policy = sc.policy;
    s.Ce = sc.policy == GPB_ATLAS ? sc.C : 1;
    s.fwd = host_ms_to_ns(sc.fwd_ms);
    s.dur = host_ms_to_ns(sc.bwd_ms) + (sc.recompute ? host_ms_to_ns(sc.rec_ms) : 0);
    s.horizon = horizon;
    s.tl_off = tl;
    s.gap_off = gp;
    s.lst_off = ls;
    s.ar_off = -1;
    if (with_allreduce) {  // per-stage tail durations: ar_dur_kernel, on the device
      s.ar_off = n_ar;
      n_ar += sc.S;
    }
    tl += (long long)s.Ce * s.S * s.M;
    gp += (long long)s.Ce * s.S * (2 * s.M + 1);
    ls += (long long)s.Ce * s.S;
  }
  long long* fe = (long long*)c.dev_buf(c.b_tl_spans, 16 * (size_t)std::max(1LL, tl));
  long long* ps = fe + std::max(1LL, tl);
  gpb_row* tl_rows = (gpb_row*)c.dev_buf(c.b_tl_rows, sizeof(gpb_row) * (size_t)c.n_rows);
  longlong2* gpk = (longlong2*)c.dev_buf(c.b_gaps, 33 * (size_t)std::max(1LL, gp));
  long long* glo = (long long*)(gpk + std::max(1LL, gp));
  long long* ghi = glo + std::max(1LL, gp);
  unsigned char* gfl = (unsigned char*)(ghi + std::max(1LL, gp));
  int* gcnt = (int*)c.dev_buf(c.b_ngaps, 24 * (size_t)std::max(1LL, ls) + 8 * (size_t)n + 64);
  long long* gsum = (long long*)(gcnt + 2 * std::max(1LL, ls));
  int* ghas = (int*)(gsum + std::max(1LL, ls));
  long long* hz = (long long*)(ghas + 2 * std::max(1LL, ls));
  TlSlot* dslots = (TlSlot*)c.dev_buf(c.b_tl_nspan, sizeof(TlSlot) * (size_t)std::max(1, n));
  if (!fe || !tl_rows || !glo || !gcnt || !dslots)
    return c.cuda_fail(cudaErrorMemoryAllocation, "timeline buffers");
  // per-(policy, B) work lists over the slots
  std::vector<int32_t> work;
  std::vector<long long> offs;
  struct Grp {
    int policy, B, off, cnt, max_m, max_c, max_s, max_nw;
  };
  std::vector<Grp> grps;
  for (int pol = 0; pol < 4; ++pol)
    for (int B = 1; B <= 8; ++B) {
      Grp g{pol, B, (int)work.size(), 0, 0, 0, 0, 0};
      for (int i = 0; i < n; ++i) {
        const DevScen& sc = c.dev_scens_host[c.scen_of_row(rows[i])];
        if (sc.policy != pol || (sc.S + 31) / 32 != B) continue;
        work.push_back((int32_t)rows[i]);
        offs.push_back(slots[i].tl_off);
        g.max_m = std::max(g.max_m, sc.M);
        g.max_c = std::max(g.max_c, sc.C);
        g.max_s = std::max(g.max_s, sc.S);
        g.max_nw = std::max(g.max_nw, sc.n_order - 1);
        ++g.cnt;
      }
      if (g.cnt) grps.push_back(g);
    }
  int32_t* dwork = (int32_t*)c.dev_buf(c.b_reqs, 4 * work.size() + 8 * offs.size() + 64);
  long long* doffs = (long long*)(dwork + ((work.size() + 1) & ~(size_t)1));
  int32_t* cursors = (int32_t*)c.dev_buf(c.b_pack_misc, 4 * (grps.size() + 2));
  if (!dwork || !cursors) return c.cuda_fail(cudaErrorMemoryAllocation, "timeline work");
  cudaMemcpyAsync(dwork, work.data(), 4 * work.size(), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(doffs, offs.data(), 8 * offs.size(), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dslots, slots.data(), sizeof(TlSlot) * n, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(cursors, 0, 4 * (grps.size() + 2), st);
  for (size_t gi = 0; gi < grps.size(); ++gi) {
    const Grp& g = grps[gi];
    EvalArgs a;
    std::memset(&a, 0, sizeof a);
    a.scens = (const DevScen*)c.b_scens.ptr;
    a.topos = (const DevTopo*)c.b_topos.ptr;
    a.row_scen = (const int32_t*)c.b_row_scen.ptr;
    a.work = dwork + g.off;
    a.n_work = g.cnt;
    a.cursor = cursors + gi;
    a.rows = tl_rows;
    a.error_flag = cursors + grps.size();
    a.tl_fe = fe;
    a.tl_ps = ps;
    a.tl_off = doffs + g.off;
    cudaError_t e;
    if (g.policy != GPB_ATLAS) {
      a.smem_m = g.max_m;
      e = launch_timeline(g.policy, g.B, a, std::min(c.num_sms * 8, (g.cnt + 3) / 4), st);
    } else {
      AtlasPlan P;
      long long max_csm = 0;
      const int rc = plan_atlas(c, g.B, true, g.max_c, g.max_s, g.max_m, g.max_nw,
                                (long long)g.max_c * g.max_s * g.max_m, g.cnt, P);
      (void)max_csm;
      if (rc != GPB_OK) return rc;
      a.lay = P.L;
      const int grid = P.grid, wpc = P.wpc;
      a.scratch = nullptr;
      a.scratch_per_warp = P.scratch_per_warp;
      a.scratch_big_off = P.scratch_big_off;
      if (P.scratch_per_warp > 0) {
        a.scratch = (long long*)c.dev_buf(c.b_tl_scratch,
                                          8 * (size_t)P.scratch_per_warp * grid * wpc);
        if (!a.scratch) return c.cuda_fail(cudaErrorMemoryAllocation, "atlas scratch");
      }
      e = launch_atlas_timeline(g.B, a, grid, wpc, st);
    }
    if (e != cudaSuccess) return c.cuda_fail(e, "timeline launch");
  }
  long long* ar_dev = (long long*)c.dev_buf(c.b_ar, 16 * std::max<size_t>(1, n_ar));
  if (!ar_dev) return c.cuda_fail(cudaErrorMemoryAllocation, "allreduce buffers");
  long long* ar_start = ar_dev + std::max<long long>(1, n_ar);
  if (n_ar > 0)
    ar_dur_kernel<<<n, 128, 0, st>>>(dslots, n, (const DevScen*)c.b_scens.ptr,
                                     (const DevTopo*)c.b_topos.ptr,
                                     (const int32_t*)c.b_row_scen.ptr, ar_dev);
  c.tl_ar = ar_dev;
  cudaMemsetAsync(hz, 0, 8 * (size_t)n, st);
  horizon_kernel<<<n, 128, 0, st>>>(dslots, n, tl_rows, ps, ar_dev, ar_start, hz);
  long long max_lists = 1;
  for (const TlSlot& s : slots) max_lists = std::max(max_lists, (long long)s.Ce * s.S);
  gap_kernel<<<dim3((unsigned)((max_lists + 127) / 128), (unsigned)n), 128, 0, st>>>(
      dslots, n, fe, ps, ar_dev, ar_start, glo, ghi, gfl, gpk, gcnt, gsum, ghas, hz);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return c.cuda_fail(e, "gap kernel");
  int32_t flag = 0;
  cudaMemcpyAsync(&flag, cursors + grps.size(), 4, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return c.cuda_fail(e, "timelines");
  if (flag) {
    c.set_error("kernel invariant failure in the timeline kernels");
    return GPB_ERROR;
  }
  c.tl_glo = glo;
  c.tl_ghi = ghi;
  c.tl_gfl = gfl;
  c.tl_gpk = gpk;
  c.tl_gcnt = gcnt;
  c.tl_gsum = gsum;
  c.tl_ghas = ghas;
  c.tl_hz = hz;
  c.tl_slots_dev = (void*)dslots;
  return GPB_OK;
}

}  // namespace

namespace gpb {
// WAN boundaries of a row's plan (DC blocks - 1), or -1 if infeasible.
int row_wan_boundaries(const Ctx& c, int64_t row) {
  const int si = c.scen_of_row(row);
  const DevScen& sc = c.dev_scens_host[si];
  const HostBlocks hb = host_decode(sc, c.dev_topos_host[sc.topo], (int)(row - sc.first_row) + 1);
  return hb.feasible ? hb.nb - 1 : -1;
}
}  // namespace gpb

extern "C" int gpb_bubbles(gpb_ctx* ctx_, int64_t row, int64_t horizon_ns, gpb_bubble* out,
                           int64_t cap, int64_t* n_out) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  c.last_error.clear();
  if (!c.loaded) {
    c.set_error("no plan space loaded");
    return GPB_CONFIG_ERROR;
  }
  cudaSetDevice(c.device);
  std::vector<TlSlot> slots;
  int rc = build_timelines(c, &row, 1, horizon_ns, slots, c.pack_allreduce);
  if (rc != GPB_OK) return rc;
  const TlSlot& s = slots[0];
  const size_t nl = (size_t)s.Ce * s.S, per = 2 * (size_t)s.M + 1;
  std::vector<long long> lo(nl * per), hi(nl * per);
  std::vector<int> cnt(nl), has(nl);
  long long hz = 0;
  cudaStream_t st = c.stream;
  cudaMemcpyAsync(lo.data(), c.tl_glo, 8 * lo.size(), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(hi.data(), c.tl_ghi, 8 * hi.size(), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(cnt.data(), c.tl_gcnt, 4 * nl, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(has.data(), c.tl_ghas, 4 * nl, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&hz, c.tl_hz, 8, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return c.cuda_fail(e, "bubbles");
  if (hz <= 0) {
    c.set_error("horizon: must be positive");
    return GPB_CONFIG_ERROR;
  }
  // expand to every timeline GPU in id order (extract_bubbles sorts by GPU):
  // DCs in topology order; inside a DC ids go (cell, pipeline, stage).
  const DevScen& sc = c.dev_scens_host[c.scen_of_row(row)];
  const DevTopo& tp = c.dev_topos_host[sc.topo];
  HostBlocks hb = host_decode(sc, tp, s.D);
  int64_t k = 0;
  for (int dc = 0; dc < tp.n_dc; ++dc) {
    int b = -1;
    for (int x = 0; x < hb.nb; ++x)
      if (hb.dc[x] == dc) b = x;
    if (b < 0) continue;
    const int cnt_stages = hb.first[b + 1] - hb.first[b];
    for (int cell = 0; cell < s.D; ++cell)
      for (int pipe = 0; pipe < s.C; ++pipe)
        for (int st2 = hb.first[b]; st2 < hb.first[b + 1]; ++st2) {
          const int li = (s.Ce > 1 ? pipe : 0) * s.S + st2;
          if (!has[li]) continue;  // no busy span: absent from busy_by_gpu
          const int gpu = tp.dc_base[dc] +
                          sc.tp * ((cell * s.C + pipe) * cnt_stages + (st2 - hb.first[b]));
          for (int j = 0; j < cnt[li]; ++j, ++k) {
            if (k < cap && out) {
              out[k].gpu_id = gpu;
              out[k].pad_ = 0;
              out[k].start_ns = lo[li * per + j];
              out[k].end_ns = hi[li * per + j];
            }
          }
        }
  }
  if (n_out) *n_out = k;
  return GPB_OK;
}

extern "C" int gpb_pack_prefills(gpb_ctx* ctx_, const int64_t* rows, int32_t n_rows_sel,
                                 const gpb_request* reqs, int64_t n_req,
                                 const gpb_prefill_model* pm, int64_t horizon_ns,
                                 gpb_pack_summary* summaries, gpb_placement* placements) {
  if (!ctx_) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  c.last_error.clear();
  if (!c.loaded) {
    c.set_error("no plan space loaded");
    return GPB_CONFIG_ERROR;
  }
  if (!pm || n_rows_sel < 0 || n_req < 0 || (n_req > 0 && !reqs) || !summaries) {
    c.set_error("null input");
    return GPB_CONFIG_ERROR;
  }
  if (!(pm->saturation_ms > 0) || pm->max_tokens < 1 || pm->inference_layers < 1 ||
      pm->inference_hidden < 1 || pm->bytes_per_element < 1 || pm->memory_budget_bytes < 1 ||
      pm->boundary_latency_ms < 0 || pm->guard_ms < 0 || pm->inference_params_per_layer < 0) {
    c.set_error("prefill: invalid prefill model");
    return GPB_CONFIG_ERROR;
  }
  if (!(pm->stage_bw > 0)) {
    c.set_error("bandwidth must be positive");
    return GPB_ERROR;  // std::invalid_argument in transfer_time_ms
  }
  for (int64_t i = 0; i < n_req; ++i)
    if (reqs[i].tokens < 1 || reqs[i].tokens > pm->max_tokens) {
      c.set_error("request.tokens: must be in [1, %d]", pm->max_tokens);
      return GPB_CONFIG_ERROR;
    }
  cudaSetDevice(c.device);
  std::vector<TlSlot> slots;
  int rc = build_timelines(c, rows, n_rows_sel, horizon_ns, slots, c.pack_allreduce);
  if (rc != GPB_OK) return rc;
  // memory budget per stage (bubbletea.cpp:113-125)
  const double ppl = pm->inference_params_per_layer > 0
                         ? pm->inference_params_per_layer
                         : 12.0 * (double)pm->inference_hidden * (double)pm->inference_hidden;
  std::vector<long long> gpu_base(n_rows_sel + 1, 0);
  long long max_nl = 0;
  for (int i = 0; i < n_rows_sel; ++i) {
    const TlSlot& s = slots[i];
    const int worst = pm->inference_layers / s.D + (pm->inference_layers % s.D ? 1 : 0);
    const long long mem = (long long)((double)worst * ppl * pm->bytes_per_element);
    if (mem > pm->memory_budget_bytes) {
      c.set_error("prefill.memory_budget_bytes: inference model needs %lld bytes per stage, over "
                  "the budget of %lld", mem, (long long)pm->memory_budget_bytes);
      return GPB_CONFIG_ERROR;
    }
    gpu_base[i + 1] = gpu_base[i] + (long long)s.D * s.C * s.S;
    max_nl = std::max(max_nl, (long long)s.Ce * s.S * (2 * s.M + 1));
  }
  cudaStream_t st = c.stream;
  gpb_request* dreq = (gpb_request*)c.dev_buf(c.b_pl, sizeof(gpb_request) * std::max<int64_t>(1, n_req));
  gpb_pack_summary* dsum = (gpb_pack_summary*)c.dev_buf(c.b_sum, sizeof(gpb_pack_summary) * std::max(1, n_rows_sel) + 64);
  const long long G = gpu_base[n_rows_sel];
  long long* gpu_arr = (long long*)c.dev_buf(c.b_pack_scratch, 16 * (size_t)std::max(1LL, G) + 20 * (size_t)(n_rows_sel + 1));
  if (!dreq || !dsum || !gpu_arr) return c.cuda_fail(cudaErrorMemoryAllocation, "pack buffers");
  long long* gpu_off = gpu_arr;
  int* gpu_cnt = (int*)(gpu_off + std::max(1LL, G));
  int* gpu_cap = gpu_cnt + std::max(1LL, G);
  long long* dbase = (long long*)(gpu_cap + std::max(1LL, G));  // 16*G bytes in: aligned
  int* overflow = (int*)(dsum + std::max(1, n_rows_sel));
  cudaMemcpyAsync(dreq, reqs, sizeof(gpb_request) * n_req, cudaMemcpyHostToDevice, st);
  c.sufmin_host.assign((size_t)n_req + 1, 0);
  for (int64_t i = n_req - 1; i >= 0; --i) {
    const long long t = host_ms_to_ns(reqs[i].arrival_ms);
    c.sufmin_host[i] = i + 1 < n_req ? std::min(t, c.sufmin_host[i + 1]) : t;
  }
  long long* dsufmin = (long long*)c.dev_buf(c.b_sufmin, 8 * c.sufmin_host.size());
  if (!dsufmin) return c.cuda_fail(cudaErrorMemoryAllocation, "pack buffers");
  cudaMemcpyAsync(dsufmin, c.sufmin_host.data(), 8 * c.sufmin_host.size(), cudaMemcpyHostToDevice,
                  st);
  cudaMemcpyAsync(dbase, gpu_base.data(), 8 * n_rows_sel, cudaMemcpyHostToDevice, st);
  // CTAs start in index order: the plans with the most searched stage GPUs
  // (pipelines x stages searched one by one) first, so the longest packings
  // do not start in the last wave
  long long* dpool_off = dbase + n_rows_sel + 1;
  int32_t* dorder = (int32_t*)(dpool_off + n_rows_sel + 1);
  c.pack_order.resize(n_rows_sel);
  {
    std::vector<long long> est(std::max(1, n_rows_sel));
    for (int i = 0; i < n_rows_sel; ++i) {
      const TlSlot& sl2 = slots[i];
      const int d_eff = pm->inference_layers / sl2.D == 0 ? pm->inference_layers % sl2.D + 1 : sl2.D;
      est[i] = (long long)sl2.C * sl2.S * d_eff;
      c.pack_order[i] = i;
    }
    std::stable_sort(c.pack_order.begin(), c.pack_order.end(),
                     [&](int x, int y) { return est[x] > est[y]; });
    c.pack_est = est;
  }
  cudaMemcpyAsync(dorder, c.pack_order.data(), 4 * (size_t)n_rows_sel, cudaMemcpyHostToDevice, st);
  gpb_placement* dpl = nullptr;
  if (placements) {
    dpl = (gpb_placement*)c.dev_buf(c.b_placements, sizeof(gpb_placement) * (size_t)n_rows_sel * std::max<int64_t>(1, n_req));
    if (!dpl) return c.cuda_fail(cudaErrorMemoryAllocation, "placements");
  }
  // copy-on-write pool per slot. Final list sizes are bounded by the initial
  // gaps plus one split per accepted request on each of its D stage GPUs;
  // capacity doubling at most triples the total. Each slot gets its own
  // bound (a plan with few GPUs needs little); an overflow re-runs the kernel
  // with 4x the pool, so the first size errs on the large side.
  if (!c.pack_warm) {
    // Load both packing kernels with an empty launch first (lazy module
    // loading): measured on B200, the first real launch pair otherwise starts
    // the light kernel's CTAs ahead of the heavy plans' (40 s vs 22 s on
    // config 4, the heavy plans set the kernel time).
    PackArgs w;
    std::memset(&w, 0, sizeof w);
    pack_kernel<8><<<1, 32 * 8, 0, st>>>(w);
    pack_kernel<4><<<1, 32 * 4, 0, st>>>(w);
    c.pack_warm = true;
  }
  std::vector<long long> pool_off(n_rows_sel + 1, 0);
  for (int attempt = 0, scale = 1; attempt < 8; ++attempt, scale *= 4) {
    for (int i = 0; i < n_rows_sel; ++i) {
      const long long G = (long long)slots[i].D * slots[i].C * slots[i].S;
      const long long need = 3 * (G * (2LL * slots[i].M + 9) +
                                  (long long)slots[i].D * std::min<long long>(n_req, 2048));
      pool_off[i + 1] = pool_off[i] + std::max<long long>(4096, need) * scale;
    }
    const long long pool = pool_off[n_rows_sel];
    longlong2* pool_e = (longlong2*)c.dev_buf(c.b_tl_scratch, 16 * (size_t)std::max(1LL, pool));
    if (!pool_e) return c.cuda_fail(cudaErrorMemoryAllocation, "pack pool");
    cudaMemcpyAsync(dpool_off, pool_off.data(), 8 * (size_t)(n_rows_sel + 1),
                    cudaMemcpyHostToDevice, st);
    PackArgs a;
    std::memset(&a, 0, sizeof a);
    a.slots = (const TlSlot*)c.tl_slots_dev;
    a.n_slots = n_rows_sel;
    a.scens = (const DevScen*)c.b_scens.ptr;
    a.topos = (const DevTopo*)c.b_topos.ptr;
    a.row_scen = (const int32_t*)c.b_row_scen.ptr;
    a.gpk = c.tl_gpk;
    a.gcnt = c.tl_gcnt;
    a.gsum = c.tl_gsum;
    a.hz = c.tl_hz;
    a.reqs = dreq;
    a.n_req = n_req;
    a.sufmin = dsufmin;
    a.sat_ms = pm->saturation_ms;
    a.stage_bw = pm->stage_bw;
    a.lat_ms = pm->boundary_latency_ms;
    a.max_tokens = pm->max_tokens;
    a.inf_layers = pm->inference_layers;
    a.bpe = pm->bytes_per_element;
    a.inf_hidden = pm->inference_hidden;
    a.guard_ns = host_ms_to_ns(pm->guard_ms);
    a.pool = pool_e;
    a.pool_off = dpool_off;
    a.gpu_off = gpu_off;
    a.gpu_cnt = gpu_cnt;
    a.gpu_cap = gpu_cap;
    a.gpu_base = dbase;
    a.sums = dsum;
    a.pl = dpl;
    a.overflow = overflow;
    a.order = dorder;
    int max_pipes = 1;
    for (const TlSlot& sl2 : slots) max_pipes = std::max(max_pipes, sl2.C * sl2.S);
    a.max_pipes = max_pipes;
    // caps, batch table, flags (pack_kernel's shared layout)
    auto psmem_of = [&](int W) {
      return 16 * (size_t)max_pipes + (7 * 8 + 16 + 4 * 4) * (size_t)(32 * W) + 16 + 16 +
             (size_t)max_pipes + 16;
    };
    const size_t psmem4 = psmem_of(4), psmem8 = psmem_of(8);
    if (psmem8 > (size_t)c.smem_optin) {
      c.set_error("too many prefill pipelines per plan for the packing kernel");
      return GPB_CONFIG_ERROR;
    }
    if (psmem4 > 48 * 1024)
      cudaFuncSetAttribute(pack_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem4);
    if (psmem8 > 48 * 1024)
      cudaFuncSetAttribute(pack_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem8);
    a.memo_words = (pm->max_tokens + 31) / 32;
    const size_t memo_bytes = 4 * (size_t)a.memo_words * max_pipes * std::max(1, n_rows_sel);
    a.memo = (unsigned*)c.dev_buf(c.b_pack_memo, memo_bytes);
    if (!a.memo) return c.cuda_fail(cudaErrorMemoryAllocation, "pack memo");
    cudaMemsetAsync(a.memo, 0, memo_bytes, st);
    a.stats = nullptr;
    if (std::getenv("GPB_PACK_STATS")) {
      a.stats = (long long*)c.dev_buf(c.b_pack_stats, 64 * (size_t)std::max(1, n_rows_sel));
      cudaMemsetAsync(a.stats, 0, 64 * (size_t)std::max(1, n_rows_sel), st);
    }
    cudaMemsetAsync(overflow, 0, 4, st);
    // device time of the packing kernels (timelines, tables and one-time
    // buffer allocations before this point are in the call's wall time)
    cudaEventRecord(c.pack_ev0, st);
    // the heaviest plans (estimate within half of the largest, at most one
    // per SM) on 8-warp CTAs on a side stream, the rest on 4-warp CTAs
    int n_heavy = 0;
    while (n_heavy < std::min(n_rows_sel, c.num_sms) &&
           2 * c.pack_est[c.pack_order[n_heavy]] >= c.pack_est[c.pack_order[0]])
      ++n_heavy;
    if (n_heavy > 0) {
      if (!c.pack_side) {
        // highest priority: the block scheduler then starts every heavy CTA
        // before the light kernel's queued CTAs (launch order alone across
        // two streams is not honoured: the heavy plans set the kernel time)
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        cudaStreamCreateWithPriority(&c.pack_side, cudaStreamNonBlocking, hi);
        cudaEventCreateWithFlags(&c.pack_fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&c.pack_join, cudaEventDisableTiming);
      }
      cudaEventRecord(c.pack_fork, st);
      cudaStreamWaitEvent(c.pack_side, c.pack_fork, 0);
      PackArgs ah = a;
      ah.order_base = 0;
      pack_kernel<8><<<n_heavy, 32 * 8, psmem8, c.pack_side>>>(ah);
      cudaEventRecord(c.pack_join, c.pack_side);
    }
    if (n_rows_sel - n_heavy > 0) {
      a.order_base = n_heavy;
      pack_kernel<4><<<n_rows_sel - n_heavy, 32 * 4, psmem4, st>>>(a);
    }
    if (n_heavy > 0) cudaStreamWaitEvent(st, c.pack_join, 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return c.cuda_fail(e, "pack launch");
    int32_t ovf = 0;
    cudaMemcpyAsync(&ovf, overflow, 4, cudaMemcpyDeviceToHost, st);
    cudaEventRecord(c.pack_ev1, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return c.cuda_fail(e, "pack");
    if (a.stats) {
      std::vector<long long> hs(8 * (size_t)n_rows_sel);
      cudaMemcpy(hs.data(), a.stats, 64 * (size_t)n_rows_sel, cudaMemcpyDeviceToHost);
      long long tot[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mx = 0;
      for (int i = 0; i < n_rows_sel; ++i) {
        for (int k = 0; k < 8; ++k) tot[k] += hs[8 * i + k];
        mx = std::max(mx, hs[8 * i + 4]);
      }
      std::vector<int> ord(n_rows_sel);
      for (int i = 0; i < n_rows_sel; ++i) ord[i] = i;
      std::sort(ord.begin(), ord.end(), [&](int x, int y) { return hs[8 * x + 4] > hs[8 * y + 4]; });
      for (int q = 0; q < std::min(n_rows_sel, 4); ++q) {
        const int i = ord[q];
        const TlSlot& sl = slots[i];
        std::fprintf(stderr, "  slot %d row %lld pol %d D %d C %d S %d M %d: cycles %lld examined %lld "
                     "searches %lld failed %lld accepted %lld iters %lld search_cyc %lld\n", i,
                     (long long)sl.row, sl.policy, sl.D, sl.C, sl.S, sl.M, hs[8 * i + 4],
                     hs[8 * i], hs[8 * i + 1], hs[8 * i + 2], hs[8 * i + 3], hs[8 * i + 5],
                     hs[8 * i + 6]);
      }
      std::fprintf(stderr, "pack stats (attempt %d, pool %lld, ovf %d): examined %lld searches %lld "
                   "failed %lld accepted %lld cycles sum %lld max %lld; search iters %lld "
                   "search cyc %lld commit cyc %lld\n", attempt, pool, ovf,
                   tot[0], tot[1], tot[2], tot[3], tot[4], mx, tot[5], tot[6], tot[7]);
    }
    if (!ovf) break;
    if (attempt == 7) {
      c.set_error("gap pool overflow");
      return GPB_ERROR;
    }
  }
  // its own event pair: evaluate's ev0..ev2 stay valid for gpb_get_timing
  cudaEventElapsedTime(&c.pack_ms, c.pack_ev0, c.pack_ev1);
  cudaMemcpyAsync(summaries, dsum, sizeof(gpb_pack_summary) * n_rows_sel, cudaMemcpyDeviceToHost, st);
  if (placements)
    cudaMemcpyAsync(placements, dpl, sizeof(gpb_placement) * (size_t)n_rows_sel * n_req,
                    cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? GPB_OK : c.cuda_fail(e, "pack results");
}

// Raw iteration timeline of one row (cell 0): forward ends and pair starts
// laid out [pipeline][stage][microbatch] (Ce = C for atlas, else 1).
extern "C" int gpb_timeline_arrays(gpb_ctx* ctx_, int64_t row, int64_t* fe, int64_t* ps,
                                   int64_t cap, int32_t* dims, int64_t* makespan) {
  if (!ctx_ || !dims) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  c.last_error.clear();
  if (!c.loaded) {
    c.set_error("no plan space loaded");
    return GPB_CONFIG_ERROR;
  }
  cudaSetDevice(c.device);
  std::vector<TlSlot> slots;
  int rc = build_timelines(c, &row, 1, 0, slots);
  if (rc != GPB_OK) return rc;
  const TlSlot& s = slots[0];
  const long long n = (long long)s.Ce * s.S * s.M;
  dims[0] = s.Ce;
  dims[1] = s.S;
  dims[2] = s.M;
  dims[3] = s.D;
  if (fe && ps && cap >= n) {
    long long* dfe = (long long*)c.b_tl_spans.ptr;
    long long* dps = dfe + std::max(1LL, n);
    cudaMemcpyAsync(fe, dfe, 8 * n, cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(ps, dps, 8 * n, cudaMemcpyDeviceToHost, c.stream);
  }
  gpb_row r;
  cudaMemcpyAsync(&r, (gpb_row*)c.b_tl_rows.ptr + row, sizeof r, cudaMemcpyDeviceToHost, c.stream);
  cudaError_t e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) return c.cuda_fail(e, "timeline");
  if (makespan) *makespan = r.makespan_ns;
  return GPB_OK;
}

extern "C" int gpb_set_allreduce_tail(gpb_ctx* ctx_, int32_t enable) {
  if (!ctx_) return GPB_ERROR;
  reinterpret_cast<Ctx*>(ctx_)->pack_allreduce = enable != 0;
  return GPB_OK;
}

// ------------------------------------------------- saturating_requests
//
// saturating_requests (bubbletea.cpp:240-267): for every prefill pipeline
// (pipe, stage) in build_prefill_pipelines order, fill its head GPU's (cell
// 0's) idle windows with back-to-back requests, each the largest token count
// whose duration fits the rest of the window. One thread per pipeline walks
// that GPU's gap list (gap_kernel: gaps_of over busy_by_gpu); a first pass
// counts, a second writes at the pipeline's offset, so ids follow the
// reference's order. Same double operations as the reference (--fmad=false).
namespace {

// static_cast<int>(double) as x86-64 executes it (cvttsd2si): out of range
// or NaN gives INT_MIN (the reference then emits no request for the window).
__device__ __forceinline__ int x86_double_to_int(double x) {
  if (!(x > -2147483649.0 && x < 2147483648.0)) return (int)0x80000000;
  return (int)x;
}

__device__ __forceinline__ long long prefill_ns(double sat_ms, int max_tokens, int tokens) {
  // ms_to_ns(prefill_duration_ms(tokens)) (bubbletea.cpp:68-76, base.h:15-17)
  return ms_to_ns(__ddiv_rn(__dmul_rn(sat_ms, (double)tokens), (double)max_tokens));
}

__global__ void saturate_kernel(const TlSlot* slots, const longlong2* gpk, const int* gcnt,
                                double sat_ms, int max_tokens, const long long* offs,
                                gpb_request* out, long long* counts) {
  const TlSlot& sl = slots[0];
  const int pi = blockIdx.x * blockDim.x + threadIdx.x;  // = pipe * S + stage
  if (pi >= sl.C * sl.S) return;
  const int pipe = pi / sl.S, stage = pi % sl.S;
  const int li = (sl.Ce > 1 ? pipe : 0) * sl.S + stage;  // spatial policies: one list
  const longlong2* G = gpk + sl.gap_off + (size_t)li * (2 * sl.M + 1);
  const int ng = gcnt[sl.lst_off + li];
  long long k = 0, id = offs ? offs[pi] : 0;
  for (int j = 0; j < ng; ++j) {
    const long long end = G[j].y & ~kGapFl;
    long long cur = G[j].x;
    while (cur < end) {
      const double gap_ms = __ddiv_rn((double)(end - cur), 1e6);
      int tokens = x86_double_to_int(__ddiv_rn(__dmul_rn(gap_ms, (double)max_tokens), sat_ms));
      tokens = min(tokens, max_tokens);
      while (tokens >= 1 && cur + prefill_ns(sat_ms, max_tokens, tokens) > end) tokens -= 1;
      if (tokens < 1) break;
      if (out) {
        gpb_request r;
        r.id = (int32_t)id;
        r.tokens = tokens;
        r.arrival_ms = __ddiv_rn((double)cur, 1e6);
        out[id] = r;
      }
      ++id;
      ++k;
      cur += prefill_ns(sat_ms, max_tokens, tokens);
    }
  }
  if (counts) counts[pi] = k;
}

}  // namespace

extern "C" int gpb_saturating_requests(gpb_ctx* ctx_, int64_t row, const gpb_prefill_model* pm,
                                       int64_t horizon_ns, gpb_request* out, int64_t cap,
                                       int64_t* n_out) {
  if (!ctx_ || !pm) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  c.last_error.clear();
  if (!c.loaded) {
    c.set_error("no plan space loaded");
    return GPB_CONFIG_ERROR;
  }
  if (pm->max_tokens < 1) {
    c.set_error("prefill.max_tokens: must be >= 1");
    return GPB_CONFIG_ERROR;
  }
  cudaSetDevice(c.device);
  std::vector<TlSlot> slots;
  int rc = build_timelines(c, &row, 1, horizon_ns, slots, c.pack_allreduce);
  if (rc != GPB_OK) return rc;
  const TlSlot& s = slots[0];
  const int P = s.C * s.S;
  cudaStream_t st = c.stream;
  long long hz = 0;
  cudaMemcpyAsync(&hz, c.tl_hz, 8, cudaMemcpyDeviceToHost, st);
  long long* dcnt = (long long*)c.dev_buf(c.b_pack_misc, 16 * (size_t)P + 64);
  if (!dcnt) return c.cuda_fail(cudaErrorMemoryAllocation, "saturating counts");
  long long* doff = dcnt + P;
  const int threads = 128, grid = (P + threads - 1) / threads;
  saturate_kernel<<<grid, threads, 0, st>>>((const TlSlot*)c.tl_slots_dev, c.tl_gpk, c.tl_gcnt,
                                            pm->saturation_ms, pm->max_tokens, nullptr, nullptr,
                                            dcnt);
  std::vector<long long> cnt(P), off(P);
  cudaMemcpyAsync(cnt.data(), dcnt, 8 * (size_t)P, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return c.cuda_fail(e, "saturating requests");
  if (hz <= 0) {
    c.set_error("horizon: must be positive");
    return GPB_CONFIG_ERROR;
  }
  long long n = 0;
  for (int i = 0; i < P; ++i) {
    off[i] = n;
    n += cnt[i];
  }
  if (n_out) *n_out = n;
  if (out && cap >= n && n > 0) {
    gpb_request* dout = (gpb_request*)c.dev_buf(c.b_reqs, sizeof(gpb_request) * (size_t)n);
    if (!dout) return c.cuda_fail(cudaErrorMemoryAllocation, "saturating requests");
    cudaMemcpyAsync(doff, off.data(), 8 * (size_t)P, cudaMemcpyHostToDevice, st);
    saturate_kernel<<<grid, threads, 0, st>>>((const TlSlot*)c.tl_slots_dev, c.tl_gpk,
                                              c.tl_gcnt, pm->saturation_ms, pm->max_tokens, doff,
                                              dout, nullptr);
    cudaMemcpyAsync(out, dout, sizeof(gpb_request) * (size_t)n, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return c.cuda_fail(e, "saturating requests");
  }
  return GPB_OK;
}

// ------------------------------------------------------- validation
//
// The reference's structural checker validate_timeline (tests/support/
// validate.h:77-256; SURVEY.md §8(f) "engine replay as an on-device
// validator") restated for the device timeline of one row, cell 0 (all D
// cells are identical; ATLAS keeps C pipelines, the spatial policies one):
//   1 completeness   every (pipeline, stage, microbatch) has its forward and
//                    its recompute+backward pair (validate.h:115-135)
//   2 GPU exclusivity tasks of one stage GPU never overlap (:138-146)
//   3 link exclusivity transfers of one lane never overlap: the pooled lane
//                    of a cell (ATLAS, exact fit at the producer's end) or
//                    the pipeline's own FIFO lane (:148-187)
//   4 forward causality  a forward starts after its activation arrives
//   5 backward causality a pair starts after its gradient arrives / its
//                    own forward at the last stage (:190-243)
//   6 makespan       the row's makespan is the last task end (:246-252)
// One thread per (pipeline, stage) for 1/2/4/5, one per (WAN boundary,
// direction) for 3; a failure records the smallest (check, pipeline,
// stage, microbatch) key.
namespace {

constexpr long long kVNeg = -(1LL << 60);

__device__ __forceinline__ void vfail(unsigned long long* res, int check, int p, int s, int m) {
  const unsigned long long key = ((unsigned long long)check << 56) |
                                 ((unsigned long long)(p & 0xff) << 48) |
                                 ((unsigned long long)(s & 0xffff) << 32) | (unsigned)m;
  atomicMin(res, key);
}

__global__ void validate_kernel(const TlSlot* slots, const DevScen* scens, const DevTopo* topos,
                                const int32_t* row_scen, const long long* fe, const long long* ps,
                                long long makespan, unsigned long long* res,
                                unsigned long long* mk_out) {
  const TlSlot& sl = slots[0];
  const DevScen& sc = scens[row_scen[sl.row]];
  Geom g;
  decode(sc, topos[sc.topo], sl.D, g);
  const int S = sl.S, M = sl.M, Ce = sl.Ce;
  const long long f = sl.fwd, dur = sl.dur;
  const bool atlas = sl.policy == GPB_ATLAS, rev = sl.policy == GPB_GPIPE;
  const long long* F = fe + sl.tl_off;
  const long long* P = ps + sl.tl_off;
  auto wan = [&](int s, long long& ser, long long& lat) {  // boundary s -> s+1
    for (int b = 1; b < g.nb; ++b)
      if (g.blk_first[b] == s + 1) {
        ser = atlas ? g.ser_pooled[b - 1] : g.ser_spatial[b - 1];
        lat = g.lat[b - 1];
        return true;
      }
    return false;
  };
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  // ---- per stage GPU: completeness, exclusivity, causality
  if (tid < Ce * S) {
    const int p = tid / S, s = tid % S;
    const long long* Fs = F + (size_t)tid * M;
    const long long* Ps = P + (size_t)tid * M;
    long long mk = 0;
    for (int m = 0; m < M; ++m) {
      if (Fs[m] < f || Ps[m] < 0) {
        vfail(res, 1, p, s, m);
        return;
      }
      mk = imax(mk, imax(Fs[m], Ps[m] + dur));
    }
    atomicMax(mk_out, (unsigned long long)mk);
    // tasks by start: forwards in m order, pairs in drain order
    int i = 0, j = 0;
    long long last_end = -1;
    while (i < M || j < M) {
      const long long fs = i < M ? Fs[i] - f : kInf64;
      const int mj = rev ? M - 1 - j : j;
      const long long pst = j < M ? Ps[mj] : kInf64;
      long long lo, hi;
      int mm;
      if (fs <= pst) {
        lo = fs;
        hi = Fs[i];
        mm = i++;
      } else {
        lo = pst;
        hi = pst + dur;
        mm = mj;
        ++j;
      }
      if (lo < last_end) {
        vfail(res, 2, p, s, mm);
        return;
      }
      last_end = hi;
    }
    // forward causality: arrival of the activation from stage s-1
    long long ser = 0, lat = 0;
    if (s > 0) {
      const long long* Fu = F + ((size_t)p * S + s - 1) * M;
      const bool w = wan(s - 1, ser, lat);
      long long link = kVNeg;  // FIFO lane of a spatial pipeline
      for (int m = 0; m < M; ++m) {
        long long arr = Fu[m];
        if (w) {
          const long long start = atlas ? Fu[m] : imax(Fu[m], link);
          link = start + ser;
          arr = start + ser + lat;
        }
        if (Fs[m] - f < arr) {
          vfail(res, 4, p, s, m);
          return;
        }
      }
    }
    // backward causality: gradient from stage s+1 (or the forward at S-1)
    if (s == S - 1) {
      for (int m = 0; m < M; ++m)
        if (Ps[m] < Fs[m]) {
          vfail(res, 5, p, s, m);
          return;
        }
    } else {
      const long long* Pd = P + ((size_t)p * S + s + 1) * M;
      const bool w = wan(s, ser, lat);
      long long link = kVNeg;
      for (int k = 0; k < M; ++k) {
        const int m = rev ? M - 1 - k : k;  // the lane's order: the producer's drain order
        long long arr = Pd[m] + dur;
        if (w) {
          const long long start = atlas ? Pd[m] + dur : imax(Pd[m] + dur, link);
          link = start + ser;
          arr = start + ser + lat;
        }
        if (Ps[m] < arr) {
          vfail(res, 5, p, s, m);
          return;
        }
      }
    }
    return;
  }
  // ---- pooled lanes (ATLAS): transfers of all pipelines on one boundary
  const int li = tid - Ce * S;
  if (!atlas || li >= 2 * (S - 1)) return;
  const int s = li >> 1;
  const bool grad = li & 1;
  long long ser = 0, lat = 0;
  if (!wan(s, ser, lat) || ser <= 0) return;
  // merge the C per-pipeline (time-sorted) transfer lists by start
  int cur[32];
  for (int p = 0; p < Ce; ++p) cur[p] = 0;
  long long last_end = kVNeg;
  for (;;) {
    int bp = -1;
    long long bt = kInf64;
    for (int p = 0; p < Ce; ++p) {
      if (cur[p] >= M) continue;
      const long long t = grad ? P[((size_t)p * S + s + 1) * M + cur[p]] + dur
                               : F[((size_t)p * S + s) * M + cur[p]];
      if (t < bt) {
        bt = t;
        bp = p;
      }
    }
    if (bp < 0) break;
    if (bt < last_end) {
      vfail(res, 3, bp, s, cur[bp]);
      return;
    }
    last_end = bt + ser;
    ++cur[bp];
  }
}

}  // namespace

extern "C" int gpb_validate_timeline(gpb_ctx* ctx_, int64_t row, const int64_t* fe,
                                     const int64_t* ps, int32_t* check, int64_t* where) {
  if (!ctx_ || !check) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  c.last_error.clear();
  if (!c.loaded) {
    c.set_error("no plan space loaded");
    return GPB_CONFIG_ERROR;
  }
  cudaSetDevice(c.device);
  std::vector<TlSlot> slots;
  int rc = build_timelines(c, &row, 1, 0, slots);
  if (rc != GPB_OK) return rc;
  const TlSlot& s = slots[0];
  if (s.Ce > 32) {
    c.set_error("validation supports at most 32 pipelines per cell");
    return GPB_CONFIG_ERROR;
  }
  const long long n = (long long)s.Ce * s.S * s.M;
  long long* dfe = (long long*)c.b_tl_spans.ptr;
  long long* dps = dfe + std::max(1LL, n);
  cudaStream_t st = c.stream;
  if (fe && ps) {  // validate the caller's arrays instead of the device's own
    cudaMemcpyAsync(dfe, fe, 8 * n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dps, ps, 8 * n, cudaMemcpyHostToDevice, st);
  }
  unsigned long long* dres = (unsigned long long*)c.dev_buf(c.b_pack_misc, 64);
  if (!dres) return c.cuda_fail(cudaErrorMemoryAllocation, "validate");
  const unsigned long long init[2] = {~0ULL, 0ULL};
  cudaMemcpyAsync(dres, init, 16, cudaMemcpyHostToDevice, st);
  gpb_row r;
  cudaMemcpyAsync(&r, (gpb_row*)c.b_tl_rows.ptr + row, sizeof r, cudaMemcpyDeviceToHost, st);
  const int threads = 128;
  const int items = s.Ce * s.S + 2 * (s.S - 1);
  validate_kernel<<<(items + threads - 1) / threads, threads, 0, st>>>(
      (const TlSlot*)c.tl_slots_dev, (const DevScen*)c.b_scens.ptr, (const DevTopo*)c.b_topos.ptr,
      (const int32_t*)c.b_row_scen.ptr, dfe, dps, 0, dres, dres + 1);
  unsigned long long out[2];
  cudaMemcpyAsync(out, dres, 16, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return c.cuda_fail(e, "validate");
  if (out[0] != ~0ULL) {
    *check = (int32_t)(out[0] >> 56);
    if (where) *where = (int64_t)(out[0] & 0x00ffffffffffffffULL);
  } else if ((long long)out[1] != r.makespan_ns) {
    *check = 6;  // makespan is not the last task end
    if (where) *where = (int64_t)out[1];
  } else {
    *check = 0;
    if (where) *where = 0;
  }
  return GPB_OK;
}

// append_allreduce (scheduler.cpp:613-650) of one row from the device: each
// stage's all-reduce starts at the stage's last backward end over every
// replica (horizon_kernel) and lasts ar_dur_kernel's duration.
extern "C" int gpb_allreduce_tail(gpb_ctx* ctx_, int64_t row, int64_t* start_ns, int64_t* dur_ns,
                                  int32_t cap, int32_t* n_stages) {
  if (!ctx_ || !n_stages) return GPB_ERROR;
  Ctx& c = *reinterpret_cast<Ctx*>(ctx_);
  c.last_error.clear();
  if (!c.loaded) {
    c.set_error("no plan space loaded");
    return GPB_CONFIG_ERROR;
  }
  cudaSetDevice(c.device);
  std::vector<TlSlot> slots;
  int rc = build_timelines(c, &row, 1, 0, slots, true);
  if (rc != GPB_OK) return rc;
  const int S = slots[0].S;
  *n_stages = S;
  if (start_ns && dur_ns && cap >= S) {
    cudaMemcpyAsync(dur_ns, c.tl_ar, 8 * (size_t)S, cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(start_ns, c.tl_ar + S, 8 * (size_t)S, cudaMemcpyDeviceToHost, c.stream);
    const cudaError_t e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) return c.cuda_fail(e, "allreduce tail");
  }
  return GPB_OK;
}
