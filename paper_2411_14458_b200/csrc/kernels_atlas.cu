// kernels_atlas.cu — the ATLAS temporal-bandwidth-sharing schedule
// (scheduler.cpp:276-538) evaluated one warp per plan row on sm_100a.
//
// Reservation lists (base.h:63-124). Every interval on a boundary's pooled
// link has the same length (that boundary's pooled serialization time), and
// one pipeline's reservations on a link are made in microbatch order at
// increasing times. A link's list is therefore kept as C append-only,
// time-sorted arrays indexed [pipeline][microbatch] (no sorted inserts);
// earliest_fit / free_at / latest_fit run over their union and return
// exactly the reference's answers (each is "the extreme feasible start",
// which the union walk preserves).
//
// Forward phase (scheduler.cpp:362-431): memory-cap admission first. The
// reference drains "the deepest stage with a ready pair" one pair at a time;
// draining stage s never readies a deeper stage, so an admission is one
// descending pass over the stages, run by lane 0 with the stage-above state
// forwarded in registers. The chain of one microbatch is then a max-plus map
// of its start t0: e_s(t0) = a_s + f + max(t0, G_s), a_s = s*f + sum of the
// WAN (ser + lat) below s, G_s = max_{j<=s}(gpu_free_j - a_j) (warp
// max-scan), so the exact-fit shift loop touches only the WAN boundaries.
//
// Drain (scheduler.cpp:452-505): the global greedy commits pairs in
// non-decreasing start time and stage s depends only on itself, its private
// gradient link and the gradient arrivals of stage s+1; it equals a per-stage
// greedy. Lanes run those per-stage greedies as a lock-step
// wavefront: stage s commits its best (t, p) only if t < last_commit(s+1) +
// pair_dur, the earliest any later gradient from s+1 can arrive.
//
// Right-pack (scheduler.cpp:506-529) runs only in the timeline variant.
#include <cuda_runtime.h>

#include "atlas_layout.h"
#include "eval_common.cuh"

namespace gpb {

constexpr int kAtlasQ = 2;  // commits per stage per wavefront round

// ------------------------------------------------------- union of lists

// first index i of a sorted start array with st[i] + len > x. Queries land
// near the tail (reservations are made in time order), so probe backwards a
// few entries before falling back to bisection.
__device__ __forceinline__ int first_end_after(const long long* st, int n, long long len,
                                               long long x) {
  int i = n;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (i == 0 || st[i - 1] + len <= x) return i;
    --i;
  }
  int lo = 0, hi = i;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (st[mid] + len > x) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// Counts of the C per-pipeline arrays of one link.
struct LinkCounts {
  const int* nm;   // nm[q * S + s] (res_bwd of stage s), or nullptr
  int S, s;
  int p, m;        // pipeline whose count is overridden by m (-1: none)
  int mode;        // 0: res_bwd counts from nm; 1: res_fwd (q<p: M, q==p: m)
  int M;
  __device__ __forceinline__ int count(int q) const {
    if (mode == 1) return q < p ? M : (q == p ? m : 0);
    return q == p ? m : nm[q * S + s];
  }
};

// earliest_fit (base.h:75-84) over the union.
__device__ __forceinline__ long long union_earliest_fit(const long long* base, int C, int M,
                                                        const LinkCounts& k, long long lo,
                                                        long long len) {
  if (len <= 0) return lo;
  long long t = lo;
  for (;;) {
    bool changed = false;
    for (int q = 0; q < C; ++q) {
      const int n = k.count(q);
      if (n == 0) continue;
      const long long* st = base + (size_t)q * M;
      if (st[n - 1] + len <= t) continue;
      int i = first_end_after(st, n, len, t);
      while (i < n && st[i] < t + len) {
        t = st[i] + len;
        ++i;
        changed = true;
      }
    }
    if (!changed) return t;
  }
}

// free_at (base.h:65-72) over the union.
__device__ __forceinline__ bool union_free_at(const long long* base, int C, int M,
                                              const LinkCounts& k, long long start,
                                              long long len) {
  if (len <= 0) return true;
  for (int q = 0; q < C; ++q) {
    const int n = k.count(q);
    if (n == 0) continue;
    const long long* st = base + (size_t)q * M;
    if (st[n - 1] + len <= start) continue;
    const int i = first_end_after(st, n, len, start);
    if (i < n && st[i] < start + len) return false;
  }
  return true;
}

// latest_fit (base.h:88-99) over the union, ignoring entry (skip_q, skip_i)
// (the pair's own reservation, unreserved by the caller).
__device__ __forceinline__ long long union_latest_fit(const long long* base, int C, int M,
                                                      const LinkCounts& k, long long lo,
                                                      long long hi, long long len, int skip_q,
                                                      int skip_i) {
  if (hi < lo) return lo - 1;
  if (len <= 0) return hi;
  long long t = hi;
  for (;;) {
    bool changed = false;
    for (int q = 0; q < C; ++q) {
      const int n = k.count(q);
      const long long* st = base + (size_t)q * M;
      int lo_i = 0, hi_i = n;  // first index with st[i] >= t + len
      while (lo_i < hi_i) {
        const int mid = (lo_i + hi_i) >> 1;
        if (st[mid] < t + len) lo_i = mid + 1; else hi_i = mid;
      }
      for (int i = lo_i - 1; i >= 0; --i) {
        if (q == skip_q && i == skip_i) continue;
        if (st[i] >= t + len) continue;
        if (st[i] + len <= t) break;
        t = st[i] - len;
        changed = true;
        if (t < lo) return lo - 1;
      }
    }
    if (!changed) return t >= lo ? t : lo - 1;
  }
}

// free_at over the union, one lane per pipeline list (warp-uniform result).
__device__ __forceinline__ bool warp_union_free_at(const long long* base, int C, int M,
                                                   const LinkCounts& k, long long start,
                                                   long long len) {
  if (len <= 0) return true;
  bool conflict = false;
  for (int q = threadIdx.x & 31; q < C; q += 32) {
    const int n = k.count(q);
    if (n == 0) continue;
    const long long* st = base + (size_t)q * M;
    if (st[n - 1] + len <= start) continue;
    const int i = first_end_after(st, n, len, start);
    if (i < n && st[i] < start + len) conflict = true;
  }
  return !__any_sync(0xffffffffu, conflict);
}

// earliest_fit over the union: every lane pushes t past the overlapping run
// of its own list; the warp max of the proposals keeps "no feasible start in
// [lo, t)" invariant, and the fixpoint is the reference's answer.
__device__ __forceinline__ long long warp_union_earliest_fit(const long long* base, int C, int M,
                                                             const LinkCounts& k, long long lo,
                                                             long long len) {
  if (len <= 0) return lo;
  long long t = lo;
  for (;;) {
    long long my = t;
    for (int q = threadIdx.x & 31; q < C; q += 32) {
      const int n = k.count(q);
      if (n == 0) continue;
      const long long* st = base + (size_t)q * M;
      if (st[n - 1] + len <= my) continue;
      int i = first_end_after(st, n, len, my);
      while (i < n && st[i] < my + len) {
        my = st[i] + len;
        ++i;
      }
    }
    long long nt = my;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nt = imax(nt, __shfl_xor_sync(0xffffffffu, nt, o));
    if (nt == t) return t;
    t = nt;
  }
}

// ------------------------------------------------------------ the warp

struct AtlasMem {
  long long *wa, *wg, *gf, *cand, *lastc, *fdl, *resf, *resb, *garr, *pub_last;
  int *wbs, *nm, *done, *firstm, *pub_nm, *pub_done;
  long long* fe;  // timeline: forward ends [C][S][M] (global)
  long long* ps;  // timeline: pair starts  [C][S][M] (global)

  __device__ void carve(unsigned char* base, const AtlasLayout& L, long long* garr_global) {
    wa = (long long*)(base + L.off_wa);
    wg = (long long*)(base + L.off_wg);
    wbs = (int*)(base + L.off_wbs);
    gf = (long long*)(base + L.off_gf);
    cand = (long long*)(base + L.off_cand);
    lastc = (long long*)(base + L.off_lastc);
    nm = (int*)(base + L.off_nm);
    done = (int*)(base + L.off_done);
    firstm = (int*)(base + L.off_firstm);
    pub_nm = (int*)(base + L.off_pub_nm);
    pub_last = (long long*)(base + L.off_pub_last);
    pub_done = (int*)(base + L.off_pub_done);
    fdl = (long long*)(base + L.off_fdl);
    resf = (long long*)(base + L.off_resf);
    resb = (long long*)(base + L.off_resb);
    garr = L.garr_in_smem ? (long long*)(base + L.off_garr) : garr_global;
    fe = ps = nullptr;
  }
};

// Candidate start of pair (p, s, m): atlas_pair_start(max(ready, gpu_free))
// (scheduler.cpp:461-485, 287-294); the caller guarantees readiness.
__device__ __forceinline__ long long atlas_cand(const Geom& g, const AtlasMem& X, int p, int s,
                                                int m, int wb, long long serb) {
  const int S = g.S, M = g.M, C = g.C;
  const long long ready = s == S - 1 ? X.fdl[p * M + m] : X.garr[((size_t)p * S + s) * M + m];
  const long long lo = imax(ready, X.gf[p * S + s]);
  if (wb < 0) return lo;
  LinkCounts k{X.nm, S, s, -1, 0, 0, M};
  return union_earliest_fit(X.resb + (size_t)wb * C * M, C, M, k, lo + g.dur, serb) - g.dur;
}

template <int B, bool TIMELINE>
__device__ long long atlas_row(const Geom& g, int mem_limit, AtlasMem& X, int& err,
                               long long* phase = nullptr) {
  const int lane = threadIdx.x & 31;
  long long ph_casc = 0, ph_chain = 0, ph_fit = 0, ph_drain = 0, ph_t = 0;
  long long n_stage_it = 0, n_pairs = 0, n_adm = 0;
  const int S = g.S, M = g.M, C = g.C;
  const long long f = g.fwd, dur = g.dur;
  const int nw = g.nb - 1;
  for (int i = lane; i < C * S; i += 32) {
    X.gf[i] = 0;
    X.nm[i] = 0;
  }
  for (int s = lane; s < S; s += 32) {
    int w;
    X.wbs[s] = (s > 0 && wan_after(g, s - 1, w)) ? w : -1;
    X.done[s] = 0;
  }
  if (lane < nw) {  // pooled serialization / latency per WAN boundary
    X.wa[8 + lane] = g.ser_pooled[lane];
    X.wg[8 + lane] = g.lat[lane];
  }
  __syncwarp();

  // Per-lane stage info and chain offsets a_s (lane prefix + warp scan).
  int wbi[B];
  long long serb[B], latb[B], a_loc[B];
  long long run = 0;
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const int s = lane * B + j;
    wbi[j] = -1;
    serb[j] = latb[j] = 0;
    a_loc[j] = run;
    if (s < S) {
      int w;
      if (s > 0 && wan_after(g, s - 1, w)) {
        wbi[j] = w;
        serb[j] = g.ser_pooled[w];
        latb[j] = g.lat[w];
      }
      run += f;
      if (s + 1 < S && wan_after(g, s, w)) run += g.ser_pooled[w] + g.lat[w];
    }
  }
  {
    long long incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = shfl_up64(incl, o);
      if (lane >= o) incl += v;
    }
    const long long excl = incl - run;
#pragma unroll
    for (int j = 0; j < B; ++j) a_loc[j] += excl;
  }

  // ------------------------------------------------------ forward phase
  // Per-lane registers for the current pipeline p: gpu_free and drained
  // counts of the owned stages (written back to shared memory per p).
  long long gfr[B];
  int drr[B];
  for (int p = 0; p < C; ++p) {
#pragma unroll
    for (int j = 0; j < B; ++j) {
      gfr[j] = 0;
      drr[j] = 0;
    }
    for (int m = 0; m < M; ++m) {
      // memory-cap admission (:366-381) + forced drains (:321-346)
      if (phase) ph_t = clock64();
      int nblk = 0;
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (lane * B + j < S && m - drr[j] >= mem_limit) ++nblk;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nblk += __shfl_xor_sync(kFull, nblk, o);
      if (nblk > 0) {
        // The cascade is one descending pass over the stages; it runs in
        // lane 0 on shared copies of this pipeline's state, forwarding the
        // gradient just produced by the stage above in a register.
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const int s = lane * B + j;
          if (s < S) {
            X.gf[p * S + s] = gfr[j];
            X.nm[p * S + s] = drr[j];
          }
        }
        __syncwarp();
        if (lane == 0) {
          long long* __restrict__ gfp = X.gf + p * S;
          int* __restrict__ nmp = X.nm + p * S;
          long long* __restrict__ garr = X.garr;
          const long long* __restrict__ fdl = X.fdl + p * M;
          int nb = nblk, up = m, carry_m = -1;
          long long carry = 0;
          // software-pipelined: stage s-1's state is loaded while s drains
          int n_dm = nmp[S - 1], n_w = X.wbs[S - 1];
          long long n_gf = gfp[S - 1];
          for (int s = S - 1; s >= 0 && nb > 0; --s) {
            int dm = n_dm;
            const int w = n_w;
            long long gfi = n_gf;
            if (s > 0) {
              n_dm = nmp[s - 1];
              n_w = X.wbs[s - 1];
              n_gf = gfp[s - 1];
            }
            const int u = up;
            up = dm;
            ++n_stage_it;
            if (dm >= M || dm >= u) {  // no ready pair: nothing new for s-1
              carry_m = -1;
              continue;
            }
            const long long ser = w >= 0 ? X.wa[8 + w] : 0;  // boundary constants
            const long long lat = w >= 0 ? X.wg[8 + w] : 0;
            long long produced = 0;
            int pm = -1;
            while (dm < M && dm < u && nb > 0) {
              const long long ready =
                  s == S - 1 ? fdl[dm]
                             : (dm == carry_m ? carry : garr[((size_t)p * S + s) * M + dm]);
              const long long lo = imax(ready, gfi);
              long long t = lo;
              if (w >= 0) {
                long long* base = X.resb + (size_t)w * C * M;
                LinkCounts k{X.nm, S, s, p, dm, 0, M};
                t = union_earliest_fit(base, C, M, k, lo + dur, ser) - dur;
                base[(size_t)p * M + dm] = t + dur;  // reserve (append to list p)
              }
              const long long e = t + dur;  // atlas_commit_pair (:298-317)
              gfi = imax(gfi, e);
              produced = w >= 0 ? e + ser + lat : e;
              pm = dm;
              if (s > 0) garr[((size_t)p * S + s - 1) * M + dm] = produced;
              if (TIMELINE) X.ps[((size_t)p * S + s) * M + dm] = t;
              if (m - dm >= mem_limit && m - (dm + 1) < mem_limit) --nb;
              ++dm;
              ++n_pairs;
            }
            gfp[s] = gfi;
            nmp[s] = dm;
            up = dm;
            carry = produced;
            carry_m = pm;
          }
          X.done[0] = nb;  // > 0: DeadlockError (unreachable)
          ++n_adm;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const int s = lane * B + j;
          if (s < S) {
            gfr[j] = X.gf[p * S + s];
            drr[j] = X.nm[p * S + s];
          }
        }
        if (X.done[0] > 0) {
          err = 1;
          return 0;
        }
      }
      if (phase) {
        const long long t1 = clock64();
        ph_casc += t1 - ph_t;
        ph_t = t1;
      }
      // chain: G_s prefix max (lane-local, then warp inclusive scan)
      long long gl[B];
      long long runmax = -kInf64;
#pragma unroll
      for (int j = 0; j < B; ++j) {
        if (lane * B + j < S) runmax = imax(runmax, gfr[j] - a_loc[j]);
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
#pragma unroll
      for (int j = 0; j < B; ++j) {
        gl[j] = imax(gl[j], prev);
        const int s = lane * B + j;
        int w;
        if (s + 1 < S && wan_after(g, s, w)) {
          X.wa[w] = a_loc[j];
          X.wg[w] = gl[j];
        }
      }
      long long t0 = __shfl_sync(kFull, gfr[0], 0);  // gpu_free of stage 0
      __syncwarp();
      if (phase) {
        const long long t1 = clock64();
        ph_chain += t1 - ph_t;
        ph_t = t1;
      }
      // exact-fit shift loop over the WAN boundaries (:383-405), one lane per
      // pipeline list of each link, then the chain's reservations (:407-430)
      {
        LinkCounts k{nullptr, S, 0, p, m, 1, M};
        for (int w = 0; w < nw;) {
          const long long e = X.wa[w] + f + imax(t0, X.wg[w]);
          const long long* base = X.resf + (size_t)w * C * M;
          const long long len = g.ser_pooled[w];
          if (!warp_union_free_at(base, C, M, k, e, len)) {
            t0 += warp_union_earliest_fit(base, C, M, k, e, len) - e;
            w = 0;  // restart the chain
          } else {
            ++w;
          }
        }
        if (lane < nw)
          X.resf[((size_t)lane * C + p) * M + m] = X.wa[lane] + f + imax(t0, X.wg[lane]);
      }
      if (phase) {
        const long long t1 = clock64();
        ph_fit += t1 - ph_t;
        ph_t = t1;
      }
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int s = lane * B + j;
        if (s < S) {
          const long long e = a_loc[j] + f + imax(t0, gl[j]);
          gfr[j] = e;
          if (s == S - 1) X.fdl[p * M + m] = e;
          if (TIMELINE) X.fe[((size_t)p * S + s) * M + m] = e;
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int s = lane * B + j;
      if (s < S) {
        X.gf[p * S + s] = gfr[j];
        X.nm[p * S + s] = drr[j];
      }
    }
    __syncwarp();
  }

  if (phase) ph_t = clock64();
  // ------------------------------------------ drain: per-stage wavefront
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const int s = lane * B + j;
    if (s < S) {
      X.lastc[s] = -kInf64;
      int all = 1;
      for (int p = 0; p < C; ++p) {
        const int i = p * S + s;
        const int m = X.nm[i];
        X.firstm[i] = m;
        all &= m >= M;
        const bool ready = m < M && (s == S - 1 || X.nm[i + 1] > m);
        X.cand[i] = ready ? atlas_cand(g, X, p, s, m, wbi[j], serb[j]) : kInf64;
      }
      X.done[s] = all;
    }
  }
  __syncwarp();
  auto publish = [&]() {
    const int s0 = lane * B;
    if (s0 < S) {
      for (int p = 0; p < C; ++p) X.pub_nm[p * 32 + lane] = X.nm[p * S + s0];
      X.pub_last[lane] = X.lastc[s0];
      X.pub_done[lane] = X.done[s0];
    } else {
      X.pub_done[lane] = 1;
    }
  };
  publish();
  __syncwarp();
  for (;;) {
    bool active = false;
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int s = lane * B + j;
      if (s < S && !X.done[s]) active = true;
    }
    if (!__any_sync(kFull, active)) break;
#pragma unroll
    for (int j = B - 1; j >= 0; --j) {
      const int s = lane * B + j;
      if (s >= S || X.done[s]) continue;
      const bool up = s + 1 < S;
      const bool up_pub = up && j == B - 1;  // stage s+1 lives in lane+1
      int up_done = 1;
      long long up_last = kInf64;
      if (up) {
        up_done = up_pub ? X.pub_done[lane + 1] : X.done[s + 1];
        up_last = up_pub ? X.pub_last[lane + 1] : X.lastc[s + 1];
      }
      for (int p = 0; p < C; ++p) {  // gradients that arrived since last round
        const int i = p * S + s;
        const int m = X.nm[i];
        if (m < M && X.cand[i] == kInf64) {
          const int un = !up ? M : (up_pub ? X.pub_nm[p * 32 + lane + 1] : X.nm[i + 1]);
          if (un > m) X.cand[i] = atlas_cand(g, X, p, s, m, wbi[j], serb[j]);
        }
      }
      const long long bound =
          (!up || up_done) ? kInf64 : (up_last == -kInf64 ? -kInf64 : up_last + dur);
      for (int q = 0; q < kAtlasQ; ++q) {
        long long bt = kInf64;
        int bp = -1;
        for (int p = 0; p < C; ++p) {
          const long long t = X.cand[p * S + s];
          if (t < bt) {  // strict: lowest p wins ties (scan order p asc)
            bt = t;
            bp = p;
          }
        }
        if (bp < 0 || bt >= bound) break;
        const int i = bp * S + s;
        const int m = X.nm[i];
        const int w = wbi[j];
        if (w >= 0) X.resb[((size_t)w * C + bp) * M + m] = bt + dur;  // reserve
        X.gf[i] = bt + dur;
        if (s > 0)
          X.garr[((size_t)bp * S + s - 1) * M + m] =
              w >= 0 ? bt + dur + serb[j] + latb[j] : bt + dur;
        if (TIMELINE) X.ps[((size_t)bp * S + s) * M + m] = bt;
        X.nm[i] = m + 1;
        X.lastc[s] = bt;
        // refresh: every pipeline of the stage when the gradient link is
        // shared (the new reservation may push them), else only bp
        for (int p = w >= 0 ? 0 : bp; p < (w >= 0 ? C : bp + 1); ++p) {
          const int i2 = p * S + s;
          const int m2 = X.nm[i2];
          const int un = !up ? M : (up_pub ? X.pub_nm[p * 32 + lane + 1] : X.nm[i2 + 1]);
          X.cand[i2] = (m2 < M && un > m2) ? atlas_cand(g, X, p, s, m2, w, serb[j]) : kInf64;
        }
      }
      int all = 1;
      for (int p = 0; p < C; ++p) all &= X.nm[p * S + s] >= M;
      X.done[s] = all;
    }
    __syncwarp();
    publish();
    __syncwarp();
  }

  if (phase && lane == 0) {
    ph_drain = clock64() - ph_t;
    phase[0] = ph_casc;
    phase[1] = ph_chain;
    phase[2] = ph_fit;
    phase[3] = ph_drain;
    phase[4] = n_stage_it;
    phase[5] = n_pairs;
    phase[6] = n_adm;
  }
  // -------------------------------------------- right-pack (timeline)
  if (TIMELINE) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        const int w = X.wbs[s];
        const long long ser = w >= 0 ? g.ser_pooled[w] : 0;
        long long* base = w >= 0 ? X.resb + (size_t)w * C * M : nullptr;
        LinkCounts k{X.nm, S, s, -1, 0, 0, M};
        for (int p = 0; p < C; ++p) {
          for (int m = M - 2; m >= X.firstm[p * S + s]; --m) {
            const size_t kk = ((size_t)p * S + s) * M + m;
            const long long cur = X.ps[kk];
            long long end_max = X.ps[kk + 1];
            if (s > 0) {
              const long long consumer = X.ps[((size_t)p * S + s - 1) * M + m];
              end_max = imin(end_max, w >= 0 ? consumer - g.lat[w] - ser : consumer);
            }
            if (end_max <= cur + dur) continue;
            if (w >= 0 && ser > 0) {
              // unreserve own slot, latest fit, reserve (index m of list p)
              const long long slot =
                  union_latest_fit(base, C, M, k, cur + dur, end_max, ser, p, m);
              X.ps[kk] = slot - dur;
              base[(size_t)p * M + m] = slot;
            } else {
              X.ps[kk] = end_max - dur;
            }
          }
        }
      }
    }
    __syncwarp();
  }
  long long mk = 0;
  for (int i = lane; i < C * S; i += 32) mk = imax(mk, X.gf[i]);
  return warp_max64(mk);
}

template <int B>
__global__ void __launch_bounds__(kEvalThreads) atlas_kernel(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + warp;
  AtlasMem X;
  X.carve(smem + (size_t)warp * a.lay.total, a.lay,
          a.scratch ? a.scratch + (size_t)gwarp * a.scratch_per_warp : nullptr);
  for (;;) {
    const int wk = next_work(a.cursor);
    if (wk >= a.n_work) break;
    const int row = a.work[wk];
    const long long t_start = clock64();
    Geom g;
    const DevScen* sc;
    const DevTopo* tp;
    if (!begin_row(a, row, g, sc, tp)) continue;
    int err = 0;
    const long long mk = atlas_row<B, false>(g, sc->mem_limit, X, err,
                                             a.row_phase ? a.row_phase + 8 * (size_t)row : nullptr);
    end_row(a, row, g, *sc, *tp, mk, err, t_start);
    __syncwarp();
  }
}

template <int B>
__global__ void __launch_bounds__(kEvalThreads) atlas_timeline_kernel(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + warp;
  AtlasMem X;
  X.carve(smem + (size_t)warp * a.lay.total, a.lay,
          a.scratch ? a.scratch + (size_t)gwarp * a.scratch_per_warp : nullptr);
  for (;;) {
    const int wk = next_work(a.cursor);
    if (wk >= a.n_work) break;
    const int row = a.work[wk];
    const long long t_start = clock64();
    Geom g;
    const DevScen* sc;
    const DevTopo* tp;
    if (!begin_row(a, row, g, sc, tp)) continue;
    X.fe = a.tl_fe + a.tl_off[wk];
    X.ps = a.tl_ps + a.tl_off[wk];
    int err = 0;
    const long long mk = atlas_row<B, true>(g, sc->mem_limit, X, err);
    end_row(a, row, g, *sc, *tp, mk, err, t_start);
    __syncwarp();
  }
}

template <int B>
static cudaError_t launch_atlas_tl_b(const EvalArgs& a, int grid, int wpc, cudaStream_t st) {
  const size_t smem = (size_t)wpc * a.lay.total;
  cudaError_t e = cudaFuncSetAttribute(atlas_timeline_kernel<B>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  atlas_timeline_kernel<B><<<grid, 32 * wpc, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_atlas_timeline(int B, const EvalArgs& a, int grid, int wpc, cudaStream_t st) {
  switch (B) {
    case 1: return launch_atlas_tl_b<1>(a, grid, wpc, st);
    case 2: return launch_atlas_tl_b<2>(a, grid, wpc, st);
    case 3: return launch_atlas_tl_b<3>(a, grid, wpc, st);
    case 4: return launch_atlas_tl_b<4>(a, grid, wpc, st);
    case 5: return launch_atlas_tl_b<5>(a, grid, wpc, st);
    case 6: return launch_atlas_tl_b<6>(a, grid, wpc, st);
    case 7: return launch_atlas_tl_b<7>(a, grid, wpc, st);
    case 8: return launch_atlas_tl_b<8>(a, grid, wpc, st);
  }
  return cudaErrorInvalidValue;
}

template <int B>
static cudaError_t launch_atlas_b(const EvalArgs& a, int grid, int wpc, cudaStream_t st) {
  const size_t smem = (size_t)wpc * a.lay.total;
  cudaError_t e = cudaFuncSetAttribute(atlas_kernel<B>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  atlas_kernel<B><<<grid, 32 * wpc, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_atlas(int B, const EvalArgs& a, int grid, int wpc, cudaStream_t st) {
  switch (B) {
    case 1: return launch_atlas_b<1>(a, grid, wpc, st);
    case 2: return launch_atlas_b<2>(a, grid, wpc, st);
    case 3: return launch_atlas_b<3>(a, grid, wpc, st);
    case 4: return launch_atlas_b<4>(a, grid, wpc, st);
    case 5: return launch_atlas_b<5>(a, grid, wpc, st);
    case 6: return launch_atlas_b<6>(a, grid, wpc, st);
    case 7: return launch_atlas_b<7>(a, grid, wpc, st);
    case 8: return launch_atlas_b<8>(a, grid, wpc, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace gpb
