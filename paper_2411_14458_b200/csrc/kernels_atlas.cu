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
// descending pass over the stages, evaluated in rounds of warp suffix scans
// (atlas_cascade, lane = stage). The chain of one microbatch is then a max-plus map
// of its start t0: e_s(t0) = a_s + f + max(t0, G_s), a_s = s*f + sum of the
// WAN (ser + lat) below s, G_s = max_{j<=s}(gpu_free_j - a_j) (warp
// max-scan), so the exact-fit shift loop touches only the WAN boundaries.
//
// Drain (scheduler.cpp:452-505): the global greedy commits pairs in
// non-decreasing start time and stage s depends only on itself, its private
// gradient link and the gradient arrivals of stage s+1; it equals a per-stage
// greedy, run from stage S-1 down: a WAN stage as a warp
// argmin over its pipelines (lane = pipeline), a run of stages without a WAN
// gradient link as segmented prefix-max scans or one 2-D wavefront.
//
// Right-pack (scheduler.cpp:506-529) runs only in the timeline variant.
#include <cuda_runtime.h>

#include <mutex>

#include "atlas_layout.h"
#include "eval_common.cuh"

namespace gpb {

// ------------------------------------------------------- union of lists

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

// ------------------------------------------------------------ the warp

struct AtlasMem {
  long long *wa, *wg, *gf, *fdl, *resf, *resb, *garr;
  long long *garr_smem, *garr_glob;
  long long garr_cap;
  int *wbs, *nm, *firstm;
  long long *mf, *mb, *mtmp;  // merged static link lists (forward phase)
  int *jf, *jb;               // their run jumps
  int* mcnt;                  // [w] |mf|, [8+w] |mb|, [16+w] mb cursor
  long long* fe;  // timeline: forward ends [C][S][M] (global)
  long long* ps;  // timeline: pair starts  [C][S][M] (global)

  // small state in the warp's shared slice; the lists ("big" region) there
  // too when they fit, else in the warp's global scratch
  __device__ void carve(unsigned char* base, const AtlasLayout& L, long long* garr_global,
                        unsigned char* big_global) {
    wa = (long long*)(base + L.off_wa);
    wg = (long long*)(base + L.off_wg);
    wbs = (int*)(base + L.off_wbs);
    gf = (long long*)(base + L.off_gf);
    nm = (int*)(base + L.off_nm);
    firstm = (int*)(base + L.off_firstm);
    mcnt = (int*)(base + L.off_mcnt);
    unsigned char* big = L.big_in_smem ? base + L.off_big : big_global;
    fdl = (long long*)(big + L.off_fdl);
    resf = (long long*)(big + L.off_resf);
    resb = (long long*)(big + L.off_resb);
    mf = (long long*)(big + L.off_mf);
    mb = (long long*)(big + L.off_mb);
    mtmp = (long long*)(big + L.off_mtmp);
    jf = (int*)(big + L.off_jf);
    jb = (int*)(big + L.off_jb);
    garr_smem = (long long*)(base + L.off_garr);
    garr_glob = garr_global;
    garr_cap = L.garr_cap;
    garr = garr_smem;
    fe = ps = nullptr;
  }
};

// ------------------------------------------- forward-phase link lists
//
// While pipeline p runs its forward phase (chains + memory-cap drains), every
// other pipeline's reservations on every link are fixed: pipelines q < p are
// finished (their remaining pairs drain after all forwards) and q > p have
// none. So each link is one static sorted list — the merge of pipelines
// 0..p-1, rebuilt when p starts — plus p's own append-only list. Queries on a
// link during p's phase come in non-decreasing time order and always start
// after p's own last reservation (gpu_free grows), so only the own tail can
// overlap: a monotone cursor over the static list plus one comparison with
// the own tail answer free_at / earliest_fit (base.h:65-84) exactly.

// past-the-end value of a list (above every time; see LinkCur)
constexpr long long kEndCur = 1LL << 60;

// A[0..na) <- merge(A, Bv[0..nb)) through tmp (warp-parallel; A wins ties).
__device__ __forceinline__ void warp_merge(long long* A, int na, const long long* Bv, int nb,
                                           long long* tmp) {
  // Merge path: lane l writes outputs [l*k, l*k + k); one bisection finds how
  // many of A precede its first output (A[i] goes before Bv[j] iff A[i] <=
  // Bv[j]), then a sequential two-cursor merge of its k outputs (one new
  // load per output instead of a bisection per element).
  const int lane = threadIdx.x & 31;
  const int n = na + nb, k = (n + 31) >> 5;
  const int d = min(lane * k, n), d_end = min(d + k, n);
  int lo = max(0, d - nb), hi = min(d, na);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] <= Bv[d - mid - 1]) lo = mid + 1; else hi = mid;
  }
  int i = lo, j = d - lo;
  long long a = i < na ? A[i] : kEndCur, b = j < nb ? Bv[j] : kEndCur;
  for (int o = d; o < d_end; ++o) {
    if (j >= nb || (i < na && a <= b)) {
      tmp[o] = a;
      ++i;
      a = i < na ? A[i] : kEndCur;
    } else {
      tmp[o] = b;
      ++j;
      b = j < nb ? Bv[j] : kEndCur;
    }
  }
  __syncwarp();
  for (int x = lane; x < n; x += 32) A[x] = tmp[x];
  __syncwarp();
}

// Cursor into a static list: index i and the entry there (kEndCur past the
// end), so the common "no advance" check needs no load.
struct LinkCur {
  int i;
  long long v;
  __device__ __forceinline__ void reset(const long long* mg, int n) {
    i = 0;
    v = n > 0 ? mg[0] : kEndCur;
  }
  __device__ __forceinline__ void set(const long long* mg, int n, int k) {
    i = k;
    v = k < n ? mg[k] : kEndCur;
  }
};

// Advance the cursor to the first static entry ending after x (gallop from
// the cursor, then bisect).
__device__ __forceinline__ void link_advance(const long long* mg, int n, LinkCur& c, long long len,
                                             long long x) {
  if (c.v + len > x) return;
  const int cur = c.i;
  // the next four entries in one round of independent loads (a query usually
  // moves the cursor by about the number of earlier pipelines); past the end
  // reads as kEndCur, which ends after every query
  const long long v1 = cur + 1 < n ? mg[cur + 1] : kEndCur,
                  v2 = cur + 2 < n ? mg[cur + 2] : kEndCur,
                  v3 = cur + 3 < n ? mg[cur + 3] : kEndCur,
                  v4 = cur + 4 < n ? mg[cur + 4] : kEndCur;
  if (v1 + len > x) {
    c.i = cur + 1;
    c.v = v1;
    return;
  }
  if (v2 + len > x) {
    c.i = cur + 2;
    c.v = v2;
    return;
  }
  if (v3 + len > x) {
    c.i = cur + 3;
    c.v = v3;
    return;
  }
  if (v4 + len > x) {
    c.i = cur + 4;
    c.v = v4;
    return;
  }
  int lo = cur + 5, step = 1;
  while (lo + step - 1 < n && mg[lo + step - 1] + len <= x) {
    lo += step;
    step <<= 1;
  }
  int hi = min(lo + step - 1, n);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (mg[mid] + len <= x) lo = mid + 1; else hi = mid;
  }
  c.set(mg, n, lo);
}

// Run jumps of a static list whose intervals all have length len:
// jmp[i] = the first j >= i after which a free gap of at least len opens
// (mg[j+1] - (mg[j] + len) >= len, or j = n-1). earliest_fit that overlaps
// entry i lands exactly at mg[jmp[i]] + len. Warp-parallel from the tail,
// 32 entries per step.
__device__ __forceinline__ void warp_jumps(const long long* mg, int n, long long len, int* jmp) {
  const int lane = threadIdx.x & 31;
  int carry = n - 1;  // first flagged index of the part already done
  for (int base = ((n - 1) >> 5) << 5; base >= 0 && n > 0; base -= 32) {
    const int i = base + lane;
    const bool flag = i < n && (i == n - 1 || mg[i + 1] - mg[i] - len >= len);
    const unsigned fm = __ballot_sync(kFull, flag) & (0xffffffffu << lane);
    if (i < n) jmp[i] = fm ? base + __ffs(fm) - 1 : carry;
    const unsigned all = __ballot_sync(kFull, flag);
    if (all) carry = base + __ffs(all) - 1;
  }
  __syncwarp();
}

// [x, x+len) overlaps a static entry (cursor `cur`, advanced) or the own tail
__device__ __forceinline__ bool link_conflict(const long long* mg, int n, LinkCur& c,
                                              long long own_last, long long len, long long x) {
  if (len <= 0) return false;
  link_advance(mg, n, c, len, x);
  if (c.v < x + len) return true;
  return own_last + len > x;
}

// earliest_fit over the static list and the own tail; a run of back-to-back
// static entries is crossed in one step through the jump table
__device__ __forceinline__ long long link_fit(const long long* mg, const int* jmp, int n, LinkCur& c,
                                              long long own_last, long long len, long long x) {
  if (len <= 0) return x;
  long long t = x;
  for (;;) {
    link_advance(mg, n, c, len, t);
    if (c.v < t + len) {
      const int k = jmp[c.i];
      t = mg[k] + len;
      c.set(mg, n, k + 1);
      continue;
    }
    if (own_last + len > t) {
      t = own_last + len;
      continue;
    }
    return t;
  }
}

// -inf of the max-plus maps (see the admission cascade below).
constexpr long long kNegMP = -(1LL << 53);

// Gradient-link queries of the admission cascade, per owned stage j (lane
// stage j's WAN gradient link wbi[j]): conflict = free_at fails, fit =
// earliest_fit (base.h:65-84), reserve = append to this pipeline's own list.
// StaticLinks: the frozen pipelines' reservations merged into one list with
// run jumps (one warp evaluates the pipelines in order).
template <int B>
struct StaticLinks {
  const AtlasMem& X;
  int C, M;
  const int (&wbi)[B];
  const long long (&ser)[B];
  long long own[B];
  LinkCur cur[B];
  int n[B];
  __device__ __forceinline__ StaticLinks(const AtlasMem& X_, int C_, int M_, const int (&wbi_)[B],
                                         const long long (&ser_)[B])
      : X(X_), C(C_), M(M_), wbi(wbi_), ser(ser_) {
#pragma unroll
    for (int j = 0; j < B; ++j) {
      own[j] = kNegMP;
      n[j] = wbi[j] >= 0 ? X.mcnt[8 + wbi[j]] : 0;
      cur[j].i = 0;
      cur[j].v = kEndCur;
      if (wbi[j] >= 0) cur[j].reset(X.mb + (size_t)wbi[j] * C * M, n[j]);
    }
  }
  __device__ __forceinline__ bool conflict(int j, long long y) {
    return link_conflict(X.mb + (size_t)wbi[j] * C * M, n[j], cur[j], own[j], ser[j], y);
  }
  __device__ __forceinline__ long long fit(int j, long long y) {
    return link_fit(X.mb + (size_t)wbi[j] * C * M, X.jb + (size_t)wbi[j] * C * M, n[j], cur[j],
                    own[j], ser[j], y);
  }
  __device__ __forceinline__ void reserve(int j, int p, int k, long long e) {
    X.resb[((size_t)wbi[j] * C + p) * M + k] = e;
    own[j] = e;
  }
};

// ------------------------------------------------ admission cascade
//
// The memory-cap admission of microbatch m of pipeline p (scheduler.cpp:
// 366-381) repeats atlas_drain_step (:321-346) — "drain the deepest stage
// with a ready pair" — while some stage s has m - drained[s] >= mem_limit.
// Stage S-1 has every forwarded pair ready; a stage's ready pairs come only
// from the stage above, so the repetition is one descending pass in which
// every stage above the lowest blocked stage s_min drains ALL its ready
// pairs (up to pair m-1, since the stage above reached m) and s_min drains
// up to pair m-mem_limit (then nothing is blocked). Closed form per stage:
//   n_s = m - dm_s (s > s_min), m - L + 1 - dm_s (s = s_min), 0 (s < s_min).
// Order within the pass only matters through data dependencies: pair k at
// stage s needs stage s's previous pair (gpu_free) and the gradient of pair
// k from stage s+1; each gradient link is written by one stage only. So the
// pass is evaluated in rounds: round j drains pair dm_s + j at every stage
// with j < n_s. Inside a round, stage s consumes stage s+1's output of the
// same round iff dm_s == dm_{s+1} ("linked"); otherwise its input was
// produced in an earlier round (memory). A round is a max-plus chain down
// the linked stages: out_s = max(in_s, gf_s) + dur + delta_s + wan_s, with
// delta_s the exact-fit shift on the stage's WAN gradient link
// (atlas_pair_start, :287-294). With the deltas fixed it is a composition
// of maps x -> max(x + a, b), evaluated by one warp suffix scan; the deltas
// are resolved top-down (the topmost conflicting WAN stage has a final
// input), rescanning after each, so a round costs 1 + (#shifted WAN stages)
// scans instead of one sequential step per pair.
// -inf of the max-plus maps. Real times and their sums along a row stay
// below 2^50 ns (13 days) and a composed map sums at most 256 terms (one
// per stage), so plain adds never overflow (|sum| < 2^62) and a map that
// includes a -inf term stays negative, below every real time (no clamping).

__device__ __forceinline__ long long mp_add(long long x, long long y) { return x + y; }

template <int B, bool TIMELINE, bool PROF, typename Links>
__device__ __forceinline__ void atlas_cascade(const Geom& g, int p, int m, int L, AtlasMem& X,
                                              long long (&gfr)[B], int (&drr)[B],
                                              const int (&wbi)[B], const long long (&serb)[B],
                                              const long long (&latb)[B], Links& links,
                                              const long long (&wsuf)[B],
                                              long long& n_pairs,
                                              long long& n_scans, long long& n_rounds,
                                              long long* cph) {
  // links: the gradient-link queries of the stages this lane owns
  long long ct = PROF ? clock64() : 0;
  const int lane = threadIdx.x & 31;
  const int S = g.S, M = g.M, C = g.C;
  const int nl = (S + B - 1) / B;  // lanes owning stages
  const long long dur = g.dur;
  // Lowest blocked stage: a pair drains at stage s only after it drained at
  // s+1 (its gradient), so drained[s] <= drained[s+1] and the callers (stage
  // 0 blocked) always have s_min = 0: stage 0 drains to m - L + 1, every
  // stage above it all its ready pairs, and the most pairs of any stage above
  // are stage 1's (the fewest drained).
  constexpr int s_min = 0;
  // pair counts, links (dm of the stage above: next local stage, or lane+1)
  int cnt[B];
  bool link[B];
  const int up_dm = __shfl_down_sync(kFull, drr[0], 1);
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const int s = lane * B + j;
    cnt[j] = s >= S || s < s_min ? 0 : (s == s_min ? m - L + 1 - drr[j] : m - drr[j]);
    const int dma = j + 1 < B ? drr[j + 1] : up_dm;
    link[j] = s + 1 < S && dma == drr[j];
  }
  const int d0 = __shfl_sync(kFull, drr[0], 0), d1 = __shfl_sync(kFull, drr[B > 1 ? 1 : 0], B > 1 ? 0 : 1);
  const int R = max(m - L + 1 - d0, S > 1 ? m - d1 : 0);
  if (PROF) {
    int tot = 0;
#pragma unroll
    for (int j = 0; j < B; ++j) tot += cnt[j];
    n_pairs += __reduce_add_sync(kFull, tot);
  }
  long long wl[B];  // WAN serialization + latency added to the pair's output
#pragma unroll
  for (int j = 0; j < B; ++j) wl[j] = wbi[j] >= 0 ? serb[j] + latb[j] : 0;

  if (PROF) n_rounds += R;
  if (PROF) {
    const long long t1 = clock64();
    cph[0] += t1 - ct;
    ct = t1;
  }
  for (int r = 0; r < R; ++r) {
    long long xin[B], dl[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int s = lane * B + j;
      dl[j] = 0;
      xin[j] = kNegMP;
      if (r < cnt[j] && !link[j]) {
        const int k = drr[j] + r;
        xin[j] = s == S - 1 ? X.fdl[p * M + k] : X.garr[((size_t)p * S + s) * M + k];
      }
    }
    long long lo[B];
    if (PROF) {
      const long long t1 = clock64();
      cph[1] += t1 - ct;
      ct = t1;
    }
    // The round as one suffix max of one value per stage. A stage's pair
    // starts at lo_s = max(in_s, gf_s); in_s is the output of the stage above
    // (linked) or a stored gradient. With c_s = dur + dl_s + wl_s (dl: the
    // exact-fit shift) and K_s = sum_{i >= s} c_i,
    //   lo_s = K_s + max_{j in seg(s)} (base_j - K_j + c_j) - c_s,
    // seg(s) = s and the linked stages above it up to the first "head" (a
    // stage that is not linked, or idle this round: its output is -inf),
    // base_j = gf_j, max(in_j, gf_j) at a head. The segments are separated
    // by adding kSegBig * (#heads at or above j): every value above a
    // segment is smaller by at least kSegBig (|base - K + c| < 2^51).
    constexpr long long kSegBig = 1LL << 53;
    long long hb[B];  // kSegBig * heads at or above the stage
    {
      int hc[B], loc = 0;
#pragma unroll
      for (int j = B - 1; j >= 0; --j) {
        const int s = lane * B + j;
        if (s < S && (r >= cnt[j] || !link[j])) ++loc;
        hc[j] = loc;
      }
      int incl = loc;
      if (B == 1) {  // one stage per lane: count the heads above by ballot
        incl = __popc(__ballot_sync(kFull, loc != 0) & (0xffffffffu << lane));
      } else {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_down_sync(kFull, incl, o);
          if (lane + o < 32) incl += v;
        }
      }
#pragma unroll
      for (int j = 0; j < B; ++j) hb[j] = kSegBig * (hc[j] + incl - loc);
    }
    long long DLs[B];  // sum of the shifts at stages >= s
#pragma unroll
    for (int j = 0; j < B; ++j) DLs[j] = 0;
    for (;;) {
      if (PROF) ++n_scans;
      long long um[B], run = kNegMP;
#pragma unroll
      for (int j = B - 1; j >= 0; --j) {
        const long long u = r < cnt[j] ? imax(xin[j], gfr[j]) - (wsuf[j] + DLs[j]) +
                                             (dur + dl[j] + wl[j])
                                       : kNegMP;
        run = imax(run, u + hb[j]);
        um[j] = run;
      }
      long long sc = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {  // inclusive suffix max over the owning lanes
        if (o >= nl) break;  // warp-uniform
        const long long ov = shfl_down64(sc, o);
        if (lane + o < nl) sc = imax(sc, ov);
      }
      long long above = shfl_down64(sc, 1);
      if (lane + 1 >= nl) above = kNegMP;
      // evaluate the lane's stages; check the WAN links at their inputs
      int conf = -1;
      long long conf_y = 0;
#pragma unroll
      for (int j = B - 1; j >= 0; --j) {
        lo[j] = wsuf[j] + DLs[j] + (imax(um[j], above) - hb[j]) - (dur + dl[j] + wl[j]);
        const int w = wbi[j];
        if (r < cnt[j] && w >= 0 && conf < 0) {
          const long long y = lo[j] + dur + dl[j];
          if (links.conflict(j, y)) {
            conf = j;
            conf_y = y;
          }
        }
      }
      const unsigned bal = __ballot_sync(kFull, conf >= 0);
      if (!bal) break;
      const int src = 31 - __clz(bal);  // topmost conflict: its input is final
      long long shift = 0;
      if (lane == src) {
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (j == conf) {
            shift = links.fit(j, conf_y) - conf_y;
            dl[j] += shift;
          }
      }
      {  // the shift enters every suffix sum at or below its stage
        const int sw = __shfl_sync(kFull, lane * B + conf, src);
        shift = shfl_idx64(shift, src);
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (lane * B + j <= sw) DLs[j] += shift;
      }
    }
    if (PROF) {
      const long long t1 = clock64();
      cph[2] += t1 - ct;
      ct = t1;
    }
    // commit the round
#pragma unroll
    for (int j = 0; j < B; ++j) {
      if (r >= cnt[j]) continue;
      const int s = lane * B + j;
      const int k = drr[j] + r;
      const long long t = lo[j] + dl[j];
      const long long e = t + dur;
      gfr[j] = e;
      if (wbi[j] >= 0) links.reserve(j, p, k, e);  // reserve (append to list p)
      if (s > 0) X.garr[((size_t)p * S + s - 1) * M + k] = e + wl[j];
      if (TIMELINE) X.ps[((size_t)p * S + s) * M + k] = t;
    }
    __syncwarp();
    if (PROF) {
      const long long t1 = clock64();
      cph[3] += t1 - ct;
      ct = t1;
    }
  }
#pragma unroll
  for (int j = 0; j < B; ++j) drr[j] += cnt[j];
}

// --------------------------------------------------------- drain phase
//
// The reference's drain (scheduler.cpp:461-505) is a global greedy over all
// (pipeline, stage) next pairs. Stage s reads only its own GPUs, its own
// gradient link (boundary s-1) and the gradient arrivals of stage s+1, and
// the greedy commits in non-decreasing start time; a pair that is not ready
// yet becomes ready only after its producer commits, strictly later (pair
// duration > 0). So the global greedy equals, stage by stage from S-1 down,
// a per-stage greedy with every input of the stage known:
//  * a stage without a WAN gradient link has no shared resource: pipeline
//    p's pairs follow e[m] = max(r[m], e[m-1]) + dur, i.e.
//    e[m] = (m+1)*dur + max(gf0 - m0*dur, max_{m0<=j<=m} (r[j] - j*dur)),
//    one segmented prefix-max over the stage's (pipeline, microbatch) pairs
//    (drain_stage_scan); a deep run of such stages with few pairs is one
//    2-D max-plus wavefront instead (drain_run_wavefront);
//  * a stage with a WAN gradient link runs the greedy over its C pipelines
//    (lane = pipeline, warp argmin, lowest pipeline on ties). Its link holds
//    the forward phase's forced drains (a static merged list) plus this
//    stage's commits, which come in non-decreasing time; every later query
//    starts at or after the last commit, so only that one can overlap.

// Stage s without a WAN gradient link: segmented prefix max, K pairs per lane.
template <bool TIMELINE>
__device__ void drain_stage_scan(const Geom& g, AtlasMem& X, int s) {
  constexpr int K = 8;
  const int lane = threadIdx.x & 31;
  const int S = g.S, M = g.M, C = g.C;
  const long long dur = g.dur;
  const int n = C * M;
  // Few pairs left (the memory cap drained most of them in the forward
  // phase, e.g. the config-2 critical row: ~8 of 256 per stage): one pass
  // over the remaining pairs only, one per lane, instead of K pairs per lane
  // over all C*M.
  {
    int rem_p = 0;
    for (int p = lane; p < C; p += 32) rem_p += M - X.nm[p * S + s];
    const int A = __reduce_add_sync(kFull, rem_p);
    if (A <= 32) {
      int p = 0, pre = 0, m0 = 0;
      bool act = lane < A;
      if (act) {  // the lane's pair: pipelines in order, pairs m0 .. M-1 of each
        for (;; ++p) {
          m0 = X.nm[p * S + s];
          if (lane < pre + M - m0) break;
          pre += M - m0;
        }
      }
      const int m = m0 + lane - pre;
      long long u = kNegMP;
      bool f = true;
      if (act) {
        const long long r = s == S - 1 ? X.fdl[p * M + m] : X.garr[((size_t)p * S + s) * M + m];
        u = r - (long long)m * dur;
        f = m == m0;
        if (f) u = imax(u, X.gf[p * S + s] - (long long)m0 * dur);
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {  // inclusive segmented max, upward
        const long long ou = shfl_up64(u, o);
        const bool of = __shfl_up_sync(kFull, (int)f, o) != 0;
        if (lane >= o) {
          if (!f) u = imax(u, ou);
          f = f || of;
        }
      }
      if (act) {
        const long long e = (long long)(m + 1) * dur + u;
        if (s > 0) X.garr[((size_t)p * S + s - 1) * M + m] = e;
        if (TIMELINE) X.ps[((size_t)p * S + s) * M + m] = e - dur;
        if (m == M - 1) X.gf[p * S + s] = e;
      }
      __syncwarp();
      for (int q = lane; q < C; q += 32) X.nm[q * S + s] = M;
      __syncwarp();
      return;
    }
  }
  long long carry = kNegMP;
  for (int base = 0; base < n; base += 32 * K) {
    const int rem = n - base < 32 * K ? n - base : 32 * K;
    const int kk = (rem + 31) / 32;
    long long u[K];
    bool rs[K], act[K];
    int rs_first = K;
    long long acc = kNegMP;
    // (p, m) of the lane's first pair, then stepped (no division per pair)
    const int idx0 = base + lane * kk;
    const int p0 = idx0 / M, mm0 = idx0 - p0 * M;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      u[i] = kNegMP;
      rs[i] = act[i] = false;
      const int idx = idx0 + i;
      if (i < kk && idx < base + rem) {
        int p = p0, m = mm0 + i;
        while (m >= M) {
          m -= M;
          ++p;
        }
        const int m0 = X.nm[p * S + s];
        if (m >= m0) {
          act[i] = true;
          const long long r = s == S - 1 ? X.fdl[p * M + m] : X.garr[((size_t)p * S + s) * M + m];
          long long v = r - (long long)m * dur;
          if (m == m0) {
            rs[i] = true;
            v = imax(v, X.gf[p * S + s] - (long long)m0 * dur);
          }
          u[i] = v;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {  // lane-local inclusive segmented max
      if (rs[i]) {
        acc = u[i];
        if (rs_first == K) rs_first = i;
      } else {
        acc = imax(acc, u[i]);
      }
      u[i] = acc;
    }
    // warp inclusive segmented scan of the lane aggregates
    bool f = rs_first < K;
    long long a = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long oa = shfl_up64(a, o);
      const bool of = __shfl_up_sync(kFull, (int)f, o) != 0;
      if (lane >= o) {
        if (!f) a = imax(a, oa);
        f = f || of;
      }
    }
    long long ex = shfl_up64(a, 1);
    bool exf = __shfl_up_sync(kFull, (int)f, 1) != 0;
    if (lane == 0) {
      ex = kNegMP;
      exf = false;
    }
    const long long pre = exf ? ex : imax(carry, ex);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (!act[i]) continue;
      int p = p0, m = mm0 + i;
      while (m >= M) {
        m -= M;
        ++p;
      }
      const long long uu = i >= rs_first ? u[i] : imax(pre, u[i]);
      const long long e = (long long)(m + 1) * dur + uu;
      if (s > 0) X.garr[((size_t)p * S + s - 1) * M + m] = e;
      if (TIMELINE) X.ps[((size_t)p * S + s) * M + m] = e - dur;
      if (m == M - 1) X.gf[p * S + s] = e;
    }
    const long long tot = f ? a : imax(carry, a);
    carry = shfl_idx64(tot, 31);
  }
  __syncwarp();
  for (int p = lane; p < C; p += 32) X.nm[p * S + s] = M;
  __syncwarp();
}

// A run of consecutive stages s_top..s_bot none of which has a WAN gradient
// link: every pair follows e[p][s][m] = max(in[p][s][m], e[p][s][m-1]) +
// dur, with in = the output of stage s+1 for the same pair (or the forward
// end at S-1), and the chain of each (p, s) starting from its gpu_free at
// its first pair not drained in the forward phase. That is a 2-D max-plus
// grid evaluated as one wavefront: lane l owns stages s_top - l*Bw - j
// (j < Bw) and handles pair k = (p, m) at step k + l, taking the output of
// the lane above from the previous step by shuffle; a pair drained in the
// forward phase passes nothing and its consumer reads the stored gradient.
// Runs longer than 32*B stages are split by the caller.
template <int B, bool TIMELINE>
__device__ void drain_run_wavefront(const Geom& g, AtlasMem& X, int s_top, int s_bot) {
  const int lane = threadIdx.x & 31;
  const int S = g.S, M = g.M, C = g.C;
  const long long dur = g.dur;
  const int R = s_top - s_bot + 1;
  const int Bw = (R + 31) / 32;  // <= B
  const int nl = (R + Bw - 1) / Bw;
  const int n = C * M;
  int sj[B], nmj[B];
  long long pe[B];
#pragma unroll
  for (int j = 0; j < B; ++j) {
    sj[j] = j < Bw && lane < nl ? s_top - lane * Bw - j : -1;
    if (sj[j] < s_bot) sj[j] = -1;
    nmj[j] = 0;
    pe[j] = 0;
  }
  long long xo = 0;  // this lane's output of the previous step
  bool fo = false;   // ... and whether its bottom stage computed it
  long long top = 0;  // inputs of the run's top stage, items [t & ~31, +32), lane i = item +i
  int wp = 0, wm = 0;
  for (int t = 0; t < n + nl - 1; ++t) {
    if ((t & 31) == 0 && t < n) {  // coalesced prefetch of the next 32 top inputs
      const int k = t + lane;
      if (k < n) {
        const int p = k / M, m = k - p * M;
        top = s_top == S - 1 ? X.fdl[p * M + m] : X.garr[((size_t)p * S + s_top) * M + m];
      }
    }
    long long x = shfl_up64(xo, 1);
    bool f = __shfl_up_sync(kFull, (int)fo, 1) != 0;
    const long long tv = shfl_idx64(top, t & 31);
    if (lane == 0) {
      x = tv;
      f = true;  // (a top stage always consumes the stored input)
    }
    const int k = t - lane;
    if (k > 0 && ++wm == M) {  // (wp, wm) = pair k, stepped with t
      wm = 0;
      ++wp;
    }
    if (lane < nl && k >= 0 && k < n) {
      const int p = wp, m = wm;
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int s = sj[j];
        if (s < 0) continue;
        if (m == 0) {
          nmj[j] = X.nm[p * S + s];
          pe[j] = X.gf[p * S + s];
        }
        if (m < nmj[j]) {  // drained in the forward phase
          f = false;
          continue;
        }
        const long long r = f ? x : (s == S - 1 ? X.fdl[p * M + m]
                                                : X.garr[((size_t)p * S + s) * M + m]);
        const long long e = imax(r, pe[j]) + dur;
        pe[j] = e;
        if (s == s_bot && s > 0) X.garr[((size_t)p * S + s - 1) * M + m] = e;
        if (TIMELINE) X.ps[((size_t)p * S + s) * M + m] = e - dur;
        if (m == M - 1) X.gf[p * S + s] = e;
        x = e;
        f = true;
      }
    }
    xo = x;
    fo = f;
  }
  __syncwarp();
  for (int i = lane; i < C * R; i += 32) X.nm[(i / R) * S + s_bot + i % R] = M;
  __syncwarp();
}

// A run s_bot..s_top of stages without a WAN gradient link in which every
// pipeline p entered the drain with the same drained count n0 at every
// stage of the run (e.g. no forced drains: mem_limit >= M, the deep config-2
// rows), evaluation rows only. The run is a rectangular max-plus grid with
// uniform cell weight dur: e[s][m] = max(e[s+1][m], e[s][m-1]) + dur,
// e[s_top+1][m] = in[m] (the stored input of the top stage), e[s][n0-1] =
// gf[s]. Every monotone path from an entry point to cell (s, m) has the same
// number of cells, so
//   e[s][m] = (m+1-s)*dur + max( max_{s <= s' <= s_top} gf[s'] + (s'-n0)*dur,
//                                max_{n0 <= j <= m} in[j] + (s_top-j)*dur ),
// exact in int64. Only what later stages and the row read is produced: the
// bottom stage's outputs (the gradients of stage s_bot-1) and each stage's
// last end (gpu_free, the makespan). O(C*(M + R)) instead of O(C*M*R).
// Returns false (nothing done) when some pipeline's counts differ across
// the run.
__device__ bool drain_run_closed(const Geom& g, AtlasMem& X, int s_top, int s_bot) {
  const int lane = threadIdx.x & 31;
  const int S = g.S, M = g.M, C = g.C;
  const long long dur = g.dur;
  const int R = s_top - s_bot + 1;
  bool bad = false;
  for (int i = lane; i < C * R; i += 32) {
    const int p = i / R, s = s_bot + i % R;
    bad |= X.nm[p * S + s] != X.nm[p * S + s_top];
  }
  if (__any_sync(kFull, bad)) return false;
  for (int p = 0; p < C; ++p) {
    const int n0 = X.nm[p * S + s_top];
    if (n0 >= M) continue;
    // the gpu_free term over the whole run (its value at the bottom stage)
    long long gs_all = kNegMP;
    for (int s = s_bot + lane; s <= s_top; s += 32)
      gs_all = imax(gs_all, X.gf[p * S + s] + (long long)(s - n0) * dur);
    gs_all = warp_max64(gs_all);
    // prefix max over the pairs of in[j] + (s_top - j) * dur: bottom outputs
    long long pm = kNegMP;
    for (int m0 = n0; m0 < M; m0 += 32) {
      const int m = m0 + lane;
      long long v = kNegMP;
      if (m < M) {
        const long long in = s_top == S - 1 ? X.fdl[p * M + m]
                                            : X.garr[((size_t)p * S + s_top) * M + m];
        v = in + (long long)(s_top - m) * dur;
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long ov = shfl_up64(v, o);
        if (lane >= o) v = imax(v, ov);
      }
      v = imax(v, pm);
      if (m < M && s_bot > 0)
        X.garr[((size_t)p * S + s_bot - 1) * M + m] =
            (long long)(m + 1 - s_bot) * dur + imax(gs_all, v);
      pm = shfl_idx64(v, 31);
    }
    // every stage's last end: suffix max of the gpu_free term, 32 stages at a
    // time from the top (each lane reads its stage before writing it)
    long long gs = kNegMP;
    for (int top = s_top; top >= s_bot; top -= 32) {
      const int s = top - lane;
      long long v = s >= s_bot ? X.gf[p * S + s] + (long long)(s - n0) * dur : kNegMP;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {  // max over lanes <= lane: stages >= s
        const long long ov = shfl_up64(v, o);
        if (lane >= o) v = imax(v, ov);
      }
      v = imax(v, gs);
      if (s >= s_bot) X.gf[p * S + s] = (long long)(M - s) * dur + imax(v, pm);
      gs = shfl_idx64(v, 31);
    }
    __syncwarp();
  }
  for (int i = lane; i < C * R; i += 32) X.nm[(i / R) * S + s_bot + i % R] = M;
  __syncwarp();
  return true;
}

// Stage s whose gradient link w crosses the WAN: per-stage greedy, lane q =
// pipeline q (C <= 32, host-checked).
template <bool TIMELINE>
__device__ void drain_stage_greedy(const Geom& g, AtlasMem& X, int s, int w) {
  const int q = threadIdx.x & 31;
  const int S = g.S, M = g.M, C = g.C;
  const long long dur = g.dur, len = g.ser_pooled[w], wl = g.ser_pooled[w] + g.lat[w];
  const long long* mg = X.mb + (size_t)w * C * M;
  const int* jg = X.jb + (size_t)w * C * M;
  const int nmg = X.mcnt[8 + w];
  int mq = q < C ? X.nm[q * S + s] : M;
  long long gfq = q < C ? X.gf[q * S + s] : 0;
  LinkCur cur;
  cur.reset(mg, nmg);
  long long last_a = kNegMP;  // start of this stage's last committed transfer
  // inputs of this stage are final (stage s+1 is drained): the next pair's
  // input is loaded one commit ahead
  auto input = [&](int m) -> long long {
    return s == S - 1 ? X.fdl[q * M + m] : X.garr[((size_t)q * S + s) * M + m];
  };
  long long rnext = q < C && mq < M ? input(mq) : 0;
  auto fresh = [&]() -> long long {
    const long long r = rnext;
    if (mq + 1 < M) rnext = input(mq + 1);
    return link_fit(mg, jg, nmg, cur, last_a, len, imax(r, gfq) + dur) - dur;
  };
  long long cand = mq < M ? fresh() : kInf64;
  int P2 = 1;  // argmin over the lowest power-of-two group holding the C lanes
  while (P2 < C) P2 <<= 1;
  for (;;) {
    long long b = cand;
    int bq = q;
    for (int o = P2 >> 1; o > 0; o >>= 1) {
      const long long ob = __shfl_xor_sync(kFull, b, o);
      const int oq = __shfl_xor_sync(kFull, bq, o);
      if (ob < b || (ob == b && oq < bq)) {
        b = ob;
        bq = oq;
      }
    }
    b = shfl_idx64(b, 0);
    bq = __shfl_sync(kFull, bq, 0);
    if (b == kInf64) break;
    if (q == bq) {  // atlas_commit_pair (:298-317) + reserve
      const long long e = b + dur;
      X.resb[((size_t)w * C + q) * M + mq] = e;
      X.garr[((size_t)q * S + s - 1) * M + mq] = e + wl;
      if (TIMELINE) X.ps[((size_t)q * S + s) * M + mq] = b;
      gfq = e;
      ++mq;
    }
    last_a = b + dur;
    if (q == bq) {
      cand = mq < M ? fresh() : kInf64;
    } else if (cand != kInf64 && cand + dur < last_a + len) {
      cand = link_fit(mg, jg, nmg, cur, last_a, len, cand + dur) - dur;  // pushed by the commit
    }
  }
  if (q < C) {
    X.gf[q * S + s] = gfq;
    X.nm[q * S + s] = M;
  }
  __syncwarp();
}

// The same per-stage greedy on one lane, for cells of at most CMAX pipelines:
// the C candidates, their cursors and gpu_free live in that lane's registers,
// so a commit is a register argmin plus one fit instead of a warp argmin of
// shuffles (measured ~4x fewer cycles per commit at C = 4).
template <bool TIMELINE, int CMAX>
__device__ void drain_stage_greedy_lane(const Geom& g, AtlasMem& X, int s, int w) {
  {  // the stage's inputs (final: stage s+1 is drained), staged by the warp
    const int S = g.S, M = g.M, C = g.C;
    for (int q = 0; q < C; ++q)
      for (int m = threadIdx.x & 31; m < M; m += 32)
        X.mtmp[q * M + m] = s == S - 1 ? X.fdl[q * M + m] : X.garr[((size_t)q * S + s) * M + m];
    __syncwarp();
  }
  if ((threadIdx.x & 31) == 0) {
    const int S = g.S, M = g.M, C = g.C;
    const long long* in = X.mtmp;  // [q][m]
    const long long dur = g.dur, len = g.ser_pooled[w], wl = g.ser_pooled[w] + g.lat[w];
    const long long* mg = X.mb + (size_t)w * C * M;
    const int* jg = X.jb + (size_t)w * C * M;
    const int nmg = X.mcnt[8 + w];
    int mq[CMAX];
    long long gfq[CMAX], cand[CMAX];
    LinkCur cur[CMAX];
    long long last_a = kNegMP;
    if (nmg == 0) {
      // No forced drains on this link (mem_limit >= M): it holds only this
      // stage's commits, in non-decreasing time, so earliest_fit of a
      // transfer at x is max(x, last + len) and every candidate's start is
      // max(raw_q, last + len - dur) with raw_q = max(input, gpu_free): the
      // greedy is an argmin of that over the pipelines' next pairs (lowest
      // pipeline on ties), no list walks.
      long long raw[CMAX];
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        mq[q] = q < C ? X.nm[q * S + s] : M;
        gfq[q] = q < C ? X.gf[q * S + s] : 0;
        raw[q] = mq[q] < M ? imax(in[q * M + mq[q]], gfq[q]) : kInf64;
      }
      long long floor_t = kNegMP;  // last + len - dur (len > 0)
      for (;;) {
        long long b = kInf64;
        int bq = -1;
#pragma unroll
        for (int q = 0; q < CMAX; ++q) {
          const long long st = imax(raw[q], floor_t);
          if (raw[q] != kInf64 && st < b) {
            b = st;
            bq = q;
          }
        }
        if (bq < 0) break;
        const long long e = b + dur;
        if (len > 0) floor_t = e + len - dur;
#pragma unroll
        for (int q = 0; q < CMAX; ++q) {
          if (q == bq) {  // atlas_commit_pair (:298-317) + reserve
            X.resb[((size_t)w * C + q) * M + mq[q]] = e;
            X.garr[((size_t)q * S + s - 1) * M + mq[q]] = e + wl;
            if (TIMELINE) X.ps[((size_t)q * S + s) * M + mq[q]] = b;
            gfq[q] = e;
            ++mq[q];
            raw[q] = mq[q] < M ? imax(in[q * M + mq[q]], e) : kInf64;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < CMAX; ++q)
        if (q < C) {
          X.gf[q * S + s] = gfq[q];
          X.nm[q * S + s] = M;
        }
    } else {
#pragma unroll
    for (int q = 0; q < CMAX; ++q) {
      cand[q] = kInf64;
      mq[q] = M;
      gfq[q] = 0;
      cur[q].reset(mg, nmg);
      if (q < C) {
        mq[q] = X.nm[q * S + s];
        gfq[q] = X.gf[q * S + s];
        if (mq[q] < M)
          cand[q] = link_fit(mg, jg, nmg, cur[q], last_a, len, imax(in[q * M + mq[q]], gfq[q]) + dur) -
                    dur;
      }
    }
    // Candidates are exact starts except that the last commit may have pushed
    // some (only the last commit can overlap a later query, see above): the
    // minimum is refitted if its transfer overlaps that commit, then the
    // minimum is taken again, so each commit refits only the candidates that
    // reach the front (lowest pipeline on ties, as the warp version).
    for (;;) {
      long long b = kInf64;
      int bq = -1;
#pragma unroll
      for (int q = 0; q < CMAX; ++q)
        if (cand[q] < b) {  // strict: the lowest pipeline on ties
          b = cand[q];
          bq = q;
        }
      if (bq < 0) break;
      if (b + dur < last_a + len) {  // pushed by the last commit: refit, retry
#pragma unroll
        for (int q = 0; q < CMAX; ++q)
          if (q == bq) cand[q] = link_fit(mg, jg, nmg, cur[q], last_a, len, b + dur) - dur;
        continue;
      }
      const long long e = b + dur;
      last_a = e;
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        if (q == bq) {  // atlas_commit_pair (:298-317) + reserve
          X.resb[((size_t)w * C + q) * M + mq[q]] = e;
          X.garr[((size_t)q * S + s - 1) * M + mq[q]] = e + wl;
          if (TIMELINE) X.ps[((size_t)q * S + s) * M + mq[q]] = b;
          gfq[q] = e;
          ++mq[q];
          cand[q] = kInf64;
          if (mq[q] < M)
            cand[q] = link_fit(mg, jg, nmg, cur[q], last_a, len, imax(in[q * M + mq[q]], e) + dur) -
                      dur;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < CMAX; ++q)
      if (q < C) {
        X.gf[q * S + s] = gfq[q];
        X.nm[q * S + s] = M;
      }
    }
  }
  __syncwarp();
}

template <bool TIMELINE>
__device__ __forceinline__ void drain_stage_wan(const Geom& g, AtlasMem& X, int s, int w) {
  if (g.C <= 4 && g.drain_lane && g.S >= g.drain_lane)
    drain_stage_greedy_lane<TIMELINE, 4>(g, X, s, w);
  else
    drain_stage_greedy<TIMELINE>(g, X, s, w);
}

constexpr int kWaveRatio = 8;

// PROF: per-row phase counters (gpb_set_profile; a separate instantiation,
// so the production kernel carries no clock reads or counters)
template <int B, bool TIMELINE, bool PROF>
__device__ long long atlas_row(const Geom& g, int mem_limit, AtlasMem& X, int& err,
                               long long* phase = nullptr) {
  const int lane = threadIdx.x & 31;
  long long ph_casc = 0, ph_chain = 0, ph_fit = 0, ph_drain = 0, ph_t = 0;
  long long n_stage_it = 0, n_pairs = 0, n_adm = 0, n_rounds = 0;
  long long cph[4] = {0, 0, 0, 0};  // cascade: setup, loads, scan rounds, commits
  const int S = g.S, M = g.M, C = g.C;
  const long long f = g.fwd, dur = g.dur;
  const int nw = g.nb - 1;
  X.garr = (long long)C * S * M <= X.garr_cap ? X.garr_smem : X.garr_glob;
  for (int i = lane; i < C * S; i += 32) {
    X.gf[i] = 0;
    X.nm[i] = 0;
  }
  for (int s = lane; s < S; s += 32) {
    int w;
    X.wbs[s] = (s > 0 && wan_after(g, s - 1, w)) ? w : -1;
  }
  if (lane < nw) {  // pooled serialization / latency per WAN boundary
    X.wa[8 + lane] = g.ser_pooled[lane];
    X.wg[8 + lane] = g.lat[lane];
  }
  __syncwarp();

  // Per-lane stage info and chain offsets a_s (lane prefix + warp scan).
  const int nl = (S + B - 1) / B;  // lanes owning stages
  int wbi[B], wfi[B];  // WAN boundary before / after the stage, or -1
  long long serb[B], latb[B], a_loc[B];
  long long run = 0;
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const int s = lane * B + j;
    wbi[j] = wfi[j] = -1;
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
      if (s + 1 < S && wan_after(g, s, w)) {
        run += g.ser_pooled[w] + g.lat[w];
        wfi[j] = w;
      }
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
  // chain offsets of the stages before each WAN boundary (lane w reads a_w)
#pragma unroll
  for (int j = 0; j < B; ++j)
    if (wfi[j] >= 0) X.wa[wfi[j]] = a_loc[j];
  const int wsrc = lane < nw ? g.blk_first[lane + 1] - 1 : lane;  // B == 1: that stage's lane
  __syncwarp();
  // wsuf[j]: sum over stages i >= s of (pair duration + WAN delay of the
  // gradient link of i) — the cascade's single-chain suffix sums
  long long wsuf[B];
  {
    long long loc = 0;
#pragma unroll
    for (int j = B - 1; j >= 0; --j) {
      const int s = lane * B + j;
      if (s < S) loc += dur + (wbi[j] >= 0 ? serb[j] + latb[j] : 0);
      wsuf[j] = loc;
    }
    long long incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = shfl_down64(incl, o);
      if (lane + o < 32) incl += v;
    }
    const long long excl = incl - loc;
#pragma unroll
    for (int j = 0; j < B; ++j) wsuf[j] += excl;
  }

  // ------------------------------------------------------ forward phase
  // Per-lane registers for the current pipeline p: gpu_free and drained
  // counts of the owned stages (written back to shared memory per p).
  long long gfr[B];
  int drr[B];
  if (lane < 8) X.mcnt[lane] = X.mcnt[8 + lane] = 0;
  __syncwarp();
  LinkCur curf;  // lane w: cursor of the static forward list of link w
  for (int p = 0; p < C; ++p) {
#pragma unroll
    for (int j = 0; j < B; ++j) {
      gfr[j] = 0;
      drr[j] = 0;
    }
    if (p > 0) {  // fold pipeline p-1 into the static lists of every link
      for (int w = 0; w < nw; ++w) {
        const int sw = g.blk_first[w + 1];  // stage whose gradient link is w
        const int nf = X.mcnt[w], nbk = X.mcnt[8 + w];
        const int add_b = X.nm[(p - 1) * S + sw];
        warp_merge(X.mf + (size_t)w * C * M, nf, X.resf + ((size_t)w * C + p - 1) * M, M, X.mtmp);
        warp_merge(X.mb + (size_t)w * C * M, nbk, X.resb + ((size_t)w * C + p - 1) * M, add_b,
                   X.mtmp);
        warp_jumps(X.mf + (size_t)w * C * M, nf + M, g.ser_pooled[w], X.jf + (size_t)w * C * M);
        warp_jumps(X.mb + (size_t)w * C * M, nbk + add_b, g.ser_pooled[w],
                   X.jb + (size_t)w * C * M);
        if (lane == 0) {
          X.mcnt[w] = nf + M;
          X.mcnt[8 + w] = nbk + add_b;
        }
        __syncwarp();
      }
    }
    __syncwarp();
    StaticLinks<B> links(X, C, M, wbi, serb);
    // lane w < nw: link w's constants for this pipeline (chain checks)
    long long aw_l = 0, lenw_l = 0, ownw_l = kNegMP;
    const long long* mgw_l = nullptr;
    const int* jgw_l = nullptr;
    int nmw_l = 0;
    if (lane < nw) {
      aw_l = X.wa[lane];
      lenw_l = X.wa[8 + lane];
      mgw_l = X.mf + (size_t)lane * C * M;
      jgw_l = X.jf + (size_t)lane * C * M;
      nmw_l = X.mcnt[lane];
      curf.reset(mgw_l, nmw_l);
    }
    for (int m = 0; m < M; ++m) {
      // memory-cap admission (:366-381) + forced drains (:321-346)
      if (PROF) ph_t = clock64();
      // some stage blocked <=> stage 0 (the least drained) is
      if (m - __shfl_sync(kFull, drr[0], 0) >= mem_limit) {
        atlas_cascade<B, TIMELINE, PROF>(g, p, m, mem_limit, X, gfr, drr, wbi, serb, latb, links,
                                         wsuf, n_pairs, n_stage_it, n_rounds, cph);
        if (PROF) ++n_adm;
      }
      if (PROF) {
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
        if (o >= nl) break;  // warp-uniform
        const long long v = shfl_up64(pre, o);
        if (lane >= o) pre = imax(pre, v);
      }
      long long prev = shfl_up64(pre, 1);
      if (lane == 0) prev = -kInf64;
      long long gw = 0;  // lane w: G of the stage before WAN boundary w
#pragma unroll
      for (int j = 0; j < B; ++j) gl[j] = imax(gl[j], prev);
      if (B == 1) {  // that stage is lane wsrc's only stage
        gw = shfl_idx64(gl[0], wsrc);
      } else {
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (wfi[j] >= 0) X.wg[wfi[j]] = gl[j];
        __syncwarp();
        if (lane < nw) gw = X.wg[lane];
      }
      long long t0 = __shfl_sync(kFull, gfr[0], 0);  // gpu_free of stage 0
      if (PROF) {
        const long long t1 = clock64();
        ph_chain += t1 - ph_t;
        ph_t = t1;
      }
      // exact-fit shift loop over the WAN boundaries (:383-405), one lane per
      // pipeline list of each link, then the chain's reservations (:407-430)
      // (lane w checks link w; the lowest conflicting link shifts t0, as the
      // reference's restart from stage 0 does)
      if (nw > 0) {
        for (;;) {
          const long long e = aw_l + f + imax(t0, gw);
          const bool conf = lane < nw && link_conflict(mgw_l, nmw_l, curf, ownw_l, lenw_l, e);
          const unsigned bal = __ballot_sync(kFull, conf);
          if (!bal) break;
          const int src = __ffs(bal) - 1;
          long long shift = 0;
          if (lane == src) shift = link_fit(mgw_l, jgw_l, nmw_l, curf, ownw_l, lenw_l, e) - e;
          t0 += shfl_idx64(shift, src);
        }
        if (lane < nw) {
          ownw_l = aw_l + f + imax(t0, gw);
          X.resf[((size_t)lane * C + p) * M + m] = ownw_l;
        }
      }
      if (PROF) {
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

  if (PROF) ph_t = clock64();
  // ------------------------------------------ drain: stage by stage
  // Pairs drained by the forward phase are excluded from the right-pack.
  for (int i = lane; i < C * S; i += 32) X.firstm[i] = X.nm[i];
  // the last pipeline's forced drains join the static gradient lists
  for (int w = 0; w < nw; ++w) {
    const int sw = g.blk_first[w + 1];
    const int nbk = X.mcnt[8 + w], add_b = X.nm[(C - 1) * S + sw];
    warp_merge(X.mb + (size_t)w * C * M, nbk, X.resb + ((size_t)w * C + C - 1) * M, add_b,
               X.mtmp);
    warp_jumps(X.mb + (size_t)w * C * M, nbk + add_b, g.ser_pooled[w], X.jb + (size_t)w * C * M);
    if (lane == 0) X.mcnt[8 + w] = nbk + add_b;
    __syncwarp();
  }
  long long dph[4] = {0, 0, 0, 0};  // drain: greedy / scan / wavefront cycles, wave steps
  for (int s = S - 1; s >= 0;) {
    const long long td = PROF ? clock64() : 0;
    const int w = X.wbs[s];
    if (w >= 0) {
      drain_stage_wan<TIMELINE>(g, X, s, w);
      --s;
      if (PROF) dph[0] += clock64() - td;
      continue;
    }
    int sb = s;  // the run of stages without a WAN gradient link below s
    while (sb > 0 && X.wbs[sb - 1] < 0) --sb;
    // per-stage scans cost ~R * ceil(CM / 256) scan steps, the wavefront
    // CM + R/B shuffle steps (kWaveRatio: measured cost ratio of the two)
    const int R = s - sb + 1, CM = C * g.M;
    if (!TIMELINE && drain_run_closed(g, X, s, sb)) {
      s = sb - 1;
      if (PROF) dph[2] += clock64() - td;
      continue;
    }
    if ((long long)(CM + (R + B - 1) / B) > (long long)kWaveRatio * R * ((CM + 255) / 256)) {
      for (; s >= sb; --s) drain_stage_scan<TIMELINE>(g, X, s);
      if (PROF) dph[1] += clock64() - td;
      continue;
    }
    constexpr int BW = B < 4 ? B : 4;  // stages per lane (register arrays)
    for (int st = s; st >= sb; st -= 32 * BW) {
      const int bot = max(sb, st - 32 * BW + 1), rr = st - bot + 1;
      drain_run_wavefront<BW, TIMELINE>(g, X, st, bot);
      if (PROF) dph[3] += CM + (rr + BW - 1) / BW;
    }
    s = sb - 1;
    if (PROF) dph[2] += clock64() - td;
  }
  if (PROF && lane == 0) {
    ph_drain = clock64() - ph_t;
    phase[0] = ph_casc;
    phase[1] = ph_chain;
    phase[2] = ph_fit;
    phase[3] = ph_drain;
    phase[4] = n_stage_it;
    phase[5] = n_pairs;
    phase[6] = n_adm;
    phase[7] = n_rounds;
    for (int k = 0; k < 4; ++k) phase[8 + k] = cph[k];
    for (int k = 0; k < 4; ++k) phase[12 + k] = dph[k];
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

// ------------------------------------------------------ wave (heavy rows)
//
// The forward phase of the reference runs pipeline 0's M microbatches, then
// pipeline 1's, ... (scheduler.cpp:362-431). Pipeline p reads the shared
// links only through free_at / earliest_fit over the reservations of the
// pipelines before it, and never affects them. So the pipelines can run
// concurrently — one warp each, the whole CTA one row — provided pipeline p
// waits, before it answers a query over the window [t, t + len) on a link,
// until every earlier pipeline q has either finished its forward phase or
// made a reservation on that link starting at or after t: q's reservations
// on a link are appended in increasing time and all have length len, so
// every later one then starts at or after t + len and cannot touch the
// window. The answers are exactly those of the sequential order; the wait
// chain only points to lower pipelines, so it cannot deadlock. The drain
// (global greedy + per-stage decomposition) starts once every pipeline is
// done, on warp 0, over the merged gradient lists. Used for the heavy ATLAS
// rows (the critical path of a small space such as config 2: S=16, C=4,
// M=64 went from one warp walking the 4 pipelines in turn to 4 warps).
constexpr int kWaveMaxC = 8;

struct WaveState {  // per CTA (one row), in shared memory
  int cnt_f[GPB_MAX_DC - 1][kWaveMaxC];  // reservations per (link, pipeline)
  int cnt_b[GPB_MAX_DC - 1][kWaveMaxC];
  int done[kWaveMaxC];
  int row;
  unsigned long long wait_cyc[kWaveMaxC];  // profiling: cycles pipeline p spent waiting
};

__device__ __forceinline__ int vload(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ long long vload(const long long* p) {
  return *(const volatile long long*)p;
}

// One lane's view of one link's lists of the pipelines before it, with the
// cursor position and entry, the list length and the time below which the
// list is known final held in registers (the common query reads no memory,
// as atlas_kernel's static cursor does). NQ >= the number of earlier
// pipelines (the wave kernel takes C <= kWaveRegC).
constexpr int kWaveRegC = 4;
template <int NQ>
struct WaveView {
  const long long* base;  // list q at base + q * M
  const int* cnt;         // published lengths
  const int* done;        // per pipeline: forward phase finished
  int M, p;
  int n[NQ], idx[NQ];
  long long val[NQ], fin[NQ];
  __device__ __forceinline__ void init(const long long* b, const int* c, const int* d, int M_,
                                       int p_) {
    base = b;
    cnt = c;
    done = d;
    M = M_;
    p = p_;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      n[q] = idx[q] = 0;
      val[q] = kEndCur;
      fin[q] = kNegMP;
    }
  }
  // list q final below t (q done, or its last reservation starts at or
  // after t: every later one starts at or after t + len)
  __device__ __forceinline__ void ensure(int q, long long t, unsigned long long* wait) {
    if (t <= fin[q]) return;
    long long t0 = 0;
    for (int spin = 0;; ++spin) {
      const int nn = vload(&cnt[q]);
      const long long last = nn > 0 ? vload(&base[(size_t)q * M + nn - 1]) : kNegMP;
      const bool d = vload(&done[q]) != 0;
      const int nf = d ? vload(&cnt[q]) : nn;
      if (last >= t || d) {
        n[q] = nf;
        fin[q] = d ? kEndCur : last;
        if (val[q] == kEndCur && idx[q] < nf) val[q] = vload(&base[(size_t)q * M + idx[q]]);
        if (spin > 0) atomicAdd(wait, (unsigned long long)(clock64() - t0));
        return;
      }
      if (spin == 0) t0 = clock64();
      __nanosleep(20);
    }
  }
  __device__ __forceinline__ void advance(int q, long long len, long long t) {
    while (val[q] + len <= t) {
      ++idx[q];
      val[q] = idx[q] < n[q] ? vload(&base[(size_t)q * M + idx[q]]) : kEndCur;
    }
  }
  // free_at(x, x + len) fails (moves cursors only past entries ending <= x)
  __device__ __forceinline__ bool conflict(long long own, long long len, long long x,
                                           unsigned long long* wait) {
    if (len <= 0) return false;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (q >= p) break;
      ensure(q, x, wait);
      advance(q, len, x);
      if (val[q] < x + len) return true;
    }
    return own + len > x;
  }
  // earliest_fit(x, len) over the union and the own tail
  __device__ __forceinline__ long long fit(long long own, long long len, long long x,
                                           unsigned long long* wait) {
    if (len <= 0) return x;
    long long t = x;
    for (;;) {
      bool moved = false;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (q >= p) break;
        ensure(q, t, wait);
        advance(q, len, t);
        while (val[q] < t + len) {
          t = val[q] + len;
          moved = true;
          ensure(q, t, wait);
          advance(q, len, t);
        }
      }
      if (own + len > t) {
        t = own + len;
        moved = true;
      }
      if (!moved) return t;
    }
  }
};

// gradient-link policy of the cascade (B = 1: the lane's one stage)
struct WaveLinks {
  AtlasMem& X;
  WaveState& W;
  WaveView<kWaveRegC - 1> v;
  int C, M, w;
  long long len, own;
  __device__ __forceinline__ long long fit(int, long long y) {
    return v.fit(own, len, y, &W.wait_cyc[v.p]);
  }
  __device__ __forceinline__ bool conflict(int, long long y) {
    return v.conflict(own, len, y, &W.wait_cyc[v.p]);
  }
  __device__ __forceinline__ void reserve(int, int pp, int k, long long e) {
    X.resb[((size_t)w * C + pp) * M + k] = e;
    own = e;
    __threadfence_block();
    *(volatile int*)&W.cnt_b[w][pp] = k + 1;
  }
};

// One pipeline's forward phase (the loop of atlas_row with wave queries).
__device__ void atlas_wave_forward(const Geom& g, int mem_limit, AtlasMem& X, WaveState& W, int p,
                                   const int (&wbi)[1], const int (&wfi)[1],
                                   const long long (&serb)[1], const long long (&latb)[1],
                                   const long long (&a_loc)[1], const long long (&wsuf)[1],
                                   int wsrc) {
  const int lane = threadIdx.x & 31;
  const int S = g.S, M = g.M, C = g.C;
  const long long f = g.fwd;
  const int nw = g.nb - 1;
  const int nl = S;  // B = 1
  long long gfr[1] = {0};
  int drr[1] = {0};
  long long n0 = 0, n1 = 0, n2 = 0;
  const int wb = wbi[0] >= 0 ? wbi[0] : 0;
  WaveLinks links{X, W, {}, C, M, wb, wbi[0] >= 0 ? serb[0] : 0, kNegMP};
  links.v.init(X.resb + (size_t)wb * C * M, W.cnt_b[wb], W.done, M, p);
  const int wf = lane < nw ? lane : 0;  // lane w < nw: forward link w
  WaveView<kWaveRegC - 1> fv;
  fv.init(X.resf + (size_t)wf * C * M, W.cnt_f[wf], W.done, M, p);
  long long aw_l = 0, lenw_l = 0, ownw_l = kNegMP;
  if (lane < nw) {
    aw_l = X.wa[lane];
    lenw_l = X.wa[8 + lane];
  }
  __syncwarp();
  for (int m = 0; m < M; ++m) {
    if (m - __shfl_sync(kFull, drr[0], 0) >= mem_limit)  // stage 0 is the least drained
      atlas_cascade<1, false, false>(g, p, m, mem_limit, X, gfr, drr, wbi, serb, latb, links,
                                     wsuf, n0, n1, n2, nullptr);
    long long gl = lane < S ? gfr[0] - a_loc[0] : -kInf64;
    for (int o = 1; o < nl; o <<= 1) {
      const long long v = shfl_up64(gl, o);
      if (lane >= o) gl = imax(gl, v);
    }
    const long long gw = shfl_idx64(gl, wsrc);
    long long t0 = __shfl_sync(kFull, gfr[0], 0);
    if (nw > 0) {
      for (;;) {
        const long long e = aw_l + f + imax(t0, gw);
        const bool conf = lane < nw && fv.conflict(ownw_l, lenw_l, e, &W.wait_cyc[p]);
        const unsigned bal = __ballot_sync(kFull, conf);
        if (!bal) break;
        const int src = __ffs(bal) - 1;  // the lowest conflicting link shifts t0
        long long shift = 0;
        if (lane == src) shift = fv.fit(ownw_l, lenw_l, e, &W.wait_cyc[p]) - e;
        t0 += shfl_idx64(shift, src);
      }
      if (lane < nw) {
        ownw_l = aw_l + f + imax(t0, gw);
        X.resf[((size_t)lane * C + p) * M + m] = ownw_l;
        __threadfence_block();
        *(volatile int*)&W.cnt_f[lane][p] = m + 1;
      }
    }
    if (lane < S) {
      const long long e = a_loc[0] + f + imax(t0, gl);
      gfr[0] = e;
      if (lane == S - 1) X.fdl[p * M + m] = e;
    }
    __syncwarp();
  }
  if (lane < S) {
    X.gf[p * S + lane] = gfr[0];
    X.nm[p * S + lane] = drr[0];
  }
  __threadfence_block();
  __syncwarp();
  if (lane == 0) *(volatile int*)&W.done[p] = 1;
}

// Drain phase of a row after the forward phases (warp 0): the gradient lists
// of all pipelines merged per link, then the per-stage decomposition.
template <int B, bool TIMELINE>
__device__ long long atlas_drain_all(const Geom& g, AtlasMem& X, const WaveState* W) {
  const int lane = threadIdx.x & 31;
  const int S = g.S, M = g.M, C = g.C;
  const int nw = g.nb - 1;
  for (int i = lane; i < C * S; i += 32) X.firstm[i] = X.nm[i];
  for (int w = 0; w < nw; ++w) {
    int nbk = 0;
    for (int q = 0; q < C; ++q) {
      const int add_b = W ? W->cnt_b[w][q] : 0;
      warp_merge(X.mb + (size_t)w * C * M, nbk, X.resb + ((size_t)w * C + q) * M, add_b, X.mtmp);
      nbk += add_b;
    }
    warp_jumps(X.mb + (size_t)w * C * M, nbk, g.ser_pooled[w], X.jb + (size_t)w * C * M);
    if (lane == 0) X.mcnt[8 + w] = nbk;
    __syncwarp();
  }
  for (int s = S - 1; s >= 0;) {
    const int w = X.wbs[s];
    if (w >= 0) {
      drain_stage_wan<TIMELINE>(g, X, s, w);
      --s;
      continue;
    }
    int sb = s;
    while (sb > 0 && X.wbs[sb - 1] < 0) --sb;
    const int R = s - sb + 1, CM = C * g.M;
    if (!TIMELINE && drain_run_closed(g, X, s, sb)) {
      s = sb - 1;
      continue;
    }
    if ((long long)(CM + (R + B - 1) / B) > (long long)kWaveRatio * R * ((CM + 255) / 256)) {
      for (; s >= sb; --s) drain_stage_scan<TIMELINE>(g, X, s);
      continue;
    }
    constexpr int BW = B < 4 ? B : 4;
    for (int st = s; st >= sb; st -= 32 * BW) {
      const int bot = max(sb, st - 32 * BW + 1);
      drain_run_wavefront<BW, TIMELINE>(g, X, st, bot);
    }
    s = sb - 1;
  }
  long long mk = 0;
  for (int i = lane; i < C * S; i += 32) mk = imax(mk, X.gf[i]);
  return warp_max64(mk);
}

// One CTA per heavy row (S <= 32, 2 <= C <= 8), warp p = pipeline p.
__global__ void __launch_bounds__(32 * kWaveMaxC, 1) atlas_wave_kernel(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WaveState& W = *reinterpret_cast<WaveState*>(smem);
  AtlasMem X;
  long long* scr = a.scratch ? a.scratch + (size_t)blockIdx.x * a.scratch_per_warp : nullptr;
  X.carve(smem + AtlasLayout::al(sizeof(WaveState)), a.lay, scr,
          scr ? (unsigned char*)(scr + a.scratch_big_off) : nullptr);
  for (;;) {
    if (threadIdx.x == 0) W.row = atomicAdd(a.cursor, 1);
    __syncthreads();
    const int wk = W.row;
    if (wk >= a.n_work) break;
    const int row = a.work[wk];
    const long long t_start = clock64();
    Geom g;
    const DevScen* sc;
    const DevTopo* tp;
    const bool ok = begin_row(a, row, g, sc, tp);  // warp 0's lane 0 writes infeasible rows
    if (!ok) {
      __syncthreads();
      continue;
    }
    const int S = g.S, C = g.C;
    const int nw = g.nb - 1;
    X.garr = (long long)C * S * g.M <= X.garr_cap ? X.garr_smem : X.garr_glob;
    if (warp == 0) {
      for (int i = lane; i < C * S; i += 32) {
        X.gf[i] = 0;
        X.nm[i] = 0;
      }
      for (int s = lane; s < S; s += 32) {
        int w;
        X.wbs[s] = (s > 0 && wan_after(g, s - 1, w)) ? w : -1;
      }
      if (lane < nw) {
        X.wa[8 + lane] = g.ser_pooled[lane];
        X.wg[8 + lane] = g.lat[lane];
      }
      for (int i = lane; i < (GPB_MAX_DC - 1) * kWaveMaxC; i += 32) {
        (&W.cnt_f[0][0])[i] = 0;
        (&W.cnt_b[0][0])[i] = 0;
      }
      if (lane < kWaveMaxC) {
        W.done[lane] = 0;
        W.wait_cyc[lane] = 0;
      }
    }
    // every warp: its lane's stage (B = 1) constants
    int wbi[1] = {-1}, wfi[1] = {-1};
    long long serb[1] = {0}, latb[1] = {0}, a_loc[1] = {0}, wsuf[1] = {0};
    {
      const int s = lane;
      long long run = 0, suf = 0;
      if (s < S) {
        int w;
        if (s > 0 && wan_after(g, s - 1, w)) {
          wbi[0] = w;
          serb[0] = g.ser_pooled[w];
          latb[0] = g.lat[w];
        }
        run = g.fwd;
        if (s + 1 < S && wan_after(g, s, w)) {
          run += g.ser_pooled[w] + g.lat[w];
          wfi[0] = w;
        }
        suf = g.dur + (wbi[0] >= 0 ? serb[0] + latb[0] : 0);
      }
      long long incl = run;
      for (int o = 1; o < 32; o <<= 1) {
        const long long v = shfl_up64(incl, o);
        if (lane >= o) incl += v;
      }
      a_loc[0] = incl - run;
      long long sincl = suf;
      for (int o = 1; o < 32; o <<= 1) {
        const long long v = shfl_down64(sincl, o);
        if (lane + o < 32) sincl += v;
      }
      wsuf[0] = sincl;
    }
    if (warp == 0 && wfi[0] >= 0) X.wa[wfi[0]] = a_loc[0];
    const int wsrc = lane < nw ? g.blk_first[lane + 1] - 1 : lane;
    __syncthreads();
    const long long t_fwd = clock64();
    if (warp < C)
      atlas_wave_forward(g, sc->mem_limit, X, W, warp, wbi, wfi, serb, latb, a_loc, wsuf, wsrc);
    const long long t_fwd_end = clock64();
    __syncthreads();
    if (warp == 0) {
      const long long t_drain = clock64();
      const long long mk = atlas_drain_all<1, false>(g, X, &W);
      int err = 0;
      end_row(a, row, g, *sc, *tp, mk, err, t_start);
      if (a.row_phase && lane == 0) {  // profiling: forward / drain / per-pipeline waits
        long long* ph = a.row_phase + 16 * (size_t)row;
        ph[0] = t_drain - t_fwd;
        ph[3] = clock64() - t_drain;
        for (int q = 0; q < kWaveMaxC; ++q) ph[8 + q] = (long long)W.wait_cyc[q];
      }
    }
    if (a.row_phase && lane == 0 && warp < C && warp < 4)
      a.row_phase[16 * (size_t)row + 4 + warp] = t_fwd_end - t_fwd;
    __syncthreads();
  }
}

int atlas_wave_smem(const AtlasLayout& L) { return (int)(AtlasLayout::al(sizeof(WaveState)) + L.total); }

int atlas_wave_blocks_per_sm(int warps, int smem) {
  cudaFuncSetAttribute(atlas_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int n = 0;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, atlas_wave_kernel, 32 * warps, smem) ==
                 cudaSuccess
             ? n
             : 1;
}

cudaError_t launch_atlas_wave(const EvalArgs& a, int grid, int warps, cudaStream_t st) {
  const int smem = atlas_wave_smem(a.lay);
  static int set_to = 0;
  if (smem > set_to) {
    const cudaError_t e = cudaFuncSetAttribute(
        atlas_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    set_to = smem;
  }
  atlas_wave_kernel<<<grid, 32 * warps, smem, st>>>(a);
  return cudaGetLastError();
}

// Blocks per SM the register allocation must allow: 3 for one stage per lane
// (162 registers, no spills: more resident warps when the space saturates
// the GPU), 1 for deeper pipelines (their larger per-lane state would spill).
#ifndef GPB_ATLAS_MIN_BLOCKS_B1
#define GPB_ATLAS_MIN_BLOCKS_B1 3
#endif

// OCC4 (one stage per lane, large spaces): 4 resident blocks per SM (128
// registers, no spills): more rows in flight where throughput sets the step
// (config 5: 207 -> 193 ms), while the latency-bound small spaces keep 3
// (their critical rows ran ~15 % slower at 4: 805 K -> 935 K cycles).
template <int B, bool PROF, bool OCC4 = false>
__global__ void __launch_bounds__(kEvalThreads, B == 1 ? (OCC4 ? 4 : GPB_ATLAS_MIN_BLOCKS_B1) : 1)
    atlas_kernel(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + warp;
  AtlasMem X;
  long long* scr = a.scratch ? a.scratch + (size_t)gwarp * a.scratch_per_warp : nullptr;
  X.carve(smem + (size_t)warp * a.lay.total, a.lay, scr,
          scr ? (unsigned char*)(scr + a.scratch_big_off) : nullptr);
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
    const long long mk =
        atlas_row<B, false, PROF>(g, sc->mem_limit, X, err,
                                  PROF ? a.row_phase + 16 * (size_t)row : nullptr);
    end_row(a, row, g, *sc, *tp, mk, err, t_start);
    __syncwarp();
  }
}

template <int B>
__global__ void __launch_bounds__(kEvalThreads, 1) atlas_timeline_kernel(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + warp;
  AtlasMem X;
  long long* scr = a.scratch ? a.scratch + (size_t)gwarp * a.scratch_per_warp : nullptr;
  X.carve(smem + (size_t)warp * a.lay.total, a.lay, scr,
          scr ? (unsigned char*)(scr + a.scratch_big_off) : nullptr);
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
    const long long mk = atlas_row<B, true, false>(g, sc->mem_limit, X, err);
    end_row(a, row, g, *sc, *tp, mk, err, t_start);
    __syncwarp();
  }
}

// Raise a kernel's dynamic shared memory limit only when a launch needs more
// than it was set to (per device; the attribute call costs host time on every
// evaluate otherwise).
template <int B, bool TL>
static cudaError_t ensure_smem_attr(size_t smem) {
  static std::mutex mu;
  static int done[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && done[dev] >= (int)smem) return cudaSuccess;
  cudaError_t e =
      TL ? cudaFuncSetAttribute(atlas_timeline_kernel<B>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
         : cudaFuncSetAttribute(atlas_kernel<B, false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && !TL)  // the profiling instantiation (gpb_set_profile)
    e = cudaFuncSetAttribute(atlas_kernel<B, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
  if constexpr (B == 1) {  // the 4-blocks-per-SM instantiations
    if (e == cudaSuccess && !TL)
      e = cudaFuncSetAttribute(atlas_kernel<1, false, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && !TL)
      e = cudaFuncSetAttribute(atlas_kernel<1, true, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  if (e == cudaSuccess && dev < 64) done[dev] = (int)smem;
  return e;
}

template <int B>
static cudaError_t launch_atlas_tl_b(const EvalArgs& a, int grid, int wpc, cudaStream_t st) {
  const size_t smem = (size_t)wpc * a.lay.total;
  cudaError_t e = ensure_smem_attr<B, true>(smem);
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
  const size_t smem = std::max((size_t)wpc * a.lay.total, (size_t)a.smem_floor);
  cudaError_t e = ensure_smem_attr<B, false>(smem);
  if (e != cudaSuccess) return e;
  if constexpr (B == 1) {
    if (a.occ4) {
      if (a.row_phase)
        atlas_kernel<1, true, true><<<grid, 32 * wpc, smem, st>>>(a);
      else
        atlas_kernel<1, false, true><<<grid, 32 * wpc, smem, st>>>(a);
      return cudaGetLastError();
    }
  }
  if (a.row_phase)
    atlas_kernel<B, true><<<grid, 32 * wpc, smem, st>>>(a);
  else
    atlas_kernel<B, false><<<grid, 32 * wpc, smem, st>>>(a);
  return cudaGetLastError();
}

// Resident blocks per SM of the ATLAS kernel (registers + shared memory).
int atlas_blocks_per_sm(int B, bool timeline, int wpc, size_t smem, bool occ4) {
  int n = 0;
  cudaError_t e = cudaSuccess;
  if (B == 1 && !timeline && occ4) {
    e = ensure_smem_attr<1, false>(smem);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, atlas_kernel<1, false, true>, 32 * wpc,
                                                        smem);
    return e == cudaSuccess ? n : 0;
  }
#define GPB_OCC(BB)                                                                         \
  case BB:                                                                                  \
    e = timeline ? ensure_smem_attr<BB, true>(smem) : ensure_smem_attr<BB, false>(smem);      \
    if (e == cudaSuccess)                                                                   \
      e = timeline ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, atlas_timeline_kernel<BB>, \
                                                                   32 * wpc, smem)          \
                   : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, atlas_kernel<BB, false>, \
                                                                   32 * wpc, smem);         \
    break;
  switch (B) {
    GPB_OCC(1) GPB_OCC(2) GPB_OCC(3) GPB_OCC(4) GPB_OCC(5) GPB_OCC(6) GPB_OCC(7) GPB_OCC(8)
  }
#undef GPB_OCC
  return e == cudaSuccess ? n : 0;
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
