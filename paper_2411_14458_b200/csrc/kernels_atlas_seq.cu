// kernels_atlas_seq.cu — ATLAS (scheduler.cpp:276-538) one THREAD per plan
// row, for the throughput-bound bulk of large plan spaces.
//
// atlas_kernel (kernels_atlas.cu) spreads one row over a warp (lane = stage)
// so that a single long row finishes fast: right for the critical path of a
// small space (config 2). A saturated space (configs 3 / 5) is mostly rows
// of shallow pipelines (S <= 16), where the warp formulation leaves most
// lanes idle and pays warp-wide scans per microbatch. Here every lane runs
// its own row with the reference's sequential recurrences, so 32 rows share
// one instruction stream.
//
// The state of a row lives in a per-thread slice of global scratch laid out
// [element][lane] per warp (lanes at the same step touch one 256-byte line):
//   GF[C][S]   gpu_free        DR[C][S]  drained counts
//   FDL[C][M]  last-stage forward ends (written once per forward)
//   GA[C][S][M] gradient arrivals at stage s (pair m's arrival exists once
//              stage s+1 has drained pair m: DR[p][s+1] > m)
//   per WAN link w: MF / MB merged static forward / gradient reservation
//   starts of the pipelines before the current one (C*M each), OF / OB the
//   current pipeline's own starts (M each).
// Reservation lists (base.h:63-124) hold intervals of one uniform length per
// link (the pooled serialization time). While pipeline p runs its forward
// phase, pipelines q < p are frozen and q > p have none on any link, so a
// link is the static merged list plus p's own append-only list; p's queries
// on a link come in non-decreasing time and start after p's own last
// reservation, so only the own tail can overlap and a forward-only cursor
// over the static list answers free_at / earliest_fit exactly (the same
// argument as atlas_kernel). The drain runs stage by stage
// (the global greedy of :461-505 equals per-stage greedies):
// a stage without a WAN gradient link is the max-plus chain per pipeline, a
// WAN stage the greedy over its C pipelines' next pairs (lowest pipeline on
// ties) against the forced drains of the forward phase plus its own last
// commit. Makespan = max gpu_free (all tasks end on some gpu_free).
#include <cuda_runtime.h>

#include "eval_common.cuh"

namespace gpb {

namespace {

constexpr long long kNegInf = -(1LL << 60);

// One thread's row state, interleaved with the other 31 lanes of its warp.
struct SeqMem {
  long long* base;  // warp base + lane
  __device__ __forceinline__ long long& at(long long k) const { return base[k * 32]; }
};

struct SeqLayout {
  long long gf, dr, fdl, ga, links, per_link;
  int C, S, M;
  __device__ __forceinline__ void make(int C_, int S_, int M_) {
    C = C_;
    S = S_;
    M = M_;
    gf = 0;
    dr = gf + (long long)C * S;
    fdl = dr + (long long)C * S;
    ga = fdl + (long long)C * M;
    links = ga + (long long)C * S * M;
    per_link = 2LL * C * M + 2LL * M;
  }
  __device__ __forceinline__ long long mf(int w) const { return links + w * per_link; }
  __device__ __forceinline__ long long mb(int w) const { return mf(w) + (long long)C * M; }
  __device__ __forceinline__ long long of(int w) const { return mb(w) + (long long)C * M; }
  __device__ __forceinline__ long long ob(int w) const { return of(w) + M; }
};

// earliest t >= x with [t, t+len) free on (static list from cursor cur) u
// (own tail: an interval [own, own+len)); the cursor only moves forward
// (queries are non-decreasing, base.h:75-84 semantics)
__device__ __forceinline__ long long fit(const SeqMem& X, long long list, int n, int& cur,
                                         long long own, long long len, long long x) {
  long long t = x;
  for (;;) {
    while (cur < n && X.at(list + cur) + len <= t) ++cur;
    if (cur < n && X.at(list + cur) < t + len) {
      t = X.at(list + cur) + len;
      continue;
    }
    if (own + len > t) {
      t = own + len;
      continue;
    }
    return t;
  }
}

// in-place merge of own[0..no) into static[0..ns) (both sorted; the static
// entry first on ties), from the back
__device__ __forceinline__ void merge_into(const SeqMem& X, long long st, int ns, long long own,
                                           int no) {
  int i = ns - 1, j = no - 1, k = ns + no - 1;
  while (j >= 0) {
    if (i >= 0 && X.at(st + i) > X.at(own + j)) {
      X.at(st + k) = X.at(st + i);
      --i;
    } else {
      X.at(st + k) = X.at(own + j);
      --j;
    }
    --k;
  }
}

}  // namespace

// One ATLAS row on one thread; returns the makespan.
__device__ long long atlas_seq_row(const Geom& g, int L, const SeqMem& X) {
  const int S = g.S, M = g.M, C = g.C;
  const long long f = g.fwd, dur = g.dur;
  SeqLayout Y;
  Y.make(C, S, M);
  const int nw = g.nb - 1;
  auto link_after = [&](int s) -> int {  // WAN link of boundary s -> s+1
    for (int b = 1; b < g.nb; ++b)
      if (g.blk_first[b] == s + 1) return b - 1;
    return -1;
  };
  for (long long i = 0; i < 2LL * C * S; ++i) X.at(Y.gf + i) = 0;
  int nf[GPB_MAX_DC], nb_[GPB_MAX_DC], of_n[GPB_MAX_DC], ob_n[GPB_MAX_DC];
  for (int w = 0; w < nw; ++w) nf[w] = nb_[w] = of_n[w] = ob_n[w] = 0;

  // ------------------------------------------------------ forward phase
  for (int p = 0; p < C; ++p) {
    if (p > 0) {  // fold pipeline p-1's lists into the static ones
      for (int w = 0; w < nw; ++w) {
        merge_into(X, Y.mf(w), nf[w], Y.of(w), of_n[w]);
        nf[w] += of_n[w];
        merge_into(X, Y.mb(w), nb_[w], Y.ob(w), ob_n[w]);
        nb_[w] += ob_n[w];
        of_n[w] = ob_n[w] = 0;
      }
    }
    int cf[GPB_MAX_DC], cb[GPB_MAX_DC];
    for (int w = 0; w < nw; ++w) cf[w] = cb[w] = 0;
    const long long gfp = Y.gf + (long long)p * S, drp = Y.dr + (long long)p * S;
    for (int m = 0; m < M; ++m) {
      // memory-cap admission (:366-381): drain the deepest stage with a ready
      // pair (atlas_drain_step, :321-346) while some stage is blocked
      for (;;) {
        bool blocked = false;
        for (int s = 0; s < S; ++s)
          if (m - (int)X.at(drp + s) >= L) {
            blocked = true;
            break;
          }
        if (!blocked) break;
        bool drained = false;
        for (int s = S - 1; s >= 0 && !drained; --s) {
          const int mm = (int)X.at(drp + s);
          if (mm >= M) continue;
          // ready: forwarded (microbatches < m are) / gradient arrived
          if (s == S - 1 ? mm >= m : (int)X.at(drp + s + 1) <= mm) continue;
          const long long ready = s == S - 1
                                      ? X.at(Y.fdl + (long long)p * M + mm)
                                      : X.at(Y.ga + ((long long)p * S + s) * M + mm);
          long long lo = imax(ready, X.at(gfp + s));
          const int w = s > 0 ? link_after(s - 1) : -1;
          long long t = lo;
          if (w >= 0) {  // atlas_pair_start (:287-294) + reserve
            const long long len = g.ser_pooled[w];
            if (len > 0) {
              const long long own = ob_n[w] > 0 ? X.at(Y.ob(w) + ob_n[w] - 1) : kNegInf;
              t = fit(X, Y.mb(w), nb_[w], cb[w], own, len, lo + dur) - dur;
              X.at(Y.ob(w) + ob_n[w]) = t + dur;
              ++ob_n[w];
            }
          }
          const long long e = t + dur;  // atlas_commit_pair (:298-317)
          X.at(gfp + s) = imax(X.at(gfp + s), e);
          if (s > 0)
            X.at(Y.ga + ((long long)p * S + s - 1) * M + mm) =
                w >= 0 ? e + g.ser_pooled[w] + g.lat[w] : e;
          X.at(drp + s) = mm + 1;
          drained = true;
        }
        if (!drained) return -1;  // DeadlockError in the reference (unreachable)
      }
      // the chain: shift t0 until every WAN transfer fits at its compute end
      long long t0 = X.at(gfp + 0);
      for (;;) {
        bool ok = true;
        long long cur = t0;
        for (int s = 0; s < S; ++s) {
          const long long e = imax(cur, X.at(gfp + s)) + f;
          if (s + 1 < S) {
            const int w = link_after(s);
            if (w >= 0) {
              const long long len = g.ser_pooled[w];
              if (len > 0) {
                const long long own = of_n[w] > 0 ? X.at(Y.of(w) + of_n[w] - 1) : kNegInf;
                const long long slot = fit(X, Y.mf(w), nf[w], cf[w], own, len, e);
                if (slot != e) {
                  t0 += slot - e;
                  ok = false;
                  break;
                }
              }
              cur = e + len + g.lat[w];
            } else {
              cur = e;
            }
          }
        }
        if (ok) break;
      }
      long long cur = t0;  // commit (:407-430)
      for (int s = 0; s < S; ++s) {
        const long long e = imax(cur, X.at(gfp + s)) + f;
        X.at(gfp + s) = e;
        if (s == S - 1) X.at(Y.fdl + (long long)p * M + m) = e;
        if (s + 1 < S) {
          const int w = link_after(s);
          if (w >= 0) {
            if (g.ser_pooled[w] > 0) {
              X.at(Y.of(w) + of_n[w]) = e;
              ++of_n[w];
            }
            cur = e + g.ser_pooled[w] + g.lat[w];
          } else {
            cur = e;
          }
        }
      }
    }
  }
  // the last pipeline's forced drains join the static gradient lists
  for (int w = 0; w < nw; ++w) {
    merge_into(X, Y.mb(w), nb_[w], Y.ob(w), ob_n[w]);
    nb_[w] += ob_n[w];
  }

  // ------------------------------------------- drain: stage by stage
  long long mk = 0;
  for (int s = S - 1; s >= 0; --s) {
    const int w = s > 0 ? link_after(s - 1) : -1;
    const long long len = w >= 0 ? g.ser_pooled[w] : 0;
    if (w < 0 || len <= 0) {  // no shared resource: e[m] = max(r[m], e[m-1]) + dur
      const long long wl2 = w >= 0 ? g.lat[w] : 0;  // len == 0 WAN stage: latency only
      for (int p = 0; p < C; ++p) {
        long long gfv = X.at(Y.gf + (long long)p * S + s);
        for (int m = (int)X.at(Y.dr + (long long)p * S + s); m < M; ++m) {
          const long long r = s == S - 1 ? X.at(Y.fdl + (long long)p * M + m)
                                         : X.at(Y.ga + ((long long)p * S + s) * M + m);
          gfv = imax(r, gfv) + dur;
          if (s > 0) X.at(Y.ga + ((long long)p * S + s - 1) * M + m) = gfv + wl2;
        }
        X.at(Y.gf + (long long)p * S + s) = gfv;
        mk = imax(mk, gfv);
      }
      continue;
    }
    // WAN gradient link: greedy over the pipelines' next pairs
    const long long wl2 = len + g.lat[w];
    long long last = kNegInf;  // start of this stage's last committed transfer
    long long cand[32];
    int mq[32], cq[32];
    for (int q = 0; q < C; ++q) {
      mq[q] = (int)X.at(Y.dr + (long long)q * S + s);
      cq[q] = 0;
      cand[q] = kInf64;
      if (mq[q] < M) {
        const long long r = s == S - 1 ? X.at(Y.fdl + (long long)q * M + mq[q])
                                       : X.at(Y.ga + ((long long)q * S + s) * M + mq[q]);
        const long long lo = imax(r, X.at(Y.gf + (long long)q * S + s));
        cand[q] = fit(X, Y.mb(w), nb_[w], cq[q], last, len, lo + dur) - dur;
      }
    }
    for (;;) {
      int bq = -1;
      long long bt = kInf64;
      for (int q = 0; q < C; ++q)
        if (cand[q] < bt) {
          bt = cand[q];
          bq = q;
        }
      if (bq < 0) break;
      const long long e = bt + dur;
      X.at(Y.gf + (long long)bq * S + s) = e;
      X.at(Y.ga + ((long long)bq * S + s - 1) * M + mq[bq]) = e + wl2;
      last = e;
      ++mq[bq];
      cand[bq] = kInf64;
      if (mq[bq] < M) {
        const long long r = s == S - 1 ? X.at(Y.fdl + (long long)bq * M + mq[bq])
                                       : X.at(Y.ga + ((long long)bq * S + s) * M + mq[bq]);
        cand[bq] = fit(X, Y.mb(w), nb_[w], cq[bq], last, len, imax(r, e) + dur) - dur;
      }
      for (int q = 0; q < C; ++q)  // candidates pushed by the new reservation
        if (q != bq && cand[q] != kInf64 && cand[q] + dur < last + len)
          cand[q] = fit(X, Y.mb(w), nb_[w], cq[q], last, len, cand[q] + dur) - dur;
    }
    for (int q = 0; q < C; ++q) mk = imax(mk, X.at(Y.gf + (long long)q * S + s));
  }
  for (long long i = 0; i < (long long)C * S; ++i) mk = imax(mk, X.at(Y.gf + i));
  return mk;
}

__global__ void __launch_bounds__(kEvalThreads) atlas_seq_kernel(EvalArgs a) {
  const int lane = threadIdx.x & 31;
  const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  SeqMem X{a.scratch + gwarp * a.scratch_per_warp + lane};  // [element][lane]
  for (;;) {
    const int wk = atomicAdd(a.cursor, 1);
    if (wk >= a.n_work) break;
    const int row = a.work[wk];
    const long long t_start = clock64();
    const int si = a.row_scen[row];
    const DevScen& sc = a.scens[si];
    const DevTopo& tp = a.topos[sc.topo];
    Geom g;
    const int d = (int)(row - sc.first_row) + 1;
    decode(sc, tp, d, g);
    gpb_row r;
    infeasible_row(r);
    r.scenario = si;
    r.d = d;
    if (g.feasible) {
      const long long mk = atlas_seq_row(g, sc.mem_limit, X);
      finish_row(sc, tp, g, mk, r);
      if (mk < 0) {
        r.feasible = -1;
        atomicExch(a.error_flag, 1);
      }
    }
    if (a.row_cycles) a.row_cycles[row] = clock64() - t_start;
    a.rows[row] = r;
  }
}

// int64 elements of one thread's slice for rows up to (C, S, M, nw)
long long atlas_seq_slice(int C, int S, int M, int nw) {
  return 2LL * C * S + (long long)C * M + (long long)C * S * M +
         (long long)nw * (2LL * C * M + 2LL * M);
}

int atlas_seq_blocks_per_sm() {
  int n = 0;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, atlas_seq_kernel, kEvalThreads, 0) ==
                 cudaSuccess
             ? n
             : 1;
}

cudaError_t launch_atlas_seq(const EvalArgs& a, int grid, cudaStream_t st) {
  atlas_seq_kernel<<<grid, kEvalThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace gpb
