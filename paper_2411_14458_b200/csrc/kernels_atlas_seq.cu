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
// The state of a row lives in a per-thread slice of global scratch:
//   GF[C][S]   gpu_free        DR[C][S]  drained counts
//   FDL[C][R]  last-stage forward ends, ring of R slots
//   GA[C][S][R] gradient arrivals at stage s, ring of R slots (pair m's
//              arrival exists once stage s+1 has drained pair m)
// A pair is "in flight" at stage s between its producer's commit (stage s+1,
// or the forward at S-1) and its own drain. The memory cap keeps at most
// L = mem_limit pairs in flight per stage: after every admission no stage
// is blocked (m - drained[s] < L), a cascade drains a stage only after the
// stage above, and after the last admission at most L pairs remain per
// stage for the drain phase. So rings of R = 2^ceil(log2(min(L, M))) slots
// indexed m & (R-1) hold every live value (the reference keeps all M).
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
constexpr int kSeqMaxC = 8;  // pipelines per cell (host-checked)

// One thread's row state: a contiguous slice, so the streams a row walks
// (its rings, list cursors, appends) stay within few cache lines. Lanes of a
// warp diverge in shape and progress, so an [element][lane] interleave buys
// no coalescing and costs a new line per element (measured: 43% L2 hits,
// long-scoreboard bound).
struct SeqMem {
  long long* base;
  __device__ __forceinline__ long long& at(long long k) const { return base[k]; }
};

// The row's small, hot scalars — per-link serialization / latency, list
// lengths and cursors, the drain's candidates — live in shared memory, one
// column per thread ([field][thread]: conflict-free). As local arrays they
// were a 720-byte stack frame per thread, 368 KB per SM at 4 blocks: more
// than L1, so every cursor step went to L2.
constexpr int kSeqLinks = GPB_MAX_DC - 1;
struct SeqSmall {
  long long* l;  // [field][thread] int64: ser[7] lat[7] T.cand(8)
  int* i;        // [field][thread] int32: nf nb ofn obn cf cb [7 each], mq cq [8 each]
  signed char* lk;  // [16][thread]: WAN link after stage s
  int t;
  __device__ __forceinline__ long long& ser(int w) const { return l[(0 + w) * kEvalThreads + t]; }
  __device__ __forceinline__ long long& lat(int w) const { return l[(7 + w) * kEvalThreads + t]; }
  __device__ __forceinline__ long long& cand(int q) const { return l[(14 + q) * kEvalThreads + t]; }
  __device__ __forceinline__ int& nf(int w) const { return i[(0 + w) * kEvalThreads + t]; }
  __device__ __forceinline__ int& nb(int w) const { return i[(7 + w) * kEvalThreads + t]; }
  __device__ __forceinline__ int& ofn(int w) const { return i[(14 + w) * kEvalThreads + t]; }
  __device__ __forceinline__ int& obn(int w) const { return i[(21 + w) * kEvalThreads + t]; }
  __device__ __forceinline__ int& cf(int w) const { return i[(28 + w) * kEvalThreads + t]; }
  __device__ __forceinline__ int& cb(int w) const { return i[(35 + w) * kEvalThreads + t]; }
  __device__ __forceinline__ int& mq(int q) const { return i[(42 + q) * kEvalThreads + t]; }
  __device__ __forceinline__ int& cq(int q) const { return i[(50 + q) * kEvalThreads + t]; }
  __device__ __forceinline__ signed char& link(int s) const { return lk[s * kEvalThreads + t]; }
};
constexpr int kSeqSmallBytes = (22 * 8 + 58 * 4 + 16) * kEvalThreads;

// ring slots for a row: the smallest power of two >= min(mem_limit, M)
__host__ __device__ __forceinline__ int seq_ring(int L, int M) {
  const int n = L < M ? L : M;
  int r = 1;
  while (r < n) r <<= 1;
  return r;
}

struct SeqLayout {
  long long gf, dr, fdl, ga, links, per_link;
  int C, S, M, R;
  __device__ __forceinline__ void make(int C_, int S_, int M_, int R_) {
    C = C_;
    S = S_;
    M = M_;
    R = R_;
    gf = 0;
    dr = gf + (long long)C * S;
    fdl = dr + (long long)C * S;
    ga = fdl + (long long)C * R;
    links = ga + (long long)C * S * R;
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

// WAN link of boundary s -> s+1, or -1
__device__ __forceinline__ int link_of(const Geom& g, int s) {
  for (int b = 1; b < g.nb; ++b)
    if (g.blk_first[b] == s + 1) return b - 1;
  return -1;
}

}  // namespace

// One ATLAS row on one thread; returns the makespan. SMAX >= S bounds the
// stage loops, which are unrolled so the current pipeline's per-stage state
// (gpu_free, drained counts, WAN links) stays in registers.
template <int SMAX>
__device__ long long atlas_seq_row(const Geom& g, int L, const SeqMem& X, const SeqSmall& T) {
  const int S = g.S, M = g.M, C = g.C;
  const long long f = g.fwd, dur = g.dur;
  SeqLayout Y;
  const int R = seq_ring(L, M), RM = R - 1;
  Y.make(C, S, M, R);
  const int nw = g.nb - 1;
  int lk[SMAX];  // WAN link of boundary s -> s+1, or -1
#pragma unroll
  for (int s = 0; s < SMAX; ++s) {
    lk[s] = -1;
    for (int b = 1; b < g.nb; ++b)
      if (g.blk_first[b] == s + 1 && s + 1 < S) lk[s] = b - 1;
  }
  for (int w = 0; w < nw; ++w) {
    T.nf(w) = T.nb(w) = T.ofn(w) = T.obn(w) = 0;
    T.ser(w) = g.ser_pooled[w];
    T.lat(w) = g.lat[w];
  }
  for (int s = 0; s < S; ++s) T.link(s) = (signed char)link_of(g, s);

  // ------------------------------------------------------ forward phase
  for (int p = 0; p < C; ++p) {
    if (p > 0) {  // fold pipeline p-1's lists into the static ones
      for (int w = 0; w < nw; ++w) {
        merge_into(X, Y.mf(w), T.nf(w), Y.of(w), T.ofn(w));
        T.nf(w) += T.ofn(w);
        merge_into(X, Y.mb(w), T.nb(w), Y.ob(w), T.obn(w));
        T.nb(w) += T.obn(w);
        T.ofn(w) = T.obn(w) = 0;
      }
    }
    for (int w = 0; w < nw; ++w) T.cf(w) = T.cb(w) = 0;
    long long gfr[SMAX];
    int drr[SMAX];
#pragma unroll
    for (int s = 0; s < SMAX; ++s) {
      gfr[s] = 0;
      drr[s] = 0;
    }
    const long long fdlp = Y.fdl + (long long)p * R, gap = Y.ga + (long long)p * S * R;
    for (int m = 0; m < M; ++m) {
      // memory-cap admission (:366-381): the reference repeats
      // atlas_drain_step (:321-346), "drain the deepest stage with a ready
      // pair", while some stage is blocked (m - drained >= L). Draining a
      // stage unblocks only itself and readies only the stage below, so the
      // repetition is: every stage above the lowest blocked one s_min drains
      // all its ready pairs (up to m-1), s_min drains to m-L+1; each
      // gradient link has one writer stage, so stages run one after another.
      int s_min = -1;
#pragma unroll
      for (int s = SMAX - 1; s >= 0; --s)
        if (s < S && m - drr[s] >= L) s_min = s;
      if (s_min >= 0) {
#pragma unroll
        for (int s = SMAX - 1; s >= 0; --s) {
          if (s >= S || s < s_min) continue;
          const int upto = s == s_min ? m - L + 1 : m;
          const int w = s > 0 ? lk[s - 1] : -1;
          const long long len = w >= 0 ? T.ser(w) : 0;
          const long long wl = w >= 0 ? len + T.lat(w) : 0;
          long long gv = gfr[s];
          for (int mm = drr[s]; mm < upto; ++mm) {
            const long long ready =
                s == S - 1 ? X.at(fdlp + (mm & RM)) : X.at(gap + (long long)s * R + (mm & RM));
            long long t = imax(ready, gv);
            if (len > 0) {  // atlas_pair_start (:287-294) + reserve
              const long long own = T.obn(w) > 0 ? X.at(Y.ob(w) + T.obn(w) - 1) : kNegInf;
              t = fit(X, Y.mb(w), T.nb(w), T.cb(w), own, len, t + dur) - dur;
              X.at(Y.ob(w) + T.obn(w)) = t + dur;
              ++T.obn(w);
            }
            gv = t + dur;  // atlas_commit_pair (:298-317)
            if (s > 0) X.at(gap + (long long)(s - 1) * R + (mm & RM)) = gv + wl;
          }
          if (upto > drr[s]) {
            gfr[s] = gv;
            drr[s] = upto;
          }
        }
      }
      // the chain: shift t0 until every WAN transfer fits at its compute end
      // (:383-405), then commit (:407-430)
      long long t0 = gfr[0];
      for (;;) {
        bool ok = true;
        long long cur = t0;
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
          if (s < S && ok) {
            const long long e = imax(cur, gfr[s]) + f;
            const int w = lk[s];
            cur = e;
            if (w >= 0) {
              const long long len = T.ser(w);
              if (len > 0) {
                const long long own = T.ofn(w) > 0 ? X.at(Y.of(w) + T.ofn(w) - 1) : kNegInf;
                const long long slot = fit(X, Y.mf(w), T.nf(w), T.cf(w), own, len, e);
                if (slot != e) {
                  t0 += slot - e;
                  ok = false;
                }
              }
              cur = e + len + T.lat(w);
            }
          }
        }
        if (ok) break;
      }
      long long cur = t0;
#pragma unroll
      for (int s = 0; s < SMAX; ++s) {
        if (s < S) {
          const long long e = imax(cur, gfr[s]) + f;
          gfr[s] = e;
          cur = e;
          const int w = lk[s];
          if (w >= 0) {
            if (T.ser(w) > 0) {
              X.at(Y.of(w) + T.ofn(w)) = e;
              ++T.ofn(w);
            }
            cur = e + T.ser(w) + T.lat(w);
          }
          if (s == S - 1) X.at(fdlp + (m & RM)) = e;
        }
      }
    }
#pragma unroll
    for (int s = 0; s < SMAX; ++s)
      if (s < S) {
        X.at(Y.gf + (long long)p * S + s) = gfr[s];
        X.at(Y.dr + (long long)p * S + s) = drr[s];
      }
  }
  // the last pipeline's forced drains join the static gradient lists
  for (int w = 0; w < nw; ++w) {
    merge_into(X, Y.mb(w), T.nb(w), Y.ob(w), T.obn(w));
    T.nb(w) += T.obn(w);
  }

  // ------------------------------------------- drain: stage by stage
  long long mk = 0;
  for (int s = S - 1; s >= 0; --s) {
    const int w = s > 0 ? (int)T.link(s - 1) : -1;
    const long long len = w >= 0 ? T.ser(w) : 0;
    if (w < 0 || len <= 0) {  // no shared resource: e[m] = max(r[m], e[m-1]) + dur
      const long long wl2 = w >= 0 ? T.lat(w) : 0;  // len == 0 WAN stage: latency only
      for (int p = 0; p < C; ++p) {
        long long gfv = X.at(Y.gf + (long long)p * S + s);
        for (int m = (int)X.at(Y.dr + (long long)p * S + s); m < M; ++m) {
          const long long r = s == S - 1 ? X.at(Y.fdl + (long long)p * R + (m & RM))
                                         : X.at(Y.ga + ((long long)p * S + s) * R + (m & RM));
          gfv = imax(r, gfv) + dur;
          if (s > 0) X.at(Y.ga + ((long long)p * S + s - 1) * R + (m & RM)) = gfv + wl2;
        }
        X.at(Y.gf + (long long)p * S + s) = gfv;
        mk = imax(mk, gfv);
      }
      continue;
    }
    // WAN gradient link: greedy over the pipelines' next pairs
    const long long wl2 = len + T.lat(w);
    long long last = kNegInf;  // start of this stage's last committed transfer
    for (int q = 0; q < C; ++q) {
      T.mq(q) = (int)X.at(Y.dr + (long long)q * S + s);
      T.cq(q) = 0;
      T.cand(q) = kInf64;
      if (T.mq(q) < M) {
        const long long r = s == S - 1 ? X.at(Y.fdl + (long long)q * R + (T.mq(q) & RM))
                                       : X.at(Y.ga + ((long long)q * S + s) * R + (T.mq(q) & RM));
        const long long lo = imax(r, X.at(Y.gf + (long long)q * S + s));
        T.cand(q) = fit(X, Y.mb(w), T.nb(w), T.cq(q), last, len, lo + dur) - dur;
      }
    }
    for (;;) {
      int bq = -1;
      long long bt = kInf64;
      for (int q = 0; q < C; ++q)
        if (T.cand(q) < bt) {
          bt = T.cand(q);
          bq = q;
        }
      if (bq < 0) break;
      const long long e = bt + dur;
      X.at(Y.gf + (long long)bq * S + s) = e;
      X.at(Y.ga + ((long long)bq * S + s - 1) * R + (T.mq(bq) & RM)) = e + wl2;
      last = e;
      ++T.mq(bq);
      T.cand(bq) = kInf64;
      if (T.mq(bq) < M) {
        const long long r = s == S - 1 ? X.at(Y.fdl + (long long)bq * R + (T.mq(bq) & RM))
                                       : X.at(Y.ga + ((long long)bq * S + s) * R + (T.mq(bq) & RM));
        T.cand(bq) = fit(X, Y.mb(w), T.nb(w), T.cq(bq), last, len, imax(r, e) + dur) - dur;
      }
      for (int q = 0; q < C; ++q)  // candidates pushed by the new reservation
        if (q != bq && T.cand(q) != kInf64 && T.cand(q) + dur < last + len)
          T.cand(q) = fit(X, Y.mb(w), T.nb(w), T.cq(q), last, len, T.cand(q) + dur) - dur;
    }
    for (int q = 0; q < C; ++q) mk = imax(mk, X.at(Y.gf + (long long)q * S + s));
  }
  for (long long i = 0; i < (long long)C * S; ++i) mk = imax(mk, X.at(Y.gf + i));
  return mk;
}

template <int SMAX>
__global__ void __launch_bounds__(kEvalThreads, 4) atlas_seq_kernel(EvalArgs a) {
  const int lane = threadIdx.x & 31;
  const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  SeqMem X{a.scratch + gwarp * a.scratch_per_warp + (long long)lane * (a.scratch_per_warp / 32)};
  extern __shared__ __align__(16) unsigned char seq_smem[];
  SeqSmall T{(long long*)seq_smem, (int*)(seq_smem + 22 * 8 * kEvalThreads),
             (signed char*)(seq_smem + (22 * 8 + 58 * 4) * kEvalThreads), (int)threadIdx.x};
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
      const long long mk = atlas_seq_row<SMAX>(g, sc.mem_limit, X, T);
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

// int64 elements of one thread's slice for rows up to (C, S, M, nw) with
// memory cap L
long long atlas_seq_slice(int C, int S, int M, int nw, int L) {
  const long long R = seq_ring(L, M);
  return 2LL * C * S + (long long)C * R + (long long)C * S * R +
         (long long)nw * (2LL * C * M + 2LL * M);
}

static void seq_smem_attrs() {
  static bool done = false;  // per process; the attribute is per function
  if (done) return;
  cudaFuncSetAttribute(atlas_seq_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kSeqSmallBytes);
  cudaFuncSetAttribute(atlas_seq_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kSeqSmallBytes);
  cudaFuncSetAttribute(atlas_seq_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kSeqSmallBytes);
  done = true;
}

int atlas_seq_blocks_per_sm(int smax) {
  seq_smem_attrs();
  int n = 0;
  const cudaError_t e =
      smax <= 4 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, atlas_seq_kernel<4>,
                                                                kEvalThreads, kSeqSmallBytes)
      : smax <= 8 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, atlas_seq_kernel<8>,
                                                                  kEvalThreads, kSeqSmallBytes)
                  : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, atlas_seq_kernel<16>,
                                                                  kEvalThreads, kSeqSmallBytes);
  return e == cudaSuccess ? n : 1;
}

// smax: 4, 8 or 16 (rows with S <= smax)
cudaError_t launch_atlas_seq(int smax, const EvalArgs& a, int grid, cudaStream_t st) {
  seq_smem_attrs();
  if (smax <= 4)
    atlas_seq_kernel<4><<<grid, kEvalThreads, kSeqSmallBytes, st>>>(a);
  else if (smax <= 8)
    atlas_seq_kernel<8><<<grid, kEvalThreads, kSeqSmallBytes, st>>>(a);
  else
    atlas_seq_kernel<16><<<grid, kEvalThreads, kSeqSmallBytes, st>>>(a);
  return cudaGetLastError();
}

}  // namespace gpb
