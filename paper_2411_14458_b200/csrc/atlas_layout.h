// atlas_layout.h — per-warp shared-memory slice of the ATLAS kernel, shared
// by the host (sizing) and the device (carving). All offsets in bytes,
// 16-byte aligned.
#pragma once

#include <cstddef>
#include <cstdint>

namespace gpb {

struct AtlasLayout {
  // inputs
  int C, S, M, nw;     // nw = max WAN boundaries (<= 7)
  long long garr_cap;  // gradient-queue entries kept in shared memory per warp
                       // (rows with C*S*M above it use the global scratch)
  // outputs
  bool big_in_smem = true;  // lists in the shared slice (else the global scratch)
  size_t off_wa, off_wg, off_wbs, off_gf, off_nm, off_firstm, off_mcnt, off_big, off_garr,
      total;
  // "big" region (lists), relative to its base
  size_t off_fdl, off_resf, off_resb, off_mf, off_mb, off_mtmp, off_jf, off_jb, big_total;
  int cap;             // list storage per WAN boundary = C * M (C lists of M)

  __host__ __device__ static size_t al(size_t x) { return (x + 15) & ~(size_t)15; }

  __host__ __device__ void compute() {
    const size_t CS = (size_t)C * S;
    cap = C * M;
    size_t o = 0;
    off_fdl = o;       o = al(o + (size_t)C * M * 8);   // last-stage forward ends
    off_resf = o;      o = al(o + (size_t)nw * cap * 8);  // per-pipeline link lists
    off_resb = o;      o = al(o + (size_t)nw * cap * 8);
    // merged static lists (pipelines < p) per WAN link, forward / gradient
    off_mf = o;        o = al(o + (size_t)nw * cap * 8);
    off_mb = o;        o = al(o + (size_t)nw * cap * 8);
    off_mtmp = o;      o = al(o + (size_t)cap * 8);
    off_jf = o;        o = al(o + (size_t)nw * cap * 4);  // run jumps of mf / mb
    off_jb = o;        o = al(o + (size_t)nw * cap * 4);
    big_total = o;
    o = 0;
    off_wa = o;        o = al(o + 16 * 8);          // a_w [0,8) | ser_w [8,16)
    off_wg = o;        o = al(o + 16 * 8);          // G_w [0,8) | lat_w [8,16)
    off_wbs = o;       o = al(o + (size_t)S * 4);   // WAN boundary before stage s
    off_gf = o;        o = al(o + CS * 8);
    off_nm = o;        o = al(o + CS * 4);
    off_firstm = o;    o = al(o + CS * 4);
    off_mcnt = o;      o = al(o + 32 * 4);          // counts / cursors
    off_big = o;
    if (big_in_smem) o = al(o + big_total);
    off_garr = o;
    o = al(o + (size_t)garr_cap * 8);
    total = o;
  }
};

}  // namespace gpb
