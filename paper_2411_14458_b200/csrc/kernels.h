// kernels.h — launch interface between the host planner (host.cpp) and the
// sm_100a kernels. Plain structs of device pointers; no torch types.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/geopipe_batch.h"
#include "atlas_layout.h"

namespace gpb {

struct DevTopo;
struct DevScen;

constexpr int kEvalThreads = 128;  // 4 warps per CTA, one plan row per warp

struct EvalArgs {
  const DevScen* scens;
  const DevTopo* topos;
  const int32_t* row_scen;    // row -> scenario
  const int32_t* work;        // rows of this bucket, in dispatch order
  int32_t n_work;
  int32_t* cursor;            // atomic work cursor (zeroed per launch)
  gpb_row* rows;              // output table
  int32_t* error_flag;
  long long* row_cycles;      // optional per-row clock64 cost (profiling)
  long long* row_phase;       // optional [row][4] atlas phase cycles (profiling)
  // timeline variant: per-work-item offsets into forward-end / pair-start
  // arrays laid out [pipeline][stage][microbatch]
  long long* tl_fe;
  long long* tl_ps;
  const long long* tl_off;
  // flush: per-warp shared fd_last buffer length (max M of the bucket)
  int32_t smem_m;
  int32_t smem_floor;         // atlas warp kernel: dynamic shared memory at least this (bytes)
  int32_t drain_lane;         // atlas: WAN-stage drain greedy on one lane when C <= 4 and S >= this (0 = never)
  int32_t occ4;               // atlas B = 1: the 4-blocks-per-SM instantiation (large spaces)
  // atlas: per-warp shared slice and (when it does not fit) global garr
  AtlasLayout lay;
  long long* scratch;
  long long scratch_per_warp; // int64 elements per warp (global garr + lists)
  long long scratch_big_off;  // int64 offset of the lists inside a warp's scratch
};

struct SelectArgs {
  const DevScen* scens;
  const int32_t* scen_list;   // scenarios to select (nullable: 0 .. n_scen-1)
  int32_t n_scen;
  gpb_row* rows;
  gpb_scenario_result* results;
  gpb_best* block_best;       // [grid]
  gpb_best* best;
};

cudaError_t launch_flush(int B, bool gpipe, const EvalArgs& a, int grid, cudaStream_t st);
// shallow pipelines (S <= gw, gw = 8 or 16): 32/gw rows per warp
cudaError_t launch_flush_group(int gw, bool gpipe, const EvalArgs& a, int grid, cudaStream_t st);
cudaError_t launch_onef1b(int B, const EvalArgs& a, int grid, cudaStream_t st);
cudaError_t launch_onef1b_group(int gw, const EvalArgs& a, int grid, cudaStream_t st);
cudaError_t launch_atlas(int B, const EvalArgs& a, int grid, int wpc, cudaStream_t st);
int atlas_blocks_per_sm(int B, bool timeline, int wpc, size_t smem, bool occ4 = false);
// one thread per ATLAS row (bulk of large spaces); scratch_per_warp = 32 x
// the per-thread slice (int64 elements) for rows up to (C, S, M, nw)
long long atlas_seq_slice(int C, int S, int M, int nw, int L);
// heavy ATLAS rows (S <= 32, 2 <= C <= 4): one CTA per row, warp = pipeline;
// the AtlasLayout slice (+ wave state) per CTA, scratch_per_warp per CTA
constexpr int kWaveMaxPipes = 4;  // = kWaveRegC (register-cached list views)
int atlas_wave_smem(const AtlasLayout& L);
int atlas_wave_blocks_per_sm(int warps, int smem);
cudaError_t launch_atlas_wave(const EvalArgs& a, int grid, int warps, cudaStream_t st);
int atlas_seq_blocks_per_sm(int smax);
cudaError_t launch_atlas_seq(int smax, const EvalArgs& a, int grid, cudaStream_t st);
cudaError_t launch_select(const SelectArgs& a, int grid, cudaStream_t st);
// select_kernel alone (per bucket) / the final reduction of the block bests
cudaError_t launch_select_part(const SelectArgs& a, int grid, cudaStream_t st);
cudaError_t launch_best_reduce(const gpb_best* in, int n, gpb_best* out, cudaStream_t st);
cudaError_t launch_timeline(int policy, int B, const EvalArgs& a, int grid, cudaStream_t st);
cudaError_t launch_atlas_timeline(int B, const EvalArgs& a, int grid, int wpc, cudaStream_t st);

}  // namespace gpb

namespace gpb {
cudaError_t launch_maxplus_bench(int kind, long long* out, int grid, int iters, cudaStream_t st);
}
