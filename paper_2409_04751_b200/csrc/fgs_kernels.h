// fgs_kernels.h — kernel argument blocks and launch entry points shared by the .cu files.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "fgs_common.cuh"

namespace fgs {

struct PreprocessArgs {
  int64_t n;
  DevCamera cam;
  int sh_degree;
  int tiles_x, tiles_y;
  const float* means;
  const float* rotations;
  const float* log_scales;
  const float* opacity;
  const float* sh;
  SortedRec* rec;        // per-Gaussian splat record
  uint8_t* state;
  uint32_t* depth_key;   // level-1 sort keys (0xFFFFFFFF for culled)
  uint32_t* touched;     // tiles touched
  ushort4* rect;         // tx0, tx1, ty0, ty1
  int32_t* radii;        // per Gaussian radius (0 = culled / degenerate)
  int32_t* rowdiff;      // tiles_y x (tiles_x + 1) row-difference tile counts
  int* error_flag;
  uint32_t* state_counts;  // [kept, degenerate]
};

struct PreprocessBackwardArgs {
  int64_t n;
  int64_t m;                 // Gaussians that touched >= 1 tile (level-1 compaction count)
  const uint32_t* cval;      // [m] their ids in source order
  const SortedRec* rec;      // K1 per-Gaussian records (alpha, clamped colours)
  DevCamera cam;
  int sh_degree;
  int full_sh;
  int accumulate;
  int view_dir;
  float jac_grad_scale[3];
  const float* means;
  const float* rotations;
  const float* log_scales;
  const float* opacity;
  const float* sh;
  const uint8_t* state;
  const uint32_t* touched;
  const uint32_t* coff;      // [m] first emission slot of cval[q]
  const ushort4* rect;       // [n] tile rectangles (K1)
  const uint32_t* emit_pos;  // [I] sorted position of each emission slot
  const float* partials;     // [I][8][9] K4a per-(intersection, block) sums, sorted order
  float* d_means;
  float* d_rotations;
  float* d_log_scales;
  float* d_opacity;
  float* d_sh;
  int aligned16;             // d_rotations and d_sh 16-byte aligned: float4 stores
};

struct BlendArgs {
  int width, height, tiles_x, tiles_y;
  const uint32_t* tile_offsets;  // T+1
  const uint32_t* sorted_gauss;  // I
  const SortedRec* srec;         // I records in sorted order (nullptr: read rec[sorted_gauss[k]])
  const SortedRec* rec;          // per-Gaussian records
  float bg[3];
  float* image;                  // H*W*3
  float* final_T;                // H*W
  uint32_t* last;                // H*W: index one past the last contributing entry
  unsigned long long* counters;  // optional: E_eval, E_contrib, culled evals, max CTA cycles
  unsigned long long* tile_cycles;  // optional (with counters): per-tile CTA cycles
  const uint32_t* tile_order;    // optional: CTA -> tile (heaviest lists first)
  int px_per_lane;               // forward blend: 1 or 2 pixels per lane
  const uint32_t* scalars;       // forward: device scalars; exit if I > isect_cap (speculative launch)
  int64_t isect_cap;
  // backward
  const float* dl_dimage;
  float* partials;               // I x 8 x 9
};

__global__ void preprocess_kernel(PreprocessArgs a);
__global__ void preprocess_backward_kernel(PreprocessBackwardArgs a);
constexpr int kPreprocessBackwardThreads = 128;  // tile-touching Gaussians per K4b CTA

// ---- binning / sorting (binning.cu) ----
constexpr int kBinThreads = 1024;
constexpr int kScalarI = 0, kScalarErr = 1, kScalarKept = 2, kScalarDegen = 3, kScalarM = 4, kScalarI2 = 5, kScalarBig = 6;

struct BinArgs {
  int n;                       // Gaussians
  int tiles_x, tiles_y, num_tiles;
  int64_t isect_cap;           // capacity of the per-intersection buffers (scatter/sort exit if I exceeds it)
  const uint32_t* touched;     // [n] tiles touched per Gaussian (K1)
  const uint32_t* depth_key;   // [n] depth key bits (K1)
  const ushort4* rect;         // [n] tile rectangle (K1)
  int32_t* rowdiff;            // [tiles_y * (tiles_x + 1)] row-difference tile counts (K1 adds, bin_scan zeroes)
  uint32_t* cval;              // [n] tile-touching Gaussians in source order (compacted)
  uint32_t* coff;              // [n] their first emission slot
  uint32_t* scalars;           // device scalars (kScalar*)
  uint32_t* part_scan;         // [2 * grid]
  uint32_t* tile_offsets;      // [num_tiles + 1]
  uint32_t* fill;              // [num_tiles] scatter cursors
  uint32_t* tile_order;        // [num_tiles] blend schedule (optional)
  // per intersection
  uint64_t* keys;              // [I] (depth_key << 32 | emission slot), grouped by tile
  uint32_t* emit_gauss;        // [I] Gaussian of each emission slot
  uint32_t* sorted_gauss;      // [I]
  uint32_t* emit_pos;          // [I] sorted position of each emission slot
  const SortedRec* rec;        // per-Gaussian splat records (K1 output)
  SortedRec* sorted_rec;       // [I] records in sorted order (optional)
};

// Words of part_scan scratch bin_scan needs.
size_t bin_part_words();
// K2a: compaction + emission offsets + I (scalars), tile ranges + blend schedule.
cudaError_t bin_scan(BinArgs& a, cudaStream_t st);
// K2b + K2c: key scatter into tile ranges, per-tile sort; returns launches. The kernels read
// I and the big-tile count from the device scalars and do nothing if I > a.isect_cap; n_big
// < 0 (unknown on the host) sizes the sort grid for the worst case.
int bin_sort(BinArgs& a, int n_big, cudaStream_t st);
// Debug: the reference's pre-sort key list (source order).
cudaError_t debug_source_order_keys(BinArgs& a, uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss,
                                    cudaStream_t st);

// ---- blend (raster.cu) ----
int blend_forward(const BlendArgs& a, cudaStream_t st);
int blend_backward(const BlendArgs& a, cudaStream_t st);
// FP32 pipe probe: returns achieved non-FMA fp32 op/s (FMUL + FADD, no contraction).
double fp32_peak_probe(cudaStream_t st);

}  // namespace fgs
