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
  const uint32_t* rank;
  const uint32_t* offsets;   // per depth rank
  const float* partials;     // I x 9 per-intersection sums (K4c output)
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
  const uint32_t* sorted_emit;   // I (emission slot of each sorted entry; backward partials)
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
  // backward
  const float* dl_dimage;
  float* partials;               // I x 8 x 9
};

__global__ void preprocess_kernel(PreprocessArgs a);
__global__ void preprocess_backward_kernel(PreprocessBackwardArgs a);
constexpr int kPreprocessBackwardThreads = 128;  // tile-touching Gaussians per K4b CTA

// ---- binning / sorting (binning.cu) ----
constexpr int kBinThreads = 1024;
constexpr int kScalarI = 0, kScalarErr = 1, kScalarKept = 2, kScalarDegen = 3, kScalarM = 4;

struct BinArgs {
  int n;                       // Gaussians
  int tiles_x, num_tiles, passes2;
  int num_isect;               // I (level 2 only; known on the host after level 1)
  const uint32_t* touched;     // [n]
  const uint32_t* depth_key_in;  // [n]
  const ushort4* rect;         // [n]
  uint32_t* ckey;              // compacted depth keys [n]
  uint32_t* cval;              // compacted Gaussian ids [n]
  uint32_t* key_a;             // ping-pong [n]
  uint32_t* val_a;
  uint32_t* key_b;
  uint32_t* val_b;             // level-1 result: Gaussian ids by depth rank
  uint32_t* offsets;           // [n] emission offset per depth rank
  uint32_t* rank;              // [n] depth rank per Gaussian
  uint32_t* scalars;           // device scalars (kScalar*)
  uint32_t* part_scan;         // [grid]
  uint32_t* part_radix;        // [grid * 256]
  // level 2
  uint32_t* tkey;              // [I] tile keys (emission order)
  uint32_t* emit;              // [I] emission slots
  uint32_t* emit_gauss;        // [I] Gaussian of each emission slot
  uint32_t* tkey_a;
  uint32_t* emit_a;
  uint32_t* tkey_b;
  uint32_t* emit_b;
  uint32_t* tile_offsets;      // [num_tiles + 1]
  uint32_t* sorted_gauss;      // [I]
  uint32_t* sorted_emit;       // [I]
  const SortedRec* rec;        // per-Gaussian splat records (K1 output)
  SortedRec* sorted_rec;       // [I] records in sorted order
  uint32_t* tile_order;        // [num_tiles] blend schedule (optional)
  unsigned long long* trace;   // debug phase timestamps (optional)
};

// Words of part_scan + part_radix scratch the persistent kernels need.
size_t bin_part_words();
// Compaction + level-1 sort + rank scan (writes scalars[kScalarM], scalars[kScalarI]).
cudaError_t bin_level1(BinArgs& a, cudaStream_t st);
// Duplication + level-2 sort + tile ranges (needs a.num_isect).
cudaError_t bin_level2(BinArgs& a, cudaStream_t st);
// Debug: the reference's pre-sort key list (source order).
cudaError_t debug_source_order_keys(BinArgs& a, uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss,
                                    cudaStream_t st);

// ---- blend (raster.cu) ----
int blend_forward(const BlendArgs& a, cudaStream_t st);
int blend_backward(const BlendArgs& a, cudaStream_t st);
// K4c: per intersection, sum the per-block partials of the blocks passing the culling test.
int combine_partials(const uint32_t* tile_keys, const uint32_t* emit_gauss, const SortedRec* rec,
                     const float* partials, float* partial_tile, int tiles_x, int ni, cudaStream_t st);
// FP32 pipe probe: returns achieved non-FMA fp32 op/s (FMUL + FADD, no contraction).
double fp32_peak_probe(cudaStream_t st);

}  // namespace fgs
