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
  float4* rec0;
  float4* rec1;
  float* rec2;
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
  const float* partials;     // I x 9
  float* d_means;
  float* d_rotations;
  float* d_log_scales;
  float* d_opacity;
  float* d_sh;
};

struct BlendArgs {
  int width, height, tiles_x, tiles_y;
  const uint32_t* tile_offsets;  // T+1
  const uint32_t* sorted_gauss;  // I
  const uint32_t* sorted_emit;   // I (emission slot of each sorted entry; backward partials)
  SplatRefs rec;
  float bg[3];
  float* image;                  // H*W*3
  float* final_T;                // H*W
  uint32_t* last;                // H*W: index one past the last contributing entry
  unsigned long long* counters;  // optional: E_eval, E_contrib
  // backward
  const float* dl_dimage;
  float* partials;               // I x 9
};

__global__ void preprocess_kernel(PreprocessArgs a);
__global__ void preprocess_backward_kernel(PreprocessBackwardArgs a);

// ---- binning / sorting (binning.cu) ----
struct SortScratch {
  uint32_t* hist;        // passes * 256 (exclusive offsets after scan)
  uint32_t* lookback;    // passes * max_tiles * 256
  uint32_t* counters;    // passes tile counters
  int max_tiles;
};
constexpr int kSortThreads = 512;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 8192
constexpr int kMaxPasses = 4;

// Stable LSD radix sort of (u32 key, u32 value) over bits [0, 8*passes). The inputs are not
// modified; passes alternate b, a, b, a. Returns where the sorted pairs are.
struct SortResult {
  uint32_t* keys;
  uint32_t* vals;
  int launches;
};
SortResult radix_sort_pairs(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_a, uint32_t* vals_a,
                            uint32_t* keys_b, uint32_t* vals_b, const uint32_t* n_dev, int n_max, int passes,
                            const SortScratch& s, bool hist_ready, cudaStream_t st);

// Status words a single-pass scan over n_max items needs.
size_t scan_status_words(int n_max);
// Stream compaction (source order) of the Gaussians touching >= 1 tile: keys_out = depth keys,
// vals_out = Gaussian indices, *count_out = their number (device); hist = the 4 digit
// histograms of the compacted keys (level-1 sort input).
int compact_visible(const uint32_t* touched, const uint32_t* depth_key, uint32_t* keys_out, uint32_t* vals_out,
                    uint32_t* count_out, int n, uint32_t* status, uint32_t* counter, uint32_t* hist,
                    cudaStream_t st);
// Exclusive scan of touched[perm[r]] over depth ranks r < *n_dev: offsets[r], rank[perm[r]] = r,
// *total_out = I (device).
int rank_scan(const uint32_t* perm, const uint32_t* touched, uint32_t* offsets, uint32_t* rank,
              const uint32_t* n_dev, int n_max, uint32_t* total_out, uint32_t* status, uint32_t* counter,
              cudaStream_t st);
// Emit (tile key, emission slot, gaussian) per intersection in depth-rank order.
int duplicate(const uint32_t* perm, const uint32_t* offsets, const uint32_t* touched, const ushort4* rect, int tiles_x,
              uint32_t* tile_keys, uint32_t* emit_vals, uint32_t* emit_gauss, const uint32_t* n_dev, int n_max,
              uint32_t* hist, int passes, cudaStream_t st);
// Per-tile ranges from sorted tile keys; sorted_gauss[k] = emit_gauss[sorted_emit[k]].
int tile_ranges(const uint32_t* sorted_tiles, const uint32_t* sorted_emit, const uint32_t* emit_gauss,
                uint32_t* tile_offsets, uint32_t* sorted_gauss, int num_isect, int num_tiles, cudaStream_t st);
// Debug: reference emission order keys (source order, ty-major, tx-minor).
void debug_source_order_keys(const uint32_t* touched, const ushort4* rect, const uint32_t* depth_key, int tiles_x,
                             int n, uint32_t* scratch_offsets, uint32_t* status, uint32_t* counter, uint32_t* total,
                             uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss, cudaStream_t st);

// ---- blend (raster.cu) ----
int blend_forward(const BlendArgs& a, cudaStream_t st);
int blend_backward(const BlendArgs& a, cudaStream_t st);
// FP32 pipe probe: returns achieved non-FMA fp32 op/s (FMUL + FADD, no contraction).
double fp32_peak_probe(cudaStream_t st);

}  // namespace fgs
