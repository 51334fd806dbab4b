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
  int vec_rot, vec_sh, vec_geo;  // rotations / sh / means+log_scales 16-byte aligned: LDG.128
  int32_t* rowdiff;      // tiles_y x (tiles_x + 1) row-difference tile counts
  int* error_flag;
  uint32_t* state_counts;  // [kept, degenerate]
};

struct PreprocessBackwardArgs {
  int64_t n;
  int64_t m;                 // Gaussians that touched >= 1 tile (level-1 compaction count)
  int64_t q_begin, q_end;    // this launch's slice of the compacted list (all: 0, m)
  int64_t id_begin, id_end;  // and the Gaussian-id range it writes (all: 0, n)
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
  int vec_rot;               // rotations 16-byte aligned: LDG.128
  const uint8_t* state;
  const uint32_t* touched;
  const uint32_t* coff;      // [m] first emission slot of cval[q]
  const float* partials;     // [I][9] K4a per-intersection sums by emission slot
  int64_t num_isect;         // I (bounds of partials, checked build)
  float* d_means;
  float* d_rotations;
  float* d_log_scales;
  float* d_opacity;
  float* d_sh;
  int aligned16;             // d_rotations and d_sh 16-byte aligned: float4 stores
};

struct BlendArgs {
  int width, height, tiles_x, tiles_y;
  int ellipse;                   // backward: exact ellipse-vs-block culling on top of the box test
  const uint32_t* tile_offsets;  // T+1
  uint32_t* sorted_gauss;        // I (written by the forward's per-tile sort, read by the backward)
  uint64_t* keys;                // forward: tile list keys (K2), sorted in place per tile
  const uint32_t* src_off;       // backward: first emission slot of each tile-touching Gaussian
  const ushort4* rect;           // backward: tile rectangle per Gaussian
  const SortedRec* rec;          // per-Gaussian records
  int64_t num_rec;               // records (rows of the TMA record tensor)
  float bg[3];
  float* image;                  // H*W*3
  float* final_T;                // H*W
  uint32_t* last;                // H*W: index one past the last contributing entry
  uint16_t* blend_count;         // optional H*W: contributions per pixel (FGS_FLAG_BLEND_COUNT / counters)
  unsigned long long* counters;  // optional: E_eval, E_contrib, culled evals, max CTA cycles
  unsigned long long* tile_cycles;  // optional (with counters): per-tile CTA cycles
  unsigned long long* tile_span;    // optional (with counters): per tile [start, end] %globaltimer (ns)
  const uint4* tile_sched;       // optional: CTA -> (tile, list begin, list end), heaviest lists first
  const uint32_t* scalars;       // forward: device scalars; exit if I > isect_cap (speculative launch)
  uint32_t* seg_cursor;          // forward: slot allocation cursor (scalars[kScalarSegPos])
  float* ckpt;                   // segment checkpoints [slot][4][256] (T, C0, C1, C2 per tile pixel)
  uint32_t* seg_items;           // [slot] tile | k << 16 (segment k >= 1 of tile), k = kSegFinal: final state
  uint32_t* tile_ckpt;           // [tile] first slot of a long list's checkpoints
  int64_t ckpt_cap;              // slots the checkpoint buffers hold
  int64_t num_seg_items;         // backward: slots of the frame (the first CTAs take the segments k >= 1)
  uint32_t* zero_next;           // forward: 16 scalars of the next frame, zeroed by CTA 0
  int64_t isect_cap;
  // backward
  const float* dl_dimage;
  float* partial_tile;           // I x 9 per-intersection sums by emission slot (K4a -> K4b)
};

// K1 / K4b launches (preprocess.cu); host_scene: the scene arrays are pinned host memory read in
// place over PCIe (separate instantiations, so profiles tell the two apart).
void preprocess_launch(const PreprocessArgs& a, bool host_scene, cudaStream_t st);
// fgs_crmath.cuh self-test (fgs_selftest_crmath): out_dev = u64[3] checked / mismatches / slow path
void crmath_selftest(int which, uint64_t begin, uint64_t count, uint64_t seed, unsigned long long* out_dev,
                     cudaStream_t st);
void preprocess_backward_launch(const PreprocessBackwardArgs& a, bool host_scene, int variant, cudaStream_t st);
constexpr int kPreprocessBackwardThreads = 128;  // tile-touching Gaussians per K4b CTA

// ---- binning / sorting (binning.cu) ----
#ifndef FGS_BIN_THREADS
#define FGS_BIN_THREADS 1024
#endif
#ifndef FGS_BIN_CTAS_PER_SM
#define FGS_BIN_CTAS_PER_SM 1
#endif
constexpr int kBinThreads = FGS_BIN_THREADS;          // K2 CTA size (experiment builds: 512 x 2 per SM)
constexpr int kBinCtasPerSm = FGS_BIN_CTAS_PER_SM;
constexpr int kScalarI = 0, kScalarErr = 1, kScalarKept = 2, kScalarDegen = 3, kScalarM = 4, kScalarI2 = 5, kScalarBig = 6,
              kScalarSegs = 7,    // backward segment slots of the frame (K2: sum over long lists of ceil(L / kSeg))
              kScalarSegPos = 8,  // K3's slot allocation cursor
              kScalarMaxList = 9, // longest tile list of the frame (K2)
              kScalarChunkQ = 10; // [kGradChunks - 1]: tile-touching Gaussians with id < c N / kGradChunks
// The backward's K4b can run as kGradChunks launches over Gaussian-id ranges [c N / C, (c+1) N / C)
// so that a multi-GPU step all-reduces each range's gradients while the next range is computed
// (fgs_fwd_bwd_views); K2 records where each range starts in the compacted list.
constexpr int kGradChunks = 4;
constexpr int kScalarReadback = kScalarChunkQ + kGradChunks - 1;  // scalars the host reads after K2
// The host's mapped copy of the scalars (one 64-byte block K2 writes): [0, kScalarReadback) the
// scalars, kHostHash a hash of them and the sequence number, kHostSeq the frame's sequence number.
constexpr int kHostBlock = 16, kHostHash = 14, kHostSeq = 15;
__host__ __device__ inline uint32_t host_block_hash_init(uint32_t seq) { return seq * 0x9E3779B1u + 0x7F4A7C15u; }
__host__ __device__ inline uint32_t host_block_hash_step(uint32_t h, uint32_t v) {
  h = (h ^ v) * 0x85EBCA6Bu;
  return h ^ (h >> 13);
}

// Backward segments: a tile list longer than kSeg entries is split into ceil(L / kSeg) segments
// that the blend backward processes as independent CTAs; the forward leaves each pixel's state
// (T and accumulated colour) at every segment boundary, plus its final (T, colour), in one
// checkpoint slot per segment (4 x 256 floats, SoA over the tile's pixels).
#ifndef FGS_SEG  // (experiment builds: 128 / 192 / 512 measured slower forward + backward at config 2)
#define FGS_SEG 256
#endif
constexpr int kSeg = FGS_SEG;
constexpr uint32_t kSegFinal = 0xFFFFu;  // item marker of a tile's final-state slot

struct BinArgs {
  int n;                       // Gaussians
  int tiles_x, tiles_y, num_tiles;
  int64_t isect_cap;           // capacity of the per-intersection buffers (the scatter is skipped if I exceeds it)
  int scatter_only;            // relaunch: phases 1-2 already ran
  int row_scatter;             // phase 3 by tile-row lists (large I) instead of source-order slots
  int fast;                    // slot order by CTA-local compaction (bin_local_kernel) when the scene fits
  unsigned long long* trace;   // debug phase timestamps (FGS_FLAG_COUNTERS), 8 slots
  const uint32_t* touched;     // [n] tiles touched per Gaussian (K1)
  const uint32_t* depth_key;   // [n] depth key bits (K1)
  const ushort4* rect;         // [n] tile rectangle (K1)
  int32_t* rowdiff;            // [tiles_y * (tiles_x + 1)] row-difference tile counts (K1 adds, bin_scan zeroes)
  uint32_t* cval;              // [n] tile-touching Gaussians in source order (compacted)
  uint32_t* coff;              // [n] their first emission slot
  uint32_t* src_off;           // [n] first emission slot by Gaussian id (tile-touching ones)
  uint32_t* scalars;           // device scalars (kScalar*)
  uint32_t* part_scan;         // [2 * grid] CTA partials, [64] schedule histogram + cursors, [tiles_y] row totals
  uint32_t* tile_offsets;      // [num_tiles + 1]
  uint32_t* fill;              // [num_tiles] scatter cursors
  uint4* tile_sched;           // [num_tiles] blend schedule: (tile, list begin, list end, 0)
  uint32_t* row_hist;          // [grid][tiles_y] per-CTA counts of (Gaussian, tile row) pairs
  // per intersection
  uint64_t* keys;              // [I] (depth_key << 32 | Gaussian id), grouped by tile
  uint32_t* row_list;          // [<= I] Gaussians per tile row (row-major), the scatter's work order
  uint32_t* host_scalars;      // mapped pinned memory: scalars[0, kScalarReadback) then seq at kHostSeq
  uint32_t seq;                // this frame's sequence number
};

// Words of part_scan scratch bin_scan needs; words of the per-CTA row histograms.
size_t bin_part_words(int tiles_y);
size_t bin_row_hist_words(int tiles_y);
constexpr int kMaxTileRows = 4096;  // binning keeps per-row state in shared memory
// K2 (one cooperative kernel): compaction + emission offsets + I and M (device scalars),
// tile ranges + blend schedule, key scatter into the tile ranges (skipped if I > isect_cap).
cudaError_t bin_launch(BinArgs& a, cudaStream_t st);
// Debug: the reference's pre-sort key list (source order).
cudaError_t debug_source_order_keys(BinArgs& a, uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss,
                                    cudaStream_t st);

// ---- blend (raster.cu) ----
int blend_forward(const BlendArgs& a, int64_t num_isect, int px_request, cudaStream_t st);
int blend_backward(const BlendArgs& a, int64_t num_isect, int variant, cudaStream_t st, int* px_used = nullptr);
// ---- training step (train.cu) ----
// L1 + D-SSIM loss and dL/drendered (inc/metrics.hpp:86-195). maps: loss_scratch_floats();
// partials: 2 * loss_partials() + 2 doubles, the last two = (sum of SSIM map, sum |x - y|).
size_t loss_scratch_floats(int width, int height);
size_t loss_partials(int width, int height);
int l1_dssim_loss(const float* rendered, const float* target, int width, int height, float lambda, float* d_rendered,
                  float* maps, double* partials, cudaStream_t st);

struct AdamArgs {  // groups: means, rotations, log_scales, opacities, sh
  float* p[5];
  const float* g[5];
  float* m[5];
  float* v[5];
  int64_t len[5];
  int width[5];  // floats per Gaussian: 3, 4, 3, 1, 48
  float lr[6];  // mean, rotation, log_scale, opacity, sh DC, sh higher bands
  float beta1, beta2, eps, bc1, bc2;
  int* nonfinite;  // min offending Gaussian index (INT_MAX = all finite)
};
int adam_check(AdamArgs& a, cudaStream_t st);
int adam_step(AdamArgs& a, cudaStream_t st);

// ---- brute-force validation renderer (bruteforce.cu), double precision ----
}  // namespace fgs
struct fgs_gaussians;
struct fgs_camera;
namespace fgs {
cudaError_t bruteforce_render(const ::fgs_gaussians& scene, const ::fgs_camera& cam, int sh_degree, const double bg[3],
                              double* image, double* transmittance, cudaStream_t st);
cudaError_t bruteforce_render_f64(int64_t n, const double* means, const double* rotations, const double* log_scales,
                                  const double* opacity, const double* sh, const ::fgs_camera& cam, int sh_degree,
                                  const double bg[3], double* image, double* transmittance, cudaStream_t st);

// FP32 pipe probe: returns achieved non-FMA fp32 op/s (FMUL + FADD, no contraction).
double fp32_peak_probe(cudaStream_t st);

}  // namespace fgs
