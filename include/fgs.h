/*
 * fgs.h — C ABI of the B200-native Fisheye-GS rasterizer (libfgs.so).
 *
 * Drop-in for the reference's render/backward path (omnisplat, a header-only C++ API):
 *   render<S>(scene, camera, options) -> {image, stats, context}
 *       /root/reference/proj/include/omnisplat/splatting.hpp:330-374
 *   backward<S>(scene, camera, context, dL/dimage, options) -> GradientBuffer
 *       /root/reference/proj/include/omnisplat/gradients.hpp:207-267
 * The reference has no FFI of its own; this header is what its C++ callers (cmd_render /
 * cmd_bench in src/cli.cpp:130,153; train in inc/optimize.hpp:247,264) bind instead, through
 * the C++ wrapper in include/fgs.hpp. See INTEGRATION.md.
 *
 * Conventions
 *  - fp32 throughout. Plain pointers + sizes; no CUDA or torch types in signatures
 *    (streams are passed as void* = cudaStream_t).
 *  - Scene layout (structure of arrays, one array per field, N Gaussians):
 *      means N*3, rotations N*4 (w,x,y,z, unnormalised), log_scales N*3,
 *      opacity_logits N, sh N*48 with per-Gaussian order [channel*16 + basis]
 *    (= the reference's Gaussian3D fields, inc/model.hpp:18-36, ShCoeffs column-major).
 *  - Image and dL/dimage: H*W*3 row-major RGB (ImageBuffer, inc/model.hpp:53-92).
 *  - Gradients: five arrays matching the scene fields; pointing them at consecutive blocks of
 *    one 59*N buffer (means, rotations, log_scales, opacities, sh) makes multi-view gradient
 *    sums a single all-reduce.
 *  - The forward state (ForwardContext, inc/splatting.hpp:309-321) lives in the context; one
 *    context serves one forward/backward pair at a time. Contexts are not thread-safe.
 *  - Errors are status codes; the C++ wrapper rethrows the reference's exception types.
 */
#ifndef FGS_H_
#define FGS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  FGS_OK = 0,
  FGS_EINVAL = 1,             /* bad shape / context-camera-scene mismatch (std::invalid_argument) */
  FGS_EDEGENERATE_QUAT = 2,   /* zero-norm quaternion (inc/model.hpp:98, "degenerate rotation") */
  FGS_ECUDA = 3,              /* CUDA runtime error */
  FGS_ENOMEM = 4,             /* device allocation failed */
  FGS_ESTATE = 5,             /* backward without a matching forward */
  FGS_ENONFINITE = 6          /* non-finite gradient in an Adam step (std::runtime_error) */
};

enum { FGS_CAMERA_PINHOLE = 0, FGS_CAMERA_FISHEYE = 1, FGS_CAMERA_PANORAMA = 2 };

/* Camera (inc/cameras.hpp:29-74): equidistant fisheye (the paper's model), pinhole, and
 * equirectangular panorama (fx..cy unused). */
typedef struct fgs_camera {
  int32_t model;
  int32_t width, height;
  float fx, fy, cx, cy;
  float rotation_wc[9];    /* row-major, world -> camera */
  float translation_wc[3];
  float fov_max;           /* culling half-angle; culled beyond fov_max + 10 deg */
} fgs_camera;

typedef struct fgs_gaussians {
  int64_t n;
  const float* means;
  const float* rotations;
  const float* log_scales;
  const float* opacity_logits;
  const float* sh;
} fgs_gaussians;

typedef struct fgs_gradients {
  float* d_means;            /* N*3 */
  float* d_rotations;        /* N*4 */
  float* d_log_scales;       /* N*3 */
  float* d_opacity_logits;   /* N   */
  float* d_sh;               /* N*48 */
} fgs_gradients;

/* RenderOptions (inc/splatting.hpp:50-55). */
typedef struct fgs_render_options {
  int32_t sh_degree;         /* 0..3 */
  int32_t use_background;    /* 0: scene background = black (the reference Scene default) */
  float background[3];
} fgs_render_options;

/* BackwardOptions (inc/gradients.hpp:57-63) plus build switches. */
typedef struct fgs_backward_options {
  float jacobian_grad_scale[3]; /* mutation hook; {1,1,1} normally */
  int32_t full_sh;              /* 1: all 48 SH gradients; 0: DC only (reference) */
  int32_t accumulate;           /* 1: add into the gradient arrays (multi-view sums) */
  int32_t sh_view_dir_grad;     /* 1: add colour -> view direction -> mean (the reference omits it,
                                   inc/gradients.hpp:255-262); 0 (default) = reference parity */
} fgs_backward_options;

/* RenderStats (inc/splatting.hpp:41-48); stage times from CUDA events. The per-tile sort runs
   inside the blend kernel: its time is part of raster_ms and sort_ms is 0. */
typedef struct fgs_stats {
  uint64_t num_intersections;
  uint32_t num_splats, num_culled, num_degenerate;
  double preprocess_ms, binning_ms, sort_ms, raster_ms;
  uint64_t peak_aux_bytes;
} fgs_stats;

typedef struct fgs_context fgs_context;

int fgs_create(int device, fgs_context** out);
int fgs_destroy(fgs_context* ctx);
/* Stream for all subsequent work (cudaStream_t; NULL = legacy default stream). Switching
   streams first waits for the work queued on the previous one (the context's buffers are
   reused by the next call). */
int fgs_set_stream(fgs_context* ctx, void* stream);
const char* fgs_last_error(const fgs_context* ctx);

/* Device-resident forward: all pointers are device memory. `radii` (N int32, 0 = culled or
 * degenerate) and `stats` may be NULL; a non-NULL `stats` synchronises the stream. */
int fgs_forward(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                const fgs_render_options* options, float* image, int32_t* radii, fgs_stats* stats);

/* Device-resident backward for the last forward of this context. */
int fgs_backward(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                 const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads);

/* Host-buffer variants with the reference's calling convention: inputs and outputs in host
 * memory, host<->device transfers included; blocking. Scene arrays in page-locked (pinned)
 * host memory are read in place over PCIe (zero copy: every Gaussian's geometry, the opacity
 * and SH rows only of the splats that survive the culls); pageable ones are copied whole. */
int fgs_render_host(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                    const fgs_render_options* options, float* image, int32_t* radii, fgs_stats* stats);
int fgs_backward_host(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                      const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads);

/* fgs_render_host for a stream of frames: returns once the frame is queued and its statistics
 * are known (the binning's scalars), with the image (and radii) still being read back on a copy
 * stream, so that the next frame's zero-copy scene reads (host -> device) overlap this frame's
 * read-back (device -> host). `image` / `radii` are valid after fgs_wait, or after the next
 * synchronous host call on this context; the scene arrays must stay unchanged until then. Two
 * frames' device images alternate, so a third call waits for the first one's read-back. */
int fgs_render_host_async(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                          const fgs_render_options* options, float* image, int32_t* radii, fgs_stats* stats);
/* fgs_backward_host for a stream of frames: returns once the backward is queued, the gradients
 * being read back on the copy stream (two device gradient buffers alternate); `grads` are valid
 * after fgs_wait or the next synchronous host call. */
int fgs_backward_host_async(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                            const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads);
/* Wait for every fgs_render_host_async / fgs_backward_host_async read-back of this context (and
 * order the context's stream after them). */
int fgs_wait(fgs_context* ctx);

/* A scene in array-of-structures form: n records of `stride` bytes in host memory, each holding
 * the float fields at the given byte offsets -- e.g. the reference's std::vector<Gaussian3D<float>>
 * (inc/model.hpp:18-36: mean 3, rotation 4 (w,x,y,z), log_scale 3, opacity_logit 1, sh 48 =
 * ShCoeffs column-major [channel*16 + basis]), described with offsetof() (include/fgs_omnisplat.hpp). */
typedef struct fgs_gaussians_aos {
  int64_t n;
  const void* data;
  int64_t stride;
  int64_t off_mean, off_rotation, off_log_scale, off_opacity_logit, off_sh;
} fgs_gaussians_aos;

/* fgs_render_host / fgs_backward_host for an AoS scene: the records go to the device in one
 * transfer and a gather kernel splits them into the structure-of-arrays layout. */
int fgs_render_host_aos(fgs_context* ctx, const fgs_gaussians_aos* scene, const fgs_camera* camera,
                        const fgs_render_options* options, float* image, int32_t* radii, fgs_stats* stats);
int fgs_backward_host_aos(fgs_context* ctx, const fgs_gaussians_aos* scene, const fgs_camera* camera,
                          const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads);

/* PCIe bytes moved by the last fgs_render_host / fgs_backward_host call: out = {h2d, d2h}. */
int fgs_last_transfer(const fgs_context* ctx, uint64_t out[2]);

/* Flags: FGS_FLAG_COUNTERS makes the forward blend count E_eval / E_contrib (atomics; slower)
 * and records the binning phase trace; FGS_FLAG_TIMING records CUDA events around every stage
 * (read with fgs_timing). FGS_FLAG_BLEND_COUNT makes the forward also write the per-pixel
 * contribution count (ForwardContext::blend_count, inc/splatting.hpp:299-301; debug name
 * "blend_count", u16[H*W]; also written with FGS_FLAG_COUNTERS). FGS_FLAG_ROW_SCATTER /
 * FGS_FLAG_SLOT_SCATTER force the binning scatter's work order (tile-row lists / source-order
 * emission slots; default: by the intersection count; same keys either way). On the slot order,
 * scenes of <= 148 x 8192 Gaussians take the CTA-local binning kernel; FGS_FLAG_GLOBAL_SLOTS forces
 * the global slot order instead (same outputs). FGS_FLAG_KEEP_KEYS is reserved (no effect).
 * Default 0. */
enum { FGS_FLAG_COUNTERS = 1, FGS_FLAG_KEEP_KEYS = 2, FGS_FLAG_TIMING = 4, FGS_FLAG_BLEND_COUNT = 8,
       FGS_FLAG_ROW_SCATTER = 16, FGS_FLAG_SLOT_SCATTER = 32, FGS_FLAG_GLOBAL_SLOTS = 64 };
int fgs_set_flags(fgs_context* ctx, uint32_t flags);

/* Device time per stage accumulated from CUDA events while FGS_FLAG_TIMING is set, and the
 * number of kernels this context launched, since the last reset:
 *   ms[0..5] = preprocess, binning, sort, raster, raster_backward, preprocess_backward;
 *   calls[0] = forward calls timed, calls[1] = backward calls timed. Synchronises. */
int fgs_timing(fgs_context* ctx, double ms[6], uint64_t calls[2], uint64_t* launches, int reset);

/* Diagnostic: FP32 pipe throughput (non-FMA fp32 op/s) of this device, measured with a
 * FMUL/FADD probe kernel; the denominator of the blend kernels' roofline. */
int fgs_measure_fp32_peak(fgs_context* ctx, double* ops_per_s);

/* Self-test of the fast correctly rounded exp / atan2 K1 and K4b use (csrc/fgs_crmath.cuh) against
 * their definition (fp32 rounding of the double evaluation): which 0 = exp over the fp32 bit
 * patterns [begin, begin + count); 1 = atan2 over `count` seeded pairs of random bit patterns;
 * 2 = atan2 over seeded pairs of the camera domain. out = {checked, mismatches, slow-path count}.
 * Synchronises. */
int fgs_selftest_crmath(fgs_context* ctx, int which, uint64_t begin, uint64_t count, uint64_t seed, uint64_t out[3]);

/* Parity/debug export of the last forward's state into host memory. Names:
 *   "state_u8" u8[N] (0 culled, 1 kept, 2 degenerate), "rec" f32[N*12] (splat records: mean_px,
 *   -conic.a/2, conic.b, -conic.c/2, alpha_max, colour, extent), "depth_key" u32[N], "radius" int32[N], "touched" u32[N],
 *   "key_tile"/"key_depth"/"key_gauss" u32[I] (pre-sort keys in the reference's emission order),
 *   "sorted_gauss" u32[I], "sorted_tile" u32[I], "offsets" u32[T+1] (tile ranges),
 *   "keys" u64[I] (depth key << 32 | Gaussian id, as the binning scatter wrote them into each tile's
 *   range), "rect" u16[N*4] (tile rectangle tx0, tx1, ty0, ty1 per Gaussian), "variants" u32[5]
 *   (forward pixels per lane, backward pixels per lane, K4b CTAs per SM, longest tile list, binning
 *   scatter by tile-row lists),
 *   "aux_bytes" u64[1] (device bytes the render/backward path holds, backward scratch included),
 *   "compact_gauss"/"compact_offsets" u32[M], "final_T" f32[H*W], "last" u32[H*W],
 *   "counters" u64[4] (E_eval, E_contrib, culled evaluations, max CTA cycles; with
 *   FGS_FLAG_COUNTERS), "counters16" u64[16], "bin_trace" u64[8], "tile_cycles" u64[T],
 *   "tile_span" / "tile_span_bwd" u64[2T] (per tile CTA start / end %globaltimer ns of the last forward
 *   / backward blend; with FGS_FLAG_COUNTERS).
 * Returns the number of bytes (dst may be NULL to query), or -1 for an unknown name. */
int64_t fgs_debug_get(fgs_context* ctx, const char* name, void* dst, int64_t dst_bytes);

/* ---- Training step: inc/metrics.hpp:86-195, inc/optimize.hpp:100-277 ---- */

/* L = (1 - lambda) L1 + lambda (1 - SSIM) of `rendered` against `target` (device H*W*3 each,
 * 11x11 Gaussian-window SSIM, zero padding); writes dL/drendered (device H*W*3) and
 * out[3] = {total, l1, dssim} (host). Synchronises. */
int fgs_l1_dssim_loss(fgs_context* ctx, const float* rendered, const float* target, int32_t width, int32_t height,
                      float lambda, float* d_rendered, double out[3]);

/* Mutable scene parameters (device arrays, the fgs_gaussians layout). */
typedef struct fgs_params {
  int64_t n;
  float* means;
  float* rotations;
  float* log_scales;
  float* opacity_logits;
  float* sh;
} fgs_params;

/* AdamParams + GroupLearningRates (inc/optimize.hpp:72-97). lr_sh_rest (SH bands 1..3) is a
 * build extension: the reference optimises the DC only; 0 reproduces that. */
typedef struct fgs_adam_options {
  float lr_mean, lr_rotation, lr_log_scale, lr_opacity, lr_sh_dc, lr_sh_rest;
  float beta1, beta2, eps;  /* 0.9, 0.999, 1e-15 in the reference */
} fgs_adam_options;

/* AdamState (inc/optimize.hpp:78-90): step count and first/second moments, device arrays in
 * the gradient layout (zero-initialised by the caller, step = 0). */
typedef struct fgs_adam_state {
  int64_t step;
  fgs_gradients m, v;
} fgs_adam_state;

/* adam_step (inc/optimize.hpp:115-145) on device arrays. A non-finite gradient in an updated
 * group returns FGS_ENONFINITE and changes nothing (the reference throws before updating). */
int fgs_adam_step(fgs_context* ctx, fgs_params* params, const fgs_gradients* grads, fgs_adam_state* state,
                  const fgs_adam_options* options);

typedef struct fgs_train_options {
  int32_t sh_degree;
  float background[3];
  float lambda;             /* loss_lambda, 0.2 in the reference */
  fgs_adam_options adam;
} fgs_train_options;

/* One iteration of the reference's train loop body (inc/optimize.hpp:237-266): render the
 * view, L1 + D-SSIM loss against `target` (device H*W*3), backward, Adam step -- all on the
 * device, parameters updated in place. loss_out = {total, l1, dssim}. */
int fgs_train_step(fgs_context* ctx, fgs_params* params, const fgs_camera* camera, const float* target,
                   const fgs_train_options* options, fgs_adam_state* state, double loss_out[3]);

/* ---- Validation ---- */

/* The reference's brute-force renderer (inc/oracle.hpp:161-270) on the GPU in double: every
 * splat in global (depth, source) order gated per 16x16 tile, with an independent projection /
 * covariance / SH transcription (no code shared with the fast path). Scene: device fp32 arrays
 * (cast to double); image: device double H*W*3; transmittance: device double H*W or NULL.
 * Synchronises. For large-scene checks of fgs_forward and for finite-difference gradchecks. */
int fgs_bruteforce_render(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera, int32_t sh_degree,
                          const double background[3], double* image, double* transmittance);
/* Same with a double-precision scene (device arrays in the fgs_gaussians layout): the
 * finite-difference gradcheck (inc/oracle.hpp:338-418) perturbs parameters in double. */
int fgs_bruteforce_render_f64(fgs_context* ctx, int64_t n, const double* means, const double* rotations,
                              const double* log_scales, const double* opacity_logits, const double* sh,
                              const fgs_camera* camera, int32_t sh_degree, const double background[3], double* image,
                              double* transmittance);

/* ---- Multi-GPU: views partitioned by camera, Gaussians replicated, the
 * per-Gaussian gradients summed over the GPUs with one NCCL all-reduce (NCCL is loaded at first
 * use; libfgs.so itself does not depend on it). ---- */
typedef struct fgs_comm fgs_comm;

/* One rank per process: rank 0 creates the 128-byte id and shares it out of band (MPI,
 * torch.distributed, a file); every rank then joins with its context (device and stream). */
int fgs_comm_get_unique_id(uint8_t id[128]);
int fgs_comm_init(fgs_context* ctx, const uint8_t id[128], int nranks, int rank, fgs_comm** out);
/* One process driving ndev devices (ncclCommInitAll): one communicator per context. */
int fgs_comm_init_all(fgs_context* const* ctxs, int ndev, fgs_comm** comms);
int fgs_comm_destroy(fgs_comm* comm);

/* In-place sum over the ranks of the five gradient arrays of n Gaussians (device memory), ordered
 * on the context's stream. */
int fgs_allreduce_gradients(fgs_comm* comm, fgs_gradients* grads, int64_t n);

/* The multi-view step of one rank: forward + backward of its `nviews` cameras (dl_dimages[v] and
 * images[v], device H*W*3 each; images may be NULL), the gradients accumulated into `grads` (the
 * first view overwrites unless options->accumulate), then -- with a communicator -- summed over
 * the ranks: the last view's preprocess backward runs in 4 Gaussian-id ranges and each range's
 * all-reduce starts on a communication stream as soon as the range is written, overlapping the
 * next range. comm = NULL: single GPU, no collective. Asynchronous on the context's stream. */
int fgs_fwd_bwd_views(fgs_context* ctx, fgs_comm* comm, const fgs_gaussians* scene, const fgs_camera* cameras,
                      int nviews, const float* const* dl_dimages, const fgs_render_options* render_options,
                      const fgs_backward_options* backward_options, fgs_gradients* grads, float* const* images);

/* Counters of the last forward: [n, num_splats, num_intersections, tiles_x, tiles_y, width, height,
 * num_culled, num_degenerate]. */
int fgs_last_counts(const fgs_context* ctx, int64_t out[9]);

#ifdef __cplusplus
}
#endif

#endif /* FGS_H_ */
