// fgs_api.cu — the C ABI (include/fgs.h): context, device memory, stage orchestration.
//
// Forward (reference render, inc/splatting.hpp:330-374):
//   K1 preprocess (+ per-tile counts) -> K2 (cooperative): emission offsets, I, tile ranges,
//   schedule, key scatter into the tile ranges -> K3 per-tile sort + blend. The host reads I
//   (32 bytes) after K2 while K3 already runs against the buffers' capacity.
// Backward (reference backward, inc/gradients.hpp:207-267):
//   K4a reverse blend (per-intersection partials) -> K4b preprocess backward.

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fgs.h"
#include "fgs_kernels.h"

namespace {

template <typename T>
struct DevBuf {  // owning device allocation that only grows (freed on destruction)
  T* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  cudaError_t ensure(size_t n) {
    if (n <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = n + n / 4 + 64;
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      return e;
    }
    cap = want;
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

// Launch-variant rules. Where two work decompositions give identical results, the choice is a
// deterministic function of the frame's statistics (no timing-based tuning, so a run's numbers
// reproduce): the intersection count I, the tile count T and the longest tile list. Measured
// at the BASELINE configs (profiles/r02_variants.md):
//   forward blend, pixels per lane: 2 amortises the per-splat work over twice the pixels and
//     wins on even lists (configs 1, 3, 4); a heavy-tailed frame (longest list > 8x the mean and
//     > 512, config 2) is bound by its longest lists, which 1 pixel per lane spreads over twice
//     the warps;
//   both blends take 1 pixel per lane on small images (< 1024 tiles, config 0: fewer CTAs than
//     a few waves over the 148 SMs);
//   backward blend: 2 pixels per lane from 32 entries per tile on average, at 6 CTAs per SM;
//   K4b: 6 CTAs per SM (80 registers) for scenes with > 1M tile-touching Gaussians, else 4 (85).
// FGS_FWD_PX / FGS_BWD_PX / FGS_BWD_MINB / FGS_K4B_MINB override (profiling).
namespace {
int env_int(const char* name) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : 0;
}
int rule_fwd_px(int64_t I, int64_t tiles, int64_t longest) {
  static const int e = env_int("FGS_FWD_PX");
  if (e == 1 || e == 2) return e;
  const int64_t mean = tiles > 0 ? I / tiles : 0;
  if (tiles < 1024) return 1;  // a small image: fewer CTAs than a few waves, use every warp
  return (longest > 512 && longest > 8 * std::max<int64_t>(mean, 1)) ? 1 : 2;
}
int rule_row_scatter(int64_t I) {
  static const int e = env_int("FGS_ROW_SCATTER");
  if (e == 1 || e == 2) return e == 1;
  return I > 2000000 ? 1 : 0;
}
// K2 on the slot order: bin_local_kernel (each CTA compacts and scatters its own range of
// Gaussians from shared memory) for scenes of <= 148 x 8192 Gaussians; FGS_BIN_FAST=1 takes
// bin_kernel's global slot order (intersection-balanced ranges, global rank search).
int rule_bin_fast() {
  static const int e = env_int("FGS_BIN_FAST");
  return e == 1 ? 0 : 1;
}
int rule_k4b_minb(int64_t m) {
  static const int e = env_int("FGS_K4B_MINB");
  if (e == 4 || e == 6) return e;
  return m > 1000000 ? 6 : 4;
}
}  // namespace

struct fgs_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t flags = 0;
  std::string err;

  // per Gaussian
  DevBuf<fgs::SortedRec> rec;
  DevBuf<uint8_t> state;
  DevBuf<uint32_t> dkey, cval, coff, src_off, touched, scan_status;
  DevBuf<ushort4> rect;
  DevBuf<int32_t> radii;
  // per intersection
  DevBuf<uint64_t> keys;
  DevBuf<uint32_t> sorted_gauss, row_list, row_hist;
  DevBuf<float> ckpt;             // backward segments: forward checkpoints [slot][4][256]
  DevBuf<uint32_t> seg_items, tile_ckpt;
  int64_t ckpt_cap = 0;           // slots of ckpt / seg_items
  int64_t num_segs = 0;           // slots of the last forward
  DevBuf<float> partial_tile;     // backward: 9 screen-space gradient sums per intersection
  // training step
  DevBuf<float> t_image, t_dimage, t_grads, t_maps;
  DevBuf<double> t_part;
  DevBuf<int> t_flag;
  // per tile / pixel
  DevBuf<uint32_t> tile_offsets, fill, last;
  DevBuf<uint4> tile_sched;
  DevBuf<int32_t> rowdiff;  // zero between frames (K2 zeroes what K1 added)
  size_t rowdiff_clean = 0; // entries known to be zero
  int64_t isect_cap = 0;    // capacity of the per-intersection buffers
  cudaEvent_t ev_k2 = nullptr;    // K2 done on the caller's stream (error detection while waiting)
  uint32_t* d_hscalars = nullptr; // device view of h_scalars (mapped pinned memory K2 writes)
  uint32_t frame_seq = 0;         // K2 writes it to h_scalars[kHostSeq] after the scalars
  uint32_t longest = 0;     // longest tile list of the last forward
  int var_fwd_px = 0, var_bwd_px = 0, var_k4b = 0, var_row_scatter = 0, var_bin_local = 0;  // launch variants (reported)
  // The device scalars alternate between two 16-word halves by frame parity; a frame's K3 zeroes
  // the other half for the next frame (whose previous readback finished before this frame began),
  // so no memset precedes K1. scalars_clean[h]: half h is known to be zero.
  int64_t frame = 0;
  bool scalars_clean[2] = {true, true};
  DevBuf<float> final_T;
  DevBuf<uint16_t> blend_count;  // per pixel (FGS_FLAG_BLEND_COUNT)
  bool have_blend_count = false;
  // misc device scalars: [0] total I, [1] error flag, [2..3] state counts, [4] compacted count M,
  // [5] scan tile counter
  DevBuf<uint32_t> scalars;
  DevBuf<unsigned long long> counters, tile_cycles, tile_span, tile_span_bwd;
  uint32_t* h_scalars = nullptr;  // pinned, mapped: the frame's scalars, written by K2 over PCIe
  // host-call staging
  DevBuf<float> h_means, h_rot, h_ls, h_op, h_sh, h_img, h_dl, h_grad;
  DevBuf<uint8_t> h_aos;  // AoS scene upload (fgs_*_host_aos)
  DevBuf<int32_t> h_radii;
  // fgs_render_host_async: device images / radii double-buffered by frame parity, read back on
  // a copy stream (created on first use) while the next frame runs on the caller's stream
  DevBuf<float> a_img[2];
  DevBuf<int32_t> a_radii[2];
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ev_rendered = nullptr, ev_copied[2] = {nullptr, nullptr};
  bool copy_recorded[2] = {false, false};
  int async_parity = 0, async_last = -1;
  // fgs_backward_host_async: device gradients double-buffered, read back on the copy stream
  DevBuf<float> a_grad[2];
  cudaEvent_t ev_bdone = nullptr, ev_gcopied[2] = {nullptr, nullptr};
  bool gcopy_recorded[2] = {false, false};
  int gasync_parity = 0, gasync_last = -1;
  cudaEvent_t ev[5] = {};
  // stage timing (FGS_FLAG_TIMING): event sets pending accumulation
  struct EventSet {
    cudaEvent_t e[5];
    int kind;  // 0 forward (4 intervals -> ms[0..3]), 1 backward (2 intervals -> ms[4..5])
  };
  std::vector<EventSet> pending, spare;
  double acc_ms[6] = {0, 0, 0, 0, 0, 0};
  uint64_t acc_calls[2] = {0, 0};
  uint64_t launches = 0;

  // last forward
  bool have_fwd = false;
  int64_t n = 0;
  fgs_camera cam{};
  int sh_degree = 3;
  float bg[3] = {0, 0, 0};
  fgs::DevCamera dcam{};
  int tiles_x = 0, tiles_y = 0;
  int64_t num_isect = 0;
  int64_t num_compact = 0;  // Gaussians touching >= 1 tile (rows the backward computes)
  int64_t chunk_q[fgs::kGradChunks + 1] = {};  // compacted-list position of each gradient-chunk boundary
  uint32_t num_splats = 0, num_degenerate = 0, num_culled = 0;
  size_t aux_bytes = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;  // PCIe bytes of the last host-buffer call
  bool scene_on_host = false;  // the scene arrays of the current call are pinned host memory
  fgs::BinArgs bin_args{};
};

namespace {

// NVTX ranges around the public calls and markers at each stage launch (header-only NVTX 3: a
// few nanoseconds when no tool is attached), so an nsys / ncu timeline shows the path's stages.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int fail(fgs_context* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(fgs_context* c, cudaError_t e, const char* where) {
  return fail(c, e == cudaErrorMemoryAllocation ? FGS_ENOMEM : FGS_ECUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define FGS_CHECK(expr)                                   \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr); \
  } while (0)

fgs::DevCamera make_dev_camera(const fgs_camera& c) {
  fgs::DevCamera d{};
  d.model = c.model;
  d.width = c.width;
  d.height = c.height;
  d.fx = c.fx; d.fy = c.fy; d.cx = c.cx; d.cy = c.cy;
  for (int i = 0; i < 9; ++i) d.W[i] = c.rotation_wc[i];
  for (int i = 0; i < 3; ++i) d.b[i] = c.translation_wc[i];
  d.fov_max = c.fov_max;
  // center = -W^T b (inc/cameras.hpp:60), summed left to right in float, no contraction
  for (int r = 0; r < 3; ++r) {
    volatile float acc = (-c.rotation_wc[0 * 3 + r]) * c.translation_wc[0];
    volatile float t1 = (-c.rotation_wc[1 * 3 + r]) * c.translation_wc[1];
    acc = acc + t1;
    volatile float t2 = (-c.rotation_wc[2 * 3 + r]) * c.translation_wc[2];
    acc = acc + t2;
    d.center[r] = acc;
  }
  return d;
}

fgs_context::EventSet* take_set(fgs_context* ctx, int kind) {
  fgs_context::EventSet es{};
  if (!ctx->spare.empty()) {
    es = ctx->spare.back();
    ctx->spare.pop_back();
  } else {
    for (auto& e : es.e) cudaEventCreate(&e);
  }
  es.kind = kind;
  ctx->pending.push_back(es);
  return &ctx->pending.back();
}

// Device bytes the render/backward path holds (RenderStats::peak_aux_bytes): per-Gaussian and
// per-intersection state, tile and pixel arrays, and the backward's scratch once allocated.
template <typename T>
size_t cap_bytes(const DevBuf<T>& b) { return b.p ? b.cap * sizeof(T) : 0; }
size_t path_bytes(const fgs_context* c) {
  return cap_bytes(c->rec) + cap_bytes(c->state) + cap_bytes(c->dkey) + cap_bytes(c->cval) + cap_bytes(c->coff) +
         cap_bytes(c->src_off) + cap_bytes(c->touched) + cap_bytes(c->scan_status) + cap_bytes(c->rect) +
         cap_bytes(c->radii) + cap_bytes(c->keys) + cap_bytes(c->sorted_gauss) + cap_bytes(c->row_list) + cap_bytes(c->row_hist) + cap_bytes(c->ckpt) + cap_bytes(c->seg_items) + cap_bytes(c->tile_ckpt) +
         cap_bytes(c->partial_tile) + cap_bytes(c->tile_offsets) + cap_bytes(c->fill) + cap_bytes(c->last) +
         cap_bytes(c->tile_sched) + cap_bytes(c->rowdiff) + cap_bytes(c->final_T);
}

// Checkpoint slots for X backward segments (grows only).
cudaError_t ensure_ckpt(fgs_context* c, int64_t X) {
  if (X <= c->ckpt_cap && c->ckpt.p) return cudaSuccess;
  const size_t slots = static_cast<size_t>(std::max<int64_t>(X, 1));
  cudaError_t e = c->ckpt.ensure(slots * 4 * fgs::kTile * fgs::kTile);
  if (e == cudaSuccess) e = c->seg_items.ensure(slots);
  if (e != cudaSuccess) return e;
  c->ckpt_cap = static_cast<int64_t>(std::min(c->ckpt.cap / (4 * fgs::kTile * fgs::kTile), c->seg_items.cap));
  return cudaSuccess;
}

// An event set taken by a call that then fails returns to the spare pool unread (its later events
// were never recorded): error paths leave no pending interval behind.
struct SetGuard {
  fgs_context* ctx;
  bool armed;
  ~SetGuard() {
    if (armed && !ctx->pending.empty()) {
      ctx->spare.push_back(ctx->pending.back());
      ctx->pending.pop_back();
    }
  }
};

void drain_sets(fgs_context* ctx, size_t keep) {
  while (ctx->pending.size() > keep) {
    fgs_context::EventSet es = ctx->pending.front();
    ctx->pending.erase(ctx->pending.begin());
    const int nint = es.kind == 0 ? 4 : 2;
    cudaEventSynchronize(es.e[nint]);
    for (int k = 0; k < nint; ++k) {
      float ms = 0.0f;
      if (es.kind == 0 && k == 2) continue;  // forward: the sort runs inside K3 (no event 3)
      if (cudaEventElapsedTime(&ms, es.e[es.kind == 0 && k == 3 ? 2 : k], es.e[k + 1]) != cudaSuccess) {
        cudaGetLastError();  // an interval of a failed call: not counted, and no sticky error left
        continue;
      }
      ctx->acc_ms[(es.kind == 0 ? 0 : 4) + k] += ms;
    }
    ctx->acc_calls[es.kind] += 1;
    ctx->spare.push_back(es);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool same_camera(const fgs_camera& a, const fgs_camera& b) {
  // the fields the reference compares (inc/gradients.hpp:213-217)
  if (a.model != b.model || a.width != b.width || a.height != b.height || a.fx != b.fx || a.fy != b.fy ||
      a.cx != b.cx || a.cy != b.cy)
    return false;
  for (int i = 0; i < 9; ++i)
    if (a.rotation_wc[i] != b.rotation_wc[i]) return false;
  for (int i = 0; i < 3; ++i)
    if (a.translation_wc[i] != b.translation_wc[i]) return false;
  return true;
}

}  // namespace

namespace {
// The copy stream of the asynchronous host calls and its events (created on first use).
cudaError_t ensure_copy_stream(fgs_context* ctx) {
  if (ctx->copy_st) return cudaSuccess;
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->copy_st, cudaStreamNonBlocking);
  for (cudaEvent_t* ev : {&ctx->ev_rendered, &ctx->ev_bdone, &ctx->ev_copied[0], &ctx->ev_copied[1],
                          &ctx->ev_gcopied[0], &ctx->ev_gcopied[1]})
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  return e;
}
}  // namespace

namespace {
// Wait for K2's scalars of this frame in the mapped h_scalars (sequence number in kHostSeq),
// watching K2's completion event for errors.
bool host_block_ready(fgs_context* ctx) {
  const volatile uint32_t* hs = ctx->h_scalars;
  if (hs[fgs::kHostSeq] != ctx->frame_seq) return false;
  std::atomic_thread_fence(std::memory_order_acquire);
  uint32_t h = fgs::host_block_hash_init(ctx->frame_seq);
  for (int t = 0; t < fgs::kScalarReadback; ++t) h = fgs::host_block_hash_step(h, hs[t]);
  return h == hs[fgs::kHostHash] && hs[fgs::kHostSeq] == ctx->frame_seq;
}
int wait_host_scalars(fgs_context* ctx) {
  for (uint64_t it = 0;; ++it) {
    if (host_block_ready(ctx)) return FGS_OK;
    if ((it & 1023) == 1023) {
      const cudaError_t q = cudaEventQuery(ctx->ev_k2);
      if (q == cudaSuccess) {  // K2 is done: its writes are visible
        if (host_block_ready(ctx)) return FGS_OK;
        return fail(ctx, FGS_ECUDA, "forward: binning finished without publishing its scalars");
      }
      if (q != cudaErrorNotReady) return fail(ctx, FGS_ECUDA, cudaGetErrorString(q));
    }
  }
}
}  // namespace

extern "C" {

int fgs_create(int device, fgs_context** out) {
  if (!out) return FGS_EINVAL;
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return FGS_ECUDA;
  auto* ctx = new fgs_context();
  ctx->device = device;
  e = cudaHostAlloc(&ctx->h_scalars, 32 * sizeof(uint32_t), cudaHostAllocMapped);
  if (e == cudaSuccess) {
    std::memset(ctx->h_scalars, 0, 32 * sizeof(uint32_t));
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->d_hscalars), ctx->h_scalars, 0);
  }
  if (e != cudaSuccess) {
    delete ctx;
    return FGS_ECUDA;
  }
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  cudaEventCreateWithFlags(&ctx->ev_k2, cudaEventDisableTiming);
  if (ctx->scalars.ensure(32) != cudaSuccess || cudaMemset(ctx->scalars.p, 0, 32 * sizeof(uint32_t)) != cudaSuccess || ctx->counters.ensure(24) != cudaSuccess ||
      false) {
    fgs_destroy(ctx);
    return FGS_ENOMEM;
  }
  *out = ctx;
  return FGS_OK;
}

int fgs_destroy(fgs_context* ctx) {
  if (ctx && ctx->copy_st) {
    cudaStreamSynchronize(ctx->copy_st);
    cudaStreamDestroy(ctx->copy_st);
    cudaEventDestroy(ctx->ev_rendered);
    cudaEventDestroy(ctx->ev_bdone);
    for (auto& e : ctx->ev_copied) cudaEventDestroy(e);
    for (auto& e : ctx->ev_gcopied) cudaEventDestroy(e);
  }
  if (!ctx) return FGS_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  else cudaDeviceSynchronize();
  for (auto* b : {&ctx->final_T, &ctx->partial_tile, &ctx->ckpt, &ctx->t_image, &ctx->t_dimage, &ctx->t_grads,
                  &ctx->t_maps, &ctx->h_means, &ctx->h_rot, &ctx->h_ls, &ctx->h_op,
                  &ctx->h_sh, &ctx->h_img, &ctx->h_dl, &ctx->h_grad})
    b->release();
  ctx->rec.release();
  ctx->state.release();
  for (auto* b : {&ctx->dkey, &ctx->cval, &ctx->coff, &ctx->src_off, &ctx->touched, &ctx->scan_status,
                  &ctx->sorted_gauss, &ctx->row_list, &ctx->row_hist, &ctx->seg_items, &ctx->tile_ckpt, &ctx->tile_offsets, &ctx->fill, &ctx->last,
                  &ctx->scalars})
    b->release();
  ctx->tile_sched.release();
  ctx->keys.release();
  ctx->t_part.release();
  ctx->t_flag.release();
  ctx->rowdiff.release();
  ctx->rect.release();
  ctx->radii.release();
  ctx->h_radii.release();
  for (int k = 0; k < 2; ++k) {
    ctx->a_img[k].release();
    ctx->a_radii[k].release();
    ctx->a_grad[k].release();
  }
  ctx->counters.release();
  ctx->tile_cycles.release();
  ctx->blend_count.release();
  ctx->h_aos.release();
  ctx->tile_span.release();
  ctx->tile_span_bwd.release();
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->ev_k2) cudaEventDestroy(ctx->ev_k2);
  for (auto* v : {&ctx->pending, &ctx->spare})
    for (auto& es : *v)
      for (auto& e : es.e) cudaEventDestroy(e);
  if (ctx->h_scalars) cudaFreeHost(ctx->h_scalars);
  delete ctx;
  return FGS_OK;
}

int fgs_set_stream(fgs_context* ctx, void* stream) {
  if (!ctx) return FGS_EINVAL;
  const cudaStream_t next = static_cast<cudaStream_t>(stream);
  if (next != ctx->stream) {
    // the context's buffers (records, keys, scalars, ...) are reused by the next call: work
    // still queued on the old stream must finish before the new stream may touch them
    FGS_CHECK(cudaSetDevice(ctx->device));
    FGS_CHECK(cudaStreamSynchronize(ctx->stream));
    ctx->stream = next;
  }
  return FGS_OK;
}

int fgs_set_flags(fgs_context* ctx, uint32_t flags) {
  if (!ctx) return FGS_EINVAL;
  ctx->flags = flags;
  return FGS_OK;
}

const char* fgs_last_error(const fgs_context* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int fgs_last_counts(const fgs_context* ctx, int64_t out[9]) {
  if (!ctx || !out) return FGS_EINVAL;
  out[0] = ctx->n;
  out[1] = ctx->num_splats;
  out[2] = ctx->num_isect;
  out[3] = ctx->tiles_x;
  out[4] = ctx->tiles_y;
  out[5] = ctx->cam.width;
  out[6] = ctx->cam.height;
  out[7] = ctx->num_culled;
  out[8] = ctx->num_degenerate;
  return FGS_OK;
}

// Exact ellipse culling in the blends (FGS_ELLIPSE=0 turns it off; profiling switch).
static int blend_ellipse() {
  static const int v = [] {
    const char* e = std::getenv("FGS_ELLIPSE");
    return e && *e ? std::atoi(e) : 1;
  }();
  return v;
}

int fgs_forward(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                const fgs_render_options* options, float* image, int32_t* radii, fgs_stats* stats) {
  if (!ctx) return FGS_EINVAL;
  NvtxRange nvtx("fgs.forward");
  if (!scene || !camera || !image) return fail(ctx, FGS_EINVAL, "forward: null argument");
  if (camera->model != FGS_CAMERA_FISHEYE && camera->model != FGS_CAMERA_PINHOLE &&
      camera->model != FGS_CAMERA_PANORAMA)
    return fail(ctx, FGS_EINVAL, "forward: unknown camera model");
  if (camera->width <= 0 || camera->height <= 0) return fail(ctx, FGS_EINVAL, "forward: empty image");
  if ((static_cast<int64_t>(camera->width) + 15) / 16 * ((static_cast<int64_t>(camera->height) + 15) / 16) > 65536)
    return fail(ctx, FGS_EINVAL, "forward: more than 65536 tiles");
  if ((camera->height + 15) / 16 > fgs::kMaxTileRows)
    return fail(ctx, FGS_EINVAL, "forward: more than 4096 tile rows (image taller than 65536 pixels)");
  const int sh_degree = options ? options->sh_degree : 3;
  if (sh_degree < 0 || sh_degree > 3) return fail(ctx, FGS_EINVAL, "forward: sh_degree must be 0..3");
  const int64_t n = scene->n;
  if (n < 0 || n >= (int64_t(1) << 31)) return fail(ctx, FGS_EINVAL, "forward: scene size out of range");
  if (n > 0 && (!scene->means || !scene->rotations || !scene->log_scales || !scene->opacity_logits || !scene->sh))
    return fail(ctx, FGS_EINVAL, "forward: null scene array");
  FGS_CHECK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  ctx->have_fwd = false;

  const int W = camera->width, H = camera->height;
  const int tiles_x = (W + fgs::kTile - 1) / fgs::kTile, tiles_y = (H + fgs::kTile - 1) / fgs::kTile;
  const int num_tiles = tiles_x * tiles_y;
  const size_t nn = static_cast<size_t>(n > 0 ? n : 1);
  const size_t npix = static_cast<size_t>(W) * H;
  FGS_CHECK(ctx->rec.ensure(nn));
  FGS_CHECK(ctx->state.ensure(nn));
  for (auto* b : {&ctx->dkey, &ctx->cval, &ctx->coff, &ctx->src_off, &ctx->touched}) FGS_CHECK(b->ensure(nn));
  const size_t part_words = fgs::bin_part_words(tiles_y);
  if (ctx->scan_status.cap < part_words) {
    FGS_CHECK(ctx->scan_status.ensure(part_words));
    ctx->rowdiff_clean = 0;  // forces the scratch memsets below
  }
  FGS_CHECK(ctx->rect.ensure(nn));
  FGS_CHECK(ctx->radii.ensure(nn));
  FGS_CHECK(ctx->tile_offsets.ensure(num_tiles + 1));
  FGS_CHECK(ctx->fill.ensure(num_tiles));
  FGS_CHECK(ctx->tile_sched.ensure(num_tiles));
  FGS_CHECK(ctx->tile_ckpt.ensure(num_tiles));
  FGS_CHECK(ctx->row_hist.ensure(std::max<size_t>(fgs::bin_row_hist_words(tiles_y), 1)));
  const size_t ndiff = static_cast<size_t>(tiles_x + 1) * tiles_y;
  if (ctx->rowdiff.cap < ndiff || ctx->rowdiff_clean < ndiff) {
    FGS_CHECK(ctx->rowdiff.ensure(ndiff));
    FGS_CHECK(cudaMemsetAsync(ctx->rowdiff.p, 0, ctx->rowdiff.cap * sizeof(int32_t), ctx->stream));
    FGS_CHECK(cudaMemsetAsync(ctx->scan_status.p, 0, ctx->scan_status.cap * sizeof(uint32_t), ctx->stream));
    ctx->rowdiff_clean = ctx->rowdiff.cap;
  }
  FGS_CHECK(ctx->last.ensure(npix));
  FGS_CHECK(ctx->final_T.ensure(npix));

  ctx->n = n;
  ctx->cam = *camera;
  ctx->sh_degree = sh_degree;
  for (int k = 0; k < 3; ++k) ctx->bg[k] = (options && options->use_background) ? options->background[k] : 0.0f;
  ctx->dcam = make_dev_camera(*camera);
  ctx->tiles_x = tiles_x;
  ctx->tiles_y = tiles_y;

  const bool timing = stats != nullptr || (ctx->flags & FGS_FLAG_TIMING);
  if (ctx->pending.size() > 64) drain_sets(ctx, 8);
  cudaEvent_t* ev = timing ? take_set(ctx, 0)->e : ctx->ev;
  SetGuard guard{ctx, timing};
  if (timing) cudaEventRecord(ev[0], st);
  uint64_t launches = 0;

  const int half = static_cast<int>(ctx->frame++ & 1);
  uint32_t* scalars = ctx->scalars.p + 16 * half;
  if (!ctx->scalars_clean[half]) FGS_CHECK(cudaMemsetAsync(scalars, 0, 16 * sizeof(uint32_t), st));
  ctx->scalars_clean[half] = false;
  if (ctx->flags & FGS_FLAG_COUNTERS) FGS_CHECK(cudaMemsetAsync(ctx->counters.p, 0, 24 * sizeof(unsigned long long), st));
  if (n > 0) {
    fgs::PreprocessArgs pa{};
    pa.n = n;
    pa.cam = ctx->dcam;
    pa.sh_degree = sh_degree;
    pa.tiles_x = tiles_x;
    pa.tiles_y = tiles_y;
    pa.means = scene->means;
    pa.rotations = scene->rotations;
    pa.log_scales = scene->log_scales;
    pa.opacity = scene->opacity_logits;
    pa.sh = scene->sh;
    pa.rec = ctx->rec.p;
    pa.state = ctx->state.p;
    pa.depth_key = ctx->dkey.p;
    pa.touched = ctx->touched.p;
    pa.rect = ctx->rect.p;
    pa.radii = ctx->radii.p;
    pa.rowdiff = ctx->rowdiff.p;
    pa.vec_rot = aligned16(scene->rotations);
    pa.vec_sh = aligned16(scene->sh);
    pa.vec_geo = aligned16(scene->means) && aligned16(scene->log_scales);
    pa.error_flag = reinterpret_cast<int*>(scalars + 1);
    pa.state_counts = scalars + 2;
    nvtxMarkA("K1 preprocess");
    fgs::preprocess_launch(pa, ctx->scene_on_host, st);
    ++launches;
  }
  if (timing) cudaEventRecord(ev[1], st);
  // K2 (one persistent cooperative kernel): emission offsets of the tile-touching Gaussians,
  // I, tile ranges from K1's per-tile counts, blend schedule, key scatter into the ranges
  fgs::BinArgs bn{};
  bn.n = static_cast<int>(n);
  bn.tiles_x = tiles_x;
  bn.tiles_y = tiles_y;
  bn.num_tiles = num_tiles;
  bn.touched = ctx->touched.p;
  bn.depth_key = ctx->dkey.p;
  bn.rect = ctx->rect.p;
  bn.rowdiff = ctx->rowdiff.p;
  bn.cval = ctx->cval.p;
  bn.coff = ctx->coff.p;
  bn.scalars = scalars;
  bn.part_scan = ctx->scan_status.p;
  bn.tile_offsets = ctx->tile_offsets.p;
  bn.fill = ctx->fill.p;
  bn.tile_sched = ctx->tile_sched.p;
  bn.isect_cap = ctx->isect_cap;
  bn.keys = ctx->keys.p;
  bn.row_list = ctx->row_list.p;
  bn.row_hist = ctx->row_hist.p;
  // binning scatter by tile-row lists when the frame has many intersections (configs 3-4:
  // K2 0.159 -> 0.141 ms, 0.141 -> 0.127), by source-order slots otherwise (config 2: 0.046 vs
  // 0.054); decided on the last frame's count, kept for the relaunch of the same frame
  bn.row_scatter = (ctx->flags & FGS_FLAG_ROW_SCATTER) ? 1 : (ctx->flags & FGS_FLAG_SLOT_SCATTER) ? 0
                                                          : rule_row_scatter(ctx->num_isect);
  ctx->var_row_scatter = bn.row_scatter;
  bn.fast = (ctx->flags & FGS_FLAG_GLOBAL_SLOTS) ? 0 : rule_bin_fast();
  bn.src_off = ctx->src_off.p;
  bn.host_scalars = ctx->d_hscalars;
  bn.seq = ++ctx->frame_seq;
  bn.trace = (ctx->flags & FGS_FLAG_COUNTERS) ? ctx->counters.p + 16 : nullptr;
  if (n > 0) {
    ctx->rowdiff_clean = 0;  // dirty until K2 has consumed K1's counts
    nvtxMarkA("K2 binning");
    FGS_CHECK(fgs::bin_launch(bn, st));
    ctx->var_bin_local = bn.fast;
    ctx->rowdiff_clean = ndiff;
    ++launches;
  } else {
    FGS_CHECK(cudaMemsetAsync(ctx->tile_offsets.p, 0, sizeof(uint32_t) * (num_tiles + 1), st));
  }
  // The frame's scalars reach the host without a copy on any stream: K2's CTA 0 writes them
  // into mapped pinned memory once they are final, then the frame's sequence number, and the
  // host waits for that (below) while K3 is already queued behind K2. (A device-to-host copy on
  // a side stream did the same until the application's streams outnumbered the GPU's hardware
  // queues: the copy then shared K3's queue and K3 waited for it, +17 us per frame.)
  const bool k2_ran = n > 0;
  if (k2_ran) {
    FGS_CHECK(cudaEventRecord(ctx->ev_k2, st));
  } else {
    FGS_CHECK(cudaMemcpyAsync(ctx->h_scalars, scalars, fgs::kScalarReadback * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  }
  if (timing) cudaEventRecord(ev[2], st);  // (no separate sort stage: K3 sorts each tile's list)

  // K3 (sort each tile's list + blend) is launched before the host knows I, against the
  // capacity of the per-intersection buffers, so the GPU never waits for the host: K2's scatter
  // and K3 read I from the device and do nothing if it exceeds the capacity, in which case
  // the host grows the buffers and launches the scatter and K3 again (first frames, growing
  // scenes).
  fgs::BlendArgs ba{};
  ba.ellipse = blend_ellipse();
  ba.width = W;
  ba.height = H;
  ba.tiles_x = tiles_x;
  ba.tiles_y = tiles_y;
  ba.tile_offsets = ctx->tile_offsets.p;
  ba.rec = ctx->rec.p;
  ba.num_rec = n;
  for (int k = 0; k < 3; ++k) ba.bg[k] = ctx->bg[k];
  ba.image = image;
  ba.final_T = ctx->final_T.p;
  ba.last = ctx->last.p;
  ba.counters = (ctx->flags & FGS_FLAG_COUNTERS) ? ctx->counters.p : nullptr;
  if (ctx->flags & (FGS_FLAG_COUNTERS | FGS_FLAG_BLEND_COUNT)) {
    FGS_CHECK(ctx->blend_count.ensure(npix));
    ba.blend_count = ctx->blend_count.p;
    ctx->have_blend_count = true;
  } else {
    ctx->have_blend_count = false;
  }
  ba.tile_sched = n > 0 ? ctx->tile_sched.p : nullptr;
  ba.scalars = scalars;
  ba.zero_next = ctx->scalars.p + 16 * (1 - half);
  if (ba.counters) {
    FGS_CHECK(ctx->tile_cycles.ensure(num_tiles));
    FGS_CHECK(cudaMemsetAsync(ctx->tile_cycles.p, 0, num_tiles * sizeof(unsigned long long), st));
    ba.tile_cycles = ctx->tile_cycles.p;
    FGS_CHECK(ctx->tile_span.ensure(2 * num_tiles));
    FGS_CHECK(cudaMemsetAsync(ctx->tile_span.p, 0, 2 * num_tiles * sizeof(unsigned long long), st));
    ba.tile_span = ctx->tile_span.p;
  }
  ba.seg_cursor = scalars + fgs::kScalarSegPos;
  ba.tile_ckpt = ctx->tile_ckpt.p;
  auto launch_blend = [&]() -> int {
    ba.isect_cap = ctx->isect_cap;
    ba.ckpt = ctx->ckpt.p;
    ba.seg_items = ctx->seg_items.p;
    ba.ckpt_cap = ctx->ckpt_cap;
    ba.keys = ctx->keys.p;
    ba.sorted_gauss = ctx->sorted_gauss.p;
    // work decomposition from this frame's statistics once known, else the last frame's
    nvtxMarkA("K3 sort + blend");
    const int px = rule_fwd_px(ctx->num_isect, num_tiles, ctx->longest);
    ctx->var_fwd_px = px;
    const int l = fgs::blend_forward(ba, ctx->num_isect, px, st);
    ctx->scalars_clean[1 - half] = true;  // K3 zeroes the other half
    if (timing) cudaEventRecord(ev[4], st);
    return l;
  };
  const bool speculative = n > 0 && ctx->isect_cap > 0;
  if (speculative) launches += launch_blend();

  if (k2_ran) {
    const int w = wait_host_scalars(ctx);
    if (w != FGS_OK) return w;
  } else {
    FGS_CHECK(cudaStreamSynchronize(st));
  }
  FGS_CHECK(cudaGetLastError());
  if (ctx->h_scalars[fgs::kScalarErr]) return fail(ctx, FGS_EDEGENERATE_QUAT, "degenerate rotation: quaternion has zero norm");
  const int64_t I = ctx->h_scalars[fgs::kScalarI];
  if (n > 0 && ctx->h_scalars[fgs::kScalarI2] != ctx->h_scalars[fgs::kScalarI])
    return fail(ctx, FGS_ECUDA, "forward: per-tile counts disagree with the intersection scan");
  ctx->num_isect = I;
  ctx->num_compact = ctx->h_scalars[fgs::kScalarM];
  ctx->chunk_q[0] = 0;
  for (int c = 1; c < fgs::kGradChunks; ++c) ctx->chunk_q[c] = n > 0 ? ctx->h_scalars[fgs::kScalarChunkQ + c - 1] : 0;
  ctx->chunk_q[fgs::kGradChunks] = ctx->num_compact;
  ctx->num_splats = ctx->h_scalars[fgs::kScalarKept];
  ctx->num_degenerate = ctx->h_scalars[fgs::kScalarDegen];
  ctx->num_culled = static_cast<uint32_t>(n) - ctx->num_splats - ctx->num_degenerate;
  if (I >= (int64_t(1) << 30)) return fail(ctx, FGS_ENOMEM, "forward: intersection count exceeds 2^30");
  const int64_t X = ctx->h_scalars[fgs::kScalarSegs];
  ctx->longest = ctx->h_scalars[fgs::kScalarMaxList];
  ctx->num_segs = X;
  if (speculative && I <= ctx->isect_cap && X > ctx->ckpt_cap) {
    // only the checkpoint slots ran short: the speculative K3 exited; grow them and blend again
    FGS_CHECK(ensure_ckpt(ctx, X));
    FGS_CHECK(cudaMemsetAsync(scalars + fgs::kScalarSegPos, 0, sizeof(uint32_t), st));
    launches += launch_blend();
  } else if (!speculative || I > ctx->isect_cap) {
    FGS_CHECK(ensure_ckpt(ctx, X));
    FGS_CHECK(cudaMemsetAsync(scalars + fgs::kScalarSegPos, 0, sizeof(uint32_t), st));
    // (re)size the per-intersection buffers (cudaFree / cudaMalloc synchronise with the
    // speculative kernels, which exited without work) and launch for real
    const size_t ni = static_cast<size_t>(I > 0 ? I : 1);
    FGS_CHECK(ctx->keys.ensure(ni));
    FGS_CHECK(ctx->sorted_gauss.ensure(ni));
    FGS_CHECK(ctx->row_list.ensure(ni));
    size_t cap = ctx->keys.cap;
    cap = std::min(cap, std::min(ctx->sorted_gauss.cap, ctx->row_list.cap));
    ctx->isect_cap = static_cast<int64_t>(cap);
    if (n > 0 && I > 0) {
      bn.isect_cap = ctx->isect_cap;
      bn.keys = ctx->keys.p;
      bn.row_list = ctx->row_list.p;
      bn.scatter_only = 1;
      FGS_CHECK(fgs::bin_launch(bn, st));
      bn.scatter_only = 0;
      ++launches;
    }
    launches += launch_blend();
  }
  ctx->bin_args = bn;
  if (radii && n > 0) FGS_CHECK(cudaMemcpyAsync(radii, ctx->radii.p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  FGS_CHECK(cudaGetLastError());
  ctx->launches += launches;

  ctx->aux_bytes = path_bytes(ctx);
  ctx->have_fwd = true;
  guard.armed = false;
  if (stats) {
    FGS_CHECK(cudaEventSynchronize(ev[4]));
    float ms[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    cudaEventElapsedTime(&ms[0], ev[0], ev[1]);
    cudaEventElapsedTime(&ms[1], ev[1], ev[2]);
    cudaEventElapsedTime(&ms[3], ev[2], ev[4]);  // sort_ms stays 0: K3 sorts each tile's list
    if (!(ctx->flags & FGS_FLAG_TIMING)) {  // stats-only timing: recycle the set now
      ctx->spare.push_back(ctx->pending.back());
      ctx->pending.pop_back();
    }
    stats->num_intersections = static_cast<uint64_t>(I);
    stats->num_splats = ctx->num_splats;
    stats->num_culled = ctx->num_culled;
    stats->num_degenerate = ctx->num_degenerate;
    stats->preprocess_ms = ms[0];
    stats->binning_ms = ms[1];
    stats->sort_ms = ms[2];
    stats->raster_ms = ms[3];
    stats->peak_aux_bytes = ctx->aux_bytes;
  }
  return FGS_OK;
}

// The backward of the last forward. K4b runs as one launch, or (chunk_done set) as kGradChunks
// launches over the Gaussian-id ranges [c n / C, (c + 1) n / C) with chunk_done(c, id0, id1)
// called after each: the multi-GPU step enqueues that range's all-reduce there
// (fgs_fwd_bwd_views), overlapping it with the next range's K4b.
int backward_impl(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera, const float* dl_dimage,
                  const fgs_backward_options* options, fgs_gradients* grads,
                  const std::function<int(int, int64_t, int64_t)>& chunk_done) {
  if (!ctx) return FGS_EINVAL;
  NvtxRange nvtx("fgs.backward");
  if (!scene || !camera || !dl_dimage || !grads) return fail(ctx, FGS_EINVAL, "backward: null argument");
  if (!ctx->have_fwd) return fail(ctx, FGS_ESTATE, "backward: no forward context");
  if (scene->n != ctx->n) return fail(ctx, FGS_EINVAL, "backward: forward context was built for a different scene");
  if (!same_camera(*camera, ctx->cam))
    return fail(ctx, FGS_EINVAL, "backward: forward context was built for a different camera");
  FGS_CHECK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int64_t n = ctx->n, I = ctx->num_isect;
  if (n == 0) return FGS_OK;
  FGS_CHECK(ctx->partial_tile.ensure(static_cast<size_t>(I > 0 ? I : 1) * 9));
  ctx->aux_bytes = path_bytes(ctx);

  fgs::BlendArgs ba{};
  ba.ellipse = blend_ellipse();
  ba.width = ctx->cam.width;
  ba.height = ctx->cam.height;
  ba.tiles_x = ctx->tiles_x;
  ba.tiles_y = ctx->tiles_y;
  ba.tile_offsets = ctx->tile_offsets.p;
  ba.sorted_gauss = ctx->sorted_gauss.p;
  ba.rec = ctx->rec.p;
  for (int k = 0; k < 3; ++k) ba.bg[k] = ctx->bg[k];
  ba.final_T = ctx->final_T.p;
  ba.last = ctx->last.p;
  ba.dl_dimage = dl_dimage;
  ba.ckpt = ctx->ckpt.p;
  ba.seg_items = ctx->seg_items.p;
  ba.tile_ckpt = ctx->tile_ckpt.p;
  ba.num_seg_items = ctx->num_segs;
  ba.num_rec = n;
  ba.isect_cap = I;  // (bounds for the checked build)
  ba.ckpt_cap = ctx->ckpt_cap;
  ba.counters = (ctx->flags & FGS_FLAG_COUNTERS) ? ctx->counters.p : nullptr;
  ba.partial_tile = ctx->partial_tile.p;
  ba.src_off = ctx->src_off.p;
  ba.rect = ctx->rect.p;
  ba.tile_sched = I > 0 ? ctx->tile_sched.p : nullptr;
  if (ba.counters) {
    const size_t nt = static_cast<size_t>(ctx->tiles_x) * ctx->tiles_y;
    FGS_CHECK(ctx->tile_span_bwd.ensure(2 * nt));
    FGS_CHECK(cudaMemsetAsync(ctx->tile_span_bwd.p, 0, 2 * nt * sizeof(unsigned long long), st));
    ba.tile_span = ctx->tile_span_bwd.p;
  }
  const bool timing = (ctx->flags & FGS_FLAG_TIMING) != 0;
  if (timing && ctx->pending.size() > 64) drain_sets(ctx, 8);
  cudaEvent_t* ev = timing ? take_set(ctx, 1)->e : nullptr;
  SetGuard guard{ctx, timing};
  if (timing) cudaEventRecord(ev[0], st);
  if (I > 0) {
    nvtxMarkA("K4a blend backward");
    ctx->launches += fgs::blend_backward(ba, I, 0, st, &ctx->var_bwd_px);
  }
  if (timing) cudaEventRecord(ev[1], st);

  fgs::PreprocessBackwardArgs pb{};
  pb.n = n;
  pb.cam = ctx->dcam;
  pb.sh_degree = ctx->sh_degree;
  pb.full_sh = options ? options->full_sh : 1;
  pb.accumulate = options ? options->accumulate : 0;
  pb.view_dir = options ? options->sh_view_dir_grad : 0;
  for (int k = 0; k < 3; ++k) pb.jac_grad_scale[k] = options ? options->jacobian_grad_scale[k] : 1.0f;
  pb.means = scene->means;
  pb.rotations = scene->rotations;
  pb.log_scales = scene->log_scales;
  pb.opacity = scene->opacity_logits;
  pb.sh = scene->sh;
  pb.vec_rot = aligned16(scene->rotations);
  pb.state = ctx->state.p;
  pb.touched = ctx->touched.p;
  pb.coff = ctx->coff.p;
  pb.partials = ctx->partial_tile.p;
  pb.num_isect = I;
  pb.d_means = grads->d_means;
  pb.d_rotations = grads->d_rotations;
  pb.d_log_scales = grads->d_log_scales;
  pb.d_opacity = grads->d_opacity_logits;
  pb.d_sh = grads->d_sh;
  pb.aligned16 = ((reinterpret_cast<uintptr_t>(grads->d_rotations) | reinterpret_cast<uintptr_t>(grads->d_sh)) & 15u) == 0;
  pb.m = ctx->num_compact;
  pb.cval = ctx->cval.p;
  pb.rec = ctx->rec.p;
  ctx->var_k4b = ctx->scene_on_host ? 6 : rule_k4b_minb(pb.m);
  const int variant = ctx->var_k4b == 4 ? 2 : 1;
  if (!chunk_done) {
    pb.q_begin = 0;
    pb.q_end = pb.m;
    pb.id_begin = 0;
    pb.id_end = n;
    if (n > 0 && (pb.m > 0 || !pb.accumulate)) {
      fgs::preprocess_backward_launch(pb, ctx->scene_on_host, variant, st);
      ++ctx->launches;
    }
  } else {
    for (int c = 0; c < fgs::kGradChunks; ++c) {
      pb.q_begin = ctx->chunk_q[c];
      pb.q_end = ctx->chunk_q[c + 1];
      pb.id_begin = n * c / fgs::kGradChunks;
      pb.id_end = n * (c + 1) / fgs::kGradChunks;
      if (pb.id_end > pb.id_begin && (pb.q_end > pb.q_begin || !pb.accumulate)) {
        fgs::preprocess_backward_launch(pb, ctx->scene_on_host, variant, st);
        ++ctx->launches;
      }
      FGS_CHECK(cudaGetLastError());
      const int rc = chunk_done(c, pb.id_begin, pb.id_end);
      if (rc != FGS_OK) return rc;
    }
  }
  if (timing) cudaEventRecord(ev[2], st);
  FGS_CHECK(cudaGetLastError());
  guard.armed = false;
  return FGS_OK;
}

int fgs_backward(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera, const float* dl_dimage,
                 const fgs_backward_options* options, fgs_gradients* grads) {
  return backward_impl(ctx, scene, camera, dl_dimage, options, grads, nullptr);
}

}  // extern "C"

// Internal entry points for comm.cu (not part of the C ABI).
int fgs_internal_fail(fgs_context* ctx, int code, const char* msg) { return fail(ctx, code, msg); }
cudaStream_t fgs_internal_stream(fgs_context* ctx) { return ctx->stream; }
int fgs_internal_device(fgs_context* ctx) { return ctx->device; }
float* fgs_internal_scratch_image(fgs_context* ctx, size_t floats) {
  return ctx->t_image.ensure(floats) == cudaSuccess ? ctx->t_image.p : nullptr;
}
int fgs_internal_backward(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                          const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads,
                          const std::function<int(int, int64_t, int64_t)>& chunk_done) {
  return backward_impl(ctx, scene, camera, dl_dimage, options, grads, chunk_done);
}

extern "C" {

namespace {
// Device address of page-locked (pinned, mapped) host memory, or nullptr for pageable memory.
const void* mapped_host(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

// The scene's five arrays as device-accessible pointers when all of them are pinned host
// memory: K1 then reads them over PCIe directly (zero copy), and only what it needs -- the
// geometry of every Gaussian, the opacity and SH rows of the visible ones.
bool mapped_scene(const fgs_gaussians* s, fgs_gaussians* out) {
  *out = *s;
  if (s->n <= 0) return false;
  const void* p[5] = {mapped_host(s->means), mapped_host(s->rotations), mapped_host(s->log_scales),
                      mapped_host(s->opacity_logits), mapped_host(s->sh)};
  for (auto* q : p)
    if (!q) return false;
  out->means = static_cast<const float*>(p[0]);
  out->rotations = static_cast<const float*>(p[1]);
  out->log_scales = static_cast<const float*>(p[2]);
  out->opacity_logits = static_cast<const float*>(p[3]);
  out->sh = static_cast<const float*>(p[4]);
  return true;
}
}  // namespace

int fgs_wait(fgs_context* ctx) {
  if (!ctx) return FGS_EINVAL;
  if (ctx->async_last < 0 && ctx->gasync_last < 0) return FGS_OK;
  FGS_CHECK(cudaSetDevice(ctx->device));
  for (cudaEvent_t e : {ctx->async_last >= 0 ? ctx->ev_copied[ctx->async_last] : nullptr,
                        ctx->gasync_last >= 0 ? ctx->ev_gcopied[ctx->gasync_last] : nullptr}) {
    if (!e) continue;
    FGS_CHECK(cudaStreamWaitEvent(ctx->stream, e, 0));
    FGS_CHECK(cudaEventSynchronize(e));
  }
  ctx->async_last = -1;
  ctx->gasync_last = -1;
  return FGS_OK;
}

namespace {
int render_host_impl(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                     const fgs_render_options* options, float* image, int32_t* radii, fgs_stats* stats, bool async) {
  if (!ctx) return FGS_EINVAL;
  if (!scene || !camera || !image) return fail(ctx, FGS_EINVAL, "render: null argument");
  FGS_CHECK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  if (!async) {
    const int w = fgs_wait(ctx);  // earlier asynchronous frames complete first
    if (w != FGS_OK) return w;
  }
  const size_t n = static_cast<size_t>(scene->n > 0 ? scene->n : 0), nn = n ? n : 1;
  const size_t npix = static_cast<size_t>(camera->width) * camera->height;
  FGS_CHECK(ctx->h_means.ensure(nn * 3));
  FGS_CHECK(ctx->h_rot.ensure(nn * 4));
  FGS_CHECK(ctx->h_ls.ensure(nn * 3));
  FGS_CHECK(ctx->h_op.ensure(nn));
  FGS_CHECK(ctx->h_sh.ensure(nn * 48));
  FGS_CHECK(ctx->h_img.ensure(npix * 3));
  FGS_CHECK(ctx->h_radii.ensure(nn));
  fgs_gaussians dev{};
  const bool zero_copy = mapped_scene(scene, &dev);
  if (!zero_copy) {  // pageable host memory: copy the whole scene
    if (n) {
      FGS_CHECK(cudaMemcpyAsync(ctx->h_means.p, scene->means, n * 3 * 4, cudaMemcpyHostToDevice, st));
      FGS_CHECK(cudaMemcpyAsync(ctx->h_rot.p, scene->rotations, n * 4 * 4, cudaMemcpyHostToDevice, st));
      FGS_CHECK(cudaMemcpyAsync(ctx->h_ls.p, scene->log_scales, n * 3 * 4, cudaMemcpyHostToDevice, st));
      FGS_CHECK(cudaMemcpyAsync(ctx->h_op.p, scene->opacity_logits, n * 4, cudaMemcpyHostToDevice, st));
      FGS_CHECK(cudaMemcpyAsync(ctx->h_sh.p, scene->sh, n * 48 * 4, cudaMemcpyHostToDevice, st));
    }
    dev = fgs_gaussians{scene->n, ctx->h_means.p, ctx->h_rot.p, ctx->h_ls.p, ctx->h_op.p, ctx->h_sh.p};
  }
  ctx->scene_on_host = zero_copy;
  float* dimg = ctx->h_img.p;
  int32_t* drad = ctx->h_radii.p;
  const int par = ctx->async_parity;
  if (async) {
    FGS_CHECK(ensure_copy_stream(ctx));
    FGS_CHECK(ctx->a_img[par].ensure(npix * 3));
    FGS_CHECK(ctx->a_radii[par].ensure(nn));
    dimg = ctx->a_img[par].p;
    drad = ctx->a_radii[par].p;
    // the read-back of the frame that used this buffer pair two frames ago must be done first
    if (ctx->copy_recorded[par]) FGS_CHECK(cudaStreamWaitEvent(st, ctx->ev_copied[par], 0));
  }
  int rc = fgs_forward(ctx, &dev, camera, options, dimg, radii ? drad : nullptr, stats);
  ctx->scene_on_host = false;
  if (rc != FGS_OK) return rc;
  if (async) {
    // the image (and radii) read back on the copy stream: device -> host while the caller's
    // next frame reads its scene host -> device (PCIe is full duplex)
    FGS_CHECK(cudaEventRecord(ctx->ev_rendered, st));
    FGS_CHECK(cudaStreamWaitEvent(ctx->copy_st, ctx->ev_rendered, 0));
    FGS_CHECK(cudaMemcpyAsync(image, dimg, npix * 3 * 4, cudaMemcpyDeviceToHost, ctx->copy_st));
    if (radii && n) FGS_CHECK(cudaMemcpyAsync(radii, drad, n * 4, cudaMemcpyDeviceToHost, ctx->copy_st));
    FGS_CHECK(cudaEventRecord(ctx->ev_copied[par], ctx->copy_st));
    ctx->copy_recorded[par] = true;
    ctx->async_last = par;
    ctx->async_parity = 1 - par;
  } else {
    FGS_CHECK(cudaMemcpyAsync(image, dimg, npix * 3 * 4, cudaMemcpyDeviceToHost, st));
    if (radii && n) FGS_CHECK(cudaMemcpyAsync(radii, drad, n * 4, cudaMemcpyDeviceToHost, st));
    FGS_CHECK(cudaStreamSynchronize(st));
  }
  // bytes over PCIe: zero copy reads 40 B of geometry and the opacity of every Gaussian and,
  // per splat that survives the culls, the SH coefficients of the evaluated degree
  const int deg = options ? options->sh_degree : 3;
  const uint64_t sh_bytes = deg == 0 ? 3 * 4 : (deg == 1 ? 3 * 16 : (deg == 2 ? 3 * 48 : 3 * 64));
  ctx->h2d_bytes = zero_copy ? n * 44 + static_cast<uint64_t>(ctx->num_splats) * sh_bytes : n * 59 * 4;
  ctx->d2h_bytes = npix * 3 * 4 + (radii ? n * 4 : 0);
  return FGS_OK;
}
}  // namespace

int fgs_render_host(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                    const fgs_render_options* options, float* image, int32_t* radii, fgs_stats* stats) {
  return render_host_impl(ctx, scene, camera, options, image, radii, stats, false);
}

int fgs_render_host_async(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                          const fgs_render_options* options, float* image, int32_t* radii, fgs_stats* stats) {
  return render_host_impl(ctx, scene, camera, options, image, radii, stats, true);
}

namespace {
// Host-buffer backward with the scene already on the device (dev) or mapped (zero_copy).
int backward_host_dev(fgs_context* ctx, const fgs_gaussians& dev, bool zero_copy, const fgs_camera* camera,
                      const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads,
                      bool async = false);
int backward_host_impl(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera, const float* dl_dimage,
                       const fgs_backward_options* options, fgs_gradients* grads, bool async);
}  // namespace

int fgs_backward_host(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera, const float* dl_dimage,
                      const fgs_backward_options* options, fgs_gradients* grads) {
  return backward_host_impl(ctx, scene, camera, dl_dimage, options, grads, false);
}

int fgs_backward_host_async(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                            const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads) {
  return backward_host_impl(ctx, scene, camera, dl_dimage, options, grads, true);
}

namespace {

int backward_host_impl(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera, const float* dl_dimage,
                       const fgs_backward_options* options, fgs_gradients* grads, bool async) {
  if (!ctx) return FGS_EINVAL;
  if (!scene || !camera || !dl_dimage || !grads) return fail(ctx, FGS_EINVAL, "backward: null argument");
  FGS_CHECK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  if (!async && ctx->gasync_last >= 0) {
    const int w = fgs_wait(ctx);
    if (w != FGS_OK) return w;
  }
  const size_t n = static_cast<size_t>(ctx->n), nn = n ? n : 1;
  if (static_cast<int64_t>(n) != scene->n)
    return fail(ctx, FGS_EINVAL, "backward: forward context was built for a different scene");
  // The reference takes the scene by value on every call: pinned host arrays are read in place
  // (zero copy, only the tile-touching Gaussians' parameters), pageable ones copied again.
  fgs_gaussians dev{};
  const bool zero_copy = mapped_scene(scene, &dev);
  if (!zero_copy) {
    FGS_CHECK(ctx->h_means.ensure(nn * 3));
    FGS_CHECK(ctx->h_rot.ensure(nn * 4));
    FGS_CHECK(ctx->h_ls.ensure(nn * 3));
    FGS_CHECK(ctx->h_op.ensure(nn));
    FGS_CHECK(ctx->h_sh.ensure(nn * 48));
    if (n) {
      FGS_CHECK(cudaMemcpyAsync(ctx->h_means.p, scene->means, n * 3 * 4, cudaMemcpyHostToDevice, st));
      FGS_CHECK(cudaMemcpyAsync(ctx->h_rot.p, scene->rotations, n * 4 * 4, cudaMemcpyHostToDevice, st));
      FGS_CHECK(cudaMemcpyAsync(ctx->h_ls.p, scene->log_scales, n * 3 * 4, cudaMemcpyHostToDevice, st));
      FGS_CHECK(cudaMemcpyAsync(ctx->h_op.p, scene->opacity_logits, n * 4, cudaMemcpyHostToDevice, st));
      FGS_CHECK(cudaMemcpyAsync(ctx->h_sh.p, scene->sh, n * 48 * 4, cudaMemcpyHostToDevice, st));
    }
    dev = fgs_gaussians{scene->n, ctx->h_means.p, ctx->h_rot.p, ctx->h_ls.p, ctx->h_op.p, ctx->h_sh.p};
  }
  const int rc = backward_host_dev(ctx, dev, zero_copy, camera, dl_dimage, options, grads, async);
  if (rc == FGS_OK && !zero_copy) ctx->h2d_bytes += n * 59 * 4;
  return rc;
}

int backward_host_dev(fgs_context* ctx, const fgs_gaussians& dev, bool zero_copy, const fgs_camera* camera,
                      const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads, bool async) {
  cudaStream_t st = ctx->stream;
  const size_t n = static_cast<size_t>(ctx->n), nn = n ? n : 1;
  const size_t npix = static_cast<size_t>(camera->width) * camera->height;
  FGS_CHECK(ctx->h_dl.ensure(npix * 3));
  FGS_CHECK(ctx->h_grad.ensure(nn * 59));
  FGS_CHECK(cudaMemcpyAsync(ctx->h_dl.p, dl_dimage, npix * 3 * 4, cudaMemcpyHostToDevice, st));
  float* g = ctx->h_grad.p;
  const int gp = ctx->gasync_parity;
  if (async) {
    FGS_CHECK(ensure_copy_stream(ctx));
    FGS_CHECK(ctx->a_grad[gp].ensure(nn * 59));
    g = ctx->a_grad[gp].p;
    // the read-back of the call that used this buffer two calls ago must be done first
    if (ctx->gcopy_recorded[gp]) FGS_CHECK(cudaStreamWaitEvent(st, ctx->ev_gcopied[gp], 0));
  }
  fgs_gradients dg{g, g + 3 * nn, g + 7 * nn, g + 10 * nn, g + 11 * nn};
  const bool acc = options && options->accumulate;
  if (acc && n) {
    FGS_CHECK(cudaMemcpyAsync(dg.d_means, grads->d_means, n * 3 * 4, cudaMemcpyHostToDevice, st));
    FGS_CHECK(cudaMemcpyAsync(dg.d_rotations, grads->d_rotations, n * 4 * 4, cudaMemcpyHostToDevice, st));
    FGS_CHECK(cudaMemcpyAsync(dg.d_log_scales, grads->d_log_scales, n * 3 * 4, cudaMemcpyHostToDevice, st));
    FGS_CHECK(cudaMemcpyAsync(dg.d_opacity_logits, grads->d_opacity_logits, n * 4, cudaMemcpyHostToDevice, st));
    FGS_CHECK(cudaMemcpyAsync(dg.d_sh, grads->d_sh, n * 48 * 4, cudaMemcpyHostToDevice, st));
  }
  ctx->scene_on_host = zero_copy;
  int rc = fgs_backward(ctx, &dev, camera, ctx->h_dl.p, options, &dg);
  ctx->scene_on_host = false;
  if (rc != FGS_OK) return rc;
  // the gradients back: on the copy stream for the asynchronous call (device -> host while the
  // caller's next frame reads its scene and uploads its dL/dimage host -> device)
  cudaStream_t cs = st;
  if (async) {
    FGS_CHECK(cudaEventRecord(ctx->ev_bdone, st));
    FGS_CHECK(cudaStreamWaitEvent(ctx->copy_st, ctx->ev_bdone, 0));
    cs = ctx->copy_st;
  }
  if (n) {
    FGS_CHECK(cudaMemcpyAsync(grads->d_means, dg.d_means, n * 3 * 4, cudaMemcpyDeviceToHost, cs));
    FGS_CHECK(cudaMemcpyAsync(grads->d_rotations, dg.d_rotations, n * 4 * 4, cudaMemcpyDeviceToHost, cs));
    FGS_CHECK(cudaMemcpyAsync(grads->d_log_scales, dg.d_log_scales, n * 3 * 4, cudaMemcpyDeviceToHost, cs));
    FGS_CHECK(cudaMemcpyAsync(grads->d_opacity_logits, dg.d_opacity_logits, n * 4, cudaMemcpyDeviceToHost, cs));
    FGS_CHECK(cudaMemcpyAsync(grads->d_sh, dg.d_sh, n * 48 * 4, cudaMemcpyDeviceToHost, cs));
  }
  if (async) {
    FGS_CHECK(cudaEventRecord(ctx->ev_gcopied[gp], cs));
    ctx->gcopy_recorded[gp] = true;
    ctx->gasync_last = gp;
    ctx->gasync_parity = 1 - gp;
  } else {
    FGS_CHECK(cudaStreamSynchronize(st));
  }
  ctx->h2d_bytes = npix * 3 * 4 + (zero_copy ? static_cast<uint64_t>(ctx->num_compact) * 44 : 0) +
                   (acc ? n * 59 * 4 : 0);
  ctx->d2h_bytes = n * 59 * 4;
  return FGS_OK;
}
}  // namespace

namespace {
// AoS -> SoA on the device: one thread per (Gaussian, float field component); consecutive threads
// read consecutive floats of a record and write consecutive entries of each field array.
__global__ void aos_to_soa_kernel(const uint8_t* __restrict__ raw, int64_t n, int64_t stride, int64_t o_mean,
                                  int64_t o_rot, int64_t o_ls, int64_t o_op, int64_t o_sh, float* means, float* rot,
                                  float* ls, float* op, float* sh) {
  const int64_t total = n * 59;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = i / 59;
    const int f = static_cast<int>(i - g * 59);
    const uint8_t* rec = raw + g * stride;
    float v;
    if (f < 3) {
      memcpy(&v, rec + o_mean + 4 * f, 4);
      means[g * 3 + f] = v;
    } else if (f < 7) {
      memcpy(&v, rec + o_rot + 4 * (f - 3), 4);
      rot[g * 4 + f - 3] = v;
    } else if (f < 10) {
      memcpy(&v, rec + o_ls + 4 * (f - 7), 4);
      ls[g * 3 + f - 7] = v;
    } else if (f == 10) {
      memcpy(&v, rec + o_op, 4);
      op[g] = v;
    } else {
      memcpy(&v, rec + o_sh + 4 * (f - 11), 4);
      sh[g * 48 + f - 11] = v;
    }
  }
}

// Uploads an AoS host scene in one transfer and splits it into the context's device SoA arrays.
int upload_aos(fgs_context* ctx, const fgs_gaussians_aos* s, fgs_gaussians* dev) {
  if (s->n < 0 || (s->n > 0 && (!s->data || s->stride < 59 * 4))) return fail(ctx, FGS_EINVAL, "scene: bad AoS layout");
  const int64_t offs[5] = {s->off_mean, s->off_rotation, s->off_log_scale, s->off_opacity_logit, s->off_sh};
  const int64_t widths[5] = {3, 4, 3, 1, 48};
  for (int k = 0; k < 5; ++k)
    if (offs[k] < 0 || offs[k] + 4 * widths[k] > s->stride) return fail(ctx, FGS_EINVAL, "scene: AoS field outside the record");
  cudaStream_t st = ctx->stream;
  const size_t n = static_cast<size_t>(s->n), nn = n ? n : 1;
  FGS_CHECK(ctx->h_means.ensure(nn * 3));
  FGS_CHECK(ctx->h_rot.ensure(nn * 4));
  FGS_CHECK(ctx->h_ls.ensure(nn * 3));
  FGS_CHECK(ctx->h_op.ensure(nn));
  FGS_CHECK(ctx->h_sh.ensure(nn * 48));
  FGS_CHECK(ctx->h_aos.ensure(nn * static_cast<size_t>(s->stride)));
  if (n) {
    FGS_CHECK(cudaMemcpyAsync(ctx->h_aos.p, s->data, n * s->stride, cudaMemcpyHostToDevice, st));
    const int64_t total = static_cast<int64_t>(n) * 59;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    aos_to_soa_kernel<<<blocks, 256, 0, st>>>(ctx->h_aos.p, s->n, s->stride, s->off_mean, s->off_rotation,
                                              s->off_log_scale, s->off_opacity_logit, s->off_sh, ctx->h_means.p,
                                              ctx->h_rot.p, ctx->h_ls.p, ctx->h_op.p, ctx->h_sh.p);
    ++ctx->launches;
    FGS_CHECK(cudaGetLastError());
  }
  *dev = fgs_gaussians{s->n, ctx->h_means.p, ctx->h_rot.p, ctx->h_ls.p, ctx->h_op.p, ctx->h_sh.p};
  return FGS_OK;
}
}  // namespace

int fgs_render_host_aos(fgs_context* ctx, const fgs_gaussians_aos* scene, const fgs_camera* camera,
                        const fgs_render_options* options, float* image, int32_t* radii, fgs_stats* stats) {
  if (!ctx) return FGS_EINVAL;
  if (!scene || !camera || !image) return fail(ctx, FGS_EINVAL, "render: null argument");
  FGS_CHECK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  fgs_gaussians dev{};
  int rc = upload_aos(ctx, scene, &dev);
  if (rc != FGS_OK) return rc;
  const size_t n = static_cast<size_t>(scene->n), nn = n ? n : 1;
  const size_t npix = static_cast<size_t>(camera->width) * camera->height;
  FGS_CHECK(ctx->h_img.ensure(npix * 3));
  FGS_CHECK(ctx->h_radii.ensure(nn));
  rc = fgs_forward(ctx, &dev, camera, options, ctx->h_img.p, radii ? ctx->h_radii.p : nullptr, stats);
  if (rc != FGS_OK) return rc;
  FGS_CHECK(cudaMemcpyAsync(image, ctx->h_img.p, npix * 3 * 4, cudaMemcpyDeviceToHost, st));
  if (radii && n) FGS_CHECK(cudaMemcpyAsync(radii, ctx->h_radii.p, n * 4, cudaMemcpyDeviceToHost, st));
  FGS_CHECK(cudaStreamSynchronize(st));
  ctx->h2d_bytes = n * static_cast<uint64_t>(scene->stride);
  ctx->d2h_bytes = npix * 3 * 4 + (radii ? n * 4 : 0);
  return FGS_OK;
}

int fgs_backward_host_aos(fgs_context* ctx, const fgs_gaussians_aos* scene, const fgs_camera* camera,
                          const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads) {
  if (!ctx) return FGS_EINVAL;
  if (!scene || !camera || !dl_dimage || !grads) return fail(ctx, FGS_EINVAL, "backward: null argument");
  FGS_CHECK(cudaSetDevice(ctx->device));
  if (scene->n != ctx->n) return fail(ctx, FGS_EINVAL, "backward: forward context was built for a different scene");
  fgs_gaussians dev{};
  int rc = upload_aos(ctx, scene, &dev);
  if (rc != FGS_OK) return rc;
  rc = backward_host_dev(ctx, dev, false, camera, dl_dimage, options, grads);
  if (rc == FGS_OK) ctx->h2d_bytes += static_cast<uint64_t>(scene->n) * static_cast<uint64_t>(scene->stride);
  return rc;
}

int fgs_last_transfer(const fgs_context* ctx, uint64_t out[2]) {
  if (!ctx || !out) return FGS_EINVAL;
  out[0] = ctx->h2d_bytes;
  out[1] = ctx->d2h_bytes;
  return FGS_OK;
}

int fgs_l1_dssim_loss(fgs_context* ctx, const float* rendered, const float* target, int32_t width, int32_t height,
                      float lambda, float* d_rendered, double out[3]) {
  if (!ctx) return FGS_EINVAL;
  if (!rendered || !target || !d_rendered || !out) return fail(ctx, FGS_EINVAL, "l1_dssim_loss: null argument");
  if (width <= 0 || height <= 0) return fail(ctx, FGS_EINVAL, "l1_dssim_loss: image dimensions differ");
  FGS_CHECK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  FGS_CHECK(ctx->t_maps.ensure(fgs::loss_scratch_floats(width, height)));
  const size_t nb = fgs::loss_partials(width, height);
  FGS_CHECK(ctx->t_part.ensure(2 * nb + 2));
  ctx->launches += fgs::l1_dssim_loss(rendered, target, width, height, lambda, d_rendered, ctx->t_maps.p,
                                      ctx->t_part.p, st);
  double sums[2];
  FGS_CHECK(cudaMemcpyAsync(sums, ctx->t_part.p + 2 * nb, sizeof(sums), cudaMemcpyDeviceToHost, st));
  FGS_CHECK(cudaStreamSynchronize(st));
  FGS_CHECK(cudaGetLastError());
  const double norm = 1.0 / (3.0 * static_cast<double>(width) * height);
  const double l1 = sums[1] * norm, dssim = 1.0 - sums[0] * norm;
  out[0] = (1.0 - lambda) * l1 + lambda * dssim;
  out[1] = l1;
  out[2] = dssim;
  return FGS_OK;
}

int fgs_adam_step(fgs_context* ctx, fgs_params* params, const fgs_gradients* grads, fgs_adam_state* state,
                  const fgs_adam_options* o) {
  if (!ctx) return FGS_EINVAL;
  if (!params || !grads || !state || !o) return fail(ctx, FGS_EINVAL, "adam_step: null argument");
  FGS_CHECK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int64_t n = params->n;
  fgs::AdamArgs a{};
  float* p[5] = {params->means, params->rotations, params->log_scales, params->opacity_logits, params->sh};
  const float* g[5] = {grads->d_means, grads->d_rotations, grads->d_log_scales, grads->d_opacity_logits, grads->d_sh};
  float* m[5] = {state->m.d_means, state->m.d_rotations, state->m.d_log_scales, state->m.d_opacity_logits,
                 state->m.d_sh};
  float* v[5] = {state->v.d_means, state->v.d_rotations, state->v.d_log_scales, state->v.d_opacity_logits,
                 state->v.d_sh};
  const int w[5] = {3, 4, 3, 1, 48};
  for (int k = 0; k < 5; ++k) {
    if (n > 0 && (!p[k] || !g[k] || !m[k] || !v[k])) return fail(ctx, FGS_EINVAL, "adam_step: null array");
    a.p[k] = p[k];
    a.g[k] = g[k];
    a.m[k] = m[k];
    a.v[k] = v[k];
    a.len[k] = n * w[k];
    a.width[k] = w[k];
  }
  const float lr[6] = {o->lr_mean, o->lr_rotation, o->lr_log_scale, o->lr_opacity, o->lr_sh_dc, o->lr_sh_rest};
  for (int k = 0; k < 6; ++k) a.lr[k] = lr[k];
  a.beta1 = o->beta1;
  a.beta2 = o->beta2;
  a.eps = o->eps;
  FGS_CHECK(ctx->t_flag.ensure(1));
  a.nonfinite = ctx->t_flag.p;
  const int big = 0x7fffffff;
  FGS_CHECK(cudaMemcpyAsync(ctx->t_flag.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  ctx->launches += fgs::adam_check(a, st);
  int first_bad = big;
  FGS_CHECK(cudaMemcpyAsync(&first_bad, ctx->t_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FGS_CHECK(cudaStreamSynchronize(st));
  if (first_bad != big)
    return fail(ctx, FGS_ENONFINITE, "adam_step: non-finite gradient for Gaussian " + std::to_string(first_bad));
  // bias corrections in double, as the reference's std::pow on its double state
  const int64_t step = state->step + 1;
  a.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(o->beta1), static_cast<double>(step)));
  a.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(o->beta2), static_cast<double>(step)));
  ctx->launches += fgs::adam_step(a, st);
  FGS_CHECK(cudaGetLastError());
  state->step = step;
  return FGS_OK;
}

int fgs_train_step(fgs_context* ctx, fgs_params* params, const fgs_camera* camera, const float* target,
                   const fgs_train_options* opt, fgs_adam_state* state, double loss_out[3]) {
  if (!ctx) return FGS_EINVAL;
  if (!params || !camera || !target || !opt || !state || !loss_out)
    return fail(ctx, FGS_EINVAL, "train_step: null argument");
  FGS_CHECK(cudaSetDevice(ctx->device));
  const int64_t n = params->n;
  const size_t npix = static_cast<size_t>(camera->width) * camera->height;
  FGS_CHECK(ctx->t_image.ensure(npix * 3));
  FGS_CHECK(ctx->t_dimage.ensure(npix * 3));
  FGS_CHECK(ctx->t_grads.ensure(static_cast<size_t>(n > 0 ? n : 1) * 59));
  const fgs_gaussians scene{n, params->means, params->rotations, params->log_scales, params->opacity_logits, params->sh};
  fgs_render_options ro{opt->sh_degree, 1, {opt->background[0], opt->background[1], opt->background[2]}};
  int rc = fgs_forward(ctx, &scene, camera, &ro, ctx->t_image.p, nullptr, nullptr);
  if (rc != FGS_OK) return rc;
  rc = fgs_l1_dssim_loss(ctx, ctx->t_image.p, target, camera->width, camera->height, opt->lambda, ctx->t_dimage.p,
                         loss_out);
  if (rc != FGS_OK) return rc;
  if (!std::isfinite(loss_out[0])) return fail(ctx, FGS_ENONFINITE, "train: loss diverged (non-finite)");
  float* gb = ctx->t_grads.p;
  const size_t nn = static_cast<size_t>(n);
  fgs_gradients gr{gb, gb + 3 * nn, gb + 7 * nn, gb + 10 * nn, gb + 11 * nn};
  fgs_backward_options bo{{1.f, 1.f, 1.f}, opt->adam.lr_sh_rest != 0.0f ? 1 : 0, 0, 0};
  rc = fgs_backward(ctx, &scene, camera, ctx->t_dimage.p, &bo, &gr);
  if (rc != FGS_OK) return rc;
  return fgs_adam_step(ctx, params, &gr, state, &opt->adam);
}

int fgs_bruteforce_render(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera, int32_t sh_degree,
                          const double background[3], double* image, double* transmittance) {
  if (!ctx) return FGS_EINVAL;
  if (!scene || !camera || !image) return fail(ctx, FGS_EINVAL, "bruteforce_render: null argument");
  if (sh_degree < 0 || sh_degree > 3) return fail(ctx, FGS_EINVAL, "bruteforce_render: sh_degree must be 0..3");
  if (camera->width <= 0 || camera->height <= 0) return fail(ctx, FGS_EINVAL, "bruteforce_render: empty image");
  FGS_CHECK(cudaSetDevice(ctx->device));
  const double zero[3] = {0.0, 0.0, 0.0};
  FGS_CHECK(fgs::bruteforce_render(*scene, *camera, sh_degree, background ? background : zero, image, transmittance,
                                   ctx->stream));
  ctx->launches += 2;
  return FGS_OK;
}

int fgs_bruteforce_render_f64(fgs_context* ctx, int64_t n, const double* means, const double* rotations,
                              const double* log_scales, const double* opacity_logits, const double* sh,
                              const fgs_camera* camera, int32_t sh_degree, const double background[3], double* image,
                              double* transmittance) {
  if (!ctx) return FGS_EINVAL;
  if (!camera || !image || (n > 0 && (!means || !rotations || !log_scales || !opacity_logits || !sh)))
    return fail(ctx, FGS_EINVAL, "bruteforce_render: null argument");
  if (sh_degree < 0 || sh_degree > 3) return fail(ctx, FGS_EINVAL, "bruteforce_render: sh_degree must be 0..3");
  if (camera->width <= 0 || camera->height <= 0) return fail(ctx, FGS_EINVAL, "bruteforce_render: empty image");
  FGS_CHECK(cudaSetDevice(ctx->device));
  const double zero[3] = {0.0, 0.0, 0.0};
  FGS_CHECK(fgs::bruteforce_render_f64(n, means, rotations, log_scales, opacity_logits, sh, *camera, sh_degree,
                                       background ? background : zero, image, transmittance, ctx->stream));
  ctx->launches += 2;
  return FGS_OK;
}

int fgs_timing(fgs_context* ctx, double ms[6], uint64_t calls[2], uint64_t* launches, int reset) {
  if (!ctx) return FGS_EINVAL;
  FGS_CHECK(cudaSetDevice(ctx->device));
  drain_sets(ctx, 0);
  if (ms)
    for (int k = 0; k < 6; ++k) ms[k] = ctx->acc_ms[k];
  if (calls) {
    calls[0] = ctx->acc_calls[0];
    calls[1] = ctx->acc_calls[1];
  }
  if (launches) *launches = ctx->launches;
  if (reset) {
    for (double& v : ctx->acc_ms) v = 0.0;
    ctx->acc_calls[0] = ctx->acc_calls[1] = 0;
    ctx->launches = 0;
  }
  return FGS_OK;
}

int fgs_measure_fp32_peak(fgs_context* ctx, double* ops_per_s) {
  if (!ctx || !ops_per_s) return FGS_EINVAL;
  FGS_CHECK(cudaSetDevice(ctx->device));
  *ops_per_s = fgs::fp32_peak_probe(ctx->stream);
  FGS_CHECK(cudaGetLastError());
  return FGS_OK;
}

int fgs_selftest_crmath(fgs_context* ctx, int which, uint64_t begin, uint64_t count, uint64_t seed, uint64_t out[3]) {
  if (!ctx || !out || which < 0 || which > 2) return FGS_EINVAL;
  FGS_CHECK(cudaSetDevice(ctx->device));
  unsigned long long* d = nullptr;
  FGS_CHECK(cudaMalloc(&d, 3 * sizeof(unsigned long long)));
  cudaError_t e = cudaMemsetAsync(d, 0, 3 * sizeof(unsigned long long), ctx->stream);
  if (e == cudaSuccess) {
    fgs::crmath_selftest(which, begin, count, seed, d, ctx->stream);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d);
  FGS_CHECK(e);
  return FGS_OK;
}

int64_t fgs_debug_get(fgs_context* ctx, const char* name, void* dst, int64_t dst_bytes) {
  if (!ctx || !name || !ctx->have_fwd) return -1;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return -1;
  cudaStream_t st = ctx->stream;
  const std::string nm(name);
  const size_t n = static_cast<size_t>(ctx->n), I = static_cast<size_t>(ctx->num_isect);
  const size_t npix = static_cast<size_t>(ctx->cam.width) * ctx->cam.height;
  const size_t nt = static_cast<size_t>(ctx->tiles_x) * ctx->tiles_y;
  auto copy = [&](const void* src, size_t bytes) -> int64_t {
    if (!dst) return static_cast<int64_t>(bytes);
    if (static_cast<int64_t>(bytes) > dst_bytes) return -1;
    if (bytes && cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess) return -1;
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    return static_cast<int64_t>(bytes);
  };
  if (nm == "state_u8") return copy(ctx->state.p, n);
  if (nm == "rec") return copy(ctx->rec.p, n * sizeof(fgs::SortedRec));
  if (nm == "depth_key") return copy(ctx->dkey.p, n * 4);
  if (nm == "radius") return copy(ctx->radii.p, n * 4);
  if (nm == "touched") return copy(ctx->touched.p, n * 4);
  if (nm == "sorted_gauss") return copy(ctx->sorted_gauss.p, I * 4);
  // hot-path state: the 64-bit (depth key << 32 | Gaussian id) keys as K2's scatter left them in
  // each tile's range (K3 sorts lists of <= 4096 keys in shared memory, longer ones in place)
  if (nm == "keys") return copy(ctx->keys.p, I * 8);
  if (nm == "rect") return copy(ctx->rect.p, n * sizeof(ushort4));
  if (nm == "compact_gauss") return copy(ctx->cval.p, static_cast<size_t>(ctx->num_compact) * 4);
  if (nm == "compact_offsets") return copy(ctx->coff.p, static_cast<size_t>(ctx->num_compact) * 4);
  if (nm == "sorted_tile") {
    // tile id of every sorted entry, expanded from the tile ranges
    if (!dst) return static_cast<int64_t>(I * 4);
    if (static_cast<int64_t>(I * 4) > dst_bytes) return -1;
    std::vector<uint32_t> off(nt + 1);
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    if (cudaMemcpy(off.data(), ctx->tile_offsets.p, (nt + 1) * 4, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    auto* out = static_cast<uint32_t*>(dst);
    for (size_t t = 0; t < nt; ++t)
      for (uint32_t k = off[t]; k < off[t + 1] && k < I; ++k) out[k] = static_cast<uint32_t>(t);
    return static_cast<int64_t>(I * 4);
  }
  if (nm == "offsets") return copy(ctx->tile_offsets.p, (nt + 1) * 4);
  if (nm == "variants") {  // launch variants of the last forward / backward, longest tile list
    const uint32_t v[6] = {static_cast<uint32_t>(ctx->var_fwd_px), static_cast<uint32_t>(ctx->var_bwd_px),
                           static_cast<uint32_t>(ctx->var_k4b), ctx->longest,
                           static_cast<uint32_t>(ctx->var_row_scatter), static_cast<uint32_t>(ctx->var_bin_local)};
    if (!dst) return sizeof(v);
    if (dst_bytes < static_cast<int64_t>(sizeof(v))) return -1;
    std::memcpy(dst, v, sizeof(v));
    return sizeof(v);
  }
  if (nm == "aux_bytes") {  // device bytes the path holds (RenderStats::peak_aux_bytes, incl. backward scratch)
    const uint64_t v = path_bytes(ctx);
    if (!dst) return sizeof(v);
    if (dst_bytes < static_cast<int64_t>(sizeof(v))) return -1;
    std::memcpy(dst, &v, sizeof(v));
    return sizeof(v);
  }
  if (nm == "final_T") return copy(ctx->final_T.p, npix * 4);
  if (nm == "blend_count") return ctx->have_blend_count ? copy(ctx->blend_count.p, npix * 2) : -1;
  if (nm == "last") return copy(ctx->last.p, npix * 4);
  if (nm == "counters") return copy(ctx->counters.p, 4 * sizeof(unsigned long long));
  if (nm == "counters16") return copy(ctx->counters.p, 16 * sizeof(unsigned long long));
  if (nm == "bin_trace") return copy(ctx->counters.p + 16, 8 * sizeof(unsigned long long));
  if (nm == "tile_cycles") return copy(ctx->tile_cycles.p, nt * sizeof(unsigned long long));
  if (nm == "tile_span") return copy(ctx->tile_span.p, 2 * nt * sizeof(unsigned long long));
  if (nm == "tile_span_bwd") return copy(ctx->tile_span_bwd.p, 2 * nt * sizeof(unsigned long long));
  if (nm == "key_tile" || nm == "key_depth" || nm == "key_gauss") {
    if (!dst) return static_cast<int64_t>(I * 4);
    // Recompute the reference's pre-sort emission order (source order) on demand.
    DevBuf<uint32_t> kt, kd, kg;
    if (kt.ensure(I + 1) || kd.ensure(I + 1) || kg.ensure(I + 1)) return -1;
    fgs::BinArgs a = ctx->bin_args;
    if (fgs::debug_source_order_keys(a, kt.p, kd.p, kg.p, st) != cudaSuccess) return -1;
    const uint32_t* src = nm == "key_tile" ? kt.p : (nm == "key_depth" ? kd.p : kg.p);
    const int64_t r = copy(src, I * 4);
    for (auto* b : {&kt, &kd, &kg}) b->release();
    return r;
  }
  return -1;
}

}  // extern "C"
