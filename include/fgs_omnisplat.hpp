// fgs_omnisplat.hpp — the drop-in for the reference's own C++ types: render / backward taking
// omnisplat::Scene<float> / Camera<float> and returning omnisplat::RenderResult<float> (image,
// RenderStats, a complete ForwardContext) / GradientBuffer<float>, computed on the B200 through the
// C ABI (include/fgs.h).
//
// Replaces (omnisplat, /root/reference/proj/include/omnisplat/):
//   template <S> RenderResult<S> render(const Scene<S>&, const Camera<S>&, const RenderOptions<S>&)
//       splatting.hpp:330-374
//   template <S> GradientBuffer<S> backward(const Scene<S>&, const Camera<S>&, const ForwardContext<S>&,
//                                           const ImageBuffer<S>&, const BackwardOptions<S>&)
//       gradients.hpp:207-267
// A caller such as cmd_bench (src/cli.cpp:138-170) switches by calling fgs::omni::render instead of
// omnisplat::render (tools/omnisplat_bench.cpp does exactly that). Include the reference's headers
// (with Eigen, or this repo's oracle/eigen_shim) before this one.
//
// Data path: the scene's std::vector<Gaussian3D<float>> goes to the device as one block and is
// split into the structure-of-arrays layout there (fgs_render_host_aos, field offsets taken from
// the record type); the context is filled from the GPU forward state: the kept splats in source
// order (Splat2D, with their camera-space means), the tile ranges and sorted splat references,
// the per-pixel final transmittance and blend count.
//
// Errors: the reference's std::invalid_argument messages for a zero quaternion, a context built for
// another scene / camera and a dL/dimage shape mismatch; std::runtime_error otherwise.
#ifndef FGS_OMNISPLAT_HPP_
#define FGS_OMNISPLAT_HPP_

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fgs.h"
#include "omnisplat/gradients.hpp"
#include "omnisplat/splatting.hpp"

namespace fgs {
namespace omni {

inline void check(int rc, const fgs_context* ctx) {
  if (rc == FGS_OK) return;
  const std::string msg = fgs_last_error(ctx);
  if (rc == FGS_EINVAL || rc == FGS_EDEGENERATE_QUAT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// The AoS record layout of Gaussian3D<float> (inc/model.hpp:18-36), from a probe record: the
// Eigen fixed-size members store their floats contiguously, ShCoeffs column-major (= [c*16 + j]).
inline fgs_gaussians_aos aos_view(const omnisplat::Scene<float>& s) {
  using G = omnisplat::Gaussian3D<float>;
  const G probe{};
  const char* base = reinterpret_cast<const char*>(&probe);
  auto off = [&](const float* p) { return static_cast<int64_t>(reinterpret_cast<const char*>(p) - base); };
  fgs_gaussians_aos a{};
  a.n = static_cast<int64_t>(s.gaussians.size());
  a.data = s.gaussians.data();
  a.stride = static_cast<int64_t>(sizeof(G));
  a.off_mean = off(probe.mean.data());
  a.off_rotation = off(probe.rotation.data());
  a.off_log_scale = off(probe.log_scale.data());
  a.off_opacity_logit = off(&probe.opacity_logit);
  a.off_sh = off(probe.sh.data());
  return a;
}

inline fgs_camera to_fgs(const omnisplat::Camera<float>& c) {
  fgs_camera o{};
  o.model = static_cast<int32_t>(c.model);  // Pinhole 0, FisheyeEquidistant 1, Panorama 2 (cameras.hpp:13)
  o.width = c.width;
  o.height = c.height;
  o.fx = c.fx;
  o.fy = c.fy;
  o.cx = c.cx;
  o.cy = c.cy;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) o.rotation_wc[r * 3 + k] = c.rotation_wc(r, k);
  for (int r = 0; r < 3; ++r) o.translation_wc[r] = c.translation_wc[r];
  o.fov_max = c.fov_max;
  return o;
}

// One device context; render() leaves the GPU forward state that backward() consumes.
class Renderer {
 public:
  explicit Renderer(int device = 0) {
    if (fgs_create(device, &ctx_) != FGS_OK) throw std::runtime_error("fgs_create failed (no CUDA device?)");
  }
  ~Renderer() { fgs_destroy(ctx_); }
  Renderer(const Renderer&) = delete;
  Renderer& operator=(const Renderer&) = delete;
  fgs_context* handle() { return ctx_; }

  omnisplat::RenderResult<float> render(const omnisplat::Scene<float>& scene, const omnisplat::Camera<float>& camera,
                                        const omnisplat::RenderOptions<float>& options = {}) {
    const omnisplat::Vec3<float> bg = options.background.value_or(scene.background);
    omnisplat::RenderResult<float> out;
    forward(scene, camera, options.sh_degree, bg, &out.image, &out.stats);
    fill_context(scene, camera, options.sh_degree, bg, &out.context);
    key_ = out.context.final_transmittance.data();
    return out;
  }

  omnisplat::GradientBuffer<float> backward(const omnisplat::Scene<float>& scene,
                                            const omnisplat::Camera<float>& camera,
                                            const omnisplat::ForwardContext<float>& ctx,
                                            const omnisplat::ImageBuffer<float>& dl_dimage,
                                            const omnisplat::BackwardOptions<float>& options = {}) {
    // the reference's argument checks, in its order (gradients.hpp:211-218, :73-74)
    if (ctx.scene_size != scene.gaussians.size())
      throw std::invalid_argument("backward: forward context was built for a different scene");
    const auto& a = ctx.camera;
    if (a.model != camera.model || a.width != camera.width || a.height != camera.height || a.fx != camera.fx ||
        a.fy != camera.fy || a.cx != camera.cx || a.cy != camera.cy || a.rotation_wc != camera.rotation_wc ||
        a.translation_wc != camera.translation_wc)
      throw std::invalid_argument("backward: forward context was built for a different camera");
    if (dl_dimage.width != a.width || dl_dimage.height != a.height)
      throw std::invalid_argument("rasterize_backward: image gradient shape does not match context");
    // the device holds the state of the last render(); a context from an earlier one is rebuilt
    // first (the forward is deterministic, so its state is the same)
    if (ctx.final_transmittance.data() != key_ || key_ == nullptr) {
      forward(scene, ctx.camera, ctx.sh_degree, ctx.background, nullptr, nullptr);
      key_ = ctx.final_transmittance.data();
    }
    const size_t n = scene.gaussians.size();
    std::vector<float> g(n * 59, 0.f);
    fgs_gradients gr{g.data(), g.data() + 3 * n, g.data() + 7 * n, g.data() + 10 * n, g.data() + 11 * n};
    fgs_backward_options bo{{options.jacobian_grad_scale[0], options.jacobian_grad_scale[1],
                             options.jacobian_grad_scale[2]},
                            0 /* DC-only SH gradients: the reference's GradientBuffer */, 0, 0};
    const fgs_gaussians_aos s = aos_view(scene);
    const fgs_camera c = to_fgs(camera);
    check(fgs_backward_host_aos(ctx_, &s, &c, dl_dimage.pixels.data(), &bo, &gr), ctx_);
    omnisplat::GradientBuffer<float> buf;
    buf.resize_zero(n);
    for (size_t i = 0; i < n; ++i) {
      buf.d_mean[i] = omnisplat::Vec3<float>(gr.d_means[3 * i], gr.d_means[3 * i + 1], gr.d_means[3 * i + 2]);
      buf.d_rotation[i] = omnisplat::Vec4<float>(gr.d_rotations[4 * i], gr.d_rotations[4 * i + 1],
                                                 gr.d_rotations[4 * i + 2], gr.d_rotations[4 * i + 3]);
      buf.d_log_scale[i] =
          omnisplat::Vec3<float>(gr.d_log_scales[3 * i], gr.d_log_scales[3 * i + 1], gr.d_log_scales[3 * i + 2]);
      buf.d_opacity_logit[i] = gr.d_opacity_logits[i];
      buf.d_sh_dc[i] = omnisplat::Vec3<float>(gr.d_sh[48 * i], gr.d_sh[48 * i + 16], gr.d_sh[48 * i + 32]);
    }
    return buf;
  }

 private:
  fgs_context* ctx_ = nullptr;
  const float* key_ = nullptr;  // final_transmittance buffer of the context the device state belongs to

  void forward(const omnisplat::Scene<float>& scene, const omnisplat::Camera<float>& camera, int sh_degree,
               const omnisplat::Vec3<float>& bg, omnisplat::ImageBuffer<float>* image, omnisplat::RenderStats* stats) {
    const fgs_gaussians_aos s = aos_view(scene);
    const fgs_camera c = to_fgs(camera);
    fgs_render_options o{sh_degree, 1, {bg[0], bg[1], bg[2]}};
    std::vector<float> scratch;
    float* pix = nullptr;
    if (image) {
      *image = omnisplat::ImageBuffer<float>(camera.width, camera.height);
      pix = image->pixels.data();
    } else {
      scratch.resize(static_cast<size_t>(camera.width) * camera.height * 3);
      pix = scratch.data();
    }
    fgs_stats st{};
    check(fgs_set_flags(ctx_, FGS_FLAG_BLEND_COUNT), ctx_);
    check(fgs_render_host_aos(ctx_, &s, &c, &o, pix, nullptr, &st), ctx_);
    if (stats) {
      stats->num_intersections = st.num_intersections;
      stats->num_splats = st.num_splats;
      stats->num_culled = st.num_culled;
      stats->num_degenerate = st.num_degenerate;
      stats->preprocess_ms = st.preprocess_ms;
      stats->binning_ms = st.binning_ms;
      stats->sort_ms = st.sort_ms;
      stats->raster_ms = st.raster_ms;
      stats->peak_aux_bytes = static_cast<size_t>(st.peak_aux_bytes);
    }
  }

  template <typename T>
  std::vector<T> get(const char* name) {
    const int64_t bytes = fgs_debug_get(ctx_, name, nullptr, 0);
    if (bytes < 0) throw std::runtime_error(std::string("forward state '") + name + "' unavailable");
    std::vector<T> v(static_cast<size_t>(bytes) / sizeof(T));
    if (fgs_debug_get(ctx_, name, v.data(), bytes) != bytes) throw std::runtime_error(std::string("reading ") + name);
    return v;
  }

  // ForwardContext (splatting.hpp:309-321) from the GPU state of the last forward.
  void fill_context(const omnisplat::Scene<float>& scene, const omnisplat::Camera<float>& camera, int sh_degree,
                    const omnisplat::Vec3<float>& bg, omnisplat::ForwardContext<float>* cx) {
    cx->camera = camera;
    cx->scene_size = scene.gaussians.size();
    cx->sh_degree = sh_degree;
    cx->background = bg;
    const std::vector<uint8_t> state = get<uint8_t>("state_u8");
    const std::vector<float> rec = get<float>("rec");  // 12 floats per Gaussian (fgs.h)
    const std::vector<uint32_t> dkey = get<uint32_t>("depth_key");
    const std::vector<int32_t> radius = get<int32_t>("radius");
    // kept splats in source order (the reference's stable compaction, splatting.hpp:125-138)
    std::vector<int32_t> splat_of(state.size(), -1);
    for (size_t i = 0; i < state.size(); ++i) {
      if (state[i] != 1) continue;
      splat_of[i] = static_cast<int32_t>(cx->splats.size());
      const float* r = rec.data() + 12 * i;
      omnisplat::Splat2D<float> sp;
      sp.mean_px = omnisplat::Vec2<float>(r[0], r[1]);
      sp.conic = omnisplat::Vec3<float>(-2.0f * r[2], r[3], -2.0f * r[4]);  // the record holds -a/2, -c/2
      const uint32_t bits = dkey[i] & 0x7FFFFFFFu;  // positive depth: the key is the bits | 0x80000000
      std::memcpy(&sp.depth, &bits, 4);
      sp.radius_px = radius[i];
      sp.color = omnisplat::Vec3<float>(r[6], r[7], r[8]);
      sp.alpha_max = r[5];
      sp.source_index = static_cast<int>(i);
      cx->splats.push_back(sp);
      cx->cam_points.push_back(omnisplat::world_to_camera(scene.gaussians[i].mean, camera));
    }
    const int tx = (camera.width + 15) / 16, ty = (camera.height + 15) / 16;
    cx->tiles.tiles_x = tx;
    cx->tiles.tiles_y = ty;
    cx->tiles.offsets = get<uint32_t>("offsets");
    const std::vector<uint32_t> sorted = get<uint32_t>("sorted_gauss");
    cx->refs.resize(sorted.size());
    for (size_t k = 0; k < sorted.size(); ++k) cx->refs[k] = static_cast<uint32_t>(splat_of[sorted[k]]);
    cx->final_transmittance = get<float>("final_T");
    cx->blend_count = get<uint16_t>("blend_count");
  }
};

inline Renderer& default_renderer() {
  thread_local std::unique_ptr<Renderer> r;
  if (!r) r.reset(new Renderer(0));
  return *r;
}

// Drop-in free functions (the reference's signatures, S = float).
inline omnisplat::RenderResult<float> render(const omnisplat::Scene<float>& scene,
                                             const omnisplat::Camera<float>& camera,
                                             const omnisplat::RenderOptions<float>& options = {}) {
  return default_renderer().render(scene, camera, options);
}

inline omnisplat::GradientBuffer<float> backward(const omnisplat::Scene<float>& scene,
                                                 const omnisplat::Camera<float>& camera,
                                                 const omnisplat::ForwardContext<float>& ctx,
                                                 const omnisplat::ImageBuffer<float>& dl_dimage,
                                                 const omnisplat::BackwardOptions<float>& options = {}) {
  return default_renderer().backward(scene, camera, ctx, dl_dimage, options);
}

}  // namespace omni
}  // namespace fgs

#endif  // FGS_OMNISPLAT_HPP_
