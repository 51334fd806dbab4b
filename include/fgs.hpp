// fgs.hpp — header-only C++ wrapper over the C ABI (include/fgs.h) with the reference's
// calling convention and exception types.
//
// Reference API being replaced (omnisplat, /root/reference/proj/include/omnisplat/):
//   RenderResult<float> render(const Scene<float>&, const Camera<float>&, const RenderOptions<float>&)
//       splatting.hpp:330-374
//   GradientBuffer<float> backward(const Scene<float>&, const Camera<float>&,
//                                  const ForwardContext<float>&, const ImageBuffer<float>&,
//                                  const BackwardOptions<float>&)          gradients.hpp:207-267
// The reference throws std::invalid_argument for a zero quaternion, a dL/dimage shape mismatch
// and a scene/camera that differs from the forward context; so does this wrapper.
#ifndef FGS_HPP_
#define FGS_HPP_

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fgs.h"

namespace fgs {

struct SceneSoA {  // host arrays, the reference's Gaussian3D fields as structure-of-arrays
  std::vector<float> means, rotations, log_scales, opacity_logits, sh;  // N*3, N*4, N*3, N, N*48
  std::array<float, 3> background{0.f, 0.f, 0.f};
  int64_t size() const { return static_cast<int64_t>(opacity_logits.size()); }
  fgs_gaussians view() const {
    return fgs_gaussians{size(), means.data(), rotations.data(), log_scales.data(), opacity_logits.data(), sh.data()};
  }
};

struct Image {  // ImageBuffer<float> (inc/model.hpp:53-92): row-major RGB
  int width = 0, height = 0;
  std::vector<float> pixels;
};

struct Gradients {  // GradientBuffer (inc/gradients.hpp:20-46) with all 48 SH coefficients
  std::vector<float> d_means, d_rotations, d_log_scales, d_opacity_logits, d_sh;
};

struct RenderResult {
  Image image;
  fgs_stats stats{};
  std::vector<int32_t> radii;
};

inline void throw_on(int rc, const fgs_context* ctx) {
  if (rc == FGS_OK) return;
  const std::string msg = fgs_last_error(ctx);
  if (rc == FGS_EINVAL || rc == FGS_EDEGENERATE_QUAT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// One device context = the reference's ForwardContext holder. Not thread-safe.
class Renderer {
 public:
  explicit Renderer(int device = 0) {
    if (fgs_create(device, &ctx_) != FGS_OK) throw std::runtime_error("fgs_create failed (no CUDA device?)");
  }
  ~Renderer() { fgs_destroy(ctx_); }
  Renderer(const Renderer&) = delete;
  Renderer& operator=(const Renderer&) = delete;

  RenderResult render(const SceneSoA& scene, const fgs_camera& camera, int sh_degree = 3) {
    RenderResult r;
    r.image.width = camera.width;
    r.image.height = camera.height;
    r.image.pixels.resize(static_cast<size_t>(camera.width) * camera.height * 3);
    r.radii.resize(static_cast<size_t>(scene.size()));
    fgs_render_options o{sh_degree, 1, {scene.background[0], scene.background[1], scene.background[2]}};
    const fgs_gaussians g = scene.view();
    throw_on(fgs_render_host(ctx_, &g, &camera, &o, r.image.pixels.data(), r.radii.data(), &r.stats), ctx_);
    return r;
  }

  Gradients backward(const SceneSoA& scene, const fgs_camera& camera, const Image& dl_dimage, bool full_sh = true) {
    if (dl_dimage.width != camera.width || dl_dimage.height != camera.height)
      throw std::invalid_argument("rasterize_backward: image gradient shape does not match context");
    const size_t n = static_cast<size_t>(scene.size());
    Gradients out;
    out.d_means.assign(n * 3, 0.f);
    out.d_rotations.assign(n * 4, 0.f);
    out.d_log_scales.assign(n * 3, 0.f);
    out.d_opacity_logits.assign(n, 0.f);
    out.d_sh.assign(n * 48, 0.f);
    fgs_gradients gr{out.d_means.data(), out.d_rotations.data(), out.d_log_scales.data(), out.d_opacity_logits.data(),
                     out.d_sh.data()};
    fgs_backward_options o{{1.f, 1.f, 1.f}, full_sh ? 1 : 0, 0, 0};
    const fgs_gaussians g = scene.view();
    throw_on(fgs_backward_host(ctx_, &g, &camera, dl_dimage.pixels.data(), &o, &gr), ctx_);
    return out;
  }

  // A stream of frames (fgs_render_host_async): the image goes into `image` (width * height * 3
  // floats, caller-owned, ideally page-locked) -- valid after wait(); the scene must stay
  // unchanged until then. Returns the frame's statistics.
  fgs_stats render_async(const SceneSoA& scene, const fgs_camera& camera, float* image, int sh_degree = 3) {
    fgs_render_options o{sh_degree, 1, {scene.background[0], scene.background[1], scene.background[2]}};
    const fgs_gaussians g = scene.view();
    fgs_stats st{};
    throw_on(fgs_render_host_async(ctx_, &g, &camera, &o, image, nullptr, &st), ctx_);
    return st;
  }
  void wait() { throw_on(fgs_wait(ctx_), ctx_); }

  fgs_context* handle() { return ctx_; }

 private:
  fgs_context* ctx_ = nullptr;
};

inline fgs_camera fisheye_camera(int w, int h, float fx, float fy, float cx, float cy,
                                 float fov_max = 1.5707963267948966f) {
  fgs_camera c{};
  c.model = FGS_CAMERA_FISHEYE;
  c.width = w;
  c.height = h;
  c.fx = fx;
  c.fy = fy;
  c.cx = cx;
  c.cy = cy;
  c.rotation_wc[0] = c.rotation_wc[4] = c.rotation_wc[8] = 1.f;
  c.fov_max = fov_max;
  return c;
}

}  // namespace fgs

#endif  // FGS_HPP_
