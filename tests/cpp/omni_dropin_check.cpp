// Drop-in check (tests/test_omnisplat_dropin.py): the same omnisplat::Scene<float> / Camera<float>
// through the reference's own render / backward (its headers, compiled here against the repo's
// Eigen shim; CPU) and through fgs::omni::render / backward (include/fgs_omnisplat.hpp; B200). Prints
// one JSON line of agreement metrics; the Python test holds the bars. Built by
// paper_2409_04751_b200/build.py where the reference headers are mounted.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>

#include "omnisplat/gradients.hpp"
#include "omnisplat/splatting.hpp"
#include "../../include/fgs_omnisplat.hpp"

using omnisplat::Camera;
using omnisplat::Scene;

namespace {

Scene<float> make_scene(int n, uint32_t seed) {
  std::mt19937 rng(seed);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::uniform_real_distribution<float> ud(0.f, 1.f);
  Scene<float> s;
  s.gaussians.resize(static_cast<size_t>(n));
  for (auto& g : s.gaussians) {
    float d[3] = {nd(rng), nd(rng), nd(rng)};
    const float len = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    const float r = std::cbrt(1.f + 999.f * ud(rng));
    for (int k = 0; k < 3; ++k) g.mean[k] = d[k] / len * r;
    for (int k = 0; k < 4; ++k) g.rotation[k] = nd(rng);
    for (int k = 0; k < 3; ++k) g.log_scale[k] = -3.5f + 0.5f * nd(rng);
    g.opacity_logit = nd(rng);
    for (int c = 0; c < 3; ++c)
      for (int j = 0; j < 16; ++j) g.sh(j, c) = (j == 0 ? 0.3f : 0.05f) * nd(rng);
  }
  return s;
}

double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

template <typename V>
void flat(const std::vector<V>& v, int w, std::vector<double>* out) {
  for (const auto& x : v)
    for (int k = 0; k < w; ++k) out->push_back(static_cast<double>(x[k]));
}

}  // namespace

int main() {
  const int W = 640, H = 480;
  const float f = 0.5f * std::hypot(float(W), float(H)) / 1.5707964f;
  Camera<float> cam = Camera<float>::fisheye(W, H, f, f, W / 2.f, H / 2.f);
  const Eigen::Matrix<float, 3, 3> rot = Eigen::AngleAxis<float>(0.3f, Eigen::Matrix<float, 3, 1>(0.f, 1.f, 0.f)).toRotationMatrix();
  cam.rotation_wc = rot;
  cam.translation_wc = Eigen::Matrix<float, 3, 1>(0.1f, -0.2f, 0.3f);
  const Scene<float> scene = make_scene(20000, 7u);
  omnisplat::RenderOptions<float> opts;
  opts.sh_degree = 3;

  const auto ref = omnisplat::render(scene, cam, opts);
  const auto gpu = fgs::omni::render(scene, cam, opts);

  double max_abs = 0, mse = 0;
  for (size_t i = 0; i < ref.image.pixels.size(); ++i) {
    const double d = double(gpu.image.pixels[i]) - double(ref.image.pixels[i]);
    max_abs = std::max(max_abs, std::fabs(d));
    mse += d * d;
  }
  mse /= double(ref.image.pixels.size());
  const double psnr = mse > 0 ? 10 * std::log10(1.0 / mse) : 999.0;
  size_t bc_equal = 0, off_equal = 0;
  double t_max = 0;
  for (size_t p = 0; p < ref.context.blend_count.size(); ++p) {
    bc_equal += ref.context.blend_count[p] == gpu.context.blend_count[p];
    t_max = std::max(t_max, std::fabs(double(ref.context.final_transmittance[p]) - gpu.context.final_transmittance[p]));
  }
  for (size_t t = 0; t < ref.context.tiles.offsets.size(); ++t) off_equal += ref.context.tiles.offsets[t] == gpu.context.tiles.offsets[t];
  // splats: same Gaussians kept, same fields
  size_t src_equal = 0;
  double mean_px_max = 0;
  const size_t ns = std::min(ref.context.splats.size(), gpu.context.splats.size());
  for (size_t i = 0; i < ns; ++i) {
    src_equal += ref.context.splats[i].source_index == gpu.context.splats[i].source_index;
    for (int k = 0; k < 2; ++k)
      mean_px_max = std::max(mean_px_max, double(std::fabs(ref.context.splats[i].mean_px[k] - gpu.context.splats[i].mean_px[k])));
  }
  size_t refs_equal = 0;
  const size_t nr = std::min(ref.context.refs.size(), gpu.context.refs.size());
  for (size_t k = 0; k < nr; ++k) refs_equal += ref.context.refs[k] == gpu.context.refs[k];

  // backward on the same dL/dimage
  omnisplat::ImageBuffer<float> dl(W, H);
  std::mt19937 rng(11u);
  std::normal_distribution<float> nd(0.f, 1.f);
  for (auto& v : dl.pixels) v = nd(rng);
  const auto gref = omnisplat::backward(scene, cam, ref.context, dl);
  const auto ggpu = fgs::omni::backward(scene, cam, gpu.context, dl);
  std::vector<double> a, b;
  double e_mean, e_rot, e_ls, e_op, e_sh;
  a.clear(); b.clear(); flat(ggpu.d_mean, 3, &a); flat(gref.d_mean, 3, &b); e_mean = rel_l2(a, b);
  a.clear(); b.clear(); flat(ggpu.d_rotation, 4, &a); flat(gref.d_rotation, 4, &b); e_rot = rel_l2(a, b);
  a.clear(); b.clear(); flat(ggpu.d_log_scale, 3, &a); flat(gref.d_log_scale, 3, &b); e_ls = rel_l2(a, b);
  a.clear(); b.clear();
  for (float v : ggpu.d_opacity_logit) a.push_back(v);
  for (float v : gref.d_opacity_logit) b.push_back(v);
  e_op = rel_l2(a, b);
  a.clear(); b.clear(); flat(ggpu.d_sh_dc, 3, &a); flat(gref.d_sh_dc, 3, &b); e_sh = rel_l2(a, b);
  // a context from an earlier render (the device state is rebuilt) gives the same gradients
  Camera<float> cam2 = cam;
  cam2.translation_wc[0] += 0.5f;
  const auto other = fgs::omni::render(scene, cam2, opts);
  const auto ggpu2 = fgs::omni::backward(scene, cam, gpu.context, dl);
  a.clear(); b.clear(); flat(ggpu2.d_mean, 3, &a); flat(ggpu.d_mean, 3, &b);
  const double e_rebuild = rel_l2(a, b);

  // the reference's error behaviour
  std::string err_cam, err_shape, err_quat;
  try {
    fgs::omni::backward(scene, cam2, gpu.context, dl);
  } catch (const std::invalid_argument& e) {
    err_cam = e.what();
  }
  try {
    fgs::omni::backward(scene, cam, gpu.context, omnisplat::ImageBuffer<float>(W - 1, H));
  } catch (const std::invalid_argument& e) {
    err_shape = e.what();
  }
  Scene<float> bad = scene;
  bad.gaussians[static_cast<size_t>(gpu.context.splats[0].source_index)].rotation.setZero();  // a visible one
  try {
    fgs::omni::render(bad, cam, opts);
  } catch (const std::invalid_argument& e) {
    err_quat = e.what();
  }
  (void)other;
  std::printf(
      "{\"image_max_abs\": %.3g, \"psnr\": %.2f, \"isect_ref\": %llu, \"isect_gpu\": %llu, \"splats_ref\": %zu, "
      "\"splats_gpu\": %zu, \"src_equal\": %zu, \"mean_px_max\": %.3g, \"offsets_equal\": %zu, \"tiles\": %zu, "
      "\"refs_equal\": %zu, \"refs\": %zu, \"blend_count_equal\": %zu, \"pixels\": %zu, \"final_T_max\": %.3g, "
      "\"grad_mean\": %.3g, \"grad_rotation\": %.3g, \"grad_log_scale\": %.3g, \"grad_opacity\": %.3g, "
      "\"grad_sh_dc\": %.3g, \"grad_rebuilt\": %.3g, \"err_camera\": \"%s\", \"err_shape\": \"%s\", "
      "\"err_quat\": \"%s\"}\n",
      max_abs, psnr, (unsigned long long)ref.stats.num_intersections, (unsigned long long)gpu.stats.num_intersections,
      ref.context.splats.size(), gpu.context.splats.size(), src_equal, mean_px_max, off_equal,
      ref.context.tiles.offsets.size(), refs_equal, ref.context.refs.size(), bc_equal, ref.context.blend_count.size(),
      t_max, e_mean, e_rot, e_ls, e_op, e_sh, e_rebuild, err_cam.c_str(), err_shape.c_str(), err_quat.c_str());
  return 0;
}
