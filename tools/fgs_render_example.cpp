// fgs_render_example — C++ host program over the C ABI via include/fgs.hpp: renders a seeded
// synthetic fisheye scene, runs a backward pass with dL/dimage = image, prints a key=value
// stats line in the style of the reference's `bench` command (src/cli.cpp:138-170).
//   fgs_render_example [n_gaussians] [width] [height]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "../include/fgs.hpp"

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 20000;
  const int w = argc > 2 ? std::atoi(argv[2]) : 512;
  const int h = argc > 3 ? std::atoi(argv[3]) : 384;
  std::mt19937_64 rng(0);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::uniform_real_distribution<float> ud(0.f, 1.f);
  fgs::SceneSoA s;
  s.means.resize(n * 3);
  s.rotations.resize(n * 4);
  s.log_scales.resize(n * 3);
  s.opacity_logits.resize(n);
  s.sh.assign(static_cast<size_t>(n) * 48, 0.f);
  for (int i = 0; i < n; ++i) {
    float d[3] = {nd(rng), nd(rng), nd(rng)};
    const float len = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]) + 1e-6f;
    const float r = std::cbrt(1.f + 999.f * ud(rng));
    for (int k = 0; k < 3; ++k) s.means[i * 3 + k] = d[k] / len * r;
    for (int k = 0; k < 4; ++k) s.rotations[i * 4 + k] = nd(rng);
    for (int k = 0; k < 3; ++k) s.log_scales[i * 3 + k] = -3.0f + 0.5f * nd(rng);
    s.opacity_logits[i] = nd(rng);
    for (int c = 0; c < 3; ++c) s.sh[i * 48 + c * 16] = 0.3f * nd(rng);
  }
  const float f = 0.5f * std::hypot(float(w), float(h)) / 1.5707963f;
  const fgs_camera cam = fgs::fisheye_camera(w, h, f, f, w / 2.f, h / 2.f);
  try {
    fgs::Renderer r(0);
    const auto t0 = std::chrono::steady_clock::now();
    const fgs::RenderResult res = r.render(s, cam, 3);
    const auto t1 = std::chrono::steady_clock::now();
    fgs::Image dl = res.image;
    const fgs::Gradients g = r.backward(s, cam, dl);
    double gsum = 0;
    for (float v : g.d_means) gsum += std::fabs(v);
    double mean = 0;
    for (float v : res.image.pixels) mean += v;
    mean /= res.image.pixels.size();
    std::printf("gaussians=%d width=%d height=%d intersections=%llu splats=%u culled=%u render_ms=%.3f "
                "image_mean=%.6f grad_mean_l1=%.6e\n",
                n, w, h, static_cast<unsigned long long>(res.stats.num_intersections), res.stats.num_splats,
                res.stats.num_culled, std::chrono::duration<double, std::milli>(t1 - t0).count(), mean, gsum);
    // the reference's error behaviour: mismatched dL/dimage shape -> std::invalid_argument
    fgs::Image bad;
    bad.width = 2;
    bad.height = 2;
    bad.pixels.assign(12, 0.f);
    try {
      r.backward(s, cam, bad);
      std::printf("error_check=missing\n");
      return 1;
    } catch (const std::invalid_argument&) {
      std::printf("error_check=ok\n");
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
