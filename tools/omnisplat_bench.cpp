// omnisplat_bench — the reference CLI's `bench` subcommand (cmd_bench, src/cli.cpp:138-170), written
// against the reference's own types (omnisplat::Scene<float>, Camera<float>, RenderResult<float>)
// with one change: render() is fgs::omni::render, the B200 drop-in of include/fgs_omnisplat.hpp.
// Built only where the reference headers are mounted (paper_2409_04751_b200/build.py), against this
// repo's Eigen-subset shim (oracle/eigen_shim). Scene and cameras are read with include/fgs_io.hpp
// (the reference's readers need nlohmann-json, which is not installed).
//
//   omnisplat_bench --scene s.ply --cameras c.json [--repeat r]
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <iostream>
#include <map>
#include <string>

#include "omnisplat/cameras.hpp"
#include "omnisplat/splatting.hpp"
#include "../include/fgs_io.hpp"
#include "../include/fgs_omnisplat.hpp"

namespace {

omnisplat::Scene<float> to_scene(const fgs::SceneSoA& s) {
  omnisplat::Scene<float> out;
  out.gaussians.resize(static_cast<size_t>(s.size()));
  for (size_t i = 0; i < out.gaussians.size(); ++i) {
    auto& g = out.gaussians[i];
    for (int k = 0; k < 3; ++k) g.mean[k] = s.means[3 * i + k];
    for (int k = 0; k < 4; ++k) g.rotation[k] = s.rotations[4 * i + k];
    for (int k = 0; k < 3; ++k) g.log_scale[k] = s.log_scales[3 * i + k];
    g.opacity_logit = s.opacity_logits[i];
    for (int k = 0; k < 48; ++k) g.sh.data()[k] = s.sh[48 * i + k];  // ShCoeffs column-major [c*16 + j]
  }
  return out;
}

omnisplat::Camera<double> to_camera(const fgs::io::CameraD& c) {
  omnisplat::Camera<double> o;
  o.model = static_cast<omnisplat::CameraModel>(c.model);
  o.width = c.width;
  o.height = c.height;
  o.fx = c.fx;
  o.fy = c.fy;
  o.cx = c.cx;
  o.cy = c.cy;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) o.rotation_wc(r, k) = c.rotation_wc[3 * r + k];
  for (int r = 0; r < 3; ++r) o.translation_wc[r] = c.translation_wc[r];
  o.fov_max = c.fov_max;
  return o;
}

}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> a;
  for (int i = 1; i + 1 < argc; i += 2) a[argv[i]] = argv[i + 1];
  if (!a.count("--scene") || !a.count("--cameras")) {
    std::cerr << "usage: omnisplat_bench --scene s.ply --cameras c.json [--repeat r]\n";
    return 2;
  }
  try {
    const int repeat = a.count("--repeat") ? std::atoi(a["--repeat"].c_str()) : 10;
    const omnisplat::Scene<float> scene = to_scene(fgs::io::load_ply(a["--scene"]).scene);
    const auto cams = fgs::io::load_cameras(a["--cameras"]).cameras;
    for (size_t i = 0; i < cams.size(); ++i) {
      const omnisplat::Camera<double> camd = to_camera(cams[i]);
      const omnisplat::Camera<float> cam = camd.cast<float>();
      omnisplat::RenderOptions<float> opts;
      double total_ms = 0, max_ms = 0;
      uint64_t intersections = 0;
      size_t aux = 0;
      for (int r = 0; r < repeat; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        const auto rr = fgs::omni::render(scene, cam, opts);
        const auto t1 = std::chrono::steady_clock::now();
        const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        total_ms += ms;
        max_ms = std::max(max_ms, ms);
        if (r == 0) intersections = rr.stats.num_intersections;
        else if (intersections != rr.stats.num_intersections)
          throw std::runtime_error("bench: intersection count changed between repeats");
        aux = std::max(aux, rr.stats.peak_aux_bytes);
      }
      std::cout << "camera=" << i << " model=" << omnisplat::camera_model_name(camd.model) << " repeats=" << repeat
                << " fps=" << (repeat * 1000.0 / total_ms) << " max_ms=" << max_ms
                << " intersections=" << intersections << " aux_bytes=" << aux << "\n";
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
