// fgs_cli — the reference CLI's `render` and `bench` subcommands (src/cli.cpp:125-170,
// :310-335) on the B200 path, reading the reference's file formats (include/fgs_io.hpp) and
// printing the reference's key=value lines, so scripts that parse `omnisplat render|bench`
// output work unchanged. `inspect` prints loader checksums (used by the tests).
//
//   fgs_cli render --scene s.ply --cameras c.json --out dir [--model-override m] [--bg r,g,b]
//                  [--sh-degree d] [--format ppm|png] [--device k]
//   fgs_cli bench  --scene s.ply --cameras c.json [--repeat r] [--device k]
//   fgs_cli inspect --scene s.ply [--cameras c.json]
#include <chrono>
#include <cstdio>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "../include/fgs_io.hpp"

namespace {

using fgs::io::CameraD;

struct Args {
  std::string cmd;
  std::map<std::string, std::string> kv;
  std::string get(const std::string& k, const std::string& def = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? def : it->second;
  }
  std::string need(const std::string& k) const {
    auto it = kv.find(k);
    if (it == kv.end()) throw std::invalid_argument(k + " is required");
    return it->second;
  }
};

std::array<float, 3> parse_rgb(const std::string& s) {
  std::array<float, 3> v{};
  char comma;
  std::istringstream is(s);
  double a, b, c;
  if (!(is >> a >> comma >> b >> comma >> c)) throw std::runtime_error("expected background as r,g,b");
  v = {static_cast<float>(a), static_cast<float>(b), static_cast<float>(c)};
  return v;
}

// src/cli.cpp:42-47
CameraD override_model(CameraD cam, int model) {
  cam.model = model;
  if (model == FGS_CAMERA_FISHEYE && !(cam.fov_max > 0)) cam.fov_max = 1.5707963267948966;
  return cam;
}

std::string frame_name(size_t i, const std::string& ext) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "frame_%03zu.%s", i, ext.c_str());
  return buf;
}

// src/cli.cpp:56-65
void print_stats_line(size_t frame, const std::string& file, const CameraD& cam, const fgs_stats& st) {
  std::cout << "frame=" << frame << " file=" << file << " model=" << fgs::io::camera_model_name(cam.model)
            << " width=" << cam.width << " height=" << cam.height << " splats=" << st.num_splats
            << " culled=" << st.num_culled << " degenerate=" << st.num_degenerate
            << " intersections=" << st.num_intersections << " preprocess_ms=" << st.preprocess_ms
            << " binning_ms=" << st.binning_ms << " sort_ms=" << st.sort_ms << " raster_ms=" << st.raster_ms
            << " aux_bytes=" << st.peak_aux_bytes << "\n";
}

void mkdirs(const std::string& dir) {
  std::string cur;
  std::istringstream is(dir);
  std::string part;
  if (!dir.empty() && dir[0] == '/') cur = "/";
  while (std::getline(is, part, '/')) {
    if (part.empty()) continue;
    cur += part + "/";
    mkdir(cur.c_str(), 0755);
  }
}

int cmd_render(const Args& a) {
  auto ply = fgs::io::load_ply(a.need("--scene"));
  for (const auto& w : ply.warnings) std::cerr << "warning: " << w << "\n";
  auto cams = fgs::io::load_cameras(a.need("--cameras"));
  for (const auto& w : cams.warnings) std::cerr << "warning: " << w << "\n";
  const std::string out = a.need("--out"), model = a.get("--model-override"), bg = a.get("--bg");
  const std::string format = a.get("--format", "ppm");
  const int sh_degree = std::stoi(a.get("--sh-degree", "3"));
  mkdirs(out);
  fgs::Renderer r(std::stoi(a.get("--device", "0")));
  for (size_t i = 0; i < cams.cameras.size(); ++i) {
    CameraD cam = cams.cameras[i];
    if (!model.empty()) cam = override_model(cam, fgs::io::camera_model_from(model, "render"));
    fgs::SceneSoA& scene = ply.scene;
    scene.background = bg.empty() ? std::array<float, 3>{0.f, 0.f, 0.f} : parse_rgb(bg);
    const auto rr = r.render(scene, cam.to_float(), sh_degree);
    const std::string file = out + "/" + frame_name(i, format);
    fgs::io::write_image(rr.image, file);
    print_stats_line(i, file, cam, rr.stats);
  }
  return 0;
}

// src/cli.cpp:138-170: per camera, `repeat` renders through the reference-facing host call;
// fps over the repeats, the slowest render, the intersection count (must not change).
int cmd_bench(const Args& a) {
  const auto ply = fgs::io::load_ply(a.need("--scene"));
  const auto cams = fgs::io::load_cameras(a.need("--cameras"));
  const int repeat = std::stoi(a.get("--repeat", "5"));
  fgs::Renderer r(std::stoi(a.get("--device", "0")));
  for (size_t i = 0; i < cams.cameras.size(); ++i) {
    const fgs_camera cam = cams.cameras[i].to_float();
    r.render(ply.scene, cam, 3);  // warm-up: allocations, lazy module load
    double total_ms = 0, max_ms = 0;
    uint64_t isect = 0, aux = 0;
    for (int k = 0; k < repeat; ++k) {
      const auto t0 = std::chrono::steady_clock::now();
      const auto rr = r.render(ply.scene, cam, 3);
      const auto t1 = std::chrono::steady_clock::now();
      const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
      total_ms += ms;
      max_ms = std::max(max_ms, ms);
      if (k == 0) isect = rr.stats.num_intersections;
      else if (isect != rr.stats.num_intersections)
        throw std::runtime_error("bench: intersection count changed between repeats");
      aux = std::max<uint64_t>(aux, rr.stats.peak_aux_bytes);
    }
    std::cout << "camera=" << i << " model=" << fgs::io::camera_model_name(cams.cameras[i].model)
              << " repeats=" << repeat << " fps=" << (repeat * 1000.0 / total_ms) << " max_ms=" << max_ms
              << " intersections=" << isect << " aux_bytes=" << aux << "\n";
  }
  return 0;
}

int cmd_inspect(const Args& a) {
  const auto ply = fgs::io::load_ply(a.need("--scene"));
  for (const auto& w : ply.warnings) std::cout << "warning=" << w << "\n";
  const auto& s = ply.scene;
  auto sum = [](const std::vector<float>& v) {
    double t = 0;
    for (float x : v) t += x;
    return t;
  };
  std::printf("gaussians=%lld means=%.17g rotations=%.17g log_scales=%.17g opacity=%.17g sh=%.17g\n",
              static_cast<long long>(s.size()), sum(s.means), sum(s.rotations), sum(s.log_scales),
              sum(s.opacity_logits), sum(s.sh));
  if (!a.get("--cameras").empty()) {
    const auto cams = fgs::io::load_cameras(a.get("--cameras"));
    for (const auto& w : cams.warnings) std::cout << "warning=" << w << "\n";
    for (size_t i = 0; i < cams.cameras.size(); ++i) {
      const auto& c = cams.cameras[i];
      std::printf("camera=%zu model=%s width=%d height=%d fx=%.17g fy=%.17g cx=%.17g cy=%.17g fov_max=%.17g rot=",
                  i, fgs::io::camera_model_name(c.model), c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.fov_max);
      for (int k = 0; k < 9; ++k) std::printf("%s%.17g", k ? "," : "", c.rotation_wc[k]);
      std::printf(" trans=%.17g,%.17g,%.17g\n", c.translation_wc[0], c.translation_wc[1], c.translation_wc[2]);
    }
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: fgs_cli render|bench|inspect [--key value ...]\n";
    return 2;
  }
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0 || i + 1 >= argc) {
      std::cerr << "error: expected --key value pairs\n";
      return 2;
    }
    a.kv[k] = argv[++i];
  }
  try {
    if (a.cmd == "render") return cmd_render(a);
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "inspect") return cmd_inspect(a);
    std::cerr << "error: unknown subcommand '" << a.cmd << "'\n";
    return 2;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
