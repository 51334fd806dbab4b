// ref_capi.cpp — C entry points around the REFERENCE's own hot-path headers.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/Makefile against the headers as they lie
// under /root/reference/proj/include (never copied into this repo) plus the repo's
// Eigen-subset shim (oracle/eigen_shim). Output: oracle/_ref/libomnisplat_ref.so, which
// serves (a) as the pin for the restatement in oracle/fgs_oracle.cpp and (b) as the CPU
// reference arm of bench.py (`--impl reference`, "kind": "reference").
//
// Calls: omnisplat::render (inc/splatting.hpp:330), omnisplat::backward
// (inc/gradients.hpp:207), omnisplat::rasterize_backward (inc/gradients.hpp:69),
// omnisplat::bruteforce_render (inc/oracle.hpp:231).

#include <cstring>
#include <memory>
#include <string>
#include <type_traits>

#include "omnisplat/gradients.hpp"
#include "omnisplat/metrics.hpp"
#include "omnisplat/optimize.hpp"
#include "omnisplat/oracle.hpp"
#include "omnisplat/splatting.hpp"

using namespace omnisplat;

namespace {

thread_local std::string g_err;

template <typename S>
Scene<S> make_scene(int64_t n, const S* means, const S* rots, const S* ls, const S* op, const S* sh, const S* bg) {
  Scene<S> s;
  s.gaussians.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    auto& g = s.gaussians[i];
    g.mean = Vec3<S>(means[i * 3], means[i * 3 + 1], means[i * 3 + 2]);
    g.rotation = Vec4<S>(rots[i * 4], rots[i * 4 + 1], rots[i * 4 + 2], rots[i * 4 + 3]);
    g.log_scale = Vec3<S>(ls[i * 3], ls[i * 3 + 1], ls[i * 3 + 2]);
    g.opacity_logit = op[i];
    std::memcpy(g.sh.data(), sh + i * 48, 48 * sizeof(S));  // column-major 16x3: [c*16 + j]
  }
  if (bg) s.background = Vec3<S>(bg[0], bg[1], bg[2]);
  return s;
}

template <typename S>
Camera<S> make_camera(const double* p) {
  Camera<S> c;
  c.model = p[0] == 0 ? CameraModel::Pinhole : (p[0] == 1 ? CameraModel::FisheyeEquidistant : CameraModel::Panorama);
  c.width = static_cast<int>(p[1]);
  c.height = static_cast<int>(p[2]);
  c.fx = S(p[3]); c.fy = S(p[4]); c.cx = S(p[5]); c.cy = S(p[6]);
  for (int i = 0; i < 9; ++i) c.rotation_wc(i / 3, i % 3) = S(p[7 + i]);
  for (int i = 0; i < 3; ++i) c.translation_wc[i] = S(p[16 + i]);
  c.fov_max = S(p[19]);
  return c;
}

template <typename S>
struct RefCtx {
  Scene<S> scene;
  Camera<S> camera;
  RenderResult<S> rr;
};

struct Any {
  int is_double;
  void* p;
};

template <typename S>
bool has_zero_quat(const Scene<S>& s) {
  for (const auto& g : s.gaussians)
    if (!(g.rotation.squaredNorm() > S(0))) return true;
  return false;
}

template <typename S>
void* do_render(int64_t n, const S* means, const S* rots, const S* ls, const S* op, const S* sh, const double* cam,
                const S* bg, int sh_degree, int threads) {
  auto c = std::make_unique<RefCtx<S>>();
  try {
    c->scene = make_scene<S>(n, means, rots, ls, op, sh, bg);
    c->camera = make_camera<S>(cam);
    RenderOptions<S> o;
    o.sh_degree = sh_degree;
    // A zero quaternion thrown inside a parallel_for worker terminates the process
    // (inc/parallel.hpp:42-44); run single-threaded so the reference's exception surfaces.
    o.threads = has_zero_quat(c->scene) ? 1 : threads;
    c->rr = render(c->scene, c->camera, o);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
  return new Any{sizeof(S) == 8, c.release()};
}

template <typename S>
int do_backward(Any* a, int64_t n, const S* dl, S* grads, const double* jgs, int threads, S* splat_grads) {
  auto* c = static_cast<RefCtx<S>*>(a->p);
  try {
    if (n != static_cast<int64_t>(c->scene.gaussians.size()))
      throw std::invalid_argument("backward: forward context was built for a different scene");
    ImageBuffer<S> img(c->camera.width, c->camera.height);
    std::memcpy(img.pixels.data(), dl, img.pixels.size() * sizeof(S));
    BackwardOptions<S> bo;
    bo.threads = threads;
    if (jgs) bo.jacobian_grad_scale = Vec3<S>(S(jgs[0]), S(jgs[1]), S(jgs[2]));
    const GradientBuffer<S> buf = backward(c->scene, c->camera, c->rr.context, img, bo);
    std::memset(grads, 0, n * 59 * sizeof(S));
    for (int64_t i = 0; i < n; ++i) {
      S* g = grads + i * 59;
      for (int k = 0; k < 3; ++k) g[k] = buf.d_mean[i][k];
      for (int k = 0; k < 4; ++k) g[3 + k] = buf.d_rotation[i][k];
      for (int k = 0; k < 3; ++k) g[7 + k] = buf.d_log_scale[i][k];
      g[10] = buf.d_opacity_logit[i];
      for (int ch = 0; ch < 3; ++ch) g[11 + ch * 16] = buf.d_sh_dc[i][ch];
    }
    if (splat_grads) {
      const SplatGradients<S> sg = rasterize_backward(c->rr.context, img, threads);
      for (size_t i = 0; i < sg.d_mean_px.size(); ++i) {
        S* o = splat_grads + i * 9;
        o[0] = sg.d_mean_px[i][0]; o[1] = sg.d_mean_px[i][1];
        for (int k = 0; k < 3; ++k) { o[2 + k] = sg.d_conic[i][k]; o[5 + k] = sg.d_color[i][k]; }
        o[8] = sg.d_alpha_max[i];
      }
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
  return 0;
}

template <typename S>
int64_t do_get(RefCtx<S>* c, const std::string& nm, void* dst) {
  const auto& ctx = c->rr.context;
  auto put = [&](const auto* src, int64_t cnt) {
    if (dst) std::memcpy(dst, src, cnt * sizeof(*src));
    return cnt;
  };
  std::vector<S> tmp;
  std::vector<int32_t> itmp;
  const int64_t nv = static_cast<int64_t>(ctx.splats.size());
  if (nm == "image") return put(c->rr.image.pixels.data(), c->rr.image.pixels.size());
  if (nm == "final_T") return put(ctx.final_transmittance.data(), ctx.final_transmittance.size());
  if (nm == "count") return put(ctx.blend_count.data(), ctx.blend_count.size());
  if (nm == "refs") return put(ctx.refs.data(), ctx.refs.size());
  if (nm == "offsets") return put(ctx.tiles.offsets.data(), ctx.tiles.offsets.size());
  if (nm == "cam_points") { for (auto& p : ctx.cam_points) for (int k = 0; k < 3; ++k) tmp.push_back(p[k]); return put(tmp.data(), 3 * nv); }
  if (nm == "mean_px") { for (auto& s : ctx.splats) { tmp.push_back(s.mean_px[0]); tmp.push_back(s.mean_px[1]); } return put(tmp.data(), 2 * nv); }
  if (nm == "conic") { for (auto& s : ctx.splats) for (int k = 0; k < 3; ++k) tmp.push_back(s.conic[k]); return put(tmp.data(), 3 * nv); }
  if (nm == "color") { for (auto& s : ctx.splats) for (int k = 0; k < 3; ++k) tmp.push_back(s.color[k]); return put(tmp.data(), 3 * nv); }
  if (nm == "depth") { for (auto& s : ctx.splats) tmp.push_back(s.depth); return put(tmp.data(), nv); }
  if (nm == "alpha") { for (auto& s : ctx.splats) tmp.push_back(s.alpha_max); return put(tmp.data(), nv); }
  if (nm == "radius") { for (auto& s : ctx.splats) itmp.push_back(s.radius_px); return put(itmp.data(), nv); }
  if (nm == "source") { for (auto& s : ctx.splats) itmp.push_back(s.source_index); return put(itmp.data(), nv); }
  return -1;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_render_f32(int64_t n, const float* m, const float* r, const float* l, const float* o, const float* sh,
                     const double* cam, const float* bg, int deg, int threads) {
  return do_render<float>(n, m, r, l, o, sh, cam, bg, deg, threads);
}
void* ref_render_f64(int64_t n, const double* m, const double* r, const double* l, const double* o,
                     const double* sh, const double* cam, const double* bg, int deg, int threads) {
  return do_render<double>(n, m, r, l, o, sh, cam, bg, deg, threads);
}
int ref_backward_f32(void* h, int64_t n, const float* dl, float* grads, const double* jgs, int threads, float* sg) {
  auto* a = static_cast<Any*>(h);
  if (a->is_double) { g_err = "precision mismatch"; return -1; }
  return do_backward<float>(a, n, dl, grads, jgs, threads, sg);
}
int ref_backward_f64(void* h, int64_t n, const double* dl, double* grads, const double* jgs, int threads, double* sg) {
  auto* a = static_cast<Any*>(h);
  if (!a->is_double) { g_err = "precision mismatch"; return -1; }
  return do_backward<double>(a, n, dl, grads, jgs, threads, sg);
}
void ref_free(void* h) {
  auto* a = static_cast<Any*>(h);
  if (!a) return;
  if (a->is_double) delete static_cast<RefCtx<double>*>(a->p);
  else delete static_cast<RefCtx<float>*>(a->p);
  delete a;
}
void ref_sizes(void* h, int64_t* out) {
  auto* a = static_cast<Any*>(h);
  auto fill = [&](auto* c) {
    out[0] = static_cast<int64_t>(c->scene.gaussians.size());
    out[1] = static_cast<int64_t>(c->rr.context.splats.size());
    out[2] = static_cast<int64_t>(c->rr.stats.num_intersections);
    out[3] = c->rr.context.tiles.tiles_x; out[4] = c->rr.context.tiles.tiles_y;
    out[5] = c->camera.width; out[6] = c->camera.height;
  };
  if (a->is_double) fill(static_cast<RefCtx<double>*>(a->p)); else fill(static_cast<RefCtx<float>*>(a->p));
}
void ref_stats(void* h, double* out) {
  auto* a = static_cast<Any*>(h);
  auto fill = [&](auto* c) {
    const auto& s = c->rr.stats;
    out[0] = double(s.num_intersections); out[1] = s.num_splats; out[2] = s.num_culled; out[3] = s.num_degenerate;
    out[4] = s.preprocess_ms; out[5] = s.binning_ms; out[6] = s.sort_ms; out[7] = s.raster_ms;
    out[8] = double(s.peak_aux_bytes); out[9] = -1; out[10] = -1;
  };
  if (a->is_double) fill(static_cast<RefCtx<double>*>(a->p)); else fill(static_cast<RefCtx<float>*>(a->p));
}
int64_t ref_get(void* h, const char* name, void* dst) {
  auto* a = static_cast<Any*>(h);
  return a->is_double ? do_get(static_cast<RefCtx<double>*>(a->p), name, dst)
                      : do_get(static_cast<RefCtx<float>*>(a->p), name, dst);
}
int ref_bruteforce_render_f64(int64_t n, const double* m, const double* r, const double* l, const double* o,
                              const double* sh, const double* cam, const double* bg, int deg, double* image) {
  try {
    const Scene<double> s = make_scene<double>(n, m, r, l, o, sh, bg);
    const Camera<double> c = make_camera<double>(cam);
    OracleOptions<double> oo;
    oo.sh_degree = deg;
    oo.max_gaussians = static_cast<size_t>(n) + 1;
    const ImageBuffer<double> img = bruteforce_render(s, c, oo);
    std::memcpy(image, img.pixels.data(), img.pixels.size() * sizeof(double));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
  return 0;
}

// L = (1 - lambda) L1 + lambda (1 - SSIM) and dL/drendered (double, as the reference trains).
int ref_l1_dssim_loss_f64(int w, int h, const double* rendered, const double* target, double lambda,
                          double* d_rendered, double* out3) {
  try {
    ImageBuffer<double> a(w, h), b(w, h);
    std::memcpy(a.pixels.data(), rendered, a.pixels.size() * sizeof(double));
    std::memcpy(b.pixels.data(), target, b.pixels.size() * sizeof(double));
    const LossResult<double> r = l1_dssim_loss(a, b, lambda);
    std::memcpy(d_rendered, r.d_rendered.pixels.data(), r.d_rendered.pixels.size() * sizeof(double));
    out3[0] = r.total;
    out3[1] = r.l1;
    out3[2] = r.dssim;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
  return 0;
}

// One adam_step on n Gaussians (params/grads/m/v as 59-float rows: mean 3, rotation 4,
// log_scale 3, opacity 1, sh 48 with DC at 11 + 16c; the reference updates the DC only).
// lr = {mean, rotation, log_scale, opacity, sh_dc}; step = the state's step before the call.
int ref_adam_step_f64(int64_t n, double* params, const double* grads, double* m, double* v, int64_t step,
                      const double* lr) {
  try {
    Scene<double> s;
    s.gaussians.resize(n);
    GradientBuffer<double> g;
    g.resize_zero(n);
    AdamState<double> st;
    st.init(n);
    st.step = step;
    auto load = [&](int64_t i, const double* row, auto& mean, auto& rot, auto& ls, double& op, auto& dc) {
      for (int k = 0; k < 3; ++k) mean[k] = row[k];
      for (int k = 0; k < 4; ++k) rot[k] = row[3 + k];
      for (int k = 0; k < 3; ++k) ls[k] = row[7 + k];
      op = row[10];
      for (int c = 0; c < 3; ++c) dc[c] = row[11 + 16 * c];
      (void)i;
    };
    for (int64_t i = 0; i < n; ++i) {
      auto& q = s.gaussians[i];
      Vec3<double> dc;
      load(i, params + i * 59, q.mean, q.rotation, q.log_scale, q.opacity_logit, dc);
      for (int c = 0; c < 3; ++c) q.sh(0, c) = dc[c];
      load(i, grads + i * 59, g.d_mean[i], g.d_rotation[i], g.d_log_scale[i], g.d_opacity_logit[i], g.d_sh_dc[i]);
      load(i, m + i * 59, st.m.d_mean[i], st.m.d_rotation[i], st.m.d_log_scale[i], st.m.d_opacity_logit[i],
           st.m.d_sh_dc[i]);
      load(i, v + i * 59, st.v.d_mean[i], st.v.d_rotation[i], st.v.d_log_scale[i], st.v.d_opacity_logit[i],
           st.v.d_sh_dc[i]);
    }
    const GroupLearningRates<double> rates{lr[0], lr[1], lr[2], lr[3], lr[4]};
    adam_step(s, g, st, rates);
    auto store = [&](double* row, const auto& mean, const auto& rot, const auto& ls, double op, const auto& dc) {
      for (int k = 0; k < 3; ++k) row[k] = mean[k];
      for (int k = 0; k < 4; ++k) row[3 + k] = rot[k];
      for (int k = 0; k < 3; ++k) row[7 + k] = ls[k];
      row[10] = op;
      for (int c = 0; c < 3; ++c) row[11 + 16 * c] = dc[c];
    };
    for (int64_t i = 0; i < n; ++i) {
      const auto& q = s.gaussians[i];
      const Vec3<double> dc(q.sh(0, 0), q.sh(0, 1), q.sh(0, 2));
      store(params + i * 59, q.mean, q.rotation, q.log_scale, q.opacity_logit, dc);
      store(m + i * 59, st.m.d_mean[i], st.m.d_rotation[i], st.m.d_log_scale[i], st.m.d_opacity_logit[i],
            st.m.d_sh_dc[i]);
      store(v + i * 59, st.v.d_mean[i], st.v.d_rotation[i], st.v.d_log_scale[i], st.v.d_opacity_logit[i],
            st.v.d_sh_dc[i]);
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
  return 0;
}

}  // extern "C"
