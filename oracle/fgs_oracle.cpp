// fgs_oracle.cpp — CPU restatement of the omnisplat fisheye render/backward hot path.
//
// TEST INFRASTRUCTURE ONLY. This file is the parity checker for the CUDA product in
// paper_2409_04751_b200/. Only tests/, __graft_entry__.smoke() and bench.py's CPU
// baseline leg may load it; the product never links or calls it.
//
// It restates, scalar by scalar, the reference algorithm in
//   /root/reference/proj/include/omnisplat/{core,model,cameras,splatting,gradients,oracle}.hpp
// (cited below as inc/<file>:<line>). Every small-matrix expression of the reference is
// expanded with the evaluation order the repo's Eigen-subset shim (oracle/eigen_shim)
// gives it: products and reductions are summed left to right, coefficient-wise
// expressions follow C++ associativity. Built with -ffp-contract=off, so fp32 results
// are bit-identical to the reference headers compiled against that shim (oracle/_ref,
// see oracle/Makefile) when `mode == ORC_MODE_LIBM`.
//
// Two transcendental modes:
//   ORC_MODE_PARITY: atan2f/expf are evaluated in double and rounded once to float
//                    (glibc-independent; the CUDA kernels implement the same definition).
//   ORC_MODE_LIBM:   std::atan2/std::exp on floats exactly as the reference calls them.
// For S = double both modes are identical.
//
// Parity of this restatement is pinned by tests/test_oracle_pins.py (the reference's own
// known-answer tests, ported) and tests/test_oracle_vs_ref.py (bit-exact vs oracle/_ref).

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

enum { ORC_MODE_PARITY = 0, ORC_MODE_LIBM = 1 };
enum { CAM_PINHOLE = 0, CAM_FISHEYE = 1, CAM_PANORAMA = 2 };

// inc/core.hpp:43-53 — constants that define the forward model.
constexpr double kAlphaClamp = 0.99;
constexpr double kAlphaSkip = 1.0 / 255.0;
constexpr double kTransmittanceStop = 1.0e-4;
constexpr double kCovarianceDilation = 0.3;
constexpr double kRadiusSigma = 3.0;
constexpr int kTileSize = 16;
constexpr double kPinholeNearClip = 0.2;
constexpr double kFisheyeCullMarginRad = 10.0 * 3.141592653589793238462643383279502884 / 180.0;
constexpr double kFisheyeSeriesW2 = 1.0e-6;  // inc/cameras.hpp:104

// inc/model.hpp:173-183
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                           -1.0925484305920792, 0.5462742152960396};
constexpr double kC3[7] = {-0.5900435899266435, 2.890611442640554,  -0.4570457994644658,
                           0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                           -0.5900435899266435};

thread_local int g_mode = ORC_MODE_PARITY;

template <typename S> inline S t_exp(S x);
template <> inline float t_exp<float>(float x) {
  return g_mode == ORC_MODE_LIBM ? std::exp(x) : static_cast<float>(std::exp(static_cast<double>(x)));
}
template <> inline double t_exp<double>(double x) { return std::exp(x); }
template <typename S> inline S t_atan2(S y, S x);
template <> inline float t_atan2<float>(float y, float x) {
  return g_mode == ORC_MODE_LIBM ? std::atan2(y, x)
                                 : static_cast<float>(std::atan2(static_cast<double>(y), static_cast<double>(x)));
}
template <> inline double t_atan2<double>(double y, double x) { return std::atan2(y, x); }

// ---------------------------------------------------------------------------------------
// parallel_for: static contiguous partition, one std::thread per worker per call
// (inc/parallel.hpp:29-47). Results are independent of the thread count.
template <typename F>
void parallel_for(int64_t n, F&& f, int threads) {
  if (n <= 0) return;
  int t = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  if (t > n) t = static_cast<int>(n);
  const int mode = g_mode;
  if (t <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> workers;
  workers.reserve(t);
  for (int w = 0; w < t; ++w) {
    const int64_t lo = n * w / t, hi = n * (w + 1) / t;
    workers.emplace_back([&f, lo, hi, mode] {
      g_mode = mode;
      for (int64_t i = lo; i < hi; ++i) f(i);
    });
  }
  for (auto& w : workers) w.join();
}

// ---------------------------------------------------------------------------------------
// Small fixed-size helpers. Row-major storage here; only the *sum order* matters and it
// is spelled out at each call site.
template <typename S> struct V2 { S v[2]; };
template <typename S> struct V3 { S v[3]; };
template <typename S> struct M3 { S m[3][3]; };
template <typename S> struct M23 { S m[2][3]; };
template <typename S> struct M2 { S m[2][2]; };

template <typename S>
struct Camera {
  int model = CAM_FISHEYE;
  int width = 0, height = 0;
  S fx = 0, fy = 0, cx = 0, cy = 0;
  S W[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};  // rotation_wc, world -> camera
  S b[3] = {0, 0, 0};                             // translation_wc
  S fov_max = S(3.141592653589793238462643383279502884L) / S(2);
};

template <typename S>
struct Scene {
  int64_t n = 0;
  std::vector<S> means, rotations, log_scales, opacity, sh;  // sh: per Gaussian [c*16 + j]
  S bg[3] = {0, 0, 0};
};

// Matrix product C = A(RxK) * B(KxC), coefficients summed left to right over k.
template <typename S, int R, int K, int C>
inline void matmul(const S (&a)[R][K], const S (&b)[K][C], S (&out)[R][C]) {
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < C; ++j) {
      S acc = a[i][0] * b[0][j];
      for (int k = 1; k < K; ++k) acc = acc + a[i][k] * b[k][j];
      out[i][j] = acc;
    }
}
template <typename S, int R, int C>
inline void transpose(const S (&a)[R][C], S (&out)[C][R]) {
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < C; ++j) out[j][i] = a[i][j];
}
// Eigen .cwiseProduct().sum() over a column-major matrix: storage order is column-major,
// summed left to right (shim order).
template <typename S, int R, int C>
inline S cwise_sum_colmajor(const S (&a)[R][C], const S (&b)[R][C]) {
  S acc = a[0][0] * b[0][0];
  bool first = true;
  for (int j = 0; j < C; ++j)
    for (int i = 0; i < R; ++i) {
      if (first) { first = false; continue; }
      acc = acc + a[i][j] * b[i][j];
    }
  return acc;
}

// ---------------------------------------------------------------------------------------
// Camera (inc/cameras.hpp)

// inc/cameras.hpp:60 — center = -R^T b
template <typename S>
inline void camera_center(const Camera<S>& cam, S out[3]) {
  for (int r = 0; r < 3; ++r) {
    S acc = (-cam.W[0][r]) * cam.b[0];
    acc = acc + (-cam.W[1][r]) * cam.b[1];
    acc = acc + (-cam.W[2][r]) * cam.b[2];
    out[r] = acc;
  }
}

// inc/cameras.hpp:76-79 — mu_c = W mu + b
template <typename S>
inline void world_to_camera(const Camera<S>& cam, const S* m, S out[3]) {
  for (int r = 0; r < 3; ++r) {
    S acc = cam.W[r][0] * m[0];
    acc = acc + cam.W[r][1] * m[1];
    acc = acc + cam.W[r][2] * m[2];
    out[r] = acc + cam.b[r];
  }
}

template <typename S> struct FisheyeTerms { S g, u, U; };

// inc/cameras.hpp:107-128 (AxisMode::Auto)
template <typename S>
inline FisheyeTerms<S> fisheye_terms(S lz2, S z, int force = 0 /*0 auto, 1 series, 2 general*/) {
  const S z2 = z * z;
  const bool series = force == 1 || (force == 0 && z > S(0) && lz2 < S(kFisheyeSeriesW2) * z2);
  FisheyeTerms<S> t;
  if (series) {
    const S w2 = lz2 / z2;
    const S z3 = z2 * z, z5 = z3 * z2;
    t.g = (S(1) - w2 / S(3) + w2 * w2 / S(5) - w2 * w2 * w2 / S(7)) / z;
    t.u = (S(-2) / S(3) + S(4) / S(5) * w2 - S(6) / S(7) * w2 * w2) / z3;
    t.U = (S(8) / S(5) - S(24) / S(7) * w2 + S(16) / S(3) * w2 * w2) / z5;
  } else {
    const S lz = std::sqrt(lz2);
    const S r2 = lz2 + z2;
    const S theta = t_atan2<S>(lz, z);
    t.g = theta / lz;
    t.u = z / (lz2 * r2) - theta / (lz2 * lz);
    t.U = S(3) * theta / (lz2 * lz2 * lz) - z / (r2 * lz2 * lz2) -
          S(2) * z * (r2 + lz2) / (lz2 * lz2 * r2 * r2);
  }
  return t;
}

// inc/cameras.hpp:180-212
template <typename S>
inline void projection_jacobian(const S p[3], const Camera<S>& cam, S j[2][3], int force = 0) {
  const S x = p[0], y = p[1], z = p[2];
  switch (cam.model) {
    case CAM_PINHOLE: {
      const S iz = S(1) / z;
      j[0][0] = cam.fx * iz; j[0][1] = S(0); j[0][2] = -cam.fx * x * iz * iz;
      j[1][0] = S(0); j[1][1] = cam.fy * iz; j[1][2] = -cam.fy * y * iz * iz;
      break;
    }
    case CAM_FISHEYE: {
      const S lz2 = x * x + y * y;
      const S r2 = lz2 + z * z;
      const auto t = fisheye_terms(lz2, z, force);
      const S fx = cam.fx, fy = cam.fy;
      j[0][0] = fx * (t.g + x * x * t.u); j[0][1] = fx * x * y * t.u; j[0][2] = -fx * x / r2;
      j[1][0] = fy * x * y * t.u; j[1][1] = fy * (t.g + y * y * t.u); j[1][2] = -fy * y / r2;
      break;
    }
    default: {  // panorama (inc/cameras.hpp:200-208)
      const S pi = S(3.141592653589793238462643383279502884L);
      const S s = x * x + z * z;
      const S rho = std::sqrt(s);
      const S r2 = s + y * y;
      const S cw = S(cam.width) / (S(2) * pi);
      const S dh = S(cam.height) / pi;
      j[0][0] = cw * z / s; j[0][1] = S(0); j[0][2] = -cw * x / s;
      j[1][0] = -dh * x * y / (rho * r2); j[1][1] = dh * rho / r2; j[1][2] = -dh * y * z / (rho * r2);
      break;
    }
  }
}

// inc/cameras.hpp:139-177. Returns visibility; pixel written whenever a finite one exists.
template <typename S>
inline bool project(const S p[3], const Camera<S>& cam, S pixel[2], S jac[2][3], int force = 0) {
  const S x = p[0], y = p[1], z = p[2];
  const S r2 = x * x + y * y + z * z;
  pixel[0] = pixel[1] = S(0);
  if (r2 < S(1e-24)) return false;
  bool visible = false;
  switch (cam.model) {
    case CAM_PINHOLE: {
      if (std::abs(z) < S(1e-12)) return false;
      pixel[0] = cam.cx + cam.fx * x / z;
      pixel[1] = cam.cy + cam.fy * y / z;
      visible = z > S(kPinholeNearClip);
      break;
    }
    case CAM_FISHEYE: {
      const S lz2 = x * x + y * y;
      if (z < S(0) && lz2 < S(1e-24) * z * z) return false;
      const S theta = t_atan2<S>(std::sqrt(lz2), z);
      const S g = fisheye_terms(lz2, z, force).g;
      pixel[0] = cam.cx + cam.fx * g * x;
      pixel[1] = cam.cy + cam.fy * g * y;
      visible = theta <= cam.fov_max + S(kFisheyeCullMarginRad);
      break;
    }
    default: {
      const S pi = S(3.141592653589793238462643383279502884L);
      const S s = x * x + z * z;
      if (s < S(1e-24) * y * y) return false;
      const S w = S(cam.width), h = S(cam.height);
      S xp = w * (t_atan2<S>(x, z) + pi) / (S(2) * pi);
      if (xp >= w) xp -= w;
      const S yp = h * (t_atan2<S>(y, std::sqrt(s)) + pi / S(2)) / pi;
      pixel[0] = xp;
      pixel[1] = yp;
      visible = true;
      break;
    }
  }
  if (visible) projection_jacobian(p, cam, jac, force);
  return visible;
}

// inc/cameras.hpp:217-271 (fisheye and pinhole branches; panorama included for completeness)
template <typename S>
inline void projection_jacobian_grad(const S p[3], const Camera<S>& cam, S d[3][2][3]) {
  const S x = p[0], y = p[1], z = p[2];
  switch (cam.model) {
    case CAM_PINHOLE: {
      const S iz2 = S(1) / (z * z);
      const S fx = cam.fx, fy = cam.fy;
      const S a[3][2][3] = {{{S(0), S(0), -fx * iz2}, {S(0), S(0), S(0)}},
                            {{S(0), S(0), S(0)}, {S(0), S(0), -fy * iz2}},
                            {{-fx * iz2, S(0), S(2) * fx * x * iz2 / z}, {S(0), -fy * iz2, S(2) * fy * y * iz2 / z}}};
      std::memcpy(d, a, sizeof(a));
      break;
    }
    case CAM_FISHEYE: {
      const S lz2 = x * x + y * y;
      const S r2 = lz2 + z * z;
      const S ir4 = S(1) / (r2 * r2);
      const auto t = fisheye_terms(lz2, z);
      const S fx = cam.fx, fy = cam.fy;
      const S x2 = x * x, y2 = y * y;
      const S ux = t.u + x2 * t.U;
      const S uy = t.u + y2 * t.U;
      d[0][0][0] = fx * x * (S(3) * t.u + x2 * t.U); d[0][0][1] = fx * y * ux; d[0][0][2] = fx * (S(2) * x2 - r2) * ir4;
      d[0][1][0] = fy * y * ux; d[0][1][1] = fy * x * uy; d[0][1][2] = S(2) * fy * x * y * ir4;
      d[1][0][0] = fx * y * ux; d[1][0][1] = fx * x * uy; d[1][0][2] = S(2) * fx * x * y * ir4;
      d[1][1][0] = fy * x * uy; d[1][1][1] = fy * y * (S(3) * t.u + y2 * t.U); d[1][1][2] = fy * (S(2) * y2 - r2) * ir4;
      d[2][0][0] = fx * (S(2) * x2 - r2) * ir4; d[2][0][1] = S(2) * fx * x * y * ir4; d[2][0][2] = S(2) * fx * x * z * ir4;
      d[2][1][0] = S(2) * fy * x * y * ir4; d[2][1][1] = fy * (S(2) * y2 - r2) * ir4; d[2][1][2] = S(2) * fy * y * z * ir4;
      break;
    }
    default: {
      const S pi = S(3.141592653589793238462643383279502884L);
      const S s = x * x + z * z;
      const S rho = std::sqrt(s);
      const S r2 = s + y * y;
      const S cw = S(cam.width) / (S(2) * pi);
      const S dh = S(cam.height) / pi;
      const S is2 = S(1) / (s * s);
      const S e = S(1) / (rho * r2);
      const S f = (r2 + S(2) * s) / (rho * s * r2 * r2);
      const S ey = S(2) * y / (rho * r2 * r2);
      d[0][0][0] = S(-2) * cw * x * z * is2; d[0][0][1] = S(0); d[0][0][2] = cw * (x * x - z * z) * is2;
      d[0][1][0] = -dh * y * (e - x * x * f); d[0][1][1] = dh * x * (y * y - s) / (rho * r2 * r2); d[0][1][2] = dh * x * y * z * f;
      d[1][0][0] = S(0); d[1][0][1] = S(0); d[1][0][2] = S(0);
      d[1][1][0] = -dh * x * (e - y * ey); d[1][1][1] = S(-2) * dh * rho * y / (r2 * r2); d[1][1][2] = -dh * z * (e - y * ey);
      d[2][0][0] = cw * (x * x - z * z) * is2; d[2][0][1] = S(0); d[2][0][2] = S(2) * cw * x * z * is2;
      d[2][1][0] = dh * x * y * z * f; d[2][1][1] = dh * z * (y * y - s) / (rho * r2 * r2); d[2][1][2] = -dh * y * (e - z * z * f);
      break;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Model (inc/model.hpp)

struct DegenerateRotation : std::invalid_argument {
  DegenerateRotation() : std::invalid_argument("degenerate rotation: quaternion has zero norm") {}
};

// inc/model.hpp:95-106
template <typename S>
inline void quaternion_to_rotation(const S* q, S r[3][3]) {
  const S n2 = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
  if (!(n2 > S(0))) throw DegenerateRotation();
  const S n = std::sqrt(n2);
  const S w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  r[0][0] = S(1) - S(2) * (y * y + z * z); r[0][1] = S(2) * (x * y - w * z); r[0][2] = S(2) * (x * z + w * y);
  r[1][0] = S(2) * (x * y + w * z); r[1][1] = S(1) - S(2) * (x * x + z * z); r[1][2] = S(2) * (y * z - w * x);
  r[2][0] = S(2) * (x * z - w * y); r[2][1] = S(2) * (y * z + w * x); r[2][2] = S(1) - S(2) * (x * x + y * y);
}

// inc/model.hpp:111-121
template <typename S>
inline void rotation_quaternion_partials(const S qn[4], S d[4][3][3]) {
  const S w = qn[0], x = qn[1], y = qn[2], z = qn[3];
  const S a[4][3][3] = {{{S(0), -z, y}, {z, S(0), -x}, {-y, x, S(0)}},
                        {{S(0), y, z}, {y, S(-2) * x, -w}, {z, w, S(-2) * x}},
                        {{S(-2) * y, x, w}, {x, S(0), z}, {-w, z, S(-2) * y}},
                        {{S(-2) * z, -w, x}, {w, S(-2) * z, y}, {x, y, S(0)}}};
  for (int k = 0; k < 4; ++k)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) d[k][i][j] = a[k][i][j] * S(2);
}

// inc/model.hpp:127-140
template <typename S>
inline void build_covariance(const S* q, const S* log_scale, S sigma[3][3]) {
  S r[3][3];
  quaternion_to_rotation(q, r);
  const S scale[3] = {t_exp<S>(log_scale[0]), t_exp<S>(log_scale[1]), t_exp<S>(log_scale[2])};
  S m[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = r[i][j] * scale[j];
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) {
      const S v = m[i][0] * m[j][0] + m[i][1] * m[j][1] + m[i][2] * m[j][2];
      sigma[i][j] = v;
      sigma[j][i] = v;
    }
}

// inc/model.hpp:144-171
template <typename S>
inline void build_covariance_backward(const S* q, const S* log_scale, const S g[3][3], S dq[4], S ds[3]) {
  const S n2 = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
  if (!(n2 > S(0))) throw DegenerateRotation();
  const S n = std::sqrt(n2);
  const S qn[4] = {q[0] / n, q[1] / n, q[2] / n, q[3] / n};
  S r[3][3];
  quaternion_to_rotation(q, r);
  const S scale[3] = {t_exp<S>(log_scale[0]), t_exp<S>(log_scale[1]), t_exp<S>(log_scale[2])};
  S m[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = r[i][j] * scale[j];
  S gs[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) gs[i][j] = g[i][j] + g[j][i];
  S dm[3][3];
  matmul<S, 3, 3, 3>(gs, m, dm);
  S dr[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) dr[i][j] = dm[i][j] * scale[j];
  for (int i = 0; i < 3; ++i) ds[i] = scale[i] * (r[0][i] * dm[0][i] + r[1][i] * dm[1][i] + r[2][i] * dm[2][i]);
  S drq[4][3][3];
  rotation_quaternion_partials(qn, drq);
  S dqn[4];
  for (int k = 0; k < 4; ++k) dqn[k] = cwise_sum_colmajor<S, 3, 3>(dr, drq[k]);
  const S dot = qn[0] * dqn[0] + qn[1] * dqn[1] + qn[2] * dqn[2] + qn[3] * dqn[3];
  for (int k = 0; k < 4; ++k) dq[k] = (dqn[k] - qn[k] * dot) / n;
}

// inc/model.hpp:187-215 — evaluated per channel; basis factors multiply coefficients in the
// reference's association order. `basis` (optional) receives the 16 basis factors Y_j.
template <typename S>
inline void eval_sh(const S* sh, const S dir[3], int degree, S out[3], S* basis = nullptr) {
  const S x = dir[0], y = dir[1], z = dir[2];
  S Y[16];
  Y[0] = S(kC0);
  if (degree >= 1) {
    Y[1] = -S(kC1) * y; Y[2] = S(kC1) * z; Y[3] = -S(kC1) * x;
  }
  S xx = 0, yy = 0, zz = 0, xy = 0, yz = 0, xz = 0;
  if (degree >= 2) {
    xx = x * x; yy = y * y; zz = z * z; xy = x * y; yz = y * z; xz = x * z;
    Y[4] = S(kC2[0]) * xy; Y[5] = S(kC2[1]) * yz; Y[6] = S(kC2[2]) * (S(2) * zz - xx - yy);
    Y[7] = S(kC2[3]) * xz; Y[8] = S(kC2[4]) * (xx - yy);
  }
  if (degree >= 3) {
    Y[9] = S(kC3[0]) * y * (S(3) * xx - yy);
    Y[10] = S(kC3[1]) * xy * z;
    Y[11] = S(kC3[2]) * y * (S(4) * zz - xx - yy);
    Y[12] = S(kC3[3]) * z * (S(2) * zz - S(3) * xx - S(3) * yy);
    Y[13] = S(kC3[4]) * x * (S(4) * zz - xx - yy);
    Y[14] = S(kC3[5]) * z * (xx - yy);
    Y[15] = S(kC3[6]) * x * (xx - yy);
  }
  for (int c = 0; c < 3; ++c) {
    const S* k = sh + c * 16;
    S v = S(kC0) * k[0];
    if (degree >= 1) {
      // -C1*y*s1 + C1*z*s2 - C1*x*s3
      const S t = (-S(kC1)) * y * k[1] + S(kC1) * z * k[2] - S(kC1) * x * k[3];
      v = v + t;
      if (degree >= 2) {
        const S t2 = S(kC2[0]) * xy * k[4] + S(kC2[1]) * yz * k[5] +
                     S(kC2[2]) * (S(2) * zz - xx - yy) * k[6] + S(kC2[3]) * xz * k[7] +
                     S(kC2[4]) * (xx - yy) * k[8];
        v = v + t2;
        if (degree >= 3) {
          const S t3 = S(kC3[0]) * y * (S(3) * xx - yy) * k[9] + S(kC3[1]) * xy * z * k[10] +
                       S(kC3[2]) * y * (S(4) * zz - xx - yy) * k[11] +
                       S(kC3[3]) * z * (S(2) * zz - S(3) * xx - S(3) * yy) * k[12] +
                       S(kC3[4]) * x * (S(4) * zz - xx - yy) * k[13] + S(kC3[5]) * z * (xx - yy) * k[14] +
                       S(kC3[6]) * x * (xx - yy) * k[15];
          v = v + t3;
        }
      }
    }
    v = v + S(0.5);
    out[c] = std::max(v, S(0));
  }
  if (basis) {
    const int nb = (degree + 1) * (degree + 1);
    for (int j = 0; j < 16; ++j) basis[j] = j < nb ? Y[j] : S(0);
  }
}

// Build extension (not in the reference): d colour_c / d dir for the SH view-direction
// path, dY_j/d(x, y, z) of the basis above. Used only when sh_view_dir_grad is on.
template <typename S>
inline void sh_basis_grad(const S dir[3], int degree, S dY[16][3]) {
  const S x = dir[0], y = dir[1], z = dir[2];
  for (int j = 0; j < 16; ++j) dY[j][0] = dY[j][1] = dY[j][2] = S(0);
  if (degree < 1) return;
  const S c1 = S(kC1);
  dY[1][1] = -c1; dY[2][2] = c1; dY[3][0] = -c1;
  if (degree < 2) return;
  const S a0 = S(kC2[0]), a1 = S(kC2[1]), a2 = S(kC2[2]), a3 = S(kC2[3]), a4 = S(kC2[4]);
  dY[4][0] = a0 * y; dY[4][1] = a0 * x;
  dY[5][1] = a1 * z; dY[5][2] = a1 * y;
  dY[6][0] = S(-2) * a2 * x; dY[6][1] = S(-2) * a2 * y; dY[6][2] = S(4) * a2 * z;
  dY[7][0] = a3 * z; dY[7][2] = a3 * x;
  dY[8][0] = S(2) * a4 * x; dY[8][1] = S(-2) * a4 * y;
  if (degree < 3) return;
  const S b0 = S(kC3[0]), b1 = S(kC3[1]), b2 = S(kC3[2]), b3 = S(kC3[3]), b4 = S(kC3[4]), b5 = S(kC3[5]),
          b6 = S(kC3[6]);
  const S xx = x * x, yy = y * y, zz = z * z;
  dY[9][0] = S(6) * b0 * x * y; dY[9][1] = b0 * (S(3) * xx - S(3) * yy);
  dY[10][0] = b1 * y * z; dY[10][1] = b1 * x * z; dY[10][2] = b1 * x * y;
  dY[11][0] = S(-2) * b2 * x * y; dY[11][1] = b2 * (S(4) * zz - xx - S(3) * yy); dY[11][2] = S(8) * b2 * y * z;
  dY[12][0] = S(-6) * b3 * x * z; dY[12][1] = S(-6) * b3 * y * z; dY[12][2] = b3 * (S(6) * zz - S(3) * xx - S(3) * yy);
  dY[13][0] = b4 * (S(4) * zz - S(3) * xx - yy); dY[13][1] = S(-2) * b4 * x * y; dY[13][2] = S(8) * b4 * x * z;
  dY[14][0] = S(2) * b5 * x * z; dY[14][1] = S(-2) * b5 * y * z; dY[14][2] = b5 * (xx - yy);
  dY[15][0] = b6 * (S(3) * xx - yy); dY[15][1] = S(-2) * b6 * x * y;
}

// inc/core.hpp:30-36
template <typename S>
inline S sigmoid(S x) {
  if (x >= S(0)) return S(1) / (S(1) + t_exp<S>(-x));
  const S e = t_exp<S>(x);
  return e / (S(1) + e);
}

// ---------------------------------------------------------------------------------------
// Forward pipeline (inc/splatting.hpp)

template <typename S>
struct Splat {
  S mean_px[2];
  S conic[3];
  S depth;
  int radius;
  S color[3];
  S alpha;
  int source;
};

template <typename S>
struct Ctx {
  Camera<S> cam;
  Scene<S> scene;
  int sh_degree = 3;
  S bg[3] = {0, 0, 0};
  std::vector<int32_t> state;  // per Gaussian: 0 culled, 1 kept, 2 degenerate
  std::vector<Splat<S>> splats;
  std::vector<S> cam_points;   // 3 per splat
  int tiles_x = 0, tiles_y = 0;
  std::vector<uint32_t> key_tile, key_splat;  // pre-sort emission order
  std::vector<uint64_t> key_depth;            // depth_key_bits (32 used for float)
  std::vector<uint32_t> refs, offsets;
  std::vector<S> image, final_T;
  std::vector<uint16_t> count;
  uint32_t num_culled = 0, num_degenerate = 0;
  double pre_ms = 0, bin_ms = 0, sort_ms = 0, raster_ms = 0;
  double aux_bytes = 0;
  uint64_t e_eval = 0, e_contrib = 0;
};

// inc/splatting.hpp:68-139
template <typename S>
void preprocess(Ctx<S>& c, int threads) {
  const int64_t n = c.scene.n;
  std::vector<Splat<S>> slots(n);
  std::vector<S> points(n * 3);
  c.state.assign(n, 0);
  S cam_center[3];
  camera_center(c.cam, cam_center);
  std::atomic<bool> degenerate_quat{false};
  parallel_for(n, [&](int64_t i) {
    const S* mean = &c.scene.means[i * 3];
    S mu[3];
    world_to_camera(c.cam, mean, mu);
    S pixel[2], jac[2][3];
    if (!project(mu, c.cam, pixel, jac)) return;
    S t[2][3];
    matmul<S, 2, 3, 3>(jac, c.cam.W, t);                        // :87
    S sigma[3][3];
    try {
      build_covariance(&c.scene.rotations[i * 4], &c.scene.log_scales[i * 3], sigma);  // :88
    } catch (const DegenerateRotation&) {
      degenerate_quat = true;
      return;
    }
    S ts[2][3], tt[3][2], sp[2][2];
    matmul<S, 2, 3, 3>(t, sigma, ts);
    transpose<S, 2, 3>(t, tt);
    matmul<S, 2, 3, 2>(ts, tt, sp);                             // :89
    sp[0][0] += S(kCovarianceDilation);                         // :90-91
    sp[1][1] += S(kCovarianceDilation);
    const S det = sp[0][0] * sp[1][1] - sp[0][1] * sp[1][0];    // :93
    if (!(det > S(0))) {
      c.state[i] = 2;
      return;
    }
    const S mid = (sp[0][0] + sp[1][1]) / S(2);                 // :99-102
    const S lambda_max = mid + std::sqrt(std::max(mid * mid - det, S(0)));
    const int radius = static_cast<int>(std::ceil(S(kRadiusSigma) * std::sqrt(lambda_max)));
    const S mx = pixel[0], my = pixel[1];                        // :106-109
    if (mx + S(radius) < S(0) || mx - S(radius) > S(c.cam.width) || my + S(radius) < S(0) ||
        my - S(radius) > S(c.cam.height))
      return;
    Splat<S>& s = slots[i];
    s.mean_px[0] = pixel[0];
    s.mean_px[1] = pixel[1];
    s.conic[0] = sp[1][1] / det;                                // :113
    s.conic[1] = -sp[0][1] / det;
    s.conic[2] = sp[0][0] / det;
    s.depth = c.cam.model == CAM_PINHOLE ? mu[2] : std::sqrt(mu[0] * mu[0] + mu[1] * mu[1] + mu[2] * mu[2]);
    s.radius = radius;
    S v[3] = {mean[0] - cam_center[0], mean[1] - cam_center[1], mean[2] - cam_center[2]};
    const S vn2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];      // Eigen normalized(): v / sqrt(|v|^2)
    S dir[3] = {v[0], v[1], v[2]};
    if (vn2 > S(0)) {
      const S nrm = std::sqrt(vn2);
      dir[0] = v[0] / nrm; dir[1] = v[1] / nrm; dir[2] = v[2] / nrm;
    }
    eval_sh(&c.scene.sh[i * 48], dir, c.sh_degree, s.color);   // :117
    s.alpha = sigmoid(c.scene.opacity[i]);                      // :118
    s.source = static_cast<int>(i);
    points[i * 3 + 0] = mu[0]; points[i * 3 + 1] = mu[1]; points[i * 3 + 2] = mu[2];
    c.state[i] = 1;
  }, threads);
  if (degenerate_quat) throw DegenerateRotation();
  c.splats.clear();
  c.cam_points.clear();
  c.num_culled = c.num_degenerate = 0;
  for (int64_t i = 0; i < n; ++i) {                              // :125-138 stable compaction
    if (c.state[i] == 1) {
      c.splats.push_back(slots[i]);
      c.cam_points.insert(c.cam_points.end(), &points[i * 3], &points[i * 3] + 3);
    } else if (c.state[i] == 2) {
      ++c.num_degenerate;
    } else {
      ++c.num_culled;
    }
  }
}

// inc/splatting.hpp:143-151
inline uint64_t depth_key_bits(float d) {
  uint32_t u;
  std::memcpy(&u, &d, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
inline uint64_t depth_key_bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// inc/splatting.hpp:154-180 — stable LSD byte radix sort, skipping constant-digit passes.
template <typename Key, typename Payload>
void radix_sort_pairs(std::vector<Key>& keys, std::vector<Payload>& payload) {
  const size_t n = keys.size();
  std::vector<Key> kt(n);
  std::vector<Payload> pt(n);
  for (int pass = 0; pass < static_cast<int>(sizeof(Key)); ++pass) {
    const int shift = pass * 8;
    size_t count[256] = {0};
    for (size_t i = 0; i < n; ++i) ++count[(keys[i] >> shift) & 0xff];
    if (count[(keys.empty() ? 0 : (keys[0] >> shift)) & 0xff] == n) continue;
    size_t sum = 0;
    for (int d = 0; d < 256; ++d) {
      const size_t cc = count[d];
      count[d] = sum;
      sum += cc;
    }
    for (size_t i = 0; i < n; ++i) {
      const size_t dst = count[(keys[i] >> shift) & 0xff]++;
      kt[dst] = keys[i];
      pt[dst] = payload[i];
    }
    keys.swap(kt);
    payload.swap(pt);
  }
}

// inc/splatting.hpp:196-249
template <typename S>
void bin_and_sort(Ctx<S>& c) {
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  const int W = c.cam.width, H = c.cam.height;
  c.tiles_x = (W + kTileSize - 1) / kTileSize;
  c.tiles_y = (H + kTileSize - 1) / kTileSize;
  c.key_tile.clear(); c.key_depth.clear(); c.key_splat.clear();
  for (size_t i = 0; i < c.splats.size(); ++i) {
    const Splat<S>& sp = c.splats[i];
    const S r = S(sp.radius);
    const int tx0 = std::max(0, static_cast<int>(std::floor((sp.mean_px[0] - r) / kTileSize)));
    const int tx1 = std::min(c.tiles_x - 1, static_cast<int>(std::floor((sp.mean_px[0] + r) / kTileSize)));
    const int ty0 = std::max(0, static_cast<int>(std::floor((sp.mean_px[1] - r) / kTileSize)));
    const int ty1 = std::min(c.tiles_y - 1, static_cast<int>(std::floor((sp.mean_px[1] + r) / kTileSize)));
    const uint64_t dk = depth_key_bits(sp.depth);
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) {
        c.key_tile.push_back(static_cast<uint32_t>(ty * c.tiles_x + tx));
        c.key_depth.push_back(dk);
        c.key_splat.push_back(static_cast<uint32_t>(i));
      }
  }
  const auto t1 = clock::now();
  const size_t I = c.key_tile.size();
  std::vector<uint64_t> tile_and_splat(I);
  for (size_t i = 0; i < I; ++i) tile_and_splat[i] = (uint64_t(c.key_tile[i]) << 32) | c.key_splat[i];
  if (sizeof(S) == 4) {
    std::vector<uint32_t> dk(I);
    for (size_t i = 0; i < I; ++i) dk[i] = static_cast<uint32_t>(c.key_depth[i]);
    radix_sort_pairs(dk, tile_and_splat);
  } else {
    std::vector<uint64_t> dk(c.key_depth);
    radix_sort_pairs(dk, tile_and_splat);
  }
  std::vector<uint32_t> tile_keys(I);
  c.refs.assign(I, 0);
  for (size_t i = 0; i < I; ++i) {
    tile_keys[i] = static_cast<uint32_t>(tile_and_splat[i] >> 32);
    c.refs[i] = static_cast<uint32_t>(tile_and_splat[i] & 0xffffffffu);
  }
  radix_sort_pairs(tile_keys, c.refs);
  c.offsets.assign(static_cast<size_t>(c.tiles_x) * c.tiles_y + 1, 0);
  for (const uint32_t t : tile_keys) ++c.offsets[t + 1];
  for (size_t t = 1; t < c.offsets.size(); ++t) c.offsets[t] += c.offsets[t - 1];
  const auto t2 = clock::now();
  c.bin_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  c.sort_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
  // inc/splatting.hpp:241-244 (capacities taken as sizes)
  c.aux_bytes = double(I) * (sizeof(S) == 4 ? 4 : 8) + double(I) * 8 + double(I) * 4 + double(I) * 4 +
                double(c.offsets.size()) * 4;
}

// inc/splatting.hpp:258-306
template <typename S>
void rasterize(Ctx<S>& c, int threads) {
  const int W = c.cam.width, H = c.cam.height;
  c.image.assign(size_t(W) * H * 3, S(0));
  c.final_T.assign(size_t(W) * H, S(1));
  c.count.assign(size_t(W) * H, 0);
  const int ntiles = c.tiles_x * c.tiles_y;
  std::vector<uint64_t> ev(ntiles, 0), ec(ntiles, 0);
  parallel_for(ntiles, [&](int64_t t) {
    const int tx = static_cast<int>(t) % c.tiles_x, ty = static_cast<int>(t) / c.tiles_x;
    const uint32_t lo = c.offsets[t], hi = c.offsets[t + 1];
    const int px0 = tx * kTileSize, px1 = std::min(W, px0 + kTileSize);
    const int py0 = ty * kTileSize, py1 = std::min(H, py0 + kTileSize);
    uint64_t n_eval = 0, n_contrib = 0;
    for (int py = py0; py < py1; ++py)
      for (int px = px0; px < px1; ++px) {
        S trans = S(1);
        S col[3] = {0, 0, 0};
        uint16_t cnt = 0;
        for (uint32_t k = lo; k < hi; ++k) {
          ++n_eval;
          const Splat<S>& sp = c.splats[c.refs[k]];
          const S dx = S(px) + S(0.5) - sp.mean_px[0];
          const S dy = S(py) + S(0.5) - sp.mean_px[1];
          const S power = S(-0.5) * (sp.conic[0] * dx * dx + sp.conic[2] * dy * dy) - sp.conic[1] * dx * dy;
          if (power > S(0)) continue;
          const S alpha = std::min(S(kAlphaClamp), sp.alpha * t_exp<S>(power));
          if (alpha < S(kAlphaSkip)) continue;
          const S next_trans = trans * (S(1) - alpha);
          if (next_trans < S(kTransmittanceStop)) break;
          for (int ch = 0; ch < 3; ++ch) col[ch] = col[ch] + sp.color[ch] * (alpha * trans);
          trans = next_trans;
          ++cnt;
        }
        n_contrib += cnt;
        const size_t pix = size_t(py) * W + px;
        for (int ch = 0; ch < 3; ++ch) c.image[pix * 3 + ch] = col[ch] + trans * c.bg[ch];
        c.final_T[pix] = trans;
        c.count[pix] = cnt;
      }
    ev[t] = n_eval;
    ec[t] = n_contrib;
  }, threads);
  c.e_eval = c.e_contrib = 0;
  for (int t = 0; t < ntiles; ++t) {
    c.e_eval += ev[t];
    c.e_contrib += ec[t];
  }
}

// inc/splatting.hpp:330-374
template <typename S>
Ctx<S>* render(Ctx<S>* c, int threads) {
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  preprocess(*c, threads);
  const auto t1 = clock::now();
  bin_and_sort(*c);
  const auto t2 = clock::now();
  rasterize(*c, threads);
  const auto t3 = clock::now();
  c->pre_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  c->raster_ms = std::chrono::duration<double, std::milli>(t3 - t2).count();
  (void)t2;
  return c;
}

// ---------------------------------------------------------------------------------------
// Backward (inc/gradients.hpp)

template <typename S>
struct SplatGrad {
  S mean_px[2] = {0, 0};
  S conic[3] = {0, 0, 0};
  S color[3] = {0, 0, 0};
  S alpha = 0;
};

// inc/gradients.hpp:69-175
template <typename S>
void rasterize_backward(const Ctx<S>& c, const S* dl, std::vector<SplatGrad<S>>& out, int threads) {
  const int W = c.cam.width, H = c.cam.height;
  out.assign(c.splats.size(), SplatGrad<S>{});
  const int ntiles = c.tiles_x * c.tiles_y;
  std::vector<std::vector<SplatGrad<S>>> scratch(ntiles);
  struct Contribution { uint32_t ref; S alpha; S trans; };
  parallel_for(ntiles, [&](int64_t t) {
    const uint32_t lo = c.offsets[t], hi = c.offsets[t + 1];
    if (lo == hi) return;
    auto& sc = scratch[t];
    sc.assign(hi - lo, SplatGrad<S>{});
    const int tx = static_cast<int>(t) % c.tiles_x, ty = static_cast<int>(t) / c.tiles_x;
    const int px0 = tx * kTileSize, px1 = std::min(W, px0 + kTileSize);
    const int py0 = ty * kTileSize, py1 = std::min(H, py0 + kTileSize);
    std::vector<Contribution> contribs;
    contribs.reserve(hi - lo);
    for (int py = py0; py < py1; ++py)
      for (int px = px0; px < px1; ++px) {
        contribs.clear();
        S trans = S(1);
        for (uint32_t k = lo; k < hi; ++k) {
          const Splat<S>& sp = c.splats[c.refs[k]];
          const S dx = S(px) + S(0.5) - sp.mean_px[0];
          const S dy = S(py) + S(0.5) - sp.mean_px[1];
          const S power = S(-0.5) * (sp.conic[0] * dx * dx + sp.conic[2] * dy * dy) - sp.conic[1] * dx * dy;
          if (power > S(0)) continue;
          const S alpha = std::min(S(kAlphaClamp), sp.alpha * t_exp<S>(power));
          if (alpha < S(kAlphaSkip)) continue;
          const S next_trans = trans * (S(1) - alpha);
          if (next_trans < S(kTransmittanceStop)) break;
          contribs.push_back({k, alpha, trans});
          trans = next_trans;
        }
        const size_t pix = size_t(py) * W + px;
        const S dc[3] = {dl[pix * 3 + 0], dl[pix * 3 + 1], dl[pix * 3 + 2]};
        S suffix[3] = {trans * c.bg[0], trans * c.bg[1], trans * c.bg[2]};
        for (size_t m = contribs.size(); m-- > 0;) {
          const Contribution& cb = contribs[m];
          const Splat<S>& sp = c.splats[c.refs[cb.ref]];
          SplatGrad<S>& slot = sc[cb.ref - lo];
          const S weight = cb.alpha * cb.trans;
          for (int ch = 0; ch < 3; ++ch) slot.color[ch] = slot.color[ch] + dc[ch] * weight;
          const S dot_c = dc[0] * sp.color[0] + dc[1] * sp.color[1] + dc[2] * sp.color[2];
          const S dot_s = dc[0] * suffix[0] + dc[1] * suffix[1] + dc[2] * suffix[2];
          const S d_alpha = dot_c * cb.trans - dot_s / (S(1) - cb.alpha);
          for (int ch = 0; ch < 3; ++ch) suffix[ch] = suffix[ch] + sp.color[ch] * weight;
          const S dx = S(px) + S(0.5) - sp.mean_px[0];
          const S dy = S(py) + S(0.5) - sp.mean_px[1];
          const S power = S(-0.5) * (sp.conic[0] * dx * dx + sp.conic[2] * dy * dy) - sp.conic[1] * dx * dy;
          const S expp = t_exp<S>(power);
          if (sp.alpha * expp > S(kAlphaClamp)) continue;
          slot.alpha = slot.alpha + d_alpha * expp;
          const S d_power = d_alpha * cb.alpha;
          slot.mean_px[0] = slot.mean_px[0] + d_power * (sp.conic[0] * dx + sp.conic[1] * dy);
          slot.mean_px[1] = slot.mean_px[1] + d_power * (sp.conic[1] * dx + sp.conic[2] * dy);
          slot.conic[0] = slot.conic[0] + d_power * (S(-0.5) * dx * dx);
          slot.conic[1] = slot.conic[1] + d_power * (-dx * dy);
          slot.conic[2] = slot.conic[2] + d_power * (S(-0.5) * dy * dy);
        }
      }
  }, threads);
  for (int t = 0; t < ntiles; ++t) {  // :161-173 fixed-order reduction
    const auto& sc = scratch[t];
    if (sc.empty()) continue;
    const uint32_t lo = c.offsets[t];
    for (size_t s = 0; s < sc.size(); ++s) {
      SplatGrad<S>& o = out[c.refs[lo + s]];
      for (int q = 0; q < 2; ++q) o.mean_px[q] = o.mean_px[q] + sc[s].mean_px[q];
      for (int q = 0; q < 3; ++q) o.conic[q] = o.conic[q] + sc[s].conic[q];
      for (int q = 0; q < 3; ++q) o.color[q] = o.color[q] + sc[s].color[q];
      o.alpha = o.alpha + sc[s].alpha;
    }
  }
}

constexpr int kGradStride = 59;  // mean 3, rotation 4, log_scale 3, opacity 1, sh 48

// inc/gradients.hpp:207-267. full_sh != 0 adds the 45 higher-band SH gradients (not in
// the reference, which returns DC only: inc/gradients.hpp:262, inc/model.hpp:219-227).
template <typename S>
void backward(const Ctx<S>& c, const S* dl, S* grads, const S jgs[3], int full_sh, int view_dir, int threads,
              std::vector<SplatGrad<S>>* sg_out) {
  std::vector<SplatGrad<S>> sg;
  rasterize_backward(c, dl, sg, threads);
  const int64_t n = c.scene.n;
  std::fill(grads, grads + n * kGradStride, S(0));
  S cam_center[3];
  camera_center(c.cam, cam_center);
  parallel_for(static_cast<int64_t>(c.splats.size()), [&](int64_t i) {
    const Splat<S>& sp = c.splats[i];
    const int src = sp.source;
    const S* mu = &c.cam_points[i * 3];
    S j[2][3];
    projection_jacobian(mu, c.cam, j);
    // :177-181 mean_backward: J^T dmean_px
    S direct[3];
    for (int k = 0; k < 3; ++k) direct[k] = j[0][k] * sg[i].mean_px[0] + j[1][k] * sg[i].mean_px[1];
    // :239-243
    const S q[2][2] = {{sp.conic[0], sp.conic[1]}, {sp.conic[1], sp.conic[2]}};
    const S gq[2][2] = {{sg[i].conic[0], sg[i].conic[1] / S(2)}, {sg[i].conic[1] / S(2), sg[i].conic[2]}};
    const S nq[2][2] = {{-q[0][0], -q[0][1]}, {-q[1][0], -q[1][1]}};
    S tmp[2][2], dsp[2][2];
    matmul<S, 2, 2, 2>(nq, gq, tmp);
    matmul<S, 2, 2, 2>(tmp, q, dsp);
    S sigma[3][3];
    build_covariance(&c.scene.rotations[src * 4], &c.scene.log_scales[src * 3], sigma);
    // :186-202 covariance_projection_backward
    S t[2][3], tt[3][2];
    matmul<S, 2, 3, 3>(j, c.cam.W, t);
    transpose<S, 2, 3>(t, tt);
    S a32[3][2], dsig[3][3];
    matmul<S, 3, 2, 2>(tt, dsp, a32);
    matmul<S, 3, 2, 3>(a32, t, dsig);
    S gs[2][2] = {{dsp[0][0] + dsp[0][0], dsp[0][1] + dsp[1][0]}, {dsp[1][0] + dsp[0][1], dsp[1][1] + dsp[1][1]}};
    S b23[2][3], dldt[2][3], wt[3][3], dldj[2][3];
    matmul<S, 2, 2, 3>(gs, t, b23);
    matmul<S, 2, 3, 3>(b23, sigma, dldt);
    transpose<S, 3, 3>(c.cam.W, wt);
    matmul<S, 2, 3, 3>(dldt, wt, dldj);
    S dj[3][2][3];
    projection_jacobian_grad(mu, c.cam, dj);
    S cov[3];
    for (int k = 0; k < 3; ++k) cov[k] = jgs[k] * cwise_sum_colmajor<S, 2, 3>(dldj, dj[k]);
    S dq[4], ds[3];
    build_covariance_backward(&c.scene.rotations[src * 4], &c.scene.log_scales[src * 3], dsig, dq, ds);
    // :251-252
    const S v[3] = {direct[0] + cov[0], direct[1] + cov[1], direct[2] + cov[2]};
    S* g = grads + int64_t(src) * kGradStride;
    for (int r = 0; r < 3; ++r) g[r] = c.cam.W[0][r] * v[0] + c.cam.W[1][r] * v[1] + c.cam.W[2][r] * v[2];
    for (int k = 0; k < 4; ++k) g[3 + k] = dq[k];
    for (int k = 0; k < 3; ++k) g[7 + k] = ds[k];
    const S a = sigmoid(c.scene.opacity[src]);
    g[10] = sg[i].alpha * a * (S(1) - a);                      // :261
    const S* mean = &c.scene.means[src * 3];
    S vv[3] = {mean[0] - cam_center[0], mean[1] - cam_center[1], mean[2] - cam_center[2]};
    const S vn2 = vv[0] * vv[0] + vv[1] * vv[1] + vv[2] * vv[2];
    S dir[3] = {vv[0], vv[1], vv[2]};
    if (vn2 > S(0)) {
      const S nrm = std::sqrt(vn2);
      dir[0] = vv[0] / nrm; dir[1] = vv[1] / nrm; dir[2] = vv[2] / nrm;
    }
    S color[3], basis[16];
    eval_sh(&c.scene.sh[src * 48], dir, c.sh_degree, color, basis);
    const int nb = full_sh ? (c.sh_degree + 1) * (c.sh_degree + 1) : 1;
    for (int ch = 0; ch < 3; ++ch) {
      if (!(color[ch] > S(0))) continue;                        // inc/model.hpp:224-225
      g[11 + ch * 16 + 0] = S(kC0) * sg[i].color[ch];
      for (int jb = 1; jb < nb; ++jb) g[11 + ch * 16 + jb] = basis[jb] * sg[i].color[ch];
    }
    if (view_dir && c.sh_degree > 0 && vn2 > S(0)) {
      // colour -> dir -> mean (omitted by the reference, inc/gradients.hpp:255-262)
      S dY[16][3];
      sh_basis_grad(dir, c.sh_degree, dY);
      const int nbd = (c.sh_degree + 1) * (c.sh_degree + 1);
      S ddir[3] = {0, 0, 0};
      for (int ch = 0; ch < 3; ++ch) {
        if (!(color[ch] > S(0))) continue;
        const S* k = &c.scene.sh[src * 48 + ch * 16];
        for (int jb = 1; jb < nbd; ++jb)
          for (int a = 0; a < 3; ++a) ddir[a] += sg[i].color[ch] * k[jb] * dY[jb][a];
      }
      const S nrm = std::sqrt(vn2);
      const S dd = dir[0] * ddir[0] + dir[1] * ddir[1] + dir[2] * ddir[2];
      for (int a = 0; a < 3; ++a) g[a] += (ddir[a] - dir[a] * dd) / nrm;
    }
  }, threads);
  if (sg_out) sg_out->swap(sg);
}

// ---------------------------------------------------------------------------------------
// Brute-force renderer (inc/oracle.hpp:161-270): independent projection in double, per
// pixel walk over all splats in global (depth, source) order behind a tile-overlap gate.

struct OSplat {
  double mx, my, a, b, c, depth, color[3], alpha;
  int radius, source;
};

inline bool oproject(const double p[3], const Camera<double>& cam, double pix[2], double jac[2][3]) {
  const double x = p[0], y = p[1], z = p[2];
  if (x * x + y * y + z * z < 1e-24) return false;
  if (cam.model == CAM_PINHOLE) {
    if (z <= kPinholeNearClip) return false;
    pix[0] = cam.cx + cam.fx * x / z; pix[1] = cam.cy + cam.fy * y / z;
    jac[0][0] = cam.fx / z; jac[0][1] = 0; jac[0][2] = -cam.fx * x / (z * z);
    jac[1][0] = 0; jac[1][1] = cam.fy / z; jac[1][2] = -cam.fy * y / (z * z);
    return true;
  }
  if (cam.model == CAM_FISHEYE) {  // inc/oracle.hpp:115-136
    const double lz = std::sqrt(x * x + y * y);
    if (z < 0.0 && lz * lz < 1e-24 * z * z) return false;
    const double theta = std::atan2(lz, z);
    if (theta > cam.fov_max + kFisheyeCullMarginRad) return false;
    const double l2 = x * x + y * y + z * z;
    if (lz < 1e-8 * std::abs(z)) {
      pix[0] = cam.cx + cam.fx * x / z; pix[1] = cam.cy + cam.fy * y / z;
      jac[0][0] = cam.fx / z; jac[0][1] = 0; jac[0][2] = -cam.fx * x / (z * z);
      jac[1][0] = 0; jac[1][1] = cam.fy / z; jac[1][2] = -cam.fy * y / (z * z);
      return true;
    }
    pix[0] = cam.cx + cam.fx * theta * x / lz; pix[1] = cam.cy + cam.fy * theta * y / lz;
    const double lz2 = lz * lz, lz3 = lz2 * lz;
    jac[0][0] = cam.fx * (x * x * z / (lz2 * l2) + y * y * theta / lz3);
    jac[0][1] = cam.fx * x * y * (z / (lz2 * l2) - theta / lz3);
    jac[0][2] = -cam.fx * x / l2;
    jac[1][0] = cam.fy * x * y * (z / (lz2 * l2) - theta / lz3);
    jac[1][1] = cam.fy * (y * y * z / (lz2 * l2) + x * x * theta / lz3);
    jac[1][2] = -cam.fy * y / l2;
    return true;
  }
  const double s = x * x + z * z;  // panorama
  if (s < 1e-24 * y * y) return false;
  const double rho = std::sqrt(s), l2 = s + y * y, two_pi = 2.0 * 3.141592653589793238462643383279502884;
  double xp = cam.width * (std::atan2(x, z) + two_pi / 2.0) / two_pi;
  if (xp >= cam.width) xp -= cam.width;
  pix[0] = xp;
  pix[1] = cam.height * (std::atan2(y, rho) + two_pi / 4.0) / (two_pi / 2.0);
  jac[0][0] = cam.width * z / (two_pi * s); jac[0][1] = 0; jac[0][2] = -cam.width * x / (two_pi * s);
  const double hpi = cam.height / (two_pi / 2.0);
  jac[1][0] = -hpi * x * y / (rho * l2); jac[1][1] = hpi * rho / l2; jac[1][2] = -hpi * y * z / (rho * l2);
  return true;
}

inline double osh(const double* k, const double d[3], int degree) {  // inc/oracle.hpp:75-99
  const double x = d[0], y = d[1], z = d[2];
  double v = 0.28209479177387814 * k[0];
  if (degree >= 1) v += -0.4886025119029199 * y * k[1] + 0.4886025119029199 * z * k[2] - 0.4886025119029199 * x * k[3];
  if (degree >= 2) {
    const double xx = x * x, yy = y * y, zz = z * z;
    v += 1.0925484305920792 * x * y * k[4] - 1.0925484305920792 * y * z * k[5] +
         0.31539156525252005 * (2.0 * zz - xx - yy) * k[6] - 1.0925484305920792 * x * z * k[7] +
         0.5462742152960396 * (xx - yy) * k[8];
  }
  if (degree >= 3) {
    const double xx = x * x, yy = y * y, zz = z * z;
    v += -0.5900435899266435 * y * (3.0 * xx - yy) * k[9] + 2.890611442640554 * x * y * z * k[10] -
         0.4570457994644658 * y * (4.0 * zz - xx - yy) * k[11] +
         0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy) * k[12] -
         0.4570457994644658 * x * (4.0 * zz - xx - yy) * k[13] + 1.445305721320277 * z * (xx - yy) * k[14] -
         0.5900435899266435 * x * (xx - yy) * k[15];
  }
  return std::max(v + 0.5, 0.0);
}

inline void bruteforce_render(const Scene<double>& sc, const Camera<double>& cam, int sh_degree, double* img,
                              double* trans_out) {
  const double* W = &cam.W[0][0];
  double center[3];
  for (int r = 0; r < 3; ++r) center[r] = -(W[0 * 3 + r] * cam.b[0] + W[1 * 3 + r] * cam.b[1] + W[2 * 3 + r] * cam.b[2]);
  std::vector<OSplat> sp;
  for (int64_t i = 0; i < sc.n; ++i) {
    const double* m = &sc.means[i * 3];
    double mu[3];
    for (int r = 0; r < 3; ++r) mu[r] = W[r * 3] * m[0] + W[r * 3 + 1] * m[1] + W[r * 3 + 2] * m[2] + cam.b[r];
    double pix[2], jac[2][3];
    if (!oproject(mu, cam, pix, jac)) continue;
    const double* q = &sc.rotations[i * 4];
    const double qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(qn > 0)) throw DegenerateRotation();
    const double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
    const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                            {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                            {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    double s2[3];
    for (int k = 0; k < 3; ++k) s2[k] = std::exp(2.0 * sc.log_scales[i * 3 + k]);
    double sig[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) sig[a][b] = R[a][0] * s2[0] * R[b][0] + R[a][1] * s2[1] * R[b][1] + R[a][2] * s2[2] * R[b][2];
    double T[2][3];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) T[a][b] = jac[a][0] * W[0 * 3 + b] + jac[a][1] * W[1 * 3 + b] + jac[a][2] * W[2 * 3 + b];
    double P[2][2];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        double acc = 0;
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) acc += T[a][k] * sig[k][l] * T[b][l];
        P[a][b] = acc;
      }
    P[0][0] += kCovarianceDilation;
    P[1][1] += kCovarianceDilation;
    const double det = P[0][0] * P[1][1] - P[0][1] * P[1][0];
    if (!(det > 0.0)) continue;
    const double mid = 0.5 * (P[0][0] + P[1][1]);
    const double lmax = mid + std::sqrt(std::max(mid * mid - det, 0.0));
    const int radius = static_cast<int>(std::ceil(kRadiusSigma * std::sqrt(lmax)));
    if (pix[0] + radius < 0 || pix[0] - radius > cam.width || pix[1] + radius < 0 || pix[1] - radius > cam.height) continue;
    OSplat o;
    o.mx = pix[0]; o.my = pix[1];
    o.a = P[1][1] / det; o.b = -P[0][1] / det; o.c = P[0][0] / det;
    o.depth = cam.model == CAM_PINHOLE ? mu[2] : std::sqrt(mu[0] * mu[0] + mu[1] * mu[1] + mu[2] * mu[2]);
    o.radius = radius;
    double d[3] = {m[0] - center[0], m[1] - center[1], m[2] - center[2]};
    const double dn = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int k = 0; k < 3; ++k) d[k] /= dn;
    for (int ch = 0; ch < 3; ++ch) o.color[ch] = osh(&sc.sh[i * 48 + ch * 16], d, sh_degree);
    o.alpha = 1.0 / (1.0 + std::exp(-sc.opacity[i]));
    o.source = static_cast<int>(i);
    sp.push_back(o);
  }
  std::sort(sp.begin(), sp.end(), [](const OSplat& a, const OSplat& b) {
    return a.depth != b.depth ? a.depth < b.depth : a.source < b.source;
  });
  for (int py = 0; py < cam.height; ++py)
    for (int px = 0; px < cam.width; ++px) {
      const int tx0 = (px / kTileSize) * kTileSize, ty0 = (py / kTileSize) * kTileSize;
      double trans = 1.0, col[3] = {0, 0, 0};
      for (const auto& s : sp) {
        if (s.mx + s.radius < tx0 || s.mx - s.radius >= tx0 + kTileSize || s.my + s.radius < ty0 ||
            s.my - s.radius >= ty0 + kTileSize)
          continue;
        const double dx = px + 0.5 - s.mx, dy = py + 0.5 - s.my;
        const double power = -0.5 * (s.a * dx * dx + s.c * dy * dy) - s.b * dx * dy;
        if (power > 0) continue;
        const double alpha = std::min(kAlphaClamp, s.alpha * std::exp(power));
        if (alpha < kAlphaSkip) continue;
        const double nt = trans * (1.0 - alpha);
        if (nt < kTransmittanceStop) break;
        for (int ch = 0; ch < 3; ++ch) col[ch] += s.color[ch] * (alpha * trans);
        trans = nt;
      }
      const size_t pix = size_t(py) * cam.width + px;
      for (int ch = 0; ch < 3; ++ch) img[pix * 3 + ch] = col[ch] + trans * sc.bg[ch];
      if (trans_out) trans_out[pix] = trans;
    }
}

thread_local std::string g_err;

template <typename S>
Scene<S> make_scene(int64_t n, const S* means, const S* rots, const S* ls, const S* op, const S* sh, const S* bg) {
  Scene<S> s;
  s.n = n;
  s.means.assign(means, means + n * 3);
  s.rotations.assign(rots, rots + n * 4);
  s.log_scales.assign(ls, ls + n * 3);
  s.opacity.assign(op, op + n);
  s.sh.assign(sh, sh + n * 48);
  if (bg) for (int k = 0; k < 3; ++k) s.bg[k] = bg[k];
  return s;
}

// cam: [model, w, h, fx, fy, cx, cy, R(9, row-major), t(3), fov_max] as doubles
template <typename S>
Camera<S> make_camera(const double* p) {
  Camera<S> c;
  c.model = static_cast<int>(p[0]);
  c.width = static_cast<int>(p[1]);
  c.height = static_cast<int>(p[2]);
  c.fx = S(p[3]); c.fy = S(p[4]); c.cx = S(p[5]); c.cy = S(p[6]);
  for (int i = 0; i < 9; ++i) c.W[i / 3][i % 3] = S(p[7 + i]);
  for (int i = 0; i < 3; ++i) c.b[i] = S(p[16 + i]);
  c.fov_max = S(p[19]);
  return c;
}

struct AnyCtx {
  int is_double = 0;
  void* p = nullptr;
};

}  // namespace orc

using namespace orc;

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

#define ORC_RENDER_IMPL(S, NAME)                                                                        \
  void* NAME(int64_t n, const S* means, const S* rots, const S* ls, const S* op, const S* sh,          \
             const double* cam, const S* bg, int sh_degree, int threads, int mode) {                   \
    g_mode = mode;                                                                                      \
    auto* c = new Ctx<S>();                                                                             \
    try {                                                                                               \
      c->scene = make_scene<S>(n, means, rots, ls, op, sh, bg);                                         \
      c->cam = make_camera<S>(cam);                                                                     \
      c->sh_degree = sh_degree;                                                                         \
      for (int k = 0; k < 3; ++k) c->bg[k] = c->scene.bg[k];                                            \
      render(c, threads);                                                                               \
    } catch (const std::exception& e) {                                                                 \
      g_err = e.what();                                                                                 \
      delete c;                                                                                         \
      return nullptr;                                                                                   \
    }                                                                                                   \
    auto* a = new AnyCtx();                                                                             \
    a->is_double = sizeof(S) == 8;                                                                      \
    a->p = c;                                                                                           \
    return a;                                                                                           \
  }
ORC_RENDER_IMPL(float, orc_render_f32)
ORC_RENDER_IMPL(double, orc_render_f64)

void orc_free(void* h) {
  auto* a = static_cast<AnyCtx*>(h);
  if (!a) return;
  if (a->is_double) delete static_cast<Ctx<double>*>(a->p);
  else delete static_cast<Ctx<float>*>(a->p);
  delete a;
}

// sizes: [n, num_splats, num_isect, tiles_x, tiles_y, width, height]
void orc_sizes(void* h, int64_t* out) {
  auto* a = static_cast<AnyCtx*>(h);
  auto fill = [&](auto* c) {
    out[0] = c->scene.n; out[1] = static_cast<int64_t>(c->splats.size());
    out[2] = static_cast<int64_t>(c->key_tile.size()); out[3] = c->tiles_x; out[4] = c->tiles_y;
    out[5] = c->cam.width; out[6] = c->cam.height;
  };
  if (a->is_double) fill(static_cast<Ctx<double>*>(a->p)); else fill(static_cast<Ctx<float>*>(a->p));
}

// stats: [num_isect, num_splats, num_culled, num_degenerate, pre_ms, bin_ms, sort_ms, raster_ms,
//         aux_bytes, e_eval, e_contrib]
void orc_stats(void* h, double* out) {
  auto* a = static_cast<AnyCtx*>(h);
  auto fill = [&](auto* c) {
    out[0] = double(c->key_tile.size()); out[1] = double(c->splats.size());
    out[2] = c->num_culled; out[3] = c->num_degenerate; out[4] = c->pre_ms; out[5] = c->bin_ms;
    out[6] = c->sort_ms; out[7] = c->raster_ms; out[8] = c->aux_bytes;
    out[9] = double(c->e_eval); out[10] = double(c->e_contrib);
  };
  if (a->is_double) fill(static_cast<Ctx<double>*>(a->p)); else fill(static_cast<Ctx<float>*>(a->p));
}

// Copy a named array out of the context (element type: S for reals, int32/uint32/uint16/uint64
// for the integer arrays). Returns the number of elements, -1 for an unknown name.
int64_t orc_get(void* h, const char* name, void* dst) {
  auto* a = static_cast<AnyCtx*>(h);
  auto get = [&](auto* c) -> int64_t {
    using S = std::remove_reference_t<decltype(c->image[0])>;
    const std::string nm(name);
    const int64_t nv = static_cast<int64_t>(c->splats.size());
    auto put = [&](const auto* src, int64_t cnt) {
      if (dst) std::memcpy(dst, src, cnt * sizeof(*src));
      return cnt;
    };
    if (nm == "state") return put(c->state.data(), c->state.size());
    if (nm == "image") return put(c->image.data(), c->image.size());
    if (nm == "final_T") return put(c->final_T.data(), c->final_T.size());
    if (nm == "count") return put(c->count.data(), c->count.size());
    if (nm == "refs") return put(c->refs.data(), c->refs.size());
    if (nm == "offsets") return put(c->offsets.data(), c->offsets.size());
    if (nm == "key_tile") return put(c->key_tile.data(), c->key_tile.size());
    if (nm == "key_splat") return put(c->key_splat.data(), c->key_splat.size());
    if (nm == "key_depth") return put(c->key_depth.data(), c->key_depth.size());
    if (nm == "cam_points") return put(c->cam_points.data(), c->cam_points.size());
    std::vector<S> tmp;
    std::vector<int32_t> itmp;
    if (nm == "mean_px") { for (auto& s : c->splats) { tmp.push_back(s.mean_px[0]); tmp.push_back(s.mean_px[1]); } return put(tmp.data(), 2 * nv); }
    if (nm == "conic") { for (auto& s : c->splats) for (int k = 0; k < 3; ++k) tmp.push_back(s.conic[k]); return put(tmp.data(), 3 * nv); }
    if (nm == "color") { for (auto& s : c->splats) for (int k = 0; k < 3; ++k) tmp.push_back(s.color[k]); return put(tmp.data(), 3 * nv); }
    if (nm == "depth") { for (auto& s : c->splats) tmp.push_back(s.depth); return put(tmp.data(), nv); }
    if (nm == "alpha") { for (auto& s : c->splats) tmp.push_back(s.alpha); return put(tmp.data(), nv); }
    if (nm == "radius") { for (auto& s : c->splats) itmp.push_back(s.radius); return put(itmp.data(), nv); }
    if (nm == "source") { for (auto& s : c->splats) itmp.push_back(s.source); return put(itmp.data(), nv); }
    return -1;
  };
  return a->is_double ? get(static_cast<Ctx<double>*>(a->p)) : get(static_cast<Ctx<float>*>(a->p));
}

// inc/gradients.hpp:207-267. grads: n x 59 (mean 3, rotation 4, log_scale 3, opacity 1, sh 48
// [c*16+j]). splat_grads (optional): num_splats x 9 (d_mean_px 2, d_conic 3, d_color 3, d_alpha 1).
// Returns 0 on success, -1 on error (orc_last_error()).
#define ORC_BACKWARD_IMPL(S, NAME)                                                                      \
  int NAME(void* h, int64_t n, const S* dl_dimage, S* grads, const double* jac_grad_scale, int full_sh, \
           int view_dir, int threads, int mode, S* splat_grads) {                                       \
    auto* a = static_cast<AnyCtx*>(h);                                                                  \
    if (!a || a->is_double != (sizeof(S) == 8)) { g_err = "backward: context precision mismatch"; return -1; } \
    auto* c = static_cast<Ctx<S>*>(a->p);                                                               \
    if (n != c->scene.n) { g_err = "backward: forward context was built for a different scene"; return -1; } \
    g_mode = mode;                                                                                      \
    const S jgs[3] = {S(jac_grad_scale ? jac_grad_scale[0] : 1.0), S(jac_grad_scale ? jac_grad_scale[1] : 1.0), \
                      S(jac_grad_scale ? jac_grad_scale[2] : 1.0)};                                     \
    try {                                                                                               \
      std::vector<SplatGrad<S>> sg;                                                                     \
      backward(*c, dl_dimage, grads, jgs, full_sh, view_dir, threads, &sg);                                       \
      if (splat_grads)                                                                                  \
        for (size_t i = 0; i < sg.size(); ++i) {                                                        \
          S* o = splat_grads + i * 9;                                                                   \
          o[0] = sg[i].mean_px[0]; o[1] = sg[i].mean_px[1];                                             \
          for (int k = 0; k < 3; ++k) { o[2 + k] = sg[i].conic[k]; o[5 + k] = sg[i].color[k]; }         \
          o[8] = sg[i].alpha;                                                                           \
        }                                                                                               \
    } catch (const std::exception& e) { g_err = e.what(); return -1; }                                 \
    return 0;                                                                                           \
  }
ORC_BACKWARD_IMPL(float, orc_backward_f32)
ORC_BACKWARD_IMPL(double, orc_backward_f64)

// inc/oracle.hpp:231-270 (double only). Returns 0 / -1.
int orc_bruteforce_render_f64(int64_t n, const double* means, const double* rots, const double* ls,
                              const double* op, const double* sh, const double* cam, const double* bg,
                              int sh_degree, double* image, double* trans) {
  try {
    auto sc = make_scene<double>(n, means, rots, ls, op, sh, bg);
    auto c = make_camera<double>(cam);
    bruteforce_render(sc, c, sh_degree, image, trans);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
  return 0;
}

// inc/oracle.hpp:273-290
uint64_t orc_bruteforce_intersections(int64_t nv, const double* mean_px, const int32_t* radius, int width,
                                      int height) {
  const int tiles_x = (width + kTileSize - 1) / kTileSize, tiles_y = (height + kTileSize - 1) / kTileSize;
  uint64_t count = 0;
  for (int64_t i = 0; i < nv; ++i) {
    const double mx = mean_px[2 * i], my = mean_px[2 * i + 1], r = radius[i];
    for (int ty = 0; ty < tiles_y; ++ty)
      for (int tx = 0; tx < tiles_x; ++tx) {
        const double x0 = tx * kTileSize, y0 = ty * kTileSize;
        if (mx + r >= x0 && mx - r < x0 + kTileSize && my + r >= y0 && my - r < y0 + kTileSize) ++count;
      }
  }
  return count;
}

// Camera-level probes used by the ported known-answer tests (double and float).
// project: returns visible; pixel[2], jac[6] row-major. force: 0 auto, 1 series, 2 general.
int orc_project_f64(const double* cam, const double* p, double* pixel, double* jac, int force) {
  auto c = make_camera<double>(cam);
  double j[2][3] = {{0, 0, 0}, {0, 0, 0}};
  const bool v = project(p, c, pixel, j, force);
  if (force && c.model == CAM_FISHEYE) projection_jacobian(p, c, j, force);
  if (jac) std::memcpy(jac, j, sizeof(j));
  return v ? 1 : 0;
}
int orc_project_f32(const double* cam, const float* p, float* pixel, float* jac, int mode) {
  g_mode = mode;
  auto c = make_camera<float>(cam);
  float j[2][3] = {{0, 0, 0}, {0, 0, 0}};
  const bool v = project(p, c, pixel, j, 0);
  if (jac) std::memcpy(jac, j, sizeof(j));
  return v ? 1 : 0;
}
void orc_jacobian_grad_f64(const double* cam, const double* p, double* out18) {
  auto c = make_camera<double>(cam);
  double d[3][2][3];
  projection_jacobian_grad(p, c, d);
  std::memcpy(out18, d, sizeof(d));
}
int orc_build_covariance_f64(const double* q, const double* s, double* sigma9) {
  try {
    double sg[3][3];
    build_covariance(q, s, sg);
    std::memcpy(sigma9, sg, sizeof(sg));
  } catch (const std::exception& e) { g_err = e.what(); return -1; }
  return 0;
}
int orc_build_covariance_backward_f64(const double* q, const double* s, const double* g9, double* dq, double* ds) {
  try {
    double g[3][3];
    std::memcpy(g, g9, sizeof(g));
    build_covariance_backward(q, s, g, dq, ds);
  } catch (const std::exception& e) { g_err = e.what(); return -1; }
  return 0;
}
void orc_eval_sh_f64(const double* sh48, const double* dir, int degree, double* out3) {
  eval_sh(sh48, dir, degree, out3);
}

// Splat-level entry (the reference tests' hand-built Splat2D lists, e.g. simple_splat in
// tests/test_splatting.cpp:44-54): bin_and_sort + rasterize over given splats, double precision.
void* orc_splats_render_f64(int64_t nv, const double* mean_px, const double* conic, const double* depth,
                            const int32_t* radius, const double* color, const double* alpha, int width, int height,
                            const double* bg, int threads) {
  auto* c = new Ctx<double>();
  c->cam.model = CAM_PINHOLE;
  c->cam.width = width;
  c->cam.height = height;
  c->scene.n = nv;
  for (int k = 0; k < 3; ++k) c->bg[k] = bg ? bg[k] : 0.0;
  for (int64_t i = 0; i < nv; ++i) {
    Splat<double> s;
    s.mean_px[0] = mean_px[2 * i]; s.mean_px[1] = mean_px[2 * i + 1];
    for (int k = 0; k < 3; ++k) { s.conic[k] = conic[3 * i + k]; s.color[k] = color[3 * i + k]; }
    s.depth = depth[i];
    s.radius = radius[i];
    s.alpha = alpha[i];
    s.source = static_cast<int>(i);
    c->splats.push_back(s);
    c->cam_points.insert(c->cam_points.end(), {0.0, 0.0, 1.0});
  }
  c->state.assign(nv, 1);
  bin_and_sort(*c);
  rasterize(*c, threads);
  auto* a = new AnyCtx();
  a->is_double = 1;
  a->p = c;
  return a;
}

// rasterize_backward only (inc/gradients.hpp:69-175): splat_grads num_splats x 9.
int orc_splats_backward_f64(void* h, const double* dl, double* splat_grads, int threads) {
  auto* a = static_cast<AnyCtx*>(h);
  if (!a || !a->is_double) { g_err = "precision mismatch"; return -1; }
  auto* c = static_cast<Ctx<double>*>(a->p);
  std::vector<SplatGrad<double>> sg;
  rasterize_backward(*c, dl, sg, threads);
  for (size_t i = 0; i < sg.size(); ++i) {
    double* o = splat_grads + i * 9;
    o[0] = sg[i].mean_px[0]; o[1] = sg[i].mean_px[1];
    for (int k = 0; k < 3; ++k) { o[2 + k] = sg[i].conic[k]; o[5 + k] = sg[i].color[k]; }
    o[8] = sg[i].alpha;
  }
  return 0;
}

}  // extern "C"
