// preprocess.cu — K1 (preprocess) and K4b (preprocess backward), sm_100a. The camera model
// (equidistant fisheye, pinhole, equirectangular panorama) only matters here: binning, sort
// and blends are camera-agnostic (splatting.hpp:65-67).
//
// Compiled with --fmad=false: every expression below is evaluated in the reference's
// operation order with IEEE-rounded fp32 ops (division and sqrt are IEEE by default), so the
// per-Gaussian outputs (pixel mean, radius, depth, conic, colour, alpha) are bit-identical to
// the oracle's parity mode (oracle/fgs_oracle.cpp), and hence the tile/depth keys are too.
// atan2f/expf use the correctly rounded definition (double evaluation, one rounding).
//
// Reference: /root/reference/proj/include/omnisplat/
//   preprocess            splatting.hpp:68-139
//   project               cameras.hpp:139-177, fisheye_terms :99-128, jacobian :180-212
//   build_covariance      model.hpp:95-140; eval_sh model.hpp:187-215; sigmoid core.hpp:30-36
//   backward per splat    gradients.hpp:226-264, covariance_projection_backward :186-202,
//                         projection_jacobian_grad cameras.hpp:217-271,
//                         build_covariance_backward model.hpp:144-171

#include "fgs_common.cuh"
#include "fgs_crmath.cuh"
#include "fgs_kernels.h"

namespace fgs {

namespace {

constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2_0 = 1.0925484305920792, kC2_1 = -1.0925484305920792, kC2_2 = 0.31539156525252005,
                 kC2_3 = -1.0925484305920792, kC2_4 = 0.5462742152960396;
constexpr double kC3_0 = -0.5900435899266435, kC3_1 = 2.890611442640554, kC3_2 = -0.4570457994644658,
                 kC3_3 = 0.3731763325901154, kC3_4 = -0.4570457994644658, kC3_5 = 1.445305721320277,
                 kC3_6 = -0.5900435899266435;

struct Terms {
  float g, u, U;
};

// cameras.hpp:107-128 (AxisMode::Auto). theta = atan2(sqrt(lz2), z): the reference evaluates it
// again in every call (visibility, pixel, Jacobian, Jacobian gradient); the value is the same, so
// it is computed once per Gaussian and passed in.
__device__ __forceinline__ Terms fisheye_terms(float lz2, float z, float theta) {
  const float z2 = z * z;
  Terms t;
  if (z > 0.0f && lz2 < kFisheyeSeriesW2 * z2) {
    const float w2 = lz2 / z2;
    const float z3 = z2 * z, z5 = z3 * z2;
    t.g = (1.0f - w2 / 3.0f + w2 * w2 / 5.0f - w2 * w2 * w2 / 7.0f) / z;
    t.u = (-2.0f / 3.0f + 4.0f / 5.0f * w2 - 6.0f / 7.0f * w2 * w2) / z3;
    t.U = (8.0f / 5.0f - 24.0f / 7.0f * w2 + 16.0f / 3.0f * w2 * w2) / z5;
  } else {
    const float lz = sqrtf(lz2);
    const float r2 = lz2 + z2;
    t.g = theta / lz;
    t.u = z / (lz2 * r2) - theta / (lz2 * lz);
    t.U = 3.0f * theta / (lz2 * lz2 * lz) - z / (r2 * lz2 * lz2) - 2.0f * z * (r2 + lz2) / (lz2 * lz2 * r2 * r2);
  }
  return t;
}

// cameras.hpp:191-198
__device__ __forceinline__ void fisheye_jacobian(const float p[3], const DevCamera& cam, const Terms& t,
                                                 float j[2][3]) {
  const float x = p[0], y = p[1], z = p[2];
  const float lz2 = x * x + y * y;
  const float r2 = lz2 + z * z;
  const float fx = cam.fx, fy = cam.fy;
  j[0][0] = fx * (t.g + x * x * t.u);
  j[0][1] = fx * x * y * t.u;
  j[0][2] = -fx * x / r2;
  j[1][0] = fy * x * y * t.u;
  j[1][1] = fy * (t.g + y * y * t.u);
  j[1][2] = -fy * y / r2;
}

constexpr float kPi = 3.14159265358979323846f;  // pi<float>() (core.hpp)

// cameras.hpp:184-189
__device__ __forceinline__ void pinhole_jacobian(const float p[3], const DevCamera& cam, float j[2][3]) {
  const float x = p[0], y = p[1], z = p[2];
  const float iz = 1.0f / z;
  j[0][0] = cam.fx * iz; j[0][1] = 0.0f; j[0][2] = -cam.fx * x * iz * iz;
  j[1][0] = 0.0f; j[1][1] = cam.fy * iz; j[1][2] = -cam.fy * y * iz * iz;
}

// cameras.hpp:200-208
__device__ __forceinline__ void panorama_jacobian(const float p[3], const DevCamera& cam, float j[2][3]) {
  const float x = p[0], y = p[1], z = p[2];
  const float s = x * x + z * z;
  const float rho = sqrtf(s);
  const float r2 = s + y * y;
  const float cw = static_cast<float>(cam.width) / (2.0f * kPi);
  const float dh = static_cast<float>(cam.height) / kPi;
  j[0][0] = cw * z / s; j[0][1] = 0.0f; j[0][2] = -cw * x / s;
  j[1][0] = -dh * x * y / (rho * r2); j[1][1] = dh * rho / r2; j[1][2] = -dh * y * z / (rho * r2);
}

// cameras.hpp:223-230
__device__ __forceinline__ void pinhole_jacobian_grad(const float p[3], const DevCamera& cam, float d[3][2][3]) {
  const float x = p[0], y = p[1], z = p[2];
  const float iz2 = 1.0f / (z * z);
  const float fx = cam.fx, fy = cam.fy;
  d[0][0][0] = 0.0f; d[0][0][1] = 0.0f; d[0][0][2] = -fx * iz2;
  d[0][1][0] = 0.0f; d[0][1][1] = 0.0f; d[0][1][2] = 0.0f;
  d[1][0][0] = 0.0f; d[1][0][1] = 0.0f; d[1][0][2] = 0.0f;
  d[1][1][0] = 0.0f; d[1][1][1] = 0.0f; d[1][1][2] = -fy * iz2;
  d[2][0][0] = -fx * iz2; d[2][0][1] = 0.0f; d[2][0][2] = 2.0f * fx * x * iz2 / z;
  d[2][1][0] = 0.0f; d[2][1][1] = -fy * iz2; d[2][1][2] = 2.0f * fy * y * iz2 / z;
}

// cameras.hpp:249-268
__device__ __forceinline__ void panorama_jacobian_grad(const float p[3], const DevCamera& cam, float d[3][2][3]) {
  const float x = p[0], y = p[1], z = p[2];
  const float s = x * x + z * z;
  const float rho = sqrtf(s);
  const float r2 = s + y * y;
  const float cw = static_cast<float>(cam.width) / (2.0f * kPi);
  const float dh = static_cast<float>(cam.height) / kPi;
  const float is2 = 1.0f / (s * s);
  const float e = 1.0f / (rho * r2);
  const float f = (r2 + 2.0f * s) / (rho * s * r2 * r2);
  const float ey = 2.0f * y / (rho * r2 * r2);
  d[0][0][0] = -2.0f * cw * x * z * is2; d[0][0][1] = 0.0f; d[0][0][2] = cw * (x * x - z * z) * is2;
  d[0][1][0] = -dh * y * (e - x * x * f); d[0][1][1] = dh * x * (y * y - s) / (rho * r2 * r2); d[0][1][2] = dh * x * y * z * f;
  d[1][0][0] = 0.0f; d[1][0][1] = 0.0f; d[1][0][2] = 0.0f;
  d[1][1][0] = -dh * x * (e - y * ey); d[1][1][1] = -2.0f * dh * rho * y / (r2 * r2); d[1][1][2] = -dh * z * (e - y * ey);
  d[2][0][0] = cw * (x * x - z * z) * is2; d[2][0][1] = 0.0f; d[2][0][2] = 2.0f * cw * x * z * is2;
  d[2][1][0] = dh * x * y * z * f; d[2][1][1] = dh * z * (y * y - s) / (rho * r2 * r2); d[2][1][2] = -dh * y * (e - z * z * f);
}

// cameras.hpp:232-247
__device__ __forceinline__ void fisheye_jacobian_grad(const float p[3], const DevCamera& cam, const Terms& t,
                                                      float d[3][2][3]) {
  const float x = p[0], y = p[1], z = p[2];
  const float lz2 = x * x + y * y;
  const float r2 = lz2 + z * z;
  const float ir4 = 1.0f / (r2 * r2);
  const float fx = cam.fx, fy = cam.fy;
  const float x2 = x * x, y2 = y * y;
  const float ux = t.u + x2 * t.U;
  const float uy = t.u + y2 * t.U;
  d[0][0][0] = fx * x * (3.0f * t.u + x2 * t.U); d[0][0][1] = fx * y * ux; d[0][0][2] = fx * (2.0f * x2 - r2) * ir4;
  d[0][1][0] = fy * y * ux; d[0][1][1] = fy * x * uy; d[0][1][2] = 2.0f * fy * x * y * ir4;
  d[1][0][0] = fx * y * ux; d[1][0][1] = fx * x * uy; d[1][0][2] = 2.0f * fx * x * y * ir4;
  d[1][1][0] = fy * x * uy; d[1][1][1] = fy * y * (3.0f * t.u + y2 * t.U); d[1][1][2] = fy * (2.0f * y2 - r2) * ir4;
  d[2][0][0] = fx * (2.0f * x2 - r2) * ir4; d[2][0][1] = 2.0f * fx * x * y * ir4; d[2][0][2] = 2.0f * fx * x * z * ir4;
  d[2][1][0] = 2.0f * fy * x * y * ir4; d[2][1][1] = fy * (2.0f * y2 - r2) * ir4; d[2][1][2] = 2.0f * fy * y * z * ir4;
}

// cameras.hpp:76-79
__device__ __forceinline__ void world_to_camera(const DevCamera& cam, const float m[3], float mu[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r) mu[r] = cam.W[r * 3 + 0] * m[0] + cam.W[r * 3 + 1] * m[1] + cam.W[r * 3 + 2] * m[2] + cam.b[r];
}

// model.hpp:95-106; returns false for a zero-norm quaternion
__device__ __forceinline__ bool quat_to_rot(const float4 q, float r[3][3]) {
  const float n2 = q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w;
  if (!(n2 > 0.0f)) return false;
  const float n = sqrtf(n2);
  const float w = q.x / n, x = q.y / n, y = q.z / n, z = q.w / n;
  r[0][0] = 1.0f - 2.0f * (y * y + z * z); r[0][1] = 2.0f * (x * y - w * z); r[0][2] = 2.0f * (x * z + w * y);
  r[1][0] = 2.0f * (x * y + w * z); r[1][1] = 1.0f - 2.0f * (x * x + z * z); r[1][2] = 2.0f * (y * z - w * x);
  r[2][0] = 2.0f * (x * z - w * y); r[2][1] = 2.0f * (y * z + w * x); r[2][2] = 1.0f - 2.0f * (x * x + y * y);
  return true;
}

// model.hpp:127-140
__device__ __forceinline__ bool build_covariance(const float4 q, const float s[3], float sigma[3][3]) {
  float r[3][3];
  if (!quat_to_rot(q, r)) return false;
  const float sc[3] = {cr_expf_fast(s[0]), cr_expf_fast(s[1]), cr_expf_fast(s[2])};
  float m[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) m[i][j] = r[i][j] * sc[j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) {
      const float v = m[i][0] * m[j][0] + m[i][1] * m[j][1] + m[i][2] * m[j][2];
      sigma[i][j] = v;
      sigma[j][i] = v;
    }
  return true;
}

// core.hpp:30-36
// (one exp of -|x| serves both branches: the same two values, one evaluation per lane)
__device__ __forceinline__ float sigmoid(float x) {
  const float e = cr_expf_fast(-fabsf(x));
  return (x >= 0.0f ? 1.0f : e) / (1.0f + e);
}

// model.hpp:187-215 — SH basis factors Y[j] in the reference's association order.
__device__ __forceinline__ void sh_basis(const float d[3], int degree, float Y[16]) {
  const float x = d[0], y = d[1], z = d[2];
  Y[0] = float(kC0);
  if (degree >= 1) {
    Y[1] = -float(kC1) * y; Y[2] = float(kC1) * z; Y[3] = -float(kC1) * x;
  }
  if (degree >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    Y[4] = float(kC2_0) * xy; Y[5] = float(kC2_1) * yz; Y[6] = float(kC2_2) * (2.0f * zz - xx - yy);
    Y[7] = float(kC2_3) * xz; Y[8] = float(kC2_4) * (xx - yy);
    if (degree >= 3) {
      Y[9] = float(kC3_0) * y * (3.0f * xx - yy);
      Y[10] = float(kC3_1) * xy * z;
      Y[11] = float(kC3_2) * y * (4.0f * zz - xx - yy);
      Y[12] = float(kC3_3) * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
      Y[13] = float(kC3_4) * x * (4.0f * zz - xx - yy);
      Y[14] = float(kC3_5) * z * (xx - yy);
      Y[15] = float(kC3_6) * x * (xx - yy);
    }
  }
}

// Colour for one channel: reference grouping (C0*s0) + ((Y1 s1 + Y2 s2) - (C1 x) s3) + ...
// Y[3] = (-C1) x = -(C1 x) exactly, so "a - (C1 x) s3" == "a + Y3 s3" bit for bit.
__device__ __forceinline__ float sh_channel(const float* k, const float Y[16], int degree) {
  float v = Y[0] * k[0];
  if (degree >= 1) {
    const float t1 = Y[1] * k[1] + Y[2] * k[2] + Y[3] * k[3];
    v = v + t1;
    if (degree >= 2) {
      const float t2 = Y[4] * k[4] + Y[5] * k[5] + Y[6] * k[6] + Y[7] * k[7] + Y[8] * k[8];
      v = v + t2;
      if (degree >= 3) {
        const float t3 = Y[9] * k[9] + Y[10] * k[10] + Y[11] * k[11] + Y[12] * k[12] + Y[13] * k[13] +
                         Y[14] * k[14] + Y[15] * k[15];
        v = v + t3;
      }
    }
  }
  v = v + 0.5f;
  return fmaxf(v, 0.0f);
}

// d colour / d dir for one channel (SH view-direction path, build extension), accumulated
// into ddir: sum_j k_j * dY_j/d(x,y,z) * dcolour.
__device__ __forceinline__ void sh_dir_grad(const float d[3], int degree, const float* k, float dc, float ddir[3]) {
  const float x = d[0], y = d[1], z = d[2];
  const float c1 = float(kC1);
  float gx = -c1 * k[3], gy = -c1 * k[1], gz = c1 * k[2];
  if (degree >= 2) {
    const float a0 = float(kC2_0), a1 = float(kC2_1), a2 = float(kC2_2), a3 = float(kC2_3), a4 = float(kC2_4);
    gx += a0 * y * k[4] - 2.0f * a2 * x * k[6] + a3 * z * k[7] + 2.0f * a4 * x * k[8];
    gy += a0 * x * k[4] + a1 * z * k[5] - 2.0f * a2 * y * k[6] - 2.0f * a4 * y * k[8];
    gz += a1 * y * k[5] + 4.0f * a2 * z * k[6] + a3 * x * k[7];
    if (degree >= 3) {
      const float b0 = float(kC3_0), b1 = float(kC3_1), b2 = float(kC3_2), b3 = float(kC3_3), b4 = float(kC3_4),
                  b5 = float(kC3_5), b6 = float(kC3_6);
      const float xx = x * x, yy = y * y, zz = z * z;
      gx += 6.0f * b0 * x * y * k[9] + b1 * y * z * k[10] - 2.0f * b2 * x * y * k[11] - 6.0f * b3 * x * z * k[12] +
            b4 * (4.0f * zz - 3.0f * xx - yy) * k[13] + 2.0f * b5 * x * z * k[14] + b6 * (3.0f * xx - yy) * k[15];
      gy += b0 * (3.0f * xx - 3.0f * yy) * k[9] + b1 * x * z * k[10] + b2 * (4.0f * zz - xx - 3.0f * yy) * k[11] -
            6.0f * b3 * y * z * k[12] - 2.0f * b4 * x * y * k[13] - 2.0f * b5 * y * z * k[14] - 2.0f * b6 * x * y * k[15];
      gz += b1 * x * y * k[10] + 8.0f * b2 * y * z * k[11] + b3 * (6.0f * zz - 3.0f * xx - 3.0f * yy) * k[12] +
            8.0f * b4 * x * z * k[13] + b5 * (xx - yy) * k[14];
    }
  }
  ddir[0] += gx * dc;
  ddir[1] += gy * dc;
  ddir[2] += gz * dc;
}

// 16-byte load of p[0..3]: one LDG.128 when the array base is 16-byte aligned (vec), else four
// scalar loads (a caller's arrays may start anywhere, e.g. field blocks of a flat 59*N buffer).
__device__ __forceinline__ float4 ld4(const float* __restrict__ p, bool vec) {
  if (vec) return __ldg(reinterpret_cast<const float4*>(p));
  return make_float4(__ldg(p), __ldg(p + 1), __ldg(p + 2), __ldg(p + 3));
}

// The 16 coefficients of one colour channel, vectorised when the SH array is 16-byte aligned
// (channel rows are then 64-byte aligned).
__device__ __forceinline__ void load_sh16(const float* __restrict__ sh, int64_t g, int ch, int degree, bool vec,
                                          float k[16]) {
  const float* p = sh + g * 48 + 16 * ch;
  if (degree == 0) {
    k[0] = __ldg(p);
#pragma unroll
    for (int j = 1; j < 16; ++j) k[j] = 0.0f;
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 v = ld4(p + 4 * q, vec);
    k[4 * q + 0] = v.x; k[4 * q + 1] = v.y; k[4 * q + 2] = v.z; k[4 * q + 3] = v.w;
  }
}

// The 16 coefficients of one colour channel (only the SH view-direction gradient needs them).
__device__ __forceinline__ void load_sh_channel(const float* __restrict__ sh, int64_t g, int ch, int degree,
                                                float k[16]) {
  const float* p = sh + g * 48 + 16 * ch;
  const int nb = (degree + 1) * (degree + 1);
#pragma unroll
  for (int j = 0; j < 16; ++j) k[j] = j < nb ? __ldg(p + j) : 0.0f;
}

__device__ __forceinline__ void view_dir(const DevCamera& cam, const float m[3], float dir[3]) {
  const float v0 = m[0] - cam.center[0], v1 = m[1] - cam.center[1], v2 = m[2] - cam.center[2];
  const float n2 = v0 * v0 + v1 * v1 + v2 * v2;
  dir[0] = v0; dir[1] = v1; dir[2] = v2;
  if (n2 > 0.0f) {
    const float n = sqrtf(n2);
    dir[0] = v0 / n; dir[1] = v1 / n; dir[2] = v2 / n;
  }
}

__device__ __forceinline__ uint32_t depth_key_bits(float d) {
  const uint32_t u = __float_as_uint(d);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Projected covariance + conic for a visible Gaussian: returns 0 kept-candidate, 2 degenerate.
struct Proj {
  Terms ft;  // fisheye terms (g, u, U) at mu (fisheye camera only)
  float mu[3];
  float pix[2];
  float j[2][3];
  float t[2][3];
  float sigma[3][3];
  float sp[2][2];
  float det;
};

// splatting.hpp:83-97. Returns -1 invisible, 2 degenerate, 1 ok, 3 zero quaternion. prefetch: the
// Gaussian's SH row, requested into L1 as soon as the Gaussian is known to be in the field of
// view, so its load after the projection finds it there.
// The SH row is requested early only for Gaussians whose centre projects within this many pixels
// of the image (0: every Gaussian in the field of view). At config 2 about 40 % of the field of
// view falls outside the image rectangle; K1 0.0608 -> 0.0594 ms at a 32-pixel margin (8 / 64 / 128:
// within 0.5 % of it).
#ifndef FGS_K1_PF_MARGIN
#define FGS_K1_PF_MARGIN 32
#endif
__device__ __forceinline__ bool pix_near_image(const DevCamera& cam, const float pix[2]) {
  const float m = static_cast<float>(FGS_K1_PF_MARGIN);
  return pix[0] > -m && pix[0] < static_cast<float>(cam.width) + m && pix[1] > -m &&
         pix[1] < static_cast<float>(cam.height) + m;
}
__device__ __forceinline__ void prefetch_row(const float* p) {
  if (!p) return;
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 32));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 47));
}

__device__ __forceinline__ int project_covariance(const DevCamera& cam, const float m[3], const float4 q,
                                                  const float ls[3], Proj& P, const float* prefetch = nullptr) {
  world_to_camera(cam, m, P.mu);
  const float x = P.mu[0], y = P.mu[1], z = P.mu[2];
  const float r2 = x * x + y * y + z * z;
  if (r2 < 1e-24f) return -1;
  if (cam.model == kCamFisheye) {
    const float lz2 = x * x + y * y;
    if (z < 0.0f && lz2 < 1e-24f * z * z) return -1;
    const float theta = cr_atan2f_fast(sqrtf(lz2), z);
    if (!(theta <= cam.fov_max + kFisheyeCullMargin)) return -1;
#if FGS_K1_PF_MARGIN == 0
    prefetch_row(prefetch);
#endif
    P.ft = fisheye_terms(lz2, z, theta);
    const float g = P.ft.g;
    P.pix[0] = cam.cx + cam.fx * g * x;
    P.pix[1] = cam.cy + cam.fy * g * y;
#if FGS_K1_PF_MARGIN > 0
    // (a hint only: the row of a Gaussian whose centre projects far outside the image is not
    // requested early; if its footprint still reaches the image it is loaded when used)
    if (pix_near_image(cam, P.pix)) prefetch_row(prefetch);
#endif
    fisheye_jacobian(P.mu, cam, P.ft, P.j);
  } else if (cam.model == kCamPinhole) {
    if (fabsf(z) < 1e-12f) return -1;
    P.pix[0] = cam.cx + cam.fx * x / z;
    P.pix[1] = cam.cy + cam.fy * y / z;
    if (!(z > kPinholeNearClip)) return -1;
    if (FGS_K1_PF_MARGIN == 0 || pix_near_image(cam, P.pix)) prefetch_row(prefetch);
    pinhole_jacobian(P.mu, cam, P.j);
  } else {
    const float s = x * x + z * z;
    if (s < 1e-24f * y * y) return -1;
    const float w = static_cast<float>(cam.width), h = static_cast<float>(cam.height);
    float xp = w * (cr_atan2f_fast(x, z) + kPi) / (2.0f * kPi);
    if (xp >= w) xp -= w;
    P.pix[0] = xp;
    P.pix[1] = h * (cr_atan2f_fast(y, sqrtf(s)) + kPi / 2.0f) / kPi;
    prefetch_row(prefetch);
    panorama_jacobian(P.mu, cam, P.j);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) P.t[i][c] = P.j[i][0] * cam.W[0 * 3 + c] + P.j[i][1] * cam.W[1 * 3 + c] + P.j[i][2] * cam.W[2 * 3 + c];
  if (!build_covariance(q, ls, P.sigma)) return 3;
  float ts[2][3];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) ts[i][c] = P.t[i][0] * P.sigma[0][c] + P.t[i][1] * P.sigma[1][c] + P.t[i][2] * P.sigma[2][c];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int c = 0; c < 2; ++c) P.sp[i][c] = ts[i][0] * P.t[c][0] + ts[i][1] * P.t[c][1] + ts[i][2] * P.t[c][2];
  P.sp[0][0] += kCovarianceDilation;
  P.sp[1][1] += kCovarianceDilation;
  P.det = P.sp[0][0] * P.sp[1][1] - P.sp[0][1] * P.sp[1][0];
  if (!(P.det > 0.0f)) return 2;
  return 1;
}

}  // namespace

// Host-scene SH rows: float4s of one colour channel row that the degree evaluates (the
// device path loads all four).
__device__ __forceinline__ int sh_row_f4(int degree) { return degree == 1 ? 1 : (degree == 2 ? 3 : 4); }
constexpr int kStageRow = 13;  // float4 per staged row: 12 + 1 pad (conflict-free LDS.128)
// dynamic shared memory of preprocess_kernel<true>
static size_t preprocess_host_smem() { return sizeof(float4) * 8 * 32 * kStageRow; }

// Warp-collective (host scene): the SH rows of the warp's lanes with `need` set, read over PCIe
// as contiguous runs by the whole warp (a lane reading its own 192-byte row issues 16-byte
// pieces 192 bytes apart, which PCIe serves at a third of the rate) into stage[lane][...].
__device__ __forceinline__ void stage_sh_rows(const float* __restrict__ sh, int64_t warp_g0, bool need, int degree,
                                              bool vec, float4* stage) {
  const int lane = threadIdx.x & 31;
  const unsigned mask = __ballot_sync(0xffffffffu, need);
  const int nq = sh_row_f4(degree), per_row = 3 * nq;
  const int total = __popc(mask) * per_row;
  for (int it = lane; it < total; it += 32) {
    const int r = it / per_row, t = it - r * per_row;
    const int src_lane = __fns(mask, 0, r + 1);  // the r-th needing lane
    const int ch = t / nq, q = t - ch * nq;
    const float* row = sh + (warp_g0 + src_lane) * 48;
    stage[src_lane * kStageRow + ch * 4 + q] = ld4(row + 4 * (ch * 4 + q), vec);
  }
  __syncwarp();
}

// K1 body for one Gaussian (every lane of the warp calls it: the host-scene variant has
// warp-collective loads). m / ls: the mean and log-scales, read by the caller.
template <bool HOST_SCENE>
__device__ __forceinline__ void preprocess_one(const PreprocessArgs& a, int64_t i, bool valid, const float m[3],
                                               const float ls[3], unsigned* s_counts, float4* stage) {
  const DevCamera& cam = a.cam;
  const float4 q = valid ? ld4(a.rotations + 4 * i, a.vec_rot) : make_float4(1.f, 0.f, 0.f, 0.f);
  // host scene: every lane reads its opacity (one coalesced 128-byte run per warp over PCIe
  // instead of scattered 4-byte reads by the kept lanes)
  const float op = valid ? __ldg(a.opacity + i) : 0.0f;  // issued early (coalesced; the host scene reads
                                                        // it as one 128-byte run per warp over PCIe)

  uint8_t state = 0;
  uint32_t key = 0xFFFFFFFFu, touched = 0;
  int radius = 0;
  ushort4 rect = make_ushort4(1, 0, 1, 0);
  float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
  float r2v = 0.f;

  Proj P;
  const int pc = valid ? project_covariance(cam, m, q, ls, P, (!HOST_SCENE && a.sh_degree > 0) ? a.sh + 48 * i : nullptr)
                       : -1;
  bool keep = false;
  float mx = 0.f, my = 0.f, rf = 0.f;
  if (pc == 3) {
    *a.error_flag = 1;
  } else if (pc == 2) {
    state = 2;
  } else if (pc == 1) {
    const float det = P.det;
    const float mid = (P.sp[0][0] + P.sp[1][1]) / 2.0f;
    const float lambda_max = mid + sqrtf(fmaxf(mid * mid - det, 0.0f));
    radius = static_cast<int>(ceilf(kRadiusSigma * sqrtf(lambda_max)));
    mx = P.pix[0], my = P.pix[1], rf = static_cast<float>(radius);
    keep = !(mx + rf < 0.0f || mx - rf > static_cast<float>(cam.width) || my + rf < 0.0f ||
             my - rf > static_cast<float>(cam.height));
  }
  if constexpr (HOST_SCENE) {
    if (a.sh_degree > 0) stage_sh_rows(a.sh, i - (threadIdx.x & 31), keep, a.sh_degree, a.vec_sh, stage);
  }
  if (keep) {
    state = 1;
    const float det = P.det;
    const float ca = P.sp[1][1] / det, cb = -P.sp[0][1] / det, cc = P.sp[0][0] / det;
    // splatting.hpp:114: z for the pinhole, the distance for fisheye / panorama
    const float depth = cam.model == kCamPinhole ? P.mu[2]
                                                 : sqrtf(P.mu[0] * P.mu[0] + P.mu[1] * P.mu[1] + P.mu[2] * P.mu[2]);
    float dir[3];
    view_dir(cam, m, dir);
    float Y[16];
    sh_basis(dir, a.sh_degree, Y);
    // one colour channel at a time (16 live coefficients instead of 48)
    float col[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float k[16];
      if (HOST_SCENE && a.sh_degree > 0) {
        const int nq = sh_row_f4(a.sh_degree);
        const float4* st = stage + (threadIdx.x & 31) * kStageRow + ch * 4;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const float4 v = qq < nq ? st[qq] : make_float4(0.f, 0.f, 0.f, 0.f);
          k[4 * qq + 0] = v.x; k[4 * qq + 1] = v.y; k[4 * qq + 2] = v.z; k[4 * qq + 3] = v.w;
        }
      } else {
        load_sh16(a.sh, i, ch, a.sh_degree, a.vec_sh, k);
      }
      col[ch] = sh_channel(k, Y, a.sh_degree);
    }
    const float col0 = col[0], col1 = col[1], col2 = col[2];
    const float alpha = sigmoid(op);
    r0 = make_float4(mx, my, ca, cb);
    r1 = make_float4(cc, alpha, col0, col1);
    r2v = col2;
    key = depth_key_bits(depth);
    // splatting.hpp:211-214 — inclusive, floor, clamped
    const int tx0 = max(0, static_cast<int>(floorf((mx - rf) / 16.0f)));
    const int tx1 = min(a.tiles_x - 1, static_cast<int>(floorf((mx + rf) / 16.0f)));
    const int ty0 = max(0, static_cast<int>(floorf((my - rf) / 16.0f)));
    const int ty1 = min(a.tiles_y - 1, static_cast<int>(floorf((my + rf) / 16.0f)));
    if (tx1 >= tx0 && ty1 >= ty0) {
      touched = static_cast<uint32_t>((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
      rect = make_ushort4(tx0, tx1, ty0, ty1);
      // per-tile counts for K2: +1 / -1 at both ends of every covered row
      const int rw = a.tiles_x + 1;
      for (int ty = ty0; ty <= ty1; ++ty) {
        atomicAdd(a.rowdiff + ty * rw + tx0, 1);
        atomicAdd(a.rowdiff + ty * rw + tx1 + 1, -1);
      }
    }
  }
  if (!valid) return;
  SortedRec rr;
  const float3 cull = splat_cull_params(r0, r1);
  // the record keeps -a/2 and -c/2 (exact power-of-two scalings): the blends' power is then
  // (a' dx) dx + (c' dy) dy - (b dx) dy, one multiplication less per (pixel, splat) pair, with
  // the reference's value bit for bit (SortedRec, fgs_common.cuh)
  rr.a = make_float4(r0.x, r0.y, -0.5f * r0.z, r0.w);
  rr.b = make_float4(-0.5f * r1.x, r1.y, r1.z, r1.w);
  rr.c = make_float4(r2v, cull.x, cull.y, cull.z);
  a.rec[i] = rr;
  a.state[i] = state;
  a.depth_key[i] = key;
  a.touched[i] = touched;
  a.rect[i] = rect;
  a.radii[i] = state == 1 ? radius : 0;
  if (state == 1) atomicAdd(s_counts, 1u);
  if (state == 2) atomicAdd(s_counts + 1, 1u);
}


// K1: one thread per Gaussian.
// HOST_SCENE: the scene arrays are pinned host memory read in place over PCIe (the host-buffer
// calls). Reads are then shaped for PCIe: the CTA's means and log-scales (3 KB runs each) are
// copied through shared memory with 16-byte loads, and SH rows are fetched warp-cooperatively.
template <bool HOST_SCENE>
#ifndef FGS_K1_MINB
#define FGS_K1_MINB 4
#endif
__global__ void __launch_bounds__(256, FGS_K1_MINB) preprocess_kernel(PreprocessArgs a) {
  __shared__ unsigned s_counts[2];
  const int64_t i0 = int64_t(blockIdx.x) * blockDim.x;
  const int64_t i = i0 + threadIdx.x;
  const bool valid = i < a.n;
  float m[3] = {0.f, 0.f, 0.f}, ls[3] = {0.f, 0.f, 0.f};
  float4* stage = nullptr;
  if constexpr (HOST_SCENE) {
    __shared__ float4 s_geo[2][192];                       // means, log-scales of 256 Gaussians
    extern __shared__ float4 s_stage[];                   // SH rows: [8 warps][32][kStageRow]
    const int64_t nrem = a.n - i0;
    const int nf = static_cast<int>((nrem < 256 ? nrem : 256) * 3);  // floats of this CTA
    const float* src[2] = {a.means + i0 * 3, a.log_scales + i0 * 3};
    // 3 * 256 floats per array; i0 * 3 * 4 bytes is a multiple of 16 (i0 is a multiple of 256)
    for (int t = threadIdx.x; t < 2 * 192; t += blockDim.x) {
      const int arr = t / 192, j = t - arr * 192;
      if (4 * j + 3 < nf) s_geo[arr][j] = ld4(src[arr] + 4 * j, a.vec_geo);
      else {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        for (int e = 0; e < 4; ++e) if (4 * j + e < nf) v[e] = __ldg(src[arr] + 4 * j + e);
        s_geo[arr][j] = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
    if (threadIdx.x < 2) s_counts[threadIdx.x] = 0;
    crm::stage_tables();
    __syncthreads();
    const float* gm = reinterpret_cast<const float*>(s_geo[0]);
    const float* gl = reinterpret_cast<const float*>(s_geo[1]);
    for (int c = 0; c < 3; ++c) {
      m[c] = gm[3 * threadIdx.x + c];
      ls[c] = gl[3 * threadIdx.x + c];
    }
    stage = s_stage + (threadIdx.x >> 5) * (32 * kStageRow);
  } else {
    if (threadIdx.x < 2) s_counts[threadIdx.x] = 0;
    crm::stage_tables();
    __syncthreads();
    if (valid) {
      for (int c = 0; c < 3; ++c) {
        m[c] = __ldg(a.means + 3 * i + c);
        ls[c] = __ldg(a.log_scales + 3 * i + c);
      }
    }
  }
  preprocess_one<HOST_SCENE>(a, i, valid, m, ls, s_counts, stage);
  __syncthreads();
  if (threadIdx.x < 2 && s_counts[threadIdx.x]) atomicAdd(a.state_counts + threadIdx.x, s_counts[threadIdx.x]);
}

// K4b per-Gaussian chain rule for Gaussian i with its summed screen-space values sg[9] (power
// moments 5, colour 3, sum of dpower; K4a); writes (or adds) its 59 gradient values.
// shstage: this lane's 20-float slot -- the SH gradient rows are Y (x) dcolour, so the lane leaves
// Y[16] (band-masked), dcolour[3] (clamp-masked) and i there and the warp writes the rows as
// contiguous 192-byte runs afterwards (sh_rows_store).
__device__ __forceinline__ void gaussian_backward(const PreprocessBackwardArgs& a, int64_t i, const float sg[9],
                                                  float* shstage) {
  float out[11];  // mean 3, rotation 4, log-scale 3, opacity 1 (SH rows are stored as computed)
#pragma unroll
  for (int k = 0; k < 11; ++k) out[k] = 0.0f;
  {
    const DevCamera& cam = a.cam;
    const float m[3] = {__ldg(a.means + 3 * i), __ldg(a.means + 3 * i + 1), __ldg(a.means + 3 * i + 2)};
    const float4 q = ld4(a.rotations + 4 * i, a.vec_rot);
    const float ls[3] = {__ldg(a.log_scales + 3 * i), __ldg(a.log_scales + 3 * i + 1), __ldg(a.log_scales + 3 * i + 2)};
    Proj P;
    project_covariance(cam, m, q, ls, P);
    const float det = P.det;
    const float conic[3] = {P.sp[1][1] / det, -P.sp[0][1] / det, P.sp[0][0] / det};
    // sg[0..4]: the summed moments M = sum dpower-gradient x (dx, dy, dx^2, dx dy, dy^2) over the
    // Gaussian's pixels (K4a); dL/dmean_px = (a M0 + b M1, b M0 + c M1) and dL/dconic =
    // -(M2 / 2, M3, M4 / 2) (gradients.hpp:153-156 per pixel, summed with the conic factored out)
    const float dmx = conic[0] * sg[0] + conic[1] * sg[1], dmy = conic[1] * sg[0] + conic[2] * sg[1];
    // mean_backward (gradients.hpp:177-181): J^T dmean_px
    float direct[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) direct[k] = P.j[0][k] * dmx + P.j[1][k] * dmy;
    // gradients.hpp:239-243: dSigma_p = (-Q) Gq Q, b-slot cotangent halved
    const float nq[2][2] = {{-conic[0], -conic[1]}, {-conic[1], -conic[2]}};
    const float Q[2][2] = {{conic[0], conic[1]}, {conic[1], conic[2]}};
    const float h3 = -0.5f * sg[3];
    const float gq[2][2] = {{-0.5f * sg[2], h3}, {h3, -0.5f * sg[4]}};
    float tmp[2][2], dsp[2][2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) tmp[r][c] = nq[r][0] * gq[0][c] + nq[r][1] * gq[1][c];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) dsp[r][c] = tmp[r][0] * Q[0][c] + tmp[r][1] * Q[1][c];
    // covariance_projection_backward (gradients.hpp:186-202)
    float a32[3][2], dsig[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) a32[r][c] = P.t[0][r] * dsp[0][c] + P.t[1][r] * dsp[1][c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) dsig[r][c] = a32[r][0] * P.t[0][c] + a32[r][1] * P.t[1][c];
    const float gs[2][2] = {{dsp[0][0] + dsp[0][0], dsp[0][1] + dsp[1][0]}, {dsp[1][0] + dsp[0][1], dsp[1][1] + dsp[1][1]}};
    float b23[2][3], dldt[2][3], dldj[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) b23[r][c] = gs[r][0] * P.t[0][c] + gs[r][1] * P.t[1][c];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) dldt[r][c] = b23[r][0] * P.sigma[0][c] + b23[r][1] * P.sigma[1][c] + b23[r][2] * P.sigma[2][c];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) dldj[r][c] = dldt[r][0] * cam.W[c * 3 + 0] + dldt[r][1] * cam.W[c * 3 + 1] + dldt[r][2] * cam.W[c * 3 + 2];
    float dj[3][2][3];
    if (cam.model == kCamFisheye) fisheye_jacobian_grad(P.mu, cam, P.ft, dj);
    else if (cam.model == kCamPinhole) pinhole_jacobian_grad(P.mu, cam, dj);
    else panorama_jacobian_grad(P.mu, cam, dj);
    float cov[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      // cwiseProduct().sum() in column-major storage order
      const float s = dldj[0][0] * dj[k][0][0] + dldj[1][0] * dj[k][1][0] + dldj[0][1] * dj[k][0][1] +
                      dldj[1][1] * dj[k][1][1] + dldj[0][2] * dj[k][0][2] + dldj[1][2] * dj[k][1][2];
      cov[k] = a.jac_grad_scale[k] * s;
    }
    // build_covariance_backward (model.hpp:144-171)
    {
      const float n2 = q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w;
      const float n = sqrtf(n2);
      const float qn[4] = {q.x / n, q.y / n, q.z / n, q.w / n};
      float r[3][3];
      quat_to_rot(q, r);
      const float sc[3] = {cr_expf_fast(ls[0]), cr_expf_fast(ls[1]), cr_expf_fast(ls[2])};
      float mm[3][3];
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int v = 0; v < 3; ++v) mm[u][v] = r[u][v] * sc[v];
      float gsym[3][3];
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int v = 0; v < 3; ++v) gsym[u][v] = dsig[u][v] + dsig[v][u];
      float dm[3][3];
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int v = 0; v < 3; ++v) dm[u][v] = gsym[u][0] * mm[0][v] + gsym[u][1] * mm[1][v] + gsym[u][2] * mm[2][v];
      float dr[3][3];
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int v = 0; v < 3; ++v) dr[u][v] = dm[u][v] * sc[v];
#pragma unroll
      for (int u = 0; u < 3; ++u) out[7 + u] = sc[u] * (r[0][u] * dm[0][u] + r[1][u] * dm[1][u] + r[2][u] * dm[2][u]);
      const float w = qn[0], x = qn[1], y = qn[2], z = qn[3];
      // rotation_quaternion_partials (model.hpp:111-121), each entry * 2; the sum runs over
      // the 3x3 product in column-major order (cwiseProduct().sum()).
      auto colsum = [&](float p00, float p01, float p02, float p10, float p11, float p12, float p20, float p21,
                        float p22) {
        float acc = dr[0][0] * (p00 * 2.0f);
        acc = acc + dr[1][0] * (p10 * 2.0f);
        acc = acc + dr[2][0] * (p20 * 2.0f);
        acc = acc + dr[0][1] * (p01 * 2.0f);
        acc = acc + dr[1][1] * (p11 * 2.0f);
        acc = acc + dr[2][1] * (p21 * 2.0f);
        acc = acc + dr[0][2] * (p02 * 2.0f);
        acc = acc + dr[1][2] * (p12 * 2.0f);
        acc = acc + dr[2][2] * (p22 * 2.0f);
        return acc;
      };
      float dqn[4];
      dqn[0] = colsum(0.0f, -z, y, z, 0.0f, -x, -y, x, 0.0f);
      dqn[1] = colsum(0.0f, y, z, y, -2.0f * x, -w, z, w, -2.0f * x);
      dqn[2] = colsum(-2.0f * y, x, w, x, 0.0f, z, -w, z, -2.0f * y);
      dqn[3] = colsum(-2.0f * z, -w, x, w, -2.0f * z, y, x, y, 0.0f);
      const float dot = qn[0] * dqn[0] + qn[1] * dqn[1] + qn[2] * dqn[2] + qn[3] * dqn[3];
#pragma unroll
      for (int kq = 0; kq < 4; ++kq) out[3 + kq] = (dqn[kq] - qn[kq] * dot) / n;
    }
    // gradients.hpp:251-252
    const float v[3] = {direct[0] + cov[0], direct[1] + cov[1], direct[2] + cov[2]};
#pragma unroll
    for (int r = 0; r < 3; ++r) out[r] = cam.W[0 * 3 + r] * v[0] + cam.W[1 * 3 + r] * v[1] + cam.W[2 * 3 + r] * v[2];
    // K1's record holds sigmoid(opacity) and the clamped colours, computed by the same code
    // in this translation unit: bit-identical to recomputing them, without the SH reads.
    const float4 rb = a.rec[i].b;
    const float colour[3] = {rb.z, rb.w, a.rec[i].c.x};
    const float al = rb.y;
    // sg[8] = sum dp = al * dL/dal (K4a), so dL/dlogit = dL/dal * al (1 - al) = sg[8] (1 - al)
    out[10] = sg[8] * (1.0f - al);
    // SH: eval_sh_dc_backward (model.hpp:219-227) + higher bands (build extension)
    float dir[3];
    view_dir(cam, m, dir);
    float Y[16];
    sh_basis(dir, a.sh_degree, Y);
    const int nb = a.full_sh ? (a.sh_degree + 1) * (a.sh_degree + 1) : 1;
    float ddir[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int jb = 0; jb < 16; ++jb) shstage[jb] = jb < nb ? (jb == 0 ? float(kC0) : Y[jb]) : 0.0f;
    shstage[19] = __int_as_float(static_cast<int>(i));
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const bool live = colour[ch] > 0.0f;  // clamped channel: no gradient
      const float dc = sg[5 + ch];
      shstage[16 + ch] = live ? dc : 0.0f;
      if (live && a.view_dir && a.sh_degree > 0) {
        float k[16];
        load_sh_channel(a.sh, i, ch, a.sh_degree, k);
        sh_dir_grad(dir, a.sh_degree, k, dc, ddir);
      }
    }
    if (a.view_dir && a.sh_degree > 0) {
      // colour -> view direction -> mean (not in the reference; opt-in)
      const float v0 = m[0] - cam.center[0], v1 = m[1] - cam.center[1], v2 = m[2] - cam.center[2];
      const float nrm = sqrtf(v0 * v0 + v1 * v1 + v2 * v2);
      if (nrm > 0.0f) {
        const float dd = dir[0] * ddir[0] + dir[1] * ddir[1] + dir[2] * ddir[2];
#pragma unroll
        for (int q2 = 0; q2 < 3; ++q2) out[q2] += (ddir[q2] - dir[q2] * dd) / nrm;
      }
    }
  }
  // write (field-major arrays)
  float* dm = a.d_means + 3 * i;
  float* drt = a.d_rotations + 4 * i;
  float* dls = a.d_log_scales + 3 * i;
  if (a.accumulate) {
#pragma unroll
    for (int k = 0; k < 3; ++k) dm[k] += out[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) drt[k] += out[3 + k];
#pragma unroll
    for (int k = 0; k < 3; ++k) dls[k] += out[7 + k];
    a.d_opacity[i] += out[10];
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) dm[k] = out[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) dls[k] = out[7 + k];
    a.d_opacity[i] = out[10];
    if (a.aligned16) {
      reinterpret_cast<float4*>(drt)[0] = make_float4(out[3], out[4], out[5], out[6]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) drt[k] = out[3 + k];
    }
  }
}

// K4b: one thread per Gaussian that touched a tile, taken in source order from the K2
// compaction list (cval), 128 per CTA. K4a left one 9-float gradient sum per intersection at
// its emission slot; the Gaussian's slots [coff[q], +touched[g]) are contiguous in ascending
// tile order and are summed here in that order:
// deterministic, no atomics (gradients.hpp:161-173). Gaussians that touched no tile have zero
// gradient; CTA b also zero-fills (after its own Gaussians), with coalesced stores, the non-touching rows between its
// predecessor's last Gaussian and its own last one -- so every sector of that source range
// is written by one CTA in a short window and L2 merges the partial-sector writes.
// One intersection's screen-space gradient (the blend backward's per-intersection sum at its
// emission slot) added into acc.
__device__ __forceinline__ void intersection_sum(const PreprocessBackwardArgs& a, uint32_t e, float* acc) {
  FGS_DCHECK(static_cast<int64_t>(e) < a.num_isect);
  const float* p = a.partials + static_cast<size_t>(e) * 9;
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = acc[q] + p[q];
}

// Slots [e, end) in order: the first ones singly up to a 4-entry boundary, then 4 entries (36
// floats) per step as 9 independent 16-byte loads -- all in flight before the adds, which keep
// the sequential order.
__device__ __forceinline__ void intersection_sums(const PreprocessBackwardArgs& a, uint32_t e, uint32_t end,
                                                  float* acc) {
#ifdef FGS_K4B_NO_UNROLL
  for (; e < end; ++e) intersection_sum(a, e, acc);
#endif
  for (; e < end && (e & 3u); ++e) intersection_sum(a, e, acc);
  for (; e + 4 <= end; e += 4) {
    FGS_DCHECK(static_cast<int64_t>(e) + 4 <= a.num_isect);
    const float4* p4 = reinterpret_cast<const float4*>(a.partials + static_cast<size_t>(e) * 9);
    float p[36];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const float4 v = __ldg(p4 + k);
      p[4 * k] = v.x;
      p[4 * k + 1] = v.y;
      p[4 * k + 2] = v.z;
      p[4 * k + 3] = v.w;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < 9; ++q) acc[q] = acc[q] + p[9 * u + q];
  }
  for (; e < end; ++e) intersection_sum(a, e, acc);
}

constexpr int kBwdThreads = kPreprocessBackwardThreads;

// The warp's SH gradient rows (one per lane with `has`), from the lanes' slots: row r's float4 c
// is Y[4 (c % 4) ..] * dcolour[c / 4]; 12 lanes cover a row with contiguous 16-byte accesses
// (a lane writing its own row issues 16-byte pieces 192 bytes apart). The products are the
// same single-rounded multiplications as per lane.
__device__ __forceinline__ void sh_rows_store(const PreprocessBackwardArgs& a, const float* stage, bool has) {
  const int lane = threadIdx.x & 31;
  const unsigned mask = __ballot_sync(0xffffffffu, has);
  const int total = __popc(mask) * 12;
  __syncwarp();
  for (int it = lane; it < total; it += 32) {
    const int r = it / 12, c = it - 12 * r;
    const int src = __fns(mask, 0, r + 1);
    const float* st = stage + src * 20;
    const int64_t i = __float_as_int(st[19]);
    const float dc = st[16 + c / 4];
    const float4 y = *reinterpret_cast<const float4*>(st + 4 * (c & 3));
    // (+ 0.0f: masked entries are +0 whatever the signs of the factors)
    const float4 g = make_float4(y.x * dc + 0.0f, y.y * dc + 0.0f, y.z * dc + 0.0f, y.w * dc + 0.0f);
    float* d = a.d_sh + 48 * i + 4 * c;
    if (a.accumulate) {
      d[0] += g.x; d[1] += g.y; d[2] += g.z; d[3] += g.w;
    } else if (a.aligned16) {
      *reinterpret_cast<float4*>(d) = g;
    } else {
      d[0] = g.x; d[1] = g.y; d[2] = g.z; d[3] = g.w;
    }
  }
}
// MINB: the register fit (6 CTAs per SM: 80 registers with a few spills; 4: 85, none) -- same
// code and results, scene-dependent speed (config 2 0.107 vs 0.099 ms, config 4 0.289 vs
// 0.305): the caller times both per context.
template <bool HOST_SCENE, int MINB>
__global__ void __launch_bounds__(kBwdThreads, MINB) preprocess_backward_kernel(PreprocessBackwardArgs a) {
#ifdef FGS_K4B_OLD_ZERO
  constexpr int kZeroRows = kBwdThreads;
#else
  constexpr int kZeroRows = 8 * kBwdThreads;  // rows per zero-fill round (one load of their tile counts)
#endif
  constexpr int kZR = kZeroRows / kBwdThreads;
  __shared__ uint8_t vis[kZeroRows];
  __shared__ __align__(16) float s_shstage[kBwdThreads * 20];  // per-lane SH gradient factors
  const int tid = threadIdx.x, lane = tid & 31;
  pdl_wait();  // (a programmatic dependent of K4a)
#ifdef FGS_FAST_CRMATH
  crm::stage_tables();
  __syncthreads();
#endif
  const int64_t q0 = a.q_begin + int64_t(blockIdx.x) * kBwdThreads;
  const int64_t q1 = q0 + kBwdThreads < a.q_end ? q0 + kBwdThreads : a.q_end;  // this CTA's slice of cval
  // the chain rule first (its dependent loads start at once), the zero rows after it (zero rows
  // first: config 2 K4b 0.0925 -> 0.0896 ms, config 1 0.0323 -> 0.0288)
  if (q0 + (tid & ~31) < q1) {
  const bool valid = q0 + tid < q1;
  {
    const int64_t i = a.cval[valid ? q0 + tid : q0];
    // Gaussians with more than 32 tiles are summed by the whole warp (lane-strided, fixed
    // shuffle tree): deterministic, and no lane walks thousands of tiles alone.
    float sg[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) sg[k] = 0.0f;
    const uint32_t cnt = valid ? a.touched[i] : 0u;
    const uint32_t base = valid ? a.coff[q0 + tid] : 0u;
    const bool big = cnt > 32;
    if (!big) intersection_sums(a, base, base + cnt, sg);
    uint32_t bigs = __ballot_sync(0xffffffffu, big);
    while (bigs) {
      const int jl = __ffs(bigs) - 1;
      bigs &= bigs - 1;
      const uint32_t bj = __shfl_sync(0xffffffffu, base, jl), cj = __shfl_sync(0xffffffffu, cnt, jl);
      float acc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = 0.0f;
      for (uint32_t e = bj + lane; e < bj + cj; e += 32) intersection_sum(a, e, acc);
#pragma unroll
      for (int k = 0; k < 9; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[k] = acc[k] + __shfl_xor_sync(0xffffffffu, acc[k], o);
        if (lane == jl) sg[k] = acc[k];
      }
    }
    float* slot = s_shstage + tid * 20;
    if (valid) gaussian_backward(a, i, sg, slot);
    sh_rows_store(a, s_shstage + (tid & ~31) * 20, valid);
  }
  }
  if (!a.accumulate) {
    // rows of this CTA's id span: from its predecessor's last Gaussian (or the launch's first id)
    const int64_t start = q0 <= a.q_begin ? a.id_begin : int64_t(a.cval[q0 - 1]) + 1;
    const int64_t end = q1 >= a.q_end ? a.id_end : int64_t(a.cval[q1 - 1]) + 1;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t c0 = start; c0 < end; c0 += kZeroRows) {  // 1024-row rounds (a CTA spans ~N / CTAs rows)
      const int nloc = static_cast<int>(end - c0 < kZeroRows ? end - c0 : kZeroRows);
      __syncthreads();
      uint8_t v8[kZR];
#pragma unroll
      for (int k = 0; k < kZR; ++k) {  // 8 independent loads in flight
        const int r = tid + k * kBwdThreads;
        v8[k] = r < nloc && __ldg(a.touched + c0 + r) > 0u;
      }
#pragma unroll
      for (int k = 0; k < kZR; ++k) vis[tid + k * kBwdThreads] = v8[k];
      __syncthreads();
      if (a.aligned16) {
        float4* sh4 = reinterpret_cast<float4*>(a.d_sh + 48 * c0);
        for (int f = tid; f < nloc * 12; f += kBwdThreads)
          if (!vis[f / 12]) sh4[f] = z;
        for (int r = tid; r < nloc; r += kBwdThreads)
          if (!vis[r]) reinterpret_cast<float4*>(a.d_rotations + 4 * c0)[r] = z;
      } else {
        for (int f = tid; f < nloc * 48; f += kBwdThreads)
          if (!vis[f / 48]) a.d_sh[48 * c0 + f] = 0.f;
        for (int f = tid; f < nloc * 4; f += kBwdThreads)
          if (!vis[f / 4]) a.d_rotations[4 * c0 + f] = 0.f;
      }
      for (int r = tid; r < nloc; r += kBwdThreads)
        if (!vis[r]) a.d_opacity[c0 + r] = 0.f;
      for (int f = tid; f < nloc * 3; f += kBwdThreads)
        if (!vis[f / 3]) {
          a.d_means[3 * c0 + f] = 0.f;
          a.d_log_scales[3 * c0 + f] = 0.f;
        }
    }
  }
}

// Self-test of fgs_crmath.cuh against the definitions: which 0 = exp over the fp32 bit patterns
// [begin, begin + count); 1 = atan2 over `count` seeded pairs of random bit patterns; 2 = over
// seeded pairs of the fisheye / panorama domain (magnitudes 2^-30..2^30, both signs of x, ratios
// near 1 and near j/16 boundaries). out: [checked, mismatches, slow-path evaluations].
namespace {
__device__ __forceinline__ uint32_t mix32(uint64_t v) {
  v ^= v >> 33;
  v *= 0xff51afd7ed558ccdull;
  v ^= v >> 33;
  v *= 0xc4ceb9fe1a85ec53ull;
  v ^= v >> 33;
  return static_cast<uint32_t>(v);
}
__device__ __forceinline__ bool same_bits(float a, float b) {
  return __float_as_uint(a) == __float_as_uint(b) || (a != a && b != b);
}
__global__ void crmath_selftest_kernel(int which, uint64_t begin, uint64_t count, uint64_t seed,
                                       unsigned long long* out) {
  for (int t = threadIdx.x; t < 64 + 17; t += blockDim.x) crm::s_tab[t] = t < 64 ? crm::kExp2J[t] : crm::kAtanJ[t - 64];
  __syncthreads();
  unsigned long long bad = 0, slow = 0, n = 0;
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < count; k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t idx = begin + k;
    bool ok;
    if (which == 0) {
      const float x = __uint_as_float(static_cast<uint32_t>(idx));
      crm::exp_fast_path(x, &ok);
      bad += !same_bits(cr_expf_fastpath(x), cr_expf(x));
      slow += !ok;
    } else {
      const uint32_t h1 = mix32(idx * 2 + seed * 0x9E3779B97F4A7C15ull), h2 = mix32(idx * 2 + 1 + seed * 0x9E3779B97F4A7C15ull);
      float y, x;
      if (which == 1) {
        y = __uint_as_float(h1);
        x = __uint_as_float(h2);
      } else {
        const float m1 = 1.0f + (h1 & 0x7FFFFF) * 0x1p-23f, m2 = 1.0f + (h2 & 0x7FFFFF) * 0x1p-23f;
        y = ldexpf(m1, static_cast<int>((h1 >> 23) % 61) - 30);
        x = ldexpf(m2, static_cast<int>((h2 >> 23) % 61) - 30);
        const uint32_t mode = (h1 ^ h2) >> 29;
        if (mode == 1) x = y * (1.0f + static_cast<float>(static_cast<int>(h2 % 64) - 32) * 0x1p-23f);  // ratio ~1
        if (mode == 2) y = x * ((h2 % 17) / 16.0f + static_cast<float>(static_cast<int>(h1 % 64) - 32) * 0x1p-22f);  // ~j/16
        if (h2 & 1u) x = -x;
        if (mode == 3 && (h1 & 2u)) y = -y;
      }
      crm::atan2_fast_path(y, x, &ok);
      bad += !same_bits(cr_atan2f_fastpath(y, x), cr_atan2f(y, x));
      slow += !ok;
    }
    ++n;
  }
  for (int o = 16; o > 0; o >>= 1) {
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    slow += __shfl_xor_sync(0xffffffffu, slow, o);
    n += __shfl_xor_sync(0xffffffffu, n, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out + 0, n);
    atomicAdd(out + 1, bad);
    atomicAdd(out + 2, slow);
  }
}
}  // namespace

void crmath_selftest(int which, uint64_t begin, uint64_t count, uint64_t seed, unsigned long long* out_dev,
                     cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  crmath_selftest_kernel<<<sms * 8, 256, 0, st>>>(which, begin, count, seed, out_dev);
}

void preprocess_launch(const PreprocessArgs& a, bool host_scene, cudaStream_t st) {
  const int blocks = div_up(static_cast<int>(a.n), 256);
  if (host_scene) {
    static PerDevice attr;
    attr.get([] {
      cudaFuncSetAttribute(preprocess_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(preprocess_host_smem()));
      return 1;
    });
    preprocess_kernel<true><<<blocks, 256, preprocess_host_smem(), st>>>(a);
  } else {
    preprocess_kernel<false><<<blocks, 256, 0, st>>>(a);
  }
}

void preprocess_backward_launch(const PreprocessBackwardArgs& a, bool host_scene, int variant, cudaStream_t st) {
  const int64_t mq = a.q_end - a.q_begin;
  const int blocks = mq > 0 ? div_up(static_cast<int>(mq), kBwdThreads) : 1;
  if (host_scene) preprocess_backward_kernel<true, 6><<<blocks, kBwdThreads, 0, st>>>(a);
  else if (variant == 2) launch_pdl(preprocess_backward_kernel<false, 4>, dim3(blocks), dim3(kBwdThreads), 0, st, a);
  else launch_pdl(preprocess_backward_kernel<false, 6>, dim3(blocks), dim3(kBwdThreads), 0, st, a);
}

}  // namespace fgs
