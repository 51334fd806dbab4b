// fgs_common.cuh — shared device definitions for the B200 Fisheye-GS kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fgs {

// Forward-model constants (reference inc/core.hpp:43-53), rounded to float exactly as the
// reference's S(...) casts do.
constexpr float kAlphaClamp = 0.99f;
constexpr float kAlphaSkip = static_cast<float>(1.0 / 255.0);
constexpr float kTransmittanceStop = 1.0e-4f;
constexpr float kCovarianceDilation = 0.3f;
constexpr float kRadiusSigma = 3.0f;
constexpr int kTile = 16;
constexpr float kFisheyeCullMargin = static_cast<float>(10.0 * 3.141592653589793238462643383279502884 / 180.0);
constexpr float kFisheyeSeriesW2 = 1.0e-6f;

// Skip power below this without evaluating exp: alpha_max < 1 (sigmoid) => alpha <=
// exp(power) < 1/255 for power < ln(1/255) = -5.5413. -5.6 keeps a margin.
constexpr float kPowerFloor = -5.6f;
// Guard band (relative) around the 1/255 and 0.99 decision thresholds inside which the
// fast exp is replaced by the correctly rounded one (SURVEY.md §7 hard part 2).
constexpr float kGuardRel = 4.0e-6f;

struct DevCamera {
  int width, height;
  float fx, fy, cx, cy;
  float W[9];   // rotation_wc row-major
  float b[3];   // translation_wc
  float fov_max;
  float center[3];  // -W^T b (inc/cameras.hpp:60), precomputed on host in the same op order
};

// Splat record for the blend (per Gaussian):
//   rec0 = (mean_px.x, mean_px.y, conic.a, conic.b), rec1 = (conic.c, alpha_max, R, G), rec2 = B
struct SplatRefs {
  const float4* rec0;
  const float4* rec1;
  const float* rec2;
};

// Splat record gathered into sorted (tile-list) order by the binning kernel, so the blends
// read each tile's list as one contiguous, 16-byte aligned stream: 48 bytes per intersection.
struct SortedRec {
  float4 a;  // mean_px.x, mean_px.y, conic.a, conic.b
  float4 b;  // conic.c, alpha_max, R, G
  float4 c;  // B, unused x3
};

// Correctly rounded fp32 exp / atan2 (double evaluation, one rounding): the definition the
// oracle's parity mode uses.
__device__ __forceinline__ float cr_expf(float x) { return static_cast<float>(exp(static_cast<double>(x))); }
__device__ __forceinline__ float cr_atan2f(float y, float x) {
  return static_cast<float>(atan2(static_cast<double>(y), static_cast<double>(x)));
}

// The blend's decision chain in the reference's exact op order, FMA-free
// (inc/splatting.hpp:284-287): power = -0.5*((a*dx)*dx + (c*dy)*dy) - (b*dx)*dy.
__device__ __forceinline__ float blend_power(float a, float b, float c, float dx, float dy) {
  const float t1 = __fmul_rn(__fmul_rn(a, dx), dx);
  const float t2 = __fmul_rn(__fmul_rn(c, dy), dy);
  const float u = __fmul_rn(-0.5f, __fadd_rn(t1, t2));
  const float v = __fmul_rn(__fmul_rn(b, dx), dy);
  return __fsub_rn(u, v);
}

// alpha_max * exp(power) with the fast MUFU exp, falling back to the correctly rounded exp
// when the product lies within the fast path's error bound of a decision threshold.
__device__ __forceinline__ float alpha_raw(float alpha_max, float power, float* expp) {
  float e = __expf(power);
  float ar = __fmul_rn(alpha_max, e);
  const bool near_skip = fabsf(ar - kAlphaSkip) <= kGuardRel * kAlphaSkip;
  const bool near_clamp = fabsf(ar - kAlphaClamp) <= kGuardRel * kAlphaClamp;
  if (near_skip || near_clamp) {
    e = cr_expf(power);
    ar = __fmul_rn(alpha_max, e);
  }
  *expp = e;
  return ar;
}

__host__ __device__ inline int div_up(int a, int b) { return (a + b - 1) / b; }

}  // namespace fgs
