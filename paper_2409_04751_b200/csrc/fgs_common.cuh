// fgs_common.cuh — shared device definitions for the B200 Fisheye-GS kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <utility>

#include <cuda_runtime.h>

namespace fgs {

// Checked build (libfgs_checked.so, -DFGS_CHECKED): device-side bounds and invariant checks at
// the kernels' indexing sites -- the memory / race checking this pool allows (compute-sanitizer is
// closed on it). A failed check prints the site and traps (the launch fails with an error).
#ifdef FGS_CHECKED
#define FGS_DCHECK(cond)                                                                          \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("FGS_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,    \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                       \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define FGS_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// Programmatic dependent launch: the next kernel of the stream may start its CTAs while this
// one's last CTAs finish (each CTA signals when its own output is written); the dependent waits
// for the whole primary grid (and its memory) before reading any of it. Both are no-ops for a
// kernel launched without the attribute. FGS_NO_PDL builds the plain launches (A/B).
__device__ __forceinline__ void pdl_wait() {
#ifndef FGS_NO_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#ifndef FGS_NO_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
#ifdef FGS_NO_PDL
  kernel<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
  return cudaGetLastError();
#else
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
#endif
}

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

constexpr float kPinholeNearClip = 0.2f;  // core.hpp:52
constexpr int kCamPinhole = 0, kCamFisheye = 1, kCamPanorama = 2;  // FGS_CAMERA_* (fgs.h)

struct DevCamera {
  int model;  // kCam*
  int width, height;
  float fx, fy, cx, cy;
  float W[9];   // rotation_wc row-major
  float b[3];   // translation_wc
  float fov_max;
  float center[3];  // -W^T b (inc/cameras.hpp:60), precomputed on host in the same op order
};

// Splat record (48 bytes, 16-byte aligned), written per Gaussian by K1 and gathered into
// sorted (tile-list) order by the binning kernel, so the blends read each tile's list as one
// contiguous stream.
struct SortedRec {
  float4 a;  // mean_px.x, mean_px.y, -conic.a / 2, conic.b
  float4 b;  // -conic.c / 2, alpha_max, R, G
  float4 c;  // B, extent x, extent y, tau (splat_cull_params)
};
// (-a/2) dx dx + (-c/2) dy dy = -((a dx dx + c dy dy) / 2) exactly: scaling by -1/2 commutes with
// every rounding (short of subnormal results, where |power| < 1e-37 leaves alpha unchanged).

// Correctly rounded fp32 exp / atan2 (double evaluation, one rounding): the definition the
// oracle's parity mode uses.
#ifdef FGS_ABL_FLOATMATH  // ablation build (timing only): fp32 libdevice transcendentals
__device__ __forceinline__ float cr_expf(float x) { return expf(x); }
__device__ __forceinline__ float cr_atan2f(float y, float x) { return atan2f(y, x); }
#else
__device__ __forceinline__ float cr_expf(float x) { return static_cast<float>(exp(static_cast<double>(x))); }
__device__ __forceinline__ float cr_atan2f(float y, float x) {
  return static_cast<float>(atan2(static_cast<double>(y), static_cast<double>(x)));
}
#endif

// The blend's decision chain in the reference's exact op order, FMA-free
// (inc/splatting.hpp:284-287): power = -0.5*((a*dx)*dx + (c*dy)*dy) - (b*dx)*dy, from the record's
// na = -a/2, nc = -c/2: ((na*dx)*dx + (nc*dy)*dy) - (b*dx)*dy, the same value.
__device__ __forceinline__ float blend_power(float na, float b, float nc, float dx, float dy) {
  const float t1 = __fmul_rn(__fmul_rn(na, dx), dx);
  const float t2 = __fmul_rn(__fmul_rn(nc, dy), dy);
  const float v = __fmul_rn(__fmul_rn(b, dx), dy);
  return __fsub_rn(__fadd_rn(t1, t2), v);
}

// Fast exp: one MUFU.EX2 with flush-to-zero (no denormal fix-up; results below 2^-126 only
// occur for power < -87, far past the skip threshold). Same value as __expf elsewhere.
__device__ __forceinline__ float fast_exp(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__fmul_rn(x, 1.4426950408889634f)));
  return y;
}

// Approximate reciprocal (MUFU.RCP, ftz) for arguments in [0.01, 1].
__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

// Instrumentation (FGS_FLAG_COUNTERS): a CTA's [start, end] in span[2 tile], span[2 tile + 1].
__device__ __forceinline__ void span_start(unsigned long long* span, int tile) {
  if (span && threadIdx.x == 0) span[2 * tile] = global_ns();
}
__device__ __forceinline__ void span_end(unsigned long long* span, int tile) {
  if (span && (threadIdx.x & 31) == 0) atomicMax(span + 2 * tile + 1, global_ns());
}

__host__ __device__ inline int div_up(int a, int b) { return (a + b - 1) / b; }

// Host-side one-time setup that is per device (function attributes, __constant__ data,
// occupancy): `get(f)` runs f() once for the current device, under a lock, and caches its
// non-zero result.
struct PerDevice {
  std::mutex m;
  int v[64] = {};
  template <typename F>
  int get(F f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(m);
    if (dev < 0 || dev >= 64) return f();
    if (!v[dev]) v[dev] = f();
    return v[dev];
  }
};

// Conservative test: can any pixel centre of the box [x0, x1] x [y0, y1] reach
// alpha >= 1/255 for this splat? alpha(d) = alpha_max * exp(-q(d)/2) with
// q = a dx^2 + 2b dx dy + c dy^2, so alpha >= 1/255 needs q <= 2 ln(255 alpha_max), whose
// bounding box has half-extents sqrt(2 tau Sigma_xx), sqrt(2 tau Sigma_yy) (Sigma = Q^-1).
// The box is inflated (0.2% + 0.1% + 1e-3 px), far beyond the ~1e-6 relative error of the
// fast-math evaluation and of the blend's fp32 power, so a culled (pixel, splat) pair is one the
// reference would `continue` on. Every op is an explicit rounding intrinsic, so the result is
// bit-identical in every translation unit (the backward writer and the K4b reader agree).
// Half-extents (ex, ey) of the splat's alpha >= 1/255 region, inflated; returns 0 when the
// splat can never reach 1/255 (alpha_max < 1/255), 2 when no finite bound applies (degenerate
// conic: never cull), 1 otherwise.
__device__ __forceinline__ int splat_extent(float4 r0, float4 r1, float& ex, float& ey) {
  const float a = r0.z, b = r0.w, c = r1.x, amax = r1.y;
  ex = ey = 0.0f;
  if (!(amax >= kAlphaSkip)) return 0;
  const float det = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, b));
  if (!(det > 0.0f) || !(a > 0.0f) || !(c > 0.0f)) return 2;
  const float tau2 = __fadd_rn(__fmul_rn(__fmul_rn(2.0f, __logf(__fmul_rn(255.0f, amax))), 1.002f), 1e-3f);
  const float k = __fdividef(tau2, det);
  ex = __fadd_rn(__fmul_rn(__fsqrt_rn(fmaxf(__fmul_rn(k, c), 0.0f)), 1.001f), 1e-3f);
  ey = __fadd_rn(__fmul_rn(__fsqrt_rn(fmaxf(__fmul_rn(k, a), 0.0f)), 1.001f), 1e-3f);
  return 1;
}

__device__ __forceinline__ bool extent_hits(int kind, float mx, float my, float ex, float ey, float x0, float x1,
                                            float y0, float y1) {
  if (kind != 1) return kind == 2;
  return __fadd_rn(mx, ex) >= x0 && __fsub_rn(mx, ex) <= x1 && __fadd_rn(my, ey) >= y0 && __fsub_rn(my, ey) <= y1;
}

__device__ __forceinline__ bool box_may_hit(float4 r0, float4 r1, float x0, float x1, float y0, float y1) {
  float ex, ey;
  const int kind = splat_extent(r0, r1, ex, ey);
  return extent_hits(kind, r0.x, r0.y, ex, ey, x0, x1, y0, y1);
}

// The culling parameters as K1 stores them in the record (SortedRec.c.y/.z/.w), computed once
// per Gaussian: the inflated half-extents and tau2, the inflated bound on the quadratic form
// (alpha >= 1/255 needs q <= 2 ln(255 alpha_max)). kind 0 -> -inf (every test fails), kind 2
// -> +inf (every test passes).
__device__ __forceinline__ float3 splat_cull_params(float4 r0, float4 r1) {
  float ex, ey;
  const int kind = splat_extent(r0, r1, ex, ey);
  if (kind == 0) return make_float3(-INFINITY, -INFINITY, -INFINITY);
  if (kind == 2) return make_float3(INFINITY, INFINITY, INFINITY);
  const float tau2 = __fadd_rn(__fmul_rn(__fmul_rn(2.0f, __logf(__fmul_rn(255.0f, r1.y))), 1.002f), 1e-3f);
  return make_float3(ex, ey, tau2);
}

// box_may_hit from the stored extent: a = record .a (mean_px in .x/.y), c = record .c.
__device__ __forceinline__ bool rec_hits(float4 a, float4 c, float x0, float x1, float y0, float y1) {
  return __fadd_rn(a.x, c.y) >= x0 && __fsub_rn(a.x, c.y) <= x1 && __fadd_rn(a.y, c.z) >= y0 &&
         __fsub_rn(a.y, c.z) <= y1;
}

// Exact form of the test above: min over the box of q(p - mean) = a dx^2 + 2b dx dy + c dy^2
// against the record's tau2. q is convex, so the minimum is 0 when the mean lies in the box and
// otherwise lies on an edge, where it is a clamped 1D minimum. The comparison carries a slack of
// 1e-5 of the terms' magnitudes (far above the fp32 rounding of q) on top of tau2's own
// inflation, so it stays conservative: a culled pair is one the reference skips. Culls ~13-19%
// of the (block, splat) pairs the box test keeps at configs 1-2. Every op is an explicit
// rounding intrinsic, so the backward's warps and its epilogue take identical decisions.
__device__ __forceinline__ bool rec_hits_ellipse(float4 ra, float4 rb, float4 rc, float x0, float x1, float y0,
                                                 float y1) {
  const float tau = rc.w;
  if (!(tau < INFINITY)) return tau > 0.0f;
  const float lx = __fsub_rn(x0, ra.x), hx = __fsub_rn(x1, ra.x);
  const float ly = __fsub_rn(y0, ra.y), hy = __fsub_rn(y1, ra.y);
  if (lx <= 0.0f && hx >= 0.0f && ly <= 0.0f && hy >= 0.0f) return true;
  const float a = -2.0f * ra.z, b = ra.w, c = -2.0f * rb.x;  // the record's -a/2, -c/2
  const float nbc = __fdiv_rn(-b, c), nba = __fdiv_rn(-b, a);
  auto q = [&](float dx, float dy) {
    const float t1 = __fmul_rn(__fmul_rn(a, dx), dx);
    const float t2 = __fmul_rn(__fmul_rn(__fmul_rn(2.0f, b), dx), dy);
    const float t3 = __fmul_rn(__fmul_rn(c, dy), dy);
    const float v = __fadd_rn(__fadd_rn(t1, t2), t3);
    return __fsub_rn(v, __fmul_rn(1e-5f, __fadd_rn(__fadd_rn(t1, fabsf(t2)), t3)));
  };
  float best = q(lx, fminf(fmaxf(__fmul_rn(nbc, lx), ly), hy));
  best = fminf(best, q(hx, fminf(fmaxf(__fmul_rn(nbc, hx), ly), hy)));
  best = fminf(best, q(fminf(fmaxf(__fmul_rn(nba, ly), lx), hx), ly));
  best = fminf(best, q(fminf(fmaxf(__fmul_rn(nba, hy), lx), hx), hy));
  return best <= tau;
}

}  // namespace fgs
