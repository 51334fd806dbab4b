// fgs_crmath.cuh — fast correctly rounded fp32 exp / atan2 for K1 / K4b (sm_100a).
//
// cr_expf / cr_atan2f (fgs_common.cuh) define the values: the fp32 rounding of libdevice's double
// exp / atan2, i.e. the correctly rounded result, which is what the reference's libm gives
// (inc/model.hpp:128-139 exp of the log-scales and the sigmoid,
// inc/cameras.hpp:121 / :157 the fisheye angle and the panorama angles). Those cost ~60 / ~140
// SASS instructions per call, a third of them materialising double constants.
//
// Here the same values come from short double evaluations whose error is a few double ulps
// (< 2^-49 relative), with the coefficients in the constant bank (DFMA reads them in place) and
// a rounding test: the double result y is rounded to fp32 only when its low 29 mantissa bits are
// more than 64 double ulps away from a float rounding midpoint -- then y and the exact value
// round the same way, and so does libdevice's evaluation (< 1 ulp), so the fp32 result equals
// cr_expf / cr_atan2f bit for bit. Otherwise (about 2.4e-7 of the inputs; zeros, infinities,
// NaNs and extreme ranges always) the full evaluation runs. fgs_selftest_crmath checks the exp
// over all 2^32 inputs and the atan2 over seeded samples on the device
// (tests/test_gpu_parity_gaps.py::test_fast_correctly_rounded_math). Measured: no faster in
// K1 / K4b, so the product build keeps the definitions (see the FGS_FAST_CRMATH note below).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace fgs {
namespace crm {

// DFMA / DADD operands straight from the constant bank
__constant__ double kC[16] = {
    0x1.71547652b82fep+6,   // 0: 64 / ln 2
    0x1.8p52,               // 1: round-to-integer shifter
    0x1.62e42fefa39efp-7,   // 2: ln 2 / 64 (high part)
    0x1.abc9e3b39803fp-62,  // 3: ln 2 / 64 - [2]
    1.0 / 120.0,            // 4..7: exp(r) = 1 + r (1 + r (1/2 + r (1/6 + r (1/24 + r / 120))))
    1.0 / 24.0,
    1.0 / 6.0,
    0.5,
    1.0 / 9.0,              // 8..11: atan(t) = t + t s (-1/3 + s (1/5 + s (-1/7 + s / 9))), s = t^2
    -1.0 / 7.0,
    1.0 / 5.0,
    -1.0 / 3.0,
    0x1.921fb54442d18p+0,   // 12: pi / 2
    0x1.921fb54442d18p+1,   // 13: pi
    1.0,
    0.0625,
};

// 2^(j/64) and atan(j/16), rounded to double; indexed per lane, so a kernel that uses the fast
// functions copies them into shared memory first (stage_tables(), then a barrier): in global
// memory the lines were evicted from L1 by K1's parameter stream and every lookup waited on L2.
__device__ const double kExp2J[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0, 0x1.0b5586cf9890fp+0,
    0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0, 0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0,
    0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0, 0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0,
    0x1.2d285a6e4030bp+0, 0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0, 0x1.4bfdad5362a27p+0,
    0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0, 0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0,
    0x1.6247eb03a5585p+0, 0x1.6623882552225p+0, 0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0,
    0x1.75feb564267c9p+0, 0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0, 0x1.9c49182a3f090p+0,
    0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0, 0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0,
    0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0, 0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0,
    0x1.d072d4a07897cp+0, 0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};
__device__ const double kAtanJ[17] = {
    0.0, 0x1.ff55bb72cfdeap-5, 0x1.fd5ba9aac2f6ep-4, 0x1.7b97b4bce5b02p-3, 0x1.f5b75f92c80ddp-3, 0x1.362773707ebccp-2,
    0x1.6f61941e4def1p-2, 0x1.a64eec3cc23fdp-2, 0x1.dac670561bb4fp-2, 0x1.0657e94db30d0p-1, 0x1.1e00babdefeb4p-1,
    0x1.345f01cce37bbp-1, 0x1.4978fa3269ee1p-1, 0x1.5d58987169b18p-1, 0x1.700a7c5784634p-1, 0x1.819d0b7158a4dp-1,
    0x1.921fb54442d18p-1};

__shared__ double s_tab[64 + 17];  // kExp2J, kAtanJ

__device__ __forceinline__ void stage_tables() {
#ifdef FGS_FAST_CRMATH
  for (int t = threadIdx.x; t < 64 + 17; t += blockDim.x) s_tab[t] = t < 64 ? kExp2J[t] : kAtanJ[t - 64];
#endif
}

// true when double y may round to fp32 differently from a value within 64 ulps of it
__device__ __forceinline__ bool near_float_midpoint(double y) {
  const uint32_t lo = static_cast<uint32_t>(__double2loint(y)) & 0x1FFFFFFFu;
  return lo - 0x10000000u + 64u <= 128u;
}

__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

// exp(x) for |x| <= 87 (normal fp32 results): 2^(k/64) = 2^(k>>6) T[k&63], r = x - k ln2/64,
// |r| <= ln2/128, a degree-5 polynomial (truncation 2^-54). *ok = false: use the full evaluation.
__device__ __forceinline__ float exp_fast_path(float x, bool* ok) {
  const double xd = static_cast<double>(x);
  const double t = fma(xd, kC[0], kC[1]);
  const int k = __double2loint(t);
  const double kd = t - kC[1];
  double r = fma(-kd, kC[2], xd);
  r = fma(-kd, kC[3], r);
  double p = fma(r, kC[4], kC[5]);
  p = fma(r, p, kC[6]);
  p = fma(r, p, kC[7]);
  p = fma(r, p, kC[14]);
  p = fma(r, p, kC[14]);
  const double y0 = s_tab[k & 63] * p;
  const double y = __hiloint2double(__double2hiint(y0) + ((k >> 6) << 20), __double2loint(y0));
  *ok = fabsf(x) <= 87.0f && !near_float_midpoint(y);
  return __double2float_rn(y);
}

// atan2(y, x) for finite nonzero |x|, |y| <= 2^100: the first-octant angle atan(n/d) (n <= d)
// as atan(c) + atan(t), c = j/16 nearest n/d, t = (n - c d) / (d + c n), |t| <= 1/32 + eps
// (series to t^9, truncation 2^-55), then the octant / quadrant / sign.
__device__ __forceinline__ float atan2_fast_path(float y, float x, bool* ok) {
  const float ax = fabsf(x), ay = fabsf(y);
  const bool swap = ay > ax;
  const float nf = swap ? ax : ay, df = swap ? ay : ax;
  // (any j in [0, 16] gives the same angle; |t| <= 0.0315 is checked, which bounds the series)
  const int j = static_cast<int>(min(static_cast<unsigned>(__float2int_rn(__fdividef(nf, df) * 16.0f)), 16u));
  const double n = nf, d = df;
  const double c = static_cast<double>(j) * kC[15];
  const double num = fma(-c, d, n);
  const double den = fma(c, n, d);
  double rc = rcp_approx(den);
  rc = fma(fma(-den, rc, kC[14]), rc, rc);
  double t = num * rc;
  t = fma(fma(-den, t, num), rc, t);
  const double s = t * t;
  double p = fma(s, kC[8], kC[9]);
  p = fma(s, p, kC[10]);
  p = fma(s, p, kC[11]);
  double res = fma(t * s, p, t) + s_tab[64 + j];
  if (swap) res = kC[12] - res;
  if (x < 0.0f) res = kC[13] - res;
  *ok = ax > 0.0f && ay > 0.0f && ax <= 0x1p100f && ay <= 0x1p100f && fabs(t) <= 0.0315 && res > 1e-30 &&
        !near_float_midpoint(res);
  const float f = __double2float_rn(res);
  return y < 0.0f ? -f : f;
}

}  // namespace crm

// K1 / K4b call cr_expf_fast / cr_atan2f_fast; they are the fast paths only in builds with
// FGS_FAST_CRMATH: on config 2 (profiles/r02d_crmath_ab.md) the fast atan2 made K1 slower
// (0.0639 vs 0.0628 ms: a longer dependent chain -- MUFU.RCP64H, Newton step, series -- in a
// latency-bound kernel) and the fast exp saved < 1 %, less than the table staging costs.
// The self-test (fgs_selftest_crmath) always exercises the fast paths.
#if !defined(FGS_FAST_CRMATH) || defined(FGS_SLOW_EXP)
__device__ __forceinline__ float cr_expf_fast(float x) { return cr_expf(x); }
#else
__device__ __forceinline__ float cr_expf_fast(float x) {
  bool ok;
  const float f = crm::exp_fast_path(x, &ok);
  if (ok) return f;
  return cr_expf(x);
}
#endif

#if !defined(FGS_FAST_CRMATH) || defined(FGS_SLOW_ATAN2)
__device__ __forceinline__ float cr_atan2f_fast(float y, float x) { return cr_atan2f(y, x); }
#else
__device__ __forceinline__ float cr_atan2f_fast(float y, float x) {
  bool ok;
  const float f = crm::atan2_fast_path(y, x, &ok);
  if (ok) return f;
  return cr_atan2f(y, x);
}
#endif

// the fast paths themselves (self-test)
__device__ __forceinline__ float cr_expf_fastpath(float x) {
  bool ok;
  const float f = crm::exp_fast_path(x, &ok);
  if (ok) return f;
  return cr_expf(x);
}
__device__ __forceinline__ float cr_atan2f_fastpath(float y, float x) {
  bool ok;
  const float f = crm::atan2_fast_path(y, x, &ok);
  if (ok) return f;
  return cr_atan2f(y, x);
}

}  // namespace fgs
