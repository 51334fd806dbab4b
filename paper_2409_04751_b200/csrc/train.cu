// train.cu — the training step around the rasterizer, on the device:
// the L1 + D-SSIM loss with its analytic image gradient (inc/metrics.hpp:86-195) and the Adam
// update with bias correction and per-group learning rates (inc/optimize.hpp:100-145).
//
// SSIM (per channel, 11x11 separable zero-padded Gaussian window, sigma 1.5):
//   ssim_maps_kernel   one CTA per 32x8 output tile and channel: stages x, y with a 5-pixel
//                      halo in shared memory, blurs x, y, x^2, y^2, xy (rows then columns, as
//                      metrics.hpp:37-61), forms the SSIM map s and the gradient maps
//                      a, b, b(mu_x - mu_y), e, e mu_y of metrics.hpp:131-145, writes the five
//                      maps and a per-CTA double sum of s;
//   ssim_grad_kernel   same tiling: blurs the five maps and combines them with x, y and the
//                      L1 sign term into dL/drendered (metrics.hpp:146-151, :186-191), plus a
//                      per-CTA double sum of |x - y|;
//   loss_reduce_kernel sums the per-CTA partials in a fixed order (deterministic loss value).
// Both stencil kernels are HBM-bound (each plane is read once per kernel, the halo re-reads
// hit L1/L2). fp32 arithmetic; the reference trains in double (tolerance-checked).

#include <algorithm>
#include <cmath>

#include "fgs_kernels.h"

namespace fgs {

namespace {

constexpr int kTX = 32, kTY = 8, kR = 5, kWin = 11;
constexpr int kHX = kTX + 2 * kR, kHY = kTY + 2 * kR;  // haloed tile
constexpr int kLossThreads = kTX * kTY;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

__constant__ float c_win[kWin];

// inc/metrics.hpp:23-34, evaluated in double on the host and rounded once.
void upload_window() {  // __constant__ memory is per device
  static PerDevice done;
  done.get([] {
    double w[kWin], sum = 0.0;
    for (int i = 0; i < kWin; ++i) {
      const double d = i - kWin / 2;
      w[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
      sum += w[i];
    }
    float wf[kWin];
    for (int i = 0; i < kWin; ++i) wf[i] = static_cast<float>(w[i] / sum);
    cudaMemcpyToSymbol(c_win, wf, sizeof(wf));
    return 1;
  });
}

// Block sum of one double per thread (kLossThreads threads); thread 0 gets the result.
__device__ double block_sum(double v, double* s_red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kLossThreads / 32; ++w) t += s_red[w];
  return t;
}

// Blurs of NQ haloed planes src[q][kHY][kHX] -> dst[q] at the tile's kTY x kTX pixels.
template <int NQ>
__device__ __forceinline__ void blur_tile(const float (*src)[kHY][kHX], float (*hbuf)[kHY][kTX], float out[NQ]) {
  const int tid = threadIdx.x;
  // rows: every haloed row, the tile's columns
  for (int idx = tid; idx < NQ * kHY * kTX; idx += kLossThreads) {
    const int q = idx / (kHY * kTX), rem = idx % (kHY * kTX), r = rem / kTX, c = rem % kTX;
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < kWin; ++k) acc = fmaf(c_win[k], src[q][r][c + k], acc);
    hbuf[q][r][c] = acc;
  }
  __syncthreads();
  const int tx = tid % kTX, ty = tid / kTX;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < kWin; ++k) acc = fmaf(c_win[k], hbuf[q][ty + k][tx], acc);
    out[q] = acc;
  }
}

struct LossArgs {
  const float* x;  // rendered H*W*3
  const float* y;  // target
  int width, height;
  float lambda;
  float* maps;           // [3][5][H*W]
  float* d_rendered;     // H*W*3
  double* part_ssim;     // [blocks]
  double* part_l1;       // [blocks]
};

__global__ void __launch_bounds__(kLossThreads) ssim_maps_kernel(LossArgs a) {
  __shared__ float src[5][kHY][kHX];
  __shared__ float hbuf[5][kHY][kTX];
  __shared__ double s_red[kLossThreads / 32];
  const int ch = blockIdx.z, tid = threadIdx.x;
  const int x0 = blockIdx.x * kTX - kR, y0 = blockIdx.y * kTY - kR;
  const size_t npx = static_cast<size_t>(a.width) * a.height;
  for (int idx = tid; idx < kHY * kHX; idx += kLossThreads) {
    const int r = idx / kHX, c = idx % kHX, gx = x0 + c, gy = y0 + r;
    float xv = 0.0f, yv = 0.0f;
    if (gx >= 0 && gx < a.width && gy >= 0 && gy < a.height) {
      const size_t p = (static_cast<size_t>(gy) * a.width + gx) * 3 + ch;
      xv = a.x[p];
      yv = a.y[p];
    }
    src[0][r][c] = xv;
    src[1][r][c] = yv;
    src[2][r][c] = xv * xv;
    src[3][r][c] = yv * yv;
    src[4][r][c] = xv * yv;
  }
  __syncthreads();
  float mu[5];
  blur_tile<5>(src, hbuf, mu);
  const int px = blockIdx.x * kTX + tid % kTX, py = blockIdx.y * kTY + tid / kTX;
  double s_sum = 0.0;
  if (px < a.width && py < a.height) {
    const float mx = mu[0], my = mu[1];
    const float sx2 = mu[2] - mx * mx, sy2 = mu[3] - my * my, sxy = mu[4] - mx * my;
    const float c1 = static_cast<float>(kC1), c2 = static_cast<float>(kC2);
    const float n1 = 2.0f * mx * my + c1, n2 = 2.0f * sxy + c2;
    const float d1 = mx * mx + my * my + c1, d2 = sx2 + sy2 + c2;
    const float s = (n1 * n2) / (d1 * d2);
    s_sum = s;
    const float am = 2.0f * n2 * (my - mx) * (my * (mx + my) + c1) / (d1 * d1 * d2);
    const float bm = -s / d2;
    const float em = 2.0f * n1 * (d2 - n2) / (d1 * d2 * d2);
    float* m = a.maps + static_cast<size_t>(ch) * 5 * npx + static_cast<size_t>(py) * a.width + px;
    m[0] = am;
    m[npx] = bm;
    m[2 * npx] = bm * (mx - my);
    m[3 * npx] = em;
    m[4 * npx] = em * my;
  }
  const double t = block_sum(s_sum, s_red);
  if (tid == 0) a.part_ssim[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
}

__global__ void __launch_bounds__(kLossThreads) ssim_grad_kernel(LossArgs a) {
  __shared__ float src[5][kHY][kHX];
  __shared__ float hbuf[5][kHY][kTX];
  __shared__ double s_red[kLossThreads / 32];
  const int ch = blockIdx.z, tid = threadIdx.x;
  const int x0 = blockIdx.x * kTX - kR, y0 = blockIdx.y * kTY - kR;
  const size_t npx = static_cast<size_t>(a.width) * a.height;
  const float* maps = a.maps + static_cast<size_t>(ch) * 5 * npx;
  for (int idx = tid; idx < 5 * kHY * kHX; idx += kLossThreads) {
    const int q = idx / (kHY * kHX), rem = idx % (kHY * kHX), r = rem / kHX, c = rem % kHX;
    const int gx = x0 + c, gy = y0 + r;
    src[q][r][c] = (gx >= 0 && gx < a.width && gy >= 0 && gy < a.height)
                       ? maps[static_cast<size_t>(q) * npx + static_cast<size_t>(gy) * a.width + gx]
                       : 0.0f;
  }
  __syncthreads();
  float cm[5];
  blur_tile<5>(src, hbuf, cm);
  const int px = blockIdx.x * kTX + tid % kTX, py = blockIdx.y * kTY + tid / kTX;
  double l1 = 0.0;
  if (px < a.width && py < a.height) {
    const size_t p = (static_cast<size_t>(py) * a.width + px) * 3 + ch;
    const float xv = a.x[p], yv = a.y[p];
    const float norm = static_cast<float>(1.0 / (3.0 * static_cast<double>(npx)));
    const float dssim = norm * (cm[0] + 2.0f * (xv - yv) * cm[1] - 2.0f * cm[2] + yv * cm[3] - cm[4]);
    const float diff = xv - yv;
    const float sign = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
    a.d_rendered[p] = (1.0f - a.lambda) * sign * norm - a.lambda * dssim;
    l1 = fabs(static_cast<double>(diff));
  }
  const double t = block_sum(l1, s_red);
  if (tid == 0) a.part_l1[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
}

// out[0] = sum of SSIM map values, out[1] = sum |x - y| (fixed summation order).
__global__ void __launch_bounds__(1024) loss_reduce_kernel(const double* ps, const double* pl, int nb, double* out) {
  __shared__ double s[2][32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += 1024) {
    a += ps[i];
    b += pl[i];
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = a;
    s[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tb = 0.0;
    for (int w = 0; w < 32; ++w) {
      ta += s[0][w];
      tb += s[1][w];
    }
    out[0] = ta;
    out[1] = tb;
  }
}

// ---- Adam (inc/optimize.hpp:100-145) ----
// Groups: 0 means, 1 rotations, 2 log-scales, 3 opacities, 4 SH (DC at basis 0 of each
// channel: lr[4]; higher bands: lr[5], which the reference does not have -- 0 = untouched).

__device__ __forceinline__ float group_lr(const AdamArgs& a, int g, int64_t k) {
  if (g < 4) return a.lr[g];
  return (k % 16) == 0 ? a.lr[4] : a.lr[5];
}

__global__ void adam_check_kernel(AdamArgs a) {
  const int g = blockIdx.y;
  const int64_t len = a.len[g];
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < len;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (group_lr(a, g, k) != 0.0f && !isfinite(a.g[g][k])) {
      atomicMin(a.nonfinite, static_cast<int>(k / a.width[g]));  // first offending Gaussian
      return;
    }
  }
}

__global__ void adam_update_kernel(AdamArgs a) {
  const int g = blockIdx.y;
  const int64_t len = a.len[g];
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < len;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float lr = group_lr(a, g, k);
    if (lr == 0.0f) continue;
    const float gr = a.g[g][k];
    const float m = a.beta1 * a.m[g][k] + (1.0f - a.beta1) * gr;
    const float v = a.beta2 * a.v[g][k] + (1.0f - a.beta2) * gr * gr;
    a.m[g][k] = m;
    a.v[g][k] = v;
    const float mhat = m / a.bc1, vhat = v / a.bc2;
    a.p[g][k] -= lr * mhat / (sqrtf(vhat) + a.eps);
  }
}

}  // namespace

size_t loss_scratch_floats(int width, int height) { return static_cast<size_t>(width) * height * 15; }
size_t loss_partials(int width, int height) {
  return static_cast<size_t>(div_up(width, kTX)) * div_up(height, kTY) * 3;
}

int l1_dssim_loss(const float* rendered, const float* target, int width, int height, float lambda, float* d_rendered,
                  float* maps, double* partials /* 2 * loss_partials + 2 */, cudaStream_t st) {
  upload_window();
  LossArgs a{rendered, target, width, height, lambda, maps, d_rendered, partials, nullptr};
  const int nb = static_cast<int>(loss_partials(width, height));
  a.part_l1 = partials + nb;
  const dim3 grid(div_up(width, kTX), div_up(height, kTY), 3);
  ssim_maps_kernel<<<grid, kLossThreads, 0, st>>>(a);
  ssim_grad_kernel<<<grid, kLossThreads, 0, st>>>(a);
  loss_reduce_kernel<<<1, 1024, 0, st>>>(partials, partials + nb, nb, partials + 2 * nb);
  return 3;
}

int adam_step(AdamArgs& a, cudaStream_t st) {
  int64_t mx = 0;
  for (int g = 0; g < 5; ++g) mx = a.len[g] > mx ? a.len[g] : mx;
  if (mx == 0) return 0;
  const dim3 grid(static_cast<unsigned>(std::min<int64_t>((mx + 255) / 256, 148 * 16)), 5);
  adam_update_kernel<<<grid, 256, 0, st>>>(a);
  return 1;
}

int adam_check(AdamArgs& a, cudaStream_t st) {
  int64_t mx = 0;
  for (int g = 0; g < 5; ++g) mx = a.len[g] > mx ? a.len[g] : mx;
  if (mx == 0) return 0;
  const dim3 grid(static_cast<unsigned>(std::min<int64_t>((mx + 255) / 256, 148 * 16)), 5);
  adam_check_kernel<<<grid, 256, 0, st>>>(a);
  return 1;
}

}  // namespace fgs
