// raster.cu — K3 forward tile blend and K4a reverse blend backward, sm_100a.
//
// One CTA of 256 threads per 16x16 tile, one pixel per thread. Splat records of a tile's
// sorted list are staged in shared memory in batches; a pixel stops at the reference's
// termination rule and the CTA exits when every pixel has stopped (__syncthreads_count).
//
// Exactness: the decision chain (dx, dy, power, alpha thresholds, transmittance stop) is
// evaluated FMA-free in the reference's op order (inc/splatting.hpp:284-292); the exp uses
// MUFU.EX2 except within a guard band of the 1/255 and 0.99 thresholds, where the correctly
// rounded exp is used (fgs_common.cuh), so skip/clamp decisions match the oracle's parity mode.
// Colour accumulation uses FMA (tolerance-checked, not bit-checked).
//
// Backward (inc/gradients.hpp:69-175): the reverse walk recovers T_before = T_after/(1-alpha)
// from the forward's final transmittance and last-contributor index, accumulates the suffix
// colour, and produces per-(pixel, splat) gradients (mean_px 2, conic 3, colour 3, alpha 1).
// They are summed over the tile's pixels in a fixed order (warp shuffle tree, then warps in
// order) and written to the intersection's emission slot: no atomics, deterministic.

#include <algorithm>

#include "fgs_kernels.h"

namespace fgs {

namespace {

constexpr int kBlend = 256;
constexpr int kBwdBatch = 128;

__global__ void __launch_bounds__(kBlend) blend_forward_kernel(BlendArgs a) {
  __shared__ float4 s0[kBlend];
  __shared__ float4 s1[kBlend];
  __shared__ float s2[kBlend];
  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int px = tx * kTile + (threadIdx.x & 15), py = ty * kTile + (threadIdx.x >> 4);
  const bool inside = px < a.width && py < a.height;
  const uint32_t lo = a.tile_offsets[tile], hi = a.tile_offsets[tile + 1];
  const float fx = static_cast<float>(px) + 0.5f, fy = static_cast<float>(py) + 0.5f;
  float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
  uint32_t last = lo;
  bool done = !inside;
  unsigned long long n_eval = 0, n_contrib = 0;

  for (uint32_t base = lo; base < hi; base += kBlend) {
    if (__syncthreads_count(done) == kBlend) break;
    const uint32_t k = base + threadIdx.x;
    if (k < hi) {
      const uint32_t g = __ldg(a.sorted_gauss + k);
      s0[threadIdx.x] = __ldg(a.rec.rec0 + g);
      s1[threadIdx.x] = __ldg(a.rec.rec1 + g);
      s2[threadIdx.x] = __ldg(a.rec.rec2 + g);
    }
    __syncthreads();
    if (!done) {
      const int cnt = static_cast<int>(min(static_cast<uint32_t>(kBlend), hi - base));
      for (int j = 0; j < cnt; ++j) {
        if (a.counters) ++n_eval;
        const float4 r0 = s0[j];
        const float dx = __fsub_rn(fx, r0.x);
        const float dy = __fsub_rn(fy, r0.y);
        const float c = s1[j].x;
        const float power = blend_power(r0.z, r0.w, c, dx, dy);
        if (power > 0.0f || power < kPowerFloor) continue;
        const float4 r1 = s1[j];
        float e;
        const float alpha = fminf(kAlphaClamp, alpha_raw(r1.y, power, &e));
        if (alpha < kAlphaSkip) continue;
        const float Tn = __fmul_rn(T, __fsub_rn(1.0f, alpha));
        if (Tn < kTransmittanceStop) {
          done = true;
          break;
        }
        const float w = __fmul_rn(alpha, T);
        C0 = fmaf(r1.z, w, C0);
        C1 = fmaf(r1.w, w, C1);
        C2 = fmaf(s2[j], w, C2);
        T = Tn;
        last = base + j + 1;
        if (a.counters) ++n_contrib;
      }
    }
  }
  if (inside) {
    const size_t pix = static_cast<size_t>(py) * a.width + px;
    a.image[pix * 3 + 0] = C0 + T * a.bg[0];
    a.image[pix * 3 + 1] = C1 + T * a.bg[1];
    a.image[pix * 3 + 2] = C2 + T * a.bg[2];
    a.final_T[pix] = T;
    a.last[pix] = last;
    if (a.counters) {
      atomicAdd(a.counters + 0, n_eval);
      atomicAdd(a.counters + 1, n_contrib);
    }
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kBlend) blend_backward_kernel(BlendArgs a) {
  constexpr int NW = kBlend / 32;
  __shared__ float4 s0[kBwdBatch];
  __shared__ float4 s1[kBwdBatch];
  __shared__ float s2[kBwdBatch];
  __shared__ uint32_t s_emit[kBwdBatch];
  __shared__ float s_part[NW][kBwdBatch][9];
  __shared__ uint32_t s_max_last;

  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int px = tx * kTile + (threadIdx.x & 15), py = ty * kTile + (threadIdx.x >> 4);
  const bool inside = px < a.width && py < a.height;
  const uint32_t lo = a.tile_offsets[tile], hi = a.tile_offsets[tile + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_max_last = lo;
  __syncthreads();

  const float fx = static_cast<float>(px) + 0.5f, fy = static_cast<float>(py) + 0.5f;
  float T = 1.0f, dl0 = 0.0f, dl1 = 0.0f, dl2 = 0.0f;
  uint32_t last = lo;
  if (inside) {
    const size_t pix = static_cast<size_t>(py) * a.width + px;
    T = a.final_T[pix];
    last = a.last[pix];
    dl0 = a.dl_dimage[pix * 3 + 0];
    dl1 = a.dl_dimage[pix * 3 + 1];
    dl2 = a.dl_dimage[pix * 3 + 2];
    atomicMax(&s_max_last, last);
  }
  float sf0 = T * a.bg[0], sf1 = T * a.bg[1], sf2 = T * a.bg[2];
  __syncthreads();
  const uint32_t end = s_max_last;

  // Entries past every pixel's last contributor get zero partials.
  for (uint32_t k = end + threadIdx.x; k < hi; k += kBlend) {
    float* p = a.partials + static_cast<size_t>(a.sorted_emit[k]) * 9;
#pragma unroll
    for (int q = 0; q < 9; ++q) p[q] = 0.0f;
  }

  for (int64_t bend = end; bend > static_cast<int64_t>(lo); bend -= kBwdBatch) {
    const uint32_t bstart = static_cast<uint32_t>(max(static_cast<int64_t>(lo), bend - kBwdBatch));
    const int cnt = static_cast<int>(bend - bstart);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const uint32_t k = bstart + threadIdx.x;
      const uint32_t g = __ldg(a.sorted_gauss + k);
      s0[threadIdx.x] = __ldg(a.rec.rec0 + g);
      s1[threadIdx.x] = __ldg(a.rec.rec1 + g);
      s2[threadIdx.x] = __ldg(a.rec.rec2 + g);
      s_emit[threadIdx.x] = __ldg(a.sorted_emit + k);
    }
    __syncthreads();
    for (int j = cnt - 1; j >= 0; --j) {
      const uint32_t k = bstart + j;
      float g[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) g[q] = 0.0f;
      bool contrib = false;
      if (k < last) {
        const float4 r0 = s0[j];
        const float4 r1 = s1[j];
        const float dx = __fsub_rn(fx, r0.x);
        const float dy = __fsub_rn(fy, r0.y);
        const float power = blend_power(r0.z, r0.w, r1.x, dx, dy);
        if (power <= 0.0f && power >= kPowerFloor) {
          float e;
          const float ar = alpha_raw(r1.y, power, &e);
          const float alpha = fminf(kAlphaClamp, ar);
          if (alpha >= kAlphaSkip) {
            contrib = true;
            const float one_m = 1.0f - alpha;
            const float Tb = T / one_m;
            const float w = alpha * Tb;
            const float b2 = s2[j];
            g[5] = dl0 * w;
            g[6] = dl1 * w;
            g[7] = dl2 * w;
            const float dot_c = dl0 * r1.z + dl1 * r1.w + dl2 * b2;
            const float dot_s = dl0 * sf0 + dl1 * sf1 + dl2 * sf2;
            const float d_alpha = dot_c * Tb - dot_s / one_m;
            sf0 = fmaf(r1.z, w, sf0);
            sf1 = fmaf(r1.w, w, sf1);
            sf2 = fmaf(b2, w, sf2);
            T = Tb;
            if (!(ar > kAlphaClamp)) {  // clamped contributions carry no geometric gradient
              g[8] = d_alpha * e;
              const float dp = d_alpha * alpha;
              g[0] = dp * (r0.z * dx + r0.w * dy);
              g[1] = dp * (r0.w * dx + r1.x * dy);
              g[2] = dp * (-0.5f * dx * dx);
              g[3] = dp * (-dx * dy);
              g[4] = dp * (-0.5f * dy * dy);
            }
          }
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
#pragma unroll
        for (int q = 0; q < 9; ++q) g[q] = warp_sum(g[q]);
      }
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 9; ++q) s_part[warp][j][q] = g[q];
      }
    }
    __syncthreads();
    // Fixed-order reduction over warps; one writer per entry.
    for (int idx = threadIdx.x; idx < cnt * 9; idx += kBlend) {
      const int j = idx / 9, q = idx - j * 9;
      float s = s_part[0][j][q];
#pragma unroll
      for (int w = 1; w < NW; ++w) s += s_part[w][j][q];
      a.partials[static_cast<size_t>(s_emit[j]) * 9 + q] = s;
    }
  }
}

}  // namespace

int blend_forward(const BlendArgs& a, cudaStream_t st) {
  blend_forward_kernel<<<a.tiles_x * a.tiles_y, kBlend, 0, st>>>(a);
  return 1;
}

int blend_backward(const BlendArgs& a, cudaStream_t st) {
  blend_backward_kernel<<<a.tiles_x * a.tiles_y, kBlend, 0, st>>>(a);
  return 1;
}

namespace {
// 8 independent FMUL->FADD chains per thread, rounding intrinsics so nothing contracts to FFMA.
__global__ void __launch_bounds__(256) fp32_probe_kernel(float* out, int iters) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0f + 1e-3f * (threadIdx.x + k);
  const float m = 0.9999f, c = 1e-4f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __fadd_rn(__fmul_rn(a[k], m), c);
  }
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678f) out[0] = s;  // keep the chains alive
}
}  // namespace

double fp32_peak_probe(cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  cudaMalloc(&out, sizeof(float));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fp32_probe_kernel<<<blocks, threads, 0, st>>>(out, 64);  // warm-up
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, st);
    fp32_probe_kernel<<<blocks, threads, 0, st>>>(out, iters);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * 8.0 * iters * double(blocks) * threads;
    if (ms > 0) best = std::max(best, ops / (ms * 1e-3));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}

}  // namespace fgs
