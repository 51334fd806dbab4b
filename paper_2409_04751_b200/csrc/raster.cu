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

constexpr int kBlend = 256;     // threads per tile CTA = pixels per tile
constexpr int kBwdBatch = 128;  // splats per backward batch
constexpr int kWarps = kBlend / 32;
constexpr int kGroup = 4;         // forward: splats whose alphas are computed together

// Warp w of a tile owns the 8x4 pixel block at (8*(w&1), 4*(w>>1)); lane l the pixel
// (l&7, l>>3) inside it. Square-ish blocks make the per-warp culling below tight.
__device__ __forceinline__ void pixel_of(int tid, int& lx, int& ly) {
  const int w = tid >> 5, l = tid & 31;
  lx = ((w & 1) << 3) + (l & 7);
  ly = ((w >> 1) << 2) + (l >> 3);
}

// Conservative per-warp visibility of one splat: bit w is set unless no pixel centre of warp
// w's 8x4 block can reach alpha >= 1/255. alpha(d) = alpha_max * exp(-q(d)/2) with
// q = a dx^2 + 2b dx dy + c dy^2, so alpha >= 1/255 needs q <= 2 ln(255 alpha_max), whose
// bounding box has half-extents sqrt(2 tau Sigma_xx), sqrt(2 tau Sigma_yy) (Sigma = Q^-1).
// The box is inflated (0.1% + 1e-3 px) far beyond fp32 rounding of the blend's power, so a
// culled (pixel, splat) pair is exactly one the reference would `continue` on: the image and
// every decision are unchanged; only evaluations that cannot contribute are skipped.
__device__ __forceinline__ uint32_t warp_mask(float4 r0, float4 r1, float tile_x0, float tile_y0) {
  const float a = r0.z, b = r0.w, c = r1.x, amax = r1.y;
  if (!(amax >= kAlphaSkip)) return 0u;
  const float det = a * c - b * b;
  if (!(det > 0.0f) || !(a > 0.0f) || !(c > 0.0f)) return 0xFFu;
  const float tau2 = 2.0f * __logf(255.0f * amax) * 1.002f + 1e-3f;
  const float ex = sqrtf(fmaxf(tau2 * c / det, 0.0f)) * 1.001f + 1e-3f;
  const float ey = sqrtf(fmaxf(tau2 * a / det, 0.0f)) * 1.001f + 1e-3f;
  // box in tile-local pixel-centre coordinates
  const float x0 = r0.x - ex - tile_x0, x1 = r0.x + ex - tile_x0;
  const float y0 = r0.y - ey - tile_y0, y1 = r0.y + ey - tile_y0;
  uint32_t m = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const float bx0 = ((w & 1) << 3) + 0.5f, bx1 = bx0 + 7.0f;
    const float by0 = ((w >> 1) << 2) + 0.5f, by1 = by0 + 3.0f;
    if (x1 >= bx0 && x0 <= bx1 && y1 >= by0 && y0 <= by1) m |= 1u << w;
  }
  return m;
}

// Each warp compacts the batch indices whose mask has its bit into s_list[warp][...].
__device__ __forceinline__ int build_list(const uint8_t* s_mask, int cnt, int warp, int lane, uint8_t* list) {
  int n = 0;
  for (int c0 = 0; c0 < cnt; c0 += 32) {
    const int j = c0 + lane;
    const bool on = j < cnt && ((s_mask[j] >> warp) & 1u);
    const uint32_t bal = __ballot_sync(0xffffffffu, on);
    if (on) list[n + __popc(bal & ((1u << lane) - 1u))] = static_cast<uint8_t>(j);
    n += __popc(bal);
  }
  __syncwarp();
  return n;
}

// Conservative test: can any pixel centre of the box [x0, x1] x [y0, y1] reach
// alpha >= 1/255 for this splat? Same bound as warp_mask, evaluated with fast-math
// (relative error ~1e-6, far inside the 0.1-0.2% margins).
__device__ __forceinline__ bool box_may_hit(float4 r0, float4 r1, float x0, float x1, float y0, float y1) {
  const float a = r0.z, b = r0.w, c = r1.x, amax = r1.y;
  if (!(amax >= kAlphaSkip)) return false;
  const float det = a * c - b * b;
  if (!(det > 0.0f) || !(a > 0.0f) || !(c > 0.0f)) return true;
  const float tau2 = 2.0f * __logf(255.0f * amax) * 1.002f + 1e-3f;
  const float k = __fdividef(tau2, det);
  const float ex = __fsqrt_rn(fmaxf(k * c, 0.0f)) * 1.001f + 1e-3f;
  const float ey = __fsqrt_rn(fmaxf(k * a, 0.0f)) * 1.001f + 1e-3f;
  return r0.x + ex >= x0 && r0.x - ex <= x1 && r0.y + ey >= y0 && r0.y - ey <= y1;
}

struct PixelState {
  float T, C0, C1, C2;
  uint32_t last, stop, contrib;
  bool done;
};

// Power of one (pixel, splat) pair in the reference's exact op order (inc/splatting.hpp:
// 284-287). t1 = (a*dx)*dx and bdx = b*dx are shared by the two pixels of a lane.
__device__ __forceinline__ float blend_power_dy(float fy, float4 r0, float c, float t1, float bdx) {
  const float dy = __fsub_rn(fy, r0.y);
  const float t2 = __fmul_rn(__fmul_rn(c, dy), dy);
  return __fsub_rn(__fmul_rn(-0.5f, __fadd_rn(t1, t2)), __fmul_rn(bdx, dy));
}

// alpha_max * exp(power) with the fast exp; *near = the product lies within the fast path's
// error bound of the 1/255 skip threshold (the caller then recomputes it exactly).
__device__ __forceinline__ float alpha_fast(float amax, float power, bool* near) {
  const float ar = __fmul_rn(amax, __expf(power));
  *near = power <= 0.0f && fabsf(ar - kAlphaSkip) <= kGuardRel * kAlphaSkip;
  return ar;
}

// Final alpha of the reference step, or -1 when it skips (power > 0 or alpha < 1/255).
__device__ __forceinline__ float alpha_final(float power, float ar) {
  const float alpha = fminf(kAlphaClamp, ar);
  return (power <= 0.0f && alpha >= kAlphaSkip) ? alpha : -1.0f;
}

// The transmittance-dependent half of one reference step (inc/splatting.hpp:291-296).
template <bool COUNTERS>
__device__ __forceinline__ void blend_apply(PixelState& p, float alpha, float cr, float cg, float cb, uint32_t k) {
  if (p.done || alpha < 0.0f) return;
  const float Tn = __fmul_rn(p.T, __fsub_rn(1.0f, alpha));
  if (Tn < kTransmittanceStop) {
    p.done = true;
    p.stop = k;
    return;
  }
  const float w = __fmul_rn(alpha, p.T);
  p.C0 = fmaf(cr, w, p.C0);
  p.C1 = fmaf(cg, w, p.C1);
  p.C2 = fmaf(cb, w, p.C2);
  p.T = Tn;
  p.last = k + 1;
  if (COUNTERS) ++p.contrib;
}

// K3 forward blend. One CTA per 16x16 tile (scheduled heaviest list first when a tile order
// is given). PX = pixels per lane: warp w owns an 8 x (4*PX) block at (8*(w&1), 4*PX*(w>>1));
// lane l the pixel(s) (l&7, (l>>3) + 4*q), q < PX, which share a column (so (a*dx)*dx and
// b*dx are computed once). Warps walk the tile's sorted list independently in 32-splat chunks
// (no CTA barriers): each lane reads one record (the list is contiguous in sorted order, two
// chunks stay in flight), tests it against the warp's block (box_may_hit), and the warp blends
// the ballot of survivors in order from warp-private shared memory, kGroup splats at a time
// (alphas first, independent of transmittance; then the sequential transmittance updates).
// A warp stops when all its pixels have met the reference's termination rule.
template <bool COUNTERS, int PX>
__global__ void __launch_bounds__(256 / PX) blend_forward_kernel(BlendArgs a) {
  constexpr int NW = 8 / PX;
  __shared__ float4 s0[NW][32];
  __shared__ float4 s1[NW][32];
  __shared__ float s2[NW][32];
  const int tile = a.tile_order ? static_cast<int>(a.tile_order[blockIdx.x]) : static_cast<int>(blockIdx.x);
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bx = tx * kTile + ((warp & 1) << 3), by = ty * kTile + (warp >> 1) * 4 * PX;
  const int px = bx + (lane & 7);
  const uint32_t lo = a.tile_offsets[tile], hi = a.tile_offsets[tile + 1];
  const float fx = static_cast<float>(px) + 0.5f;
  const float bx0 = static_cast<float>(bx) + 0.5f, by0 = static_cast<float>(by) + 0.5f;
  const long long t_start = COUNTERS ? clock64() : 0;
  unsigned long long warp_evals = 0;
  PixelState ps[PX];
  int py[PX];
  float fy[PX];
#pragma unroll
  for (int q = 0; q < PX; ++q) {
    py[q] = by + (lane >> 3) + 4 * q;
    fy[q] = static_cast<float>(py[q]) + 0.5f;
    ps[q] = PixelState{1.0f, 0.0f, 0.0f, 0.0f, lo, hi, 0u, !(px < a.width && py[q] < a.height)};
  }
  auto all_done = [&]() {
    bool d = true;
#pragma unroll
    for (int q = 0; q < PX; ++q) d = d && ps[q].done;
    return d;
  };

  const SortedRec zero{make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
  SortedRec cur = lo + lane < hi ? a.srec[lo + lane] : zero;
  SortedRec nxt = lo + 32 + lane < hi ? a.srec[lo + 32 + lane] : zero;
  for (uint32_t base = lo; base < hi; base += 32) {
    if (__all_sync(0xffffffffu, all_done())) break;
    const bool pass = base + lane < hi && box_may_hit(cur.a, cur.b, bx0, bx0 + 7.0f, by0, by0 + (4.0f * PX - 1.0f));
    s0[warp][lane] = cur.a;
    s1[warp][lane] = cur.b;
    s2[warp][lane] = cur.c.x;
    uint32_t mask = __ballot_sync(0xffffffffu, pass);
    if (COUNTERS) warp_evals += __popc(mask);
    cur = nxt;
    if (base + 64 + lane < hi) nxt = a.srec[base + 64 + lane];
    __syncwarp();
    while (mask) {
      int js[kGroup];
#pragma unroll
      for (int q = 0; q < kGroup; ++q) {
        js[q] = mask ? __ffs(mask) - 1 : -1;
        mask &= mask - 1;
      }
      float al[kGroup][PX], pw[kGroup][PX], am[kGroup], cr[kGroup], cg_[kGroup], cb[kGroup];
      bool any_near = false;
#pragma unroll
      for (int q = 0; q < kGroup; ++q) {
        const int jj = js[q] >= 0 ? js[q] : 0;
        const float4 r0 = s0[warp][jj];
        const float4 r1 = s1[warp][jj];
        cr[q] = r1.z;
        cg_[q] = r1.w;
        cb[q] = s2[warp][jj];
        am[q] = r1.y;
        const float dx = __fsub_rn(fx, r0.x);
        const float t1 = __fmul_rn(__fmul_rn(r0.z, dx), dx);
        const float bdx = __fmul_rn(r0.w, dx);
#pragma unroll
        for (int u = 0; u < PX; ++u) {
          pw[q][u] = blend_power_dy(fy[u], r0, r1.x, t1, bdx);
          bool nr;
          al[q][u] = alpha_fast(r1.y, pw[q][u], &nr);
          any_near |= nr && !ps[u].done;
        }
      }
      if (__any_sync(0xffffffffu, any_near)) {  // rare: exact exp near the skip threshold
#pragma unroll
        for (int q = 0; q < kGroup; ++q)
#pragma unroll
          for (int u = 0; u < PX; ++u) {
            bool nr;
            alpha_fast(am[q], pw[q][u], &nr);
            if (nr) al[q][u] = __fmul_rn(am[q], cr_expf(pw[q][u]));
          }
      }
#pragma unroll
      for (int q = 0; q < kGroup; ++q) {
        if (js[q] < 0) break;
#pragma unroll
        for (int u = 0; u < PX; ++u)
          blend_apply<COUNTERS>(ps[u], alpha_final(pw[q][u], al[q][u]), cr[q], cg_[q], cb[q], base + js[q]);
      }
    }
    __syncwarp();
  }
  if (COUNTERS) {
    const long long t_cta = clock64() - t_start;
    unsigned long long ev = 0, ec = 0;
#pragma unroll
    for (int q = 0; q < PX; ++q)
      if (px < a.width && py[q] < a.height) {
        // E_eval as the reference counts it: k-loop iterations entered, including the one
        // that terminates (inc/splatting.hpp:282-292).
        ev += (ps[q].stop < hi) ? (ps[q].stop - lo + 1) : (hi - lo);
        ec += ps[q].contrib;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ev += __shfl_xor_sync(0xffffffffu, ev, o);
      ec += __shfl_xor_sync(0xffffffffu, ec, o);
    }
    if (lane == 0) {
      atomicAdd(a.counters + 0, ev);
      atomicAdd(a.counters + 1, ec);
      atomicAdd(a.counters + 2, warp_evals * (32 * PX));
      atomicMax(a.counters + 3, static_cast<unsigned long long>(t_cta));
      if (a.tile_cycles) atomicMax(a.tile_cycles + tile, static_cast<unsigned long long>(t_cta));
    }
  }
#pragma unroll
  for (int q = 0; q < PX; ++q) {
    const PixelState& p = ps[q];
    if (px < a.width && py[q] < a.height) {
      const size_t pix = static_cast<size_t>(py[q]) * a.width + px;
      a.image[pix * 3 + 0] = p.C0 + p.T * a.bg[0];
      a.image[pix * 3 + 1] = p.C1 + p.T * a.bg[1];
      a.image[pix * 3 + 2] = p.C2 + p.T * a.bg[2];
      a.final_T[pix] = p.T;
      a.last[pix] = p.last;
    }
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kBlend) blend_backward_kernel(BlendArgs a) {
  __shared__ float4 s0[kBwdBatch];
  __shared__ float4 s1[kBwdBatch];
  __shared__ float s2[kBwdBatch];
  __shared__ uint32_t s_emit[kBwdBatch];
  __shared__ uint8_t s_mask[kBwdBatch];
  __shared__ uint8_t s_list[kWarps][kBwdBatch];
  __shared__ float s_part[kWarps][kBwdBatch][9];
  __shared__ uint32_t s_max_last;
  __shared__ uint32_t s_wl[kWarps];

  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int lx, ly;
  pixel_of(threadIdx.x, lx, ly);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < a.width && py < a.height;
  const uint32_t lo = a.tile_offsets[tile], hi = a.tile_offsets[tile + 1];
  const float tile_x0 = static_cast<float>(tx * kTile), tile_y0 = static_cast<float>(ty * kTile);
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
  }
  const uint32_t warp_last = __reduce_max_sync(0xffffffffu, last);
  if (lane == 0) {
    atomicMax(&s_max_last, warp_last);
    s_wl[warp] = warp_last;
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
      const SortedRec rr = a.srec[k];
      const float4 r0 = rr.a;
      const float4 r1 = rr.b;
      s0[threadIdx.x] = r0;
      s1[threadIdx.x] = r1;
      s2[threadIdx.x] = rr.c.x;
      s_emit[threadIdx.x] = __ldg(a.sorted_emit + k);
      s_mask[threadIdx.x] = static_cast<uint8_t>(warp_mask(r0, r1, tile_x0, tile_y0));
    }
    __syncthreads();
    // a warp whose pixels all stopped before an entry cannot take a gradient from it
    const int wcnt = static_cast<int>(min(static_cast<int64_t>(cnt), static_cast<int64_t>(warp_last) - bstart));
    const int nl = wcnt > 0 ? build_list(s_mask, wcnt, warp, lane, s_list[warp]) : 0;
    for (int i = nl - 1; i >= 0; --i) {
      const int j = s_list[warp][i];
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
    // Fixed-order reduction over the warps that listed the entry; one writer per entry.
    for (int idx = threadIdx.x; idx < cnt * 9; idx += kBlend) {
      const int j = idx / 9, q = idx - j * 9;
      const uint32_t m = s_mask[j];
      const int64_t kk = static_cast<int64_t>(bstart) + j;
      float s = 0.0f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        // listed by warp w iff its mask bit is set and the entry is below warp w's last
        const bool listed = ((m >> w) & 1u) && kk < static_cast<int64_t>(s_wl[w]);
        if (listed) s += s_part[w][j][q];
      }
      a.partials[static_cast<size_t>(s_emit[j]) * 9 + q] = s;
    }
  }
}

}  // namespace

int blend_forward(const BlendArgs& a, cudaStream_t st) {
  const int px = a.px_per_lane == 2 ? 2 : 1;
  const int threads = 256 / px;
  if (a.counters) {
    if (px == 2) blend_forward_kernel<true, 2><<<a.tiles_x * a.tiles_y, threads, 0, st>>>(a);
    else blend_forward_kernel<true, 1><<<a.tiles_x * a.tiles_y, threads, 0, st>>>(a);
  } else {
    if (px == 2) blend_forward_kernel<false, 2><<<a.tiles_x * a.tiles_y, threads, 0, st>>>(a);
    else blend_forward_kernel<false, 1><<<a.tiles_x * a.tiles_y, threads, 0, st>>>(a);
  }
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
