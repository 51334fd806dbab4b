// raster.cu — K3 forward tile blend and K4a reverse blend backward, sm_100a.
//
// One CTA per 16x16 tile; it first sorts the tile's list (fgs_sort.cuh), then each warp walks
// the sorted list independently for its pixel block, the next chunk's records arriving in
// shared memory by cp.async; a pixel stops at the reference's termination rule and a warp when
// all its pixels have stopped.
//
// Exactness: the decision chain (dx, dy, power, alpha thresholds, transmittance stop) is
// evaluated FMA-free in the reference's op order (inc/splatting.hpp:284-292); the exp uses
// MUFU.EX2 except within a guard band of the 1/255 and 0.99 thresholds, where the correctly
// rounded exp is used (fgs_common.cuh), so skip/clamp decisions match the oracle's parity mode.
// Colour accumulation uses FMA (tolerance-checked, not bit-checked).
//
// Backward (inc/gradients.hpp:69-175): the reverse walk recovers T_before = T_after/(1-alpha)
// from the forward's final transmittance and last-contributor index, accumulates the suffix
// colour (as its dot product with dL/dpixel), and produces per-(pixel, splat) gradients
// (mean_px 2, conic 3, colour 3, alpha 1). They are summed over the tile's pixels in a fixed
// order (warp shuffle tree, then warp blocks in order) and written to the intersection's
// emission slot: no atomics, deterministic.

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include <cuda.h>

#include "fgs_sort.cuh"

namespace fgs {

namespace {

// forward: splats whose alphas are computed together (measured: 4 for 1 pixel per lane, 3 for 2)
template <int PX>
#ifndef FGS_FWD_G1  // (build knobs; re-measured late round 2: 3 / 5 at 1 pixel, 2 / 4 at 2 pixels slower)
#define FGS_FWD_G1 4
#endif
#ifndef FGS_FWD_G2
#define FGS_FWD_G2 3
#endif
constexpr int kGroup = PX == 1 ? FGS_FWD_G1 : FGS_FWD_G2;

struct PixelState {
  float T, C0, C1, C2;
  uint32_t last, stop, contrib;
  bool done;
};

// Power of one (pixel, splat) pair with the reference's value (inc/splatting.hpp:284-287; see
// blend_power): t1 = (na*dx)*dx and bdx = b*dx are shared by the two pixels of a lane, nc = -c/2.
__device__ __forceinline__ float blend_power_dy(float fy, float4 r0, float nc, float t1, float bdx) {
  const float dy = __fsub_rn(fy, r0.y);
  const float t2 = __fmul_rn(__fmul_rn(nc, dy), dy);
  return __fsub_rn(__fadd_rn(t1, t2), __fmul_rn(bdx, dy));
}

// alpha_max * exp(power) with the fast exp; *near = the product lies within the fast path's
// error bound of the 1/255 skip threshold (the caller then recomputes it exactly).
// (ar >= 0: its bit patterns order like the values, so the window is one unsigned range test; a
// pixel with power > 0 may also land in it -- the exact exp then runs for a skipped step.)
// The fp32 values with |ar - 1/255| <= kGuardRel / 255 are the bit patterns 0x3B808060..0x3B8080A2;
// the range below contains them with 8 ulps to spare on each side.
constexpr uint32_t kNearLo = 0x3B808058u;
constexpr uint32_t kNearSpan = 0x0000005Au;
__device__ __forceinline__ float alpha_fast(float amax, float power, bool* near) {
  const float ar = __fmul_rn(amax, fast_exp(power));
  *near = __float_as_uint(ar) - kNearLo <= kNearSpan;  // (float compares: config 4 blend +5 %)
  return ar;
}

// The transmittance-dependent half of one reference step (inc/splatting.hpp:288-296), branch-free:
// skip (power > 0 or alpha < 1/255), stop (T' < 1e-4: the pixel is done before accumulating) or
// accumulate. A skipped or stopped step adds cr * 0 = +0 to the (non-negative) colours.
template <bool CONTRIB>
__device__ __forceinline__ void blend_apply(PixelState& p, float power, float ar, float cr, float cg, float cb,
                                            uint32_t k) {
  const float alpha = fminf(kAlphaClamp, ar);
  const bool live = !p.done && power <= 0.0f && alpha >= kAlphaSkip;
  const float Tn = __fmul_rn(p.T, __fsub_rn(1.0f, alpha));
  const bool stop = live && Tn < kTransmittanceStop;
  const bool add = live && !stop;
  const float w = add ? __fmul_rn(alpha, p.T) : 0.0f;
  p.C0 = fmaf(cr, w, p.C0);
  p.C1 = fmaf(cg, w, p.C1);
  p.C2 = fmaf(cb, w, p.C2);
  p.T = add ? Tn : p.T;
  p.last = add ? k + 1 : p.last;
  p.stop = stop ? k : p.stop;
  p.done = p.done || stop;
  if (CONTRIB) p.contrib += add ? 1u : 0u;
}

// K3 forward blend. One CTA per 16x16 tile (scheduled heaviest list first when a tile order
// is given). PX = pixels per lane: warp w owns an 8 x (4*PX) block at (8*(w&1), 4*PX*(w>>1));
// lane l the pixel(s) (l&7, (l>>3) + 4*q), q < PX, which share a column (so (a*dx)*dx and
// b*dx are computed once). Warps walk the tile's sorted list independently in 32-splat chunks
// (no CTA barriers): each lane takes one record of the chunk (fetched by cp.async one chunk
// ahead), tests it against the warp's block (rec_hits on the extent K1 stored), the survivors
// are compacted in list order into warp-private staging slots, and the warp blends them
// kGroup<PX> splats at a time (alphas first, independent of transmittance; then the sequential
// transmittance updates).
// A warp stops when all its pixels have met the reference's termination rule.
// MODE: 0 the product kernel; kModeCounters: work counters + timing instrumentation (global
// atomics) and the per-pixel blend count; kModeBlendCount: the per-pixel blend count only (the
// reference's ForwardContext::blend_count, inc/splatting.hpp:299-301).
constexpr int kModeCounters = 1, kModeBlendCount = 2;
// TMA: the chunk's records are fetched by TMA gather4 (cp.async.bulk.tensor.2d ... tile::gather4:
// 4 records of the 2D record tensor per instruction, 8 lanes issue one each, completion on a
// per-warp mbarrier) instead of 3 x 16-byte cp.async per lane (profiles A/B).
template <int MODE, int PX, bool TMA = false>
__global__ void __launch_bounds__(256 / PX) blend_forward_kernel(BlendArgs a, const __grid_constant__ CUtensorMap tmap) {
  constexpr bool COUNTERS = MODE == kModeCounters;
  constexpr bool CONTRIB = MODE != 0;
  constexpr int NW = 8 / PX;
  __shared__ __align__(128) uint64_t skeys[kSortCap];  // tile list sort; then the sorted ids and the raw records
  __shared__ float4 s01[2][NW][32];  // record staging (s0, s1); the radix sort's digit counters before
  __shared__ float s2[NW][32];
  __shared__ uint32_t sk[NW][32];    // list index of each staged record
  float4 (*s0)[32] = s01[0];
  float4 (*s1)[32] = s01[1];
  pdl_wait();  // (a programmatic dependent of K2: everything below reads K2's output)
  if (a.zero_next && blockIdx.x == 0 && threadIdx.x < 16) a.zero_next[threadIdx.x] = 0u;
  // the work item (loaded first: independent of the check below, so the two loads overlap)
  uint4 w = make_uint4(blockIdx.x, 0u, 0u, 0u);
  if (a.tile_sched) w = a.tile_sched[blockIdx.x];
  // speculative launch with buffers too small: the host grows them and launches again
  if (a.scalars && (a.scalars[kScalarI] > a.isect_cap || a.scalars[kScalarSegs] > a.ckpt_cap)) return;
  int tile = static_cast<int>(w.x);
  uint32_t lo, hi;
  if (a.tile_sched) {
    lo = w.y;
    hi = w.z;
  } else {
    lo = a.tile_offsets[tile];
    hi = a.tile_offsets[tile + 1];
  }
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bx = tx * kTile + ((warp & 1) << 3), by = ty * kTile + (warp >> 1) * 4 * PX;
  const int px = bx + (lane & 7);
  FGS_DCHECK(tile < a.tiles_x * a.tiles_y && lo == a.tile_offsets[tile] && hi == a.tile_offsets[tile + 1] && lo <= hi && static_cast<int64_t>(hi) <= a.isect_cap);
  const long long t_start = COUNTERS ? clock64() : 0;
  if (COUNTERS) span_start(a.tile_span, tile);
  // long list: reserve its segments' checkpoint slots (segments k = 1.. of the backward, then
  // the final state) in tile_ckpt[tile] (0xFFFFFFFF: none), which the CTA's other threads read
  // after the sort's barriers (a shared word would cost the 2-pixel kernel its 6th CTA per SM)
  const int nseg = static_cast<int>((hi - lo + kSeg - 1) / kSeg);
  if (threadIdx.x == 0 && nseg > 1) {
    a.tile_ckpt[tile] = 0xFFFFFFFFu;
    if (a.ckpt) {
      const uint32_t pos = atomicAdd(a.seg_cursor, static_cast<uint32_t>(nseg));
      if (pos + nseg <= a.ckpt_cap) {
        a.tile_ckpt[tile] = pos;
        for (int k = 1; k < nseg; ++k) a.seg_items[pos + k - 1] = static_cast<uint32_t>(tile) | (static_cast<uint32_t>(k) << 16);
        a.seg_items[pos + nseg - 1] = static_cast<uint32_t>(tile) | (kSegFinal << 16);
      }
    }
  }
  // sort the tile's (depth, emission slot) keys; the ids stay in shared memory when they fit
  static_assert(sizeof(s01) == NW * 256 * sizeof(uint32_t), "digit counters overlay the staging");
  const int id_off = sort_tile_list<256 / PX>(a.keys, a.sorted_gauss, lo, static_cast<int>(hi - lo), skeys,
                                              reinterpret_cast<uint32_t(*)[256]>(&s01[0][0][0]));
  if (COUNTERS && threadIdx.x == 0) {
    // sort-phase instrumentation: [4] sort cycles of small lists, [5] of long lists, [6] count long
    const unsigned long long sc = static_cast<unsigned long long>(clock64() - t_start);
    const bool big = hi - lo > 256;
    atomicAdd(a.counters + (big ? 5 : 4), sc);
    if (big) atomicAdd(a.counters + 6, 1ull);
    atomicAdd(a.counters + 7, 1ull);
  }
  uint32_t* s32 = reinterpret_cast<uint32_t*>(skeys);
  // raw records of the warp's next chunk (32 x 48 bytes), filled by cp.async; they sit in the
  // part of the sort buffer the ids do not use (ids at word 0 for short lists, at 2 kRadixCap
  // for the radix range, in global memory otherwise)
  // (TMA: each gather4 group of 4 records at a 128-byte aligned 256-byte slot, record j at float4
  // 16 (j / 4) + 3 (j % 4); else record j at float4 3 j)
  constexpr int kRawF4 = TMA ? 128 : 96;
  float4* raw = reinterpret_cast<float4*>(s32 + (id_off == 0 ? 2 * kRadixCap : 0)) + warp * kRawF4;
  static_assert(sizeof(skeys) >= (2 * kRadixCap + NW * kRawF4 * 4) * 4, "raw record buffers fit the sort buffer");
  const int rawj = TMA ? 16 * (lane >> 2) + 3 * (lane & 3) : 3 * lane;  // this lane's record
  const float fx = static_cast<float>(px) + 0.5f;
  const float bx0 = static_cast<float>(bx) + 0.5f, by0 = static_cast<float>(by) + 0.5f;
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
  // issue the copies of chunk [base, base + 32)'s records into raw (one record per lane)
  __shared__ __align__(8) uint64_t s_mbar[TMA ? NW : 1];
  const uint32_t mbar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar[TMA ? warp : 0]));
  uint32_t mbar_phase = 0;
  bool tma_pending = false;
  if (TMA && lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto prefetch = [&](uint32_t base) {
    if constexpr (TMA) {
      // lanes 0..ng-1 each gather 4 records (the last group repeats the chunk's last id)
      const int n = static_cast<int>(min(hi - base, 32u)), ng = (n + 3) / 4;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(ng * 192) : "memory");
      if (lane < ng) {
        int32_t g4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t k = base + min(4 * lane + q, n - 1);
          FGS_DCHECK(k < hi && (id_off < 0 || id_off + (k - lo) < 2 * kSortCap));
          g4[q] = static_cast<int32_t>(id_off >= 0 ? s32[id_off + (k - lo)] : __ldg(a.sorted_gauss + k));
          FGS_DCHECK(g4[q] >= 0 && g4[q] < a.num_rec);
        }
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(raw + lane * 16));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5, %6}], [%7];" ::"r"(dst),
            "l"(&tmap), "r"(0), "r"(g4[0]), "r"(g4[1]), "r"(g4[2]), "r"(g4[3]), "r"(mbar)
            : "memory");
      }
      tma_pending = true;
    } else {
      const uint32_t k = base + lane;
      if (k < hi) {
        FGS_DCHECK(id_off < 0 || id_off + (k - lo) < 2 * kSortCap);
        const uint32_t g = id_off >= 0 ? s32[id_off + (k - lo)] : __ldg(a.sorted_gauss + k);
        FGS_DCHECK(g < a.num_rec);
        const float4* src = reinterpret_cast<const float4*>(a.rec + g);
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(raw + lane * 3));
#pragma unroll
        for (int q = 0; q < 3; ++q)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * q), "l"(src + q) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  auto await_chunk = [&]() {
    if constexpr (TMA) {
      if (tma_pending) {
        asm volatile(
            "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}" ::"r"(mbar),
            "r"(mbar_phase)
            : "memory");
        mbar_phase ^= 1u;
        tma_pending = false;
      }
    } else {
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
  };
  const unsigned lt = (1u << lane) - 1u;
  prefetch(lo);
  // one checkpoint: (T, C) of the lane's pixels before entries >= the boundary (or final). The
  // slot and pixel index are re-derived here (shared memory / thread index) to keep the hot
  // loop's registers free. tile_ckpt is only read for lists longer than kSeg, whose sort has
  // barriers after thread 0 wrote it.
  auto checkpoint = [&](int k, bool fin) {
    const uint32_t slot0 = *reinterpret_cast<volatile const uint32_t*>(a.tile_ckpt + tile);
    if (slot0 == 0xFFFFFFFFu) return;
    FGS_DCHECK(static_cast<int64_t>(slot0) + k < a.ckpt_cap);
    float* c = a.ckpt + static_cast<size_t>(slot0 + k) * (4 * kTile * kTile);
    const int lpix = ((warp >> 1) * 4 * PX + (lane >> 3)) * kTile + ((warp & 1) << 3) + (lane & 7);
#pragma unroll
    for (int q = 0; q < PX; ++q) {
      const PixelState& p = ps[q];
      const int l = lpix + 64 * q;
      c[l] = p.T;
      c[256 + l] = fin ? p.C0 + p.T * a.bg[0] : p.C0;
      c[512 + l] = fin ? p.C1 + p.T * a.bg[1] : p.C1;
      c[768 + l] = fin ? p.C2 + p.T * a.bg[2] : p.C2;
    }
  };
  for (uint32_t base = lo; base < hi; base += 32) {
    if (__all_sync(0xffffffffu, all_done())) break;
    if (base > lo && (base - lo) % kSeg == 0) checkpoint(static_cast<int>((base - lo) / kSeg) - 1, false);
    await_chunk();
    __syncwarp();
    // (the exact ellipse test, which the backward uses, costs the forward more than the ~13%
    // of pairs it removes at config 2)
    const float4 ra = raw[rawj], rc = raw[rawj + 2];
    const bool pass = base + lane < hi && rec_hits(ra, rc, bx0, bx0 + 7.0f, by0, by0 + (4.0f * PX - 1.0f));
    // survivors compacted, in list order, into the warp's staging slots
    const uint32_t mask = __ballot_sync(0xffffffffu, pass);
    const int nsurv = __popc(mask);
    if (COUNTERS) warp_evals += nsurv;
    if (pass) {
      const int pos = __popc(mask & lt);
      FGS_DCHECK(pos < 32);
      s0[warp][pos] = ra;
      s1[warp][pos] = raw[rawj + 1];
      s2[warp][pos] = rc.x;
      sk[warp][pos] = base + lane;
    }
    __syncwarp();
    if (base + 32 < hi) prefetch(base + 32);
    // survivors [j0, j0 + NG): alphas first (independent of the transmittance), then the
    // sequential steps; full groups of kGroup<PX>, the chunk's remainder as one smaller group
    // (no padded slots)
    auto group = [&](int j0, auto ng_tag) {
      constexpr int NG = decltype(ng_tag)::value;
      float al[NG][PX], pw[NG][PX], am[NG], cr[NG], cg_[NG], cb[NG];
      bool any_near = false;
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const float4 r0 = s0[warp][j0 + q];
        const float4 r1 = s1[warp][j0 + q];
        cr[q] = r1.z;
        cg_[q] = r1.w;
        cb[q] = s2[warp][j0 + q];
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
        for (int q = 0; q < NG; ++q)
#pragma unroll
          for (int u = 0; u < PX; ++u) {
            bool nr;
            alpha_fast(am[q], pw[q][u], &nr);
            if (nr) al[q][u] = __fmul_rn(am[q], cr_expf(pw[q][u]));
          }
      }
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const uint32_t k = sk[warp][j0 + q];
#pragma unroll
        for (int u = 0; u < PX; ++u)
          blend_apply<CONTRIB>(ps[u], pw[q][u], al[q][u], cr[q], cg_[q], cb[q], k);
      }
    };
    constexpr int G = kGroup<PX>;
    int j0 = 0;
    for (; j0 + G <= nsurv; j0 += G) group(j0, std::integral_constant<int, G>{});
    const int rem = nsurv - j0;  // warp-uniform, < G
    if (rem == 1) group(j0, std::integral_constant<int, 1>{});
    else if (rem == 2) group(j0, std::integral_constant<int, 2>{});
    else if (rem == 3) group(j0, std::integral_constant<int, (G > 3 ? 3 : 1)>{});
    else if (rem == 4) group(j0, std::integral_constant<int, (G > 4 ? 4 : 1)>{});
    else if (rem == 5) group(j0, std::integral_constant<int, (G > 5 ? 5 : 1)>{});
    else if (rem == 6) group(j0, std::integral_constant<int, (G > 6 ? 6 : 1)>{});
    else if (rem == 7) group(j0, std::integral_constant<int, (G > 7 ? 7 : 1)>{});
    __syncwarp();
  }
  await_chunk();  // (a warp that stopped early still has its last fetch in flight)
  if (hi - lo > kSeg) checkpoint(static_cast<int>((hi - lo + kSeg - 1) / kSeg) - 1, true);  // final: T, image value
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
    span_end(a.tile_span, tile);
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
      if (CONTRIB && a.blend_count) a.blend_count[pix] = static_cast<uint16_t>(min(p.contrib, 65535u));
    }
  }
  pdl_trigger();
}

// alpha_raw's guard test: the fast-exp product lies within the error bound of a threshold.
// (Two unsigned range tests on the bits, as in the forward's alpha_fast, measured slower here:
// config 2 0.2546 -> 0.2626 ms.)
__device__ __forceinline__ bool near_threshold(float ar) {
  return fabsf(ar - kAlphaSkip) <= kGuardRel * kAlphaSkip || fabsf(ar - kAlphaClamp) <= kGuardRel * kAlphaClamp;
}

// K4a backward blend (inc/gradients.hpp:69-175). One CTA per tile, PX pixels per lane: 8/PX
// warps, warp w owns the 8 x 4PX block of bwd_box<PX>, lane l the pixels (l&7, (l>>3) + 4u),
// u < PX (one column, so dx and its products are shared).
//
// The CTA walks the tile's list backwards in 32-entry chunks, from the last contributor of any
// of its pixels, all warps on the same chunk:
//   * the chunk's 48-byte records (and each entry's emission slot) are staged in shared memory
//     once per CTA by cp.async, two chunks ahead;
//   * each warp culls the chunk against its block (box test on K1's extent, then the exact
//     ellipse test), and for every surviving splat, latest first, recovers T_before =
//     T_after / (1 - alpha), accumulates the suffix colour and forms 9 per-pixel values (the
//     power-gradient moments dp (dx, dy, dx^2, dx dy, dy^2) -- the mean / conic gradients are
//     linear in them, K4b applies the conic --, colour 3, and dp itself, alpha_max times the
//     alpha_max gradient), summed over the lane's
//     pixels and then the warp by a butterfly reduce-scatter; the warp's 9 sums per surviving entry and its survivor mask
//     go to shared memory;
//   * after one CTA barrier per chunk, the CTA adds, per entry, the sums of the warps whose mask
//     has it, in warp order, and stores the 9 values at the intersection's emission slot (K4b
//     then reads each Gaussian's intersections contiguously).
// Per-entry sums never leave the SM; deterministic (fixed summation order, no atomics).
template <int PX>
__device__ __forceinline__ void bwd_box(int tx, int ty, int w, float& x0, float& x1, float& y0, float& y1) {
  x0 = static_cast<float>(tx * kTile + ((w & 1) << 3)) + 0.5f;
  x1 = x0 + 7.0f;
  y0 = static_cast<float>(ty * kTile + (w >> 1) * 4 * PX) + 0.5f;
  y1 = y0 + (4.0f * PX - 1.0f);
}

// emission slot of tile (tx, ty) in Gaussian g's intersection list: g's first slot + the tile's
// index in its rectangle (ty-major, tx-minor; splatting.hpp:216-221)
__device__ __forceinline__ uint32_t emission_slot(const BlendArgs& a, uint32_t g, int tx, int ty) {
  const ushort4 rc = a.rect[g];
  return a.src_off[g] + static_cast<uint32_t>((ty - rc.z) * (rc.y - rc.x + 1) + (tx - rc.x));
}

// K4a's reduce-scatter: before the stage of width `half`, slot i (< 2 half) holds the sum of the
// slots t == i (mod 2 half); the stage pairs slots i and i + half, i.e. t == i (mod half). With
// NG splats' 9 values at SQ q + c, the pair needs a shuffle only if one of those t is a value.
template <int NG, int NV, int SQ>
__host__ __device__ constexpr bool live_slot(int i, int half) {
  for (int t = i; t < NV; t += half)
    if (t % SQ < 9 && t / SQ < NG) return true;
  return false;
}

// MINB: CTAs per SM the register allocation is fitted to (a launch-bounds variant: same code,
// same results, different occupancy).
template <int PX, int MINB>
__global__ void __launch_bounds__(256 / PX, MINB) blend_backward_kernel(BlendArgs a) {
  constexpr int NT = 256 / PX, NW = 8 / PX;
  __shared__ float4 s_rec[2][96];          // chunk records, double buffered
  __shared__ uint32_t s_ids[kSeg];         // the segment's Gaussian ids (entries below top)
  __shared__ uint32_t s_eslot[kSeg];       // and their emission slots
  __shared__ float s_part[2][NW][32 * 9];  // per-warp sums of the chunk's entries
  __shared__ uint32_t s_mask[2][NW];       // per-warp survivor masks (bit j: entry cs + j)
  __shared__ uint32_t s_top[NW];
  pdl_wait();  // (a programmatic dependent of the forward's K3)
  // work item: segment `seg` of a tile's list (the first num_seg_items CTAs take the segments
  // k >= 1 of long lists, the rest segment 0 of every tile, heaviest lists first)
  int tile, seg = 0;
  uint32_t tlo, thi;  // the tile's list
  if (static_cast<int64_t>(blockIdx.x) < a.num_seg_items) {
    const uint32_t item = a.seg_items[blockIdx.x];
    seg = static_cast<int>(item >> 16);
    if (seg == static_cast<int>(kSegFinal)) return;  // a final-state slot: no work item
    tile = static_cast<int>(item & 0xFFFFu);
    FGS_DCHECK(seg >= 1);
    tlo = a.tile_offsets[tile];
    thi = a.tile_offsets[tile + 1];
  } else {
    const uint32_t b = blockIdx.x - static_cast<uint32_t>(a.num_seg_items);
    if (a.tile_sched) {
      const uint4 w = a.tile_sched[b];
      tile = static_cast<int>(w.x);
      tlo = w.y;
      thi = w.z;
    } else {
      tile = static_cast<int>(b);
      tlo = a.tile_offsets[tile];
      thi = a.tile_offsets[tile + 1];
    }
  }
  FGS_DCHECK(tile >= 0 && tile < a.tiles_x * a.tiles_y);
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (seg == 0) span_start(a.tile_span, tile);
  float bx0, bx1, by0, by1;
  bwd_box<PX>(tx, ty, warp, bx0, bx1, by0, by1);
  const int px = static_cast<int>(bx0) + (lane & 7);
  FGS_DCHECK(tlo == a.tile_offsets[tile] && thi == a.tile_offsets[tile + 1]);
  // this item's entries [lo, hi)
  const uint32_t lo = tlo + static_cast<uint32_t>(seg) * kSeg;
  const uint32_t hi = min(thi, lo + static_cast<uint32_t>(kSeg));
  const int nseg = static_cast<int>((thi - tlo + kSeg - 1) / kSeg);
  FGS_DCHECK(tlo <= thi && static_cast<int64_t>(thi) <= a.isect_cap && (seg == 0 || seg < nseg));
  const float* ck = nullptr;   // checkpoint at hi (state before entries >= hi), for hi < thi
  const float* fin = nullptr;  // the tile's final state (T, image value)
  if (nseg > 1) {
    const uint32_t slot0 = a.tile_ckpt[tile];
    // the forward reserved this long list's slots (the host grows the buffers and re-renders
    // until they fit)
    FGS_DCHECK(slot0 != 0xFFFFFFFFu && static_cast<int64_t>(slot0) + nseg <= a.ckpt_cap);
    fin = a.ckpt + static_cast<size_t>(slot0 + nseg - 1) * (4 * kTile * kTile);
    if (seg + 1 < nseg) ck = a.ckpt + static_cast<size_t>(slot0 + seg) * (4 * kTile * kTile);
  }
  const float fx = static_cast<float>(px) + 0.5f;
  // ds: dL/dpixel . (suffix colour), the suffix colour T_final * bg + sum_{j later} c_j w_j
  // (gradients.hpp:132, :143) kept only through its dot product with dL/dpixel. A pixel whose last
  // contributor lies past this segment starts from the forward's checkpoint at hi: T there, and
  // the suffix colour = (image value) - (colour accumulated before hi).
  // the segment's Gaussian ids first (their loads in flight with the pixels' below; the emission
  // slots after the pixels' state, so the two dependent-load chains overlap)
  constexpr int kEnt = (kSeg + NT - 1) / NT;  // entries per thread
  uint32_t gk[kEnt];
#pragma unroll
  for (int t = 0; t < kEnt; ++t) {
    const uint32_t k = lo + tid + t * NT;
    gk[t] = k < hi ? __ldg(a.sorted_gauss + k) : 0u;
  }
  float T[PX], dl[PX][3], ds[PX], fy[PX];
  uint32_t last[PX];
  uint32_t mylast = lo;
#pragma unroll
  for (int u = 0; u < PX; ++u) {
    const int py = static_cast<int>(by0) + (lane >> 3) + 4 * u;
    fy[u] = static_cast<float>(py) + 0.5f;
    T[u] = 1.0f;
    dl[u][0] = dl[u][1] = dl[u][2] = 0.0f;
    last[u] = lo;
    float suf[3] = {0.0f, 0.0f, 0.0f};
    if (px < a.width && py < a.height) {
      const size_t pix = static_cast<size_t>(py) * a.width + px;
      const uint32_t lp = a.last[pix];
      FGS_DCHECK(lp >= tlo && lp <= thi);
      dl[u][0] = a.dl_dimage[pix * 3 + 0];
      dl[u][1] = a.dl_dimage[pix * 3 + 1];
      dl[u][2] = a.dl_dimage[pix * 3 + 2];
      if (lp > hi) {
        const int l = (py - ty * kTile) * kTile + (px - tx * kTile);
        T[u] = ck[l];
#pragma unroll
        for (int c3 = 0; c3 < 3; ++c3) suf[c3] = fin[256 * (c3 + 1) + l] - ck[256 * (c3 + 1) + l];
        last[u] = hi;
      } else {
        T[u] = a.final_T[pix];
#pragma unroll
        for (int c3 = 0; c3 < 3; ++c3) suf[c3] = T[u] * a.bg[c3];
        last[u] = max(lp, lo);
      }
    }
    ds[u] = dl[u][0] * suf[0] + dl[u][1] * suf[1] + dl[u][2] * suf[2];
    mylast = max(mylast, last[u]);
  }
  const uint32_t wlast = __reduce_max_sync(0xffffffffu, mylast);
  if (lane == 0) s_top[warp] = wlast;
  // every entry's emission slot (two dependent loads each, all in flight at once), with its id in
  // shared memory for the chunk loop's record copies and the reduction's stores
#pragma unroll
  for (int t = 0; t < kEnt; ++t) {
    const uint32_t k = lo + tid + t * NT;
    if (k < hi) {
      FGS_DCHECK(gk[t] < a.num_rec);
      const uint32_t e = emission_slot(a, gk[t], tx, ty);
      FGS_DCHECK(static_cast<int64_t>(e) < a.isect_cap);
      s_ids[k - lo] = gk[t];
      s_eslot[k - lo] = e;
    }
  }
  __syncthreads();  // top, ids, slots
  uint32_t top = lo;
#pragma unroll
  for (int w = 0; w < NW; ++w) top = max(top, s_top[w]);
  // entries past every pixel's last contributor add nothing: zero sums at their slots
  for (uint32_t k = top + tid; k < hi; k += NT) {
    float* o = a.partial_tile + static_cast<size_t>(s_eslot[k - lo]) * 9;
#pragma unroll
    for (int q = 0; q < 9; ++q) o[q] = 0.0f;
  }
  const int nch = static_cast<int>((top - lo + 31) / 32);
  // chunk c covers [max(lo, top - 32 (c + 1)), top - 32 c)
  auto chunk_lo = [&](int c) {
    return static_cast<uint32_t>(max(static_cast<int64_t>(lo), static_cast<int64_t>(top) - 32 * (c + 1)));
  };
  auto prefetch = [&](int c) {  // records of chunk c into s_rec[c & 1] (ids from shared memory)
    if (c < nch) {
      const uint32_t cs = chunk_lo(c), n = top - 32 * c - cs;
#pragma unroll
      for (int t = tid; t < 96; t += NT) {
        const uint32_t j = t / 3, q = t - 3 * j;
        if (j < n) {
          const float4* src = reinterpret_cast<const float4*>(a.rec + s_ids[cs - lo + j]) + q;
          const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&s_rec[c & 1][t]));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch(0);
  prefetch(1);
  asm volatile("cp.async.wait_group 1;" ::: "memory");
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int b = c & 1;
    const uint32_t cs = chunk_lo(c), ce = top - 32 * c;
    const float4* rec = s_rec[b];
    // ---- this warp's gradients of the chunk ----
    uint32_t mask = 0;
    if (cs < wlast) {  // warp-uniform
      const uint32_t k = cs + lane;
      if (k < ce && k < wlast) {
        const float4 ra = rec[3 * lane], rb = rec[3 * lane + 1], rc = rec[3 * lane + 2];
        if (rec_hits(ra, rc, bx0, bx1, by0, by1) && (!a.ellipse || rec_hits_ellipse(ra, rb, rc, bx0, bx1, by0, by1)))
          mask = 1u;
      }
      mask = __ballot_sync(0xffffffffu, mask != 0);
    }
    if (lane == 0) s_mask[b][warp] = mask;
    float* part = s_part[b][warp];
    // Groups of 3 surviving splats, latest first (the chunk's remainder as one smaller group).
    // Their alphas are independent of the transmittance and are computed together; the
    // transmittance/suffix recurrence then runs in list order, leaving NG x 9 per-lane gradients
    // (summed over the lane's pixels), which one butterfly reduce-scatter over the warp sums (31
    // shuffles); lane l ends with value l.
    uint32_t m = mask;
    auto group = [&](auto ng_tag) {
      constexpr int NG = decltype(ng_tag)::value;
      int js[NG];
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        js[q] = 31 - __clz(m);
        m &= ~(1u << js[q]);
      }
      float pw[NG][PX], ex[NG][PX], ar[NG][PX], dys[NG][PX];
      bool any_near = false;
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const float4 r0 = rec[3 * js[q]];
        const float amax = rec[3 * js[q] + 1].y;
        const float dx = __fsub_rn(fx, r0.x);
#pragma unroll
        for (int u = 0; u < PX; ++u) {
          dys[q][u] = __fsub_rn(fy[u], r0.y);
          pw[q][u] = blend_power(r0.z, r0.w, rec[3 * js[q] + 1].x, dx, dys[q][u]);
          ex[q][u] = fast_exp(pw[q][u]);
          ar[q][u] = __fmul_rn(amax, ex[q][u]);
          any_near |= near_threshold(ar[q][u]);
        }
      }
      if (__any_sync(0xffffffffu, any_near)) {  // rare: exact exp near the 1/255 or 0.99 threshold
#pragma unroll
        for (int q = 0; q < NG; ++q)
#pragma unroll
          for (int u = 0; u < PX; ++u)
            if (near_threshold(ar[q][u])) {
              ex[q][u] = cr_expf(pw[q][u]);
              ar[q][u] = __fmul_rn(rec[3 * js[q] + 1].y, ex[q][u]);
            }
      }
      // Branch-free: every lane evaluates all steps and gates them (a non-contributing step
      // leaves T and the suffix colour unchanged and gives zero gradients; all operands are
      // finite: conic <= 1/0.3, one_m >= 0.01).
      // value slots: splat q's component c at 9 q + c (3 splats), 16 q + c (1 or 2 splats: the
      // reduce-scatter below then skips the pairs of slots that are both zero)
      constexpr int SQ = NG == 3 ? 9 : 16;
      float v[32];
      bool contrib_any = false;
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const uint32_t kk = cs + js[q];
        const float4 r0 = rec[3 * js[q]], r1 = rec[3 * js[q] + 1];
        const float b2 = rec[3 * js[q] + 2].x;
        const float dx = __fsub_rn(fx, r0.x);
#pragma unroll
        for (int c9 = 5; c9 < 8; ++c9) v[SQ * q + c9] = 0.0f;
        float p0 = 0.0f, p1 = 0.0f, p2 = 0.0f;
#pragma unroll
        for (int u = 0; u < PX; ++u) {
          const float alpha = fminf(kAlphaClamp, ar[q][u]);
          const bool cc = kk < last[u] && pw[q][u] <= 0.0f && pw[q][u] >= kPowerFloor && alpha >= kAlphaSkip;
          contrib_any |= cc;
          const float dy = dys[q][u];
          const float inv = fast_rcp(1.0f - alpha);
          const float Tb = T[u] * inv;
          const float w = cc ? alpha * Tb : 0.0f;
          v[SQ * q + 5] += dl[u][0] * w;
          v[SQ * q + 6] += dl[u][1] * w;
          v[SQ * q + 7] += dl[u][2] * w;
          const float dot_c = dl[u][0] * r1.z + dl[u][1] * r1.w + dl[u][2] * b2;
          // clamped contributions carry no geometric gradient
          const float d_alpha = (cc && !(ar[q][u] > kAlphaClamp)) ? dot_c * Tb - ds[u] * inv : 0.0f;
          ds[u] = fmaf(dot_c, w, ds[u]);
          T[u] = cc ? Tb : T[u];
          // the mean / conic terms through the lane's moments of dpower (its pixels share dx)
          const float dp = d_alpha * alpha;
          p0 += dp;
          p1 = fmaf(dp, dy, p1);
          p2 = fmaf(dp * dy, dy, p2);
        }
        // the moments sum_u dp (dx, dy, dx^2, dx dy, dy^2); the mean / conic gradients are linear
        // in them with the splat's conic as coefficients (K4b forms them from the summed moments)
        const float m0 = dx * p0;
        v[SQ * q + 0] = m0;
        v[SQ * q + 1] = p1;
        v[SQ * q + 2] = dx * m0;
        v[SQ * q + 3] = dx * p1;
        v[SQ * q + 4] = p2;
        // sum dp = alpha_max * dL/dalpha_max (dp = d_alpha * alpha_max * exp(power) unclamped,
        // 0 clamped): K4b's opacity-logit gradient is then sum dp (1 - alpha_max)
        v[SQ * q + 8] = p0;
      }
      // (one splat's 9 values: a 16-wide reduce-scatter over the half-warps, then one shuffle
      // across them -- 16 shuffles instead of 31; two splats: 24)
      constexpr int NV = NG == 1 ? 16 : 32;
#pragma unroll
      for (int s = 0; s < NV; ++s)
        if (!(s % SQ < 9 && s / SQ < NG)) v[s] = 0.0f;
      if (__any_sync(0xffffffffu, contrib_any)) {
#pragma unroll
        for (int half = NV / 2; half >= 1; half >>= 1) {
          const bool up = (lane & half) != 0;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            if (!live_slot<NG, NV, SQ>(i, half)) continue;
            const float send = up ? v[i] : v[i + half];
            const float keep = up ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
          }
        }
        if (NV == 16) v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16);
      } else {
        v[0] = 0.0f;
      }
      // lane l now holds slot l % NV: component (l % NV) % SQ of splat (l % NV) / SQ
      const int sl = lane & (NV - 1);
      const int q = sl / SQ, c = sl - SQ * q;
      int jq = js[0];  // (no dynamic register indexing)
#pragma unroll
      for (int t = 1; t < NG; ++t) jq = q == t ? js[t] : jq;
      if (c < 9 && q < NG && lane < NV) part[jq * 9 + c] = v[0];
    };
    const int nsurv = __popc(mask);
    for (int t = 0; t + 3 <= nsurv; t += 3) group(std::integral_constant<int, 3>{});
    if (nsurv % 3 == 1) group(std::integral_constant<int, 1>{});
    else if (nsurv % 3 == 2) group(std::integral_constant<int, 2>{});
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // ---- per entry of the chunk: the passing warps' sums in warp order, at the emission slot ----
    const uint32_t n = ce - cs;
    for (uint32_t idx = tid; idx < n * 9; idx += NT) {
      const uint32_t j = idx / 9, q = idx - 9 * j;
      float sg = 0.0f;
#pragma unroll
      for (int w = 0; w < NW; ++w)
        if ((s_mask[b][w] >> j) & 1u) sg = sg + s_part[b][w][idx];
      const uint32_t e = s_eslot[cs - lo + j];
      FGS_DCHECK(static_cast<int64_t>(e) < a.isect_cap);
      a.partial_tile[static_cast<size_t>(e) * 9 + q] = sg;
    }
    prefetch(c + 2);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (seg == 0) span_end(a.tile_span, tile);
  pdl_trigger();
}
}  // namespace

namespace {
// The record array as a 2D tensor (12 floats x N rows) for TMA gather4, rebuilt when the buffer
// moves or grows. cuTensorMapEncodeTiled is reached through the runtime's driver entry point.
struct RecTensorMap {
  CUtensorMap map{};
  const void* ptr = nullptr;
  int64_t rows = 0;
  bool ok = false;
};

bool encode_rec_map(RecTensorMap& m, const void* rec, int64_t rows) {
  if (m.ok && m.ptr == rec && m.rows == rows) return true;
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<Encode>(nullptr);
    return reinterpret_cast<Encode>(fn);
  }();
  if (!encode || rows <= 0) return false;
  const cuuint64_t dims[2] = {12, static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {48};
  const cuuint32_t box[2] = {12, 1};
  const cuuint32_t estr[2] = {1, 1};
  m.ok = encode(&m.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(rec), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  m.ptr = rec;
  m.rows = rows;
  return m.ok;
}
}  // namespace

namespace {
int env_carveout(const char* name, int dflt) {  // (experiments: a percent from the environment)
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}
}  // namespace

int blend_forward(const BlendArgs& a, int64_t num_isect, int px_request, cudaStream_t st) {
  static PerDevice attrs;
  attrs.get([] {
    // Shared-memory carveout: the 2-pixel kernel fits 6 CTAs per SM only with the largest
    // carveout; the 1-pixel kernel (4 CTAs, register-bound) needs ~78% and gets the rest as L1,
    // where the 8 warps of a tile re-read each chunk's records (config 2 blend 0.177 -> 0.172 ms).
    for (const void* f : {reinterpret_cast<const void*>(blend_forward_kernel<kModeCounters, 1>),
                          reinterpret_cast<const void*>(blend_forward_kernel<kModeBlendCount, 1>),
                          reinterpret_cast<const void*>(blend_forward_kernel<0, 1>),
                          reinterpret_cast<const void*>(blend_forward_kernel<0, 1, true>)})
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, env_carveout("FGS_FWD1_CARVEOUT", 78));
    for (const void* f : {reinterpret_cast<const void*>(blend_forward_kernel<kModeCounters, 2>),
                          reinterpret_cast<const void*>(blend_forward_kernel<kModeBlendCount, 2>),
                          reinterpret_cast<const void*>(blend_forward_kernel<0, 2>)})
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return 1;
  });
  // 2 pixels per lane (4 warps of 8x8 blocks) amortise the per-splat work and idle fewer warps
  // while a CTA sorts its list; 1 pixel per lane (8x4 blocks) culls and terminates finer and
  // gives a long list twice the warps. The caller picks (fgs_api.cu, rule_fwd_px); the choice only
  // changes the work decomposition, never a pixel's value.
  (void)num_isect;
  const int tiles = a.tiles_x * a.tiles_y;
  const int px = px_request == 1 ? 1 : 2;
  // record staging by TMA gather4 (FGS_FWD_TMA=1; product kernel, 1 pixel per lane): the A/B of
  // off by default
  static const int env_tma = [] {
    const char* v = std::getenv("FGS_FWD_TMA");
    return v ? std::atoi(v) : 0;
  }();
  static thread_local RecTensorMap rec_map;
  const bool tma = env_tma == 1 && px == 1 && !a.counters && !a.blend_count &&
                   encode_rec_map(rec_map, a.rec, a.num_rec);
  const CUtensorMap& tm = rec_map.map;
  if (px == 1) {
    if (a.counters) blend_forward_kernel<kModeCounters, 1><<<tiles, 256, 0, st>>>(a, tm);
    else if (a.blend_count) blend_forward_kernel<kModeBlendCount, 1><<<tiles, 256, 0, st>>>(a, tm);
    else if (tma) blend_forward_kernel<0, 1, true><<<tiles, 256, 0, st>>>(a, tm);
    else launch_pdl(blend_forward_kernel<0, 1>, dim3(tiles), dim3(256), 0, st, a, tm);
  } else {
    if (a.counters) blend_forward_kernel<kModeCounters, 2><<<tiles, 128, 0, st>>>(a, tm);
    else if (a.blend_count) blend_forward_kernel<kModeBlendCount, 2><<<tiles, 128, 0, st>>>(a, tm);
    else launch_pdl(blend_forward_kernel<0, 2>, dim3(tiles), dim3(128), 0, st, a, tm);
  }
  return 1;
}

int blend_backward(const BlendArgs& a, int64_t num_isect, int variant, cudaStream_t st, int* px_used) {
  // 8x8 warp blocks with 2 pixels per lane amortise the per-splat overhead (culling, the
  // 27-value warp reduction) over twice the pixels: faster from ~32 entries per tile on average
  // (profiles/r02_variants.md: configs 1-4), while a small image (config 0: 256 tiles) keeps 8x4
  // blocks and twice the warps. FGS_BWD_PX=1|2 overrides.
  static const int env = [] {
    const char* v = std::getenv("FGS_BWD_PX");
    return v ? std::atoi(v) : 0;
  }();
  const int tiles = a.tiles_x * a.tiles_y;
  const int px = env == 1 || env == 2 ? env
                 : (tiles >= 1024 && num_isect >= 32 * static_cast<int64_t>(tiles) ? 2 : 1);
  // 2 pixels per lane: fitted to 8 CTAs per SM (64 registers, a few spills) or 6 (77, none);
  // identical results. Since the segment's ids / slots moved to shared memory, 8 is faster at
  // every config (config 2 0.2526 -> 0.2463 ms, config 1 0.1276 -> 0.1240, configs 3 / 4 -0.4 %
  // / -0.1 %; it was 7 % slower before). FGS_BWD_MINB=6|8 overrides.
  static const int env_minb = [] {
    const char* v = std::getenv("FGS_BWD_MINB");
    return v ? std::atoi(v) : 0;
  }();
  const int minb = env_minb == 6 || env_minb == 8 ? env_minb : 8;
  (void)variant;
  static PerDevice attrs;
  attrs.get([] {
    // shared-memory carveout of the backward blends (FGS_BWD_CARVEOUT=percent; default: the
    // driver's choice)
    const char* v = std::getenv("FGS_BWD_CARVEOUT");
    if (v && *v)
      for (const void* f : {reinterpret_cast<const void*>(blend_backward_kernel<1, 4>),
                            reinterpret_cast<const void*>(blend_backward_kernel<2, 6>),
                            reinterpret_cast<const void*>(blend_backward_kernel<2, 8>)})
        cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(v));
    return 1;
  });
  if (px_used) *px_used = px;
  // one CTA per (tile, segment): the long lists' segments k >= 1 first, then every tile's first
  const int grid = tiles + static_cast<int>(a.num_seg_items);
  if (px == 1) launch_pdl(blend_backward_kernel<1, 4>, dim3(grid), dim3(256), 0, st, a);
  else if (minb == 8) launch_pdl(blend_backward_kernel<2, 8>, dim3(grid), dim3(128), 0, st, a);
  else launch_pdl(blend_backward_kernel<2, 6>, dim3(grid), dim3(128), 0, st, a);
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
