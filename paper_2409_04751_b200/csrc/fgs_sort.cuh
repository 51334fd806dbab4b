// fgs_sort.cuh — per-tile bitonic sort of the (depth_key << 32 | Gaussian id) keys, run by
// the forward blend's CTA on its own tile before blending (raster.cu).
//
// Ascending comparators only: stage (k, j) pairs index i with its mirror in the k-block
// (i ^ (k - 1)) when j == k/2, else with i ^ j; the smaller key goes to the lower index. Pads
// (index >= L) hold +inf and never move, so the global variant never materialises them.
// Register form (one warp, 32*E keys, "striped": key i = r*32 + lane lives in register r of
// lane `lane`): partners with j < 32 are in another lane (shuffles), partners with j >= 32 in
// another register of the same lane. Lists of <= 256 keys are sorted by one warp in registers;
// up to kSortCap keys by the CTA in shared memory (registers for the stages inside 256-key
// chunks); longer lists by kSortCap-chunks in shared memory with the cross-chunk stages on
// global memory.
#pragma once

#include <type_traits>

#include "fgs_kernels.h"

namespace fgs {
namespace {

constexpr int kSortCap = 4096;     // keys sorted entirely in shared memory


__device__ __forceinline__ uint64_t kmin(uint64_t x, uint64_t y) { return y < x ? y : x; }
__device__ __forceinline__ uint64_t kmax(uint64_t x, uint64_t y) { return y < x ? x : y; }

// Stage (k, j) with j < 32: partner in lane ^ mask, same register.
template <int E>
__device__ __forceinline__ void xlane_stage(uint64_t (&x)[E], int lane, int mask, int half) {
  const bool lower = (lane & half) == 0;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const uint64_t y = __shfl_xor_sync(0xffffffffu, x[r], mask);
    x[r] = lower ? kmin(x[r], y) : kmax(x[r], y);
  }
}

// Half-cleaner stage with j = 32 * RJ: partner register r | RJ of the same lane.
template <int E, int RJ>
__device__ __forceinline__ void inlane_pairs(uint64_t (&x)[E]) {
#pragma unroll
  for (int r = 0; r < E; ++r)
    if ((r & RJ) == 0) {
      const uint64_t l = kmin(x[r], x[r | RJ]), h = kmax(x[r], x[r | RJ]);
      x[r] = l;
      x[r | RJ] = h;
    }
}

// Mirror stage of level k = 64 * RB (RM = (k - 1) >> 5): partner lane ^ 31, register r ^ RM;
// the lower index is the one whose register has bit RB clear.
template <int E, int RM, int RB>
__device__ __forceinline__ void inlane_mirror(uint64_t (&x)[E]) {
  // registers r and r ^ RM exchange with the partner lane as a pair (two live temporaries)
#pragma unroll
  for (int r = 0; r < E; ++r) {
    if (r < (r ^ RM)) {
      const int q = r ^ RM;
      const uint64_t ya = __shfl_xor_sync(0xffffffffu, x[q], 31);  // partner's x[q] pairs with x[r]
      const uint64_t yb = __shfl_xor_sync(0xffffffffu, x[r], 31);  // partner's x[r] pairs with x[q]
      x[r] = (r & RB) == 0 ? kmin(x[r], ya) : kmax(x[r], ya);
      x[q] = (q & RB) == 0 ? kmin(x[q], yb) : kmax(x[q], yb);
    }
  }
}

// One stage (k, j) on a warp's 32*E striped keys (k = 0: a half-cleaner stage of a merge
// level above 32E).
template <int E>
__device__ __forceinline__ void warp_stage(uint64_t (&x)[E], int lane, int k, int j) {
  if (j < 32) {
    const bool mir = j == (k >> 1);
    xlane_stage<E>(x, lane, mir ? k - 1 : j, mir ? (k >> 1) : j);
    return;
  }
  if constexpr (E >= 2) {
    if (j == (k >> 1)) {
      if (k == 64) inlane_mirror<E, 1, 1>(x);
      if constexpr (E >= 4)
        if (k == 128) inlane_mirror<E, 3, 2>(x);
      if constexpr (E >= 8)
        if (k == 256) inlane_mirror<E, 7, 4>(x);
    } else {
      if (j == 32) inlane_pairs<E, 1>(x);
      if constexpr (E >= 4)
        if (j == 64) inlane_pairs<E, 2>(x);
      if constexpr (E >= 8)
        if (j == 128) inlane_pairs<E, 4>(x);
    }
  }
}

// Full ascending sort of the warp's 32*E striped keys.
template <int E>
__device__ __forceinline__ void warp_sort(uint64_t (&x)[E], int lane) {
#pragma unroll 1
  for (int k = 2; k <= 32 * E; k <<= 1)
#pragma unroll 1
    for (int j = k >> 1; j >= 1; j >>= 1) warp_stage<E>(x, lane, k, j);
}

// The half-cleaner stages j = 16E .. 1 of a merge level k > 32E (no mirror stage).
template <int E>
__device__ __forceinline__ void warp_halfclean(uint64_t (&x)[E], int lane) {
#pragma unroll 1
  for (int j = 16 * E; j >= 1; j >>= 1) warp_stage<E>(x, lane, 0, j);
}

__device__ __forceinline__ void ce_index(int c, int k, int j, int& i, int& p) {
  i = 2 * c - (c & (j - 1));
  p = (j == (k >> 1)) ? (i ^ (k - 1)) : (i + j);
}

__device__ __forceinline__ void ce(uint64_t* s, int i, int p) {
  const uint64_t x = s[i], y = s[p];
  if (y < x) {
    s[i] = y;
    s[p] = x;
  }
}

constexpr int kChunk = 256;  // keys per warp register chunk (E = 8)
#ifndef FGS_SORT_WARP_MAX
#define FGS_SORT_WARP_MAX 256
#endif
constexpr int kWarpSortMax = FGS_SORT_WARP_MAX;  // longer lists: the CTA sorts (one warp below)
static_assert(kWarpSortMax <= kChunk, "one warp sorts at most one register chunk");

// Register phase over the shared array s[0, n) (n a multiple of the chunk 32*E): every warp
// loads its chunks, runs a full sort (first) or the half-cleaner stages j < 32E of a merge
// level, and stores them back. Callers barrier before and after.
template <int NT, int E, bool kFull>
__device__ __forceinline__ void chunk_phase(uint64_t* s, int n) {
  constexpr int CH = 32 * E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp * CH; c < n; c += (NT / 32) * CH) {
    uint64_t x[E];
#pragma unroll
    for (int r = 0; r < E; ++r) x[r] = s[c + r * 32 + lane];
    if (kFull) warp_sort<E>(x, lane);
    else warp_halfclean<E>(x, lane);
#pragma unroll
    for (int r = 0; r < E; ++r) s[c + r * 32 + lane] = x[r];
  }
}

// Ascending sort of s[0, n) (n a power of two, n >= 256 * E / 8... i.e. a multiple of 32E) by
// the whole CTA: chunks of 32E keys sorted in registers, then every merge level's stages with
// j >= 32E in shared memory and the rest in registers. E is chosen so that the first phase
// keeps all warps busy (n / 32E >= kSortWarps where possible).
template <int NT, int E>
__device__ void cta_sort_e(uint64_t* s, int n) {
  constexpr int CH = 32 * E;
  __syncthreads();
  chunk_phase<NT, E, true>(s, n);
  for (int k = 2 * CH; k <= n; k <<= 1) {
    for (int j = k >> 1; j >= CH; j >>= 1) {
      __syncthreads();
      for (int c = threadIdx.x; c < (n >> 1); c += NT) {
        int i, p;
        ce_index(c, k, j, i, p);
        ce(s, i, p);
      }
    }
    __syncthreads();
    chunk_phase<NT, E, false>(s, n);
  }
  __syncthreads();
}

// E = n / (32 * warps) where possible, so the first (register) phase keeps every warp busy.
template <int NT>
__device__ void cta_sort(uint64_t* s, int n) {
  constexpr int W = NT / 32;
  if (n <= 64 * W) cta_sort_e<NT, 2>(s, n);
  else if (n <= 128 * W) cta_sort_e<NT, 4>(s, n);
  else cta_sort_e<NT, 8>(s, n);
}

// Stages j = C/2 .. 1 of a merge level k > C on the shared chunk s[0, C) (C = kSortCap).
template <int NT>
__device__ void cta_halfclean(uint64_t* s) {
  for (int j = kSortCap >> 1; j >= kChunk; j >>= 1) {
    __syncthreads();
    for (int c = threadIdx.x; c < (kSortCap >> 1); c += NT) {
      const int i = 2 * c - (c & (j - 1));
      ce(s, i, i + j);
    }
  }
  __syncthreads();
  chunk_phase<NT, 8, false>(s, kSortCap);
  __syncthreads();
}

// CTA radix sort of L <= kRadixCap tile-list keys by depth key, then Gaussian id.
// Stable LSD radix over the 32-bit depth key (4 passes of 8 bits, ping-pong between the two
// halves of the shared key buffer, the last pass writing the sorted 64-bit keys) with the id
// as payload; keys tied in depth (rare) are then
// put in id order by one thread per run. Every warp owns a contiguous segment of the list and
// walks it in order, so ranks follow list order: per-warp digit counts (peers by eight
// ballots), one CTA scan over (digit, warp), then the scatter. 4 passes x 3 barriers
// replace the bitonic network's O(log^2 L) stages.
constexpr int kRadixCap = 2048;
constexpr int kRadixMin = 512;  // shorter lists: the bitonic network is faster (measured)

// Lanes holding the same 8-bit digit as this lane (among the lanes with `ok`): eight ballots.
__device__ __forceinline__ unsigned digit_peers(uint32_t d, bool ok) {
  unsigned peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const unsigned bit = (d >> b) & 1u;
    const unsigned bb = __ballot_sync(0xffffffffu, bit);
    peers &= bb ^ (bit - 1u);  // bit set: bb; clear: ~bb
  }
  return peers;
}

template <int NT>
__device__ void cta_radix_sort(uint32_t* s32, int L, uint32_t (*hist)[256]) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int seg = ((L + NW - 1) / NW + 31) & ~31;  // keys per warp, whole rows
  const int b0 = warp * seg, b1 = min(L, b0 + seg);
  uint32_t* ka = s32;                 // buffer A: keys [0, kRadixCap), ids [kRadixCap, 2 kRadixCap)
  uint32_t* kb = s32 + 2 * kRadixCap;  // buffer B; the last pass writes (id, key) pairs over A
#pragma unroll 1
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = 8 * pass;
    uint32_t* src = (pass & 1) ? kb : ka;
    uint32_t* dst = (pass & 1) ? ka : kb;
    for (int d = lane; d < 256; d += 32) hist[warp][d] = 0;
    __syncwarp();
    for (int r = b0; r < b1; r += 32) {
      const int i = r + lane;
      const uint32_t d = i < b1 ? (src[i] >> sh) & 0xffu : 0u;
      const unsigned peers = digit_peers(d, i < b1);
      if (i < b1 && (peers & lt) == 0) hist[warp][d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // exclusive offsets in (digit, warp) order
    for (int d = tid; d < 256; d += NT) {
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) t += hist[w][d];
      hist[0][d] = hist[0][d] | (t << 16);  // stash the digit total in the high half (L < 65536)
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t run = 0;
#pragma unroll 1
      for (int c = 0; c < 256; c += 32) {
        const uint32_t t = hist[0][c + lane] >> 16;
        uint32_t x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        const uint32_t excl = run + x - t;
        run += __shfl_sync(0xffffffffu, x, 31);
        // per-warp offsets of digit c + lane
        uint32_t acc = excl;
        const uint32_t h0 = hist[0][c + lane] & 0xffffu;
        hist[0][c + lane] = acc;
        acc += h0;
#pragma unroll
        for (int w = 1; w < NW; ++w) {
          const uint32_t hw = hist[w][c + lane];
          hist[w][c + lane] = acc;
          acc += hw;
        }
      }
    }
    __syncthreads();
    for (int r = b0; r < b1; r += 32) {
      const int i = r + lane;
      const bool ok = i < b1;
      const uint32_t key = ok ? src[i] : 0u;
      const uint32_t id = ok ? src[kRadixCap + i] : 0u;
      const uint32_t d = (key >> sh) & 0xffu;
      const unsigned peers = digit_peers(d, ok);
      if (ok) {
        const uint32_t pos = hist[warp][d] + __popc(peers & lt);
        if (pass == 3) {  // last pass: (id, key) pairs, i.e. the 64-bit keys, into buffer A's space
          s32[2 * pos] = id;
          s32[2 * pos + 1] = key;
        } else {
          dst[pos] = key;
          dst[kRadixCap + pos] = id;
        }
      }
      __syncwarp();
      if (ok && (peers & lt) == 0) hist[warp][d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
  }
  // ties in depth: ids ascending within each run of equal keys (runs are rare and short)
  auto key_at = [&](int k) { return s32[2 * k + 1]; };
  bool tie = false;
  for (int i = tid + 1; i < L; i += NT) tie |= key_at(i) == key_at(i - 1);
  if (__syncthreads_or(tie)) {
    for (int i = tid; i < L - 1; i += NT) {
      if (key_at(i) == key_at(i + 1) && (i == 0 || key_at(i - 1) != key_at(i))) {
        int e = i + 1;
        while (e + 1 < L && key_at(e + 1) == key_at(i)) ++e;
        for (int x = i + 1; x <= e; ++x) {
          const uint32_t t = s32[2 * x];
          int y = x - 1;
          while (y >= i && s32[2 * y] > t) {
            s32[2 * (y + 1)] = s32[2 * y];
            --y;
          }
          s32[2 * (y + 1)] = t;
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Sort the tile list keys[lo, lo + L) (CTA-wide call, all NT threads) by
// (depth key, Gaussian id) and write the sorted Gaussian ids (sorted_gauss[lo + k]). Returns the
// word offset in s at which the ids are also left in shared memory (g of entry k at
// ((uint32_t*)s)[offset + k]: 0 for lists of <= 256, 2 kRadixCap for the radix range), or -1
// (read sorted_gauss).
// hist (NT/32 x 256 counters): enables the radix path for kRadixMin < L <= kRadixCap.
template <int NT>
__device__ int sort_tile_list(uint64_t* keys, uint32_t* sorted_gauss, uint32_t lo, int L, uint64_t* s,
                              uint32_t (*hist)[256] = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31;
  uint32_t* s32 = reinterpret_cast<uint32_t*>(s);
  uint64_t* g = keys + lo;
  if (L <= 0) return 0;
  if (L <= kWarpSortMax) {
    if (tid < 32) {
      auto run = [&](auto e_tag) {
        constexpr int E = decltype(e_tag)::value;
        uint64_t x[E];
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int i = r * 32 + lane;
          x[r] = i < L ? g[i] : ~0ull;
        }
        warp_sort<E>(x, lane);
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int i = r * 32 + lane;
          if (i < L) {
            const uint32_t gi = static_cast<uint32_t>(x[r]);
            sorted_gauss[lo + i] = gi;
            s32[i] = gi;
          }
        }
      };
      if (L <= 32) run(std::integral_constant<int, 1>{});
      else if (L <= 64) run(std::integral_constant<int, 2>{});
      else if (L <= 128) run(std::integral_constant<int, 4>{});
      else run(std::integral_constant<int, 8>{});
    }
    __syncthreads();
    return 0;
  }
  if (L <= kRadixCap && L > kRadixMin && hist) {
    for (int k = tid; k < L; k += NT) {
      const uint64_t v = g[k];
      s32[k] = static_cast<uint32_t>(v >> 32);
      s32[kRadixCap + k] = static_cast<uint32_t>(v);
    }
    __syncthreads();
    cta_radix_sort<NT>(s32, L, hist);  // leaves the sorted 64-bit keys in s[0, L)
    for (int k = tid; k < L; k += NT) {
      const uint32_t gi = s32[2 * k];
      sorted_gauss[lo + k] = gi;
      s32[2 * kRadixCap + k] = gi;
    }
    __syncthreads();
    return 2 * kRadixCap;
  }
  const int P = pow2_ceil(L);
  if (P <= kSortCap) {
    for (int k = tid; k < P; k += NT) s[k] = k < L ? g[k] : ~0ull;
    cta_sort<NT>(s, P);
    // lists up to 2048 keys: the ids also go to the upper half of the buffer (free: the keys
    // used s[0, P) = words [0, 2P)), as for the radix range
    const bool keep = P <= kRadixCap;
    for (int k = tid; k < L; k += NT) {
      const uint32_t gi = static_cast<uint32_t>(s[k]);
      sorted_gauss[lo + k] = gi;
      if (keep) s32[2 * kRadixCap + k] = gi;
    }
    __syncthreads();
    return keep ? 2 * kRadixCap : -1;
  }
  constexpr int C = kSortCap;
  for (int c0 = 0; c0 < L; c0 += C) {
    __syncthreads();
    for (int k = tid; k < C; k += NT) s[k] = c0 + k < L ? g[c0 + k] : ~0ull;
    cta_sort<NT>(s, C);
    for (int k = tid; k < C && c0 + k < L; k += NT) g[c0 + k] = s[k];
  }
  for (int k = 2 * C; k <= P; k <<= 1) {
    for (int j = k >> 1; j >= C; j >>= 1) {
      __syncthreads();
      for (int c = tid; c < (P >> 1); c += NT) {
        int i, p;
        ce_index(c, k, j, i, p);
        if (p < L) {
          const uint64_t x = g[i], y = g[p];
          if (y < x) {
            g[i] = y;
            g[p] = x;
          }
        }
      }
    }
    for (int c0 = 0; c0 < L; c0 += C) {
      __syncthreads();
      for (int q = tid; q < C; q += NT) s[q] = c0 + q < L ? g[c0 + q] : ~0ull;
      cta_halfclean<NT>(s);
      for (int q = tid; q < C && c0 + q < L; q += NT) g[c0 + q] = s[q];
    }
  }
  __syncthreads();
  for (int k = tid; k < L; k += NT) {
    sorted_gauss[lo + k] = static_cast<uint32_t>(g[k]);
  }
  __syncthreads();
  return -1;
}

}  // namespace
}  // namespace fgs
