// binning.cu — K2: depth-rank scan, key duplication, onesweep LSD radix sort, tile ranges.
//
// Ordering contract (reference inc/splatting.hpp:192-249): the per-tile
// lists are sorted by (tile id, depth key bits, source index). The reference duplicates keys
// in source order and runs two stable LSD sorts (depth, then tile). Here the same order is
// produced with less traffic:
//   level 1: stable sort of the N Gaussians by depth key (ties keep source order);
//   duplicate in depth-rank order (tiles ascending within a Gaussian);
//   level 2: stable sort of the I intersections by tile id.
// Stability of both levels gives exactly (tile, depth, source).
//
// The radix sort is a single-pass-per-digit "onesweep" LSD sort: one histogram kernel for all
// digit passes, then per pass one kernel whose CTAs take tiles in launch order from an atomic
// counter, rank their keys with warp match-based multisplit, resolve global digit offsets by
// decoupled look-back, and scatter through shared memory.

#include "fgs_kernels.h"

namespace fgs {

namespace {

constexpr uint32_t kFlagAgg = 1u, kFlagInc = 2u;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Block-wide exclusive scan of one value per thread (blockDim.x == 256 or 1024).
template <int THREADS>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = THREADS / 32;
    uint32_t w = lane < NW ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NW) s_warp[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const uint32_t warp_prefix = warp ? s_warp[warp - 1] : 0u;
  if (total) *total = s_warp[THREADS / 32 - 1];
  return warp_prefix + x - v;
}

template <int PASSES>
__global__ void __launch_bounds__(256) radix_hist_kernel(const uint32_t* __restrict__ keys, int n,
                                                         uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[PASSES * 256];
  for (int j = threadIdx.x; j < PASSES * 256; j += 256) h[j] = 0;
  __syncthreads();
  const int n4 = n >> 2;
  const uint4* k4 = reinterpret_cast<const uint4*>(keys);
  for (int idx = blockIdx.x * 256 + threadIdx.x; idx < n4; idx += gridDim.x * 256) {
    const uint4 k = __ldg(k4 + idx);
#pragma unroll
    for (int p = 0; p < PASSES; ++p) {
      atomicAdd(&h[p * 256 + ((k.x >> (8 * p)) & 255u)], 1u);
      atomicAdd(&h[p * 256 + ((k.y >> (8 * p)) & 255u)], 1u);
      atomicAdd(&h[p * 256 + ((k.z >> (8 * p)) & 255u)], 1u);
      atomicAdd(&h[p * 256 + ((k.w >> (8 * p)) & 255u)], 1u);
    }
  }
  if (blockIdx.x == 0)
    for (int idx = (n4 << 2) + threadIdx.x; idx < n; idx += 256) {
      const uint32_t k = keys[idx];
#pragma unroll
      for (int p = 0; p < PASSES; ++p) atomicAdd(&h[p * 256 + ((k >> (8 * p)) & 255u)], 1u);
    }
  __syncthreads();
  for (int j = threadIdx.x; j < PASSES * 256; j += 256)
    if (h[j]) atomicAdd(&hist[j], h[j]);
}

// One CTA per pass: exclusive scan of the 256 digit counts.
__global__ void __launch_bounds__(256) radix_hist_scan_kernel(uint32_t* hist) {
  __shared__ uint32_t s_warp[8];
  uint32_t* h = hist + blockIdx.x * 256;
  const uint32_t v = h[threadIdx.x];
  const uint32_t ex = block_exclusive_scan<256>(v, s_warp, nullptr);
  h[threadIdx.x] = ex;
}

__global__ void __launch_bounds__(kSortThreads) onesweep_kernel(const uint32_t* __restrict__ keys_in,
                                                                const uint32_t* __restrict__ vals_in,
                                                                uint32_t* __restrict__ keys_out,
                                                                uint32_t* __restrict__ vals_out, int n, int shift,
                                                                const uint32_t* __restrict__ digit_offsets,
                                                                uint32_t* __restrict__ lookback,
                                                                uint32_t* __restrict__ tile_counter) {
  constexpr int W = kSortThreads / 32;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp_hist[W][256];
  __shared__ uint32_t s_local_start[256];
  __shared__ uint32_t s_global_start[256];
  __shared__ uint32_t s_scan[W];
  __shared__ uint32_t s_keys[kSortTile];
  __shared__ uint32_t s_vals[kSortTile];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int j = tid; j < W * 256; j += kSortThreads) (&s_warp_hist[0][0])[j] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int base = static_cast<int>(tile) * kSortTile;
  const int warp_base = base + warp * (32 * kSortItems);

  uint32_t k[kSortItems], v[kSortItems], rank[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int idx = warp_base + i * 32 + lane;
    const bool valid = idx < n;
    k[i] = valid ? __ldg(keys_in + idx) : 0xFFFFFFFFu;
    v[i] = valid ? __ldg(vals_in + idx) : 0u;
  }
  uint32_t* wh = s_warp_hist[warp];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const bool valid = (warp_base + i * 32 + lane) < n;
    const uint32_t d = (k[i] >> shift) & 255u;
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? d : 0x100u);
    uint32_t before = 0;
    if (valid) before = wh[d];
    __syncwarp();
    if (valid) {
      rank[i] = before + __popc(peers & lt);
      if ((peers & lt) == 0) wh[d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // Per digit (thread = digit): exclusive scan over warps, CTA total.
  uint32_t total = 0;
  {
    const int d = tid;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t c = s_warp_hist[w][d];
      s_warp_hist[w][d] = total;
      total += c;
    }
  }
  const uint32_t local_start = block_exclusive_scan<kSortThreads>(total, s_scan, nullptr);
  s_local_start[tid] = local_start;
  // Decoupled look-back for this digit.
  {
    const int d = tid;
    uint32_t* mine = lookback + static_cast<size_t>(tile) * 256 + d;
    uint32_t prefix = 0;
    if (tile == 0) {
      st_volatile(mine, (total << 2) | kFlagInc);
    } else {
      st_volatile(mine, (total << 2) | kFlagAgg);
      int j = static_cast<int>(tile) - 1;
      while (true) {
        const uint32_t s = ld_volatile(lookback + static_cast<size_t>(j) * 256 + d);
        const uint32_t flag = s & 3u;
        if (flag == 0) continue;
        prefix += s >> 2;
        if (flag == kFlagInc) break;
        --j;
      }
      st_volatile(mine, ((prefix + total) << 2) | kFlagInc);
    }
    s_global_start[d] = digit_offsets[d] + prefix;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const bool valid = (warp_base + i * 32 + lane) < n;
    if (valid) {
      const uint32_t d = (k[i] >> shift) & 255u;
      const uint32_t pos = s_local_start[d] + s_warp_hist[warp][d] + rank[i];
      s_keys[pos] = k[i];
      s_vals[pos] = v[i];
    }
  }
  __syncthreads();
  const int n_tile = min(kSortTile, n - base);
  for (int p = tid; p < n_tile; p += kSortThreads) {
    const uint32_t key = s_keys[p];
    const uint32_t d = (key >> shift) & 255u;
    const uint32_t gi = s_global_start[d] + (static_cast<uint32_t>(p) - s_local_start[d]);
    keys_out[gi] = key;
    vals_out[gi] = s_vals[p];
  }
}

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;  // ranks per CTA

__device__ __forceinline__ uint32_t touched_at(const uint32_t* perm, const uint32_t* touched, int r, int n) {
  if (r >= n) return 0u;
  const uint32_t g = perm ? __ldg(perm + r) : static_cast<uint32_t>(r);
  return __ldg(touched + g);
}

__global__ void __launch_bounds__(kScanThreads) scan_block_sums_kernel(const uint32_t* __restrict__ perm,
                                                                       const uint32_t* __restrict__ touched,
                                                                       uint32_t* __restrict__ block_sums, int n) {
  __shared__ uint32_t s_warp[kScanThreads / 32];
  const int r0 = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) s += touched_at(perm, touched, r0 + i, n);
  uint32_t tot;
  block_exclusive_scan<kScanThreads>(s, s_warp, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) scan_top_kernel(uint32_t* block_sums, int nb, uint32_t* total_out) {
  __shared__ uint32_t s_warp[32];
  uint32_t carry = 0;
  for (int b0 = 0; b0 < nb; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? block_sums[b] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<1024>(v, s_warp, &tot);
    if (b < nb) block_sums[b] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_out = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const uint32_t* __restrict__ perm,
                                                                  const uint32_t* __restrict__ touched,
                                                                  const uint32_t* __restrict__ block_sums,
                                                                  uint32_t* __restrict__ offsets,
                                                                  uint32_t* __restrict__ rank, int n) {
  __shared__ uint32_t s_warp[kScanThreads / 32];
  const int r0 = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint32_t c[kScanItems], s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    c[i] = touched_at(perm, touched, r0 + i, n);
    s += c[i];
  }
  uint32_t run = block_sums[blockIdx.x] + block_exclusive_scan<kScanThreads>(s, s_warp, nullptr);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int r = r0 + i;
    if (r < n) {
      offsets[r] = run;
      if (rank) rank[perm ? perm[r] : r] = static_cast<uint32_t>(r);
    }
    run += c[i];
  }
}

__global__ void __launch_bounds__(256) duplicate_kernel(const uint32_t* __restrict__ perm,
                                                        const uint32_t* __restrict__ offsets,
                                                        const uint32_t* __restrict__ touched,
                                                        const ushort4* __restrict__ rect, int tiles_x,
                                                        uint32_t* __restrict__ tile_keys,
                                                        uint32_t* __restrict__ emit_vals,
                                                        uint32_t* __restrict__ emit_gauss, int n) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t g = __ldg(perm + r);
  if (__ldg(touched + g) == 0) return;
  const ushort4 b = rect[g];
  uint32_t e = __ldg(offsets + r);
  for (int ty = b.z; ty <= b.w; ++ty)
    for (int tx = b.x; tx <= b.y; ++tx) {
      tile_keys[e] = static_cast<uint32_t>(ty * tiles_x + tx);
      emit_vals[e] = e;
      emit_gauss[e] = g;
      ++e;
    }
}

__global__ void __launch_bounds__(256) tile_ranges_kernel(const uint32_t* __restrict__ sorted_tiles,
                                                          const uint32_t* __restrict__ sorted_emit,
                                                          const uint32_t* __restrict__ emit_gauss,
                                                          uint32_t* __restrict__ tile_offsets,
                                                          uint32_t* __restrict__ sorted_gauss, int ni, int nt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ni) return;
  const int t = static_cast<int>(sorted_tiles[k]);
  const int tp = k > 0 ? static_cast<int>(sorted_tiles[k - 1]) : -1;
  for (int tt = tp + 1; tt <= t; ++tt) tile_offsets[tt] = static_cast<uint32_t>(k);
  if (k == ni - 1)
    for (int tt = t + 1; tt <= nt; ++tt) tile_offsets[tt] = static_cast<uint32_t>(ni);
  sorted_gauss[k] = __ldg(emit_gauss + __ldg(sorted_emit + k));
}

__global__ void __launch_bounds__(256) debug_keys_kernel(const uint32_t* __restrict__ offsets,
                                                         const uint32_t* __restrict__ touched,
                                                         const ushort4* __restrict__ rect,
                                                         const uint32_t* __restrict__ depth_key, int tiles_x,
                                                         uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss,
                                                         int n) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n || touched[g] == 0) return;
  const ushort4 b = rect[g];
  uint32_t e = offsets[g];
  for (int ty = b.z; ty <= b.w; ++ty)
    for (int tx = b.x; tx <= b.y; ++tx) {
      key_tile[e] = static_cast<uint32_t>(ty * tiles_x + tx);
      key_depth[e] = depth_key[g];
      key_gauss[e] = static_cast<uint32_t>(g);
      ++e;
    }
}

}  // namespace

SortResult radix_sort_pairs(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_a, uint32_t* vals_a,
                            uint32_t* keys_b, uint32_t* vals_b, int n, int passes, const SortScratch& s,
                            cudaStream_t st) {
  SortResult r{const_cast<uint32_t*>(keys_in), const_cast<uint32_t*>(vals_in), 0};
  if (n <= 0 || passes <= 0) return r;
  const int tiles = div_up(n, kSortTile);
  cudaMemsetAsync(s.hist, 0, sizeof(uint32_t) * 256 * passes, st);
  cudaMemsetAsync(s.lookback, 0, sizeof(uint32_t) * 256 * static_cast<size_t>(tiles) * passes, st);
  cudaMemsetAsync(s.counters, 0, sizeof(uint32_t) * passes, st);
  const int hist_grid = max(1, min(div_up(n, 256 * 16), 148 * 4));
  switch (passes) {
    case 1: radix_hist_kernel<1><<<hist_grid, 256, 0, st>>>(keys_in, n, s.hist); break;
    case 2: radix_hist_kernel<2><<<hist_grid, 256, 0, st>>>(keys_in, n, s.hist); break;
    case 3: radix_hist_kernel<3><<<hist_grid, 256, 0, st>>>(keys_in, n, s.hist); break;
    default: radix_hist_kernel<4><<<hist_grid, 256, 0, st>>>(keys_in, n, s.hist); break;
  }
  radix_hist_scan_kernel<<<passes, 256, 0, st>>>(s.hist);
  r.launches = 2 + passes;
  const uint32_t *ki = keys_in, *vi = vals_in;
  for (int p = 0; p < passes; ++p) {
    uint32_t* ko = (p & 1) ? keys_a : keys_b;
    uint32_t* vo = (p & 1) ? vals_a : vals_b;
    onesweep_kernel<<<tiles, kSortThreads, 0, st>>>(ki, vi, ko, vo, n, 8 * p, s.hist + 256 * p,
                                                   s.lookback + static_cast<size_t>(256) * tiles * p,
                                                   s.counters + p);
    ki = ko;
    vi = vo;
    r.keys = ko;
    r.vals = vo;
  }
  return r;
}

int rank_scan(const uint32_t* perm, const uint32_t* touched, uint32_t* offsets, uint32_t* rank, uint32_t* block_sums,
              uint32_t* total_out, int n, cudaStream_t st) {
  const int nb = max(1, div_up(n, kScanTile));
  scan_block_sums_kernel<<<nb, kScanThreads, 0, st>>>(perm, touched, block_sums, n);
  scan_top_kernel<<<1, 1024, 0, st>>>(block_sums, nb, total_out);
  scan_apply_kernel<<<nb, kScanThreads, 0, st>>>(perm, touched, block_sums, offsets, rank, n);
  return 3;
}

int duplicate(const uint32_t* perm, const uint32_t* offsets, const uint32_t* touched, const ushort4* rect, int tiles_x,
              uint32_t* tile_keys, uint32_t* emit_vals, uint32_t* emit_gauss, int n, cudaStream_t st) {
  if (n <= 0) return 0;
  duplicate_kernel<<<div_up(n, 256), 256, 0, st>>>(perm, offsets, touched, rect, tiles_x, tile_keys, emit_vals,
                                                   emit_gauss, n);
  return 1;
}

int tile_ranges(const uint32_t* sorted_tiles, const uint32_t* sorted_emit, const uint32_t* emit_gauss,
                uint32_t* tile_offsets, uint32_t* sorted_gauss, int num_isect, int num_tiles, cudaStream_t st) {
  if (num_isect <= 0) {
    cudaMemsetAsync(tile_offsets, 0, sizeof(uint32_t) * (num_tiles + 1), st);
    return 0;
  }
  tile_ranges_kernel<<<div_up(num_isect, 256), 256, 0, st>>>(sorted_tiles, sorted_emit, emit_gauss, tile_offsets,
                                                             sorted_gauss, num_isect, num_tiles);
  return 1;
}

void debug_source_order_keys(const uint32_t* touched, const ushort4* rect, const uint32_t* depth_key, int tiles_x,
                             int n, uint32_t* scratch_offsets, uint32_t* block_sums, uint32_t* total,
                             uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss, cudaStream_t st) {
  if (n <= 0) return;
  rank_scan(nullptr, touched, scratch_offsets, nullptr, block_sums, total, n, st);
  debug_keys_kernel<<<div_up(n, 256), 256, 0, st>>>(scratch_offsets, touched, rect, depth_key, tiles_x, key_tile,
                                                    key_depth, key_gauss, n);
}

}  // namespace fgs
