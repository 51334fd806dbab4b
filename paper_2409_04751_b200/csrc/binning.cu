// binning.cu — K2: compaction, depth-rank scan, key duplication, onesweep LSD radix sort,
// tile ranges.
//
// Ordering contract (reference inc/splatting.hpp:192-249): the per-tile
// lists are sorted by (tile id, depth key bits, source index). The reference duplicates keys
// in source order and runs two stable LSD sorts (depth, then tile). Here the same order is
// produced with less traffic:
//   compact the Gaussians that touch >= 1 tile (source order kept);
//   level 1: stable sort of those by depth key (ties keep source order);
//   duplicate in depth-rank order (tiles ascending within a Gaussian);
//   level 2: stable sort of the I intersections by tile id.
// Stability of both levels gives exactly (tile, depth, source).
//
// The radix sort is a single-pass-per-digit "onesweep" LSD sort: the digit histograms of all
// passes are accumulated by the kernel that produces the keys (compaction / duplication),
// then per pass one kernel whose CTAs take tiles in launch order from an atomic
// counter, rank their keys with warp match-based multisplit, resolve global digit offsets by
// decoupled look-back (each digit's thread loads 16 predecessor statuses per step), and
// scatter through shared memory. Element counts may live in device memory (written by the
// previous kernel), so the grid is sized for the maximum and surplus CTAs exit.

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

__device__ __forceinline__ int load_n(const uint32_t* n_dev, int n_max) {
  return n_dev ? static_cast<int>(min(*n_dev, static_cast<uint32_t>(n_max))) : n_max;
}

// Block-wide exclusive scan of one value per thread.
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

// Decoupled look-back of one 30-bit value for tile `tile` (status words: value<<2 | flag),
// predecessors at status[j * stride]. Called by a single thread; issues 16 independent loads
// per step (nearest first) so that a tile whose predecessors all run concurrently walks
// back 16 tiles per memory round trip.
__device__ __forceinline__ uint32_t look_back(const uint32_t* status, size_t stride, int tile) {
  constexpr int K = 16;
  uint32_t prefix = 0;
  int j = tile - 1;
  while (true) {
    uint32_t s[K];
#pragma unroll
    for (int q = 0; q < K; ++q) s[q] = j - q >= 0 ? ld_volatile(status + static_cast<size_t>(j - q) * stride) : 0u;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      uint32_t v = s[q];
      while ((v & 3u) == 0u) v = ld_volatile(status + static_cast<size_t>(j - q) * stride);
      prefix += v >> 2;
      if ((v & 3u) == kFlagInc) return prefix;
    }
    j -= K;
  }
}

template <int PASSES>
__global__ void __launch_bounds__(256) radix_hist_kernel(const uint32_t* __restrict__ keys, const uint32_t* n_dev,
                                                         int n_max, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[PASSES * 256];
  const int n = load_n(n_dev, n_max);
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

// Dynamic shared memory layout of onesweep_kernel.
struct OnesweepSmem {
  uint32_t keys[kSortTile];
  uint32_t vals[kSortTile];
  uint32_t warp_hist[kSortThreads / 32][256];
  uint32_t local_start[256];
  uint32_t global_start[256];
  uint32_t scan[kSortThreads / 32];
  uint32_t tile;
};

__global__ void __launch_bounds__(kSortThreads) onesweep_kernel(const uint32_t* __restrict__ keys_in,
                                                                const uint32_t* __restrict__ vals_in,
                                                                uint32_t* __restrict__ keys_out,
                                                                uint32_t* __restrict__ vals_out,
                                                                const uint32_t* n_dev, int n_max, int shift,
                                                                const uint32_t* __restrict__ digit_counts,
                                                                uint32_t* __restrict__ lookback,
                                                                uint32_t* __restrict__ tile_counter) {
  constexpr int W = kSortThreads / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OnesweepSmem& sm = *reinterpret_cast<OnesweepSmem*>(smem_raw);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = load_n(n_dev, n_max);
  if (tid == 0) sm.tile = atomicAdd(tile_counter, 1u);
  for (int j = tid; j < W * 256; j += kSortThreads) (&sm.warp_hist[0][0])[j] = 0;
  __syncthreads();
  const uint32_t tile = sm.tile;
  const int base = static_cast<int>(tile) * kSortTile;
  if (base >= n) return;  // surplus CTA (count known only on device)
  const int warp_base = base + warp * (32 * kSortItems);

  uint32_t k[kSortItems], v[kSortItems], rank[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int idx = warp_base + i * 32 + lane;
    const bool valid = idx < n;
    k[i] = valid ? __ldg(keys_in + idx) : 0xFFFFFFFFu;
    v[i] = valid ? __ldg(vals_in + idx) : 0u;
  }
  // this pass's global digit offsets: exclusive scan of the pass histogram (every CTA
  // computes it; 256 values)
  const uint32_t dcount = tid < 256 ? __ldg(digit_counts + tid) : 0u;
  uint32_t* wh = sm.warp_hist[warp];
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
  if (tid < 256) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t c = sm.warp_hist[w][tid];
      sm.warp_hist[w][tid] = total;
      total += c;
    }
  }
  // Publish this tile's aggregate for digit tid, then look back ([tile][digit] layout: a
  // warp's 32 digits of one predecessor are one 128-byte line).
  uint32_t prefix = 0;
  if (tid < 256) {
    uint32_t* mine = lookback + static_cast<size_t>(tile) * 256 + tid;
    if (tile == 0) {
      st_volatile(mine, (total << 2) | kFlagInc);
    } else {
      st_volatile(mine, (total << 2) | kFlagAgg);
      prefix = look_back(lookback + tid, 256, static_cast<int>(tile));
      st_volatile(mine, ((prefix + total) << 2) | kFlagInc);
    }
  }
  const uint32_t goff = block_exclusive_scan<kSortThreads>(dcount, sm.scan, nullptr);
  if (tid < 256) sm.global_start[tid] = goff + prefix;
  __syncthreads();
  const uint32_t lstart = block_exclusive_scan<kSortThreads>(total, sm.scan, nullptr);
  if (tid < 256) sm.local_start[tid] = lstart;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const bool valid = (warp_base + i * 32 + lane) < n;
    if (valid) {
      const uint32_t d = (k[i] >> shift) & 255u;
      const uint32_t pos = sm.local_start[d] + sm.warp_hist[warp][d] + rank[i];
      sm.keys[pos] = k[i];
      sm.vals[pos] = v[i];
    }
  }
  __syncthreads();
  const int n_tile = min(kSortTile, n - base);
  for (int p = tid; p < n_tile; p += kSortThreads) {
    const uint32_t key = sm.keys[p];
    const uint32_t d = (key >> shift) & 255u;
    const uint32_t gi = sm.global_start[d] + (static_cast<uint32_t>(p) - sm.local_start[d]);
    keys_out[gi] = key;
    vals_out[gi] = sm.vals[p];
  }
}

// ---- single-pass scans (chained, decoupled look-back) ----
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

enum ScanMode { kCompact = 0, kRank = 1, kPlain = 2 };

struct ScanArgs {
  const uint32_t* touched;
  const uint32_t* perm;       // kRank
  const uint32_t* depth_key;  // kCompact
  uint32_t* keys_out;         // kCompact
  uint32_t* vals_out;         // kCompact
  uint32_t* offsets;          // kRank / kPlain
  uint32_t* rank;             // kRank
  const uint32_t* n_dev;
  int n_max;
  uint32_t* status;           // one word per tile, zeroed
  uint32_t* counter;          // tile counter, zeroed
  uint32_t* total_out;
  uint32_t* hist;             // kCompact: 4 x 256 digit counts of the compacted keys (zeroed)
};

template <int MODE>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(ScanArgs a) {
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t s_warp[kScanThreads / 32];
  __shared__ uint32_t s_hist[MODE == kCompact ? 4 * 256 : 1];
  if (MODE == kCompact)
    for (int j = threadIdx.x; j < 4 * 256; j += kScanThreads) s_hist[j] = 0;
  const int n = load_n(a.n_dev, a.n_max);
  if (threadIdx.x == 0) s_tile = atomicAdd(a.counter, 1u);
  __syncthreads();
  const int tile = static_cast<int>(s_tile);
  const int r0 = tile * kScanTile;
  if (r0 >= n && !(tile == 0 && n == 0)) return;
  // thread-contiguous items: r = r0 + threadIdx.x * kScanItems + i
  const int rt = r0 + threadIdx.x * kScanItems;
  uint32_t c[kScanItems], g[kScanItems];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int r = rt + i;
    g[i] = 0;
    c[i] = 0;
    if (r < n) {
      if (MODE == kRank) {
        g[i] = __ldg(a.perm + r);
        c[i] = __ldg(a.touched + g[i]);
      } else if (MODE == kCompact) {
        c[i] = __ldg(a.touched + r) > 0 ? 1u : 0u;
      } else {
        c[i] = __ldg(a.touched + r);
      }
    }
  }
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) sum += c[i];
  uint32_t tot;
  const uint32_t ex_t = block_exclusive_scan<kScanThreads>(sum, s_warp, &tot);
  if (threadIdx.x == 0) {
    uint32_t prefix = 0;
    if (tile == 0) {
      st_volatile(a.status, (tot << 2) | kFlagInc);
    } else {
      st_volatile(a.status + tile, (tot << 2) | kFlagAgg);
      prefix = look_back(a.status, 1, tile);
      st_volatile(a.status + tile, ((prefix + tot) << 2) | kFlagInc);
    }
    s_prefix = prefix;
    if (r0 + kScanTile >= n) *a.total_out = prefix + tot;
  }
  __syncthreads();
  uint32_t pos = s_prefix + ex_t;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int r = rt + i;
    if (r < n) {
      if (MODE == kCompact) {
        if (c[i]) {
          const uint32_t key = __ldg(a.depth_key + r);
          a.keys_out[pos] = key;
          a.vals_out[pos] = static_cast<uint32_t>(r);
#pragma unroll
          for (int p = 0; p < 4; ++p) atomicAdd(&s_hist[p * 256 + ((key >> (8 * p)) & 255u)], 1u);
        }
      } else {
        a.offsets[r] = pos;
        if (MODE == kRank) a.rank[g[i]] = static_cast<uint32_t>(r);
      }
    }
    pos += c[i];
  }
  if (MODE == kCompact) {
    __syncthreads();
    for (int j = threadIdx.x; j < 4 * 256; j += kScanThreads)
      if (s_hist[j]) atomicAdd(&a.hist[j], s_hist[j]);
  }
}

__global__ void __launch_bounds__(256) duplicate_kernel(const uint32_t* __restrict__ perm,
                                                        const uint32_t* __restrict__ offsets,
                                                        const uint32_t* __restrict__ touched,
                                                        const ushort4* __restrict__ rect, int tiles_x,
                                                        uint32_t* __restrict__ tile_keys,
                                                        uint32_t* __restrict__ emit_vals,
                                                        uint32_t* __restrict__ emit_gauss, const uint32_t* n_dev,
                                                        int n_max, uint32_t* __restrict__ hist, int passes) {
  __shared__ uint32_t s_hist[2 * 256];
  for (int j = threadIdx.x; j < 2 * 256; j += blockDim.x) s_hist[j] = 0;
  __syncthreads();
  const int n = load_n(n_dev, n_max);
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) {
    const uint32_t g = __ldg(perm + r);
    if (__ldg(touched + g) != 0) {
      const ushort4 b = rect[g];
      uint32_t e = __ldg(offsets + r);
      for (int ty = b.z; ty <= b.w; ++ty)
        for (int tx = b.x; tx <= b.y; ++tx) {
          const uint32_t t = static_cast<uint32_t>(ty * tiles_x + tx);
          tile_keys[e] = t;
          emit_vals[e] = e;
          emit_gauss[e] = g;
          ++e;
          atomicAdd(&s_hist[t & 255u], 1u);
          if (passes > 1) atomicAdd(&s_hist[256 + ((t >> 8) & 255u)], 1u);
        }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < passes * 256; j += blockDim.x)
    if (s_hist[j]) atomicAdd(&hist[j], s_hist[j]);
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

int launch_scan(int mode, ScanArgs a, cudaStream_t st) {
  const int tiles = max(1, div_up(a.n_max, kScanTile));
  cudaMemsetAsync(a.status, 0, sizeof(uint32_t) * (tiles + 1), st);
  cudaMemsetAsync(a.counter, 0, sizeof(uint32_t), st);
  if (mode == kCompact) scan_kernel<kCompact><<<tiles, kScanThreads, 0, st>>>(a);
  else if (mode == kRank) scan_kernel<kRank><<<tiles, kScanThreads, 0, st>>>(a);
  else scan_kernel<kPlain><<<tiles, kScanThreads, 0, st>>>(a);
  return 1;
}

}  // namespace

size_t scan_status_words(int n_max) { return static_cast<size_t>(max(1, div_up(n_max, kScanTile))) + 2; }

SortResult radix_sort_pairs(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_a, uint32_t* vals_a,
                            uint32_t* keys_b, uint32_t* vals_b, const uint32_t* n_dev, int n_max, int passes,
                            const SortScratch& s, bool hist_ready, cudaStream_t st) {
  SortResult r{const_cast<uint32_t*>(keys_in), const_cast<uint32_t*>(vals_in), 0};
  if (n_max <= 0 || passes <= 0) return r;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(onesweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(OnesweepSmem));
    configured = true;
  }
  const int tiles = div_up(n_max, kSortTile);
  cudaMemsetAsync(s.lookback, 0, sizeof(uint32_t) * 256 * static_cast<size_t>(tiles) * passes, st);
  cudaMemsetAsync(s.counters, 0, sizeof(uint32_t) * passes, st);
  if (!hist_ready) {
    cudaMemsetAsync(s.hist, 0, sizeof(uint32_t) * 256 * passes, st);
    const int hist_grid = max(1, min(div_up(n_max, 256 * 16), 148 * 4));
    switch (passes) {
      case 1: radix_hist_kernel<1><<<hist_grid, 256, 0, st>>>(keys_in, n_dev, n_max, s.hist); break;
      case 2: radix_hist_kernel<2><<<hist_grid, 256, 0, st>>>(keys_in, n_dev, n_max, s.hist); break;
      case 3: radix_hist_kernel<3><<<hist_grid, 256, 0, st>>>(keys_in, n_dev, n_max, s.hist); break;
      default: radix_hist_kernel<4><<<hist_grid, 256, 0, st>>>(keys_in, n_dev, n_max, s.hist); break;
    }
    r.launches += 1;
  }
  r.launches += passes;
  const uint32_t *ki = keys_in, *vi = vals_in;
  for (int p = 0; p < passes; ++p) {
    uint32_t* ko = (p & 1) ? keys_a : keys_b;
    uint32_t* vo = (p & 1) ? vals_a : vals_b;
    onesweep_kernel<<<tiles, kSortThreads, sizeof(OnesweepSmem), st>>>(
        ki, vi, ko, vo, n_dev, n_max, 8 * p, s.hist + 256 * p, s.lookback + static_cast<size_t>(256) * tiles * p,
        s.counters + p);
    ki = ko;
    vi = vo;
    r.keys = ko;
    r.vals = vo;
  }
  return r;
}

int compact_visible(const uint32_t* touched, const uint32_t* depth_key, uint32_t* keys_out, uint32_t* vals_out,
                    uint32_t* count_out, int n, uint32_t* status, uint32_t* counter, uint32_t* hist,
                    cudaStream_t st) {
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 256 * 4, st);
  ScanArgs a{};
  a.hist = hist;
  a.touched = touched;
  a.depth_key = depth_key;
  a.keys_out = keys_out;
  a.vals_out = vals_out;
  a.n_dev = nullptr;
  a.n_max = n;
  a.status = status;
  a.counter = counter;
  a.total_out = count_out;
  return launch_scan(kCompact, a, st);
}

int rank_scan(const uint32_t* perm, const uint32_t* touched, uint32_t* offsets, uint32_t* rank,
              const uint32_t* n_dev, int n_max, uint32_t* total_out, uint32_t* status, uint32_t* counter,
              cudaStream_t st) {
  ScanArgs a{};
  a.touched = touched;
  a.perm = perm;
  a.offsets = offsets;
  a.rank = rank;
  a.n_dev = n_dev;
  a.n_max = n_max;
  a.status = status;
  a.counter = counter;
  a.total_out = total_out;
  return launch_scan(kRank, a, st);
}

int duplicate(const uint32_t* perm, const uint32_t* offsets, const uint32_t* touched, const ushort4* rect, int tiles_x,
              uint32_t* tile_keys, uint32_t* emit_vals, uint32_t* emit_gauss, const uint32_t* n_dev, int n_max,
              uint32_t* hist, int passes, cudaStream_t st) {
  if (n_max <= 0) return 0;
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 256 * passes, st);
  duplicate_kernel<<<div_up(n_max, 256), 256, 0, st>>>(perm, offsets, touched, rect, tiles_x, tile_keys, emit_vals,
                                                       emit_gauss, n_dev, n_max, hist, passes);
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
                             int n, uint32_t* scratch_offsets, uint32_t* status, uint32_t* counter, uint32_t* total,
                             uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss, cudaStream_t st) {
  if (n <= 0) return;
  ScanArgs a{};
  a.touched = touched;
  a.offsets = scratch_offsets;
  a.n_max = n;
  a.status = status;
  a.counter = counter;
  a.total_out = total;
  launch_scan(kPlain, a, st);
  debug_keys_kernel<<<div_up(n, 256), 256, 0, st>>>(scratch_offsets, touched, rect, depth_key, tiles_x, key_tile,
                                                    key_depth, key_gauss, n);
}

}  // namespace fgs
