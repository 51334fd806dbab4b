// binning.cu — K2: intersection scan, tile ranges, key duplication and per-tile sort.
//
// Ordering contract (reference inc/splatting.hpp:192-249): the per-tile
// lists are sorted by (tile id, depth key bits, source index). The reference duplicates keys
// in source order and runs two stable LSD sorts over all I intersections (depth, then tile).
// Here no global sort runs at all; the same order is produced tile-locally:
//
//   K1 (preprocess.cu) also adds each kept Gaussian's tile rectangle into a row-difference
//      array over the tile grid (+1 at (ty, tx0), -1 at (ty, tx1 + 1) for each of its rows);
//   K2a bin_scan_kernel (persistent cooperative, one grid barrier): exclusive scan of the
//      per-Gaussian tile counts in source order -> emission offset of every tile-touching
//      Gaussian (compacted list), the intersection count I; then CTA 0 turns the row-difference
//      array into per-tile counts, the tile ranges (offsets[0..T]) and the blend schedule;
//   [host reads I (16 bytes) to size the per-intersection buffers]
//   K2b bin_scatter_kernel: each intersection (Gaussian g, tile t, emission slot e) claims a
//      slot in tile t's range with one atomicAdd and writes the 64-bit key (depth_key << 32 | e);
//   K2c tile_sort_kernel: one CTA per tile sorts its keys (bitonic, in shared memory up to 4096
//      entries, a chunked global/shared hybrid beyond) and writes the sorted Gaussian list.
//
// Emission slots e are assigned in source order (Gaussian-major, tiles ascending within a
// Gaussian), so among the entries of one tile e increases with the source index: sorting by
// (depth_key, e) is sorting by (depth_key, source index) -- the reference's order, bit-exact,
// whatever order the atomics handed out the slots in.

#include <cooperative_groups.h>

#include "fgs_kernels.h"

namespace cg = cooperative_groups;

namespace fgs {

namespace {

constexpr int kT = kBinThreads;       // threads per persistent CTA
constexpr int kW = kBinThreads / 32;  // warps per persistent CTA
constexpr int kItems = 8;             // items per thread per sub-tile (thread-contiguous)
constexpr int kSortThreads = 256;     // tile sort CTA
constexpr int kSortCap = 4096;        // keys sorted entirely in shared memory
constexpr int kScatterThreads = 512;  // scatter CTA
constexpr int kScatterSlots = 4096;   // emission slots per scatter CTA
constexpr int kSchedBuckets = 18;     // blend schedule: log2 list-length buckets
constexpr int kPrivTiles = 16384;     // scatter: per-CTA shared tile counters up to this many tiles

struct ScanSmem {
  uint32_t warp_tmp[kW];
  uint32_t warp_tmp2[kW];
  uint32_t hist[32];
  uint32_t run[32];
  uint32_t scalar[4];
};

// Block-wide exclusive scan of one value per thread (kT threads).
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
    uint32_t w = lane < kW ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kW) s_warp[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const uint32_t warp_prefix = warp ? s_warp[warp - 1] : 0u;
  const uint32_t t = s_warp[kW - 1];
  __syncthreads();  // s_warp may be reused right after
  if (total) *total = t;
  return warp_prefix + x - v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void chunk_of(int m, int& lo, int& hi) {
  lo = static_cast<int>(static_cast<int64_t>(m) * blockIdx.x / gridDim.x);
  hi = static_cast<int>(static_cast<int64_t>(m) * (blockIdx.x + 1) / gridDim.x);
}

// Sum over CTAs c' < blockIdx.x (prefix) and over all CTAs (total) of part[stride * c'].
__device__ __forceinline__ void cta_prefix(const uint32_t* part, int stride, uint32_t* s_warp, uint32_t& prefix,
                                           uint32_t& total) {
  uint32_t p = 0, t = 0;
  for (int c = threadIdx.x; c < static_cast<int>(gridDim.x); c += kT) {
    const uint32_t v = part[stride * c];
    t += v;
    if (c < static_cast<int>(blockIdx.x)) p += v;
  }
  uint32_t pt, tt;
  block_exclusive_scan(p, s_warp, &pt);
  block_exclusive_scan(t, s_warp, &tt);
  prefix = pt;
  total = tt;
}

__device__ __forceinline__ int sched_bucket(uint32_t c) {
  return c == 0 ? kSchedBuckets - 1 : 16 - min(16, 31 - __clz(c));
}

// K2a. Phase A1/A2 over all CTAs, phase A3 on CTA 0.
__global__ void __launch_bounds__(kT, 1) bin_scan_kernel(BinArgs a) {
  __shared__ ScanSmem sm;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  int lo, hi;
  chunk_of(a.n, lo, hi);
  // ---- A1: this CTA's number of tile-touching Gaussians and their tile total ----
  {
    uint32_t c1 = 0, c2 = 0;
    for (int i = lo + tid; i < hi; i += kT) {
      const uint32_t t = a.touched[i];
      c1 += t > 0 ? 1u : 0u;
      c2 += t;
    }
    uint32_t t1, t2;
    block_exclusive_scan(c1, sm.warp_tmp, &t1);
    block_exclusive_scan(c2, sm.warp_tmp2, &t2);
    if (tid == 0) {
      a.part_scan[2 * blockIdx.x] = t1;
      a.part_scan[2 * blockIdx.x + 1] = t2;
    }
  }
  grid.sync();
  // ---- A2: compaction (source order) with emission offsets ----
  {
    uint32_t p1, tot1, p2, tot2;
    cta_prefix(a.part_scan, 2, sm.warp_tmp, p1, tot1);
    cta_prefix(a.part_scan + 1, 2, sm.warp_tmp, p2, tot2);
    if (blockIdx.x == 0 && tid == 0) {
      a.scalars[kScalarM] = tot1;
      a.scalars[kScalarI] = tot2;
    }
    uint32_t run1 = p1, run2 = p2;
    for (int sb = lo; sb < hi; sb += kT * kItems) {
      const int r0 = sb + tid * kItems;
      uint32_t c[kItems], s1 = 0, s2 = 0;
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        c[i] = r0 + i < hi ? a.touched[r0 + i] : 0u;
        s1 += c[i] > 0 ? 1u : 0u;
        s2 += c[i];
      }
      uint32_t t1, t2;
      uint32_t pos = run1 + block_exclusive_scan(s1, sm.warp_tmp, &t1);
      uint32_t off = run2 + block_exclusive_scan(s2, sm.warp_tmp2, &t2);
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        if (c[i]) {
          a.cval[pos] = static_cast<uint32_t>(r0 + i);
          a.coff[pos] = off;
          ++pos;
          off += c[i];
        }
      }
      run1 += t1;
      run2 += t2;
    }
  }
  if (blockIdx.x != 0) return;
  __syncthreads();
  // ---- A3 (CTA 0): row-difference array -> per-tile counts -> tile ranges + schedule ----
  // rowdiff is (tiles_y) x (tiles_x + 1), row-major; every +1 of a row has its -1 in the same
  // row, so one running inclusive sum over the flattened array gives the count of every
  // (row, column < tiles_x) cell. The array is zeroed as it is read (ready for the next frame).
  const int rw = a.tiles_x + 1;
  const int nd = rw * a.tiles_y;
  const int lane = tid & 31;
  const uint32_t lt = lanemask_lt();
  const bool single = nd <= kT * kItems;  // one pass: the counts stay in registers
  if (tid < 32) sm.hist[tid] = 0;
  uint32_t carry_d = 0, carry_o = 0;
  uint32_t cnt[kItems];
  int cell_tile[kItems];
  for (int sb = 0; sb < nd; sb += kT * kItems) {
    const int d0 = sb + tid * kItems;
    int32_t v[kItems];
    int32_t s = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      v[i] = d0 + i < nd ? a.rowdiff[d0 + i] : 0;
      s += v[i];
    }
#pragma unroll
    for (int i = 0; i < kItems; ++i)
      if (d0 + i < nd && v[i]) a.rowdiff[d0 + i] = 0;
    uint32_t td;
    uint32_t run = carry_d + block_exclusive_scan(static_cast<uint32_t>(s), sm.warp_tmp, &td);
    uint32_t cs = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int d = d0 + i;
      run += static_cast<uint32_t>(v[i]);
      const bool cell = d < nd && d % rw < a.tiles_x;
      cnt[i] = cell ? run : 0u;
      cell_tile[i] = cell ? (d / rw) * a.tiles_x + d % rw : -1;
      cs += cnt[i];
    }
    uint32_t to;
    uint32_t off = carry_o + block_exclusive_scan(cs, sm.warp_tmp2, &to);
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int t = cell_tile[i];
      if (t >= 0) {
        a.tile_offsets[t] = off;
        a.fill[t] = off;
        off += cnt[i];
      }
      // schedule histogram, warp-aggregated (bucket 31 = no cell)
      const int b = t >= 0 ? sched_bucket(cnt[i]) : 31;
      const uint32_t peers = __match_any_sync(0xffffffffu, b);
      if (b != 31 && (peers & lt) == 0) atomicAdd(&sm.hist[b], __popc(peers));
    }
    carry_d += td;
    carry_o += to;
  }
  __syncthreads();
  if (tid == 0) {
    a.tile_offsets[a.num_tiles] = carry_o;
    a.scalars[kScalarI2] = carry_o;
    // blend schedule: tiles by descending list length (log2 buckets), empty tiles last.
    // The first `big` entries (lists of >= 256 keys) are CTA-sorted by K2c.
    uint32_t r = 0, big = 0;
    for (int b = 0; b < kSchedBuckets; ++b) {
      const uint32_t c = sm.hist[b];
      if (16 - b >= 8) big += c;
      sm.run[b] = r;
      r += c;
    }
    a.scalars[kScalarBig] = big;
  }
  __syncthreads();
  if (single) {
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int t = cell_tile[i];
      const int b = t >= 0 ? sched_bucket(cnt[i]) : 31;
      const uint32_t peers = __match_any_sync(0xffffffffu, b);
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (b != 31 && lane == leader) base = atomicAdd(&sm.run[b], __popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (t >= 0) a.tile_order[base + __popc(peers & lt)] = static_cast<uint32_t>(t);
    }
  } else {
    for (int t = tid; t < a.num_tiles; t += kT) {
      const uint32_t c = a.tile_offsets[t + 1] - a.tile_offsets[t];
      a.tile_order[atomicAdd(&sm.run[sched_bucket(c)], 1u)] = static_cast<uint32_t>(t);
    }
  }
}

// Largest r in [0, m) with offs[r] <= v (offs ascending, offs[0] = 0): repeated
// blockDim-ary search by the whole CTA.
__device__ int cta_upper_rank(const uint32_t* offs, int m, uint32_t v, uint32_t* s_res) {
  const int tid = threadIdx.x, nt = blockDim.x;
  int base = 0, range = m;
  while (true) {
    const int step = (range + nt - 1) / nt;
    if (tid == 0) *s_res = static_cast<uint32_t>(base);
    __syncthreads();
    const int r = base + tid * step;
    if (tid * step < range && offs[r] <= v) atomicMax(s_res, static_cast<uint32_t>(r));
    __syncthreads();
    const int nb = static_cast<int>(*s_res);
    __syncthreads();
    if (step == 1) return nb;
    base = nb;
    range = min(step, m - nb);
  }
}

// K2b. CTA c handles emission slots [kScatterSlots * c, +kScatterSlots), one slot per thread
// per step (so a Gaussian covering thousands of tiles is spread over the whole grid). The
// CTA's Gaussian range comes from a CTA search over the compacted emission offsets; the
// offsets of that range are staged in shared memory and every slot finds its Gaussian there
// by binary search. Positions in a tile's range are claimed in two levels (PRIV): the CTA
// counts its slots per tile with shared-memory atomics, then one global atomicAdd per
// (CTA, tile) reserves the block -- heavy tiles see one global atomic per CTA instead of one
// per intersection. All loads and atomics of a thread's slots are issued before use.
template <bool PRIV>
__global__ void __launch_bounds__(kScatterThreads) bin_scatter_kernel(BinArgs a) {
  extern __shared__ uint32_t s_cnt[];  // [num_tiles] (PRIV)
  __shared__ uint32_t s_res;
  __shared__ uint32_t s_off[kScatterSlots];
  constexpr int U = kScatterSlots / kScatterThreads;
  const int tid = threadIdx.x;
  const uint32_t I = a.scalars[kScalarI];
  if (I > a.isect_cap) return;  // speculative launch with too small buffers: the host relaunches
  const int m = static_cast<int>(a.scalars[kScalarM]);
  const uint32_t lo = blockIdx.x * kScatterSlots, hi = min(I, lo + kScatterSlots);
  if (lo >= hi) return;
  if (PRIV)
    for (int t = tid; t < a.num_tiles; t += kScatterThreads) s_cnt[t] = 0;
  const int r_lo = cta_upper_rank(a.coff, m, lo, &s_res);
  const int r_hi = cta_upper_rank(a.coff, m, hi - 1, &s_res);
  const int nr = r_hi - r_lo + 1;  // <= kScatterSlots: every Gaussian here owns >= 1 slot
  for (int i = tid; i < nr; i += kScatterThreads) s_off[i] = a.coff[r_lo + i];
  __syncthreads();
  uint32_t ev[U], gv[U], tv[U], pv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    ev[u] = lo + u * kScatterThreads + tid;
    int l = 0, h = nr - 1;
    while (l < h) {
      const int mid = (l + h + 1) >> 1;
      if (s_off[mid] <= ev[u]) l = mid;
      else h = mid - 1;
    }
    tv[u] = static_cast<uint32_t>(l);  // local rank for now
  }
#pragma unroll
  for (int u = 0; u < U; ++u) gv[u] = ev[u] < hi ? a.cval[r_lo + tv[u]] : 0u;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (ev[u] >= hi) continue;
    const ushort4 rc = a.rect[gv[u]];
    const int wx = rc.y - rc.x + 1;
    const int j = static_cast<int>(ev[u] - s_off[tv[u]]);
    tv[u] = static_cast<uint32_t>((rc.z + j / wx) * a.tiles_x + rc.x + j % wx);
  }
  if (PRIV) {
#pragma unroll
    for (int u = 0; u < U; ++u) pv[u] = ev[u] < hi ? atomicAdd(s_cnt + tv[u], 1u) : 1u;
    __syncthreads();
    // the slot that took local position 0 reserves the CTA's block of tile tv[u]
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (pv[u] == 0) s_cnt[tv[u]] = atomicAdd(a.fill + tv[u], s_cnt[tv[u]]);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ev[u] < hi) pv[u] += s_cnt[tv[u]];
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u) pv[u] = ev[u] < hi ? atomicAdd(a.fill + tv[u], 1u) : 0u;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (ev[u] >= hi) continue;
    a.keys[pv[u]] = (static_cast<uint64_t>(a.depth_key[gv[u]]) << 32) | ev[u];
    a.emit_gauss[ev[u]] = gv[u];
  }
}

// ---- bitonic sort, ascending comparators only ----
// Stage (k, j): for j == k/2 the partner of index i is its mirror in the k-block (i ^ (k - 1)),
// otherwise i ^ j; the smaller key goes to the lower index. Pads (index >= L) hold +inf and
// never move, so the global variant never has to materialise them.
//
// Register form (one warp, 32*E keys, "striped": key i = r*32 + lane lives in register r of
// lane `lane`): partners with j < 32 are in another lane (shuffles), partners with j >= 32 in
// another register of the same lane.

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
  uint64_t y[E];
#pragma unroll
  for (int r = 0; r < E; ++r) y[r] = __shfl_xor_sync(0xffffffffu, x[r ^ RM], 31);
#pragma unroll
  for (int r = 0; r < E; ++r) x[r] = (r & RB) == 0 ? kmin(x[r], y[r]) : kmax(x[r], y[r]);
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
constexpr int kSortWarps = kSortThreads / 32;

// Register phase over the shared array s[0, n) (n a multiple of kChunk): every warp loads its
// 256-key chunks, runs a full sort (first) or the half-cleaner stages j < 256 of a merge level,
// and stores them back. Callers barrier before and after.
template <bool kFull>
__device__ __forceinline__ void chunk_phase(uint64_t* s, int n) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp * kChunk; c < n; c += kSortWarps * kChunk) {
    uint64_t x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) x[r] = s[c + r * 32 + lane];
    if (kFull) warp_sort<8>(x, lane);
    else warp_halfclean<8>(x, lane);
#pragma unroll
    for (int r = 0; r < 8; ++r) s[c + r * 32 + lane] = x[r];
  }
}

// Ascending sort of s[0, n), n a power of two in [kChunk, kSortCap], by the whole CTA.
__device__ void cta_sort(uint64_t* s, int n) {
  __syncthreads();
  chunk_phase<true>(s, n);
  for (int k = 2 * kChunk; k <= n; k <<= 1) {
    for (int j = k >> 1; j >= kChunk; j >>= 1) {
      __syncthreads();
      for (int c = threadIdx.x; c < (n >> 1); c += kSortThreads) {
        int i, p;
        ce_index(c, k, j, i, p);
        ce(s, i, p);
      }
    }
    __syncthreads();
    chunk_phase<false>(s, n);
  }
  __syncthreads();
}

// Stages j = C/2 .. 1 of a merge level k > C on the shared chunk s[0, C) (C = kSortCap).
__device__ void cta_halfclean(uint64_t* s) {
  for (int j = kSortCap >> 1; j >= kChunk; j >>= 1) {
    __syncthreads();
    for (int c = threadIdx.x; c < (kSortCap >> 1); c += kSortThreads) {
      const int i = 2 * c - (c & (j - 1));
      ce(s, i, i + j);
    }
  }
  __syncthreads();
  chunk_phase<false>(s, kSortCap);
  __syncthreads();
}

__device__ __forceinline__ int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Output of one sorted entry at position pos: Gaussian id, emission slot -> position map,
// optionally the record in sorted order.
__device__ __forceinline__ void emit_sorted(const BinArgs& a, uint32_t pos, uint64_t key) {
  const uint32_t e = static_cast<uint32_t>(key);
  const uint32_t gi = a.emit_gauss[e];
  a.emit_pos[e] = pos;
  a.sorted_gauss[pos] = gi;
  if (a.sorted_rec) a.sorted_rec[pos] = a.rec[gi];
}

// Tiles with <= 32*E keys: one warp, registers only.
template <int E>
__device__ __forceinline__ void warp_tile_sort(const BinArgs& a, uint32_t lo, int L, int lane) {
  uint64_t x[E];
  const uint64_t* g = a.keys + lo;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int i = r * 32 + lane;
    x[r] = i < L ? g[i] : ~0ull;
  }
  warp_sort<E>(x, lane);
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int i = r * 32 + lane;
    if (i < L) emit_sorted(a, lo + i, x[r]);
  }
}

// K2c. The blend schedule lists tiles by descending list length; its first n_big entries
// (lists > 256 keys, counted by K2a) get one CTA each, sorted in shared memory (registers for
// the stages inside 256-key chunks); the remaining tiles get one warp each, registers only.
__global__ void __launch_bounds__(kSortThreads) tile_sort_kernel(BinArgs a) {
  __shared__ uint64_t s[kSortCap];
  if (a.scalars[kScalarI] > a.isect_cap) return;  // speculative launch with too small buffers
  const int n_big = static_cast<int>(a.scalars[kScalarBig]);
  const int tid = threadIdx.x;
  if (static_cast<int>(blockIdx.x) >= n_big) {
    const int idx = n_big + (static_cast<int>(blockIdx.x) - n_big) * kSortWarps + (tid >> 5);
    if (idx >= a.num_tiles) return;
    const int tile = static_cast<int>(a.tile_order[idx]);
    const uint32_t lo = a.tile_offsets[tile];
    const int L = static_cast<int>(a.tile_offsets[tile + 1] - lo);
    const int lane = tid & 31;
    if (L <= 0) return;
    if (L <= 32) warp_tile_sort<1>(a, lo, L, lane);
    else if (L <= 64) warp_tile_sort<2>(a, lo, L, lane);
    else if (L <= 128) warp_tile_sort<4>(a, lo, L, lane);
    else warp_tile_sort<8>(a, lo, L, lane);
    return;
  }
  const int tile = static_cast<int>(a.tile_order[blockIdx.x]);
  const uint32_t lo = a.tile_offsets[tile], hi = a.tile_offsets[tile + 1];
  const int L = static_cast<int>(hi - lo);
  uint64_t* g = a.keys + lo;
  const int P = pow2_ceil(L);
  if (P <= kSortCap) {
    for (int k = tid; k < P; k += kSortThreads) s[k] = k < L ? g[k] : ~0ull;
    cta_sort(s, P);
    for (int k = tid; k < L; k += kSortThreads) emit_sorted(a, lo + k, s[k]);
    return;
  }
  // Long list: sort kSortCap-chunks in shared memory, then for every larger k run the stages
  // with j >= kSortCap on global memory and finish each chunk's j < kSortCap stages in
  // shared memory.
  constexpr int C = kSortCap;
  for (int c0 = 0; c0 < L; c0 += C) {
    __syncthreads();
    for (int k = tid; k < C; k += kSortThreads) s[k] = c0 + k < L ? g[c0 + k] : ~0ull;
    cta_sort(s, C);
    for (int k = tid; k < C && c0 + k < L; k += kSortThreads) g[c0 + k] = s[k];
  }
  for (int k = 2 * C; k <= P; k <<= 1) {
    for (int j = k >> 1; j >= C; j >>= 1) {
      __syncthreads();
      for (int c = tid; c < (P >> 1); c += kSortThreads) {
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
      for (int q = tid; q < C; q += kSortThreads) s[q] = c0 + q < L ? g[c0 + q] : ~0ull;
      cta_halfclean(s);
      for (int q = tid; q < C && c0 + q < L; q += kSortThreads) g[c0 + q] = s[q];
    }
  }
  __syncthreads();
  for (int k = tid; k < L; k += kSortThreads) emit_sorted(a, lo + k, g[k]);
}

// Debug export: the reference's pre-sort key list (source order, ty-major, tx-minor).
__global__ void __launch_bounds__(kT, 1) debug_keys_kernel(BinArgs a, uint32_t* key_tile, uint32_t* key_depth,
                                                           uint32_t* key_gauss) {
  const int m = static_cast<int>(a.scalars[kScalarM]);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    const uint32_t g = a.cval[r];
    uint32_t e = a.coff[r];
    const ushort4 b = a.rect[g];
    for (int ty = b.z; ty <= b.w; ++ty)
      for (int tx = b.x; tx <= b.y; ++tx) {
        key_tile[e] = static_cast<uint32_t>(ty * a.tiles_x + tx);
        key_depth[e] = a.depth_key[g];
        key_gauss[e] = g;
        ++e;
      }
  }
}

int grid_size() {
  static int g = 0;
  if (!g) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(tile_sort_kernel),
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(bin_scatter_kernel<true>),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kPrivTiles * 4);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(bin_scatter_kernel<true>),
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bin_scan_kernel, kT, 0);
    g = sms * (per_sm > 0 ? 1 : 0);
  }
  return g;
}

}  // namespace

size_t bin_part_words() { return static_cast<size_t>(grid_size()) * 2 + 64; }

cudaError_t bin_scan(BinArgs& a, cudaStream_t st) {
  const int g = grid_size();
  if (g <= 0) return cudaErrorCooperativeLaunchTooLarge;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(bin_scan_kernel), g, kT, args, 0, st);
}

int bin_sort(BinArgs& a, int n_big, cudaStream_t st) {
  // Grid sizes from the host's bounds: the capacity (>= I when the buffers fit) and n_big
  // (or num_tiles when unknown: every CTA past the work exits at once).
  if (a.isect_cap <= 0) return 0;
  grid_size();
  const int nb = n_big >= 0 ? n_big : a.num_tiles;
  const int scatter_ctas = div_up(static_cast<int>(a.isect_cap), kScatterSlots);
  if (a.num_tiles <= kPrivTiles)
    bin_scatter_kernel<true><<<scatter_ctas, kScatterThreads, a.num_tiles * 4, st>>>(a);
  else
    bin_scatter_kernel<false><<<scatter_ctas, kScatterThreads, 0, st>>>(a);
  const int sort_ctas = n_big >= 0 ? n_big + div_up(a.num_tiles - n_big, kSortWarps) : a.num_tiles;
  (void)nb;
  tile_sort_kernel<<<sort_ctas, kSortThreads, 0, st>>>(a);
  return 2;
}

cudaError_t debug_source_order_keys(BinArgs& a, uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss,
                                    cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  debug_keys_kernel<<<div_up(a.n, kT), kT, 0, st>>>(a, key_tile, key_depth, key_gauss);
  return cudaGetLastError();
}

}  // namespace fgs
