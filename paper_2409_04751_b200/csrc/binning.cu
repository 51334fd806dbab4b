// binning.cu — K2: compaction, depth sort, depth-rank scan, key duplication, tile sort,
// tile ranges, as two persistent cooperative kernels.
//
// Ordering contract (reference inc/splatting.hpp:192-249): the per-tile
// lists are sorted by (tile id, depth key bits, source index). The reference duplicates keys
// in source order and runs two stable LSD sorts (depth, then tile). Here the same order is
// produced with less traffic:
//   compact the Gaussians that touch >= 1 tile (source order kept);
//   level 1: stable LSD radix sort of those by the 32-bit depth key (ties keep source order);
//   duplicate in depth-rank order (tiles ascending within a Gaussian);
//   level 2: stable LSD radix sort of the I intersections by the 13-bit tile id.
// Stability of both levels gives exactly (tile, depth, source).
//
// Execution model (B200-first). At the frame sizes of this path (~0.3-3M keys) every
// sort/scan phase is latency bound: measured on B200 (profiles/micro/), a back-to-back launch
// costs ~4-5 us and a decoupled look-back onesweep pass ~14-20 us when all tiles run in the
// first wave, while cooperative grid.sync() costs ~1.1 us. So all phases run inside two
// persistent kernels, one 1024-thread CTA per SM:
//   bin_level1_kernel: compaction -> 4 radix passes (8-bit digits) -> rank scan (I);
//   [host reads I (8 bytes) to size the per-intersection buffers]
//   bin_level2_kernel: duplication -> 1-2 radix passes -> tile ranges + records gathered
//   into sorted order (the blends then stream each tile's list contiguously).
// Each radix pass sweeps every CTA's contiguous chunk once for its digit histogram, resolves
// the global digit offsets across CTAs with two grid barriers (reduce-then-scan over the 148
// per-CTA histograms: each digit's column is scanned in parallel by one CTA, no look-back
// chains), then ranks keys in 8192-key sub-tiles with a
// ballot-based warp multisplit and scatters through shared memory (stable).

#include <cooperative_groups.h>

#include "fgs_kernels.h"

namespace cg = cooperative_groups;

namespace fgs {

namespace {

constexpr int kT = kBinThreads;       // threads per CTA
constexpr int kW = kBinThreads / 32;  // warps per CTA
constexpr int kItems = 8;             // keys per thread per sub-tile
constexpr int kSub = kT * kItems;     // keys per sub-tile

struct BinSmem {
  uint32_t keys[kSub];
  uint32_t vals[kSub];
  uint32_t wh[kW][256];
  uint32_t hist[256];
  uint32_t run[256];
  uint32_t local_start[256];
  uint32_t warp_tmp[kW];
  uint32_t scalar[4];
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Debug phase trace (FGS_FLAG_COUNTERS): CTA 0 records %globaltimer at phase boundaries.
__device__ __forceinline__ void trace(unsigned long long* t, int slot) {
  if (t && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    t[slot] = v;
  }
}

__device__ __forceinline__ void chunk_of(int m, int& lo, int& hi) {
  lo = static_cast<int>(static_cast<int64_t>(m) * blockIdx.x / gridDim.x);
  hi = static_cast<int>(static_cast<int64_t>(m) * (blockIdx.x + 1) / gridDim.x);
}

// Block-wide exclusive scan of one value per thread.
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

// Sum over CTAs c' < blockIdx.x (prefix) and over all CTAs (total) of part[c'].
__device__ __forceinline__ void cta_prefix(const uint32_t* part, uint32_t* s_warp, uint32_t& prefix,
                                           uint32_t& total) {
  uint32_t p = 0, t = 0;
  for (int c = threadIdx.x; c < static_cast<int>(gridDim.x); c += kT) {
    const uint32_t v = part[c];
    t += v;
    if (c < static_cast<int>(blockIdx.x)) p += v;
  }
  uint32_t pt, tt;
  block_exclusive_scan(p, s_warp, &pt);
  block_exclusive_scan(t, s_warp, &tt);
  prefix = pt;
  total = tt;
}

// One stable LSD radix pass of (kin, vin)[0, m) into (kout, vout) on digit (key >> shift) & 255.
__device__ void radix_pass(cg::grid_group& grid, BinSmem& sm, const uint32_t* __restrict__ kin,
                           const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
                           uint32_t* __restrict__ vout, int m, int shift, uint32_t* __restrict__ part,
                           unsigned long long* tr = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int lo, hi;
  chunk_of(m, lo, hi);
  // 1. digit histogram of this CTA's chunk
  if (tid < 256) sm.hist[tid] = 0;
  __syncthreads();
  for (int i = lo + tid; i < hi; i += kT) atomicAdd(&sm.hist[(kin[i] >> shift) & 255u], 1u);
  __syncthreads();
  if (tid < 256) part[blockIdx.x * 256 + tid] = sm.hist[tid];
  trace(tr, 0);
  grid.sync();
  trace(tr, 1);
  // 2. per digit, exclusive scan over CTAs: digit d is owned by CTA d mod grid, whose threads
  //    (one per CTA c) load part[c][d] in one parallel burst, scan it in place and publish the
  //    digit total. Then every CTA reads its own 256 offsets + the 256 totals (coalesced).
  uint32_t* totals = part + gridDim.x * 256;
  for (int d = blockIdx.x; d < 256; d += gridDim.x) {
    const uint32_t v = tid < static_cast<int>(gridDim.x) ? part[tid * 256 + d] : 0u;
    uint32_t t;
    const uint32_t ex = block_exclusive_scan(v, sm.warp_tmp, &t);
    if (tid < static_cast<int>(gridDim.x)) part[tid * 256 + d] = ex;
    if (tid == 0) totals[d] = t;
  }
  trace(tr, 2);
  grid.sync();
  trace(tr, 3);
  const uint32_t tot = tid < 256 ? totals[tid] : 0u;
  const uint32_t pre = tid < 256 ? part[blockIdx.x * 256 + tid] : 0u;
  const uint32_t dstart = block_exclusive_scan(tot, sm.warp_tmp, nullptr);
  if (tid < 256) sm.run[tid] = dstart + pre;
  __syncthreads();
  // 3. rank + scatter the chunk in order, one sub-tile at a time
  const uint32_t lt = lanemask_lt();
  for (int sb = lo; sb < hi; sb += kSub) {
    const int end = min(hi, sb + kSub);
    for (int j = tid; j < kW * 256; j += kT) (&sm.wh[0][0])[j] = 0;
    __syncthreads();
    const int wbase = sb + warp * (32 * kItems);
    uint32_t k[kItems], v[kItems], rk[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int idx = wbase + i * 32 + lane;
      const bool valid = idx < end;
      k[i] = valid ? kin[idx] : 0u;
      v[i] = valid ? vin[idx] : 0u;
    }
    uint32_t* wh = sm.wh[warp];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const bool valid = wbase + i * 32 + lane < end;
      const uint32_t d = (k[i] >> shift) & 255u;
      uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
      }
      uint32_t before = 0;
      if (valid) before = wh[d];
      __syncwarp();
      if (valid) {
        rk[i] = before + __popc(peers & lt);
        if ((peers & lt) == 0) wh[d] = before + __popc(peers);
      }
      __syncwarp();
    }
    __syncthreads();
    uint32_t total = 0;
    if (tid < 256) {
#pragma unroll 8
      for (int w = 0; w < kW; ++w) {
        const uint32_t c = sm.wh[w][tid];
        sm.wh[w][tid] = total;
        total += c;
      }
    }
    const uint32_t ls = block_exclusive_scan(total, sm.warp_tmp, nullptr);
    if (tid < 256) sm.local_start[tid] = ls;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      if (wbase + i * 32 + lane < end) {
        const uint32_t d = (k[i] >> shift) & 255u;
        const uint32_t pos = sm.local_start[d] + sm.wh[warp][d] + rk[i];
        sm.keys[pos] = k[i];
        sm.vals[pos] = v[i];
      }
    }
    __syncthreads();
    for (int p = tid; p < end - sb; p += kT) {
      const uint32_t key = sm.keys[p];
      const uint32_t d = (key >> shift) & 255u;
      const uint32_t gi = sm.run[d] + (static_cast<uint32_t>(p) - sm.local_start[d]);
      kout[gi] = key;
      vout[gi] = sm.vals[p];
    }
    __syncthreads();
    if (tid < 256) sm.run[tid] += total;
    __syncthreads();
  }
  trace(tr, 4);
  grid.sync();
  trace(tr, 5);
}

__global__ void __launch_bounds__(kT, 1) bin_level1_kernel(BinArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BinSmem& sm = *reinterpret_cast<BinSmem*>(smem_raw);
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  const int n = a.n;
  int lo, hi;

  trace(a.trace, 0);
  // ---- compaction of Gaussians touching >= 1 tile (source order) ----
  chunk_of(n, lo, hi);
  {
    uint32_t cnt = 0;
    for (int i = lo + tid; i < hi; i += kT) cnt += a.touched[i] > 0 ? 1u : 0u;
    uint32_t tot;
    block_exclusive_scan(cnt, sm.warp_tmp, &tot);
    if (tid == 0) a.part_scan[blockIdx.x] = tot;
  }
  grid.sync();
  {
    uint32_t prefix, total;
    cta_prefix(a.part_scan, sm.warp_tmp, prefix, total);
    if (blockIdx.x == 0 && tid == 0) a.scalars[kScalarM] = total;
    uint32_t run = prefix;
    for (int sb = lo; sb < hi; sb += kT * kItems) {
      const int r0 = sb + tid * kItems;  // thread-contiguous items keep source order
      uint32_t f[kItems], s = 0;
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        f[i] = (r0 + i < hi && a.touched[r0 + i] > 0) ? 1u : 0u;
        s += f[i];
      }
      uint32_t t;
      uint32_t pos = run + block_exclusive_scan(s, sm.warp_tmp, &t);
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        if (f[i]) {
          a.ckey[pos] = a.depth_key_in[r0 + i];
          a.cval[pos] = static_cast<uint32_t>(r0 + i);
        }
        pos += f[i];
      }
      run += t;
    }
    if (tid == 0) sm.scalar[0] = total;
  }
  grid.sync();
  const int m = static_cast<int>(sm.scalar[0]);
  trace(a.trace, 1);

  // ---- level 1: stable sort by depth key (4 x 8-bit digits): in -> a -> b -> a -> b ----
  radix_pass(grid, sm, a.ckey, a.cval, a.key_a, a.val_a, m, 0, a.part_radix);
  trace(a.trace, 2);
  radix_pass(grid, sm, a.key_a, a.val_a, a.key_b, a.val_b, m, 8, a.part_radix, a.trace ? a.trace + 16 : nullptr);
  trace(a.trace, 3);
  radix_pass(grid, sm, a.key_b, a.val_b, a.key_a, a.val_a, m, 16, a.part_radix);
  trace(a.trace, 4);
  radix_pass(grid, sm, a.key_a, a.val_a, a.key_b, a.val_b, m, 24, a.part_radix);
  trace(a.trace, 5);
  const uint32_t* perm = a.val_b;

  // ---- exclusive scan of tile counts in depth order: offsets[r], rank[perm[r]] = r, I ----
  chunk_of(m, lo, hi);
  {
    uint32_t s = 0;
    for (int r = lo + tid; r < hi; r += kT) s += a.touched[perm[r]];
    uint32_t tot;
    block_exclusive_scan(s, sm.warp_tmp, &tot);
    if (tid == 0) a.part_scan[blockIdx.x] = tot;
  }
  grid.sync();
  {
    uint32_t prefix, total;
    cta_prefix(a.part_scan, sm.warp_tmp, prefix, total);
    if (blockIdx.x == 0 && tid == 0) a.scalars[kScalarI] = total;
    trace(a.trace, 6);
    uint32_t run = prefix;
    for (int sb = lo; sb < hi; sb += kT * kItems) {
      const int r0 = sb + tid * kItems;
      uint32_t c[kItems], g[kItems], s = 0;
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        g[i] = r0 + i < hi ? perm[r0 + i] : 0u;
        c[i] = r0 + i < hi ? a.touched[g[i]] : 0u;
        s += c[i];
      }
      uint32_t t;
      uint32_t pos = run + block_exclusive_scan(s, sm.warp_tmp, &t);
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        if (r0 + i < hi) {
          a.offsets[r0 + i] = pos;
          a.rank[g[i]] = static_cast<uint32_t>(r0 + i);
        }
        pos += c[i];
      }
      run += t;
    }
  }
}

// Largest rank r in [0, m) with offsets[r] <= v (offsets ascending, offsets[0] = 0):
// two rounds of a 1024-ary search by the whole CTA.
__device__ int cta_upper_rank(const uint32_t* offsets, int m, uint32_t v, BinSmem& sm) {
  const int tid = threadIdx.x;
  if (tid == 0) sm.scalar[1] = 0;
  __syncthreads();
  // round 1: sample every step-th rank
  const int step = max(1, (m + kT - 1) / kT);
  {
    const int r = tid * step;
    if (r < m && offsets[r] <= v) atomicMax(&sm.scalar[1], static_cast<uint32_t>(r));
  }
  __syncthreads();
  const int base = static_cast<int>(sm.scalar[1]);
  __syncthreads();
  // round 2: scan [base, base + step) (step <= kT * ceil); loop for huge m
  for (int r = base + tid; r < min(m, base + step); r += kT)
    if (offsets[r] <= v) atomicMax(&sm.scalar[1], static_cast<uint32_t>(r));
  __syncthreads();
  const int res = static_cast<int>(sm.scalar[1]);
  __syncthreads();
  return res;
}

// Emit slots [e_b, e_e) of Gaussian g (slot off is its first tile; tiles ty-major, tx-minor),
// lanes lane0, lane0 + stride, ...
__device__ __forceinline__ void emit_slots(const BinArgs& a, uint32_t g, ushort4 rc, uint32_t off, uint32_t e_b,
                                           uint32_t e_e, int lane0, int stride) {
  const int wx = rc.y - rc.x + 1;
  for (uint32_t e = e_b + lane0; e < e_e; e += stride) {
    const int j = static_cast<int>(e - off);
    const int ty = rc.z + j / wx, tx = rc.x + j % wx;
    a.tkey[e] = static_cast<uint32_t>(ty * a.tiles_x + tx);
    a.emit[e] = e;
    a.emit_gauss[e] = g;
  }
}

__global__ void __launch_bounds__(kT, 1) bin_level2_kernel(BinArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BinSmem& sm = *reinterpret_cast<BinSmem*>(smem_raw);
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  const int m = static_cast<int>(a.scalars[kScalarM]);
  const int I = a.num_isect;
  const uint32_t* perm = a.val_b;
  int lo, hi;

  trace(a.trace, 8);
  // ---- duplication in depth-rank order (tiles ascending within a Gaussian) ----
  // Balanced by intersections: CTA c emits slots [I*c/G, I*(c+1)/G). Its rank range comes
  // from two 1024-ary searches over the depth-rank offsets; lanes emit their own Gaussian's
  // slots when it has <= 32 of them in range, and whole warps share the big ones (a Gaussian
  // near the camera can cover thousands of tiles).
  chunk_of(I, lo, hi);
  if (lo < hi) {
    const int r_lo = cta_upper_rank(a.offsets, m, static_cast<uint32_t>(lo), sm);
    const int r_hi = cta_upper_rank(a.offsets, m, static_cast<uint32_t>(hi - 1), sm);
    const int lane = tid & 31, warp = tid >> 5;
    for (int rb = r_lo + warp * 32; rb <= r_hi; rb += kT) {
      const int r = rb + lane;
      uint32_t g = 0, e_b = 0, e_e = 0, off = 0;
      ushort4 rc = make_ushort4(0, 0, 0, 0);
      if (r <= r_hi) {
        g = perm[r];
        off = a.offsets[r];
        rc = a.rect[g];
        const uint32_t cnt = a.touched[g];
        e_b = max(off, static_cast<uint32_t>(lo));
        e_e = min(off + cnt, static_cast<uint32_t>(hi));
      }
      const bool big = e_e > e_b + 32;
      if (!big) emit_slots(a, g, rc, off, e_b, e_e, 0, 1);
      uint32_t bigs = __ballot_sync(0xffffffffu, big);
      while (bigs) {
        const int j = __ffs(bigs) - 1;
        bigs &= bigs - 1;
        const uint32_t gj = __shfl_sync(0xffffffffu, g, j);
        const uint32_t oj = __shfl_sync(0xffffffffu, off, j);
        const uint32_t bj = __shfl_sync(0xffffffffu, e_b, j);
        const uint32_t ej = __shfl_sync(0xffffffffu, e_e, j);
        ushort4 rj;
        rj.x = __shfl_sync(0xffffffffu, rc.x, j);
        rj.y = __shfl_sync(0xffffffffu, rc.y, j);
        rj.z = __shfl_sync(0xffffffffu, rc.z, j);
        rj.w = __shfl_sync(0xffffffffu, rc.w, j);
        emit_slots(a, gj, rj, oj, bj, ej, lane, 32);
      }
    }
  }
  grid.sync();
  trace(a.trace, 9);

  // ---- level 2: stable sort by tile id ----
  const uint32_t *sk = a.tkey, *sv = a.emit;
  if (a.passes2 >= 1) {
    radix_pass(grid, sm, a.tkey, a.emit, a.tkey_a, a.emit_a, I, 0, a.part_radix);
    sk = a.tkey_a;
    sv = a.emit_a;
  }
  if (a.passes2 >= 2) {
    radix_pass(grid, sm, a.tkey_a, a.emit_a, a.tkey_b, a.emit_b, I, 8, a.part_radix);
    sk = a.tkey_b;
    sv = a.emit_b;
  }

  trace(a.trace, 10);
  // ---- per-tile ranges, sorted Gaussian list, records gathered into sorted order ----
  // 4 entries per thread per step so the dependent gathers (emission slot -> Gaussian ->
  // 48-byte record) of several entries are in flight at once.
  chunk_of(I, lo, hi);
  for (int k0 = lo + tid; k0 < hi; k0 += 4 * kT) {
    uint32_t e[4], g[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + u * kT;
      e[u] = k < hi ? sv[k] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) g[u] = k0 + u * kT < hi ? a.emit_gauss[e[u]] : 0u;
    SortedRec r[4];
    if (a.sorted_rec)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k0 + u * kT < hi) r[u] = a.rec[g[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + u * kT;
      if (k >= hi) break;
      const int t = static_cast<int>(sk[k]);
      const int tp = k > 0 ? static_cast<int>(sk[k - 1]) : -1;
      for (int tt = tp + 1; tt <= t; ++tt) a.tile_offsets[tt] = static_cast<uint32_t>(k);
      if (k == I - 1)
        for (int tt = t + 1; tt <= a.num_tiles; ++tt) a.tile_offsets[tt] = static_cast<uint32_t>(I);
      a.sorted_emit[k] = e[u];
      a.sorted_gauss[k] = g[u];
      if (a.sorted_rec) a.sorted_rec[k] = r[u];
    }
  }
  trace(a.trace, 11);
  if (a.tile_order == nullptr) return;
  grid.sync();
  trace(a.trace, 12);
  // ---- blend schedule: tiles by descending list length (log2 buckets), empty tiles last ----
  if (blockIdx.x != 0) return;
  constexpr int kB = 18;
  if (tid < kB) sm.hist[tid] = 0;
  __syncthreads();
  for (int t = tid; t < a.num_tiles; t += kT) {
    const uint32_t c = a.tile_offsets[t + 1] - a.tile_offsets[t];
    const int b = c == 0 ? kB - 1 : 16 - min(16, 31 - __clz(c));
    atomicAdd(&sm.hist[b], 1u);
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t run = 0;
    for (int b = 0; b < kB; ++b) {
      const uint32_t c = sm.hist[b];
      sm.run[b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int t = tid; t < a.num_tiles; t += kT) {
    const uint32_t c = a.tile_offsets[t + 1] - a.tile_offsets[t];
    const int b = c == 0 ? kB - 1 : 16 - min(16, 31 - __clz(c));
    a.tile_order[atomicAdd(&sm.run[b], 1u)] = static_cast<uint32_t>(t);
  }
  __syncthreads();
  trace(a.trace, 13);
}

// Debug export: the reference's pre-sort key list (source order, ty-major, tx-minor).
__global__ void __launch_bounds__(kT, 1) debug_keys_kernel(BinArgs a, uint32_t* key_tile, uint32_t* key_depth,
                                                           uint32_t* key_gauss) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BinSmem& sm = *reinterpret_cast<BinSmem*>(smem_raw);
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  int lo, hi;
  chunk_of(a.n, lo, hi);
  uint32_t s = 0;
  for (int i = lo + tid; i < hi; i += kT) s += a.touched[i];
  uint32_t tot;
  block_exclusive_scan(s, sm.warp_tmp, &tot);
  if (tid == 0) a.part_scan[blockIdx.x] = tot;
  grid.sync();
  uint32_t prefix, total;
  cta_prefix(a.part_scan, sm.warp_tmp, prefix, total);
  uint32_t run = prefix;
  for (int sb = lo; sb < hi; sb += kT * kItems) {
    const int r0 = sb + tid * kItems;
    uint32_t c[kItems], ss = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      c[i] = r0 + i < hi ? a.touched[r0 + i] : 0u;
      ss += c[i];
    }
    uint32_t t;
    uint32_t e = run + block_exclusive_scan(ss, sm.warp_tmp, &t);
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      if (c[i]) {
        const int g = r0 + i;
        const ushort4 b = a.rect[g];
        for (int ty = b.z; ty <= b.w; ++ty)
          for (int tx = b.x; tx <= b.y; ++tx) {
            key_tile[e] = static_cast<uint32_t>(ty * a.tiles_x + tx);
            key_depth[e] = a.depth_key_in[g];
            key_gauss[e] = static_cast<uint32_t>(g);
            ++e;
          }
      }
    }
    run += t;
  }
}

int grid_size() {
  static int g = 0;
  if (!g) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (auto* f : {reinterpret_cast<const void*>(bin_level1_kernel), reinterpret_cast<const void*>(bin_level2_kernel),
                    reinterpret_cast<const void*>(debug_keys_kernel)})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(BinSmem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bin_level1_kernel, kT, sizeof(BinSmem));
    g = sms * (per_sm > 0 ? 1 : 0);
  }
  return g;
}

cudaError_t launch_coop(const void* f, BinArgs& a, cudaStream_t st) {
  const int g = grid_size();
  if (g <= 0) return cudaErrorCooperativeLaunchTooLarge;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel(f, g, kT, args, sizeof(BinSmem), st);
}

}  // namespace

size_t bin_part_words() { return static_cast<size_t>(grid_size() + 2) * 256 + 64; }

cudaError_t bin_level1(BinArgs& a, cudaStream_t st) {
  return launch_coop(reinterpret_cast<const void*>(bin_level1_kernel), a, st);
}

cudaError_t bin_level2(BinArgs& a, cudaStream_t st) {
  if (a.num_isect <= 0) return cudaMemsetAsync(a.tile_offsets, 0, sizeof(uint32_t) * (a.num_tiles + 1), st);
  return launch_coop(reinterpret_cast<const void*>(bin_level2_kernel), a, st);
}

cudaError_t debug_source_order_keys(BinArgs& a, uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss,
                                    cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const int g = grid_size();
  void* args[] = {&a, &key_tile, &key_depth, &key_gauss};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(debug_keys_kernel), g, kT, args, sizeof(BinSmem),
                                     st);
}

}  // namespace fgs
