// binning.cu — K2: intersection scan, tile ranges and key scatter (one cooperative kernel).
//
// Ordering contract (reference inc/splatting.hpp:192-249): the per-tile
// lists are sorted by (tile id, depth key bits, source index). The reference duplicates keys
// in source order and runs two stable LSD sorts over all I intersections (depth, then tile).
// Here no global sort runs at all; the same order is produced tile-locally:
//
//   K1 (preprocess.cu) also adds each kept Gaussian's tile rectangle into a row-difference
//      array over the tile grid (+1 at (ty, tx0), -1 at (ty, tx1 + 1) for each of its rows);
//   K2 bin_kernel (persistent cooperative, two grid barriers):
//      phase 1: per-CTA counts of tile-touching Gaussians / intersections; one warp per tile
//               row turns the row-difference array into per-tile counts, row totals, the
//               schedule histogram, the longest list and the backward's segment count;
//      phase 2: exclusive scan in source order -> emission offset of every tile-touching
//               Gaussian (compacted list), I, the gradient-chunk boundaries; the tile ranges
//               (offsets[0..T]), scatter cursors and the blend schedule;
//      phase 3: each intersection (Gaussian g, tile t) claims a position in tile t's range
//               (per-CTA shared-memory counts, one global atomicAdd per (CTA, tile)) and its
//               64-bit key (depth_key << 32 | g) is written there;
//   K2 bin_local_kernel (same phases and outputs; scenes of <= 148 x 8192 Gaussians, configs 0-2):
//      each CTA compacts its own range of Gaussians once in shared memory (phase 1), writes the
//      compacted list with the CTAs' prefix added (phase 2) and scatters its own intersections
//      from the shared list (phase 3), with no global rank search or second pass over touched[];
//      larger scenes take bin_kernel's slot order or tile-row lists;
//   [host reads I and the frame's scalars, off the critical path; K3 is already queued]
//   K3 (raster.cu) sorts each tile's keys at the start of its CTA (fgs_sort.cuh).
//
// The key is the reference's own sort key within a tile, (depth key bits, source index), so
// sorting a tile's keys gives the reference's order bit-exactly, whatever order the atomics
// handed out the positions in. Emission slots (source order, tiles ascending within a
// Gaussian) index the backward's per-intersection gradients: slot = src_off[g] + the tile's
// index in g's rectangle.

#include <cooperative_groups.h>

#include <utility>

#include "fgs_kernels.h"

namespace cg = cooperative_groups;

namespace fgs {

namespace {

constexpr int kT = kBinThreads;       // threads per persistent CTA
constexpr int kW = kBinThreads / 32;  // warps per persistent CTA
constexpr int kItems = 8;             // items per thread per sub-tile (thread-contiguous)
constexpr int kSchedBuckets = 18;     // blend schedule: log2 list-length buckets
constexpr int kPrivTiles = 16384;     // scatter: per-CTA shared tile counters up to this many tiles

struct ScanSmem {
  uint32_t warp_tmp[kW];
  uint32_t warp_tmp2[kW];
  uint32_t hist[32];
  uint32_t run[32];
  uint32_t scalar[4];
};

#ifdef FGS_CHECKED
// Checked build: key position p lies in tile t's range (and the buffer); a rectangle is in the grid.
__device__ __forceinline__ bool key_slot_ok(const BinArgs& a, uint32_t t, uint32_t p) {
  return t < static_cast<uint32_t>(a.num_tiles) && p >= a.tile_offsets[t] && p < a.tile_offsets[t + 1] &&
         static_cast<int64_t>(p) < a.isect_cap;
}
__device__ __forceinline__ bool rect_ok(const BinArgs& a, ushort4 rc) {
  return rc.x <= rc.y && rc.y < a.tiles_x && rc.z <= rc.w && rc.w < a.tiles_y;
}
#endif

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

// Sum over CTAs c' < blockIdx.x (prefix) and over all `parts` CTAs (total) of part[stride * c'].
__device__ __forceinline__ void cta_prefix(const uint32_t* part, int stride, int parts, uint32_t* s_warp,
                                           uint32_t& prefix, uint32_t& total) {
  uint32_t p = 0, t = 0;
  for (int c = threadIdx.x; c < parts; c += kT) {
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

// Debug phase profile (FGS_FLAG_COUNTERS): thread 0 of CTA `cta` adds the %globaltimer time since
// its previous call to slot (ns, accumulated over the kernel's loops). Slots: 0 counts, row counts
// and row histograms, 1 compaction, tile offsets and row lists, 2 the two grid barriers, 3 scatter:
// counter zeroing, 4 count pass, 5 (unused), 6 tile reservations (global atomics), 7 key pass.
__device__ __forceinline__ void trace(unsigned long long* t, int cta, int slot) {
  if (t && static_cast<int>(blockIdx.x) == cta && threadIdx.x == 0) {
    static __shared__ unsigned long long prev;
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    if (slot >= 0) t[slot] += v - prev;
    prev = v;
  }
}

__device__ __forceinline__ int sched_bucket(uint32_t c) {
  return c == 0 ? kSchedBuckets - 1 : 16 - min(16, 31 - __clz(c));
}

// ---- tile ranges, one warp per tile row (spread over the whole grid) ----
// rowdiff is (tiles_y) x (tiles_x + 1), row-major: K1 added +1 at (ty, tx0) and -1 at
// (ty, tx1 + 1) for every covered row, so a row's running sum gives its tiles' list lengths.
// Rows are independent; the tile offsets need only the row totals' prefix on top.
// Scratch (BinArgs::part_scan layout): hist[32] schedule buckets, cur[32] bucket cursors,
// rowtot[tiles_y]; hist / cur are zero between frames (zeroed after their last use).
constexpr int kRowItems = 8;

// Phase 1: counts of row ty into fill[] (tile-major), its total into rowtot[ty], the schedule
// histogram (warp-aggregated global atomics); rowdiff zeroed as read.
__device__ void row_counts(const BinArgs& a, int ty, uint32_t* hist, uint32_t* rowtot) {
  const int lane = threadIdx.x & 31, rw = a.tiles_x + 1;
  const uint32_t lt = lanemask_lt();
  int32_t* rd = a.rowdiff + static_cast<size_t>(ty) * rw;
  uint32_t carry = 0, tot = 0, segs = 0, longest = 0;
  for (int c0 = 0; c0 < rw; c0 += 32 * kRowItems) {
    int32_t v[kRowItems];
    int32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kRowItems; ++i) {
      const int x = c0 + lane * kRowItems + i;
      v[i] = x < rw ? rd[x] : 0;
      sum += v[i];
      if (x < rw && v[i]) rd[x] = 0;
    }
    uint32_t incl = static_cast<uint32_t>(sum);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t run = carry + incl - static_cast<uint32_t>(sum);
#pragma unroll
    for (int i = 0; i < kRowItems; ++i) {
      const int x = c0 + lane * kRowItems + i;
      run += static_cast<uint32_t>(v[i]);
      const bool cell = x < a.tiles_x;
      if (cell) {
        a.fill[static_cast<size_t>(ty) * a.tiles_x + x] = run;
        tot += run;
        if (run > kSeg) segs += (run + kSeg - 1) / kSeg;  // the backward's segments of a long list
        longest = max(longest, run);
      }
      const int bk = cell ? sched_bucket(run) : 31;
      const uint32_t peers = __match_any_sync(0xffffffffu, bk);
      if (bk != 31 && (peers & lt) == 0) atomicAdd(hist + bk, __popc(peers));
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tot += __shfl_xor_sync(0xffffffffu, tot, o);
    segs += __shfl_xor_sync(0xffffffffu, segs, o);
  }
  longest = __reduce_max_sync(0xffffffffu, longest);
  if (lane == 0) {
    rowtot[ty] = tot;
    if (segs) atomicAdd(a.scalars + kScalarSegs, segs);
    if (longest) atomicMax(a.scalars + kScalarMaxList, longest);
  }
}

// Phase 2: tile offsets and scatter cursors of row ty (row prefix + in-row exclusive scan),
// blend schedule slots (tiles by descending list length: log2 buckets, empty tiles last).
__device__ void row_offsets(const BinArgs& a, int ty, const uint32_t* rowtot, const uint32_t* hist, uint32_t* cur,
                            uint32_t bprefix_lane, uint32_t* wsm) {
  const int lane = threadIdx.x & 31;
  uint32_t pre = 0;
  for (int r = lane; r < ty; r += 32) pre += rowtot[r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  uint32_t carry = pre;
  for (int c0 = 0; c0 < a.tiles_x; c0 += 32 * kRowItems) {
    uint32_t c[kRowItems], sum = 0;
#pragma unroll
    for (int i = 0; i < kRowItems; ++i) {
      const int x = c0 + lane * kRowItems + i;
      c[i] = x < a.tiles_x ? a.fill[static_cast<size_t>(ty) * a.tiles_x + x] : 0u;
      sum += c[i];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t off = carry + incl - sum;
    const uint32_t off0 = off;
    // schedule slots: ranks within the row's bucket counts (warp-private shared counters), then
    // one global reservation per bucket for the whole row
    wsm[lane] = 0u;
    __syncwarp();
    uint32_t rk[kRowItems];
#pragma unroll
    for (int i = 0; i < kRowItems; ++i) {
      const int x = c0 + lane * kRowItems + i;
      const bool cell = x < a.tiles_x;
      const int t = ty * a.tiles_x + x;
      if (cell) {
        a.tile_offsets[t] = off;
        a.fill[t] = off;
        rk[i] = atomicAdd(wsm + sched_bucket(c[i]), 1u);
      }
      off += c[i];
    }
    __syncwarp();
    if (lane < kSchedBuckets && wsm[lane]) wsm[32 + lane] = atomicAdd(cur + lane, wsm[lane]) + bprefix_lane;
    __syncwarp();
    uint32_t o = off0;
#pragma unroll
    for (int i = 0; i < kRowItems; ++i) {
      const int x = c0 + lane * kRowItems + i;
      if (x < a.tiles_x)  // the blend CTA's work item: tile and its range in one 16-byte load
        a.tile_sched[wsm[32 + sched_bucket(c[i])] + rk[i]] = make_uint4(static_cast<uint32_t>(ty * a.tiles_x + x), o, o + c[i], 0u);
      o += c[i];
    }
    __syncwarp();
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (ty == a.tiles_y - 1 && lane == 0) {
    a.tile_offsets[a.num_tiles] = carry;
    a.scalars[kScalarI2] = carry;
  }
}

// Largest r in [0, m) with offs[r] <= v (offs ascending, offs[0] = 0), for two values: repeated
// blockDim-ary search by the whole CTA.
__device__ void cta_upper_rank2(const uint32_t* offs, int m, uint32_t v0, uint32_t v1, uint32_t* s_res, int& r0,
                                int& r1) {
  // the two searches share their rounds (and barriers)
  const int tid = threadIdx.x, nt = blockDim.x;
  int base[2] = {0, 0}, range[2] = {m, m};
  const uint32_t v[2] = {v0, v1};
  while (true) {
    int step[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) step[q] = (range[q] + nt - 1) / nt;
    if (tid < 2) s_res[tid] = static_cast<uint32_t>(base[tid]);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = base[q] + tid * step[q];
      if (tid * step[q] < range[q] && offs[r] <= v[q]) atomicMax(s_res + q, static_cast<uint32_t>(r));
    }
    __syncthreads();
    const int nb0 = static_cast<int>(s_res[0]), nb1 = static_cast<int>(s_res[1]);
    __syncthreads();
    if (step[0] <= 1 && step[1] <= 1) {
      r0 = nb0;
      r1 = nb1;
      return;
    }
    base[0] = nb0;
    base[1] = nb1;
    range[0] = step[0] <= 1 ? 1 : min(step[0], m - nb0);
    range[1] = step[1] <= 1 ? 1 : min(step[1], m - nb1);
  }
}

// Scatter of emission slots [lo, hi) (<= kSub) by one CTA: every slot finds its Gaussian by
// binary search over the range's compacted emission offsets (staged in shared memory), and
// claims a position in its tile's range. PRIV: two levels -- the CTA counts its slots per
// tile with shared-memory atomics, then one global atomicAdd per (CTA, tile) reserves the
// block, so a heavy tile sees one global atomic per CTA instead of one per intersection. All
// loads and atomics of a thread's slots are issued before their results are used.
constexpr int kSub = 8 * kT;  // emission slots per source-order scatter sub-range

template <bool PRIV>
__device__ void scatter_range(const BinArgs& a, int m, uint32_t lo, uint32_t hi, uint32_t* s_cnt, uint32_t* s_off,
                              uint32_t* s_res) {
  constexpr int U = kSub / kT;
  const int tid = threadIdx.x;
  if (PRIV)
    for (int t = tid; t < a.num_tiles; t += kT) s_cnt[t] = 0;
  int r_lo, r_hi;
  cta_upper_rank2(a.coff, m, lo, hi - 1, s_res, r_lo, r_hi);
  const int nr = r_hi - r_lo + 1;  // <= kSub: every Gaussian here owns >= 1 slot
  for (int i = tid; i < nr; i += kT) s_off[i] = a.coff[r_lo + i];
  __syncthreads();
  trace(a.trace, 0, 3);
  uint32_t ev[U], gv[U], tv[U], pv[U];
  // each thread owns un <= U consecutive slots (every thread busy when the range is short): one
  // binary search for the first, then a forward walk (a Gaussian owns ~3 slots on average, so
  // the walk advances a step or two)
  {
    const uint32_t un = (hi - lo + kT - 1) / kT;
    const uint32_t e0 = lo + static_cast<uint32_t>(tid) * un;
    int l = 0, h = nr - 1;
    while (l < h) {
      const int mid = (l + h + 1) >> 1;
      if (s_off[mid] <= e0) l = mid;
      else h = mid - 1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ev[u] = u < static_cast<int>(un) ? e0 + u : hi;  // hi: no slot
      if (ev[u] < hi)
        while (l + 1 < nr && s_off[l + 1] <= ev[u]) ++l;
      tv[u] = static_cast<uint32_t>(l);  // local rank for now
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) gv[u] = ev[u] < hi ? a.cval[r_lo + tv[u]] : 0u;
  uint32_t dk[U];  // depth keys, in flight across the atomics
#pragma unroll
  for (int u = 0; u < U; ++u) dk[u] = a.depth_key[gv[u]];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (ev[u] >= hi) continue;
    const ushort4 rc = a.rect[gv[u]];
    FGS_DCHECK(rect_ok(a, rc) && ev[u] >= s_off[tv[u]]);
    const int wx = rc.y - rc.x + 1;
    const int j = static_cast<int>(ev[u] - s_off[tv[u]]);
    tv[u] = static_cast<uint32_t>((rc.z + j / wx) * a.tiles_x + rc.x + j % wx);
  }
  if (a.trace) { __syncthreads(); trace(a.trace, 0, 4); }
  if (PRIV) {
#pragma unroll
    for (int u = 0; u < U; ++u) pv[u] = ev[u] < hi ? atomicAdd(s_cnt + tv[u], 1u) : 1u;
    __syncthreads();
    trace(a.trace, 0, 5);
    // the slot that took local position 0 reserves the CTA's block of tile tv[u]
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (pv[u] == 0) s_cnt[tv[u]] = atomicAdd(a.fill + tv[u], s_cnt[tv[u]]);
    __syncthreads();
    trace(a.trace, 0, 6);
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
    FGS_DCHECK(key_slot_ok(a, tv[u], pv[u]) && gv[u] < static_cast<uint32_t>(a.n));
    a.keys[pv[u]] = (static_cast<uint64_t>(dk[u]) << 32) | gv[u];
  }
  __syncthreads();  // s_cnt / s_off reused by the next range
  trace(a.trace, 0, 7);
  trace(a.trace, 0, 7);
}

constexpr int kMaxRows = kMaxTileRows;  // tile rows the row-list phases keep in shared memory

// The row lists' layout (every CTA, from the row histograms of all CTAs): s_start[ty] = first
// entry of row ty in the concatenated row lists (s_start[tiles_y] = entries), s_cur[ty] = where
// this CTA's entries of row ty begin (rows in order, CTAs in order within a row).
__device__ void row_layout(const BinArgs& a, uint32_t* s_start, uint32_t* s_cur, uint32_t* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
  for (int ty = warp; ty < a.tiles_y; ty += kW) {
    uint32_t tot = 0, pre = 0;
    for (int c = lane; c < G; c += 32) {
      const uint32_t v = a.row_hist[static_cast<size_t>(c) * a.tiles_y + ty];
      tot += v;
      if (c < b) pre += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
      pre += __shfl_xor_sync(0xffffffffu, pre, o);
    }
    if (lane == 0) {
      s_start[ty] = tot;
      s_cur[ty] = pre;
    }
  }
  __syncthreads();
  // exclusive scan of the row totals (kMaxRows / kT = 4 rows per thread)
  constexpr int R = kMaxRows / kT;
  uint32_t v[R], sum = 0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int ty = tid * R + k;
    v[k] = ty < a.tiles_y ? s_start[ty] : 0u;
    sum += v[k];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan(sum, s_warp, &total);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int ty = tid * R + k;
    if (ty < a.tiles_y) {
      s_start[ty] = run;
      s_cur[ty] += run;
    }
    run += v[k];
  }
  if (tid == 0) s_start[a.tiles_y] = total;
  __syncthreads();
}

// The CTA's row-list entries for one tile-touching Gaussian i: listed once per tile row its
// rectangle covers (positions from the CTA's per-row cursors; order within a row free).
__device__ __forceinline__ void row_emit_one(const BinArgs& a, int i, uint32_t* s_cur) {
  const ushort4 rc = a.rect[i];
  FGS_DCHECK(rect_ok(a, rc));
  for (int ty = rc.z; ty <= rc.w; ++ty) {
    const uint32_t p = atomicAdd(s_cur + ty, 1u);
    FGS_DCHECK(static_cast<int64_t>(p) < a.isect_cap);
    a.row_list[p] = static_cast<uint32_t>(i);
  }
}

__device__ void row_emit(const BinArgs& a, int lo, int hi, uint32_t* s_cur) {
  for (int i = lo + static_cast<int>(threadIdx.x); i < hi; i += kT)
    if (a.touched[i]) row_emit_one(a, i, s_cur);
  __syncthreads();
}

// Row of row-list entry e: the last row whose start is <= e (s_start ascending).
__device__ __forceinline__ int row_of(const uint32_t* s_start, int rows, uint32_t e) {
  int l = 0, h = rows - 1;
  while (l < h) {
    const int mid = (l + h + 1) >> 1;
    if (s_start[mid] <= e) l = mid;
    else h = mid - 1;
  }
  return l;
}

// Phase 3: the intersections of row-list entries [e0, e1) -- a contiguous run of the row-major
// lists, so it spans one or a few tile rows and touches few tiles: the CTA counts its slots per
// tile in shared memory, reserves each tile's block with one global atomicAdd on the tile's
// cursor (few CTAs share a row, so little contention), then writes the keys at their positions.
// Rows are taken in windows whose tiles fit the shared counters; a single row wider than that
// falls back to one global atomic per slot.
__device__ void scatter_rows(const BinArgs& a, uint32_t e0, uint32_t e1, const uint32_t* s_start, uint32_t* s_cnt) {
  const int tid = threadIdx.x;
  if (e0 >= e1) return;
  const int tx = a.tiles_x;
  int ty = row_of(s_start, a.tiles_y, e0);
  const int ty_last = row_of(s_start, a.tiles_y, e1 - 1);
  while (ty <= ty_last) {
    // window of rows [ty, ty_end]
    const int rows_fit = max(1, kPrivTiles / tx);
    const int ty_end = min(ty_last, ty + rows_fit - 1);
    const uint32_t w0 = max(e0, s_start[ty]), w1 = min(e1, s_start[ty_end + 1]);
    const int span0 = ty * tx, span = (ty_end - ty + 1) * tx;
    if (span <= kPrivTiles) {
      for (int t = tid; t < span; t += kT) s_cnt[t] = 0;
      __syncthreads();
      trace(a.trace, 0, 3);
      // (a thread's entries ascend, so its row only moves forward)
      int r = ty;
      for (uint32_t e = w0 + tid; e < w1; e += kT) {
        while (s_start[r + 1] <= e) ++r;
        const ushort4 rc = a.rect[a.row_list[e]];
        for (int x = rc.x; x <= rc.y; ++x) atomicAdd(s_cnt + (r * tx + x - span0), 1u);
      }
      __syncthreads();
      trace(a.trace, 0, 4);
      for (int t = tid; t < span; t += kT)
        if (s_cnt[t]) s_cnt[t] = atomicAdd(a.fill + span0 + t, s_cnt[t]);
      __syncthreads();
      trace(a.trace, 0, 6);
      r = ty;
      for (uint32_t e = w0 + tid; e < w1; e += kT) {
        while (s_start[r + 1] <= e) ++r;
        const uint32_t g = a.row_list[e];
        const ushort4 rc = a.rect[g];
        const uint64_t key = (static_cast<uint64_t>(a.depth_key[g]) << 32) | g;
        FGS_DCHECK(rect_ok(a, rc) && r >= rc.z && r <= rc.w);
        for (int x = rc.x; x <= rc.y; ++x) {
          const uint32_t p = atomicAdd(s_cnt + (r * tx + x - span0), 1u);
          FGS_DCHECK(key_slot_ok(a, static_cast<uint32_t>(r * tx + x), p));
          a.keys[p] = key;
        }
      }
      __syncthreads();
      trace(a.trace, 0, 7);
    } else {
      for (uint32_t e = w0 + tid; e < w1; e += kT) {
        const int r = row_of(s_start, a.tiles_y, e);
        const uint32_t g = a.row_list[e];
        const ushort4 rc = a.rect[g];
        const uint64_t key = (static_cast<uint64_t>(a.depth_key[g]) << 32) | g;
        FGS_DCHECK(rect_ok(a, rc) && r >= rc.z && r <= rc.w);
        for (int x = rc.x; x <= rc.y; ++x) {
          const uint32_t p = atomicAdd(a.fill + r * tx + x, 1u);
          FGS_DCHECK(key_slot_ok(a, static_cast<uint32_t>(r * tx + x), p));
          a.keys[p] = key;
        }
      }
    }
    ty = ty_end + 1;
  }
}

// The frame's scalars (final since the second grid barrier) to the host's mapped buffer, by CTA 0
// once its own scatter is done (so its scatter starts without waiting for the loads): one
// 64-byte posted write of them, the sequence number and a hash binding the two (no fence: the
// host accepts the block once the sequence number and the hash agree).
__device__ __forceinline__ void publish_host_scalars(const BinArgs& a, int b) {
  pdl_trigger();  // (this CTA's part of K2 is done)
  if (b != 0 || threadIdx.x >= 32 || !a.host_scalars) return;
  const int tid = threadIdx.x;
  const uint32_t v = tid < kScalarReadback ? *reinterpret_cast<volatile const uint32_t*>(a.scalars + tid) : 0u;
  uint32_t h = host_block_hash_init(a.seq);
  for (int t = 0; t < kScalarReadback; ++t) h = host_block_hash_step(h, __shfl_sync(0xffffffffu, v, t));
  if (tid < kHostBlock)
    a.host_scalars[tid] = tid < kScalarReadback ? v : (tid == kHostHash ? h : (tid == kHostSeq ? a.seq : 0u));
}

// K2: one persistent cooperative kernel, two grid barriers.
//   phase 1: every CTA counts its chunk's tile-touching Gaussians and intersections; one warp
//            per tile row turns K1's row-difference array into per-tile list lengths (fill[]),
//            row totals and the schedule histogram;
//   phase 2: compaction of the tile-touching Gaussians (source order) with their emission
//            offsets (cval, coff, src_off); M and I to the device scalars; the row warps write
//            the tile offsets, scatter cursors and blend schedule (descending list length);
//   phase 3: all CTAs scatter the I emission slots (balanced by intersections) into the tile
//            ranges -- unless I exceeds the buffers' capacity (speculative launch: the host
//            grows them and launches again).
// ROWS: phase 3 by row lists (few tiles per CTA: little contention on the tile cursors; wins for
// large I, configs 3 and 4) or by emission slots in source order (no row-list passes; config 2).
template <bool ROWS>
__global__ void __launch_bounds__(kT, kBinCtasPerSm) bin_kernel(BinArgs a) {
  extern __shared__ uint32_t s_cnt[];  // [min(num_tiles, kPrivTiles)] phase-3 tile counters
  __shared__ ScanSmem sm;
  __shared__ uint32_t s_rowoff[kW * 64];         // row_offsets scratch, 64 words per warp
  __shared__ uint32_t s_big[2 * kMaxRows + 8];   // ROWS: s_start + s_cur; else the scatter's s_off
  __shared__ uint32_t s_res[2];
  static_assert(2 * kMaxRows + 8 >= kSub, "s_off fits");
  uint32_t* s_start = s_big;                     // row lists: first entry of every tile row
  uint32_t* s_cur = s_big + kMaxRows + 4;        // this CTA's next entry of every tile row
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  const int G = static_cast<int>(gridDim.x);
  const int b = static_cast<int>(blockIdx.x);
  const int lane = tid & 31, nw = G * kW;
  uint32_t* hist = a.part_scan + 2 * G;
  uint32_t* cur = hist + 32;
  uint32_t* rowtot = cur + 32;
  int lo = static_cast<int>(static_cast<int64_t>(a.n) * b / G);
  int hi = static_cast<int>(static_cast<int64_t>(a.n) * (b + 1) / G);
  trace(a.trace, 0, -1);
  if (a.scatter_only) goto scatter;  // relaunch after the buffers grew: phases 1-2 are done
  {
    // counts, and (ROWS) the CTA's row histogram (per tile row, the tile-touching Gaussians covering it)
    if (ROWS) {
      for (int t = tid; t < a.tiles_y; t += kT) s_cur[t] = 0;
      __syncthreads();
    }
    uint32_t c1 = 0, c2 = 0;
    for (int i = lo + tid; i < hi; i += kT) {
      const uint32_t t = a.touched[i];
      c1 += t > 0 ? 1u : 0u;
      c2 += t;
      if (ROWS && t) {
        const ushort4 rc = a.rect[i];
        for (int ty = rc.z; ty <= rc.w; ++ty) atomicAdd(s_cur + ty, 1u);
      }
    }
    if (ROWS) {
      __syncthreads();
      for (int t = tid; t < a.tiles_y; t += kT) a.row_hist[static_cast<size_t>(b) * a.tiles_y + t] = s_cur[t];
    }
    uint32_t t1, t2;
    block_exclusive_scan(c1, sm.warp_tmp, &t1);
    block_exclusive_scan(c2, sm.warp_tmp2, &t2);
    if (tid == 0) {
      a.part_scan[2 * b] = t1;
      a.part_scan[2 * b + 1] = t2;
    }
  }
  // rows spread over CTAs first (row ty -> CTA ty mod G), so no CTA gets two
  for (int ty = b + G * (tid >> 5); ty < a.tiles_y; ty += nw) row_counts(a, ty, hist, rowtot);
  trace(a.trace, 0, 0);
  grid.sync();
  trace(a.trace, 0, 2);
  {
    uint32_t p1, tot1, p2, tot2;
    cta_prefix(a.part_scan, 2, G, sm.warp_tmp, p1, tot1);
    cta_prefix(a.part_scan + 1, 2, G, sm.warp_tmp, p2, tot2);
    // schedule bucket prefix (lane k holds bucket k's start) and the long-list count
    const uint32_t hk = lane < kSchedBuckets ? hist[lane] : 0u;
    uint32_t incl = hk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t bprefix = incl - hk;
    if (b == 0 && tid == 0) {
      a.scalars[kScalarM] = tot1;
      a.scalars[kScalarI] = tot2;
    }
    if (b == 0 && tid < 32) {
      // the first n_big schedule slots hold the lists of >= 256 keys (log2 buckets 0..8)
      uint32_t big = lane < kSchedBuckets && 16 - lane >= 8 ? hk : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) big += __shfl_xor_sync(0xffffffffu, big, o);
      if (lane == 0) a.scalars[kScalarBig] = big;
    }
    for (int ty = b + G * (tid >> 5); ty < a.tiles_y; ty += nw)
      row_offsets(a, ty, rowtot, hist, cur, bprefix, s_rowoff + 64 * (tid >> 5));
    // the row lists' layout; their entries are written with the compaction (<= I entries: they
    // fit the per-intersection buffers when I does)
    if (ROWS) row_layout(a, s_start, s_cur, sm.warp_tmp);
    const bool emit = ROWS && tot2 <= a.isect_cap;
    uint32_t run1 = p1, run2 = p2;
    int gchunk[kGradChunks];
#pragma unroll
    for (int cb = 0; cb < kGradChunks; ++cb) gchunk[cb] = static_cast<int>(static_cast<int64_t>(a.n) * cb / kGradChunks);
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
        // a gradient-chunk boundary c N / C at this id: the compacted position there
#pragma unroll
        for (int cb = 1; cb < kGradChunks; ++cb)
          if (r0 + i == gchunk[cb]) a.scalars[kScalarChunkQ + cb - 1] = pos;
        if (c[i]) {
          a.cval[pos] = static_cast<uint32_t>(r0 + i);
          a.coff[pos] = off;
          a.src_off[r0 + i] = off;
          ++pos;
          off += c[i];
          if (emit) row_emit_one(a, r0 + i, s_cur);
        }
      }
      run1 += t1;
      run2 += t2;
    }
  }
  trace(a.trace, 0, 1);
  grid.sync();
  trace(a.trace, 0, 2);
  if (b == 0 && tid < 64) hist[tid] = 0;  // hist + cur: last read before this barrier
  if (ROWS) {
    const uint32_t I = a.scalars[kScalarI];
    if (I <= a.isect_cap && I != 0) {
      const uint32_t E = s_start[a.tiles_y];
      scatter_rows(a, static_cast<uint32_t>(static_cast<uint64_t>(E) * b / G),
                   static_cast<uint32_t>(static_cast<uint64_t>(E) * (b + 1) / G), s_start, s_cnt);
    }
    publish_host_scalars(a, b);
    return;
  }
scatter : {
  const uint32_t I = a.scalars[kScalarI];
  if (I > a.isect_cap || I == 0) {
    if (!a.scatter_only) publish_host_scalars(a, b);
    return;
  }
  if (ROWS) {
    // relaunch after the buffers grew: phases 1-2 ran (row histograms in row_hist); the row
    // lists are written now, then the scatter
    row_layout(a, s_start, s_cur, sm.warp_tmp);
    row_emit(a, lo, hi, s_cur);
    grid.sync();
    const uint32_t E = s_start[a.tiles_y];
    scatter_rows(a, static_cast<uint32_t>(static_cast<uint64_t>(E) * b / G),
                 static_cast<uint32_t>(static_cast<uint64_t>(E) * (b + 1) / G), s_start, s_cnt);
  } else {
    // the emission slots, balanced by intersections, in source order
    const int m = static_cast<int>(a.scalars[kScalarM]);
    const uint32_t s_lo = static_cast<uint32_t>(static_cast<uint64_t>(I) * b / G);
    const uint32_t s_hi = static_cast<uint32_t>(static_cast<uint64_t>(I) * (b + 1) / G);
    for (uint32_t x = s_lo; x < s_hi; x += kSub)
      scatter_range<true>(a, m, x, min(s_hi, x + kSub), s_cnt, s_big, s_res);
  }
  if (!a.scatter_only) publish_host_scalars(a, b);
}
}

// ---- K2 with CTA-local compaction (the slot order for scenes of <= grid x 8192 Gaussians) ----
// Each CTA owns one contiguous range of Gaussians (<= kLocG) for the whole kernel. Phase 1 loads
// its touched counts once and compacts them in shared memory (local position and local
// intersection prefix of every tile-touching Gaussian, kept across the grid barriers); phase 2
// only adds the CTAs' prefix to write cval / coff / src_off (no second pass over touched[]);
// phase 3 scatters the CTA's own intersections from the shared list: one binary search per
// thread over the compacted offsets, then a forward walk (no global rank search, no staging of
// coff, no per-slot Gaussian lookups), shared-memory counts per tile, one global atomicAdd per
// (CTA, tile), then the keys. Same outputs as bin_kernel<false> (the key positions inside a
// tile's range differ, the per-tile sort orders them).
constexpr int kLocG = kT * kItems;  // Gaussians per CTA
constexpr int kLocalSmem = (kLocG + 1 + kLocG / 2) * 4;  // dynamic shared memory before the tile counters

// The CTA's tile-touching Gaussians of [lo, hi) compacted in shared memory: s_lo[q] = their
// local exclusive intersection prefix, s_lg[q] = local index; returns (count, intersections).
// `between` runs while the touched loads are in flight (the row warps' phase-1 work).
template <typename F>
__device__ __forceinline__ uint2 local_compact(const BinArgs& a, int lo, int hi, uint32_t* s_lo, uint16_t* s_lg,
                                               ScanSmem& sm, F&& between) {
  const int tid = threadIdx.x, r0 = lo + tid * kItems;
  uint32_t c[kItems], s1 = 0, s2 = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) c[i] = r0 + i < hi ? a.touched[r0 + i] : 0u;
  between();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    s1 += c[i] > 0 ? 1u : 0u;
    s2 += c[i];
  }
  uint32_t m, r;
  uint32_t pos = block_exclusive_scan(s1, sm.warp_tmp, &m);
  uint32_t off = block_exclusive_scan(s2, sm.warp_tmp2, &r);
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if (c[i]) {
      s_lo[pos] = off;
      s_lg[pos] = static_cast<uint16_t>(tid * kItems + i);
      ++pos;
      off += c[i];
    }
  if (tid == 0) s_lo[m] = r;  // sentinel
  __syncthreads();
  return make_uint2(m, r);
}

// Phase 3 of the local variant: the CTA's R intersections from its compacted list (m entries),
// in passes of <= kSub.
__device__ void scatter_local(const BinArgs& a, int lo, uint32_t m, uint32_t R, const uint32_t* s_lo,
                              const uint16_t* s_lg, uint32_t* s_cnt) {
  constexpr int U = kSub / kT;
  const int tid = threadIdx.x;
  for (uint32_t x0 = 0; x0 < R; x0 += kSub) {
    const uint32_t hi = min(R, x0 + kSub);
    for (int t = tid; t < a.num_tiles; t += kT) s_cnt[t] = 0;
    __syncthreads();
    trace(a.trace, 0, 3);
    uint32_t ev[U], gv[U], tv[U], pv[U], dk[U];
    {
      const uint32_t un = (hi - x0 + kT - 1) / kT;
      const uint32_t e0 = x0 + static_cast<uint32_t>(tid) * un;
      int l = 0, h = static_cast<int>(m) - 1;  // largest q with s_lo[q] <= e0
      while (l < h) {
        const int mid = (l + h + 1) >> 1;
        if (s_lo[mid] <= e0) l = mid;
        else h = mid - 1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ev[u] = u < static_cast<int>(un) ? e0 + u : hi;  // hi: no slot
        if (ev[u] < hi)
          while (s_lo[l + 1] <= ev[u]) ++l;  // (s_lo[m] = R > ev)
        tv[u] = static_cast<uint32_t>(l);
        gv[u] = static_cast<uint32_t>(lo + s_lg[l]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) dk[u] = ev[u] < hi ? a.depth_key[gv[u]] : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (ev[u] >= hi) continue;
      const ushort4 rc = a.rect[gv[u]];
      FGS_DCHECK(rect_ok(a, rc) && ev[u] >= s_lo[tv[u]] && gv[u] < static_cast<uint32_t>(a.n));
      const int wx = rc.y - rc.x + 1;
      const int j = static_cast<int>(ev[u] - s_lo[tv[u]]);
      tv[u] = static_cast<uint32_t>((rc.z + j / wx) * a.tiles_x + rc.x + j % wx);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) pv[u] = ev[u] < hi ? atomicAdd(s_cnt + tv[u], 1u) : 1u;
    __syncthreads();
    trace(a.trace, 0, 4);
    // the slot that took local position 0 reserves the CTA's block of tile tv[u]
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (pv[u] == 0) s_cnt[tv[u]] = atomicAdd(a.fill + tv[u], s_cnt[tv[u]]);
    __syncthreads();
    trace(a.trace, 0, 6);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (ev[u] >= hi) continue;
      pv[u] += s_cnt[tv[u]];
      FGS_DCHECK(key_slot_ok(a, tv[u], pv[u]));
      a.keys[pv[u]] = (static_cast<uint64_t>(dk[u]) << 32) | gv[u];
    }
    __syncthreads();  // s_cnt reused by the next pass
    trace(a.trace, 0, 7);
  }
}

__global__ void __launch_bounds__(kT, kBinCtasPerSm) bin_local_kernel(BinArgs a) {
  extern __shared__ uint32_t s_dyn[];  // [kLocG + 1] s_lo, [kLocG / 2] s_lg, [num_tiles] tile counters
  __shared__ ScanSmem sm;
  __shared__ uint32_t s_rowoff[kW * 64];
  uint32_t* s_lo = s_dyn;
  uint16_t* s_lg = reinterpret_cast<uint16_t*>(s_dyn + kLocG + 1);
  uint32_t* s_cnt = s_dyn + kLocG + 1 + kLocG / 2;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31;
  const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x), nw = G * kW;
  uint32_t* hist = a.part_scan + 2 * G;
  uint32_t* cur = hist + 32;
  uint32_t* rowtot = cur + 32;
  const int lo = static_cast<int>(static_cast<int64_t>(a.n) * b / G);
  const int hi = static_cast<int>(static_cast<int64_t>(a.n) * (b + 1) / G);
  trace(a.trace, 0, -1);
  // the tile rows' counts by the CTAs' last warps (rows b, b + G, ... of CTA b), overlapping the
  // touched loads of the local compaction
  const uint2 mr = local_compact(a, lo, hi, s_lo, s_lg, sm, [&] {
    if (!a.scatter_only)
      for (int ty = b + G * (kW - 1 - (tid >> 5)); ty < a.tiles_y; ty += nw) row_counts(a, ty, hist, rowtot);
  });
  if (!a.scatter_only) {
    if (tid == 0) {
      a.part_scan[2 * b] = mr.x;
      a.part_scan[2 * b + 1] = mr.y;
    }
    trace(a.trace, 0, 0);
    grid.sync();
    trace(a.trace, 0, 2);
    const uint32_t hk = lane < kSchedBuckets ? hist[lane] : 0u;
    uint32_t incl = hk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    // the row warps (the CTAs' last warps) write their rows' offsets and schedule slots while
    // warp 0 sums the CTAs' partials (no block scans); one barrier hands the prefix to the CTA
    for (int ty = b + G * (kW - 1 - (tid >> 5)); ty < a.tiles_y; ty += nw)
      row_offsets(a, ty, rowtot, hist, cur, incl - hk, s_rowoff + 64 * (tid >> 5));
    if (tid < 32) {
      uint32_t v4[4] = {0u, 0u, 0u, 0u};  // p1, p2, tot1, tot2
      for (int c = lane; c < G; c += 32) {
        const uint32_t m1 = a.part_scan[2 * c], m2 = a.part_scan[2 * c + 1];
        v4[2] += m1;
        v4[3] += m2;
        if (c < b) {
          v4[0] += m1;
          v4[1] += m2;
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) v4[k] = __reduce_add_sync(0xffffffffu, v4[k]);
      if (lane == 0) {
        sm.scalar[0] = v4[0];
        sm.scalar[1] = v4[1];
        if (b == 0) {
          a.scalars[kScalarM] = v4[2];
          a.scalars[kScalarI] = v4[3];
        }
      }
    }
    __syncthreads();
    const uint32_t p1 = sm.scalar[0], p2 = sm.scalar[1];
    if (b == 0 && tid < 32) {
      uint32_t big = lane < kSchedBuckets && 16 - lane >= 8 ? hk : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) big += __shfl_xor_sync(0xffffffffu, big, o);
      if (lane == 0) a.scalars[kScalarBig] = big;
    }
    // gradient-chunk boundaries c N / C inside this CTA's range: the compacted position there
    if (tid > 0 && tid < kGradChunks) {
      const int gc = static_cast<int>(static_cast<int64_t>(a.n) * tid / kGradChunks);
      if (gc >= lo && gc < hi) {
        uint32_t q = 0, h = mr.x;  // first compacted entry with id >= gc
        while (q < h) {
          const uint32_t mid = (q + h) >> 1;
          if (lo + static_cast<int>(s_lg[mid]) < gc) q = mid + 1;
          else h = mid;
        }
        a.scalars[kScalarChunkQ + tid - 1] = p1 + q;
      }
    }
    for (uint32_t q = tid; q < mr.x; q += kT) {
      const uint32_t g = static_cast<uint32_t>(lo + s_lg[q]), off = p2 + s_lo[q];
      a.cval[p1 + q] = g;
      a.coff[p1 + q] = off;
      a.src_off[g] = off;
    }
    trace(a.trace, 0, 1);
    grid.sync();
    trace(a.trace, 0, 2);
    if (b == 0 && tid < 64) hist[tid] = 0;  // hist + cur: last read before this barrier
  }
  const uint32_t I = a.scalars[kScalarI];
  if (I <= a.isect_cap && I != 0) scatter_local(a, lo, mr.x, mr.y, s_lo, s_lg, s_cnt);
  if (!a.scatter_only) publish_host_scalars(a, b);
}

// Debug export: the reference's pre-sort key list (source order, ty-major, tx-minor).
__global__ void __launch_bounds__(kT, kBinCtasPerSm) debug_keys_kernel(BinArgs a, uint32_t* key_tile, uint32_t* key_depth,
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
  static PerDevice cache;
  return cache.get([] {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int ok = 1;
    const std::pair<const void*, int> ks[] = {{reinterpret_cast<const void*>(bin_kernel<true>), kPrivTiles * 4},
                                              {reinterpret_cast<const void*>(bin_kernel<false>), kPrivTiles * 4},
                                              {reinterpret_cast<const void*>(bin_local_kernel), kLocalSmem + kPrivTiles * 4}};
    for (const auto& k : ks) {
      cudaFuncSetAttribute(k.first, cudaFuncAttributeMaxDynamicSharedMemorySize, k.second);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.first, kT, k.second);
      ok = ok && per_sm >= kBinCtasPerSm;
    }
    return ok ? sms * kBinCtasPerSm : -1;  // -1: cooperative launch impossible
  });
}

}  // namespace

size_t bin_part_words(int tiles_y) { return static_cast<size_t>(std::max(grid_size(), 0)) * 2 + 64 + tiles_y; }
size_t bin_row_hist_words(int tiles_y) { return static_cast<size_t>(std::max(grid_size(), 0)) * tiles_y; }

cudaError_t bin_launch(BinArgs& a, cudaStream_t st) {
  const int g = grid_size();
  if (g < 2) return cudaErrorCooperativeLaunchTooLarge;
  if (a.tiles_y > kMaxRows) return cudaErrorInvalidValue;
  void* args[] = {&a};
  const size_t smem = static_cast<size_t>(std::min(a.num_tiles, kPrivTiles)) * 4;
  // the source-order scatter needs every tile's counter in shared memory
  const bool rows = a.row_scatter || a.num_tiles > kPrivTiles;
  a.fast = !rows && a.fast && static_cast<int64_t>(a.n) <= static_cast<int64_t>(g) * kLocG;  // (reported back)
  if (a.fast)
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(bin_local_kernel), g, kT, args, kLocalSmem + smem, st);
  return cudaLaunchCooperativeKernel(rows ? reinterpret_cast<const void*>(bin_kernel<true>)
                                          : reinterpret_cast<const void*>(bin_kernel<false>),
                                     g, kT, args, smem, st);
}

cudaError_t debug_source_order_keys(BinArgs& a, uint32_t* key_tile, uint32_t* key_depth, uint32_t* key_gauss,
                                    cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  debug_keys_kernel<<<div_up(a.n, kT), kT, 0, st>>>(a, key_tile, key_depth, key_gauss);
  return cudaGetLastError();
}

}  // namespace fgs
