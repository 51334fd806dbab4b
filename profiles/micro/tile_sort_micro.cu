// Per-tile sort cost of fgs_sort.cuh's sort_tile_list as K3 runs it (256 threads, the radix
// digit counters passed): average cycles per CTA for list length L, keys in global memory
// (L2-resident), many CTAs resident per SM as in K3. Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2409_04751_b200/csrc \
//     tile_sort_micro.cu -o /tmp/tsm && /tmp/tsm
// Measured (the product paths): L 16-32: 0.013 ms per 2368 tiles, 100: 0.019, 256: 0.027,
// 300-512 (CTA bitonic): 0.045, 700: 0.076, 1000: 0.093, 2048 (radix): 0.148, 2572-4096: 0.335.
// A CTA merge sort (warp-sorted chunks, merge-path levels between two shared buffers) measured
// 20-30 % faster here for 257..2048 keys (2048: 0.124 ms) but made K3 slower at config 2
// (0.152 -> 0.157 ms): in K3 the sort runs beside other CTAs' blends, and the merge levels'
// shared-memory traffic competes with the blends' staging reads (config 4: 0.615 -> 0.600).
#include <cstdio>
#include <random>
#include <vector>
#include <algorithm>
#include "fgs_sort.cuh"

using namespace fgs;

__global__ void __launch_bounds__(256) sort_kernel(uint64_t* keys, uint32_t* out, int L, unsigned long long* cyc) {
  __shared__ __align__(128) uint64_t s[kSortCap];
  __shared__ uint32_t hist[8][256];
  const long long t0 = clock64();
  const int off = sort_tile_list<256>(keys, out, static_cast<uint32_t>(blockIdx.x) * L, L, s, hist);
  if (threadIdx.x == 0) atomicAdd(cyc, static_cast<unsigned long long>(clock64() - t0) + (off == 12345));
}

int main() {
  const int Ls[] = {16, 32, 64, 100, 128, 200, 256, 300, 400, 512, 700, 1000, 1500, 2048, 2572, 4096};
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  std::mt19937_64 rng(1);
  for (int L : Ls) {
    const int tiles = 592 * 4;  // several waves
    std::vector<uint64_t> h(static_cast<size_t>(tiles) * L);
    for (auto& v : h) v = (rng() & 0xFFFFFFFF00000000ull) | (rng() & 0xFFFFF);
    uint64_t* d;
    uint32_t* o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(cyc, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    sort_kernel<<<tiles, 256>>>(d, o, L, cyc);  // warm (the sort is in place)
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(cyc, 0, 8);
    cudaEventRecord(e0);
    sort_kernel<<<tiles, 256>>>(d, o, L, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // check: the ids of every tile in (depth, id) order
    std::vector<uint32_t> ho(h.size());
    cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int t = 0; t < tiles && !bad; ++t) {
      std::vector<uint64_t> ref(h.begin() + static_cast<size_t>(t) * L, h.begin() + static_cast<size_t>(t + 1) * L);
      std::sort(ref.begin(), ref.end());
      for (int k = 0; k < L; ++k)
        if (static_cast<uint32_t>(ref[k]) != ho[static_cast<size_t>(t) * L + k]) bad = 1;
    }
    printf("%s ", bad ? "WRONG" : "ok");
    printf("L %5d  cycles/CTA %8.0f  (%.2f us at 1.965 GHz)  kernel %.3f ms for %d tiles\n", L, double(c) / tiles,
           double(c) / tiles / 1965.0, ms, tiles);
    cudaFree(d);
    cudaFree(o);
  }
  return 0;
}
