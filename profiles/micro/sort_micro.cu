// Microbenchmark of the per-tile sort paths in fgs_sort.cuh: cycles per tile list for the
// CTA path (256 threads, shared memory) and the warp path (registers), with and without the
// global key loads. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2409_04751_b200/csrc
#include <cstdio>
#include <vector>
#include <random>
#include "fgs_sort.cuh"

using namespace fgs;

__global__ void cta_kernel(uint64_t* keys, uint32_t* out, int L, unsigned long long* cyc) {
  __shared__ uint64_t s[kSortCap];
  const long long t0 = clock64();
  sort_tile_list(keys, out, blockIdx.x * L, L, s);
  if (threadIdx.x == 0) atomicAdd(cyc, static_cast<unsigned long long>(clock64() - t0));
}

__global__ void smem_only_kernel(int P, unsigned long long* cyc, uint64_t seed) {
  __shared__ uint64_t s[kSortCap];
  for (int k = threadIdx.x; k < P; k += 256) s[k] = (seed * (k + 1) * 2654435761ull) ^ (k * 977);
  __syncthreads();
  const long long t0 = clock64();
  cta_sort(s, P);
  if (threadIdx.x == 0) atomicAdd(cyc, static_cast<unsigned long long>(clock64() - t0));
}

__global__ void warp8_kernel(unsigned long long* cyc, uint64_t seed) {
  uint64_t x[8];
  const int lane = threadIdx.x & 31;
  for (int r = 0; r < 8; ++r) x[r] = (seed * (r * 32 + lane + 1) * 2654435761ull) ^ lane;
  const long long t0 = clock64();
  warp_sort<8>(x, lane);
  const long long t1 = clock64();
  uint64_t acc = 0;
  for (int r = 0; r < 8; ++r) acc ^= x[r];
  if (lane == 0) atomicAdd(cyc, static_cast<unsigned long long>(t1 - t0) + (acc == 12345 ? 1 : 0));
}

int main() {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  for (int L : {300, 600, 1000, 2000, 4000}) {
    const int tiles = 860;
    std::vector<uint64_t> h(static_cast<size_t>(tiles) * L);
    std::mt19937_64 rng(1);
    for (auto& v : h) v = rng();
    uint64_t* d;
    uint32_t* o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(cyc, 0, 8);
    cta_kernel<<<tiles, 256>>>(d, o, L, cyc);  // warm
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(cyc, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cta_kernel<<<tiles, 256>>>(d, o, L, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    int P = 1;
    while (P < L) P <<= 1;
    cudaMemset(cyc, 0, 8);
    smem_only_kernel<<<1, 256>>>(P, cyc, 7);
    unsigned long long cs;
    cudaDeviceSynchronize();
    cudaMemcpy(&cs, cyc, 8, cudaMemcpyDeviceToHost);
    printf("L=%d P=%d: %d tiles in %.1f us, avg %.0f cycles/tile (incl loads+writes); smem-only sort alone %llu cycles\n",
           L, P, tiles, ms * 1e3, double(c) / tiles, cs);
    cudaFree(d);
    cudaFree(o);
  }
  cudaMemset(cyc, 0, 8);
  warp8_kernel<<<1, 32>>>(cyc, 3);
  unsigned long long cw;
  cudaDeviceSynchronize();
  cudaMemcpy(&cw, cyc, 8, cudaMemcpyDeviceToHost);
  printf("warp_sort<8> alone: %llu cycles\n", cw);
  return 0;
}
