// zero-copy (mapped pinned host) read bandwidth by access pattern
#include <cstdio>
#include <cuda_runtime.h>
__global__ void per_lane_rows(const float4* __restrict__ src, int64_t rows, int row_f4, float* out) {
  // each thread reads its own row of row_f4 float4 (like SH AoS per Gaussian)
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float acc = 0.f;
  if (i < rows) for (int j = 0; j < row_f4; ++j) { float4 v = __ldg(src + i * row_f4 + j); acc += v.x + v.y + v.z + v.w; }
  if (acc == 1234.5f) out[0] = acc;
}
__global__ void warp_rows(const float4* __restrict__ src, int64_t rows, int row_f4, float* out) {
  // each warp reads 32 consecutive rows cooperatively: lane l reads float4 l, l+32, ... of the block
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; int lane = threadIdx.x & 31;
  float acc = 0.f;
  int64_t base = w * 32 * row_f4, n = 32 * (int64_t)row_f4;
  if (w * 32 < rows) for (int64_t j = lane; j < n; j += 32) { float4 v = __ldg(src + base + j); acc += v.x + v.y + v.z + v.w; }
  if (acc == 1234.5f) out[0] = acc;
}
__global__ void sparse_rows(const float4* __restrict__ src, int64_t rows, int row_f4, float* out, int keep_mod) {
  // warp-cooperative per selected row: for each selected row (1 in keep_mod ... pseudo-random), the warp loads it with row_f4 lanes
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int r = 0; r < 32; ++r) {
    int64_t row = w * 32 + r; if (row >= rows) break;
    unsigned h = (unsigned)row * 2654435761u; if ((h >> 16) % keep_mod) continue;
    if (lane < row_f4) { float4 v = __ldg(src + row * row_f4 + lane); acc += v.x + v.y + v.z + v.w; }
  }
  if (acc == 1234.5f) out[0] = acc;
}
__global__ void sparse_lane(const float4* __restrict__ src, int64_t rows, int row_f4, float* out, int keep_mod) {
  int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float acc = 0.f;
  if (row < rows) { unsigned h = (unsigned)row * 2654435761u; if (!((h >> 16) % keep_mod)) for (int j = 0; j < row_f4; ++j) { float4 v = __ldg(src + row * row_f4 + j); acc += v.x + v.y + v.z + v.w; } }
  if (acc == 1234.5f) out[0] = acc;
}
int main() {
  const int64_t rows = 1 << 20; const int row_f4 = 12;  // 192 B rows, 201 MB
  size_t bytes = rows * row_f4 * 16;
  float4* h; cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  memset(h, 0, bytes);
  float4* d; cudaHostGetDevicePointer(&d, h, 0);
  float4* dev; cudaMalloc(&dev, bytes);
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto f, double useful) {
    for (int it = 0; it < 2; ++it) f();
    cudaEventRecord(e0); for (int it = 0; it < 5; ++it) f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-40s %8.3f ms  %7.1f GB/s useful\n", name, ms, useful / ms / 1e6);
  };
  run("memcpy H2D", [&] { cudaMemcpyAsync(dev, h, bytes, cudaMemcpyHostToDevice); }, bytes);
  run("per-lane 192B rows", [&] { per_lane_rows<<<rows / 256, 256>>>(d, rows, row_f4, out); }, bytes);
  run("warp-coalesced rows", [&] { warp_rows<<<rows / 256, 256>>>(d, rows, row_f4, out); }, bytes);
  for (int km : {2, 3}) {
    double useful = 0; for (int64_t r = 0; r < rows; ++r) { unsigned hh = (unsigned)r * 2654435761u; if (!((hh >> 16) % km)) useful += row_f4 * 16; }
    char nm[64];
    snprintf(nm, 64, "sparse 1/%d per-lane", km); run(nm, [&] { sparse_lane<<<rows / 256, 256>>>(d, rows, row_f4, out, km); }, useful);
    snprintf(nm, 64, "sparse 1/%d warp-per-row", km); run(nm, [&] { sparse_rows<<<rows / 256, 256>>>(d, rows, row_f4, out, km); }, useful);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
