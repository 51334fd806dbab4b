// Microbenchmark: where does a single-pass (decoupled look-back) scan spend its time at
// ~1M items on B200? Variants: empty kernel, counter-only, full scan with look-back, scan with
// the prefix taken from a precomputed array (no look-back).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int K>
__device__ uint32_t look_back(const uint32_t* status, int tile) {
  uint32_t prefix = 0;
  int j = tile - 1;
  while (true) {
    uint32_t s[K];
#pragma unroll
    for (int q = 0; q < K; ++q) s[q] = j - q >= 0 ? ld_volatile(status + (j - q)) : 0u;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      uint32_t v = s[q];
      while ((v & 3u) == 0u) v = ld_volatile(status + (j - q));
      prefix += v >> 2;
      if ((v & 3u) == 2u) return prefix;
    }
    j -= K;
  }
}

__global__ void empty_kernel(int* x) { if (threadIdx.x == 12345) x[0] = 1; }
__global__ void counter_kernel(uint32_t* c, uint32_t* out) {
  __shared__ uint32_t t;
  if (threadIdx.x == 0) t = atomicAdd(c, 1u);
  __syncthreads();
  if (threadIdx.x == 0 && t == 0xFFFFFFFF) out[0] = 1;
}

template <int K, bool LB>
__global__ void __launch_bounds__(1024) scan_kernel(const uint32_t* in, uint32_t* out, int n, uint32_t* status,
                                                   uint32_t* counter, const uint32_t* pre) {
  __shared__ uint32_t s_tile, s_prefix, s_warp[32];
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const int tile = s_tile;
  const int r0 = tile * 8192 + threadIdx.x * 8;
  uint32_t c[8], sum = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i] = r0 + i < n ? in[r0 + i] : 0u; sum += c[i]; }
  // block scan
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { uint32_t y = __shfl_up_sync(~0u, x, o); if (lane >= o) x += y; }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t v = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { uint32_t y = __shfl_up_sync(~0u, v, o); if (lane >= o) v += y; }
    s_warp[lane] = v;
  }
  __syncthreads();
  const uint32_t tot = s_warp[31];
  const uint32_t ex = (w ? s_warp[w - 1] : 0u) + x - sum;
  if (threadIdx.x == 0) {
    uint32_t prefix = 0;
    if (LB) {
      if (tile == 0) st_volatile(status, (tot << 2) | 2u);
      else {
        st_volatile(status + tile, (tot << 2) | 1u);
        prefix = look_back<K>(status, tile);
        st_volatile(status + tile, ((prefix + tot) << 2) | 2u);
      }
    } else {
      prefix = pre[tile];
    }
    s_prefix = prefix;
  }
  __syncthreads();
  uint32_t pos = s_prefix + ex;
#pragma unroll
  for (int i = 0; i < 8; ++i) { if (r0 + i < n) out[r0 + i] = pos; pos += c[i]; }
}

int main() {
  const int n = 1 << 20, tiles = (n + 8191) / 8192;
  uint32_t *in, *out, *status, *counter, *pre;
  int* x;
  cudaMalloc(&in, n * 4); cudaMalloc(&out, n * 4); cudaMalloc(&status, tiles * 4 + 64);
  cudaMalloc(&counter, 64); cudaMalloc(&pre, tiles * 4); cudaMalloc(&x, 4);
  std::vector<uint32_t> h(n, 1);
  cudaMemcpy(in, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemset(pre, 0, tiles * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 10; ++i) fn();
    cudaDeviceSynchronize();
    const int reps = 200;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %8.2f us/iter (incl. memsets if any)\n", name, 1000.0f * ms / reps);
  };
  timeit("empty 128x1024", [&] { empty_kernel<<<tiles, 1024>>>(x); });
  timeit("memset x2 only", [&] { cudaMemsetAsync(status, 0, tiles * 4 + 8); cudaMemsetAsync(counter, 0, 4); });
  timeit("counter 128x1024 (+memset)", [&] { cudaMemsetAsync(counter, 0, 4); counter_kernel<<<tiles, 1024>>>(counter, out); });
  timeit("scan no-lookback (+memset)", [&] { cudaMemsetAsync(counter, 0, 4); scan_kernel<1, false><<<tiles, 1024>>>(in, out, n, status, counter, pre); });
  timeit("scan lookback K=1 (+2 memsets)", [&] { cudaMemsetAsync(status, 0, tiles * 4 + 8); cudaMemsetAsync(counter, 0, 4); scan_kernel<1, true><<<tiles, 1024>>>(in, out, n, status, counter, pre); });
  timeit("scan lookback K=16 (+2 memsets)", [&] { cudaMemsetAsync(status, 0, tiles * 4 + 8); cudaMemsetAsync(counter, 0, 4); scan_kernel<16, true><<<tiles, 1024>>>(in, out, n, status, counter, pre); });
  cudaMemcpy(h.data(), out, n * 4, cudaMemcpyDeviceToHost);
  printf("check out[n-1] = %u (expect %d)\n", h[n - 1], n - 1);
  return 0;
}
