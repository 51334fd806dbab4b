// Microbenchmark: cost of cooperative_groups grid.sync() on B200 for persistent kernels
// (one or two CTAs per SM), and of a persistent kernel doing R phases separated by syncs.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void phases_kernel(int rounds, unsigned* out) {
  cg::grid_group g = cg::this_grid();
  unsigned acc = 0;
  for (int r = 0; r < rounds; ++r) {
    acc += threadIdx.x ^ r;
    g.sync();
  }
  if (acc == 0xFFFFFFFFu) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    for (int per_sm : {1, 2}) {
      int maxb = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, phases_kernel, threads, 0);
      if (per_sm > maxb) continue;
      dim3 grid(sms * per_sm), block(threads);
      for (int rounds : {0, 1, 16}) {
        void* args[] = {&rounds, &out};
        for (int i = 0; i < 5; ++i) cudaLaunchCooperativeKernel((void*)phases_kernel, grid, block, args, 0, 0);
        cudaDeviceSynchronize();
        const int reps = 100;
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i) cudaLaunchCooperativeKernel((void*)phases_kernel, grid, block, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("threads %4d ctas/sm %d rounds %2d: %7.2f us per launch\n", threads, per_sm, rounds, 1000 * ms / reps);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
