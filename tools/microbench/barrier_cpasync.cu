// Does an outstanding cp.async (DRAM-bound prefetch) slow down grid.sync()?  Per-iteration
// time of: barrier only / prefetch-then-barrier / prefetch(L2 hint)-then-barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void cp16(void* smem, const void* g) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g));
}

__global__ void k(int iters, const char* big, long long stride, int mode) {
  extern __shared__ __align__(16) char sm[];
  cg::grid_group g = cg::this_grid();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int i = 0; i < iters; ++i) {
    const char* src = big + ((gw * 131 + (long long)i * 7919) % 100000) * stride;
    if (mode == 1) {
      for (int k2 = 0; k2 < 19; ++k2) cp16(sm + w * 9728 + 16 * (lane + 32 * k2), src + 16 * (lane + 32 * k2));
      asm volatile("cp.async.commit_group;");
    } else if (mode == 2) {
      for (int l = lane; l < 76; l += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 128 * l));
    } else if (mode == 3) {
      for (int k2 = 0; k2 < 19; ++k2) cp16(sm + w * 9728 + 16 * (lane + 32 * k2), src + 16 * (lane + 32 * k2));
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    g.sync();
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

int main() {
  char* big;
  const long long stride = 10240;
  cudaMalloc(&big, 100000LL * stride + 65536);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 9728);
  for (int blocks : {31, 148})
    for (int mode = 0; mode < 4; ++mode) {
      int iters = 1000;
      void* args[] = {&iters, &big, (void*)&stride, &mode};
      cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 8 * 9728, 0);
      cudaDeviceSynchronize();
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 8 * 9728, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const char* names[] = {"barrier only", "cp.async then barrier", "prefetch.L2 then barrier", "cp.async+wait then barrier"};
      printf("blocks=%3d %-28s %.3f us/iter (%s)\n", blocks, names[mode], 1000 * ms / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
