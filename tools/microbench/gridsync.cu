// Microbenchmark: cost of cooperative-groups grid.sync() vs a hand-rolled sense-reversing
// barrier, as a function of the number of CTAs (B200 sizing of the SGS wave barrier).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

__device__ unsigned int g_count = 0;
__device__ volatile unsigned int g_gen = 0;

__device__ __forceinline__ void my_barrier(unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int target = gen + 1;
    if (atomicAdd(&g_count, 1) == nblocks - 1) {
      g_count = 0;
      __threadfence();
      g_gen = target;
    } else {
      while (g_gen != target) {
      }
    }
    gen = target;
  }
  __syncthreads();
}

__global__ void k_my(int iters, long long* out) {
  unsigned int gen = g_gen;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) my_barrier(gridDim.x, gen);
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

__global__ void k_lat(const double* p, int n, long long* out, double* sink) {
  // pointer-chase-ish: dependent L2 loads with ld.cg
  long long t0 = clock64();
  int idx = 0;
  double acc = 0;
  for (int i = 0; i < 1000; ++i) {
    double v = __ldcg(p + idx);
    acc += v;
    idx = ((int)v + i * 977) % n;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *out = t1 - t0; *sink = acc; }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int threads : {256, 1024})
    for (int blocks : {8, 16, 32, 64, 148, 296}) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg, threads, 0);
      if (blocks > per_sm * 148) continue;
      int iters = 2000;
      void* args[] = {&iters, &d};
      cudaLaunchCooperativeKernel((void*)k_cg, blocks, threads, args, 0, 0);
      cudaDeviceSynchronize();
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, blocks, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_my, blocks, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms2;
      cudaEventElapsedTime(&ms2, a, b);
      printf("threads=%4d blocks=%4d cg.sync=%.3f us  custom=%.3f us  (%s)\n", threads, blocks, 1000 * ms / iters,
             1000 * ms2 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  double* p;
  int n = 1 << 22;
  cudaMalloc(&p, 8 * n);
  cudaMemset(p, 0, 8 * n);
  double* sink;
  cudaMalloc(&sink, 8);
  k_lat<<<1, 32>>>(p, n, d, sink);
  cudaDeviceSynchronize();
  k_lat<<<1, 32>>>(p, n, d, sink);
  long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("dependent ld.cg latency (L2-resident): %.1f cycles = %.3f us at %d kHz\n", cyc / 1000.0,
         cyc / 1000.0 / (clk / 1000.0), clk);
  return 0;
}
