// Measured FP64 (DFMA) throughput of this B200: 148 SMs x independent FMA chains.
#include <cstdio>
__global__ void k(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 42.0) out[0] = a0;
}
int main() {
  double* d;
  cudaMalloc(&d, 8);
  const int iters = 20000, blocks = 148 * 8, threads = 256;
  k<<<blocks, threads>>>(d, 100);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<<<blocks, threads>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  const double flops = 2.0 * 8 * iters * (double)blocks * threads;
  printf("{\"fp64_fma_tflops\": %.2f, \"ms\": %.3f}\n", flops / best / 1e9, best);
}
