// Latency of one warp computing one 125-slot block-row product (the coarse SGS row update)
// with different load flavours; synthetic 32^3 lattice, H in DRAM or L2.
#include <cstdio>
#include <vector>
constexpr int P = 128;
__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int MODE>
__global__ void k(const int* cols, const double* H, double* x, int* rows, int nrows, long long* out) {
  const int lane = threadIdx.x & 31;
  long long tot = 0;
  double sink = 0;
  for (int t = 0; t < nrows; ++t) {
    const int i = rows[t];
    long long t0 = clock64();
    const int* c = cols + (long long)i * P;
    const double* h = H + (long long)i * 9 * P;
    int cc[4];
    for (int kk = 0; kk < 4; ++kk) cc[kk] = __ldg(c + lane + 32 * kk);
    double xv[4][3];
    for (int kk = 0; kk < 4; ++kk) {
      const double* xp = x + 3 * (cc[kk] >= 0 ? cc[kk] : 0);
      for (int a = 0; a < 3; ++a) xv[kk][a] = MODE & 1 ? __ldcg(xp + a) : __ldg(xp + a);
    }
    double a0 = 0, a1 = 0, a2 = 0;
    for (int kk = 0; kk < 4; ++kk) {
      const int s = lane + 32 * kk;
      double hv[9];
      for (int e = 0; e < 9; ++e) hv[e] = MODE & 2 ? __ldcs(h + e * P + s) : __ldg(h + e * P + s);
      a0 += hv[0] * xv[kk][0] + hv[1] * xv[kk][1] + hv[2] * xv[kk][2];
      a1 += hv[3] * xv[kk][0] + hv[4] * xv[kk][1] + hv[5] * xv[kk][2];
      a2 += hv[6] * xv[kk][0] + hv[7] * xv[kk][1] + hv[8] * xv[kk][2];
    }
    a0 = wsum(a0); a1 = wsum(a1); a2 = wsum(a2);
    if (lane == 0) x[3 * i] = a0 + a1 + a2;
    __syncwarp();
    sink += a0;
    tot += clock64() - t0;
  }
  if (lane == 0) { out[0] = tot / nrows; out[1] = (long long)sink; }
}
int main() {
  const int N = 32, n = N * N * N;
  std::vector<int> cols((size_t)n * P, -1);
  for (int i = 0; i < N; ++i) for (int j = 0; j < N; ++j) for (int kk = 0; kk < N; ++kk) {
    int r = (i * N + j) * N + kk;
    for (int s = 0; s < 125; ++s) {
      int a = i + s / 25 - 2, b = j + (s / 5) % 5 - 2, c = kk + s % 5 - 2;
      if (a >= 0 && a < N && b >= 0 && b < N && c >= 0 && c < N) cols[(size_t)r * P + s] = (a * N + b) * N + c;
    }
  }
  int *dc, *drows; double *dH, *dx; long long* dout;
  cudaMalloc(&dc, cols.size() * 4); cudaMemcpy(dc, cols.data(), cols.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&dH, (size_t)n * 9 * P * 8); cudaMemset(dH, 0, (size_t)n * 9 * P * 8);
  cudaMalloc(&dx, (size_t)n * 3 * 8); cudaMemset(dx, 0, (size_t)n * 3 * 8);
  std::vector<int> rows(200);
  for (int t = 0; t < 200; ++t) rows[t] = (t * 7919 + 13) % n;
  cudaMalloc(&drows, 800); cudaMemcpy(drows, rows.data(), 800, cudaMemcpyHostToDevice);
  cudaMalloc(&dout, 16);
  long long h[2];
  auto run = [&](auto kern, const char* name) {
    kern<<<1, 32>>>(dc, dH, dx, drows, 200, dout);  // cold (DRAM)
    cudaMemcpy(h, dout, 16, cudaMemcpyDeviceToHost);
    long long cold = h[0];
    kern<<<1, 32>>>(dc, dH, dx, drows, 200, dout);  // warm (L2)
    cudaMemcpy(h, dout, 16, cudaMemcpyDeviceToHost);
    printf("%-28s cold %6lld cyc (%.2f us)  warm %6lld cyc (%.2f us)\n", name, cold, cold / 1965.0, h[0], h[0] / 1965.0);
  };
  run(k<0>, "ldg x, ldg H");
  run(k<1>, "ldcg x, ldg H");
  run(k<2>, "ldg x, ldcs H");
  run(k<3>, "ldcg x, ldcs H");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
