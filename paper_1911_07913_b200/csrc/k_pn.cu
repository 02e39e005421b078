// Projected-Newton baselines on B200 (solvers.hpp:235-300): the block-Jacobi / V-cycle
// preconditioned CG pieces the host-driven PCG (pcg.hpp:17-46) needs, and the matrix-free
// Hessian product and block diagonal (objective.hpp:366-440) on the per-particle tensors of
// k_particle_tensors (kappa*T packed, W_k = F^nT grad w_k).  Deterministic: node sums are
// warp gathers in a fixed order; no float atomics.
#include <cuda_runtime.h>

#include <algorithm>

#include "hot_internal.h"
#include "hot_particle.cuh"

namespace hotb200 {

namespace {

constexpr int kTS = kRecStride;  // per-particle tensor record (hot_particle.cuh)

int pgrid(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  const long long cap = (long long)num_sms() * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

/// z_i = Dinv_i r_i (the block-Jacobi preconditioner, solvers.hpp:272-277).
__global__ void k_block_apply(const double* __restrict__ dinv, const double* __restrict__ r, double* __restrict__ z,
                              int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double* D = dinv + 9 * i;
    const double r0 = r[3 * i], r1 = r[3 * i + 1], r2 = r[3 * i + 2];
    z[3 * i] = D[0] * r0 + D[1] * r1 + D[2] * r2;
    z[3 * i + 1] = D[3] * r0 + D[4] * r1 + D[5] * r2;
    z[3 * i + 2] = D[6] * r0 + D[7] * r1 + D[8] * r2;
  }
}

/// x += alpha p ; r -= alpha Ap  (pcg.hpp:36-37, uncontracted like the CPU)
__global__ void k_pcg_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                         const double* __restrict__ Ap, double alpha, long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    x[t] = __dadd_rn(x[t], __dmul_rn(alpha, p[t]));
    r[t] = __dsub_rn(r[t], __dmul_rn(alpha, Ap[t]));
  }
}

/// p = z + beta p  (pcg.hpp:43)
__global__ void k_pcg_p(double* __restrict__ p, const double* __restrict__ z, double beta, long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    p[t] = __dadd_rn(z[t], __dmul_rn(beta, p[t]));
}

/// Matrix-free product, particle pass (objective.hpp:414-427): dF = sum_k um_k (x) W_k,
/// dP = kappa T : dF, stored SoA [9][np].  um = u with Dirichlet rows zeroed.
__global__ void __launch_bounds__(128) k_mf_particle(ParticlesView P, GridView g, const double* __restrict__ Tu,
                                                     const double* __restrict__ u, double* __restrict__ dP) {
  const long long n = P.n;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const double* T = Tu + p * kTS;
    const int* nb = g.nb27 + 27LL * P.bin[p];
    double dF[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) dF[q] = 0.0;
#pragma unroll
    for (int k = 0; k < 27; ++k) {
      const int node = __ldg(nb + k);
      if (node < 0) continue;  // outside the active set: zero weight (W_k = 0)
      if (g.dir[node]) continue;
      const double w0 = T[kRecW + 3 * k], w1 = T[kRecW + 3 * k + 1], w2 = T[kRecW + 3 * k + 2];
      const double u0 = __ldg(u + 3 * node), u1 = __ldg(u + 3 * node + 1), u2 = __ldg(u + 3 * node + 2);
      dF[0] += u0 * w0;
      dF[1] += u0 * w1;
      dF[2] += u0 * w2;
      dF[3] += u1 * w0;
      dF[4] += u1 * w1;
      dF[5] += u1 * w2;
      dF[6] += u2 * w0;
      dF[7] += u2 * w1;
      dF[8] += u2 * w2;
    }
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 9; ++c) s += T[kRecT + tslot(r, c)] * dF[c];
      dP[r * n + p] = s;
    }
  }
}

/// Matrix-free product, node pass (objective.hpp:429-438): y_i = sum_p dP_p W_{p,a} + m_i um_i,
/// y_i = u_i on Dirichlet rows.  One warp per node over its 27 bins.
__global__ void __launch_bounds__(256) k_mf_node(ParticlesView P, BinsView bins, GridView g,
                                                 const double* __restrict__ Tu, const double* __restrict__ dP,
                                                 const double* __restrict__ u, double* __restrict__ y) {
  const long long n = P.n;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < g.n; i += nw) {
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    warp_node_gather(g, bins, i, lane, [&](int p, int o) {
      const double* W = Tu + (long long)p * kTS + kRecW + 3 * (26 - o);
      const double w0 = W[0], w1 = W[1], w2 = W[2];
      y0 += dP[p] * w0 + dP[n + p] * w1 + dP[2 * n + p] * w2;
      y1 += dP[3 * n + p] * w0 + dP[4 * n + p] * w1 + dP[5 * n + p] * w2;
      y2 += dP[6 * n + p] * w0 + dP[7 * n + p] * w1 + dP[8 * n + p] * w2;
    });
    y0 = warp_sum_d(y0);
    y1 = warp_sum_d(y1);
    y2 = warp_sum_d(y2);
    if (lane == 0) {
      if (g.dir[i]) {
        y[3 * i] = u[3 * i];
        y[3 * i + 1] = u[3 * i + 1];
        y[3 * i + 2] = u[3 * i + 2];
      } else {
        const double m = g.mass[i];
        y[3 * i] = y0 + m * u[3 * i];
        y[3 * i + 1] = y1 + m * u[3 * i + 1];
        y[3 * i + 2] = y2 + m * u[3 * i + 2];
      }
    }
  }
}

/// Block diagonal of the projected system (objective.hpp:366-392) and its inverse: per node
/// sum_p sym(W_a^T kappa T W_a) + m I (I on Dirichlet rows).
__global__ void __launch_bounds__(256) k_mf_diag(ParticlesView P, BinsView bins, GridView g,
                                                 const double* __restrict__ Tu, double* __restrict__ dinv) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < g.n; i += nw) {
    double D[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) D[q] = 0.0;
    warp_node_gather(g, bins, i, lane, [&](int p, int o) {
      const double* T = Tu + (long long)p * kTS;
      const double* W = T + kRecW + 3 * (26 - o);
      const double w[3] = {W[0], W[1], W[2]};
      double C[9];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          double s = 0.0;
#pragma unroll
          for (int f = 0; f < 3; ++f)
#pragma unroll
            for (int gg = 0; gg < 3; ++gg) s += w[f] * T[kRecT + tslot(3 * c + f, 3 * e + gg)] * w[gg];
          C[3 * c + e] = s;
        }
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int e = 0; e < 3; ++e) D[3 * c + e] += 0.5 * (C[3 * c + e] + C[3 * e + c]);
    });
#pragma unroll
    for (int q = 0; q < 9; ++q) D[q] = warp_sum_d(D[q]);
    if (lane == 0) {
      M3 B;
      if (g.dir[i]) {
#pragma unroll
        for (int q = 0; q < 9; ++q) B.m[q] = (q % 4 == 0) ? 1.0 : 0.0;
      } else {
        const double m = g.mass[i];
#pragma unroll
        for (int q = 0; q < 9; ++q) B.m[q] = D[q] + ((q % 4 == 0) ? m : 0.0);
      }
      double det;
      const M3 Bi = m3_inverse(B, &det);
#pragma unroll
      for (int q = 0; q < 9; ++q) dinv[9LL * i + q] = Bi.m[q];
    }
  }
}

}  // namespace

void launch_block_apply(const double* dinv, const double* r, double* z, int n, cudaStream_t s) {
  if (n) { k_block_apply<<<pgrid(n, 256), 256, 0, s>>>(dinv, r, z, n); count_launches(1); }
}
void launch_pcg_xr(double* x, double* r, const double* p, const double* Ap, double alpha, long long n, cudaStream_t s) {
  if (n) { k_pcg_xr<<<pgrid(n, 256), 256, 0, s>>>(x, r, p, Ap, alpha, n); count_launches(1); }
}
void launch_pcg_p(double* p, const double* z, double beta, long long n, cudaStream_t s) {
  if (n) { k_pcg_p<<<pgrid(n, 256), 256, 0, s>>>(p, z, beta, n); count_launches(1); }
}
void launch_mf_multiply(const ParticlesView& P, BinsView bins, GridView g, const double* Tu, const double* u,
                        double* dP, double* y, cudaStream_t s) {
  if (P.n) { k_mf_particle<<<pgrid(P.n, 128), 128, 0, s>>>(P, g, Tu, u, dP); count_launches(1); }
  if (g.n) {
    const int blocks = resident_blocks((const void*)k_mf_node, 256, 0);
    k_mf_node<<<std::min<long long>(blocks, (32LL * g.n + 255) / 256), 256, 0, s>>>(P, bins, g, Tu, dP, u, y);
    count_launches(1);
  }
}
void launch_mf_block_diag_inv(const ParticlesView& P, BinsView bins, GridView g, const double* Tu, double* dinv,
                              cudaStream_t s) {
  if (g.n) {
    const int blocks = resident_blocks((const void*)k_mf_diag, 256, 0);
    k_mf_diag<<<std::min<long long>(blocks, (32LL * g.n + 255) / 256), 256, 0, s>>>(P, bins, g, Tu, dinv);
    count_launches(1);
  }
}

}  // namespace hotb200
