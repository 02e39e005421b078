// Shared per-particle device helpers (virtual deformation gradient).
#pragma once

#include "hot_internal.h"

namespace hotb200 {

/// Virtual deformation gradient (objective.hpp:218-230) at dv + alpha * p.
__device__ __forceinline__ bool virtual_F(const ParticlesView& P, long long p, const GridView& g, double dx, double dt,
                                          const double* __restrict__ dv, const double* __restrict__ pd, double alpha,
                                          M3& F, M3& Fn) {
  const long long n = P.n;
  double c[3];
  int base[3];
  Axis3 ax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    c[a] = P.x[a * n + p] / dx;
    base[a] = stencil_base_1d(c[a]);
    axis_weights(c[a], base[a], ax[a]);
  }
  double G[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) G[k] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double w = ax[0].w[i] * ax[1].w[j] * ax[2].w[k];
        if (w <= 0.0) continue;
        const int node = dense_lookup(g.map, base[0] + i, base[1] + j, base[2] + k);
        const double gr0 = ax[0].dw[i] / dx * ax[1].w[j] * ax[2].w[k];
        const double gr1 = ax[1].dw[j] / dx * ax[0].w[i] * ax[2].w[k];
        const double gr2 = ax[2].dw[k] / dx * ax[0].w[i] * ax[1].w[j];
        double u[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double d = dv[3 * node + a];
          if (pd) d = __dadd_rn(d, __dmul_rn(alpha, pd[3 * node + a]));
          u[a] = g.vel[3 * node + a] + d;
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          G[a * 3] += u[a] * gr0;
          G[a * 3 + 1] += u[a] * gr1;
          G[a * 3 + 2] += u[a] * gr2;
        }
      }
#pragma unroll
  for (int k = 0; k < 9; ++k) Fn.m[k] = P.F[k * n + p];
  M3 A;
#pragma unroll
  for (int k = 0; k < 9; ++k) A.m[k] = ((k % 4 == 0) ? 1.0 : 0.0) + dt * G[k];
  F = m3_mul(A, Fn);
  return m3_finite(F);
}

}  // namespace hotb200
