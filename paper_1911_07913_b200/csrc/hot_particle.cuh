// Shared per-particle device helpers (virtual deformation gradient).
#pragma once

#include <type_traits>

#include "hot_internal.h"

namespace hotb200 {

/// A particle's tensor record (k_particle_tensors; 1008 B = 63 x 16 B): W_k[g] = (F^nT grad w_k)[g]
/// at kRecW + 3k + g for the 27 stencil positions, then kappa*T (45 packed entries) at
/// kRecT + tslot(r, c).  W comes first so that the suffix a row gather needs (positions k >= kmin,
/// and T) is one contiguous range.
constexpr int kRecW = 0;
constexpr int kRecT = 81;
constexpr int kRecStride = 126;

/// Slot of kappa*T[r][c] (symmetric 9x9) in the record's T part (k_particle_tensors,
/// read by k_assemble_rows and the matrix-free PN kernels): the packed upper-triangle index,
/// permuted so that the assembly's B-fragment loads (for each f, the lanes' T[3c+f][3e+g] and
/// T[6+f][6+g]) fall on distinct shared-memory bank pairs within each half-warp.  The
/// permutation came from a small backtracking search; any bijection of 0..44 is correct.
__host__ __device__ constexpr int tperm(int q) {
  constexpr int perm[45] = {44, 2, 26, 23, 25, 3, 24, 22, 29, 31, 6, 36, 42, 37, 12, 16, 43, 18, 33, 39, 20, 9, 30, 15, 35, 34, 10, 0, 7, 38, 17, 40, 4, 27, 19, 28, 1, 21, 41, 5, 14, 32, 8, 13, 11};
  return perm[q];
}
/// Inverse of tperm: the packed index stored at T slot t.
__host__ __device__ constexpr int tperm_inv(int t) {
  int q = 0;
  while (q < 45 && tperm(q) != t) ++q;
  return q;
}
__host__ __device__ constexpr int tpack_index(int r, int c) {
  return r > c ? c * 9 - c * (c - 1) / 2 + (r - c) : r * 9 - r * (r - 1) / 2 + (c - r);
}
__host__ __device__ constexpr int tslot(int r, int c) { return tperm(tpack_index(r, c)); }
static_assert(tslot(0, 0) != tslot(8, 8) && tslot(3, 5) == tslot(5, 3), "record slot table");

/// Virtual deformation gradient (objective.hpp:218-230) from precomputed nodal velocities
/// u = vel + (dv + alpha p) (launch_node_u).  The particle's stencil nodes come from its bin's
/// 27-neighbour table (P.bin, g.nb27): no lattice lookups per particle.
__device__ __forceinline__ bool virtual_F(const ParticlesView& P, long long p, const GridView& g, double dx, double dt,
                                          const double* __restrict__ u, M3& F, M3& Fn) {
  const long long n = P.n;
  double c[3];
  int base[3];
  Axis3 ax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    c[a] = P.x[a * n + p] / dx;
    base[a] = stencil_base_1d(c[a]);
    axis_weights(c[a], base[a], ax[a]);
    axis_dw_over_dx(ax[a], dx);
  }
  const int* nb = g.nb27 + 27LL * P.bin[p];
  double G[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) G[k] = 0.0;
  // The x-axis loop stays rolled (select instead of indexing) to keep the kernels that inline
  // this small enough for the instruction cache; the 9 (y, z) nodes per x-plane are unrolled.
#pragma unroll 1
  for (int i = 0; i < 3; ++i) {
    const double wi = i == 0 ? ax[0].w[0] : (i == 1 ? ax[0].w[1] : ax[0].w[2]);
    const double dwi = i == 0 ? ax[0].dw[0] : (i == 1 ? ax[0].dw[1] : ax[0].dw[2]);
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double w = wi * ax[1].w[j] * ax[2].w[k];
        if (w <= 0.0) continue;
        const int node = __ldg(nb + 9 * i + 3 * j + k);
        const double gr0 = dwi * ax[1].w[j] * ax[2].w[k];
        const double gr1 = ax[1].dw[j] * wi * ax[2].w[k];
        const double gr2 = ax[2].dw[k] * wi * ax[1].w[j];
        const double u0 = __ldg(u + 3 * node), u1 = __ldg(u + 3 * node + 1), u2 = __ldg(u + 3 * node + 2);
        G[0] += u0 * gr0;
        G[1] += u0 * gr1;
        G[2] += u0 * gr2;
        G[3] += u1 * gr0;
        G[4] += u1 * gr1;
        G[5] += u1 * gr2;
        G[6] += u2 * gr0;
        G[7] += u2 * gr1;
        G[8] += u2 * gr2;
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

/// Warp-cooperative node gather: calls body(p) -- or body(p, o) with o the bin offset index
/// (bin node = i + o - 1, lexicographic in {0,1,2}^3; node i is stencil position 26 - o of
/// that bin) -- for every particle slot p in the 27 bins around node i, lanes striding over
/// the concatenated slot list, so consecutive lanes read consecutive particles.  All 32 lanes
/// must call it.
template <class Body>
__device__ __forceinline__ void warp_node_gather(const GridView& g, const BinsView& bins, int i, int lane, Body body) {
  int st = 0, cnt = 0;
  if (lane < 27) {
    const int j = __ldg(g.nb27 + 27LL * i + lane);
    if (j >= 0) {
      st = __ldg(bins.start + j);
      cnt = __ldg(bins.start + j + 1) - st;
    }
  }
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 26);
  for (int base = 0; base < total; base += 32) {
    const int f = base + lane;
    int o = 0;  // first bin whose inclusive count exceeds f
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const int probe = min(o + s - 1, 26);
      const int v = __shfl_sync(0xffffffffu, incl, probe);
      if (o + s - 1 <= 26 && v <= f) o += s;
    }
    o = min(o, 26);
    const int so = __shfl_sync(0xffffffffu, st, o);
    const int eo = __shfl_sync(0xffffffffu, incl - cnt, o);
    if (f < total) {
      if constexpr (std::is_invocable_v<Body, int, int>)
        body(so + (f - eo), o);
      else
        body(so + (f - eo));
    }
  }
}

/// Deterministic warp sum (xor butterfly); lane 0's value is the result.
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace hotb200
