// Level-0 system matrix H = M + dt^2 d2Phi/dx2 on B200 (objective.hpp:318-363).
//
// Stage 1 (one thread per particle): virtual F -> SVD -> dP/dF projected in the diagonal
//   space -> kappa * T stored as the 45-entry upper triangle (SoA, coalesced).
// Stage 2 (one warp per row): gather over the 27 neighbouring particle bins.  Lane l owns
//   stencil position kb = l of the current particle and accumulates the 3x3 pair block into
//   the row's upper-triangle slot in shared memory (distinct slots per particle, so no
//   atomics).  Each unordered block pair is computed once by the row with the smaller
//   index and written together with its transpose, so block (i,j) == block(j,i)^T exactly
//   (the reference's symmetry_error() == 0 invariant).  The mass diagonal and the Dirichlet
//   projection (objective.hpp:133-144) are fused into the write-out.
#include <cuda_runtime.h>

#include "hot_internal.h"
#include "hot_particle.cuh"

namespace hotb200 {

namespace {

constexpr int kAsmWarps = 4;
constexpr int kUpper = 63;  // slots 62..124

__global__ void k_particle_tensors(ParticlesView P, GridView g, double dx, double dt,
                                   const DevMaterial* __restrict__ mats, const double* __restrict__ dv, int project,
                                   double* __restrict__ Tu, int* bad) {
  const long long n = P.n;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    M3 F, Fn;
    if (!virtual_F(P, p, g, dx, dt, dv, nullptr, 0.0, F, Fn)) {
      atomicExch(bad, 1);
      continue;
    }
    const DevMaterial mt = mats[P.mat[p]];
    M3 U, V;
    double s[3];
    svd3(F, U, s, V);
    double T[45];
    fcr_dpdf_projected(U, s, V, mt.mu, mt.lambda, dt * dt * P.vol[p], project != 0, T);
#pragma unroll
    for (int q = 0; q < 45; ++q) Tu[q * n + p] = T[q];
  }
}

__global__ void k_fill_cols(LevelView L, int* __restrict__ cols) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)L.n * kSlotPitch;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / kSlotPitch), s = (int)(t % kSlotPitch);
    int c = -1;
    if (s < kSlots)
      c = dense_lookup(L.map, L.coords[3 * i] + s / 25 - 2, L.coords[3 * i + 1] + (s / 5) % 5 - 2,
                       L.coords[3 * i + 2] + s % 5 - 2);
    cols[t] = c;
  }
}

template <int R, int C>
__device__ __forceinline__ double Tget(const double* T) {
  if constexpr (R <= C)
    return T[R * 9 - (R * (R - 1)) / 2 + (C - R)];
  else
    return T[C * 9 - (C * (C - 1)) / 2 + (R - C)];
}

template <int c, int e>
__device__ __forceinline__ double pair_entry(const double* T, const double wa[3], const double wb[3]) {
  // sum_f wa_f sum_g T[(3c+f),(3e+g)] wb_g  (objective.hpp:304-310)
  double acc = 0.0;
#define HOT_ROW(f)                                                                                      \
  acc += wa[f] * (Tget<3 * c + f, 3 * e>(T) * wb[0] + Tget<3 * c + f, 3 * e + 1>(T) * wb[1] + \
                  Tget<3 * c + f, 3 * e + 2>(T) * wb[2]);
  HOT_ROW(0)
  HOT_ROW(1)
  HOT_ROW(2)
#undef HOT_ROW
  return acc;
}

__global__ void __launch_bounds__(kAsmWarps * 32) k_assemble_rows(ParticlesView P, BinsView bins, GridView g,
                                                                   LevelView L, double dx,
                                                                   const double* __restrict__ Tu) {
  __shared__ double acc_s[kAsmWarps][kUpper * 9];
  __shared__ double stage_s[kAsmWarps][64];  // T (45), F (9), x (3)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* acc = acc_s[wid];
  double* st = stage_s[wid];
  const long long n = P.n;
  const int kb0 = lane / 9, kb1 = (lane / 3) % 3, kb2 = lane % 3;
  const int nwarps = gridDim.x * kAsmWarps;
  for (int i = blockIdx.x * kAsmWarps + wid; i < L.n; i += nwarps) {
    for (int k = lane; k < kUpper * 9; k += 32) acc[k] = 0.0;
    __syncwarp();
    const int ci0 = L.coords[3 * i], ci1 = L.coords[3 * i + 1], ci2 = L.coords[3 * i + 2];
    for (int o = 0; o < 27; ++o) {
      const int o0 = o / 9, o1 = (o / 3) % 3, o2 = o % 3;
      const int j = dense_lookup(L.map, ci0 + o0 - 1, ci1 + o1 - 1, ci2 + o2 - 1);
      if (j < 0) continue;
      // stencil position of row i inside a particle centred at j: ka = 2 - o
      const int ka0 = 2 - o0, ka1 = 2 - o1, ka2 = 2 - o2;
      // slot of node b = base + kb relative to row i: kb - ka + 2 = kb + o
      const int s = 25 * (kb0 + o0) + 5 * (kb1 + o1) + (kb2 + o2);
      const bool mine = lane < 27 && s >= kDiagSlot;
      const int e = bins.start[j + 1];
      for (int t = bins.start[j]; t < e; ++t) {
        const int p = bins.pid[t];
        if (lane < 45) st[lane] = Tu[(long long)lane * n + p];
        if (lane + 32 < 45) st[lane + 32] = Tu[(long long)(lane + 32) * n + p];
        if (lane >= 13 && lane < 22) st[45 + lane - 13] = P.F[(long long)(lane - 13) * n + p];
        if (lane >= 22 && lane < 25) st[54 + lane - 22] = P.x[(long long)(lane - 22) * n + p];
        __syncwarp();
        if (mine) {
          const double c0 = st[54] / dx, c1 = st[55] / dx, c2 = st[56] / dx;
          const int b0 = ci0 + o0 - 2, b1 = ci1 + o1 - 2, b2 = ci2 + o2 - 2;  // stencil base of p
          const double oa0 = c0 - (double)(b0 + ka0), oa1 = c1 - (double)(b1 + ka1), oa2 = c2 - (double)(b2 + ka2);
          const double ob0 = c0 - (double)(b0 + kb0), ob1 = c1 - (double)(b1 + kb1), ob2 = c2 - (double)(b2 + kb2);
          const double wa0 = bspline_w(oa0), wa1 = bspline_w(oa1), wa2 = bspline_w(oa2);
          const double wb0 = bspline_w(ob0), wb1 = bspline_w(ob1), wb2 = bspline_w(ob2);
          if (wa0 * wa1 * wa2 > 0.0 && wb0 * wb1 * wb2 > 0.0) {
            const double ga[3] = {bspline_dw(oa0) / dx * wa1 * wa2, bspline_dw(oa1) / dx * wa0 * wa2,
                                  bspline_dw(oa2) / dx * wa0 * wa1};
            const double gb[3] = {bspline_dw(ob0) / dx * wb1 * wb2, bspline_dw(ob1) / dx * wb0 * wb2,
                                  bspline_dw(ob2) / dx * wb0 * wb1};
            const double* Fm = st + 45;
            double wa[3], wb[3];  // F^T grad
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              wa[a] = Fm[a] * ga[0] + Fm[3 + a] * ga[1] + Fm[6 + a] * ga[2];
              wb[a] = Fm[a] * gb[0] + Fm[3 + a] * gb[1] + Fm[6 + a] * gb[2];
            }
            double C[9];
            C[0] = pair_entry<0, 0>(st, wa, wb);
            C[1] = pair_entry<0, 1>(st, wa, wb);
            C[2] = pair_entry<0, 2>(st, wa, wb);
            C[3] = pair_entry<1, 0>(st, wa, wb);
            C[4] = pair_entry<1, 1>(st, wa, wb);
            C[5] = pair_entry<1, 2>(st, wa, wb);
            C[6] = pair_entry<2, 0>(st, wa, wb);
            C[7] = pair_entry<2, 1>(st, wa, wb);
            C[8] = pair_entry<2, 2>(st, wa, wb);
            if (s == kDiagSlot) {
              const double t01 = 0.5 * (C[1] + C[3]), t02 = 0.5 * (C[2] + C[6]), t12 = 0.5 * (C[5] + C[7]);
              C[1] = C[3] = t01;
              C[2] = C[6] = t02;
              C[5] = C[7] = t12;
            }
            double* a = acc + (s - kDiagSlot) * 9;
#pragma unroll
            for (int k = 0; k < 9; ++k) a[k] += C[k];
          }
        }
        __syncwarp();
      }
    }
    // write-out: upper slots + transposed mirror, mass diagonal, Dirichlet projection
    const bool di = g.dir[i] != 0;
    const double mi = g.mass[i];
    for (int u = lane; u < kUpper; u += 32) {
      const int s = kDiagSlot + u;
      const int col = L.cols[(long long)i * kSlotPitch + s];
      if (col < 0) continue;
      double C[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) C[k] = acc[u * 9 + k];
      const bool zero = di || g.dir[col] != 0;
      if (s == kDiagSlot) {
        if (di) {
#pragma unroll
          for (int k = 0; k < 9; ++k) C[k] = (k % 4 == 0) ? 1.0 : 0.0;
        } else {
          C[0] += mi;
          C[4] += mi;
          C[8] += mi;
        }
      } else if (zero) {
#pragma unroll
        for (int k = 0; k < 9; ++k) C[k] = 0.0;
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) L.H[((long long)i * 9 + k) * kSlotPitch + s] = C[k];
      if (s != kDiagSlot) {
        const int sm = kSlots - 1 - s;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) L.H[((long long)col * 9 + 3 * r + c) * kSlotPitch + sm] = C[3 * c + r];
      }
    }
    __syncwarp();
  }
}

int agrid(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  const long long cap = (long long)num_sms() * 16;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

void launch_particle_tensors(const ParticlesView& P, GridView g, double dx, double dt, const DevMaterial* mats,
                             const double* dv, int project, double* Tu, int* bad_flag, cudaStream_t s) {
  if (P.n == 0) return;
  { k_particle_tensors<<<agrid(P.n, 128), 128, 0, s>>>(P, g, dx, dt, mats, dv, project, Tu, bad_flag); count_launches(1); }
}

void launch_fill_cols(LevelView L, cudaStream_t s) {
  if (L.n == 0) return;
  { k_fill_cols<<<agrid((long long)L.n * kSlotPitch, 256), 256, 0, s>>>(L, const_cast<int*>(L.cols)); count_launches(1); }
}

void launch_assemble_rows(const ParticlesView& P, BinsView bins, GridView g, LevelView L, double dx,
                          const double* Tu, cudaStream_t s) {
  if (L.n == 0) return;
  long long blocks = (L.n + kAsmWarps - 1) / kAsmWarps;
  const long long cap = (long long)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  { k_assemble_rows<<<(int)blocks, kAsmWarps * 32, 0, s>>>(P, bins, g, L, dx, Tu); count_launches(1); }
}

}  // namespace hotb200
