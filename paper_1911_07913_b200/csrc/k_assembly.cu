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

constexpr int kTensorStride = 72;  // per particle (bin order): 45 upper-triangle kappa*T, 9 w, 9 dw/dx, 9 F^n

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
    double* out = Tu + p * kTensorStride;
#pragma unroll
    for (int q = 0; q < 45; ++q) out[q] = T[q];
    // per-axis stencil weights and derivatives (grid.hpp:22-73) for the row gather
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double c = P.x[a * n + p] / dx;
      Axis3 ax;
      axis_weights(c, stencil_base_1d(c), ax);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        out[45 + 3 * a + k] = ax.w[k];
        out[54 + 3 * a + k] = ax.dw[k] / dx;
      }
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) out[63 + k] = Fn.m[k];
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

__constant__ unsigned char c_tri_r[45], c_tri_c[45];

/// Row gather (objective.hpp:331-357).  Per (row a, particle p) the warp first forms
/// M[c][e][g] = sum_f wa_f T[(3c+f),(3e+g)] (27 lanes, 3 FMA each), then every lane owning an
/// upper-triangle stencil position kb contracts C[c][e] = sum_g M[c][e][g] wb_g (27 FMA).
__global__ void __launch_bounds__(kAsmWarps * 32) k_assemble_rows(BinsView bins, GridView g, LevelView L,
                                                                   const double* __restrict__ Tu) {
  __shared__ double acc_s[kAsmWarps][kUpper * 9];
  __shared__ double T_s[kAsmWarps][81];
  __shared__ double X_s[kAsmWarps][28];  // w[9], dwdx[9], F[9]
  __shared__ double M_s[kAsmWarps][28];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* acc = acc_s[wid];
  double* Ts = T_s[wid];
  double* Xs = X_s[wid];
  double* Ms = M_s[wid];
  const int kb0 = lane / 9, kb1 = (lane / 3) % 3, kb2 = lane % 3;
  // lane's M entry (c,e,g) = (kb0,kb1,kb2): T indices for f = 0..2
  const int mrow = 3 * kb0, mcol = 3 * kb1 + kb2;
  const int nwarps = gridDim.x * kAsmWarps;
  for (int i = blockIdx.x * kAsmWarps + wid; i < L.n; i += nwarps) {
    for (int k = lane; k < kUpper * 9; k += 32) acc[k] = 0.0;
    const int ci0 = L.coords[3 * i], ci1 = L.coords[3 * i + 1], ci2 = L.coords[3 * i + 2];
    for (int o = 0; o < 27; ++o) {
      const int o0 = o / 9, o1 = (o / 3) % 3, o2 = o % 3;
      const int j = dense_lookup(L.map, ci0 + o0 - 1, ci1 + o1 - 1, ci2 + o2 - 1);
      if (j < 0) continue;
      const int ka0 = 2 - o0, ka1 = 2 - o1, ka2 = 2 - o2;
      const int s = 25 * (kb0 + o0) + 5 * (kb1 + o1) + (kb2 + o2);
      const bool mine = lane < 27 && s >= kDiagSlot;
      const int e = bins.start[j + 1];
      for (int t = bins.start[j]; t < e; ++t) {
        const double* pt = Tu + (long long)t * kTensorStride;  // bin order: slot t is the particle
        __syncwarp();
        {
          const double v0 = pt[lane];
          const double v1 = pt[32 + lane];
          const double v2 = lane < 8 ? pt[64 + lane] : 0.0;
          const int r0 = c_tri_r[lane], q0 = c_tri_c[lane];
          Ts[r0 * 9 + q0] = v0;
          Ts[q0 * 9 + r0] = v0;
          if (lane < 13) {
            const int r1 = c_tri_r[32 + lane], q1 = c_tri_c[32 + lane];
            Ts[r1 * 9 + q1] = v1;
            Ts[q1 * 9 + r1] = v1;
          } else {
            Xs[lane - 13] = v1;  // q = 45..63
          }
          if (lane < 8) Xs[19 + lane] = v2;  // q = 64..71
        }
        __syncwarp();
        // row node a: weight and wa = F^T grad w_a
        const double wa0 = Xs[ka0], wa1 = Xs[3 + ka1], wa2 = Xs[6 + ka2];
        if (!(wa0 * wa1 * wa2 > 0.0)) continue;
        const double ga0 = Xs[9 + ka0] * wa1 * wa2, ga1 = Xs[12 + ka1] * wa0 * wa2, ga2 = Xs[15 + ka2] * wa0 * wa1;
        const double* Fm = Xs + 18;
        const double wA0 = Fm[0] * ga0 + Fm[3] * ga1 + Fm[6] * ga2;
        const double wA1 = Fm[1] * ga0 + Fm[4] * ga1 + Fm[7] * ga2;
        const double wA2 = Fm[2] * ga0 + Fm[5] * ga1 + Fm[8] * ga2;
        if (lane < 27)
          Ms[lane] = wA0 * Ts[mrow * 9 + mcol] + wA1 * Ts[(mrow + 1) * 9 + mcol] + wA2 * Ts[(mrow + 2) * 9 + mcol];
        __syncwarp();
        if (mine) {
          const double wb0 = Xs[kb0], wb1 = Xs[3 + kb1], wb2 = Xs[6 + kb2];
          if (wb0 * wb1 * wb2 > 0.0) {
            const double gb0 = Xs[9 + kb0] * wb1 * wb2, gb1 = Xs[12 + kb1] * wb0 * wb2, gb2 = Xs[15 + kb2] * wb0 * wb1;
            const double wB0 = Fm[0] * gb0 + Fm[3] * gb1 + Fm[6] * gb2;
            const double wB1 = Fm[1] * gb0 + Fm[4] * gb1 + Fm[7] * gb2;
            const double wB2 = Fm[2] * gb0 + Fm[5] * gb1 + Fm[8] * gb2;
            double C[9];
#pragma unroll
            for (int ce = 0; ce < 9; ++ce) C[ce] = Ms[3 * ce] * wB0 + Ms[3 * ce + 1] * wB1 + Ms[3 * ce + 2] * wB2;
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
      }
    }
    __syncwarp();
    // write-out: upper slots + transposed mirror, mass diagonal, Dirichlet projection
    const bool di = g.dir[i] != 0;
    const double mi = g.mass[i];
    for (int s = lane; s < kSlotPitch; s += 32) {  // inactive / pad slots hold zeros
      if (s >= kSlots || L.cols[(long long)i * kSlotPitch + s] < 0)
#pragma unroll
        for (int k = 0; k < 9; ++k) L.H[((long long)i * 9 + k) * kSlotPitch + s] = 0.0;
    }
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
  static bool tri_ready = false;
  if (!tri_ready) {
    unsigned char r[45], c[45];
    int q = 0;
    for (int a = 0; a < 9; ++a)
      for (int b = a; b < 9; ++b) {
        r[q] = (unsigned char)a;
        c[q] = (unsigned char)b;
        ++q;
      }
    cudaMemcpyToSymbol(c_tri_r, r, 45);
    cudaMemcpyToSymbol(c_tri_c, c, 45);
    tri_ready = true;
  }
  (void)dx;
  long long blocks = (L.n + kAsmWarps - 1) / kAsmWarps;
  const long long cap = (long long)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  { k_assemble_rows<<<(int)blocks, kAsmWarps * 32, 0, s>>>(bins, g, L, Tu); count_launches(1); }
}

}  // namespace hotb200
