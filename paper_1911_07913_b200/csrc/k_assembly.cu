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

constexpr int kTensorStride = 162;  // per particle (bin order): kappa*T (81, full symmetric), W (27 x 3): W_k = F^nT grad w_k (0 where w_k = 0)

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
    {
      int q = 0;
#pragma unroll
      for (int r = 0; r < 9; ++r)
#pragma unroll
        for (int c = r; c < 9; ++c) {
          out[r * 9 + c] = T[q];
          out[c * 9 + r] = T[q];
          ++q;
        }
    }
    // W_k = F^nT grad w_k for the 27 stencil nodes (grid.hpp:58-73, objective.hpp:337-339); nodes
    // with zero weight get W = 0, which is how the reference skips them (transfer.hpp:36-37)
    Axis3 ax[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double c = P.x[a * n + p] / dx;
      axis_weights(c, stencil_base_1d(c), ax[a]);
    }
#pragma unroll
    for (int k = 0; k < 27; ++k) {
      const int k0 = k / 9, k1 = (k / 3) % 3, k2 = k % 3;
      const double w0 = ax[0].w[k0], w1 = ax[1].w[k1], w2 = ax[2].w[k2];
      double W[3] = {0.0, 0.0, 0.0};
      if (w0 * w1 * w2 > 0.0) {
        const double g0 = ax[0].dw[k0] / dx * w1 * w2, g1 = ax[1].dw[k1] / dx * w0 * w2, g2 = ax[2].dw[k2] / dx * w0 * w1;
#pragma unroll
        for (int q = 0; q < 3; ++q) W[q] = Fn.m[q] * g0 + Fn.m[3 + q] * g1 + Fn.m[6 + q] * g2;
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) out[81 + 3 * k + q] = W[q];
    }
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

/// Row gather (objective.hpp:331-357).  Per (row a, particle p) the warp first forms
/// M[c][e][g] = sum_f wa_f T[(3c+f),(3e+g)] (27 lanes, 3 FMA each), then every lane owning an
/// upper-triangle stencil position kb contracts C[c][e] = sum_g M[c][e][g] wb_g (27 FMA).
/// A bin's particles are contiguous (bin order), so they are staged in chunks with cp.async,
/// and within a bin a lane's target slot is fixed: its block accumulates in registers and is
/// folded into the row's shared-memory accumulator once per bin.
constexpr int kAsmChunk = 4;

__device__ __forceinline__ void asm_cp16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}

__global__ void __launch_bounds__(kAsmWarps * 32) k_assemble_rows(BinsView bins, GridView g, LevelView L,
                                                                   const double* __restrict__ Tu) {
  __shared__ double acc_s[kAsmWarps][kUpper * 9];
  __shared__ __align__(16) double S_s[kAsmWarps][kAsmChunk * kTensorStride];  // T | w | dw/dx | F per particle
  __shared__ __align__(16) double M_s[kAsmWarps][36];                          // M[ce][g], g padded to 4
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* acc = acc_s[wid];
  double* Ms = M_s[wid];
  const int kb0 = lane / 9, kb1 = (lane / 3) % 3, kb2 = lane % 3;
  const int tb = 27 * kb0 + 3 * kb1 + kb2;  // lane's M entry (c,e,g) reads T[(3c+f)*9 + 3e+g]
  const int mslot = 4 * (3 * kb0 + kb1) + kb2;
  const int nwarps = gridDim.x * kAsmWarps;
  for (int i = blockIdx.x * kAsmWarps + wid; i < L.n; i += nwarps) {
    for (int k = lane; k < kUpper * 9; k += 32) acc[k] = 0.0;
    const int ci0 = L.coords[3 * i], ci1 = L.coords[3 * i + 1], ci2 = L.coords[3 * i + 2];
    for (int o = 0; o < 27; ++o) {
      const int o0 = o / 9, o1 = (o / 3) % 3, o2 = o % 3;
      const int j = dense_lookup(L.map, ci0 + o0 - 1, ci1 + o1 - 1, ci2 + o2 - 1);
      if (j < 0) continue;
      const int ka3 = 3 * (9 * (2 - o0) + 3 * (2 - o1) + (2 - o2));
      const int s = 25 * (kb0 + o0) + 5 * (kb1 + o1) + (kb2 + o2);
      const bool mine = lane < 27 && s >= kDiagSlot;
      double Cr[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) Cr[k] = 0.0;
      const int pb = bins.start[j], pe = bins.start[j + 1];
      for (int c0 = pb; c0 < pe; c0 += kAsmChunk) {
        const int cnt = min(kAsmChunk, pe - c0);
        __syncwarp();
        {
          const char* src = reinterpret_cast<const char*>(Tu + (long long)c0 * kTensorStride);
          char* dst = reinterpret_cast<char*>(S_s[wid]);
          const int chunks = cnt * kTensorStride * 8 / 16;
          for (int q = lane; q < chunks; q += 32) asm_cp16(dst + 16 * q, src + 16 * q);
          asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        for (int t = 0; t < cnt; ++t) {
          const double* Ts = S_s[wid] + t * kTensorStride;
          const double* Ws = Ts + 81;
          const double wA0 = Ws[ka3], wA1 = Ws[ka3 + 1], wA2 = Ws[ka3 + 2];  // zero when w_a = 0
          __syncwarp();
          if (lane < 27) Ms[mslot] = wA0 * Ts[tb] + wA1 * Ts[tb + 9] + wA2 * Ts[tb + 18];
          __syncwarp();
          if (mine) {
            const double wB0 = Ws[3 * lane], wB1 = Ws[3 * lane + 1], wB2 = Ws[3 * lane + 2];
#pragma unroll
            for (int ce = 0; ce < 9; ++ce) {
              const double2 m01 = *reinterpret_cast<const double2*>(Ms + 4 * ce);
              const double m2 = Ms[4 * ce + 2];
              Cr[ce] += m01.x * wB0 + m01.y * wB1 + m2 * wB2;
            }
          }
        }
      }
      if (mine) {
        if (s == kDiagSlot) {  // symmetrise the diagonal contribution (objective.hpp:349-351)
          const double t01 = 0.5 * (Cr[1] + Cr[3]), t02 = 0.5 * (Cr[2] + Cr[6]), t12 = 0.5 * (Cr[5] + Cr[7]);
          Cr[1] = Cr[3] = t01;
          Cr[2] = Cr[6] = t02;
          Cr[5] = Cr[7] = t12;
        }
        double* ap = acc + (s - kDiagSlot) * 9;
#pragma unroll
        for (int k = 0; k < 9; ++k) ap[k] += Cr[k];
      }
    }
    __syncwarp();
    // write-out: upper slots + transposed mirror, mass diagonal, Dirichlet projection
    const bool di = g.dir[i] != 0;
    const double mi = g.mass[i];
    for (int s = lane; s < kSlotPitch; s += 32) {  // inactive / pad slots hold zeros
      if (s >= kSlots || L.cols[(long long)i * kSlotPitch + s] < 0)
#pragma unroll
        for (int k = 0; k < 9; ++k) __stcs(L.H + ((long long)i * 9 + k) * kSlotPitch + s, 0.0);
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
      for (int k = 0; k < 9; ++k) __stcs(L.H + ((long long)i * 9 + k) * kSlotPitch + s, C[k]);
      if (s != kDiagSlot) {
        const int sm = kSlots - 1 - s;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) __stcs(L.H + ((long long)col * 9 + 3 * r + c) * kSlotPitch + sm, C[3 * c + r]);
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
  (void)dx;
  long long blocks = (L.n + kAsmWarps - 1) / kAsmWarps;
  const long long cap = (long long)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  { k_assemble_rows<<<(int)blocks, kAsmWarps * 32, 0, s>>>(bins, g, L, Tu); count_launches(1); }
}

}  // namespace hotb200
