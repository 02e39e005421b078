// Grid-to-particle transfer, strain update with plastic return map and advection, fused
// into one pass per particle (transfer.hpp:68-120), plus the CFL speed reduction
// (simulation.hpp:290-291).  All three reference loops read the same x^n stencil and the
// converged grid velocity, so fusing them changes no value.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "hot_internal.h"

namespace hotb200 {

namespace {

template <int NT>
__global__ void __launch_bounds__(NT) k_g2p_strain_advect(ParticlesView P, GridView g, double dx, double dt,
                                                          const DevMaterial* __restrict__ mats, int* inverted) {
  const long long n = P.n;
  const double dinv = 4.0 / (dx * dx);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    double xp[3], c[3];
    int base[3];
    Axis3 ax[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      xp[a] = P.x[a * n + p];
      c[a] = xp[a] / dx;
      base[a] = stencil_base_1d(c[a]);
      axis_weights(c[a], base[a], ax[a]);
      axis_dw_over_dx(ax[a], dx);
    }
    double v[3] = {0.0, 0.0, 0.0}, B[9], G[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) B[k] = G[k] = 0.0;
    // stencil nodes from the bin's 27-neighbour table; the x-axis loop stays rolled (select, not
    // indexing) so the kernel fits the instruction cache
    const int* nb = g.nb27 + 27LL * P.bin[p];
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
          const double vi[3] = {g.vel[3 * node], g.vel[3 * node + 1], g.vel[3 * node + 2]};
          const double d[3] = {(double)(base[0] + i) * dx - xp[0], (double)(base[1] + j) * dx - xp[1],
                               (double)(base[2] + k) * dx - xp[2]};
          const double gr[3] = {dwi * ax[1].w[j] * ax[2].w[k], ax[1].dw[j] * wi * ax[2].w[k],
                                ax[2].dw[k] * wi * ax[1].w[j]};
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const double wv = w * vi[a];
            v[a] += wv;
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              B[a * 3 + b] += wv * d[b];
              G[a * 3 + b] += vi[a] * gr[b];
            }
          }
        }
    }
    M3 Fn, A;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      Fn.m[k] = P.F[k * n + p];
      A.m[k] = ((k % 4 == 0) ? 1.0 : 0.0) + dt * G[k];
    }
    M3 F = m3_mul(A, Fn);
    const DevMaterial mt = mats[P.mat[p]];
    bool skip_map = false;
    if (m3_det(F) <= 0.0) {
      atomicAdd(inverted, 1);
      skip_map = mt.plasticity == 1 || mt.plasticity == 3;  // Hencky-strain maps (Drucker-Prager: extension)
    }
    if (!skip_map) {
      double jp = P.Jp ? P.Jp[p] : 1.0;
      return_map(F, mt, &jp);
      if (P.Jp) P.Jp[p] = jp;
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      P.F[k * n + p] = F.m[k];
      P.C[k * n + p] = B[k] * dinv;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      P.v[a * n + p] = v[a];
      P.x[a * n + p] = xp[a] + dt * v[a];
    }
  }
}

__global__ void k_check_ids(const int* __restrict__ ids, long long n, int limit, int* bad) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    if (ids[p] < 0 || ids[p] >= limit) atomicExch(bad, 1);
}

__global__ void k_vmax(const double* __restrict__ v, long long n, unsigned long long* vmax_bits) {
  double m = 0.0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const double a = v[p], b = v[n + p], c = v[2 * n + p];
    m = fmax(m, sqrt(a * a + b * b + c * c));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  // block maximum, then one atomic per block; non-negative doubles order like their bit patterns
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    atomicMax(vmax_bits, (unsigned long long)__double_as_longlong(m));
  }
}

int tgrid(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  const long long cap = (long long)num_sms() * 32;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

void launch_g2p_strain_advect(const ParticlesView& P, GridView g, double dx, double dt, const DevMaterial* mats,
                              int* inverted, cudaStream_t s) {
  if (P.n == 0) return;
  // 512 threads per block.  cfg2 per step: 512 0.265 ms, 384 0.323, 256 0.454, 128 0.453: wide
  // blocks keep a bin-ordered run of particles, whose stencils overlap, on one SM (L1 hits on
  // the node velocities), which outweighs the register cap's spills
  k_g2p_strain_advect<512><<<tgrid(P.n, 512), 512, 0, s>>>(P, g, dx, dt, mats, inverted);
  count_launches(1);
}

void launch_check_ids(const int* ids, long long n, int limit, int* bad, cudaStream_t s) {
  if (n) { k_check_ids<<<(int)std::min<long long>((n + 255) / 256, (long long)num_sms() * 8), 256, 0, s>>>(ids, n, limit, bad); count_launches(1); }
}

void launch_vmax(const ParticlesView& P, unsigned long long* vmax_bits, cudaStream_t s) {
  if (P.n == 0) return;
  { k_vmax<<<std::min(tgrid(P.n, 256), 4 * num_sms()), 256, 0, s>>>(P.v, P.n, vmax_bits); count_launches(1); }
}

}  // namespace hotb200

namespace hotb200 {
namespace {
__global__ void k_aos_to_soa(const double* __restrict__ in, double* __restrict__ out, long long n, int comps) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * comps;
       t += (long long)gridDim.x * blockDim.x) {
    const long long p = t / comps;
    const int k = (int)(t % comps);
    out[k * n + p] = in[t];
  }
}
__global__ void k_soa_to_aos(const double* __restrict__ in, double* __restrict__ out, long long n, int comps) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * comps;
       t += (long long)gridDim.x * blockDim.x) {
    const long long p = t / comps;
    const int k = (int)(t % comps);
    out[t] = in[k * n + p];
  }
}
__global__ void k_soa_to_aos_perm(const double* __restrict__ in, double* __restrict__ out, long long n, int comps,
                                  const int* __restrict__ perm) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * comps;
       t += (long long)gridDim.x * blockDim.x) {
    const long long p = t / comps;
    const int k = (int)(t % comps);
    out[(long long)perm[p] * comps + k] = in[k * n + p];
  }
}
__global__ void k_iota(int* out, long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    out[t] = (int)t;
}
}  // namespace

void launch_soa_to_aos_perm(const double* in, double* out, long long n, int comps, const int* perm, cudaStream_t s) {
  if (n) { k_soa_to_aos_perm<<<tgrid(n * comps, 256), 256, 0, s>>>(in, out, n, comps, perm); count_launches(1); }
}
__global__ void k_gather_perm(const double* __restrict__ in, double* __restrict__ out, long long n,
                              const int* __restrict__ perm) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    out[t] = in[perm[t]];
}
__global__ void k_fill(double* __restrict__ out, long long n, double value) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    out[t] = value;
}
void launch_gather_perm(const double* in, double* out, long long n, const int* perm, cudaStream_t s) {
  if (n) { k_gather_perm<<<tgrid(n, 256), 256, 0, s>>>(in, out, n, perm); count_launches(1); }
}
void launch_fill(double* out, long long n, double value, cudaStream_t s) {
  if (n) { k_fill<<<tgrid(n, 256), 256, 0, s>>>(out, n, value); count_launches(1); }
}

void launch_iota(int* out, long long n, cudaStream_t s) {
  if (n) { k_iota<<<tgrid(n, 256), 256, 0, s>>>(out, n); count_launches(1); }
}

void launch_aos_to_soa(const double* in, double* out, long long n, int comps, cudaStream_t s) {
  if (n) { k_aos_to_soa<<<tgrid(n * comps, 256), 256, 0, s>>>(in, out, n, comps); count_launches(1); }
}
void launch_soa_to_aos(const double* in, double* out, long long n, int comps, cudaStream_t s) {
  if (n) { k_soa_to_aos<<<tgrid(n * comps, 256), 256, 0, s>>>(in, out, n, comps); count_launches(1); }
}
}  // namespace hotb200
