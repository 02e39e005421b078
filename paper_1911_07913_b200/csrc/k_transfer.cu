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
                                                          const DevMaterial* __restrict__ mats, int* inverted,
                                                          int own_lo, int own_hi) {
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
      // counted by the particle's owner only (particle partition: ghosts are counted there)
      const int pl = g.coords[3 * P.bin[p]];
      if (pl >= own_lo && pl < own_hi) atomicAdd(inverted, 1);
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
                              int* inverted, cudaStream_t s, int own_lo, int own_hi) {
  if (P.n == 0) return;
  // 512 threads per block.  cfg2 per step: 512 0.265 ms, 384 0.323, 256 0.454, 128 0.453: wide
  // blocks keep a bin-ordered run of particles, whose stencils overlap, on one SM (L1 hits on
  // the node velocities), which outweighs the register cap's spills
  k_g2p_strain_advect<512><<<tgrid(P.n, 512), 512, 0, s>>>(P, g, dx, dt, mats, inverted, own_lo, own_hi);
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

// ------------------------------------------------------------------------------------------
// Particle partition of the slab-sharded step: each rank stores the particles
// whose stencil-centre plane (axis 0) lies in its band [P - gL, Q + gR): the ones it owns (plane
// in [P, Q)) and ghost copies of its neighbours' particles.  After advection every rank sends
// its owned particles that left its slab or lie within the bands other ranks copy, one record
// each, through one allgather; every rank keeps the records inside its band.
// ------------------------------------------------------------------------------------------
namespace hotb200 {
namespace {

/// Stencil-centre plane (axis 0) of a position: stencil_base + 1 (grid.hpp:78-100), the bin the
/// next activation puts the particle in.
__device__ __forceinline__ int centre_plane(double x0, double dx) { return stencil_base_1d(x0 / dx) + 1; }

/// keep[p]: owned before the step (its bin's plane in [P, Q)), still owned and not in a band
/// other ranks copy (stays here, unpacked); pack[p]: owned before the step and either leaving the
/// slab or inside [P, P + gR) u [Q - gL, Q) (sent to every rank).  Ghosts are dropped: their
/// owners send them again.
__global__ void k_pp_classify(ParticlesView Pv, const int* __restrict__ coords, int owned_lo, int owned_hi,
                              int pre_lo, int pre_hi, int gL, int gR, double dx, int* __restrict__ keep,
                              int* __restrict__ pack) {
  const long long n = Pv.n;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    int k = 0, s = 0;
    const int pre = coords ? coords[3 * Pv.bin[p]] : centre_plane(Pv.x[p], dx);
    if (pre >= pre_lo && pre < pre_hi) {
      const int np_ = centre_plane(Pv.x[p], dx);
      const bool mine = np_ >= owned_lo && np_ < owned_hi;
      const bool band = np_ < owned_lo + gR || np_ >= owned_hi - gL;
      k = mine && !band;
      s = !mine || band;
    }
    keep[p] = k;
    pack[p] = s;
  }
}

/// Packed particle record: x3 v3 F9 C9 mass vol Jp orig mat plane (30 doubles, 240 B).
constexpr int kPPRec = 30;

__global__ void k_pp_pack(ParticlesView Pv, const int* __restrict__ orig, const int* __restrict__ flag,
                          const int* __restrict__ pos, double dx, double* __restrict__ out) {
  const long long n = Pv.n;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    if (!flag[p]) continue;
    double* r = out + (long long)pos[p] * kPPRec;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      r[a] = Pv.x[a * n + p];
      r[3 + a] = Pv.v[a * n + p];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      r[6 + k] = Pv.F[k * n + p];
      r[15 + k] = Pv.C[k * n + p];
    }
    r[24] = Pv.mass[p];
    r[25] = Pv.vol[p];
    r[26] = Pv.Jp ? Pv.Jp[p] : 1.0;
    r[27] = (double)orig[p];
    r[28] = (double)Pv.mat[p];
    r[29] = (double)centre_plane(Pv.x[p], dx);
  }
}

__global__ void k_pp_recv_flag(const double* __restrict__ rec, long long m, int lo, int hi, int* __restrict__ flag) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
    const int pl = (int)rec[t * kPPRec + 29];
    flag[t] = pl >= lo && pl < hi;
  }
}

/// New local arrays Q: the kept particles of P (in their order), then the kept records.
__global__ void k_pp_rebuild_keep(ParticlesView Pv, const int* __restrict__ orig, const int* __restrict__ keep,
                                  const int* __restrict__ pos, ParticlesView Qv, int* __restrict__ qorig) {
  const long long n = Pv.n, m = Qv.n;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    if (!keep[p]) continue;
    const long long t = pos[p];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Qv.x[a * m + t] = Pv.x[a * n + p];
      Qv.v[a * m + t] = Pv.v[a * n + p];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      Qv.F[k * m + t] = Pv.F[k * n + p];
      Qv.C[k * m + t] = Pv.C[k * n + p];
    }
    Qv.mass[t] = Pv.mass[p];
    Qv.vol[t] = Pv.vol[p];
    Qv.mat[t] = Pv.mat[p];
    if (Qv.Jp) Qv.Jp[t] = Pv.Jp[p];
    qorig[t] = orig[p];
  }
}

__global__ void k_pp_rebuild_recv(const double* __restrict__ rec, long long mrec, const int* __restrict__ flag,
                                  const int* __restrict__ pos, long long base, ParticlesView Qv,
                                  int* __restrict__ qorig) {
  const long long m = Qv.n;
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < mrec; s += (long long)gridDim.x * blockDim.x) {
    if (!flag[s]) continue;
    const long long t = base + pos[s];
    const double* r = rec + s * kPPRec;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Qv.x[a * m + t] = r[a];
      Qv.v[a * m + t] = r[3 + a];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      Qv.F[k * m + t] = r[6 + k];
      Qv.C[k * m + t] = r[15 + k];
    }
    Qv.mass[t] = r[24];
    Qv.vol[t] = r[25];
    if (Qv.Jp) Qv.Jp[t] = r[26];
    qorig[t] = (int)r[27];
    Qv.mat[t] = (int)r[28];
  }
}

/// Records -> the caller's interleaved arrays at their original ids (x, v: 3, F, C: 9, Jp: 1 per
/// particle; null outputs skipped).
__global__ void k_pp_unpack_caller(const double* __restrict__ rec, long long m, double* x, double* v, double* F,
                                   double* C, double* Jp) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < m; s += (long long)gridDim.x * blockDim.x) {
    const double* r = rec + s * kPPRec;
    const long long o = (long long)r[27];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (x) x[3 * o + a] = r[a];
      if (v) v[3 * o + a] = r[3 + a];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      if (F) F[9 * o + k] = r[6 + k];
      if (C) C[9 * o + k] = r[15 + k];
    }
    if (Jp) Jp[o] = r[26];
  }
}

int pgrid(long long n) {
  long long b = (n + 255) / 256;
  const long long cap = (long long)num_sms() * 16;
  return (int)std::max<long long>(1, std::min(b, cap));
}

}  // namespace

void launch_pp_classify(const ParticlesView& P, const int* coords, int owned_lo, int owned_hi, int pre_lo, int pre_hi,
                        int gL, int gR, double dx, int* keep, int* pack, cudaStream_t s) {
  if (P.n) {
    k_pp_classify<<<pgrid(P.n), 256, 0, s>>>(P, coords, owned_lo, owned_hi, pre_lo, pre_hi, gL, gR, dx, keep, pack);
    count_launches(1);
  }
}
void launch_pp_pack(const ParticlesView& P, const int* orig, const int* flag, const int* pos, double dx, double* out,
                    cudaStream_t s) {
  if (P.n) { k_pp_pack<<<pgrid(P.n), 256, 0, s>>>(P, orig, flag, pos, dx, out); count_launches(1); }
}
void launch_pp_recv_flag(const double* rec, long long m, int lo, int hi, int* flag, cudaStream_t s) {
  if (m) { k_pp_recv_flag<<<pgrid(m), 256, 0, s>>>(rec, m, lo, hi, flag); count_launches(1); }
}
void launch_pp_rebuild(const ParticlesView& P, const int* orig, const int* keep, const int* keep_pos, const double* rec,
                       long long mrec, const int* rflag, const int* rpos, long long n_keep, const ParticlesView& Q,
                       int* qorig, cudaStream_t s) {
  if (P.n) { k_pp_rebuild_keep<<<pgrid(P.n), 256, 0, s>>>(P, orig, keep, keep_pos, Q, qorig); count_launches(1); }
  if (mrec) { k_pp_rebuild_recv<<<pgrid(mrec), 256, 0, s>>>(rec, mrec, rflag, rpos, n_keep, Q, qorig); count_launches(1); }
}
int pp_record_doubles() { return kPPRec; }
void launch_pp_unpack_caller(const double* rec, long long m, double* x, double* v, double* F, double* C, double* Jp,
                             cudaStream_t s) {
  if (m) { k_pp_unpack_caller<<<pgrid(m), 256, 0, s>>>(rec, m, x, v, F, C, Jp); count_launches(1); }
}

}  // namespace hotb200
