// Incremental potential on B200: per-particle energy/stress at a nodal velocity increment
// (objective.hpp:236-257), node-centric gradient gather (objective.hpp:260-287) fused with
// the characteristic-norm residual (objective.hpp:476-486), and the L-BFGS vector algebra
// (solvers.hpp:82-129) as fused, deterministic reductions (fixed block partials summed in
// fixed order; no float atomics).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "hot_internal.h"
#include "hot_particle.cuh"

namespace hotb200 {

namespace {

constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

/// Deterministic block sum (fixed tree); result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[NT / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) r += ws[w];
  }
  __syncthreads();
  return r;
}

constexpr int kEnergyThreads = 128;  // ~146 registers: 3 blocks (12 warps) per SM

template <int NT, int MINB, bool CONTIG = false>
__global__ void __launch_bounds__(NT, MINB) k_particle_energy(ParticlesView P, GridView g, double dx, double dt,
                                                                 const DevMaterial* __restrict__ mats,
                                                                 const double* __restrict__ u,
                                                                 double* __restrict__ stress,
                                                                 double* __restrict__ svd_out,
                                                                 double* __restrict__ pe, int* bad, long long plo,
                                                                 long long phi) {
  const long long n = P.n;
  // CONTIG: each block walks one contiguous chunk of the (bin-ordered) particles, so the
  // stencil nodes its particles share stay in its SM's L1; otherwise a grid stride
  const long long chunk = CONTIG ? (phi - plo + gridDim.x - 1) / gridDim.x : 0;
  const long long p0 = CONTIG ? plo + blockIdx.x * chunk : plo + blockIdx.x * (long long)blockDim.x;
  const long long p1 = CONTIG ? min(phi, p0 + chunk) : phi;
  const long long stride = CONTIG ? (long long)blockDim.x : (long long)gridDim.x * blockDim.x;
  for (long long p = p0 + threadIdx.x; p < p1; p += stride) {
    M3 F, Fn;
    if (!virtual_F(P, p, g, dx, dt, u, F, Fn)) {
      atomicExch(bad, 1);
      pe[p] = 0.0;
      continue;
    }
    const DevMaterial mt = mats[P.mat[p]];
    double mu, la;
    particle_lame(mt, P.Jp, p, mu, la);
    M3 U, V;
    double s[3];
    svd3(F, U, s, V);
    if (svd_out) {  // kept for the assembly at the same dv (k_particle_tensors)
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        svd_out[k * n + p] = U.m[k];
        svd_out[(12 + k) * n + p] = V.m[k];
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) svd_out[(9 + k) * n + p] = s[k];
    }
    const double vol = P.vol[p];
    pe[p] = vol * model_psi(s, mu, la, mt.elasticity);
    if (stress) {
      const M3 Pk = model_P(F, U, V, mu, la, mt.elasticity);
      const M3 PFt = m3_mul_bt(Pk, Fn);
#pragma unroll
      for (int k = 0; k < 9; ++k) stress[k * n + p] = vol * PFt.m[k];
    }
  }
}

/// Node energy terms (objective.hpp:247-255) plus the elastic energy of the node's bin (its
/// particles in bin order): ne[i] per row i in [lo, hi).  The total is a fixed-tree sum over
/// ne[0, n), which does not depend on how rows are split between GPUs.
__global__ void __launch_bounds__(kRedThreads) k_node_energy(GridView g, BinsView bins, const double* __restrict__ pe,
                                                             double dt, double g0, double g1, double g2,
                                                             const double* __restrict__ dv,
                                                             const double* __restrict__ pd, double alpha,
                                                             double* __restrict__ ne, int lo, int hi) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    const int pb = __ldg(bins.start + i), pend = __ldg(bins.start + i + 1);
    for (int q = pb; q < pend; ++q) acc += __ldg(pe + q);
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      d[a] = dv[3 * i + a];
      if (pd) d[a] = __dadd_rn(d[a], __dmul_rn(alpha, pd[3 * i + a]));
    }
    const double m = g.mass[i];
    const double sq = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    const double gu = g0 * (g.vel[3 * i] + d[0]) + g1 * (g.vel[3 * i + 1] + d[1]) + g2 * (g.vel[3 * i + 2] + d[2]);
    ne[i] = acc + (0.5 * m * sq - dt * m * gu);
  }
}

/// Gradient, particle half (objective.hpp:276-280): for bin j and stencil position k, the sum
/// over the bin's particles (bin order) of (V P F^nT)_p grad w_k(x_p), into S[j][k][0..2].  One
/// warp per bin, lane k < 27; the particle's data is a broadcast load.  Every (bin, k) pair
/// feeds exactly one node, so each particle is read once per gradient instead of once per
/// stencil node, and the node pass reads each S entry once.  Empty bins write zeros.
constexpr int kBinWarps = 8;
__global__ void __launch_bounds__(kBinWarps * 32) k_bin_force(ParticlesView P, BinsView bins, GridView g, double dx,
                                                             const double* __restrict__ stress,
                                                             double* __restrict__ S, int jlo, int jhi) {
  // per warp: the current chunk of <= 32 bin particles, [field][slot] (x 3, V P F^T 9), loaded
  // coalesced (lanes over particles) and read back as broadcasts by the stencil lanes
  __shared__ double stage[kBinWarps][12][32];
  const long long n = P.n;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  double(*sm)[32] = stage[wib];
  // 1D weights: lane 9u + 3a + k (< 27) evaluates axis a, node k of particle t + u, so one
  // division sequence serves three particles; the stencil lanes (lane = 9 k0 + 3 k1 + k2) take
  // theirs by shuffle
  const int wu = min(lane / 9, 2), la = (lane % 9) / 3, lk = lane % 3;
  const int s0 = lane / 9, s1 = 3 + (lane / 3) % 3, s2 = 6 + lane % 3;
  for (int j = jlo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); j < jhi; j += nw) {
    const int pb = __ldg(bins.start + j), pe = __ldg(bins.start + j + 1);
    const double ca = (double)(g.coords[3 * j + la] + lk - 1);
    double f0 = 0.0, f1 = 0.0, f2 = 0.0;
    for (int c0 = pb; c0 < pe; c0 += 32) {
      const int cnt = min(32, pe - c0);
      __syncwarp();
      if (lane < cnt) {
#pragma unroll
        for (int a = 0; a < 3; ++a) sm[a][lane] = __ldg(P.x + a * n + c0 + lane);
#pragma unroll
        for (int q = 0; q < 9; ++q) sm[3 + q][lane] = __ldg(stress + q * n + c0 + lane);
      }
      __syncwarp();
      for (int t0 = 0; t0 < cnt; t0 += 3) {
        const double o = sm[la][min(t0 + wu, cnt - 1)] / dx - ca;
        const double wa = bspline_w(o), dwa = bspline_dw(o) / dx;
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int t = t0 + u;
          if (t >= cnt) break;
          const double w0 = __shfl_sync(0xffffffffu, wa, 9 * u + s0), w1 = __shfl_sync(0xffffffffu, wa, 9 * u + s1),
                       w2 = __shfl_sync(0xffffffffu, wa, 9 * u + s2);
          const double d0 = __shfl_sync(0xffffffffu, dwa, 9 * u + s0),
                       d1 = __shfl_sync(0xffffffffu, dwa, 9 * u + s1),
                       d2 = __shfl_sync(0xffffffffu, dwa, 9 * u + s2);
          if (w0 * w1 * w2 <= 0.0) continue;
          const double gr0 = d0 * w1 * w2;
          const double gr1 = d1 * w0 * w2;
          const double gr2 = d2 * w0 * w1;
          f0 += sm[3][t] * gr0 + sm[4][t] * gr1 + sm[5][t] * gr2;
          f1 += sm[6][t] * gr0 + sm[7][t] * gr1 + sm[8][t] * gr2;
          f2 += sm[9][t] * gr0 + sm[10][t] * gr1 + sm[11][t] * gr2;
        }
      }
    }
    if (lane < 27) {  // [bin][stencil position][field]
      double* out = S + 81LL * j + 3 * lane;
      out[0] = f0;
      out[1] = f1;
      out[2] = f2;
    }
  }
}

/// Node gradient (objective.hpp:260-287): one thread per node sums its 27 bins' contributions
/// in offset order (bin at offset o - 1, where the node is stencil position 26 - o), fused with
/// the node's scaled-norm term (objective.hpp:476-486) nt[i] = |g_i|^2 / scale_i^2, rows
/// [lo, hi).  The norm is a fixed-tree sum over nt[0, n) (split-independent).
template <int NT>
__global__ void __launch_bounds__(NT) k_node_gradient(GridView g, double dt, double g0, double g1, double g2,
                                                               const double* __restrict__ S,
                                                               const double* __restrict__ dv, double* __restrict__ gout,
                                                               double* __restrict__ nt, int* bad, int lo, int hi) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    double f0 = 0.0, f1 = 0.0, f2 = 0.0;
    const int* nbi = g.nb27 + 27LL * i;
#pragma unroll 9
    for (int o = 0; o < 27; ++o) {
      const int j = __ldg(nbi + o);
      if (j < 0) continue;
      const double* sv = S + 81LL * j + 3 * (26 - o);
      f0 += __ldg(sv);
      f1 += __ldg(sv + 1);
      f2 += __ldg(sv + 2);
    }
    const double m = g.mass[i];
    double gi[3] = {dt * f0 + m * (dv[3 * i] - dt * g0), dt * f1 + m * (dv[3 * i + 1] - dt * g1),
                    dt * f2 + m * (dv[3 * i + 2] - dt * g2)};
    if (g.dir[i]) gi[0] = gi[1] = gi[2] = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) gout[3 * i + a] = gi[a];
    const double sc = g.cn_scale[i];
    if (!(sc > 0.0)) atomicExch(bad, 2);
    nt[i] = (gi[0] * gi[0] + gi[1] * gi[1] + gi[2] * gi[2]) / (sc * sc);
  }
}

__global__ void __launch_bounds__(kRedThreads) k_sum_array(const double* __restrict__ a, long long n,
                                                           double* __restrict__ partials) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc += a[i];
  const double r = block_sum<kRedThreads>(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

__global__ void __launch_bounds__(kRedThreads) k_sum_partials(const double* __restrict__ partials, int n,
                                                              double* out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
  const double b = block_sum<kRedThreads>(acc);
  if (threadIdx.x == 0) *out = b;
}

__global__ void __launch_bounds__(kRedThreads) k_dot_partials(const double* __restrict__ a,
                                                              const double* __restrict__ b, long long n,
                                                              double* __restrict__ partials) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc += a[i] * b[i];
  const double r = block_sum<kRedThreads>(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

__global__ void __launch_bounds__(kRedThreads) k_axpy_dot(double* __restrict__ q, const double* __restrict__ y,
                                                          const double* __restrict__ coef_dev, int idx, int add,
                                                          const double* __restrict__ s, long long n,
                                                          double* __restrict__ partials) {
  const double c = y ? coef_dev[idx] : 0.0;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double v = q[i];
    if (y) {
      const double cy = __dmul_rn(c, y[i]);
      v = add ? __dadd_rn(v, cy) : __dsub_rn(v, cy);
      q[i] = v;
    }
    if (s) acc += s[i] * v;
  }
  if (partials) {
    const double r = block_sum<kRedThreads>(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = r;
  }
}

__global__ void __launch_bounds__(kRedThreads) k_finalize_coef(const double* __restrict__ partials, int n, double rho,
                                                               const double* __restrict__ alpha_dev, int idx,
                                                               double* coef_dev) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
  const double b = block_sum<kRedThreads>(acc);
  if (threadIdx.x == 0) coef_dev[idx] = alpha_dev ? alpha_dev[idx] - rho * b : rho * b;
}

__global__ void k_neg_copy(const double* __restrict__ a, double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = -a[i];
}
__global__ void k_add_scaled(const double* __restrict__ a, const double* __restrict__ b, double alpha,
                             double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(a[i], __dmul_rn(alpha, b[i]));
}
__global__ void k_scale(const double* __restrict__ a, double alpha, double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = alpha * a[i];
}
__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                      long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] - b[i];
}

__global__ void __launch_bounds__(kRedThreads) k_ys_dots(const double* __restrict__ gn, const double* __restrict__ go,
                                                         double* __restrict__ y, const double* __restrict__ s,
                                                         long long n, double* __restrict__ partials) {
  double ys = 0.0, yy = 0.0, ss = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double yi = gn[i] - go[i];
    y[i] = yi;
    const double si = s[i];
    ys += yi * si;
    yy += yi * yi;
    ss += si * si;
  }
  const double a = block_sum<kRedThreads>(ys);
  const double b = block_sum<kRedThreads>(yy);
  const double c = block_sum<kRedThreads>(ss);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = a;
    partials[gridDim.x + blockIdx.x] = b;
    partials[2 * gridDim.x + blockIdx.x] = c;
  }
}

__global__ void k_zero_dir_copy(const double* __restrict__ in, double* __restrict__ out, const uint8_t* __restrict__ dir,
                                int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const bool z = dir[i] != 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) out[3 * i + a] = z ? 0.0 : in[3 * i + a];
  }
}

/// v^{n+1} = v^n + dv, Dirichlet nodes carry bc_velocity exactly (solvers.hpp:376-379).
__global__ void k_final_velocity(GridView g, const double* __restrict__ dv, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
      out[3 * i + a] = g.dir[i] ? g.bc_vel[3 * i + a] : g.vel[3 * i + a] + dv[3 * i + a];
  }
}

int vgrid(long long n) {
  long long b = (n + 255) / 256;
  const long long cap = (long long)num_sms() * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

template <int NT, int MINB, bool CONTIG = false>
void launch_particle_energy_t(const ParticlesView& P, GridView g, double dx, double dt, const DevMaterial* mats,
                              const double* u, double* stress, double* svd_out, double* pe, int nblocks, int* bad_flag,
                              cudaStream_t s, long long plo, long long phi, int grid_scale = 1) {
  // grid_scale x the thread count of nblocks x 128 threads over the particles (grid-stride)
  const long long want = (phi - plo + NT - 1) / NT;
  const long long cap = (long long)nblocks * kEnergyThreads * grid_scale / NT;
  k_particle_energy<NT, MINB, CONTIG><<<(int)std::max<long long>(1, std::min<long long>(cap, want)), NT, 0, s>>>(
      P, g, dx, dt, mats, u, stress, svd_out, pe, bad_flag, plo, phi);
  count_launches(1);
}

void launch_particle_energy(const ParticlesView& P, GridView g, double dx, double dt, const DevMaterial* mats,
                            const double* u, double* stress, double* svd_out, double* pe, int nblocks, int* bad_flag,
                            cudaStream_t s, long long plo, long long phi) {
  if (phi < 0) phi = P.n;
  if (phi <= plo) return;
  // 512 threads x 1 CTA per SM, one resident wave.  cfg2 particle energy per step: 0.672 ms,
  // against 0.676 (two waves), 0.755 (256 x 2), 0.80 (128 x 4), 0.73 / 0.82 / 0.86 (512 / 256 /
  // 128 with contiguous per-block chunks) and 0.99 (128 x 3, 128 x 2): wide blocks keep a
  // bin-ordered run of particles, whose stencils overlap, on one SM
  launch_particle_energy_t<512, 1>(P, g, dx, dt, mats, u, stress, svd_out, pe, nblocks / 2, bad_flag, s, plo, phi);
}

void launch_node_energy(GridView g, BinsView bins, const double* pe, double dt, const double* grav, const double* dv,
                        const double* p, double alpha, double* ne, int lo, int hi, cudaStream_t s) {
  if (hi <= lo) return;
  k_node_energy<<<std::max(1, std::min((hi - lo + kRedThreads - 1) / kRedThreads, 16 * num_sms())), kRedThreads, 0, s>>>(
      g, bins, pe, dt, grav[0], grav[1], grav[2], dv, p, alpha, ne, lo, hi);
  count_launches(1);
}

void launch_node_gradient(const ParticlesView& P, BinsView bins, GridView g, double dx, double dt, const double* grav,
                          const double* stress, const double* dv, double* gout, double* bin_part, double* nt,
                          int* bad_flag, cudaStream_t s, int jlo, int jhi, int lo, int hi) {
  if (jhi < 0) jhi = g.n;
  if (hi < 0) hi = g.n;
  if (jhi > jlo) {
    const int bin_blocks = resident_blocks((const void*)k_bin_force, kBinWarps * 32, 0);
    k_bin_force<<<std::min<long long>(bin_blocks, (jhi - jlo + kBinWarps - 1) / kBinWarps), kBinWarps * 32, 0, s>>>(
        P, bins, g, dx, stress, bin_part, jlo, jhi);
    count_launches(1);
  }
  if (hi > lo) {
    k_node_gradient<256><<<std::max(1, std::min((hi - lo + 255) / 256, 16 * num_sms())), 256, 0, s>>>(
        g, dt, grav[0], grav[1], grav[2], bin_part, dv, gout, nt, bad_flag, lo, hi);
    count_launches(1);
  }
}

void launch_sum_array(const double* a, long long n, double* partials, int nblocks, cudaStream_t s) {
  k_sum_array<<<nblocks, kRedThreads, 0, s>>>(a, n, partials);
  count_launches(1);
}

void launch_sum_partials(const double* partials, int n, double* out, cudaStream_t s) {
  { k_sum_partials<<<1, kRedThreads, 0, s>>>(partials, n, out); count_launches(1); }
}

void launch_dot_partials(const double* a, const double* b, long long n, double* partials, int nblocks, cudaStream_t s) {
  { k_dot_partials<<<nblocks, kRedThreads, 0, s>>>(a, b, n, partials); count_launches(1); }
}

void launch_axpy_dot(double* q, const double* y, const double* coef_dev, int coef_idx, double coef_scale,
                     const double* s_vec, long long n, double* partials, int nblocks, cudaStream_t s) {
  { k_axpy_dot<<<nblocks, kRedThreads, 0, s>>>(q, y, coef_dev, coef_idx, coef_scale > 0 ? 1 : 0, s_vec, n, partials); count_launches(1); }
}

void launch_finalize_coef(const double* partials, int n, double rho, const double* alpha_dev, int idx, double* coef_dev,
                          cudaStream_t s) {
  { k_finalize_coef<<<1, kRedThreads, 0, s>>>(partials, n, rho, alpha_dev, idx, coef_dev); count_launches(1); }
}

void launch_neg_copy(const double* a, double* out, long long n, cudaStream_t s) {
  if (n) { k_neg_copy<<<vgrid(n), 256, 0, s>>>(a, out, n); count_launches(1); }
}
void launch_add_scaled(const double* a, const double* b, double alpha, double* out, long long n, cudaStream_t s) {
  if (n) { k_add_scaled<<<vgrid(n), 256, 0, s>>>(a, b, alpha, out, n); count_launches(1); }
}
void launch_scale(const double* a, double alpha, double* out, long long n, cudaStream_t s) {
  if (n) { k_scale<<<vgrid(n), 256, 0, s>>>(a, alpha, out, n); count_launches(1); }
}
void launch_sub(const double* a, const double* b, double* out, long long n, cudaStream_t s) {
  if (n) { k_sub<<<vgrid(n), 256, 0, s>>>(a, b, out, n); count_launches(1); }
}
void launch_ys_dots(const double* g_new, const double* g_old, double* y, const double* s, long long n,
                    double* partials, int nblocks, cudaStream_t st) {
  { k_ys_dots<<<nblocks, kRedThreads, 0, st>>>(g_new, g_old, y, s, n, partials); count_launches(1); }
}
void launch_zero_dirichlet_copy(const double* in, double* out, const uint8_t* dir, int n, cudaStream_t s) {
  if (n) { k_zero_dir_copy<<<vgrid(n), 256, 0, s>>>(in, out, dir, n); count_launches(1); }
}
void launch_final_velocity(GridView g, const double* dv, double* out, cudaStream_t s) {
  if (g.n) { k_final_velocity<<<vgrid(g.n), 256, 0, s>>>(g, dv, out); count_launches(1); }
}

}  // namespace hotb200
