// Node-embedding Galerkin multigrid on B200 (multigrid.hpp:14-392, pcg.hpp:17-46).
//
//   build_restriction  dense coarse flags + scan (same lexicographic order as the
//                      reference's sort/unique); the linear embedding weights are implicit.
//   galerkin_coarsen   one warp per coarse row: every upper-triangle coarse block
//                      H_c(A,B) = sum_{i in ch(A), l in ch(B)} w_iA w_lB H_f(i,l) is gathered
//                      (deterministic, no atomics) and mirrored, so H_c is exactly symmetric.
//   smooth_sgs         the reference's serial colour-ordered symmetric Gauss-Seidel
//                      (multigrid.hpp:298-316) reproduced exactly by a wave schedule: level 0
//                      uses its 27 mod-3 colours (same-colour nodes never couple at radius 2);
//                      coarse levels (mod-2 colours, radius 2) use t = 8*colour + 4a + 2b + c on
//                      the colour sub-lattice, which is strictly increasing along every coupled
//                      predecessor of the serial order, so rows of one wave are independent and
//                      every row sees exactly the neighbour values the serial sweep sees.  One
//                      cooperative persistent kernel per sweep, grid barrier between waves.
//   coarse_solve/pcg   Jacobi-PCG from zero as one cooperative kernel (3 grid barriers per
//                      iteration, deterministic block reductions).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "hot_internal.h"

namespace cg = cooperative_groups;

namespace hotb200 {

namespace {

constexpr int kMgThreads = 256;
constexpr int kMgWarps = kMgThreads / 32;
constexpr int kSgsThreads = 512;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int floor_div2(int x) { return x >> 1; }  // arithmetic shift = floor

__global__ void k_mark_parents(LevelView f, DenseMap cmap, uint8_t* __restrict__ flags) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < f.n; i += gridDim.x * blockDim.x) {
    int lo[3], cnt[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int c = f.coords[3 * i + a];
      lo[a] = floor_div2(c);
      cnt[a] = (c & 1) ? 2 : 1;
    }
    for (int x = 0; x < cnt[0]; ++x)
      for (int y = 0; y < cnt[1]; ++y)
        for (int z = 0; z < cnt[2]; ++z) {
          const long long l = dense_lin(cmap, lo[0] + x, lo[1] + y, lo[2] + z);
          flags[l] = 1;
        }
  }
}

__global__ void k_coarse_dirichlet(LevelView f, DenseMap cmap, uint8_t* __restrict__ cdir) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < f.n; i += gridDim.x * blockDim.x) {
    if (!f.dir[i]) continue;
    int lo[3], cnt[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int c = f.coords[3 * i + a];
      lo[a] = floor_div2(c);
      cnt[a] = (c & 1) ? 2 : 1;
    }
    for (int x = 0; x < cnt[0]; ++x)
      for (int y = 0; y < cnt[1]; ++y)
        for (int z = 0; z < cnt[2]; ++z) cdir[dense_lookup(cmap, lo[0] + x, lo[1] + y, lo[2] + z)] = 1;
  }
}

/// Valid (delta_i, delta_l) per axis for coarse offset O: |2O + dl - di| <= 2.
__device__ __forceinline__ bool axis_ok(int O, int di, int dl) {
  const int f = 2 * O + dl - di;
  return f >= -2 && f <= 2;
}

__global__ void __launch_bounds__(kMgThreads) k_galerkin(LevelView f, LevelView c) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int A = gw; A < c.n; A += nw) {
    const int A0 = c.coords[3 * A], A1 = c.coords[3 * A + 1], A2 = c.coords[3 * A + 2];
    const bool dA = c.dir[A] != 0;
    for (int s = kDiagSlot; s < kSlots; ++s) {
      const int B = c.cols[(long long)A * kSlotPitch + s];
      if (B < 0) continue;
      const int O0 = s / 25 - 2, O1 = (s / 5) % 5 - 2, O2 = s % 5 - 2;
      double acc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = 0.0;
      for (int t = lane; t < 729; t += 32) {
        const int t0 = t / 81, t1 = (t / 9) % 9, t2 = t % 9;
        const int di0 = t0 / 3 - 1, dl0 = t0 % 3 - 1;
        const int di1 = t1 / 3 - 1, dl1 = t1 % 3 - 1;
        const int di2 = t2 / 3 - 1, dl2 = t2 % 3 - 1;
        if (!axis_ok(O0, di0, dl0) || !axis_ok(O1, di1, dl1) || !axis_ok(O2, di2, dl2)) continue;
        const int i = dense_lookup(f.map, 2 * A0 + di0, 2 * A1 + di1, 2 * A2 + di2);
        if (i < 0) continue;
        const int fs = 25 * (2 * O0 + dl0 - di0 + 2) + 5 * (2 * O1 + dl1 - di1 + 2) + (2 * O2 + dl2 - di2 + 2);
        if (f.cols[(long long)i * kSlotPitch + fs] < 0) continue;
        const double wi = (di0 ? 0.5 : 1.0) * (di1 ? 0.5 : 1.0) * (di2 ? 0.5 : 1.0);
        const double wl = (dl0 ? 0.5 : 1.0) * (dl1 ? 0.5 : 1.0) * (dl2 ? 0.5 : 1.0);
        const double w = wi * wl;
        const double* h = f.H + (long long)i * 9 * kSlotPitch + fs;
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] += w * h[k * kSlotPitch];
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = wsum(acc[k]);
      if (lane == 0) {
        double C[9];
        if (s == kDiagSlot) {
          // exact symmetry: keep the upper elements and mirror
          C[0] = acc[0];
          C[4] = acc[4];
          C[8] = acc[8];
          C[1] = C[3] = acc[1];
          C[2] = C[6] = acc[2];
          C[5] = C[7] = acc[5];
          if (dA) {
#pragma unroll
            for (int k = 0; k < 9; ++k) C[k] = (k % 4 == 0) ? 1.0 : 0.0;
          }
        } else {
          const bool zero = dA || c.dir[B] != 0;
#pragma unroll
          for (int k = 0; k < 9; ++k) C[k] = zero ? 0.0 : acc[k];
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) c.H[((long long)A * 9 + k) * kSlotPitch + s] = C[k];
        if (s != kDiagSlot) {
          const int sm = kSlots - 1 - s;
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int q = 0; q < 3; ++q) c.H[((long long)B * 9 + 3 * r + q) * kSlotPitch + sm] = C[3 * q + r];
        }
      }
    }
  }
}

__global__ void k_finalize_level(LevelView L, int coarse, int* __restrict__ wave_of, int* minmax, int* singular) {
  int wmin = INT_MAX, wmax = INT_MIN;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L.n; i += gridDim.x * blockDim.x) {
    M3 D;
#pragma unroll
    for (int k = 0; k < 9; ++k) D.m[k] = L.H[((long long)i * 9 + k) * kSlotPitch + kDiagSlot];
    double det;
    const M3 Di = m3_inverse(D, &det);
    if (!(fabs(det) > 0.0)) atomicExch(singular, 1);
#pragma unroll
    for (int k = 0; k < 9; ++k) L.dinv[9 * i + k] = Di.m[k];
    const int c0 = L.coords[3 * i], c1 = L.coords[3 * i + 1], c2 = L.coords[3 * i + 2];
    int w;
    if (!coarse) {
      w = (((c0 % 3) + 3) % 3 * 3 + ((c1 % 3) + 3) % 3) * 3 + ((c2 % 3) + 3) % 3;
    } else {
      const int col = ((c0 & 1) * 2 + (c1 & 1)) * 2 + (c2 & 1);
      w = 8 * col + 4 * (c0 >> 1) + 2 * (c1 >> 1) + (c2 >> 1);
    }
    wave_of[i] = w;
    wmin = min(wmin, w);
    wmax = max(wmax, w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    wmin = min(wmin, __shfl_xor_sync(0xffffffffu, wmin, o));
    wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(minmax, wmin);
    atomicMax(minmax + 1, wmax);
  }
}

__global__ void k_wave_count(const int* __restrict__ wave_of, int n, int wmin, int* counts) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(counts + (wave_of[i] - wmin), 1);
}
__global__ void k_wave_scatter(const int* __restrict__ wave_of, int n, int wmin, int* cursor, int* rows) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    rows[atomicAdd(cursor + (wave_of[i] - wmin), 1)] = i;
}

/// y_i (3) = sum_s H(i,s) x_col (objective.hpp:66-77), one warp per row.
__device__ __forceinline__ void row_product(const LevelView& L, int i, const double* __restrict__ x, int lane,
                                            double& y0, double& y1, double& y2, bool cg_load) {
  y0 = y1 = y2 = 0.0;
  const int* cols = L.cols + (long long)i * kSlotPitch;
  const double* h = L.H + (long long)i * 9 * kSlotPitch;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int s = lane + 32 * k;
    if (s >= kSlots) break;
    const int c = __ldg(cols + s);
    if (c < 0) continue;
    double x0, x1, x2;
    if (cg_load) {
      x0 = __ldcg(x + 3 * c);
      x1 = __ldcg(x + 3 * c + 1);
      x2 = __ldcg(x + 3 * c + 2);
    } else {
      x0 = __ldg(x + 3 * c);
      x1 = __ldg(x + 3 * c + 1);
      x2 = __ldg(x + 3 * c + 2);
    }
    const double h0 = __ldcs(h + s), h1 = __ldcs(h + kSlotPitch + s), h2 = __ldcs(h + 2 * kSlotPitch + s);
    const double h3 = __ldcs(h + 3 * kSlotPitch + s), h4 = __ldcs(h + 4 * kSlotPitch + s),
                 h5 = __ldcs(h + 5 * kSlotPitch + s);
    const double h6 = __ldcs(h + 6 * kSlotPitch + s), h7 = __ldcs(h + 7 * kSlotPitch + s),
                 h8 = __ldcs(h + 8 * kSlotPitch + s);
    y0 += h0 * x0 + h1 * x1 + h2 * x2;
    y1 += h3 * x0 + h4 * x1 + h5 * x2;
    y2 += h6 * x0 + h7 * x1 + h8 * x2;
  }
  y0 = wsum(y0);
  y1 = wsum(y1);
  y2 = wsum(y2);
}

__global__ void __launch_bounds__(kMgThreads) k_spmv(LevelView L, const double* __restrict__ x, double* __restrict__ y,
                                                     const double* __restrict__ b) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < L.n; i += nw) {
    double y0, y1, y2;
    row_product(L, i, x, lane, y0, y1, y2, false);
    if (lane == 0) {
      if (b) {
        y[3 * i] = b[3 * i] - y0;
        y[3 * i + 1] = b[3 * i + 1] - y1;
        y[3 * i + 2] = b[3 * i + 2] - y2;
      } else {
        y[3 * i] = y0;
        y[3 * i + 1] = y1;
        y[3 * i + 2] = y2;
      }
    }
  }
}

__global__ void k_restrict(LevelView f, LevelView c, const double* __restrict__ rf, double* __restrict__ bc) {
  for (int J = blockIdx.x * blockDim.x + threadIdx.x; J < c.n; J += gridDim.x * blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (!c.dir[J]) {
      const int J0 = c.coords[3 * J], J1 = c.coords[3 * J + 1], J2 = c.coords[3 * J + 2];
      for (int t = 0; t < 27; ++t) {
        const int d0 = t / 9 - 1, d1 = (t / 3) % 3 - 1, d2 = t % 3 - 1;
        const int i = dense_lookup(f.map, 2 * J0 + d0, 2 * J1 + d1, 2 * J2 + d2);
        if (i < 0) continue;
        const double w = (d0 ? 0.5 : 1.0) * (d1 ? 0.5 : 1.0) * (d2 ? 0.5 : 1.0);
        a0 += w * rf[3 * i];
        a1 += w * rf[3 * i + 1];
        a2 += w * rf[3 * i + 2];
      }
    }
    bc[3 * J] = a0;
    bc[3 * J + 1] = a1;
    bc[3 * J + 2] = a2;
  }
}

__global__ void k_prolong_add(LevelView f, LevelView c, const double* __restrict__ uc, double* __restrict__ uf) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < f.n; i += gridDim.x * blockDim.x) {
    int lo[3], cnt[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int cc = f.coords[3 * i + a];
      lo[a] = floor_div2(cc);
      cnt[a] = (cc & 1) ? 2 : 1;
    }
    const double w = (cnt[0] == 2 ? 0.5 : 1.0) * (cnt[1] == 2 ? 0.5 : 1.0) * (cnt[2] == 2 ? 0.5 : 1.0);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int x = 0; x < cnt[0]; ++x)
      for (int y = 0; y < cnt[1]; ++y)
        for (int z = 0; z < cnt[2]; ++z) {
          const int J = dense_lookup(c.map, lo[0] + x, lo[1] + y, lo[2] + z);
          a0 += w * uc[3 * J];
          a1 += w * uc[3 * J + 1];
          a2 += w * uc[3 * J + 2];
        }
    uf[3 * i] += a0;
    uf[3 * i + 1] += a1;
    uf[3 * i + 2] += a2;
  }
}

__global__ void __launch_bounds__(kSgsThreads) k_sgs(LevelView L, const int* __restrict__ wave_start,
                                                    const int* __restrict__ wave_rows, int nwaves, double* u,
                                                    const double* __restrict__ b) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int pass = 0; pass < 2; ++pass) {
    for (int k = 0; k < nwaves; ++k) {
      const int w = pass == 0 ? k : nwaves - 1 - k;
      const int e = wave_start[w + 1];
      for (int r = wave_start[w] + gw; r < e; r += nw) {
        const int i = wave_rows[r];
        double y0, y1, y2;
        row_product(L, i, u, lane, y0, y1, y2, true);
        if (lane == 0) {
          const double r0 = b[3 * i] - y0, r1 = b[3 * i + 1] - y1, r2 = b[3 * i + 2] - y2;
          const double* D = L.dinv + 9 * i;
          u[3 * i] = __ldcg(u + 3 * i) + (D[0] * r0 + D[1] * r1 + D[2] * r2);
          u[3 * i + 1] = __ldcg(u + 3 * i + 1) + (D[3] * r0 + D[4] * r1 + D[5] * r2);
          u[3 * i + 2] = __ldcg(u + 3 * i + 2) + (D[6] * r0 + D[7] * r1 + D[8] * r2);
        }
      }
      grid.sync();
    }
  }
}

/// Deterministic grid reduction: every block sums all block partials in the same fixed tree.
__device__ __forceinline__ double grid_total(const double* partials, int nparts) {
  __shared__ double ws[kMgWarps];
  __shared__ double res;
  double v = 0.0;
  for (int k = threadIdx.x; k < nparts; k += blockDim.x) v += __ldcg(partials + k);
  v = wsum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kMgWarps; ++w) t += ws[w];
    res = t;
  }
  __syncthreads();
  const double r = res;
  __syncthreads();
  return r;
}

__device__ __forceinline__ void block_partial(double v, double* partials) {
  __shared__ double ws[kMgWarps];
  v = wsum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kMgWarps; ++w) t += ws[w];
    partials[blockIdx.x] = t;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kMgThreads) k_pcg(LevelView L, const double* __restrict__ b, double* x, double* r,
                                                    double* z, double* p, double* Ap, double rel, int cap,
                                                    double* partials, int* stat, int* iter_acc) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  const int nb = gridDim.x;
  // x = 0, r = b, z = D^-1 r, p = z, rho = r.z
  double loc = 0.0;
  for (int i = tid; i < L.n; i += nt) {
    const double* D = L.dinv + 9 * i;
    const double r0 = b[3 * i], r1 = b[3 * i + 1], r2 = b[3 * i + 2];
    const double z0 = D[0] * r0 + D[1] * r1 + D[2] * r2;
    const double z1 = D[3] * r0 + D[4] * r1 + D[5] * r2;
    const double z2 = D[6] * r0 + D[7] * r1 + D[8] * r2;
    x[3 * i] = x[3 * i + 1] = x[3 * i + 2] = 0.0;
    r[3 * i] = r0;
    r[3 * i + 1] = r1;
    r[3 * i + 2] = r2;
    z[3 * i] = p[3 * i] = z0;
    z[3 * i + 1] = p[3 * i + 1] = z1;
    z[3 * i + 2] = p[3 * i + 2] = z2;
    loc += r0 * z0 + r1 * z1 + r2 * z2;
  }
  block_partial(loc, partials);
  grid.sync();
  double rho = grid_total(partials, nb);
  int its = 0;
  int status = 0;
  if (!(rho > 0.0)) {
    if (rho < 0.0) status = 1;
  } else {
    const double threshold = rel * rel * rho;
    for (int it = 0; it < cap; ++it) {
      grid.sync();  // p complete; partials free
      loc = 0.0;
      for (int i = gw; i < L.n; i += nw) {
        double y0, y1, y2;
        row_product(L, i, p, lane, y0, y1, y2, true);
        if (lane == 0) {
          Ap[3 * i] = y0;
          Ap[3 * i + 1] = y1;
          Ap[3 * i + 2] = y2;
          loc += __ldcg(p + 3 * i) * y0 + __ldcg(p + 3 * i + 1) * y1 + __ldcg(p + 3 * i + 2) * y2;
        }
      }
      block_partial(loc, partials);
      grid.sync();
      const double pAp = grid_total(partials, nb);
      if (!(pAp > 0.0)) {
        status = 2;
        break;
      }
      const double alpha = rho / pAp;
      grid.sync();  // everyone has read partials
      loc = 0.0;
      for (int i = tid; i < L.n; i += nt) {
        const double* D = L.dinv + 9 * i;
        double rr[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          x[3 * i + a] = __dadd_rn(x[3 * i + a], __dmul_rn(alpha, __ldcg(p + 3 * i + a)));
          rr[a] = __dsub_rn(r[3 * i + a], __dmul_rn(alpha, __ldcg(Ap + 3 * i + a)));
          r[3 * i + a] = rr[a];
        }
        const double z0 = D[0] * rr[0] + D[1] * rr[1] + D[2] * rr[2];
        const double z1 = D[3] * rr[0] + D[4] * rr[1] + D[5] * rr[2];
        const double z2 = D[6] * rr[0] + D[7] * rr[1] + D[8] * rr[2];
        z[3 * i] = z0;
        z[3 * i + 1] = z1;
        z[3 * i + 2] = z2;
        loc += rr[0] * z0 + rr[1] * z1 + rr[2] * z2;
      }
      block_partial(loc, partials);
      grid.sync();
      const double rho_new = grid_total(partials, nb);
      its = it + 1;
      if (rho_new <= threshold) break;
      const double beta = rho_new / rho;
      for (int i = tid; i < L.n; i += nt)
#pragma unroll
        for (int a = 0; a < 3; ++a) p[3 * i + a] = __dadd_rn(z[3 * i + a], __dmul_rn(beta, p[3 * i + a]));
      rho = rho_new;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    stat[0] = status;
    stat[1] = its;
    if (iter_acc) *iter_acc += its;
  }
}

int mgrid(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  const long long cap = (long long)num_sms() * 16;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

int coop_blocks(const void* fn, int threads) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
  if (per_sm < 1) per_sm = 1;
  return per_sm * num_sms();
}

}  // namespace

int sgs_max_blocks() {
  static int v = 0;
  if (!v) v = coop_blocks((const void*)k_sgs, kSgsThreads);
  return v;
}
int pcg_max_blocks() {
  static int v = 0;
  if (!v) v = coop_blocks((const void*)k_pcg, kMgThreads);
  return v;
}

void launch_mark_parents(LevelView fine, DenseMap cmap, uint8_t* flags, cudaStream_t s) {
  if (fine.n) { k_mark_parents<<<mgrid(fine.n, 256), 256, 0, s>>>(fine, cmap, flags); count_launches(1); }
}
void launch_coarse_dirichlet(LevelView fine, DenseMap cmap, uint8_t* cdir, cudaStream_t s) {
  if (fine.n) { k_coarse_dirichlet<<<mgrid(fine.n, 256), 256, 0, s>>>(fine, cmap, cdir); count_launches(1); }
}
void launch_galerkin(LevelView fine, LevelView coarse, cudaStream_t s) {
  if (coarse.n) { k_galerkin<<<mgrid((long long)coarse.n * 32, kMgThreads), kMgThreads, 0, s>>>(fine, coarse); count_launches(1); }
}
void launch_finalize_level(LevelView L, int coarse, int* wave_of, int* wave_minmax, int* singular_flag,
                           cudaStream_t s) {
  if (L.n) { k_finalize_level<<<mgrid(L.n, 256), 256, 0, s>>>(L, coarse, wave_of, wave_minmax, singular_flag); count_launches(1); }
}
void launch_bucket_rows(const int* wave_of, int n, int wmin, int* counts, int* start, int* cursor, int* rows,
                        int nwaves, int* scan_tmp, cudaStream_t s) {
  cudaMemsetAsync(counts, 0, sizeof(int) * (nwaves + 1), s);
  if (n) { k_wave_count<<<mgrid(n, 256), 256, 0, s>>>(wave_of, n, wmin, counts); count_launches(1); }
  launch_exclusive_scan(counts, start, nwaves + 1, scan_tmp, nullptr, s);
  cudaMemcpyAsync(cursor, start, sizeof(int) * nwaves, cudaMemcpyDeviceToDevice, s);
  if (n) { k_wave_scatter<<<mgrid(n, 256), 256, 0, s>>>(wave_of, n, wmin, cursor, rows); count_launches(1); }
}
void launch_spmv(LevelView L, const double* x, double* y, cudaStream_t s) {
  if (L.n) { k_spmv<<<mgrid((long long)L.n * 32, kMgThreads), kMgThreads, 0, s>>>(L, x, y, nullptr); count_launches(1); }
}
void launch_residual(LevelView L, const double* b, const double* u, double* r, cudaStream_t s) {
  if (L.n) { k_spmv<<<mgrid((long long)L.n * 32, kMgThreads), kMgThreads, 0, s>>>(L, u, r, b); count_launches(1); }
}
void launch_restrict(LevelView fine, LevelView coarse, const double* rf, double* bc, cudaStream_t s) {
  if (coarse.n) { k_restrict<<<mgrid(coarse.n, 128), 128, 0, s>>>(fine, coarse, rf, bc); count_launches(1); }
}
void launch_prolong_add(LevelView fine, LevelView coarse, const double* uc, double* uf, cudaStream_t s) {
  if (fine.n) { k_prolong_add<<<mgrid(fine.n, 128), 128, 0, s>>>(fine, coarse, uc, uf); count_launches(1); }
}
void launch_sgs(LevelView L, const int* wave_start, const int* wave_rows, int nwaves, double* u, const double* b,
                int grid_blocks, cudaStream_t s) {
  if (L.n == 0 || nwaves == 0) return;
  void* args[] = {&L, (void*)&wave_start, (void*)&wave_rows, &nwaves, &u, (void*)&b};
  { cudaLaunchCooperativeKernel((const void*)k_sgs, grid_blocks, kSgsThreads, args, 0, s); count_launches(1); }
}
void launch_pcg(LevelView L, const double* b, double* x, double* r, double* z, double* p, double* Ap, double rel,
                int cap, double* partials, int* stat, int* iter_acc, int grid_blocks, cudaStream_t s) {
  void* args[] = {&L, (void*)&b, &x, &r, &z, &p, &Ap, &rel, &cap, &partials, &stat, &iter_acc};
  { cudaLaunchCooperativeKernel((const void*)k_pcg, grid_blocks, kMgThreads, args, 0, s); count_launches(1); }
}

}  // namespace hotb200
