// Grid activation, particle binning, APIC P2G (+ node characteristic norm) and collider
// boundary scripts on B200.
//
//   activate_grid   grid.hpp:137-165   dense bounding-box flags + scan: the scan over the
//                                       row-major box IS the lexicographic order, so node
//                                       indices equal the reference's sort+unique indices
//                                       bit for bit, with no sort.
//   p2g             transfer.hpp:46-64 node-centric gather over particles binned by their
//                                       stencil-centre node: deterministic, no float atomics.
//   compute_node_cn objective.hpp:450-473  fused into the P2G gather.
//   apply_boundary_scripts simulation.hpp:259-272
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <tuple>

#include "hot_internal.h"
#include "hot_particle.cuh"

namespace hotb200 {

namespace {

constexpr int kTile = 4096;      // scan tile (256 threads x 16 items)
constexpr int kScanThreads = 256;

__device__ __forceinline__ int warp_incl_scan(int v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += t;
  }
  return v;
}

/// Block-wide exclusive scan of one int per thread (blockDim = 256); returns the block total.
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
  __shared__ int warp_sums[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) warp_sums[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int ws = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
    const int wi = warp_incl_scan(ws);
    if (lane < kScanThreads / 32) warp_sums[lane] = wi - ws;
    if (lane == kScanThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  const int r = inc - v + warp_sums[wid];
  __syncthreads();
  return r;
}

__global__ void k_particle_bounds(const double* __restrict__ x, long long n, double dx, int* bounds6, int* bad) {
  int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double xa = x[a * n + p];
      if (!isfinite(xa)) {
        atomicExch(bad, 1);
        continue;
      }
      const int b = stencil_base_1d(xa / dx);
      mn[a] = min(mn[a], b);
      mx[a] = max(mx[a], b);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
  }
  // block reduction, then one set of atomics per block (a few hundred blocks, not one per warp)
  __shared__ int red[6][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      red[a][wid] = mn[a];
      red[3 + a][wid] = mx[a];
    }
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int a = threadIdx.x;
    int v = red[a][0];
    for (int w = 1; w < nwarp; ++w) v = a < 3 ? min(v, red[a][w]) : max(v, red[a][w]);
    if (a < 3) atomicMin(bounds6 + a, v);
    else atomicMax(bounds6 + a, v);
  }
}

/// Marks every node with nonzero quadratic weight (grid.hpp:147-152).  weight > 0 iff every
/// 1D factor > 0 (the factors are bounded below by ~1e-32, so the product never underflows).
__global__ void k_mark_active(const double* __restrict__ x, long long n, double dx, DenseMap map,
                              uint8_t* __restrict__ flags) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    double c[3];
    int base[3];
    bool ok[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      c[a] = x[a * n + p] / dx;
      base[a] = stencil_base_1d(c[a]);
#pragma unroll
      for (int k = 0; k < 3; ++k) ok[a][k] = bspline_w(c[a] - (double)(base[a] + k)) > 0.0;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (!ok[0][i]) continue;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (!ok[1][j]) continue;
        const long long row = ((long long)(base[0] + i - map.lo[0]) * map.ext[1] + (base[1] + j - map.lo[1])) * map.ext[2];
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if (ok[2][k]) flags[row + (base[2] + k - map.lo[2])] = 1;
      }
    }
  }
}

__global__ void k_tile_counts(const uint8_t* __restrict__ flags, long long len, int* tile_sums) {
  const long long t0 = (long long)blockIdx.x * kTile + threadIdx.x * 16;
  int cnt = 0;
  if (t0 + 16 <= len) {
    const uint4 v = *reinterpret_cast<const uint4*>(flags + t0);
    cnt = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);  // flags are 0/1 bytes
  } else {
    for (long long i = t0; i < len; ++i) cnt += flags[i];
  }
  __shared__ int tot;
  block_excl_scan(cnt, &tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

/// Single-block exclusive scan of n ints in place; writes the grand total.
__global__ void k_scan_small(int* data, int n, int* total) {
  __shared__ int carry_s, tot;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < n; base += kScanThreads) {
    const int i = base + threadIdx.x;
    const int v = i < n ? data[i] : 0;
    const int ex = block_excl_scan(v, &tot);
    const int carry = carry_s;
    if (i < n) data[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry_s;
}

__global__ void k_tile_index(const uint8_t* __restrict__ flags, long long len, int e1, int e2, int lo0, int lo1,
                             int lo2, const int* __restrict__ tile_sums, int* __restrict__ idx,
                             int* __restrict__ coords) {
  const long long t0 = (long long)blockIdx.x * kTile + threadIdx.x * 16;
  uint8_t f[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = (t0 + i < len) ? flags[t0 + i] : 0;
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) cnt += f[i];
  __shared__ int tot;
  int r = block_excl_scan(cnt, &tot) + tile_sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const long long l = t0 + i;
    if (l >= len) break;
    if (f[i]) {
      idx[l] = r;
      const int z = (int)(l % e2);
      const long long q = l / e2;
      const int y = (int)(q % e1);
      const int xx = (int)(q / e1);
      coords[3 * r] = xx + lo0;
      coords[3 * r + 1] = y + lo1;
      coords[3 * r + 2] = z + lo2;
      ++r;
    } else {
      idx[l] = -1;
    }
  }
}

__global__ void k_int_tile_sums(const int* __restrict__ in, int n, int* tile_sums) {
  int s = 0;
  const long long t0 = (long long)blockIdx.x * kTile + threadIdx.x * 16;
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if (t0 + i < n) s += in[t0 + i];
  __shared__ int tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void k_int_tile_scan(const int* __restrict__ in, int n, const int* __restrict__ tile_sums, int* out) {
  const long long t0 = (long long)blockIdx.x * kTile + threadIdx.x * 16;
  int v[16];
  int s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = (t0 + i < n) ? in[t0 + i] : 0;
    s += v[i];
  }
  __shared__ int tot;
  int r = block_excl_scan(s, &tot) + tile_sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (t0 + i < n) out[t0 + i] = r;
    r += v[i];
  }
}

__global__ void k_bin_count(const double* __restrict__ x, long long n, double dx, DenseMap map, int* bin_of,
                            int* counts) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = stencil_base_1d(x[a * n + p] / dx) + 1;
    const int j = dense_lookup(map, c[0], c[1], c[2]);  // the centre node always has weight > 0
    bin_of[p] = j;
    atomicAdd(counts + j, 1);
  }
}

__global__ void k_bin_scatter(const int* __restrict__ bin_of, long long n, int* cursor, int* pid) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const int pos = atomicAdd(cursor + bin_of[p], 1);
    pid[pos] = (int)p;
  }
}

/// Canonical (ascending particle id) order inside each bin, so every gather below is
/// run-to-run deterministic.
/// Particles of a bin in ascending ORIGINAL id (the caller's upload order): the order every
/// per-bin sum uses, the same whichever subset of the particles a rank stores (particle
/// partition), so the sharded sums are bitwise the single-GPU ones.
__global__ void k_bin_sort(const int* __restrict__ start, int n_nodes, int* pid, const int* __restrict__ orig) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_nodes; j += gridDim.x * blockDim.x) {
    const int b = start[j], e = start[j + 1];
    for (int i = b + 1; i < e; ++i) {
      const int v = pid[i];
      const int ov = orig[v];
      int k = i - 1;
      while (k >= b && orig[pid[k]] > ov) {
        pid[k + 1] = pid[k];
        --k;
      }
      pid[k + 1] = v;
    }
  }
}

/// P2G, particle half (transfer.hpp:46-64, objective.hpp:445-463): for bin j and stencil
/// position k, the sums over the bin's particles (bin order) of w m, w m (v + C (x_i - x_p)) and
/// w m xi, into B[j][k][0..4].  One warp per bin, lane k < 27, particle data broadcast.  Every
/// (bin, k) pair feeds exactly one node.  Empty bins write zeros.
constexpr int kBinWarps = 8;
__global__ void __launch_bounds__(kBinWarps * 32) k_bin_p2g(ParticlesView P, BinsView bins, GridView g, double dx,
                                                           const DevMaterial* __restrict__ mats,
                                                           double* __restrict__ B, int jlo, int jhi) {
  // per warp: the current chunk of <= 32 bin particles, [field][slot] (x 3, v 3, C 9, m, m xi),
  // loaded coalesced (lanes over particles) and read back as broadcasts by the stencil lanes
  __shared__ double stage[kBinWarps][17][32];
  const long long n = P.n;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  double(*sm)[32] = stage[wib];
  // 1D weights: lane 9u + 3a + k (< 27) evaluates axis a, node k of particle t + u, so one
  // division serves three particles; the stencil lanes (lane = 9 k0 + 3 k1 + k2) take theirs by
  // shuffle
  const int wu = min(lane / 9, 2), la = (lane % 9) / 3, lk = lane % 3;
  const int s0 = lane / 9, s1 = 3 + (lane / 3) % 3, s2 = 6 + lane % 3;
  const int k0 = lane / 9 - 1, k1 = (lane / 3) % 3 - 1, k2 = lane % 3 - 1;
  for (int j = jlo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); j < jhi; j += nw) {
    const int pb = __ldg(bins.start + j), pe = __ldg(bins.start + j + 1);
    const int ci0 = g.coords[3 * j] + k0, ci1 = g.coords[3 * j + 1] + k1, ci2 = g.coords[3 * j + 2] + k2;
    const double xi0 = (double)ci0 * dx, xi1 = (double)ci1 * dx, xi2 = (double)ci2 * dx;
    const double ca = (double)(g.coords[3 * j + la] + lk - 1);
    double m = 0.0, mom0 = 0.0, mom1 = 0.0, mom2 = 0.0, num = 0.0;
    for (int c0 = pb; c0 < pe; c0 += 32) {
      const int cnt = min(32, pe - c0);
      __syncwarp();
      if (lane < cnt) {
        const long long p = c0 + lane;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          sm[a][lane] = __ldg(P.x + a * n + p);
          sm[3 + a][lane] = __ldg(P.v + a * n + p);
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) sm[6 + q][lane] = __ldg(P.C + q * n + p);
        const double mp = __ldg(P.mass + p);
        sm[15][lane] = mp;
        sm[16][lane] = mp * mats[__ldg(P.mat + p)].xi;
      }
      __syncwarp();
      for (int t0 = 0; t0 < cnt; t0 += 3) {
        const double wa = bspline_w(sm[la][min(t0 + wu, cnt - 1)] / dx - ca);
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int t = t0 + u;
          if (t >= cnt) break;
          const double w = __shfl_sync(0xffffffffu, wa, 9 * u + s0) * __shfl_sync(0xffffffffu, wa, 9 * u + s1) *
                           __shfl_sync(0xffffffffu, wa, 9 * u + s2);
          if (w <= 0.0) continue;
          const double px0 = sm[0][t], px1 = sm[1][t], px2 = sm[2][t];
          const double wm = w * sm[15][t];
          const double d0 = xi0 - px0, d1 = xi1 - px1, d2 = xi2 - px2;
          const double a0 = sm[3][t] + (sm[6][t] * d0 + sm[7][t] * d1 + sm[8][t] * d2);
          const double a1 = sm[4][t] + (sm[9][t] * d0 + sm[10][t] * d1 + sm[11][t] * d2);
          const double a2 = sm[5][t] + (sm[12][t] * d0 + sm[13][t] * d1 + sm[14][t] * d2);
          m += wm;
          mom0 += wm * a0;
          mom1 += wm * a1;
          mom2 += wm * a2;
          num += w * sm[16][t];
        }
      }
    }
    if (lane < 27) {  // [bin][stencil position][field]
      double* out = B + 135LL * j + 5 * lane;
      out[0] = m;
      out[1] = mom0;
      out[2] = mom1;
      out[3] = mom2;
      out[4] = num;
    }
  }
}

/// P2G, node half: one thread per node sums its 27 bins' contributions in offset order (bin at
/// offset o - 1, where the node is stencil position 26 - o), then v = mom / m and the characteristic-norm scale
/// (objective.hpp:445-463); resets the boundary fields.
template <int NT>
__global__ void __launch_bounds__(NT) k_p2g(GridView g, const double* __restrict__ B, double ell, double dt, int lo,
                                            int hi) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    double m = 0.0, mom0 = 0.0, mom1 = 0.0, mom2 = 0.0, num = 0.0;
    const int* nbi = g.nb27 + 27LL * i;
#pragma unroll 9
    for (int o = 0; o < 27; ++o) {
      const int j = __ldg(nbi + o);
      if (j < 0) continue;
      const double* bv = B + 135LL * j + 5 * (26 - o);
      m += __ldg(bv);
      mom0 += __ldg(bv + 1);
      mom1 += __ldg(bv + 2);
      mom2 += __ldg(bv + 3);
      num += __ldg(bv + 4);
    }
    g.mass[i] = m;
    g.mom[3 * i] = mom0;
    g.mom[3 * i + 1] = mom1;
    g.mom[3 * i + 2] = mom2;
    if (m > 0.0) {
      g.vel[3 * i] = mom0 / m;
      g.vel[3 * i + 1] = mom1 / m;
      g.vel[3 * i + 2] = mom2 / m;
    } else {
      g.vel[3 * i] = g.vel[3 * i + 1] = g.vel[3 * i + 2] = 0.0;
    }
    const double xi = m > 0.0 ? num / m : 0.0;
    g.cn_scale[i] = ell * xi * dt;
    g.dir[i] = 0;
    g.bc_vel[3 * i] = g.bc_vel[3 * i + 1] = g.bc_vel[3 * i + 2] = 0.0;
  }
}

// Collider tests mirror simulation.hpp:20-65 with explicit round-to-nearest arithmetic so the
// Dirichlet set matches the CPU's uncontracted evaluation bit for bit.
__device__ __forceinline__ double dot3_rn(const double a[3], const double b[3]) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}

__device__ bool inside_collider(const DevCollider& c, const double x[3]) {
  switch (c.shape) {
    case 0:
      for (int a = 0; a < 3; ++a)
        if (x[a] < c.a[a] || x[a] > c.b[a]) return false;
      return true;
    case 1: {
      double r[3];
      for (int a = 0; a < 3; ++a) r[a] = __dsub_rn(x[a], c.a[a]);
      return __dsqrt_rn(dot3_rn(r, r)) <= c.radius;
    }
    case 2: {
      double r[3];
      for (int a = 0; a < 3; ++a) r[a] = __dsub_rn(x[a], c.a[a]);
      return dot3_rn(r, c.b) <= 0.0;
    }
    case 3: {
      double r[3];
      for (int a = 0; a < 3; ++a) r[a] = __dsub_rn(x[a], c.a[a]);
      const double t = dot3_rn(r, c.b);
      double q[3];
      for (int a = 0; a < 3; ++a) q[a] = __dsub_rn(r[a], __dmul_rn(t, c.b[a]));
      return __dsqrt_rn(dot3_rn(q, q)) <= c.radius;
    }
  }
  return false;
}

__global__ void k_apply_bc(GridView g, double dx, const DevCollider* __restrict__ cols, int n_cols) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    const double x[3] = {__dmul_rn((double)g.coords[3 * i], dx), __dmul_rn((double)g.coords[3 * i + 1], dx),
                         __dmul_rn((double)g.coords[3 * i + 2], dx)};
    for (int k = 0; k < n_cols; ++k) {
      const DevCollider c = cols[k];
      if (!inside_collider(c, x)) continue;
      double v[3] = {0.0, 0.0, 0.0};
      if (c.motion == 1) {
        v[0] = c.vel[0];
        v[1] = c.vel[1];
        v[2] = c.vel[2];
      } else if (c.motion == 2) {
        const double r0 = x[0] - c.rot_center[0], r1 = x[1] - c.rot_center[1], r2 = x[2] - c.rot_center[2];
        v[0] = c.rot_w[1] * r2 - c.rot_w[2] * r1;
        v[1] = c.rot_w[2] * r0 - c.rot_w[0] * r2;
        v[2] = c.rot_w[0] * r1 - c.rot_w[1] * r0;
      }
      g.dir[i] = 1;
      for (int a = 0; a < 3; ++a) {
        g.vel[3 * i + a] = v[a];
        g.bc_vel[3 * i + a] = v[a];
      }
      break;
    }
  }
}

/// Gathers every particle array into bin order (stable, ascending ids inside a bin) so each
/// bin is a contiguous range: the node-centric gathers then stream contiguous particle data.
__global__ void k_reorder(ParticlesView src, ParticlesView dst, const int* __restrict__ pid,
                          const int* __restrict__ bin_of, const int* __restrict__ orig_src,
                          int* __restrict__ orig_dst) {
  const long long n = src.n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long p = pid[t];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      dst.x[a * n + t] = src.x[a * n + p];
      dst.v[a * n + t] = src.v[a * n + p];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      dst.F[k * n + t] = src.F[k * n + p];
      dst.C[k * n + t] = src.C[k * n + p];
    }
    dst.mass[t] = src.mass[p];
    dst.vol[t] = src.vol[p];
    if (src.Jp) dst.Jp[t] = src.Jp[p];
    dst.mat[t] = src.mat[p];
    dst.bin[t] = bin_of[p];
    orig_dst[t] = orig_src[p];
  }
}

__global__ void k_fill_nb27(GridView g, int* __restrict__ nb27) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)g.n * 27;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / 27), k = (int)(t - 27LL * i);
    nb27[t] = dense_lookup(g.map, g.coords[3 * i] + k / 9 - 1, g.coords[3 * i + 1] + (k / 3) % 3 - 1,
                           g.coords[3 * i + 2] + k % 3 - 1);
  }
}

/// The nodal velocity of virtual_F (objective.hpp:218-230): vel + (dv + alpha p), rounded
/// exactly as the per-particle expression it replaces.
__global__ void k_node_u(GridView g, const double* __restrict__ dv, const double* __restrict__ pd, double alpha,
                         double* __restrict__ u) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 3LL * g.n;
       t += (long long)gridDim.x * blockDim.x) {
    double d = dv[t];
    if (pd) d = __dadd_rn(d, __dmul_rn(alpha, pd[t]));
    u[t] = g.vel[t] + d;
  }
}

int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  const long long cap = (long long)num_sms() * 32;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

namespace {
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
std::mutex g_dev_mutex;
}  // namespace

int num_sms() {
  // per device: a process may drive contexts on several GPUs
  static int n[kMaxDevices] = {};
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return 148;
  if (n[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

void set_max_dynamic_smem(const void* fn, int smem) {
  if (smem <= 48 * 1024) return;
  static std::set<std::tuple<int, const void*, int>> done;
  const auto key = std::make_tuple(current_device(), fn, smem);
  std::lock_guard<std::mutex> lk(g_dev_mutex);
  if (done.count(key)) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  done.insert(key);
}

int resident_blocks(const void* fn, int threads, int smem) {
  static std::map<std::tuple<int, const void*, int, int>, int> memo;
  const auto key = std::make_tuple(current_device(), fn, threads, smem);
  {
    std::lock_guard<std::mutex> lk(g_dev_mutex);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  set_max_dynamic_smem(fn, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  if (per_sm < 1) per_sm = 1;
  const int v = per_sm * num_sms();
  std::lock_guard<std::mutex> lk(g_dev_mutex);
  memo[key] = v;
  return v;
}

void launch_particle_bounds(const ParticlesView& P, double dx, int* bounds6, int* bad_flag, cudaStream_t s) {
  if (P.n == 0) return;
  { k_particle_bounds<<<std::min(grid_for(P.n, 256), 4 * num_sms()), 256, 0, s>>>(P.x, P.n, dx, bounds6, bad_flag); count_launches(1); }
}

void launch_mark_active(const ParticlesView& P, double dx, DenseMap map, uint8_t* flags, cudaStream_t s) {
  if (P.n == 0) return;
  { k_mark_active<<<grid_for(P.n, 256), 256, 0, s>>>(P.x, P.n, dx, map, flags); count_launches(1); }
}

void launch_flags_to_index(const uint8_t* flags, long long len, const int* ext, const int* lo, int* idx, int* coords,
                           int* tile_sums, int* count_dev, cudaStream_t s) {
  const int tiles = (int)((len + kTile - 1) / kTile);
  if (tiles == 0) {
    cudaMemsetAsync(count_dev, 0, sizeof(int), s);
    return;
  }
  { k_tile_counts<<<tiles, kScanThreads, 0, s>>>(flags, len, tile_sums); count_launches(1); }
  { k_scan_small<<<1, kScanThreads, 0, s>>>(tile_sums, tiles, count_dev); count_launches(1); }
  { k_tile_index<<<tiles, kScanThreads, 0, s>>>(flags, len, ext[1], ext[2], lo[0], lo[1], lo[2], tile_sums, idx, coords); count_launches(1); }
}

void launch_exclusive_scan(const int* in, int* out, int n, int* tmp, int* total_dev, cudaStream_t s) {
  const int tiles = (n + kTile - 1) / kTile;
  if (tiles == 0) {
    if (total_dev) cudaMemsetAsync(total_dev, 0, sizeof(int), s);
    return;
  }
  { k_int_tile_sums<<<tiles, kScanThreads, 0, s>>>(in, n, tmp); count_launches(1); }
  { k_scan_small<<<1, kScanThreads, 0, s>>>(tmp, tiles, total_dev); count_launches(1); }
  { k_int_tile_scan<<<tiles, kScanThreads, 0, s>>>(in, n, tmp, out); count_launches(1); }
}

void launch_bin_particles(const ParticlesView& P, double dx, DenseMap map, int n_nodes, int* bin_of, int* counts,
                          int* start, int* cursor, int* pid, int* scan_tmp, const int* orig, cudaStream_t s) {
  cudaMemsetAsync(counts, 0, sizeof(int) * (n_nodes + 1), s);
  if (P.n > 0) { k_bin_count<<<grid_for(P.n, 256), 256, 0, s>>>(P.x, P.n, dx, map, bin_of, counts); count_launches(1); }
  launch_exclusive_scan(counts, start, n_nodes + 1, scan_tmp, nullptr, s);
  cudaMemcpyAsync(cursor, start, sizeof(int) * n_nodes, cudaMemcpyDeviceToDevice, s);
  if (P.n > 0) { k_bin_scatter<<<grid_for(P.n, 256), 256, 0, s>>>(bin_of, P.n, cursor, pid); count_launches(1); }
  if (n_nodes > 0) { k_bin_sort<<<grid_for(n_nodes, 128), 128, 0, s>>>(start, n_nodes, pid, orig); count_launches(1); }
}

void launch_p2g(const ParticlesView& P, BinsView bins, GridView g, double dx, const DevMaterial* mats, double ell,
                double dt, double* bin_part, cudaStream_t s, int jlo, int jhi, int lo, int hi) {
  if (g.n == 0) return;
  if (jhi < 0) jhi = g.n;
  if (hi < 0) hi = g.n;
  const int blocks = resident_blocks((const void*)k_p2g<256>, 256, 0);
  const int bin_blocks = resident_blocks((const void*)k_bin_p2g, kBinWarps * 32, 0);
  if (jhi > jlo) {
    k_bin_p2g<<<std::min<long long>(bin_blocks, (jhi - jlo + kBinWarps - 1) / kBinWarps), kBinWarps * 32, 0, s>>>(
        P, bins, g, dx, mats, bin_part, jlo, jhi);
    count_launches(1);
  }
  if (hi > lo) {
    k_p2g<256><<<std::min<long long>(blocks, (hi - lo + 255) / 256), 256, 0, s>>>(g, bin_part, ell, dt, lo, hi);
    count_launches(1);
  }
}

void launch_fill_nb27(GridView g, int* nb27, cudaStream_t s) {
  if (g.n == 0) return;
  { k_fill_nb27<<<grid_for(27LL * g.n, 256), 256, 0, s>>>(g, nb27); count_launches(1); }
}

void launch_node_u(GridView g, const double* dv, const double* p, double alpha, double* u, cudaStream_t s) {
  if (g.n == 0) return;
  { k_node_u<<<grid_for(3LL * g.n, 256), 256, 0, s>>>(g, dv, p, alpha, u); count_launches(1); }
}

void launch_reorder_particles(const ParticlesView& src, const ParticlesView& dst, const int* pid, const int* bin_of,
                              const int* orig_src,
                              int* orig_dst, cudaStream_t s) {
  if (src.n == 0) return;
  { k_reorder<<<grid_for(src.n, 256), 256, 0, s>>>(src, dst, pid, bin_of, orig_src, orig_dst); count_launches(1); }
}

void launch_apply_bc(GridView g, double dx, const DevCollider* cols, int n_cols, cudaStream_t s) {
  if (g.n == 0 || n_cols == 0) return;
  { k_apply_bc<<<grid_for(g.n, 128), 128, 0, s>>>(g, dx, cols, n_cols); count_launches(1); }
}

}  // namespace hotb200
