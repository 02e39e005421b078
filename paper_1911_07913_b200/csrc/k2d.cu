// The 2D (dim = 2) device path of the HOT step: the reference's own test suite
// is mostly 2D (test_solvers.cpp, test_multigrid.cpp, test_objective.cpp instantiate d = 2) and
// its CLI instantiates advance_step<2> (cli.cpp:145).
//
// Same algorithm and boundary as the 3D path, sized for the small 2D problems: every stage is a
// deterministic gather (no float atomics) --
//   activation      dense flags over the stencil bounding box + scan (lexicographic = row-major),
//   binning         particles by stencil base cell, ascending ids within a cell,
//   P2G / gradient  one thread per node over the 3x3 base cells whose stencils reach it,
//   energy          per-particle psi, node terms, fixed-tree sums,
//   assembly        one thread per (row, upper slot) over the cells shared by both nodes, the
//                   block written with its transpose (exact symmetry),
//   Galerkin        one thread per (coarse row, upper slot) over child pairs,
//   smoother        the reference's serial colour-sorted sweep as wave launches (rows of a
//                   wave never couple: DESIGN.md §4.1 with 2D wave ids),
//   coarse PCG, L-BFGS two-loop, line search: host-driven over device vectors.
// Level matrices are AoS 2x2 blocks: H[(row * S + slot) * 4 + (2r + c)], S = (2R+1)^2 slots in the
// reference's lexicographic order (objective.hpp:24-32).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <memory>
#include <vector>

#include "hot2d.h"
#include "hot2d_math.cuh"

namespace hotb200 {

using d2::M2;

namespace {

#define H2_CUDA(x)                                                                                       \
  do {                                                                                                   \
    cudaError_t e_ = (x);                                                                                \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));             \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  Buf() = default;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  ~Buf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) H2_CUDA(cudaFree(p));
    p = nullptr;
    const size_t nb = std::max<size_t>(bytes + bytes / 4, 256);
    H2_CUDA(cudaMalloc(&p, nb));
    cap = nb;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

inline int gridn(long long n, int t = 256) { return (int)std::max<long long>(1, std::min<long long>((n + t - 1) / t, 65535LL * 8)); }

enum Flag : int { kBadX = 0, kBadF, kAsym, kZeroScale, kSingular, kRhoNeg, kPapNeg, kNonFiniteDv, kNumFlags };

struct Map2 {
  int lo[2], ext[2];
  const int* idx;
  __device__ int at(int x, int y) const {
    const int a = x - lo[0], b = y - lo[1];
    if (a < 0 || b < 0 || a >= ext[0] || b >= ext[1]) return -1;
    return idx[(long long)a * ext[1] + b];
  }
};

struct Cells {  // particles by stencil base cell (dense over the base-cell box)
  int lo[2], ext[2];
  const int* start;  // ext0*ext1 + 1
  const int* pid;
  __device__ void range(int x, int y, int& s, int& e) const {
    const int a = x - lo[0], b = y - lo[1];
    if (a < 0 || b < 0 || a >= ext[0] || b >= ext[1]) {
      s = e = 0;
      return;
    }
    const long long c = (long long)a * ext[1] + b;
    s = start[c];
    e = start[c + 1];
  }
};

struct Parts {
  const double *x, *v, *F, *C, *m, *vol, *jp;
  const int* mat;
  long long n;
};

// --------------------------------------------------------------------------- reductions
constexpr int kRedT = 1024;
__device__ double block_sum(double v, double* sh) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int o = kRedT / 2; o > 0; o >>= 1) {
    if (t < o) sh[t] += sh[t + o];
    __syncthreads();
  }
  return sh[0];
}
/// out[slot] = sum a[i] (b[i]) over [0, n): fixed per-thread strides + fixed tree (deterministic)
__global__ void __launch_bounds__(kRedT) k2_dot(const double* a, const double* b, long long n, double* out, int slot) {
  __shared__ double sh[kRedT];
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += kRedT) acc += b ? a[i] * b[i] : a[i];
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) out[slot] = s;
}
__global__ void k2_vmax(const double* v, long long n, unsigned long long* out) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const double s = sqrt(v[2 * p] * v[2 * p] + v[2 * p + 1] * v[2 * p + 1]);
    atomicMax(out, (unsigned long long)__double_as_longlong(s));  // s >= 0: bit order = value order
  }
}

// --------------------------------------------------------------------------- activation (grid.hpp:137-165)
__global__ void k2_bounds(Parts P, double dx, int* mm, int* flags) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P.n; p += (long long)gridDim.x * blockDim.x) {
    const double x0 = P.x[2 * p], x1 = P.x[2 * p + 1];
    if (!isfinite(x0) || !isfinite(x1)) {
      flags[kBadX] = 1;
      continue;
    }
    int b0, b1;
    d2::stencil2(x0, x1, dx, b0, b1);
    atomicMin(mm + 0, b0);
    atomicMin(mm + 1, b1);
    atomicMax(mm + 2, b0);
    atomicMax(mm + 3, b1);
  }
}
/// flags over the node box: the stencil nodes with positive weight (grid.hpp:150-152)
__global__ void k2_mark(Parts P, double dx, int lo0, int lo1, int ext1, int* fl) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P.n; p += (long long)gridDim.x * blockDim.x) {
    const double x0 = P.x[2 * p], x1 = P.x[2 * p + 1];
    int b0, b1;
    d2::stencil2(x0, x1, dx, b0, b1);
    for (int k = 0; k < 9; ++k) {
      const int n0 = b0 + k / 3, n1 = b1 + k % 3;
      double g0, g1;
      if (d2::wgrad2(x0, x1, dx, n0, n1, g0, g1) > 0.0) fl[(long long)(n0 - lo0) * ext1 + (n1 - lo1)] = 1;
    }
  }
}
__global__ void k2_compact(const int* fl, const int* sc, long long len, int lo0, int lo1, int ext1, int* idx, int* coords) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < len; t += (long long)gridDim.x * blockDim.x) {
    const int i = fl[t] ? sc[t] : -1;
    idx[t] = i;
    if (i >= 0) {
      coords[2 * i] = lo0 + (int)(t / ext1);
      coords[2 * i + 1] = lo1 + (int)(t % ext1);
    }
  }
}

// --------------------------------------------------------------------------- binning
__global__ void k2_cell_of(Parts P, double dx, int lo0, int lo1, int ext1, int* cell, int* cnt) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P.n; p += (long long)gridDim.x * blockDim.x) {
    int b0, b1;
    d2::stencil2(P.x[2 * p], P.x[2 * p + 1], dx, b0, b1);
    const int c = (b0 - lo0) * ext1 + (b1 - lo1);
    cell[p] = c;
    atomicAdd(cnt + c, 1);
  }
}
__global__ void k2_cell_fill(const int* cell, long long n, int* cursor, int* pid) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    pid[atomicAdd(cursor + cell[p], 1)] = (int)p;
}
__global__ void k2_cell_sort(const int* start, int ncell, int* pid) {  // ascending ids within a cell
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
    const int s = start[c], e = start[c + 1];
    for (int i = s + 1; i < e; ++i) {
      const int v = pid[i];
      int j = i - 1;
      while (j >= s && pid[j] > v) {
        pid[j + 1] = pid[j];
        --j;
      }
      pid[j + 1] = v;
    }
  }
}

// --------------------------------------------------------------------------- P2G (transfer.hpp:46-64) + node CN
/// Per node, over the particles of the 3x3 base cells whose stencils reach it; also the CN
/// numerator / denominator of compute_node_cn (objective.hpp:450-473).
__global__ void k2_p2g(Parts P, Cells cells, const int* coords, int n, double dx, const DevMaterial* mats, double ell,
                       double dt, double* mass, double* mom, double* vel, double* cn) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int X = coords[2 * i], Y = coords[2 * i + 1];
    const double xi0 = dx * (double)X, xi1 = dx * (double)Y;
    double m = 0.0, q0 = 0.0, q1 = 0.0, num = 0.0, den = 0.0;
    for (int k = 0; k < 9; ++k) {
      int s, e;
      cells.range(X - k / 3, Y - k % 3, s, e);
      for (int t = s; t < e; ++t) {
        const int p = cells.pid[t];
        const double x0 = P.x[2 * p], x1 = P.x[2 * p + 1];
        double g0, g1;
        const double w = d2::wgrad2(x0, x1, dx, X, Y, g0, g1);
        if (w <= 0.0) continue;
        const double pm = P.m[p];
        const double d0 = xi0 - x0, d1 = xi1 - x1;
        const double* Cp = P.C + 4 * p;
        const double a0 = P.v[2 * p] + (Cp[0] * d0 + Cp[1] * d1);
        const double a1 = P.v[2 * p + 1] + (Cp[2] * d0 + Cp[3] * d1);
        const double wm = w * pm;
        m += wm;
        q0 += wm * a0;
        q1 += wm * a1;
        num += w * (pm * mats[P.mat[p]].xi);
        den += w * pm;
      }
    }
    mass[i] = m;
    mom[2 * i] = q0;
    mom[2 * i + 1] = q1;
    vel[2 * i] = m > 0.0 ? q0 / m : 0.0;
    vel[2 * i + 1] = m > 0.0 ? q1 / m : 0.0;
    const double xi = den > 0.0 ? num / den : 0.0;
    cn[i] = ell * xi * dt;
  }
}

// --------------------------------------------------------------------------- boundary scripts (simulation.hpp:20-65,259-272)
__device__ bool inside2(const DevCollider& c, double x0, double x1) {
  switch (c.shape) {
    case 0:
      return !(x0 < c.a[0] || x0 > c.b[0] || x1 < c.a[1] || x1 > c.b[1]);
    case 1:
    case 3: {  // sphere; the 2D cylinder is a disc (simulation.hpp:31-33)
      const double r0 = __dsub_rn(x0, c.a[0]), r1 = __dsub_rn(x1, c.a[1]);
      return __dsqrt_rn(__dadd_rn(__dmul_rn(r0, r0), __dmul_rn(r1, r1))) <= c.radius;
    }
    case 2: {
      const double r0 = __dsub_rn(x0, c.a[0]), r1 = __dsub_rn(x1, c.a[1]);
      return __dadd_rn(__dmul_rn(r0, c.b[0]), __dmul_rn(r1, c.b[1])) <= 0.0;
    }
  }
  return false;
}
__global__ void k2_bc(int n, const int* coords, double dx, const DevCollider* cols, int ncol, double* vel, double* bcv,
                      uint8_t* dir) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x0 = __dmul_rn(dx, (double)coords[2 * i]), x1 = __dmul_rn(dx, (double)coords[2 * i + 1]);
    dir[i] = 0;
    bcv[2 * i] = bcv[2 * i + 1] = 0.0;
    for (int k = 0; k < ncol; ++k) {
      const DevCollider c = cols[k];
      if (!inside2(c, x0, x1)) continue;
      double v0 = 0.0, v1 = 0.0;
      if (c.motion == 1) {
        v0 = c.vel[0];
        v1 = c.vel[1];
      } else if (c.motion == 2) {  // omega about the centre: (-w r1, w r0)
        const double r0 = x0 - c.rot_center[0], r1 = x1 - c.rot_center[1];
        v0 = c.rot_w[2] * -r1;
        v1 = c.rot_w[2] * r0;
      }
      dir[i] = 1;
      vel[2 * i] = bcv[2 * i] = v0;
      vel[2 * i + 1] = bcv[2 * i + 1] = v1;
      break;
    }
  }
}

// --------------------------------------------------------------------------- objective (objective.hpp:218-287)
/// u = vel + (dv + alpha p), rounded as the reference's trial dv then u (objective.hpp:225)
__global__ void k2_node_u(int n2, const double* vel, const double* dv, const double* p, double alpha, double* u) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x)
    u[k] = vel[k] + (p ? dv[k] + alpha * p[k] : dv[k]);
}
/// virtual F = (I + dt sum_k u_k grad_k^T) F^n (objective.hpp:218-230) over the stencil in order
__device__ M2 vf2(const Parts& P, long long p, const Map2& map, double dx, double dt, const double* u) {
  const double x0 = P.x[2 * p], x1 = P.x[2 * p + 1];
  int b0, b1;
  d2::stencil2(x0, x1, dx, b0, b1);
  M2 G = d2::m2_zero();
  for (int k = 0; k < 9; ++k) {
    double g0, g1;
    if (d2::wgrad2(x0, x1, dx, b0 + k / 3, b1 + k % 3, g0, g1) <= 0.0) continue;
    const int i = map.at(b0 + k / 3, b1 + k % 3);
    if (i < 0) continue;
    const double u0 = u[2 * i], u1 = u[2 * i + 1];
    G.a[0] += u0 * g0;
    G.a[1] += u0 * g1;
    G.a[2] += u1 * g0;
    G.a[3] += u1 * g1;
  }
  M2 A;
  for (int k = 0; k < 4; ++k) A.a[k] = ((k % 3 == 0) ? 1.0 : 0.0) + dt * G.a[k];
  M2 Fn;
  for (int k = 0; k < 4; ++k) Fn.a[k] = P.F[4 * p + k];
  return d2::m2_mul(A, Fn);
}
/// pe[p] = V psi(F); PFt[4p] = P F^n T (gradient's stress) when requested
__global__ void k2_energy_particle(Parts P, Map2 map, double dx, double dt, const DevMaterial* mats, const double* u,
                                   double* pe, double* PFt, int* flags) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P.n; p += (long long)gridDim.x * blockDim.x) {
    const M2 F = vf2(P, p, map, dx, dt, u);
    if (!d2::m2_finite(F)) {
      flags[kBadF] = 1;
      pe[p] = 0.0;
      continue;
    }
    const DevMaterial mt = mats[P.mat[p]];
    double mu, la;
    d2::lame2(mt, P.jp ? P.jp[p] : 1.0, mu, la);
    pe[p] = P.vol[p] * d2::psi2(F, mu, la, mt.elasticity);
    if (PFt) {
      const M2 S = d2::stress2(F, mu, la, mt.elasticity);
      M2 Fn;
      for (int k = 0; k < 4; ++k) Fn.a[k] = P.F[4 * p + k];
      const M2 R = d2::m2_mul(S, d2::m2_t(Fn));
      for (int k = 0; k < 4; ++k) PFt[4 * p + k] = R.a[k];
    }
  }
}
/// node energy terms 0.5 m |dv|^2 - dt m g.u (objective.hpp:250-255)
__global__ void k2_node_energy(int n, const double* mass, const double* vel, const double* dv, const double* p,
                               double alpha, double dt, double g0, double g1, double* ne) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double d0 = p ? dv[2 * i] + alpha * p[2 * i] : dv[2 * i];
    const double d1 = p ? dv[2 * i + 1] + alpha * p[2 * i + 1] : dv[2 * i + 1];
    const double u0 = vel[2 * i] + d0, u1 = vel[2 * i + 1] + d1;
    const double m = mass[i];
    ne[i] = 0.5 * m * (d0 * d0 + d1 * d1) - dt * m * (g0 * u0 + g1 * u1);
  }
}
/// g_i = dt sum_p V (P F^nT) grad w + m (dv - dt g); 0 on Dirichlet; nt[i] = |g_i|^2 / scale_i^2
__global__ void k2_gradient(Parts P, Cells cells, const int* coords, int n, double dx, double dt, double g0, double g1,
                            const double* PFt, const double* mass, const double* dv, const uint8_t* dir,
                            const double* cn, double* g, double* nt, int* flags) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int X = coords[2 * i], Y = coords[2 * i + 1];
    double a0 = 0.0, a1 = 0.0;
    for (int k = 0; k < 9; ++k) {
      int s, e;
      cells.range(X - k / 3, Y - k % 3, s, e);
      for (int t = s; t < e; ++t) {
        const int p = cells.pid[t];
        double w0, w1;
        if (d2::wgrad2(P.x[2 * p], P.x[2 * p + 1], dx, X, Y, w0, w1) <= 0.0) continue;
        const double* S = PFt + 4 * p;
        const double V = P.vol[p];
        a0 += dt * (V * (S[0] * w0 + S[1] * w1));
        a1 += dt * (V * (S[2] * w0 + S[3] * w1));
      }
    }
    const double m = mass[i];
    a0 += m * (dv[2 * i] - dt * g0);
    a1 += m * (dv[2 * i + 1] - dt * g1);
    if (dir[i]) a0 = a1 = 0.0;
    g[2 * i] = a0;
    g[2 * i + 1] = a1;
    const double sc = cn[i];
    if (!(sc > 0.0)) flags[kZeroScale] = 1;
    nt[i] = (a0 * a0 + a1 * a1) / (sc * sc);
  }
}

// --------------------------------------------------------------------------- assembly (objective.hpp:293-363)
constexpr int kRec2 = 16 + 18 + 1;  // T (4x4), W_k = F^nT grad w_k (9 x 2; 0 where w = 0), kappa
__global__ void k2_tensors(Parts P, Map2 map, double dx, double dt, const DevMaterial* mats, const double* u, int project,
                           double* rec, int* flags) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P.n; p += (long long)gridDim.x * blockDim.x) {
    double* R = rec + p * kRec2;
    const M2 F = vf2(P, p, map, dx, dt, u);
    if (!d2::m2_finite(F)) {
      flags[kBadF] = 1;
      continue;
    }
    const DevMaterial mt = mats[P.mat[p]];
    double mu, la;
    d2::lame2(mt, P.jp ? P.jp[p] : 1.0, mu, la);
    double T[16];
    d2::dpdf2(F, mu, la, mt.elasticity, T);
    if (project && !d2::project_spd4(T)) flags[kAsym] = 1;
    for (int k = 0; k < 16; ++k) R[k] = T[k];
    const double x0 = P.x[2 * p], x1 = P.x[2 * p + 1];
    int b0, b1;
    d2::stencil2(x0, x1, dx, b0, b1);
    const double* Fn = P.F + 4 * p;
    for (int k = 0; k < 9; ++k) {
      double g0, g1;
      const bool on = d2::wgrad2(x0, x1, dx, b0 + k / 3, b1 + k % 3, g0, g1) > 0.0;
      R[16 + 2 * k] = on ? Fn[0] * g0 + Fn[2] * g1 : 0.0;  // (F^T grad)_0
      R[17 + 2 * k] = on ? Fn[1] * g0 + Fn[3] * g1 : 0.0;
    }
    R[34] = dt * dt * P.vol[p];
  }
}
/// C(c,e) = wa^T T[(c.),(e.)] wb (objective.hpp:304-310)
__device__ __forceinline__ void contract2(const double* T, const double* wa, const double* wb, double (&C)[4]) {
  for (int c = 0; c < 2; ++c)
    for (int e = 0; e < 2; ++e) {
      double tb[2];
      for (int f = 0; f < 2; ++f) tb[f] = T[(2 * c + f) * 4 + 2 * e] * wb[0] + T[(2 * c + f) * 4 + 2 * e + 1] * wb[1];
      C[2 * c + e] = wa[0] * tb[0] + wa[1] * tb[1];
    }
}
__device__ __forceinline__ int slot_of2(int o0, int o1, int R) {
  const int W = 2 * R + 1;
  return (o0 + R) * W + (o1 + R);
}
/// Row i, upper offset u (lexicographic >= 0, radius 2): the block over the cells whose stencils
/// hold both nodes, mirrored into (j, -off); mass diagonal; Dirichlet projection (objective.hpp:133-144).
__global__ void k2_assemble(Cells cells, const int* coords, int n, Map2 map, const double* rec, const double* mass,
                            const uint8_t* dir, double* H, int* cols) {
  const int S = 25, D = 12;  // slots, diagonal slot
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n * 13;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / 13), uo = (int)(t % 13);
    const int s = D + uo;  // upper slots 12..24
    const int o0 = s / 5 - 2, o1 = s % 5 - 2;
    const int X = coords[2 * i], Y = coords[2 * i + 1];
    const int j = map.at(X + o0, Y + o1);
    cols[(long long)i * S + s] = j;
    if (uo && j >= 0) cols[(long long)j * S + (S - 1 - s)] = i;  // the mirrored lower slot
    if (j < 0) {
      for (int e = 0; e < 4; ++e) H[((long long)i * S + s) * 4 + e] = 0.0;
      continue;
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    // cells b with i - b and j - b in {0,1,2}^2
    for (int c0 = max(X, X + o0) - 2; c0 <= min(X, X + o0); ++c0)
      for (int c1 = max(Y, Y + o1) - 2; c1 <= min(Y, Y + o1); ++c1) {
        int st, en;
        cells.range(c0, c1, st, en);
        const int ka = (X - c0) * 3 + (Y - c1), kb = (X + o0 - c0) * 3 + (Y + o1 - c1);
        for (int q = st; q < en; ++q) {
          const double* R = rec + (long long)cells.pid[q] * kRec2;
          const double* wa = R + 16 + 2 * ka;
          const double* wb = R + 16 + 2 * kb;
          if ((wa[0] == 0.0 && wa[1] == 0.0) || (wb[0] == 0.0 && wb[1] == 0.0)) continue;  // w = 0 node
          double C[4];
          contract2(R, wa, wb, C);
          const double kap = R[34];
          for (int e = 0; e < 4; ++e) C[e] = kap * C[e];
          if (uo == 0) {
            const double t01 = 0.5 * (C[1] + C[2]);
            C[0] = 0.5 * (C[0] + C[0]);
            C[3] = 0.5 * (C[3] + C[3]);
            C[1] = C[2] = t01;
          }
          for (int e = 0; e < 4; ++e) acc[e] += C[e];
        }
      }
    if (uo == 0) {
      acc[0] += mass[i];
      acc[3] += mass[i];
      if (dir[i]) {
        acc[0] = acc[3] = 1.0;
        acc[1] = acc[2] = 0.0;
      }
    } else if (dir[i] || dir[j]) {
      acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
    }
    for (int e = 0; e < 4; ++e) H[((long long)i * S + s) * 4 + e] = acc[e];
    if (uo) {
      const long long m = ((long long)j * S + (S - 1 - s)) * 4;
      H[m + 0] = acc[0];
      H[m + 1] = acc[2];
      H[m + 2] = acc[1];
      H[m + 3] = acc[3];
    }
  }
}
/// lower slots whose column is inactive (never written by a mirror): zero block, col -1
__global__ void k2_lower_inactive(const int* coords, int n, Map2 map, int R, double* H, int* cols) {
  const int W = 2 * R + 1, S = W * W, D = S / 2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n * D;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / D), s = (int)(t % D);
    const int j = map.at(coords[2 * i] + s / W - R, coords[2 * i + 1] + s % W - R);
    if (j >= 0) continue;
    cols[(long long)i * S + s] = -1;
    for (int e = 0; e < 4; ++e) H[((long long)i * S + s) * 4 + e] = 0.0;
  }
}

// --------------------------------------------------------------------------- multigrid (multigrid.hpp)
__device__ __forceinline__ int floor_div2(int x) { return x >= 0 ? x / 2 : (x - 1) / 2; }
/// embedding_entries_1d (multigrid.hpp:64-95): parents of fine coordinate c
__device__ __forceinline__ int parents1(int quad, int c, int (&pc)[3], double (&pw)[3]) {
  if (!quad) {
    const int b = floor_div2(c);
    if (c % 2 == 0) {
      pc[0] = b;
      pw[0] = 1.0;
      return 1;
    }
    pc[0] = b;
    pw[0] = 0.5;
    pc[1] = b + 1;
    pw[1] = 0.5;
    return 2;
  }
  if (c % 2 == 0) {
    const int mid = c / 2;
    pc[0] = mid - 1;
    pw[0] = 0.125;
    pc[1] = mid;
    pw[1] = 0.75;
    pc[2] = mid + 1;
    pw[2] = 0.125;
    return 3;
  }
  const int b = floor_div2(c);
  pc[0] = b;
  pw[0] = 0.5;
  pc[1] = b + 1;
  pw[1] = 0.5;
  return 2;
}
/// weight of coarse A in fine c's embedding (0 when A is not a parent)
__device__ __forceinline__ double weight1(int quad, int c, int A) {
  int pc[3];
  double pw[3];
  const int k = parents1(quad, c, pc, pw);
  for (int q = 0; q < k; ++q)
    if (pc[q] == A) return pw[q];
  return 0.0;
}
__global__ void k2_mark_parents(const int* coords, const uint8_t* dir, int n, int quad, int lo0, int lo1, int ext1,
                                int* fl, uint8_t* cdir_dense) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int p0[3], p1[3];
    double w0[3], w1[3];
    const int k0 = parents1(quad, coords[2 * i], p0, w0), k1 = parents1(quad, coords[2 * i + 1], p1, w1);
    for (int a = 0; a < k0; ++a)
      for (int b = 0; b < k1; ++b) {
        const long long l = (long long)(p0[a] - lo0) * ext1 + (p1[b] - lo1);
        fl[l] = 1;
        if (dir[i]) cdir_dense[l] = 1;
      }
  }
}
__global__ void k2_gather_dir(const uint8_t* cdir_dense, const int* coords, int n, int lo0, int lo1, int ext1, uint8_t* dir) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dir[i] = cdir_dense[(long long)(coords[2 * i] - lo0) * ext1 + (coords[2 * i + 1] - lo1)];
}
/// children of coarse coordinate A along one axis (the fine c whose embedding holds A) + weights
__device__ __forceinline__ int children1(int quad, int A, int (&c)[5], double (&w)[5]) {
  const int span = quad ? 2 : 1;
  int k = 0;
#pragma unroll 1
  for (int f = 2 * A - span; f <= 2 * A + span; ++f) {
    const double wt = weight1(quad, f, A);
    if (wt == 0.0) continue;
    c[k] = f;
    w[k++] = wt;
  }
  return k;
}
/// H_c(A, A+off) = sum_{i child of A, l child of B} w_iA w_lB H_f(i, l) (multigrid.hpp:162-202); on the
/// diagonal each unordered child pair adds (C + C^T) once, so the block is exactly symmetric.  The
/// loops stay rolled (unrolled, this kernel took the compiler tens of minutes).
__global__ void k2_galerkin(const int* ccoords, int nc, Map2 cmap, int Rc, const int* fcoords, Map2 fmap, int Rf,
                            const double* Hf, int quad, const uint8_t* cdir, double* Hc, int* ccols) {
  const int Wc = 2 * Rc + 1, Sc = Wc * Wc, Dc = Sc / 2, U = Sc - Dc;
  const int Wf = 2 * Rf + 1, Sf = Wf * Wf;
  (void)fcoords;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)nc * U;
       t += (long long)gridDim.x * blockDim.x) {
    const int A = (int)(t / U), s = Dc + (int)(t % U);
    const int AX = ccoords[2 * A], AY = ccoords[2 * A + 1];
    const int o0 = s / Wc - Rc, o1 = s % Wc - Rc;
    const int B = cmap.at(AX + o0, AY + o1);
    ccols[(long long)A * Sc + s] = B;
    if (B >= 0 && s != Dc) ccols[(long long)B * Sc + (Sc - 1 - s)] = A;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (B >= 0) {
      int a0c[5], a1c[5], b0c[5], b1c[5];
      double a0w[5], a1w[5], b0w[5], b1w[5];
      const int na0 = children1(quad, AX, a0c, a0w), na1 = children1(quad, AY, a1c, a1w);
      const int nb0 = children1(quad, AX + o0, b0c, b0w), nb1 = children1(quad, AY + o1, b1c, b1w);
#pragma unroll 1
      for (int p = 0; p < na0; ++p)
#pragma unroll 1
        for (int q = 0; q < na1; ++q) {
          const int i0 = a0c[p], i1 = a1c[q];
          const int fi = fmap.at(i0, i1);
          if (fi < 0) continue;
          const double wa = a0w[p] * a1w[q];
#pragma unroll 1
          for (int r = 0; r < nb0; ++r) {
            const int l0 = b0c[r];
            if (l0 - i0 < -Rf || l0 - i0 > Rf) continue;
#pragma unroll 1
            for (int u = 0; u < nb1; ++u) {
              const int l1 = b1c[u];
              if (l1 - i1 < -Rf || l1 - i1 > Rf) continue;
              const int fl = fmap.at(l0, l1);
              if (fl < 0) continue;
              if (s == Dc && fl < fi) continue;  // diagonal: unordered pairs
              const double* Bf = Hf + ((long long)fi * Sf + slot_of2(l0 - i0, l1 - i1, Rf)) * 4;
              const double sc = wa * (b0w[r] * b1w[u]);
              if (s == Dc && fl != fi) {
                const double c0 = sc * Bf[0], c1 = sc * Bf[1], c2 = sc * Bf[2], c3 = sc * Bf[3];
                acc[0] += c0 + c0;
                acc[1] += c1 + c2;
                acc[2] += c2 + c1;
                acc[3] += c3 + c3;
              } else {
                acc[0] += sc * Bf[0];
                acc[1] += sc * Bf[1];
                acc[2] += sc * Bf[2];
                acc[3] += sc * Bf[3];
              }
            }
          }
        }
      if (s == Dc) {
        if (cdir[A]) {
          acc[0] = acc[3] = 1.0;
          acc[1] = acc[2] = 0.0;
        }
      } else if (cdir[A] || cdir[B]) {
        acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
      }
    }
    for (int e = 0; e < 4; ++e) Hc[((long long)A * Sc + s) * 4 + e] = acc[e];
    if (B >= 0 && s != Dc) {
      const long long m = ((long long)B * Sc + (Sc - 1 - s)) * 4;
      Hc[m + 0] = acc[0];
      Hc[m + 1] = acc[2];
      Hc[m + 2] = acc[1];
      Hc[m + 3] = acc[3];
    }
  }
}
/// finalize_level (multigrid.hpp:227-251): D^-1 + singular check; wave id of the colour-sorted
/// serial sweep (level 0 / R < q: colour; coarse: 4 colour + 2 (x div q) + (y div q)).
__global__ void k2_finalize(const int* coords, int n, int S, const double* H, int q, int R, int a0, int b0,
                            double* dinv, int* wave, int* flags) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    M2 D;
    for (int e = 0; e < 4; ++e) D.a[e] = H[((long long)i * S + S / 2) * 4 + e];
    const double det = d2::m2_det(D);
    if (!(fabs(det) > 0.0)) flags[kSingular] = 1;
    const M2 I = d2::m2_inv(D);
    for (int e = 0; e < 4; ++e) dinv[4 * i + e] = I.a[e];
    const int x = coords[2 * i], y = coords[2 * i + 1];
    const int colour = (((x % q) + q) % q) * q + (((y % q) + q) % q);
    if (R < q) {
      wave[i] = colour;
    } else {
      const int a = (x >= 0 ? x / q : -((-x + q - 1) / q)) - a0, b = (y >= 0 ? y / q : -((-y + q - 1) / q)) - b0;
      wave[i] = 4 * colour + 2 * a + b;
    }
  }
}
/// one wave of the symmetric Gauss-Seidel sweep (multigrid.hpp:298-316): rows of a wave never couple
__global__ void k2_sgs_wave(const int* rows, int cnt, int S, const double* H, const int* cols, const double* dinv,
                            const double* b, double* u) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const int i = rows[t];
    double r0 = b[2 * i], r1 = b[2 * i + 1];
    for (int s = 0; s < S; ++s) {
      const int c = cols[(long long)i * S + s];
      if (c < 0) continue;
      const double* B = H + ((long long)i * S + s) * 4;
      const double u0 = u[2 * c], u1 = u[2 * c + 1];
      r0 = r0 - (B[0] * u0 + B[1] * u1);
      r1 = r1 - (B[2] * u0 + B[3] * u1);
    }
    const double* Di = dinv + 4 * i;
    u[2 * i] += Di[0] * r0 + Di[1] * r1;
    u[2 * i + 1] += Di[2] * r0 + Di[3] * r1;
  }
}
/// y = H x (objective.hpp:66-77), or r = b - H x when b is given
__global__ void k2_spmv(int n, int S, const double* H, const int* cols, const double* x, const double* b, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double y0 = 0.0, y1 = 0.0;
    for (int s = 0; s < S; ++s) {
      const int c = cols[(long long)i * S + s];
      if (c < 0) continue;
      const double* B = H + ((long long)i * S + s) * 4;
      y0 += B[0] * x[2 * c] + B[1] * x[2 * c + 1];
      y1 += B[2] * x[2 * c] + B[3] * x[2 * c + 1];
    }
    if (b) {
      y0 = b[2 * i] - y0;
      y1 = b[2 * i + 1] - y1;
    }
    y[2 * i] = y0;
    y[2 * i + 1] = y1;
  }
}
/// restrict_to_coarse (multigrid.hpp:24-31): children in fine index order, Dirichlet rows zeroed
__global__ void k2_restrict(const int* ccoords, int nc, const uint8_t* cdir, Map2 fmap, int quad, const double* rf,
                            double* bc) {
  const int span = quad ? 2 : 1;
  for (int A = blockIdx.x * blockDim.x + threadIdx.x; A < nc; A += gridDim.x * blockDim.x) {
    const int AX = ccoords[2 * A], AY = ccoords[2 * A + 1];
    double a0 = 0.0, a1 = 0.0;
    for (int i0 = 2 * AX - span; i0 <= 2 * AX + span; ++i0) {
      const double w0 = weight1(quad, i0, AX);
      if (w0 == 0.0) continue;
      for (int i1 = 2 * AY - span; i1 <= 2 * AY + span; ++i1) {
        const double w1 = weight1(quad, i1, AY);
        if (w1 == 0.0) continue;
        const int fi = fmap.at(i0, i1);
        if (fi < 0) continue;
        const double w = w0 * w1;
        a0 += w * rf[2 * fi];
        a1 += w * rf[2 * fi + 1];
      }
    }
    bc[2 * A] = cdir[A] ? 0.0 : a0;
    bc[2 * A + 1] = cdir[A] ? 0.0 : a1;
  }
}
/// prolong_add (multigrid.hpp:33-39): parents in embedding order
__global__ void k2_prolong(const int* fcoords, int nf, Map2 cmap, int quad, const double* uc, double* uf) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
    int p0[3], p1[3];
    double w0[3], w1[3];
    const int k0 = parents1(quad, fcoords[2 * i], p0, w0), k1 = parents1(quad, fcoords[2 * i + 1], p1, w1);
    double a0 = 0.0, a1 = 0.0;
    for (int a = 0; a < k0; ++a)
      for (int b = 0; b < k1; ++b) {
        const int A = cmap.at(p0[a], p1[b]);
        const double w = w0[a] * w1[b];
        a0 = a0 + w * uc[2 * A];
        a1 = a1 + w * uc[2 * A + 1];
      }
    uf[2 * i] += a0;
    uf[2 * i + 1] += a1;
  }
}
__global__ void k2_zero_dir(int n, const uint8_t* dir, double* x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (dir[i]) x[2 * i] = x[2 * i + 1] = 0.0;
}
/// z = D^-1 r per node (block Jacobi)
__global__ void k2_block_apply(int n, const double* dinv, const double* r, double* z) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double* D = dinv + 4 * i;
    const double r0 = r[2 * i], r1 = r[2 * i + 1];
    z[2 * i] = D[0] * r0 + D[1] * r1;
    z[2 * i + 1] = D[2] * r0 + D[3] * r1;
  }
}

// --------------------------------------------------------------------------- vectors
/// out = a + s b (b may be null: out = a); separate rounding of the product and the sum
__global__ void k2_axpy(long long n, const double* a, double s, const double* b, double* out) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    out[k] = b ? __dadd_rn(a[k], __dmul_rn(s, b[k])) : a[k];
}
__global__ void k2_scale(long long n, double s, const double* a, double* out) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    out[k] = s * a[k];
}
__global__ void k2_sub(long long n, const double* a, const double* b, double* out) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    out[k] = a[k] - b[k];
}
/// g^T D^-1 g per node (the adaptive PN tolerance, solvers.hpp:252-257)
__global__ void k2_gpg(int n, const double* dinv, const double* g, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double* D = dinv + 4 * i;
    const double g0 = g[2 * i], g1 = g[2 * i + 1];
    out[i] = g0 * (D[0] * g0 + D[1] * g1) + g1 * (D[2] * g0 + D[3] * g1);
  }
}
/// v^{n+1} = vel + dv, Dirichlet nodes take their scripted velocity (solvers.hpp:376-379)
__global__ void k2_final_velocity(int n, const double* vel, const double* dv, const uint8_t* dir, const double* bcv,
                                  double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int a = 0; a < 2; ++a) out[2 * i + a] = dir[i] ? bcv[2 * i + a] : vel[2 * i + a] + dv[2 * i + a];
}

// --------------------------------------------------------------------------- matrix-free (objective.hpp:366-440)
/// per particle dP = T : dF with dF = sum_k um_k W_k^T (um: u with Dirichlet nodes zeroed)
__global__ void k2_mf_particle(long long np, const double* rec, Map2 map, const double* xpos, double dx, const double* u,
                               const uint8_t* dir, double* dP) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < np; p += (long long)gridDim.x * blockDim.x) {
    const double* R = rec + p * kRec2;
    int b0, b1;
    d2::stencil2(xpos[2 * p], xpos[2 * p + 1], dx, b0, b1);
    double dF[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < 9; ++k) {
      const double w0 = R[16 + 2 * k], w1 = R[17 + 2 * k];
      if (w0 == 0.0 && w1 == 0.0) continue;
      const int i = map.at(b0 + k / 3, b1 + k % 3);
      if (i < 0 || dir[i]) continue;
      const double u0 = u[2 * i], u1 = u[2 * i + 1];
      dF[0] += u0 * w0;
      dF[1] += u0 * w1;
      dF[2] += u1 * w0;
      dF[3] += u1 * w1;
    }
    for (int r = 0; r < 4; ++r) {
      double acc = R[r * 4] * dF[0];
      for (int c = 1; c < 4; ++c) acc += R[r * 4 + c] * dF[c];
      dP[4 * p + r] = acc;
    }
  }
}
/// y_i = sum_p kappa dP W_k + m_i um_i; y_i = u_i on Dirichlet nodes
__global__ void k2_mf_node(Cells cells, const int* coords, int n, const double* rec, const double* dP, const double* mass,
                           const uint8_t* dir, const double* u, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int X = coords[2 * i], Y = coords[2 * i + 1];
    double a0 = 0.0, a1 = 0.0;
    for (int k = 0; k < 9; ++k) {
      int s, e;
      cells.range(X - k / 3, Y - k % 3, s, e);
      const int kk = (k / 3) * 3 + k % 3;  // node i is stencil position (X - c0, Y - c1)
      for (int t = s; t < e; ++t) {
        const int p = cells.pid[t];
        const double* R = rec + (long long)p * kRec2;
        const double w0 = R[16 + 2 * kk], w1 = R[17 + 2 * kk];
        if (w0 == 0.0 && w1 == 0.0) continue;
        const double* D = dP + 4 * p;
        a0 += R[34] * (D[0] * w0 + D[1] * w1);
        a1 += R[34] * (D[2] * w0 + D[3] * w1);
      }
    }
    if (dir[i]) {
      y[2 * i] = u[2 * i];
      y[2 * i + 1] = u[2 * i + 1];
    } else {
      y[2 * i] = a0 + mass[i] * u[2 * i];
      y[2 * i + 1] = a1 + mass[i] * u[2 * i + 1];
    }
  }
}
/// inverse of the block diagonal of the projected system (objective.hpp:368-396)
__global__ void k2_mf_diag_inv(Cells cells, const int* coords, int n, const double* rec, const double* mass,
                               const uint8_t* dir, double* dinv, int* flags) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int X = coords[2 * i], Y = coords[2 * i + 1];
    double D[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < 9; ++k) {
      int s, e;
      cells.range(X - k / 3, Y - k % 3, s, e);
      for (int t = s; t < e; ++t) {
        const double* R = rec + (long long)cells.pid[t] * kRec2;
        const double* w = R + 16 + 2 * k;
        if (w[0] == 0.0 && w[1] == 0.0) continue;
        double C[4];
        contract2(R, w, w, C);
        for (int q = 0; q < 4; ++q) C[q] = R[34] * C[q];
        const double t01 = 0.5 * (C[1] + C[2]);
        D[0] += 0.5 * (C[0] + C[0]);
        D[1] += t01;
        D[2] += t01;
        D[3] += 0.5 * (C[3] + C[3]);
      }
    }
    D[0] += mass[i];
    D[3] += mass[i];
    if (dir[i]) {
      D[0] = D[3] = 1.0;
      D[1] = D[2] = 0.0;
    }
    M2 Dm{{D[0], D[1], D[2], D[3]}};
    if (!(fabs(d2::m2_det(Dm)) > 0.0)) flags[kSingular] = 1;
    const M2 I = d2::m2_inv(Dm);
    for (int q = 0; q < 4; ++q) dinv[4 * i + q] = I.a[q];
  }
}

// --------------------------------------------------------------------------- G2P, strain, advection (transfer.hpp:68-120)
__global__ void k2_g2p(Parts P, double* x, double* v, double* F, double* C, double* jp, Map2 map, double dx, double dt,
                       const DevMaterial* mats, const double* vel, int* inverted) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P.n; p += (long long)gridDim.x * blockDim.x) {
    const double x0 = P.x[2 * p], x1 = P.x[2 * p + 1];
    int b0, b1;
    d2::stencil2(x0, x1, dx, b0, b1);
    double v0 = 0.0, v1 = 0.0;
    M2 B = d2::m2_zero(), G = d2::m2_zero();
    for (int k = 0; k < 9; ++k) {
      const int n0 = b0 + k / 3, n1 = b1 + k % 3;
      double g0, g1;
      const double w = d2::wgrad2(x0, x1, dx, n0, n1, g0, g1);
      if (w <= 0.0) continue;
      const int i = map.at(n0, n1);
      if (i < 0) continue;
      const double u0 = vel[2 * i], u1 = vel[2 * i + 1];
      const double wu0 = w * u0, wu1 = w * u1;
      const double d0 = dx * (double)n0 - x0, d1 = dx * (double)n1 - x1;
      v0 = v0 + wu0;
      v1 = v1 + wu1;
      B.a[0] += wu0 * d0;
      B.a[1] += wu0 * d1;
      B.a[2] += wu1 * d0;
      B.a[3] += wu1 * d1;
      G.a[0] += u0 * g0;
      G.a[1] += u0 * g1;
      G.a[2] += u1 * g0;
      G.a[3] += u1 * g1;
    }
    const double dinv = 4.0 / (dx * dx);
    v[2 * p] = v0;
    v[2 * p + 1] = v1;
    for (int k = 0; k < 4; ++k) C[4 * p + k] = dinv * B.a[k];
    M2 A, Fn;
    for (int k = 0; k < 4; ++k) {
      A.a[k] = ((k % 3 == 0) ? 1.0 : 0.0) + dt * G.a[k];
      Fn.a[k] = P.F[4 * p + k];
    }
    M2 Fp = d2::m2_mul(A, Fn);
    const DevMaterial mt = mats[P.mat[p]];
    bool skip = false;
    if (d2::m2_det(Fp) <= 0.0) {
      atomicAdd(inverted, 1);
      skip = mt.plasticity == 1 || mt.plasticity == 3;
    }
    if (!skip) Fp = d2::return_map2(Fp, mt, jp ? jp + p : nullptr);
    for (int k = 0; k < 4; ++k) F[4 * p + k] = Fp.a[k];
    x[2 * p] = x0 + dt * v0;
    x[2 * p + 1] = x1 + dt * v1;
  }
}

}  // namespace

// =========================================================================== host context
struct Lvl2 {
  int n = 0, R = 2, S = 25;
  int lo[2] = {0, 0}, ext[2] = {0, 0};
  Buf coords, map, cols, H, dinv, dir, wave, rows;
  Buf u, b, r;  // V-cycle vectors
  std::vector<int> wave_start;  // rows of wave w: rows[wave_start[w], wave_start[w+1])
  Map2 view_map() const { return Map2{{lo[0], lo[1]}, {ext[0], ext[1]}, map.as<int>()}; }
};

struct Context2D {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // scene
  double dx = 0, fps = 24, cn_factor = 24, grav[2] = {0, 0};
  std::vector<DevMaterial> mats_h;
  std::vector<DevCollider> cols_h;
  Buf mats_d, cols_d;
  bool track_jp = false;
  hot_solver_config cfg{};
  // particles (interleaved, the caller's order)
  long long np = 0;
  Buf x, v, F, C, m, vol, jp, mat, x2, v2, F2, C2, jp2;
  // grid / level 0
  Lvl2 L[16];
  int nlevels = 0;
  bool have_state = false, have_H = false;
  int cell_lo[2] = {0, 0}, cell_ext[2] = {0, 0};
  Buf cell_of, cell_cnt, cell_start, cell_cur, cell_pid, scan_tmp, scan_total;
  Buf gmass, gmom, gvel, gbc, gcn, flags_buf, iscal, dscal, vmax;
  double dt = 0;
  // solver vectors
  Buf dv, g, gnew, pdir, u, trial, pe, ne, PFt, rec, nterm, vout, tmpv, dP, pn_dinv;
  struct Hist {
    std::unique_ptr<Buf> s, y;
    double rho;
  };
  std::deque<Hist> hist;
  // time
  double time = 0;
  int frame = 0;
  long long step_index = 0, inversions = 0;
  std::vector<hot_diag_row> diag;

  Parts parts() const {
    return Parts{x.as<double>(), v.as<double>(), F.as<double>(), C.as<double>(), m.as<double>(), vol.as<double>(),
                 track_jp ? jp.as<double>() : nullptr, mat.as<int>(), np};
  }
  Cells cells() const {
    return Cells{{cell_lo[0], cell_lo[1]}, {cell_ext[0], cell_ext[1]}, cell_start.as<int>(), cell_pid.as<int>()};
  }
  int n0() const { return L[0].n; }
  void sync() { H2_CUDA(cudaStreamSynchronize(stream)); }
  /// stream-ordered copy, then wait (the context stream does not synchronise with the legacy stream)
  void copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    if (!bytes) return;
    H2_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, stream));
    sync();
  }
  void check() { H2_CUDA(cudaGetLastError()); }

  // ------------------------------------------------------------------ scalars and flags
  double dsum(const double* a, const double* b, long long len, int slot = 0) {
    k2_dot<<<1, kRedT, 0, stream>>>(a, b, len, dscal.as<double>(), slot);
    count_launches(1);
    double out = 0.0;
    H2_CUDA(cudaMemcpyAsync(&out, dscal.as<double>() + slot, sizeof(double), cudaMemcpyDeviceToHost, stream));
    sync();
    return out;
  }
  void clear_flags() { H2_CUDA(cudaMemsetAsync(flags_buf.p, 0, sizeof(int) * kNumFlags, stream)); }
  void check_flags() {
    int f[kNumFlags];
    H2_CUDA(cudaMemcpyAsync(f, flags_buf.p, sizeof(f), cudaMemcpyDeviceToHost, stream));
    sync();
    check();
    if (f[kBadX]) throw std::invalid_argument("activate_grid: non-finite particle position");
    if (f[kBadF]) throw std::invalid_argument("fcr_energy_density: non-finite deformation gradient");
    if (f[kAsym]) throw std::invalid_argument("project_spd: input is not symmetric");
    if (f[kZeroScale]) throw std::logic_error("scaled_norm: zero characteristic scale (material misconfiguration)");
    if (f[kSingular]) throw std::logic_error("multigrid: singular diagonal block");
  }

  void init(int dev) {
    device = dev;
    H2_CUDA(cudaSetDevice(dev));
    H2_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    flags_buf.ensure(sizeof(int) * kNumFlags);
    iscal.ensure(sizeof(int) * 8);
    dscal.ensure(sizeof(double) * 8);
    vmax.ensure(8);
    scan_total.ensure(8);
  }
  ~Context2D() {
    if (stream) cudaStreamDestroy(stream);
  }

  void set_scene(const hot_scene& s) {
    if (!(s.dx > 0)) throw std::invalid_argument("activate_grid: dx must be positive");
    dx = s.dx;
    fps = s.fps;
    cn_factor = s.cn_length_factor;
    grav[0] = s.gravity[0];
    grav[1] = s.gravity[1];
    mats_h.clear();
    for (int i = 0; i < s.n_materials; ++i) mats_h.push_back(make_dev_material(s.materials[i], 2));
    track_jp = false;
    for (const DevMaterial& mm : mats_h) track_jp = track_jp || mm.plasticity == 2;
    cols_h.clear();
    for (int i = 0; i < s.n_colliders; ++i) {
      const hot_collider& c = s.colliders[i];
      DevCollider d{};
      d.shape = c.shape.kind;
      d.motion = c.motion.kind;
      d.radius = c.shape.radius;
      for (int a = 0; a < 3; ++a) {
        if (c.shape.kind == 0) {
          d.a[a] = c.shape.min[a];
          d.b[a] = c.shape.max[a];
        } else if (c.shape.kind == 2) {
          d.a[a] = c.shape.point[a];
          d.b[a] = c.shape.normal[a];
        } else {
          d.a[a] = c.shape.center[a];
        }
        d.vel[a] = c.motion.velocity[a];
        d.rot_center[a] = c.motion.center[a];
      }
      d.rot_w[2] = c.motion.omega;  // 2D rotation: omega about the out-of-plane axis (simulation.hpp:56-59)
      cols_h.push_back(d);
    }
    mats_d.ensure(sizeof(DevMaterial) * std::max<size_t>(1, mats_h.size()));
    if (!mats_h.empty())
      copy(mats_d.p, mats_h.data(), sizeof(DevMaterial) * mats_h.size(), cudaMemcpyHostToDevice);
    cols_d.ensure(sizeof(DevCollider) * std::max<size_t>(1, cols_h.size()));
    if (!cols_h.empty())
      copy(cols_d.p, cols_h.data(), sizeof(DevCollider) * cols_h.size(), cudaMemcpyHostToDevice);
    cfg = hot_solver_config{s.epsilon, s.tau, s.levels, s.window, 0.5, 1e-4, 30, 10000, 1000,
                            s.solver, s.embedding, 256, s.cn_length_factor};
  }

  // ------------------------------------------------------------------ particles
  void upload(long long n, const double* xh, const double* vh, const double* mh, const double* volh, const double* Fh,
              const double* Ch, const int* math) {
    if (n < 0 || (n > 0 && !xh)) throw std::invalid_argument("particles: x is required");
    np = n;
    const size_t nn = (size_t)std::max<long long>(n, 1);
    x.ensure(16 * nn);
    v.ensure(16 * nn);
    F.ensure(32 * nn);
    C.ensure(32 * nn);
    m.ensure(8 * nn);
    vol.ensure(8 * nn);
    jp.ensure(8 * nn);
    mat.ensure(4 * nn);
    std::vector<double> tmp;
    auto put = [&](Buf& b, const double* src, size_t count, double fill, const double* eye) {
      if (src) {
        copy(b.p, src, 8 * count, cudaMemcpyHostToDevice);
        return;
      }
      tmp.assign(count, fill);
      if (eye)
        for (size_t k = 0; k < count; ++k) tmp[k] = eye[k % 4];
      copy(b.p, tmp.data(), 8 * count, cudaMemcpyHostToDevice);
    };
    const double I[4] = {1.0, 0.0, 0.0, 1.0};
    if (n > 0) {
      put(x, xh, 2 * n, 0.0, nullptr);
      put(v, vh, 2 * n, 0.0, nullptr);
      put(m, mh, n, 0.0, nullptr);
      put(vol, volh, n, 0.0, nullptr);
      put(F, Fh, 4 * n, 0.0, I);
      put(C, Ch, 4 * n, 0.0, nullptr);
      put(jp, nullptr, n, 1.0, nullptr);
      std::vector<int> mt(n, 0);
      if (math) std::memcpy(mt.data(), math, 4 * n);
      for (int k : mt)
        if (k < 0 || k >= (int)mats_h.size()) throw std::invalid_argument("particle material index out of range");
      copy(mat.p, mt.data(), 4 * n, cudaMemcpyHostToDevice);
    }
    have_state = have_H = false;
    nlevels = 0;
  }
  void download(double* xh, double* vh, double* Fh, double* Ch) {
    if (np == 0) return;
    if (xh) H2_CUDA(cudaMemcpyAsync(xh, x.p, 16 * np, cudaMemcpyDeviceToHost, stream));
    if (vh) H2_CUDA(cudaMemcpyAsync(vh, v.p, 16 * np, cudaMemcpyDeviceToHost, stream));
    if (Fh) H2_CUDA(cudaMemcpyAsync(Fh, F.p, 32 * np, cudaMemcpyDeviceToHost, stream));
    if (Ch) H2_CUDA(cudaMemcpyAsync(Ch, C.p, 32 * np, cudaMemcpyDeviceToHost, stream));
    sync();
  }

  // ------------------------------------------------------------------ grid
  /// grid.hpp:137-165 + the particle cells of the gathers
  void activate() {
    Lvl2& l = L[0];
    clear_flags();
    int mm[4] = {1 << 30, 1 << 30, -(1 << 30), -(1 << 30)};
    H2_CUDA(cudaMemcpyAsync(iscal.p, mm, sizeof(mm), cudaMemcpyHostToDevice, stream));
    if (np > 0) {
      k2_bounds<<<gridn(np), 256, 0, stream>>>(parts(), dx, iscal.as<int>(), flags_buf.as<int>());
      count_launches(1);
    }
    H2_CUDA(cudaMemcpyAsync(mm, iscal.p, sizeof(mm), cudaMemcpyDeviceToHost, stream));
    check_flags();
    if (np == 0) {
      l.n = 0;
      cell_ext[0] = cell_ext[1] = 0;
      return;
    }
    cell_lo[0] = mm[0];
    cell_lo[1] = mm[1];
    cell_ext[0] = mm[2] - mm[0] + 1;
    cell_ext[1] = mm[3] - mm[1] + 1;
    l.lo[0] = mm[0];
    l.lo[1] = mm[1];
    l.ext[0] = cell_ext[0] + 2;
    l.ext[1] = cell_ext[1] + 2;
    const long long len = (long long)l.ext[0] * l.ext[1];
    if (len > (1LL << 31) - 2) throw std::invalid_argument("activate_grid: particle extent too large for the dense map");
    Buf& fl = tmpv;  // int flags + scan over the box
    fl.ensure(8 * (size_t)len + 16);
    int* flags = fl.as<int>();
    int* scan = flags + len;
    H2_CUDA(cudaMemsetAsync(flags, 0, 4 * len, stream));
    k2_mark<<<gridn(np), 256, 0, stream>>>(parts(), dx, l.lo[0], l.lo[1], l.ext[1], flags);
    scan_tmp.ensure(4 * (size_t)(len / 4096 + 2));
    launch_exclusive_scan(flags, scan, (int)len, scan_tmp.as<int>(), scan_total.as<int>(), stream);
    int n = 0;
    H2_CUDA(cudaMemcpyAsync(&n, scan_total.p, 4, cudaMemcpyDeviceToHost, stream));
    sync();
    l.n = n;
    l.R = 2;
    l.S = 25;
    l.map.ensure(4 * (size_t)len);
    l.coords.ensure(8 * (size_t)std::max(n, 1));
    k2_compact<<<gridn(len), 256, 0, stream>>>(flags, scan, len, l.lo[0], l.lo[1], l.ext[1], l.map.as<int>(),
                                               l.coords.as<int>());
    // particles by stencil base cell, ascending ids within a cell
    const int ncell = cell_ext[0] * cell_ext[1];
    cell_of.ensure(4 * (size_t)np);
    cell_cnt.ensure(4 * (size_t)(ncell + 1));
    cell_start.ensure(4 * (size_t)(ncell + 1));
    cell_cur.ensure(4 * (size_t)(ncell + 1));
    cell_pid.ensure(4 * (size_t)np);
    scan_tmp.ensure(4 * (size_t)(std::max<long long>(len, ncell + 1) / 4096 + 2));
    H2_CUDA(cudaMemsetAsync(cell_cnt.p, 0, 4 * (size_t)(ncell + 1), stream));
    k2_cell_of<<<gridn(np), 256, 0, stream>>>(parts(), dx, cell_lo[0], cell_lo[1], cell_ext[1], cell_of.as<int>(),
                                              cell_cnt.as<int>());
    launch_exclusive_scan(cell_cnt.as<int>(), cell_start.as<int>(), ncell + 1, scan_tmp.as<int>(), nullptr, stream);
    H2_CUDA(cudaMemcpyAsync(cell_cur.p, cell_start.p, 4 * (size_t)ncell, cudaMemcpyDeviceToDevice, stream));
    k2_cell_fill<<<gridn(np), 256, 0, stream>>>(cell_of.as<int>(), np, cell_cur.as<int>(), cell_pid.as<int>());
    k2_cell_sort<<<gridn(ncell, 128), 128, 0, stream>>>(cell_start.as<int>(), ncell, cell_pid.as<int>());
    count_launches(6);
    check();
  }

  /// activation, P2G, boundary scripts and the objective state's node CN (simulation.hpp:296-304)
  void prepare(double dt_in, double t_now) {
    dt = dt_in;
    activate();
    const int n = n0();
    const size_t nn = (size_t)std::max(n, 1);
    gmass.ensure(8 * nn);
    gmom.ensure(16 * nn);
    gvel.ensure(16 * nn);
    gbc.ensure(16 * nn);
    gcn.ensure(8 * nn);
    L[0].dir.ensure(nn);
    if (n > 0) {
      k2_p2g<<<gridn(n, 128), 128, 0, stream>>>(parts(), cells(), L[0].coords.as<int>(), n, dx, mats_d.as<DevMaterial>(),
                                                cn_factor * dx * dx, dt, gmass.as<double>(), gmom.as<double>(),
                                                gvel.as<double>(), gcn.as<double>());
      k2_bc<<<gridn(n), 256, 0, stream>>>(n, L[0].coords.as<int>(), dx, cols_d.as<DevCollider>(), (int)cols_h.size(),
                                          gvel.as<double>(), gbc.as<double>(), L[0].dir.as<uint8_t>());
      count_launches(2);
    }
    (void)t_now;  // inside tests do not depend on time (simulation.hpp:20)
    for (Buf* b : {&dv, &g, &gnew, &pdir, &u, &trial, &vout, &nterm, &ne})
      b->ensure(16 * nn);
    pe.ensure(8 * (size_t)std::max<long long>(np, 1));
    PFt.ensure(32 * (size_t)std::max<long long>(np, 1));
    check();
    have_state = true;
    have_H = false;
    nlevels = 0;
  }

  // ------------------------------------------------------------------ objective
  /// energy at dv + alpha p (objective.hpp:236-257); PFt stored when want_stress
  double energy(const double* dvp, const double* p, double alpha, bool want_stress) {
    const int n = n0();
    clear_flags();
    k2_node_u<<<gridn(2 * n), 256, 0, stream>>>(2 * n, gvel.as<double>(), dvp, p, alpha, u.as<double>());
    if (np > 0)
      k2_energy_particle<<<gridn(np, 128), 128, 0, stream>>>(parts(), L[0].view_map(), dx, dt, mats_d.as<DevMaterial>(),
                                                             u.as<double>(), pe.as<double>(),
                                                             want_stress ? PFt.as<double>() : nullptr,
                                                             flags_buf.as<int>());
    k2_node_energy<<<gridn(n), 256, 0, stream>>>(n, gmass.as<double>(), gvel.as<double>(), dvp, p, alpha, dt, grav[0],
                                                 grav[1], ne.as<double>());
    count_launches(3);
    const double ep = np > 0 ? dsum(pe.as<double>(), nullptr, np, 0) : 0.0;
    const double en = dsum(ne.as<double>(), nullptr, n, 1);
    check_flags();
    return ep + en;
  }
  /// gradient + scaled norm at dv (PFt from the energy pass at the same dv)
  double gradient(const double* dvp, double* gout) {
    const int n = n0();
    clear_flags();
    k2_gradient<<<gridn(n, 128), 128, 0, stream>>>(parts(), cells(), L[0].coords.as<int>(), n, dx, dt, grav[0], grav[1],
                                                   PFt.as<double>(), gmass.as<double>(), dvp, L[0].dir.as<uint8_t>(),
                                                   gcn.as<double>(), gout, nterm.as<double>(), flags_buf.as<int>());
    count_launches(1);
    const double s = dsum(nterm.as<double>(), nullptr, n, 2);
    check_flags();
    return std::sqrt(s);
  }
  double energy_and_gradient(const double* dvp, double* gout, double* e) {
    *e = energy(dvp, nullptr, 0.0, true);
    return gradient(dvp, gout);
  }

  // ------------------------------------------------------------------ assembly + hierarchy
  void tensors(const double* dvp, bool project) {
    const int n = n0();
    clear_flags();
    rec.ensure(8 * (size_t)kRec2 * std::max<long long>(np, 1));
    k2_node_u<<<gridn(2 * n), 256, 0, stream>>>(2 * n, gvel.as<double>(), dvp, nullptr, 0.0, u.as<double>());
    if (np > 0)
      k2_tensors<<<gridn(np, 128), 128, 0, stream>>>(parts(), L[0].view_map(), dx, dt, mats_d.as<DevMaterial>(),
                                                     u.as<double>(), project ? 1 : 0, rec.as<double>(),
                                                     flags_buf.as<int>());
    count_launches(2);
    check_flags();
  }
  void assemble(const double* dvp, bool project) {
    tensors(dvp, project);
    Lvl2& l = L[0];
    const int n = l.n;
    l.cols.ensure(4 * (size_t)std::max(n, 1) * l.S);
    l.H.ensure(32 * (size_t)std::max(n, 1) * l.S);
    if (n > 0) {
      k2_lower_inactive<<<gridn((long long)n * 12), 256, 0, stream>>>(l.coords.as<int>(), n, l.view_map(), 2,
                                                                       l.H.as<double>(), l.cols.as<int>());
      k2_assemble<<<gridn((long long)n * 13, 128), 128, 0, stream>>>(cells(), l.coords.as<int>(), n, l.view_map(),
                                                                      rec.as<double>(), gmass.as<double>(),
                                                                      l.dir.as<uint8_t>(), l.H.as<double>(),
                                                                      l.cols.as<int>());
      count_launches(2);
    }
    check();
    have_H = true;
    nlevels = 1;
  }
  void finalize(int m, int q) {
    Lvl2& l = L[m];
    const int n = l.n;
    l.dinv.ensure(32 * (size_t)std::max(n, 1));
    l.wave.ensure(4 * (size_t)std::max(n, 1));
    l.rows.ensure(4 * (size_t)std::max(n, 1));
    for (Buf* b : {&l.u, &l.b, &l.r}) b->ensure(16 * (size_t)std::max(n, 1));
    const int a0 = l.lo[0] >= 0 ? l.lo[0] / q : -((-l.lo[0] + q - 1) / q);
    const int b0 = l.lo[1] >= 0 ? l.lo[1] / q : -((-l.lo[1] + q - 1) / q);
    clear_flags();
    if (n > 0) {
      k2_finalize<<<gridn(n), 256, 0, stream>>>(l.coords.as<int>(), n, l.S, l.H.as<double>(), q, l.R, a0, b0,
                                                l.dinv.as<double>(), l.wave.as<int>(), flags_buf.as<int>());
      count_launches(1);
    }
    check_flags();
    // bucket rows by wave on the host (stable: ascending row index within a wave)
    std::vector<int> w(n);
    if (n > 0) copy(w.data(), l.wave.p, 4 * (size_t)n, cudaMemcpyDeviceToHost);
    int nw = 0;
    for (int t : w) nw = std::max(nw, t + 1);
    std::vector<int> cnt(nw + 1, 0), rows(n);
    for (int t : w) ++cnt[t + 1];
    for (int k = 0; k < nw; ++k) cnt[k + 1] += cnt[k];
    std::vector<int> cur(cnt.begin(), cnt.end() - 1);
    for (int i = 0; i < n; ++i) rows[cur[w[i]]++] = i;
    l.wave_start.clear();
    for (int k = 0; k <= nw; ++k)  // drop empty waves
      if (k == nw || cnt[k + 1] > cnt[k]) l.wave_start.push_back(cnt[k]);
    if (n > 0) copy(l.rows.p, rows.data(), 4 * (size_t)n, cudaMemcpyHostToDevice);
  }
  /// build_hierarchy (multigrid.hpp:258-294)
  void build_hierarchy(int levels, int embedding) {
    if (levels < 1) throw std::invalid_argument("build_hierarchy: need at least one level");
    const int quad = embedding == 0 ? 1 : 0;
    finalize(0, 3);
    nlevels = 1;
    for (int mlev = 1; mlev < levels && mlev < 16; ++mlev) {
      Lvl2& f = L[mlev - 1];
      Lvl2& c = L[mlev];
      if (f.n == 0) break;
      c.R = quad ? 3 : 2;
      c.S = (2 * c.R + 1) * (2 * c.R + 1);
      // coarse box: parents of the fine box
      c.lo[0] = (f.lo[0] >= 0 ? f.lo[0] / 2 : (f.lo[0] - 1) / 2) - 1;
      c.lo[1] = (f.lo[1] >= 0 ? f.lo[1] / 2 : (f.lo[1] - 1) / 2) - 1;
      c.ext[0] = f.ext[0] / 2 + 4;
      c.ext[1] = f.ext[1] / 2 + 4;
      const long long len = (long long)c.ext[0] * c.ext[1];
      Buf& tmp = tmpv;
      tmp.ensure(9 * (size_t)len + 16);
      int* flags = tmp.as<int>();
      int* scan = flags + len;
      uint8_t* cdd = reinterpret_cast<uint8_t*>(scan + len);
      H2_CUDA(cudaMemsetAsync(flags, 0, 4 * (size_t)len, stream));
      H2_CUDA(cudaMemsetAsync(cdd, 0, (size_t)len, stream));
      k2_mark_parents<<<gridn(f.n), 256, 0, stream>>>(f.coords.as<int>(), f.dir.as<uint8_t>(), f.n, quad, c.lo[0],
                                                      c.lo[1], c.ext[1], flags, cdd);
      scan_tmp.ensure(4 * (size_t)(len / 4096 + 2));
      launch_exclusive_scan(flags, scan, (int)len, scan_tmp.as<int>(), scan_total.as<int>(), stream);
      int n = 0;
      H2_CUDA(cudaMemcpyAsync(&n, scan_total.p, 4, cudaMemcpyDeviceToHost, stream));
      sync();
      if (n == 0) break;  // truncated
      c.n = n;
      c.map.ensure(4 * (size_t)len);
      c.coords.ensure(8 * (size_t)n);
      c.dir.ensure((size_t)n);
      c.cols.ensure(4 * (size_t)n * c.S);
      c.H.ensure(32 * (size_t)n * c.S);
      k2_compact<<<gridn(len), 256, 0, stream>>>(flags, scan, len, c.lo[0], c.lo[1], c.ext[1], c.map.as<int>(),
                                                 c.coords.as<int>());
      k2_gather_dir<<<gridn(n), 256, 0, stream>>>(cdd, c.coords.as<int>(), n, c.lo[0], c.lo[1], c.ext[1],
                                                  c.dir.as<uint8_t>());
      k2_lower_inactive<<<gridn((long long)n * (c.S / 2)), 256, 0, stream>>>(c.coords.as<int>(), n, c.view_map(), c.R,
                                                                             c.H.as<double>(), c.cols.as<int>());
      const int U = c.S - c.S / 2;
      k2_galerkin<<<gridn((long long)n * U, 128), 128, 0, stream>>>(c.coords.as<int>(), n, c.view_map(), c.R,
                                                                     f.coords.as<int>(), f.view_map(), f.R,
                                                                     f.H.as<double>(), quad, c.dir.as<uint8_t>(),
                                                                     c.H.as<double>(), c.cols.as<int>());
      count_launches(5);
      check();
      finalize(mlev, quad ? 3 : 2);
      nlevels = mlev + 1;
    }
  }

  // ------------------------------------------------------------------ multigrid cycle
  void sgs(int mlev, double* uu, const double* bb) {
    Lvl2& l = L[mlev];
    const int nw = (int)l.wave_start.size() - 1;
    auto wave = [&](int w) {
      const int s = l.wave_start[w], cnt = l.wave_start[w + 1] - s;
      k2_sgs_wave<<<gridn(cnt, 128), 128, 0, stream>>>(l.rows.as<int>() + s, cnt, l.S, l.H.as<double>(),
                                                       l.cols.as<int>(), l.dinv.as<double>(), bb, uu);
    };
    for (int w = 0; w < nw; ++w) wave(w);
    for (int w = nw - 1; w >= 0; --w) wave(w);
    count_launches(2 * nw);
  }
  void spmv(int mlev, const double* xx, const double* bb, double* yy) {
    Lvl2& l = L[mlev];
    k2_spmv<<<gridn(l.n, 128), 128, 0, stream>>>(l.n, l.S, l.H.as<double>(), l.cols.as<int>(), xx, bb, yy);
    count_launches(1);
  }
  /// Jacobi-PCG from zero (pcg.hpp:17-46) with host scalars; returns iterations
  template <class ApplyA, class ApplyP>
  int pcg(ApplyA&& apply_a, ApplyP&& apply_p, const double* bb, double* xx, long long len, double rel, int cap,
          bool& converged, Buf& rb, Buf& zb, Buf& pb, Buf& apb) {
    for (Buf* b : {&rb, &zb, &pb, &apb}) b->ensure(8 * (size_t)std::max<long long>(len, 1));
    double *r = rb.as<double>(), *z = zb.as<double>(), *p = pb.as<double>(), *Ap = apb.as<double>();
    H2_CUDA(cudaMemsetAsync(xx, 0, 8 * len, stream));
    H2_CUDA(cudaMemcpyAsync(r, bb, 8 * len, cudaMemcpyDeviceToDevice, stream));
    apply_p(r, z);
    double rho = dsum(r, z, len);
    converged = true;
    if (!(rho > 0.0)) {
      if (rho < 0.0) throw SolverFailure("pcg: preconditioner is not positive definite");
      return 0;
    }
    const double threshold = rel * rel * rho;
    H2_CUDA(cudaMemcpyAsync(p, z, 8 * len, cudaMemcpyDeviceToDevice, stream));
    for (int it = 0; it < cap; ++it) {
      apply_a(p, Ap);
      const double pAp = dsum(p, Ap, len);
      if (!(pAp > 0.0)) throw SolverFailure("pcg: system matrix is not positive definite");
      const double alpha = rho / pAp;
      k2_axpy<<<gridn(len), 256, 0, stream>>>(len, xx, alpha, p, xx);
      k2_axpy<<<gridn(len), 256, 0, stream>>>(len, r, -alpha, Ap, r);
      count_launches(2);
      apply_p(r, z);
      const double rho_new = dsum(r, z, len);
      if (rho_new <= threshold) return it + 1;
      const double beta = rho_new / rho;
      k2_axpy<<<gridn(len), 256, 0, stream>>>(len, z, beta, p, p);
      count_launches(1);
      rho = rho_new;
    }
    converged = false;
    return cap;
  }
  Buf cr, cz, cp, cap_;
  /// vcycle (multigrid.hpp:363-392); returns coarse PCG iterations
  int vcycle(const double* b0, double* out, bool pinned, int pinned_cap) {
    const int M = nlevels;
    H2_CUDA(cudaMemcpyAsync(L[0].b.p, b0, 16 * (size_t)L[0].n, cudaMemcpyDeviceToDevice, stream));
    k2_zero_dir<<<gridn(L[0].n), 256, 0, stream>>>(L[0].n, L[0].dir.as<uint8_t>(), L[0].b.as<double>());
    count_launches(1);
    for (int mlev = 0; mlev < M - 1; ++mlev) {
      Lvl2& l = L[mlev];
      H2_CUDA(cudaMemsetAsync(l.u.p, 0, 16 * (size_t)l.n, stream));
      sgs(mlev, l.u.as<double>(), l.b.as<double>());
      spmv(mlev, l.u.as<double>(), l.b.as<double>(), l.r.as<double>());
      Lvl2& c = L[mlev + 1];
      k2_restrict<<<gridn(c.n), 256, 0, stream>>>(c.coords.as<int>(), c.n, c.dir.as<uint8_t>(), l.view_map(),
                                                  cfg.embedding == 0 ? 1 : 0, l.r.as<double>(), c.b.as<double>());
      count_launches(1);
    }
    Lvl2& bot = L[M - 1];
    bool conv = true;
    const long long len = 2LL * bot.n;
    const int it = pcg(
        [&](const double* xx, double* yy) { spmv(M - 1, xx, nullptr, yy); },
        [&](const double* rr, double* zz) {
          k2_block_apply<<<gridn(bot.n), 256, 0, stream>>>(bot.n, bot.dinv.as<double>(), rr, zz);
          count_launches(1);
        },
        bot.b.as<double>(), bot.u.as<double>(), len, pinned ? 1e-14 : 0.5, pinned ? pinned_cap : 10000, conv, cr,
        cz, cp, cap_);
    for (int mlev = M - 2; mlev >= 0; --mlev) {
      Lvl2& l = L[mlev];
      k2_prolong<<<gridn(l.n), 256, 0, stream>>>(l.coords.as<int>(), l.n, L[mlev + 1].view_map(),
                                                 cfg.embedding == 0 ? 1 : 0, L[mlev + 1].u.as<double>(),
                                                 l.u.as<double>());
      count_launches(1);
      sgs(mlev, l.u.as<double>(), l.b.as<double>());
    }
    H2_CUDA(cudaMemcpyAsync(out, L[0].u.p, 16 * (size_t)L[0].n, cudaMemcpyDeviceToDevice, stream));
    check();
    return it;
  }

  // ------------------------------------------------------------------ the solve (solvers.hpp)
  struct SolveOut {
    int outer = 0;
    long long inner = 0;
    bool converged = false;
  };
  double e_curr = 0, residual = 0, target = 0;
  long long work = 0;
  std::chrono::steady_clock::time_point t0;
  int cur_frame = 0;
  long long cur_step = 0;

  /// OuterLoop (solvers.hpp:137-187): init at dv = 0
  void outer_init(int frame_no, long long step_no) {
    const int n = n0();
    cur_frame = frame_no;
    cur_step = step_no;
    t0 = std::chrono::steady_clock::now();
    work = 0;
    target = cfg.epsilon * std::sqrt((double)n);
    H2_CUDA(cudaMemsetAsync(dv.p, 0, 16 * (size_t)n, stream));
    residual = energy_and_gradient(dv.as<double>(), g.as<double>(), &e_curr);
  }
  /// accept (solvers.hpp:160-186): line search along p, s = alpha p, y = g_new - g
  void accept(const double* p, int outer, long long inner_this, Buf* s_out, Buf* y_out) {
    const long long len = 2LL * n0();
    const double gdotp = dsum(g.as<double>(), p, len);
    if (!(gdotp < 0.0)) throw SolverFailure("line_search: not a descent direction");
    double alpha = 1.0, e = 0.0;
    bool ok = false;
    for (int k = 0; k < cfg.ls_max_steps; ++k) {
      k2_axpy<<<gridn(len), 256, 0, stream>>>(len, dv.as<double>(), alpha, p, trial.as<double>());
      count_launches(1);
      e = energy(trial.as<double>(), nullptr, 0.0, false);
      if (e <= e_curr + cfg.ls_armijo * alpha * gdotp) {
        ok = true;
        break;
      }
      alpha *= cfg.ls_shrink;
    }
    if (!ok) throw SolverFailure("line_search: no acceptable step (gradient/Hessian inconsistency)");
    if (s_out) {
      s_out->ensure(8 * (size_t)len);
      k2_scale<<<gridn(len), 256, 0, stream>>>(len, alpha, p, s_out->as<double>());
      k2_axpy<<<gridn(len), 256, 0, stream>>>(len, dv.as<double>(), 1.0, s_out->as<double>(), dv.as<double>());
    } else {
      k2_scale<<<gridn(len), 256, 0, stream>>>(len, alpha, p, tmpv_s());
      k2_axpy<<<gridn(len), 256, 0, stream>>>(len, dv.as<double>(), 1.0, tmpv_s(), dv.as<double>());
    }
    count_launches(2);
    double enew = 0.0;
    residual = energy_and_gradient(dv.as<double>(), gnew.as<double>(), &enew);
    if (y_out) {
      y_out->ensure(8 * (size_t)len);
      k2_sub<<<gridn(len), 256, 0, stream>>>(len, gnew.as<double>(), g.as<double>(), y_out->as<double>());
      count_launches(1);
    }
    std::swap(g.p, gnew.p);
    std::swap(g.cap, gnew.cap);
    e_curr = e;
    work += inner_this;
    diag.push_back(hot_diag_row{cur_frame, cur_step, outer, residual, e_curr, alpha, inner_this, work,
                                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count()});
  }
  Buf sbuf;
  double* tmpv_s() {
    sbuf.ensure(16 * (size_t)std::max(n0(), 1));
    return sbuf.as<double>();
  }
  /// lbfgs_direction (solvers.hpp:114-129) with the V-cycle initializer
  long long lbfgs_direction(double* out) {
    const long long len = 2LL * n0();
    Buf& q = pdir;
    k2_scale<<<gridn(len), 256, 0, stream>>>(len, -1.0, g.as<double>(), q.as<double>());
    count_launches(1);
    const int mh = (int)hist.size();
    std::vector<double> alpha(mh);
    for (int k = 0; k < mh; ++k) {
      const Hist& h = hist[hist.size() - 1 - k];
      alpha[k] = h.rho * dsum(h.s->as<double>(), q.as<double>(), len);
      k2_axpy<<<gridn(len), 256, 0, stream>>>(len, q.as<double>(), -alpha[k], h.y->as<double>(), q.as<double>());
      count_launches(1);
    }
    const int it = vcycle(q.as<double>(), out, false, 0);
    for (int k = mh - 1; k >= 0; --k) {
      const Hist& h = hist[hist.size() - 1 - k];
      const double beta = h.rho * dsum(h.y->as<double>(), out, len);
      k2_axpy<<<gridn(len), 256, 0, stream>>>(len, out, alpha[k] - beta, h.s->as<double>(), out);
      count_launches(1);
    }
    return it;
  }
  /// solve_quasi_newton (solvers.hpp:191-231)
  SolveOut solve_qn(int levels, int frame_no, long long step_no) {
    SolveOut out;
    outer_init(frame_no, step_no);
    if (residual <= target) {
      out.converged = true;
      return out;
    }
    assemble(dv.as<double>(), true);
    build_hierarchy(levels, cfg.embedding);
    hist.clear();
    const long long len = 2LL * n0();
    Buf dir_buf;
    dir_buf.ensure(8 * (size_t)std::max<long long>(len, 1));
    for (int outer = 1; outer <= cfg.outer_cap; ++outer) {
      const long long inner_this = lbfgs_direction(dir_buf.as<double>());
      Hist h{std::make_unique<Buf>(), std::make_unique<Buf>(), 0.0};
      accept(dir_buf.as<double>(), outer, inner_this, h.s.get(), h.y.get());
      // LBFGSHistory::push (solvers.hpp:86-93)
      const double ys = dsum(h.y->as<double>(), h.s->as<double>(), len);
      const double yy = dsum(h.y->as<double>(), h.y->as<double>(), len);
      const double ss = dsum(h.s->as<double>(), h.s->as<double>(), len);
      if (ys > 1e-12 * std::sqrt(yy) * std::sqrt(ss)) {
        if ((int)hist.size() == std::max(1, cfg.window)) hist.pop_front();
        h.rho = 1.0 / ys;
        hist.push_back(std::move(h));
      }
      out.outer = outer;
      out.inner += inner_this;
      if (residual <= target) {
        out.converged = true;
        break;
      }
    }
    if (!out.converged)
      throw SolverFailure("quasi-newton solve: outer iteration cap reached (residual " + std::to_string(residual) + ")");
    return out;
  }
  Buf pr, pz, pp, pap, pn_rhs, pn_x;
  /// solve_projected_newton (solvers.hpp:235-310): 1 assembled, 2 matrix-free, 3 multigrid
  SolveOut solve_pn(int variant, int frame_no, long long step_no) {
    SolveOut out;
    outer_init(frame_no, step_no);
    if (residual <= target) {
      out.converged = true;
      return out;
    }
    const int n = n0();
    const long long len = 2LL * n;
    pn_dinv.ensure(32 * (size_t)std::max(n, 1));
    pn_rhs.ensure(8 * (size_t)std::max<long long>(len, 1));
    pn_x.ensure(8 * (size_t)std::max<long long>(len, 1));
    for (int outer = 1; outer <= cfg.outer_cap; ++outer) {
      double* dinv;
      if (variant == 2) {
        tensors(dv.as<double>(), true);
        clear_flags();
        k2_mf_diag_inv<<<gridn(n, 128), 128, 0, stream>>>(cells(), L[0].coords.as<int>(), n, rec.as<double>(),
                                                          gmass.as<double>(), L[0].dir.as<uint8_t>(),
                                                          pn_dinv.as<double>(), flags_buf.as<int>());
        count_launches(1);
        check_flags();
        dinv = pn_dinv.as<double>();
      } else {
        assemble(dv.as<double>(), true);
        if (variant == 3) build_hierarchy(cfg.levels, cfg.embedding);
        else finalize(0, 3);
        dinv = L[0].dinv.as<double>();
      }
      k2_gpg<<<gridn(n), 256, 0, stream>>>(n, dinv, g.as<double>(), nterm.as<double>());
      count_launches(1);
      const double gpg = dsum(nterm.as<double>(), nullptr, n);
      const double k = std::min(0.5, std::sqrt(std::max(std::sqrt(gpg), cfg.tau)));  // solvers.hpp:59-62
      k2_scale<<<gridn(len), 256, 0, stream>>>(len, -1.0, g.as<double>(), pn_rhs.as<double>());
      count_launches(1);
      long long inner_this = 0;
      bool conv = true;
      auto jacobi = [&](const double* r, double* z) {
        k2_block_apply<<<gridn(n), 256, 0, stream>>>(n, dinv, r, z);
        count_launches(1);
      };
      if (variant == 2) {
        dP.ensure(32 * (size_t)std::max<long long>(np, 1));
        auto mf = [&](const double* xx, double* yy) {
          if (np > 0)
            k2_mf_particle<<<gridn(np, 128), 128, 0, stream>>>(np, rec.as<double>(), L[0].view_map(), x.as<double>(), dx,
                                                               xx, L[0].dir.as<uint8_t>(), dP.as<double>());
          k2_mf_node<<<gridn(n, 128), 128, 0, stream>>>(cells(), L[0].coords.as<int>(), n, rec.as<double>(),
                                                        dP.as<double>(), gmass.as<double>(), L[0].dir.as<uint8_t>(),
                                                        xx, yy);
          count_launches(2);
        };
        inner_this = pcg(mf, jacobi, pn_rhs.as<double>(), pn_x.as<double>(), len, k, cfg.cg_cap, conv, pr, pz, pp, pap);
      } else if (variant == 1) {
        inner_this = pcg([&](const double* xx, double* yy) { spmv(0, xx, nullptr, yy); }, jacobi, pn_rhs.as<double>(),
                         pn_x.as<double>(), len, k, cfg.cg_cap, conv, pr, pz, pp, pap);
      } else {
        long long vc = 0;
        auto mg = [&](const double* r, double* z) { vc += vcycle(r, z, true, cfg.pinned_coarse_iterations); };
        inner_this = pcg([&](const double* xx, double* yy) { spmv(0, xx, nullptr, yy); }, mg, pn_rhs.as<double>(),
                         pn_x.as<double>(), len, k, cfg.cg_cap, conv, pr, pz, pp, pap);
        inner_this += vc;
      }
      accept(pn_x.as<double>(), outer, inner_this, nullptr, nullptr);
      out.outer = outer;
      out.inner += inner_this;
      if (residual <= target) {
        out.converged = true;
        break;
      }
    }
    if (!out.converged)
      throw SolverFailure("projected newton solve: outer iteration cap reached (residual " + std::to_string(residual) +
                          ")");
    return out;
  }
  /// step_grid (solvers.hpp:354-381)
  SolveOut step_grid(int frame_no, long long step_no) {
    switch (cfg.kind) {
      case 0: return solve_qn(cfg.levels, frame_no, step_no);
      case 4: return solve_qn(1, frame_no, step_no);
      case 1: return solve_pn(1, frame_no, step_no);
      case 2: return solve_pn(2, frame_no, step_no);
      case 3: return solve_pn(3, frame_no, step_no);
    }
    throw std::invalid_argument("unknown solver kind");
  }
  void final_velocity() {
    const int n = n0();
    k2_final_velocity<<<gridn(n), 256, 0, stream>>>(n, gvel.as<double>(), dv.as<double>(), L[0].dir.as<uint8_t>(),
                                                    gbc.as<double>(), vout.as<double>());
    count_launches(1);
  }

  /// advance_step (simulation.hpp:286-323)
  void advance(double frame_end, hot_step_stats* st) {
    double vm = 0.0;
    if (np > 0) {
      H2_CUDA(cudaMemsetAsync(vmax.p, 0, 8, stream));
      k2_vmax<<<gridn(np), 256, 0, stream>>>(v.as<double>(), np, vmax.as<unsigned long long>());
      count_launches(1);
      unsigned long long bits = 0;
      H2_CUDA(cudaMemcpyAsync(&bits, vmax.p, 8, cudaMemcpyDeviceToHost, stream));
      sync();
      std::memcpy(&vm, &bits, 8);
    }
    const double frame = 1.0 / fps;  // cfl_dt (grid.hpp:168-173)
    double dtn = vm <= 0.0 ? frame : std::min(frame, 0.6 * dx / vm);
    if (frame_end > 0.0) dtn = std::min(dtn, frame_end - time);
    if (!(dtn > 0.0)) throw SolverFailure("advance_step: non-positive time step");
    prepare(dtn, time);
    SolveOut so;
    try {
      so = step_grid(frame, step_index);
    } catch (const SolverFailure& e) {
      throw SolverFailure("step " + std::to_string(step_index) + ": " + e.what());
    }
    final_velocity();
    // G2P, strain + return map, advection into fresh buffers (failure above leaves particles as they were)
    const size_t nn = (size_t)std::max<long long>(np, 1);
    x2.ensure(16 * nn);
    v2.ensure(16 * nn);
    F2.ensure(32 * nn);
    C2.ensure(32 * nn);
    jp2.ensure(8 * nn);
    H2_CUDA(cudaMemsetAsync(iscal.p, 0, 4, stream));
    if (np > 0) {
      H2_CUDA(cudaMemcpyAsync(jp2.p, jp.p, 8 * np, cudaMemcpyDeviceToDevice, stream));
      k2_g2p<<<gridn(np, 128), 128, 0, stream>>>(parts(), x2.as<double>(), v2.as<double>(), F2.as<double>(),
                                                 C2.as<double>(), track_jp ? jp2.as<double>() : nullptr,
                                                 L[0].view_map(), dx, dtn, mats_d.as<DevMaterial>(), vout.as<double>(),
                                                 iscal.as<int>());
      count_launches(1);
    }
    int inv = 0;
    H2_CUDA(cudaMemcpyAsync(&inv, iscal.p, 4, cudaMemcpyDeviceToHost, stream));
    sync();
    check();
    for (auto pr2 : {std::make_pair(&x, &x2), std::make_pair(&v, &v2), std::make_pair(&F, &F2), std::make_pair(&C, &C2),
                     std::make_pair(&jp, &jp2)}) {
      std::swap(pr2.first->p, pr2.second->p);
      std::swap(pr2.first->cap, pr2.second->cap);
    }
    inversions += inv;
    time += dtn;
    ++step_index;
    if (st) *st = hot_step_stats{dtn, so.outer, so.inner, n0(), so.converged ? 1 : 0};
  }
};

// =========================================================================== entry points
Context2D* ctx2d_new(int device, const hot_scene& s) {
  auto c = std::make_unique<Context2D>();
  c->init(device);
  c->set_scene(s);
  return c.release();
}
void ctx2d_delete(Context2D* c) { delete c; }
void ctx2d_set_solver(Context2D* c, const hot_solver_config& cfg) { c->cfg = cfg; }
void ctx2d_upload(Context2D* c, long long n, const double* x, const double* v, const double* mass, const double* vol,
                  const double* F, const double* C, const int* mat) {
  c->upload(n, x, v, mass, vol, F, C, mat);
}
void ctx2d_download(Context2D* c, double* x, double* v, double* F, double* C) { c->download(x, v, F, C); }
void ctx2d_set_plastic_state(Context2D* c, const double* Jp) {
  if (c->np > 0) c->copy(c->jp.p, Jp, 8 * c->np, cudaMemcpyHostToDevice);
}
void ctx2d_get_plastic_state(Context2D* c, double* Jp) {
  if (c->np > 0) c->copy(Jp, c->jp.p, 8 * c->np, cudaMemcpyDeviceToHost);
}
long long ctx2d_particle_count(Context2D* c) { return c->np; }
void ctx2d_set_time(Context2D* c, double time, int frame, long long step) {
  c->time = time;
  c->frame = frame;
  c->step_index = step;
}
void ctx2d_get_time(Context2D* c, double* time, int* frame, long long* step, long long* inversions) {
  if (time) *time = c->time;
  if (frame) *frame = c->frame;
  if (step) *step = c->step_index;
  if (inversions) *inversions = c->inversions;
}
void ctx2d_advance(Context2D* c, double frame_end, hot_step_stats* out) { c->advance(frame_end, out); }
int ctx2d_diagnostics(Context2D* c, hot_diag_row* rows, int cap) {
  const int cnt = (int)c->diag.size();
  if (rows)
    for (int i = 0; i < std::min(cap, cnt); ++i) rows[i] = c->diag[i];
  return cnt;
}
void ctx2d_clear_diagnostics(Context2D* c) { c->diag.clear(); }
void ctx2d_prepare(Context2D* c, double dt, double time) {
  c->prepare(dt, time);
  c->sync();
}
int ctx2d_node_count(Context2D* c) { return c->L[0].n; }
static void need_state2(Context2D* c) {
  if (!c->have_state) throw std::logic_error("no prepared grid state (call hot_stage_prepare)");
}
void ctx2d_grid(Context2D* c, int* coords, double* mass, double* velocity, double* momentum, unsigned char* dirichlet,
                double* bc_velocity, double* cn_scale) {
  need_state2(c);
  const int n = c->L[0].n;
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    if (dst && bytes) H2_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  };
  cp(coords, c->L[0].coords.p, 8 * (size_t)n);
  cp(mass, c->gmass.p, 8 * (size_t)n);
  cp(velocity, c->gvel.p, 16 * (size_t)n);
  cp(momentum, c->gmom.p, 16 * (size_t)n);
  cp(dirichlet, c->L[0].dir.p, (size_t)n);
  cp(bc_velocity, c->gbc.p, 16 * (size_t)n);
  cp(cn_scale, c->gcn.p, 8 * (size_t)n);
  c->sync();
}
void ctx2d_set_grid(Context2D* c, const double* velocity, const unsigned char* dirichlet, const double* bc_velocity) {
  need_state2(c);
  const int n = c->L[0].n;
  if (velocity) c->copy(c->gvel.p, velocity, 16 * (size_t)n, cudaMemcpyHostToDevice);
  if (dirichlet) c->copy(c->L[0].dir.p, dirichlet, (size_t)n, cudaMemcpyHostToDevice);
  if (bc_velocity) c->copy(c->gbc.p, bc_velocity, 16 * (size_t)n, cudaMemcpyHostToDevice);
}
static void upload_dv(Context2D* c, const double* dv) {
  const int n = c->L[0].n;
  std::vector<double> h(dv, dv + 2 * (size_t)n);
  for (double v : h)
    if (!std::isfinite(v)) throw std::invalid_argument("energy: non-finite dv");
  c->copy(c->trial.p, dv, 16 * (size_t)n, cudaMemcpyHostToDevice);
}
void ctx2d_energy(Context2D* c, const double* dv, double* energy) {
  need_state2(c);
  upload_dv(c, dv);
  *energy = c->energy(c->trial.as<double>(), nullptr, 0.0, false);
}
void ctx2d_gradient(Context2D* c, const double* dv, double* gout, double* scaled_norm) {
  need_state2(c);
  upload_dv(c, dv);
  double e = 0.0;
  const double nrm = c->energy_and_gradient(c->trial.as<double>(), c->gnew.as<double>(), &e);
  if (gout) c->copy(gout, c->gnew.p, 16 * (size_t)c->L[0].n, cudaMemcpyDeviceToHost);
  if (scaled_norm) *scaled_norm = nrm;
}
void ctx2d_assemble(Context2D* c, const double* dv, int project) {
  need_state2(c);
  upload_dv(c, dv);
  c->assemble(c->trial.as<double>(), project != 0);
  c->sync();
}
void ctx2d_build_hierarchy(Context2D* c, int levels, int embedding) {
  if (!c->have_H) throw std::logic_error("no matrix assembled");
  c->cfg.embedding = embedding;
  c->build_hierarchy(levels, embedding);
}
int ctx2d_level_count(Context2D* c) { return c->nlevels; }
void ctx2d_level_shape(Context2D* c, int level, int* rows, int* slots) {
  if (level < 0 || level >= c->nlevels) throw std::logic_error("no such level");
  *rows = c->L[level].n;
  *slots = c->L[level].S;
}
void ctx2d_level_matrix(Context2D* c, int level, double* blocks, int* cols, int* coords, unsigned char* dirichlet) {
  if (level < 0 || level >= c->nlevels) throw std::logic_error("no such level");
  const Lvl2& l = c->L[level];
  const size_t n = (size_t)l.n;
  std::vector<int> cl((cols || blocks) ? n * l.S : 0);
  if (!cl.empty()) c->copy(cl.data(), l.cols.p, 4 * cl.size(), cudaMemcpyDeviceToHost);
  if (cols) std::memcpy(cols, cl.data(), 4 * cl.size());
  if (blocks) {
    c->copy(blocks, l.H.p, 32 * n * l.S, cudaMemcpyDeviceToHost);
    for (size_t k = 0; k < n * l.S; ++k)
      if (cl[k] < 0)
        for (int e = 0; e < 4; ++e) blocks[4 * k + e] = 0.0;
  }
  if (coords) c->copy(coords, l.coords.p, 8 * n, cudaMemcpyDeviceToHost);
  if (dirichlet) c->copy(dirichlet, l.dir.p, n, cudaMemcpyDeviceToHost);
}
void ctx2d_matvec(Context2D* c, int level, const double* x, double* y) {
  if (level < 0 || level >= c->nlevels) throw std::logic_error("no such level");
  Lvl2& l = c->L[level];
  l.b.ensure(16 * (size_t)std::max(l.n, 1));
  l.r.ensure(16 * (size_t)std::max(l.n, 1));
  c->copy(l.b.p, x, 16 * (size_t)l.n, cudaMemcpyHostToDevice);
  c->spmv(level, l.b.as<double>(), nullptr, l.r.as<double>());
  c->copy(y, l.r.p, 16 * (size_t)l.n, cudaMemcpyDeviceToHost);
  c->check();
}
void ctx2d_vcycle(Context2D* c, const double* b, double* u, int* coarse_iterations) {
  if (c->nlevels < 1) throw std::logic_error("no hierarchy");
  const int n = c->L[0].n;
  c->copy(c->trial.p, b, 16 * (size_t)n, cudaMemcpyHostToDevice);
  const int it = c->vcycle(c->trial.as<double>(), c->vout.as<double>(), false, 0);
  c->copy(u, c->vout.p, 16 * (size_t)n, cudaMemcpyDeviceToHost);
  if (coarse_iterations) *coarse_iterations = it;
}
void ctx2d_step_grid(Context2D* c, double* velocity, double* dv, int* outer, long long* inner, int* converged, int frame,
                     long long step) {
  need_state2(c);
  const auto so = c->step_grid(frame, step);
  c->final_velocity();
  const int n = c->L[0].n;
  if (velocity) H2_CUDA(cudaMemcpyAsync(velocity, c->vout.p, 16 * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  if (dv) H2_CUDA(cudaMemcpyAsync(dv, c->dv.p, 16 * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (outer) *outer = so.outer;
  if (inner) *inner = so.inner;
  if (converged) *converged = so.converged ? 1 : 0;
}
void* ctx2d_stream(Context2D* c) { return c->stream; }

}  // namespace hotb200
