// Device-side math for the B200 HOT step: quadratic B-spline weights, 3x3 fp64 algebra,
// the sign-corrected 3x3 SVD, fixed-corotated energy / stress / projected stress
// derivative, and the plastic return maps.  Everything is fp64 and 3D.
//
// Reference semantics (file:line under /root/reference/proj/include/hotmpm):
//   kernel_weight_1d / kernel_derivative_1d / kernel_gradient  grid.hpp:22-73
//   svd_rv (sigma descending, sign of det F on sigma[2])         constitutive.hpp:66-82
//   fcr_energy_density / fcr_stress / fcr_stress_derivative      constitutive.hpp:115-199
//   project_spd (eigen-clamp at 0, identity when nothing clamps)  constitutive.hpp:203-219
//   return_map (snow clamp, von Mises on Hencky strain)           constitutive.hpp:224-251
// Extensions the reference does not have, restated from the oracle
// (oracle/hot_oracle.hpp nh_*, return_map): Neo-Hookean psi / P / dP/dF, the snow map's plastic
// volume ratio (hardening), the Drucker-Prager return map.
#pragma once

#include <cstdint>

#include <math_constants.h>

namespace hotb200 {

constexpr int kSlots = 125;       // (2*2+1)^3 diagonal-storage slots, radius 2 (objective.hpp:329)
constexpr int kSlotPitch = 128;   // padded slot count per row component
constexpr int kDiagSlot = 62;     // centre slot
constexpr int kMaxMaterials = 16;

struct DevMaterial {
  double mu, lambda, xi;  // Lame parameters, stiffness scale (constitutive.hpp:255-258)
  double yield_stress, clamp_lo, clamp_hi;
  double hardening;       // snow: Stomakhin hardening xi (extension; 0 = the reference's clamp)
  double dp_alpha;        // Drucker-Prager friction coefficient (extension)
  int plasticity;         // 0 none, 1 von Mises, 2 snow clamp, 3 Drucker-Prager (extension)
  int elasticity;         // 0 fixed-corotated (the reference), 1 Neo-Hookean (extension)
};

struct DenseMap {
  int lo[3];
  int ext[3];
  const int* idx;  // node index or -1, row-major over ext (axis 0 slowest = lexicographic)
};

__device__ __forceinline__ long long dense_lin(const DenseMap& m, int x, int y, int z) {
  const int a = x - m.lo[0], b = y - m.lo[1], c = z - m.lo[2];
  if ((unsigned)a >= (unsigned)m.ext[0] || (unsigned)b >= (unsigned)m.ext[1] || (unsigned)c >= (unsigned)m.ext[2])
    return -1;
  return ((long long)a * m.ext[1] + b) * m.ext[2] + c;
}

__device__ __forceinline__ int dense_lookup(const DenseMap& m, int x, int y, int z) {
  const long long l = dense_lin(m, x, y, z);
  return l < 0 ? -1 : __ldg(m.idx + l);
}

// ------------------------------------------------------------------------------------
// Quadratic B-spline (grid.hpp:22-73).  Offsets are x/dx - node in cell units.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ double bspline_w(double x) {
  const double a = fabs(x);
  if (a < 0.5) return 0.75 - x * x;
  if (a < 1.5) {
    const double t = 1.5 - a;
    return 0.5 * t * t;
  }
  return 0.0;
}
__device__ __forceinline__ double bspline_dw(double x) {
  const double a = fabs(x);
  if (a < 0.5) return -2.0 * x;
  if (a < 1.5) return x > 0.0 ? a - 1.5 : 1.5 - a;
  return 0.0;
}

/// Stencil base (grid.hpp:78-89) from c = x / dx (true division, computed by the caller).
__device__ __forceinline__ int stencil_base_1d(double c) { return (int)floor(c + 0.5) - 1; }

/// Per-axis weights/derivatives for the 3 stencil nodes of one axis, plus the weight > 0 mask.
struct Axis3 {
  double w[3], dw[3];
};
__device__ __forceinline__ void axis_weights(double c, int base, Axis3& ax) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double off = c - (double)(base + k);
    ax.w[k] = bspline_w(off);
    ax.dw[k] = bspline_dw(off);
  }
}

/// dw/dx in place (the reference's kernel_gradient divides each 1D derivative by dx before the
/// products, grid.hpp:58-73): 3 divisions per axis instead of one per stencil node.
__device__ __forceinline__ void axis_dw_over_dx(Axis3& ax, double dx) {
#pragma unroll
  for (int k = 0; k < 3; ++k) ax.dw[k] = ax.dw[k] / dx;
}

// ------------------------------------------------------------------------------------
// 3x3 fp64 algebra, row-major m[i*3+j]
// ------------------------------------------------------------------------------------
struct M3 {
  double m[9];
};

__device__ __forceinline__ M3 m3_mul(const M3& A, const M3& B) {
  M3 C;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) C.m[i * 3 + j] = A.m[i * 3] * B.m[j] + A.m[i * 3 + 1] * B.m[3 + j] + A.m[i * 3 + 2] * B.m[6 + j];
  return C;
}
__device__ __forceinline__ M3 m3_mul_bt(const M3& A, const M3& B) {  // A * B^T
  M3 C;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      C.m[i * 3 + j] = A.m[i * 3] * B.m[j * 3] + A.m[i * 3 + 1] * B.m[j * 3 + 1] + A.m[i * 3 + 2] * B.m[j * 3 + 2];
  return C;
}
__device__ __forceinline__ double m3_det(const M3& A) {
  const double* m = A.m;
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[3] * (m[1] * m[8] - m[2] * m[7]) + m[6] * (m[1] * m[5] - m[2] * m[4]);
}
__device__ __forceinline__ M3 m3_cofactor(const M3& F) {  // constitutive.hpp:85-105
  const double* f = F.m;
  M3 A;
  A.m[0] = f[4] * f[8] - f[5] * f[7];
  A.m[1] = f[5] * f[6] - f[3] * f[8];
  A.m[2] = f[3] * f[7] - f[4] * f[6];
  A.m[3] = f[2] * f[7] - f[1] * f[8];
  A.m[4] = f[0] * f[8] - f[2] * f[6];
  A.m[5] = f[1] * f[6] - f[0] * f[7];
  A.m[6] = f[1] * f[5] - f[2] * f[4];
  A.m[7] = f[2] * f[3] - f[0] * f[5];
  A.m[8] = f[0] * f[4] - f[1] * f[3];
  return A;
}
__device__ __forceinline__ M3 m3_inverse(const M3& A, double* det_out) {
  const double* m = A.m;
  const double c00 = m[4] * m[8] - m[5] * m[7];
  const double c01 = m[5] * m[6] - m[3] * m[8];
  const double c02 = m[3] * m[7] - m[4] * m[6];
  const double det = m[0] * c00 + m[1] * c01 + m[2] * c02;
  *det_out = det;
  M3 r;
  r.m[0] = c00 / det;
  r.m[3] = c01 / det;
  r.m[6] = c02 / det;
  r.m[1] = (m[2] * m[7] - m[1] * m[8]) / det;
  r.m[4] = (m[0] * m[8] - m[2] * m[6]) / det;
  r.m[7] = (m[1] * m[6] - m[0] * m[7]) / det;
  r.m[2] = (m[1] * m[5] - m[2] * m[4]) / det;
  r.m[5] = (m[2] * m[3] - m[0] * m[5]) / det;
  r.m[8] = (m[0] * m[4] - m[1] * m[3]) / det;
  return r;
}

// ------------------------------------------------------------------------------------
// Sign-corrected SVD (constitutive.hpp:66-82): two-sided Jacobi on the scaled matrix,
// singular values sorted by magnitude descending, U and V proper rotations, inversion
// carried by the sign of sigma[2].
// ------------------------------------------------------------------------------------
struct Rot {
  double c, s;
};

template <int I>
struct IdxC {
  static constexpr int value = I;
};

// rows (p,q) of A <- J (x,y) = (c x + s y, -s x + c y)
template <int P, int Q>
__device__ __forceinline__ void rot_rows(double* A, Rot j) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double x = A[P * 3 + i], y = A[Q * 3 + i];
    A[P * 3 + i] = j.c * x + j.s * y;
    A[Q * 3 + i] = -j.s * x + j.c * y;
  }
}
// columns (p,q) of A rotated by J^T: (x,y) -> (c x - s y, s x + c y)
template <int P, int Q>
__device__ __forceinline__ void rot_cols(double* A, Rot j) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double x = A[i * 3 + P], y = A[i * 3 + Q];
    A[i * 3 + P] = j.c * x - j.s * y;
    A[i * 3 + Q] = j.s * x + j.c * y;
  }
}

template <int P, int Q>
__device__ __forceinline__ void jacobi_pair(double* W, double* U, double* V, double& max_diag) {
  const double threshold = fmax(2.2250738585072014e-308, 4.440892098500626e-16 * max_diag);
  const double wpq = W[P * 3 + Q], wqp = W[Q * 3 + P];
  if (!(fabs(wpq) > threshold || fabs(wqp) > threshold)) return;
  // 2x2 block [[a b][c d]] -> symmetrise with rot1, then diagonalise with a Jacobi rotation
  double a = W[P * 3 + P], b = wpq, c = wqp, d = W[Q * 3 + Q];
  Rot r1;
  const double t = a + d, dd = c - b;
  if (fabs(dd) < 2.2250738585072014e-308) {
    r1.c = 1.0;
    r1.s = 0.0;
  } else {
    const double u = t / dd;
    const double inv = rsqrt(1.0 + u * u);  // 1 / sqrt(1 + u^2): one reciprocal root for s and c
    r1.s = inv;
    r1.c = u * inv;
  }
  // m <- rot1 applied on the left
  const double a1 = r1.c * a + r1.s * c, b1 = r1.c * b + r1.s * d;
  const double d1 = -r1.s * b + r1.c * d;
  Rot jr;
  const double deno = 2.0 * fabs(b1);
  if (deno < 2.2250738585072014e-308) {
    jr.c = 1.0;
    jr.s = 0.0;
  } else {
    const double tau = (a1 - d1) / deno;
    const double w = sqrt(tau * tau + 1.0);
    const double tt = tau > 0.0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
    const double sign_t = tt > 0.0 ? 1.0 : -1.0;
    const double n = rsqrt(tt * tt + 1.0);
    jr.s = -sign_t * copysign(1.0, b1) * fabs(tt) * n;  // b1 / |b1| (b1 != 0 here)
    jr.c = n;
  }
  // j_left = rot1 * j_right^T
  Rot jl;
  jl.c = r1.c * jr.c + r1.s * jr.s;
  jl.s = -r1.c * jr.s + r1.s * jr.c;
  rot_rows<P, Q>(W, jl);
  // U <- U * j_left^T  (columns rotated by j_left)
  {
    Rot jt{jl.c, -jl.s};
    rot_cols<P, Q>(U, jt);
  }
  rot_cols<P, Q>(W, jr);
  rot_cols<P, Q>(V, jr);
  max_diag = fmax(max_diag, fmax(fabs(W[P * 3 + P]), fabs(W[Q * 3 + Q])));
}

__device__ __forceinline__ void svd3(const M3& F, M3& Uo, double s[3], M3& Vo) {
  double scale = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) scale = fmax(scale, fabs(F.m[i]));
  if (scale == 0.0) scale = 1.0;
  double W[9], U[9], V[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    W[i] = F.m[i] / scale;
    U[i] = (i % 4 == 0) ? 1.0 : 0.0;
    V[i] = U[i];
  }
  double max_diag = fmax(fabs(W[0]), fmax(fabs(W[4]), fabs(W[8])));
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double thr = fmax(2.2250738585072014e-308, 4.440892098500626e-16 * max_diag);
    const bool off = fabs(W[3]) > thr || fabs(W[1]) > thr || fabs(W[6]) > thr || fabs(W[2]) > thr ||
                     fabs(W[7]) > thr || fabs(W[5]) > thr;
    if (!off) break;
    jacobi_pair<1, 0>(W, U, V, max_diag);
    jacobi_pair<2, 0>(W, U, V, max_diag);
    jacobi_pair<2, 1>(W, U, V, max_diag);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double a = W[i * 4];
    s[i] = fabs(a);
    if (a < 0.0) {
      U[i] = -U[i];
      U[3 + i] = -U[3 + i];
      U[6 + i] = -U[6 + i];
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) s[i] *= scale;
  // selection sort, descending, first maximum wins (static indices: stays in registers)
  auto swap_cols = [&](auto X, auto Y) {
    constexpr int x = decltype(X)::value, y = decltype(Y)::value;
    const double ts = s[x];
    s[x] = s[y];
    s[y] = ts;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double t0 = U[r * 3 + x];
      U[r * 3 + x] = U[r * 3 + y];
      U[r * 3 + y] = t0;
      t0 = V[r * 3 + x];
      V[r * 3 + x] = V[r * 3 + y];
      V[r * 3 + y] = t0;
    }
  };
  {
    int pos = 0;
    double mx = s[0];
    if (s[1] > mx) {
      mx = s[1];
      pos = 1;
    }
    if (s[2] > mx) {
      mx = s[2];
      pos = 2;
    }
    if (mx != 0.0) {
      if (pos == 1) swap_cols(IdxC<0>{}, IdxC<1>{});
      if (pos == 2) swap_cols(IdxC<0>{}, IdxC<2>{});
      if (s[2] > s[1]) swap_cols(IdxC<1>{}, IdxC<2>{});  // max of s[1..2] is s[2] > 0 here
    }
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    Uo.m[i] = U[i];
    Vo.m[i] = V[i];
  }
  if (m3_det(Uo) < 0.0) {
    Uo.m[2] = -Uo.m[2];
    Uo.m[5] = -Uo.m[5];
    Uo.m[8] = -Uo.m[8];
    s[2] = -s[2];
  }
  if (m3_det(Vo) < 0.0) {
    Vo.m[2] = -Vo.m[2];
    Vo.m[5] = -Vo.m[5];
    Vo.m[8] = -Vo.m[8];
    s[2] = -s[2];
  }
}

__device__ __forceinline__ bool m3_finite(const M3& F) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 9; ++i) ok = ok && isfinite(F.m[i]);
  return ok;
}

/// psi (constitutive.hpp:115-123) from signed singular values.
__device__ __forceinline__ double fcr_psi(const double s[3], double mu, double la) {
  const double J = s[0] * s[1] * s[2];
  double e = (s[0] - 1.0) * (s[0] - 1.0);
  e += (s[1] - 1.0) * (s[1] - 1.0);
  e += (s[2] - 1.0) * (s[2] - 1.0);
  return mu * e + 0.5 * la * (J - 1.0) * (J - 1.0);
}

/// P (constitutive.hpp:126-133): 2 mu (F - U V^T) + lambda (det F - 1) cof(F)
__device__ __forceinline__ M3 fcr_P(const M3& F, const M3& U, const M3& V, double mu, double la) {
  const M3 R = m3_mul_bt(U, V);
  const double J = m3_det(F);
  const M3 cof = m3_cofactor(F);
  const double tmu = 2.0 * mu, lj = la * (J - 1.0);
  M3 P;
#pragma unroll
  for (int i = 0; i < 9; ++i) P.m[i] = tmu * (F.m[i] - R.m[i]) + lj * cof.m[i];
  return P;
}

/// Neo-Hookean psi = mu/2 (sum s^2 - 3) - mu log J + lambda/2 (log J)^2 (extension; +inf for
/// J <= 0, where the model is undefined: the line search backtracks).
__device__ __forceinline__ double nh_psi(const double s[3], double mu, double la) {
  const double J = s[0] * s[1] * s[2];
  if (!(J > 0.0)) return CUDART_INF;
  const double q = s[0] * s[0] + s[1] * s[1] + s[2] * s[2];
  const double lj = log(J);
  return 0.5 * mu * (q - 3.0) - mu * lj + 0.5 * la * lj * lj;
}

/// Neo-Hookean P = mu F + (lambda log J - mu) cof(F) / J (extension); NaN for J <= 0 (the
/// oracle throws domain_error there; a NaN gradient is reported the same way by the solve).
__device__ __forceinline__ M3 nh_P(const M3& F, double mu, double la) {
  const double J = m3_det(F);
  M3 P;
  if (!(J > 0.0)) {
#pragma unroll
    for (int i = 0; i < 9; ++i) P.m[i] = CUDART_NAN;
    return P;
  }
  const M3 cof = m3_cofactor(F);
  const double c = (la * log(J) - mu) / J;
#pragma unroll
  for (int i = 0; i < 9; ++i) P.m[i] = mu * F.m[i] + c * cof.m[i];
  return P;
}

/// The material's elastic energy density / first Piola stress (FCR: the reference's).
__device__ __forceinline__ double model_psi(const double s[3], double mu, double la, int elasticity) {
  return elasticity == 1 ? nh_psi(s, mu, la) : fcr_psi(s, mu, la);
}
__device__ __forceinline__ M3 model_P(const M3& F, const M3& U, const M3& V, double mu, double la, int elasticity) {
  return elasticity == 1 ? nh_P(F, mu, la) : fcr_P(F, U, V, mu, la);
}

/// Lame parameters of particle p's material with the snow hardening factor exp(xi (1 - J_p))
/// (extension; 1 -- and the material's own values, bit for bit -- without hardening).
__device__ __forceinline__ void particle_lame(const DevMaterial& m, const double* __restrict__ Jp, long long p,
                                              double& mu, double& la) {
  mu = m.mu;
  la = m.lambda;
  if (m.plasticity == 2 && m.hardening > 0.0) {
    const double h = exp(m.hardening * (1.0 - Jp[p]));
    mu *= h;
    la *= h;
  }
}

/// Symmetric 3x3 eigen-decomposition by cyclic Jacobi (for the diagonal-space block of
/// dP/dF).  A is overwritten with a diagonal; Q columns are eigenvectors.
__device__ __forceinline__ void sym3_eig(double A[3][3], double Q[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Q[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    const double dg = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
    if (off <= 1e-34 * dg || off < 1e-300) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double apq = A[p][q];
      if (fabs(apq) < 1e-300) continue;
      const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
      const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double akp = A[k][p], akq = A[k][q];
        A[k][p] = c * akp - s * akq;
        A[k][q] = s * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double apk = A[p][k], aqk = A[q][k];
        A[p][k] = c * apk - s * aqk;
        A[q][k] = s * apk + c * aqk;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double qkp = Q[k][p], qkq = Q[k][q];
        Q[k][p] = c * qkp - s * qkq;
        Q[k][q] = s * qkp + c * qkq;
      }
    }
  }
}

/// Projected, kappa-scaled dP/dF as the upper triangle (45 entries, row-major (r<=c)) of the
/// 9x9 tensor T[(ij),(kl)] (constitutive.hpp:138-199 + project_spd :203-219).
///
/// The projection is done in the diagonal space: with Q[(ij),(mn)] = U_im V_jn orthogonal,
/// eig(Q Mhat Q^T) = eig(Mhat) and Mhat is block diagonal (one 3x3 block on the (mm) indices,
/// three 2x2 blocks on the (mn),(nm) pairs), so clamping Mhat's eigenvalues and conjugating
/// back equals the reference's 9x9 eigen-clamp up to rounding.  When no eigenvalue is
/// negative the unclamped Mhat is used (the reference returns its input unchanged).
///
/// elasticity 1 (Neo-Hookean, extension) uses the same construction with its derivatives of
/// psi(sigma) (oracle nh_stress_derivative): psi_i = mu s_i + (lambda log J - mu) / s_i,
/// psi_ii = mu + (mu - lambda (log J - 1)) / s_i^2, psi_ij = lambda / (s_i s_j), and
/// (psi_i - psi_j) / (s_i - s_j) = mu + (mu - lambda log J) / (s_i s_j).
__device__ __forceinline__ void model_dpdf_projected(const M3& U, const double s[3], const M3& V, double mu,
                                                     double la, int elasticity, double kappa, bool project,
                                                     double Tu[45]) {
  const double J = s[0] * s[1] * s[2];
  const bool nh = elasticity == 1;
  const double lj = nh ? log(J) : 0.0;  // NaN for J <= 0: the record is poisoned like the oracle's throw
  const double Jp[3] = {s[1] * s[2], s[0] * s[2], s[0] * s[1]};
  double psi[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    psi[i] = nh ? mu * s[i] + (la * lj - mu) / s[i] : 2.0 * mu * (s[i] - 1.0) + la * (J - 1.0) * Jp[i];
  // 3x3 block on the (mm) indices
  double A[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double a;
      if (nh) {
        a = i == j ? mu + (mu - la * (lj - 1.0)) / (s[i] * s[i]) : la / (s[i] * s[j]);
      } else {
        a = la * Jp[i] * Jp[j];
        if (i == j)
          a += 2.0 * mu;
        else
          a += la * (J - 1.0) * s[3 - i - j];
      }
      A[i][j] = a;
    }
  // 2x2 blocks: pairs (0,1), (0,2), (1,2): diag value e1, off value e2
  double bdiag[3], boff[3];
  const int pi[3] = {0, 0, 1}, pj[3] = {1, 2, 2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int i = pi[k], j = pj[k];
    const double bd = nh ? mu + (mu - la * lj) / (s[i] * s[j]) : 2.0 * mu - la * (J - 1.0) * s[3 - i - j];
    double sum = s[i] + s[j];
    const double mag = fmax(fabs(sum), 1e-6);
    sum = sum >= 0.0 ? mag : -mag;
    const double bs = (psi[i] + psi[j]) / sum;
    bdiag[k] = 0.5 * (bd + bs);
    boff[k] = 0.5 * (bd - bs);
  }
  // eigen-clamp
  if (project) {
    // 2x2 [[d o][o d]]: eigenvalues d+o (vector (1,1)/sqrt2) and d-o (vector (1,-1)/sqrt2)
    bool neg = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) neg = neg || (bdiag[k] + boff[k] < 0.0) || (bdiag[k] - boff[k] < 0.0);
    double E[3][3], Qe[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) E[i][j] = A[i][j];
    sym3_eig(E, Qe);
    const bool neg3 = E[0][0] < 0.0 || E[1][1] < 0.0 || E[2][2] < 0.0;
    if (neg || neg3) {
      // the reference clamps the whole 9x9 spectrum when anything is negative
      const double l0 = fmax(E[0][0], 0.0), l1 = fmax(E[1][1], 0.0), l2 = fmax(E[2][2], 0.0);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) A[i][j] = Qe[i][0] * l0 * Qe[j][0] + Qe[i][1] * l1 * Qe[j][1] + Qe[i][2] * l2 * Qe[j][2];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i + 1; j < 3; ++j) {
          const double t = 0.5 * (A[i][j] + A[j][i]);
          A[i][j] = A[j][i] = t;
        }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double lp = fmax(bdiag[k] + boff[k], 0.0), lm = fmax(bdiag[k] - boff[k], 0.0);
        bdiag[k] = 0.5 * (lp + lm);
        boff[k] = 0.5 * (lp - lm);
      }
    }
  }
  // T = Q X Q^T with Q[(ij),(mn)] = U_im V_jn; X has the (mm,pp) block A and the 2x2 blocks.
  // Column vectors of Q: B_mn[(ij)] = U_im V_jn.
  // T = sum_{m,p} A_mp B_mm B_pp^T + sum_k [bdiag_k (B_ij B_ij^T + B_ji B_ji^T) + boff_k (B_ij B_ji^T + B_ji B_ij^T)]
  double Bmm[3][9];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Bmm[m][i * 3 + j] = U.m[i * 3 + m] * V.m[j * 3 + m];
  // G[m][(ij)] = sum_p A_mp B_pp[(ij)]
  double G[3][9];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int r = 0; r < 9; ++r) G[m][r] = A[m][0] * Bmm[0][r] + A[m][1] * Bmm[1][r] + A[m][2] * Bmm[2][r];
  int o = 0;
#pragma unroll
  for (int r = 0; r < 9; ++r)
#pragma unroll
    for (int c = r; c < 9; ++c) {
      double t = Bmm[0][r] * G[0][c] + Bmm[1][r] * G[1][c] + Bmm[2][r] * G[2][c];
      Tu[o++] = t;
    }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int m = pi[k], n = pj[k];
    double Bij[9], Bji[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        Bij[i * 3 + j] = U.m[i * 3 + m] * V.m[j * 3 + n];
        Bji[i * 3 + j] = U.m[i * 3 + n] * V.m[j * 3 + m];
      }
    const double dk = bdiag[k], ok = boff[k];
    int q = 0;
#pragma unroll
    for (int r = 0; r < 9; ++r)
#pragma unroll
      for (int c = r; c < 9; ++c) {
        Tu[q++] += dk * (Bij[r] * Bij[c] + Bji[r] * Bji[c]) + ok * (Bij[r] * Bji[c] + Bji[r] * Bij[c]);
      }
  }
#pragma unroll
  for (int q = 0; q < 45; ++q) Tu[q] *= kappa;
}

/// Index of (r, c), r <= c, in the 45-entry row-major upper triangle of a 9x9.
__host__ __device__ __forceinline__ int tri9(int r, int c) { return r * 9 - (r * (r - 1)) / 2 + (c - r); }

/// Plastic return map (constitutive.hpp:224-251).  Leaves F for von Mises on a non-positive
/// singular value, which the caller never reaches (update_strain skips inverted von Mises
/// particles, transfer.hpp:107-110).  Extensions: the snow map multiplies the plastic volume
/// ratio *Jp by det(F_trial) / det(F_clamped); Drucker-Prager (Klar et al. 2016) projects the
/// Hencky strain onto the friction cone (expansion: onto its tip, sigma = 1).
__device__ __forceinline__ void return_map(M3& F, const DevMaterial& m, double* Jp) {
  if (m.plasticity == 0) return;
  M3 U, V;
  double s[3];
  svd3(F, U, s, V);
  if (m.plasticity == 2) {
    const double Jt = s[0] * s[1] * s[2];
#pragma unroll
    for (int i = 0; i < 3; ++i) s[i] = fmin(fmax(s[i], m.clamp_lo), m.clamp_hi);
    *Jp *= Jt / (s[0] * s[1] * s[2]);
  } else if (m.plasticity == 3) {
    if (!(fmin(s[0], fmin(s[1], s[2])) > 0.0)) return;
    double eps[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) eps[i] = log(s[i]);
    const double tr = eps[0] + eps[1] + eps[2];
    if (tr >= 0.0) {
      s[0] = s[1] = s[2] = 1.0;
    } else {
      double dev[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) dev[i] = eps[i] - tr / 3.0;
      const double nd = sqrt(dev[0] * dev[0] + dev[1] * dev[1] + dev[2] * dev[2]);
      const double dgamma = nd + (3.0 * m.lambda + 2.0 * m.mu) / (2.0 * m.mu) * tr * m.dp_alpha;
      if (dgamma <= 0.0 || nd == 0.0) return;
#pragma unroll
      for (int i = 0; i < 3; ++i) s[i] = exp(eps[i] - dgamma * dev[i] / nd);
    }
  } else {
    if (!(fmin(s[0], fmin(s[1], s[2])) > 0.0)) return;
    double eps[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) eps[i] = log(s[i]);
    const double trace = eps[0] + eps[1] + eps[2];
    double dev[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) dev[i] = eps[i] - trace / 3.0;
    const double dev_stress = 2.0 * m.mu * sqrt(dev[0] * dev[0] + dev[1] * dev[1] + dev[2] * dev[2]);
    if (dev_stress <= m.yield_stress) return;
#pragma unroll
    for (int i = 0; i < 3; ++i) s[i] = exp(trace / 3.0 + dev[i] * (m.yield_stress / dev_stress));
  }
  // F = U diag(s) V^T
  M3 US;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) US.m[i * 3 + j] = U.m[i * 3 + j] * s[j];
  F = m3_mul_bt(US, V);
}

}  // namespace hotb200
