// Device math of the 2D (d = 2) HOT step: 2x2 matrices, the reference's Jacobi SVD convention,
// the constitutive models and return maps, the 4x4 SPD projection.  Every function restates the
// reference routine it cites (/root/reference/proj/include/hotmpm/*.hpp) for d = 2; the 3D path
// has its own specialised versions in hot_device.cuh.
#pragma once

#include <cuda_runtime.h>

#include <cfloat>

#include "hot_device.cuh"

namespace hotb200 {
namespace d2 {

/// Row-major 2x2 (the reference stores Eigen column-major; only the layout differs).
struct M2 {
  double a[4];
  __device__ double& operator()(int i, int j) { return a[2 * i + j]; }
  __device__ double operator()(int i, int j) const { return a[2 * i + j]; }
};

__device__ __forceinline__ M2 m2_identity() { return M2{{1.0, 0.0, 0.0, 1.0}}; }
__device__ __forceinline__ M2 m2_zero() { return M2{{0.0, 0.0, 0.0, 0.0}}; }
__device__ __forceinline__ M2 m2_mul(const M2& x, const M2& y) {
  M2 r;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) r(i, j) = x(i, 0) * y(0, j) + x(i, 1) * y(1, j);
  return r;
}
__device__ __forceinline__ M2 m2_t(const M2& x) { return M2{{x.a[0], x.a[2], x.a[1], x.a[3]}}; }
__device__ __forceinline__ double m2_det(const M2& m) { return m.a[0] * m.a[3] - m.a[1] * m.a[2]; }
__device__ __forceinline__ bool m2_finite(const M2& m) {
  return isfinite(m.a[0]) && isfinite(m.a[1]) && isfinite(m.a[2]) && isfinite(m.a[3]);
}
/// common.hpp inverse (2x2: adjugate / det).
__device__ __forceinline__ M2 m2_inv(const M2& m) {
  const double det = m2_det(m);
  return M2{{m.a[3] / det, -m.a[1] / det, -m.a[2] / det, m.a[0] / det}};
}
/// constitutive.hpp:85-105 (d = 2)
__device__ __forceinline__ M2 m2_cof(const M2& F) { return M2{{F.a[3], -F.a[2], -F.a[1], F.a[0]}}; }

// --------------------------------------------------------------------------- Jacobi SVD
// The reference's svd_rv (constitutive.hpp:66-82) wraps Eigen::JacobiSVD: two-sided Jacobi with
// Eigen's 2x2 real step and rotation conventions, singular values sorted descending, then the
// sign fix that makes U and V rotations (sigma_1 may turn negative).
struct Rot {
  double c, s;
};
__device__ __forceinline__ Rot rot_t(const Rot& j) { return Rot{j.c, -j.s}; }
__device__ __forceinline__ Rot rot_mul(const Rot& x, const Rot& o) {
  return Rot{x.c * o.c - x.s * o.s, x.c * o.s + x.s * o.c};
}
/// rows (p, q) <- J (x, y) = (c x + s y, -s x + c y)
__device__ __forceinline__ void rot_left(M2& m, int p, int q, const Rot& j) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double x = m(p, i), y = m(q, i);
    m(p, i) = j.c * x + j.s * y;
    m(q, i) = -j.s * x + j.c * y;
  }
}
/// columns (p, q) rotated with J^T (Eigen applyOnTheRight)
__device__ __forceinline__ void rot_right(M2& m, int p, int q, const Rot& j) {
  const Rot t = rot_t(j);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double x = m(i, p), y = m(i, q);
    m(i, p) = t.c * x + t.s * y;
    m(i, q) = -t.s * x + t.c * y;
  }
}
__device__ __forceinline__ Rot make_jacobi(double x, double y, double z) {
  Rot r{1.0, 0.0};
  const double deno = 2.0 * fabs(y);
  if (deno < DBL_MIN) return r;
  const double tau = (x - z) / deno;
  const double w = sqrt(tau * tau + 1.0);
  const double t = tau > 0.0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
  const double sign_t = t > 0.0 ? 1.0 : -1.0;
  const double n = 1.0 / sqrt(t * t + 1.0);
  r.s = -sign_t * (y / fabs(y)) * fabs(t) * n;
  r.c = n;
  return r;
}
__device__ __forceinline__ void jacobi_2x2_step(const M2& matrix, int p, int q, Rot& jl, Rot& jr) {
  M2 m;
  m(0, 0) = matrix(p, p);
  m(0, 1) = matrix(p, q);
  m(1, 0) = matrix(q, p);
  m(1, 1) = matrix(q, q);
  Rot rot1{1.0, 0.0};
  const double t = m(0, 0) + m(1, 1);
  const double dd = m(1, 0) - m(0, 1);
  if (!(fabs(dd) < DBL_MIN)) {
    const double u = t / dd;
    const double tmp = sqrt(1.0 + u * u);
    rot1.s = 1.0 / tmp;
    rot1.c = u / tmp;
  }
  rot_left(m, 0, 1, rot1);
  jr = make_jacobi(m(0, 0), m(0, 1), m(1, 1));
  jl = rot_mul(rot1, rot_t(jr));
}
/// svd_rv (constitutive.hpp:66-82): F = U diag(s) V^T with det U = det V = +1.
__device__ __noinline__ void svd2(const M2& A, M2& U, double (&s)[2], M2& V) {
  double scale = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) scale = fmax(scale, fabs(A.a[k]));
  if (scale == 0.0) scale = 1.0;
  M2 w;
#pragma unroll
  for (int k = 0; k < 4; ++k) w.a[k] = A.a[k] / scale;
  U = m2_identity();
  V = m2_identity();
  const double precision = 2.0 * DBL_EPSILON;
  double max_diag = fmax(fabs(w(0, 0)), fabs(w(1, 1)));
  bool finished = false;
  for (int sweep = 0; !finished && sweep < 100; ++sweep) {
    finished = true;
    const double threshold = fmax(DBL_MIN, precision * max_diag);
    if (fabs(w(1, 0)) > threshold || fabs(w(0, 1)) > threshold) {
      finished = false;
      Rot jl, jr;
      jacobi_2x2_step(w, 1, 0, jl, jr);
      rot_left(w, 1, 0, jl);
      rot_right(U, 1, 0, rot_t(jl));
      rot_right(w, 1, 0, jr);
      rot_right(V, 1, 0, jr);
      max_diag = fmax(max_diag, fmax(fabs(w(1, 1)), fabs(w(0, 0))));
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double a = w(i, i);
    s[i] = fabs(a);
    if (a < 0.0) {
      U(0, i) = -U(0, i);
      U(1, i) = -U(1, i);
    }
  }
  s[0] *= scale;
  s[1] *= scale;
  if (s[1] > s[0] && s[1] != 0.0) {  // sort descending, columns with them
    const double t = s[0];
    s[0] = s[1];
    s[1] = t;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      double x = U(r, 0);
      U(r, 0) = U(r, 1);
      U(r, 1) = x;
      x = V(r, 0);
      V(r, 0) = V(r, 1);
      V(r, 1) = x;
    }
  }
  if (m2_det(U) < 0.0) {
    U(0, 1) = -U(0, 1);
    U(1, 1) = -U(1, 1);
    s[1] = -s[1];
  }
  if (m2_det(V) < 0.0) {
    V(0, 1) = -V(0, 1);
    V(1, 1) = -V(1, 1);
    s[1] = -s[1];
  }
}

__device__ __forceinline__ M2 usvt(const M2& U, double s0, double s1, const M2& V) {
  M2 S{{s0, 0.0, 0.0, s1}};
  return m2_mul(m2_mul(U, S), m2_t(V));
}

// --------------------------------------------------------------------------- materials
/// Lame parameters of the particle (snow hardening factor exp(xi (1 - J_p)) when set; extension).
__device__ __forceinline__ void lame2(const DevMaterial& m, double jp, double& mu, double& la) {
  mu = m.mu;
  la = m.lambda;
  if (m.plasticity == 2 && m.hardening > 0.0) {
    const double h = exp(m.hardening * (1.0 - jp));
    if (h != 1.0) {
      mu *= h;
      la *= h;
    }
  }
}

/// constitutive.hpp:115-123 (FCR) / the Neo-Hookean extension: psi(F).
__device__ __noinline__ double psi2(const M2& F, double mu, double la, int elasticity) {
  M2 U, V;
  double s[2];
  svd2(F, U, s, V);
  const double J = s[0] * s[1];
  if (elasticity == 1) {
    if (!(J > 0.0)) return CUDART_INF;
    const double lj = log(J);
    return 0.5 * mu * ((s[0] * s[0] + s[1] * s[1]) - 2.0) - mu * lj + 0.5 * la * lj * lj;
  }
  const double e = (s[0] - 1.0) * (s[0] - 1.0) + (s[1] - 1.0) * (s[1] - 1.0);
  return mu * e + 0.5 * la * (J - 1.0) * (J - 1.0);
}

/// constitutive.hpp:126-133 (FCR) / Neo-Hookean: P(F); NaN for NH at J <= 0 (the oracle throws).
__device__ __noinline__ M2 stress2(const M2& F, double mu, double la, int elasticity) {
  M2 P;
  const double J = m2_det(F);
  const M2 cf = m2_cof(F);
  if (elasticity == 1) {
    const double c = (la * log(J) - mu) / J;
#pragma unroll
    for (int k = 0; k < 4; ++k) P.a[k] = mu * F.a[k] + c * cf.a[k];
    return P;
  }
  M2 U, V;
  double s[2];
  svd2(F, U, s, V);
  const M2 R = m2_mul(U, m2_t(V));
  const double c = la * (J - 1.0);
#pragma unroll
  for (int k = 0; k < 4; ++k) P.a[k] = (2.0 * mu) * (F.a[k] - R.a[k]) + c * cf.a[k];
  return P;
}

/// constitutive.hpp:138-199 (d = 2) and its Neo-Hookean analogue: dP/dF as a symmetrised 4x4,
/// row-major over (ij),(kl).
__device__ __noinline__ void dpdf2(const M2& F, double mu, double la, int elasticity, double (&out)[16]) {
  M2 U, V;
  double s[2];
  svd2(F, U, s, V);
  const double J = s[0] * s[1];
  double Mh[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) Mh[k] = 0.0;
  double bd, psi0, psi1;
  if (elasticity == 1) {
    const double lj = log(J);
    psi0 = mu * s[0] + (la * lj - mu) / s[0];
    psi1 = mu * s[1] + (la * lj - mu) / s[1];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        Mh[(3 * i) * 4 + 3 * j] = i == j ? mu + (mu - la * (lj - 1.0)) / (s[i] * s[i]) : la / (s[i] * s[j]);
    bd = mu + (mu - la * lj) / (s[0] * s[1]);
  } else {
    const double Jp[2] = {s[1], s[0]};
    psi0 = 2.0 * mu * (s[0] - 1.0) + la * (J - 1.0) * Jp[0];
    psi1 = 2.0 * mu * (s[1] - 1.0) + la * (J - 1.0) * Jp[1];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double a = la * Jp[i] * Jp[j];
        if (i == j)
          a += 2.0 * mu;
        else
          a += la * (J - 1.0);
        Mh[(3 * i) * 4 + 3 * j] = a;
      }
    bd = 2.0 * mu - la * (J - 1.0);
  }
  double sum = s[0] + s[1];
  const double mag = fmax(fabs(sum), 1e-6);
  sum = sum >= 0.0 ? mag : -mag;
  const double bs = (psi0 + psi1) / sum;
  Mh[1 * 4 + 1] = Mh[2 * 4 + 2] = 0.5 * (bd + bs);
  Mh[1 * 4 + 2] = Mh[2 * 4 + 1] = 0.5 * (bd - bs);
  double Q[16];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int l = 0; l < 2; ++l) Q[(2 * i + j) * 4 + 2 * k + l] = U(i, k) * V(j, l);
  double QM[16];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc += Q[r * 4 + k] * Mh[k * 4 + c];
      QM[r * 4 + c] = acc;
    }
  double o[16];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc += QM[r * 4 + k] * Q[c * 4 + k];
      o[r * 4 + c] = acc;
    }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) out[r * 4 + c] = 0.5 * (o[r * 4 + c] + o[c * 4 + r]);
}

/// constitutive.hpp:203-219 for the 4x4 dP/dF: cyclic Jacobi eigen-decomposition (standing in for
/// Eigen::SelfAdjointEigenSolver), negative eigenvalues clamped to zero, rebuilt and symmetrised;
/// unchanged when nothing is clamped.  Returns false on asymmetric input (the reference throws).
__device__ __noinline__ bool project_spd4(double (&A)[16]) {
  double mx = 0.0, asym = 0.0;
#pragma unroll 1
  for (int i = 0; i < 4; ++i)
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      mx = fmax(mx, fabs(A[i * 4 + j]));
      asym = fmax(asym, fabs(A[i * 4 + j] - A[j * 4 + i]));
    }
  if (asym > 1e-12 * fmax(1.0, mx)) return false;
  double W[16], Vv[16];
#pragma unroll 1
  for (int k = 0; k < 16; ++k) {
    W[k] = A[k];
    Vv[k] = (k % 5 == 0) ? 1.0 : 0.0;
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
#pragma unroll 1
    for (int p = 0; p < 4; ++p)
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        if (p == q)
          diag += W[p * 4 + q] * W[p * 4 + q];
        else
          off += W[p * 4 + q] * W[p * 4 + q];
      }
    if (off <= 1e-34 * diag || off < 1e-300) break;
#pragma unroll 1
    for (int p = 0; p < 3; ++p)
#pragma unroll 1
      for (int q = p + 1; q < 4; ++q) {
        const double apq = W[p * 4 + q];
        if (fabs(apq) < 1e-300) continue;
        const double app = W[p * 4 + p], aqq = W[q * 4 + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          const double akp = W[k * 4 + p], akq = W[k * 4 + q];
          W[k * 4 + p] = c * akp - s * akq;
          W[k * 4 + q] = s * akp + c * akq;
        }
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          const double apk = W[p * 4 + k], aqk = W[q * 4 + k];
          W[p * 4 + k] = c * apk - s * aqk;
          W[q * 4 + k] = s * apk + c * aqk;
        }
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          const double vkp = Vv[k * 4 + p], vkq = Vv[k * 4 + q];
          Vv[k * 4 + p] = c * vkp - s * vkq;
          Vv[k * 4 + q] = s * vkp + c * vkq;
        }
      }
  }
  double ev[4];
  bool changed = false;
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    ev[i] = W[i * 4 + i];
    if (ev[i] < 0.0) {
      ev[i] = 0.0;
      changed = true;
    }
  }
  if (!changed) return true;
  double B[16];
#pragma unroll 1
  for (int i = 0; i < 4; ++i)
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      double acc = 0.0;
#pragma unroll 1
      for (int k = 0; k < 4; ++k) acc += Vv[i * 4 + k] * ev[k] * Vv[j * 4 + k];
      B[i * 4 + j] = acc;
    }
#pragma unroll 1
  for (int i = 0; i < 4; ++i)
#pragma unroll 1
    for (int j = 0; j < 4; ++j) A[i * 4 + j] = 0.5 * (B[i * 4 + j] + B[j * 4 + i]);
  return true;
}

/// constitutive.hpp:224-251 (d = 2): von Mises, snow clamp (with the J_p update of the hardening
/// extension) and the Drucker-Prager extension.  The caller skips the Hencky maps for det F <= 0.
__device__ __noinline__ M2 return_map2(const M2& Ft, const DevMaterial& m, double* jp) {
  if (m.plasticity == 0) return Ft;
  M2 U, V;
  double s[2];
  svd2(Ft, U, s, V);
  if (m.plasticity == 2) {
    const double Jt = s[0] * s[1];
    const double c0 = fmin(fmax(s[0], m.clamp_lo), m.clamp_hi), c1 = fmin(fmax(s[1], m.clamp_lo), m.clamp_hi);
    if (jp) *jp *= Jt / (c0 * c1);
    return usvt(U, c0, c1, V);
  }
  const double e0 = log(s[0]), e1 = log(s[1]);
  if (m.plasticity == 3) {
    const double tr = e0 + e1;
    if (tr >= 0.0) return usvt(U, 1.0, 1.0, V);
    const double d0 = e0 - tr / 2, d1 = e1 - tr / 2;
    const double nd = sqrt(d0 * d0 + d1 * d1);
    const double dgamma = nd + (2 * m.lambda + 2.0 * m.mu) / (2.0 * m.mu) * tr * m.dp_alpha;
    if (dgamma <= 0.0 || nd == 0.0) return Ft;
    return usvt(U, exp(e0 - dgamma * d0 / nd), exp(e1 - dgamma * d1 / nd), V);
  }
  // von Mises
  const double trace = e0 + e1;
  double d0 = e0 - trace / 2, d1 = e1 - trace / 2;
  const double dev_stress = 2.0 * m.mu * sqrt(d0 * d0 + d1 * d1);
  if (dev_stress <= m.yield_stress) return Ft;
  d0 *= m.yield_stress / dev_stress;
  d1 *= m.yield_stress / dev_stress;
  return usvt(U, exp(trace / 2 + d0), exp(trace / 2 + d1), V);
}

// --------------------------------------------------------------------------- B-spline (grid.hpp)
__device__ __forceinline__ double bw1(double x) {  // grid.hpp:22-34
  const double a = fabs(x);
  if (a < 0.5) return 0.75 - x * x;
  if (a < 1.5) {
    const double t = 1.5 - a;
    return 0.5 * t * t;
  }
  return 0.0;
}
__device__ __forceinline__ double bdw1(double x) {  // grid.hpp:36-46
  const double a = fabs(x);
  if (a < 0.5) return -2.0 * x;
  if (a < 1.5) return x > 0.0 ? a - 1.5 : 1.5 - a;
  return 0.0;
}
/// The particle's 3x3 stencil (grid.hpp:49-100): base node, per-axis offsets x/dx - node.
__device__ __forceinline__ void stencil2(double x0, double x1, double dx, int& b0, int& b1) {
  b0 = (int)floor(x0 / dx + 0.5) - 1;
  b1 = (int)floor(x1 / dx + 0.5) - 1;
}
/// weight and gradient at node (n0, n1) (grid.hpp:49-73: offsets x/dx - node evaluated per axis)
__device__ __forceinline__ double wgrad2(double x0, double x1, double dx, int n0, int n1, double& g0, double& g1) {
  const double o0 = x0 / dx - (double)n0, o1 = x1 / dx - (double)n1;
  const double w0 = bw1(o0), w1 = bw1(o1);
  g0 = bdw1(o0) / dx * w1;
  g1 = bdw1(o1) / dx * w0;
  return w0 * w1;
}

}  // namespace d2
}  // namespace hotb200
