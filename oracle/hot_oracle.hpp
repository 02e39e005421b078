// TEST INFRASTRUCTURE ONLY — the CPU parity oracle ("port") for the HOT implicit-MPM step.
//
// This header is a plain C++20 restatement (no Eigen) of the reference solver under
// /root/reference/proj/include/hotmpm/*.hpp.  The reference itself cannot be built here
// (Eigen3, doctest and CLI11 are absent), so this file is the
// checker that the CUDA product path is compared against.  Only tests/, bench.py's
// cpu_baseline / --impl reference leg and __graft_entry__.smoke() may load it; the product
// library never links or calls it.
//
// Every function cites the reference file:line it restates.  Serial accumulation orders,
// the parallel_for regions and the default thread count (1) are preserved.  Eigen's
// JacobiSVD (constitutive.hpp:68) and SelfAdjointEigenSolver (constitutive.hpp:208) are
// restated as two-sided / cyclic Jacobi; bitwise agreement with Eigen is "parity
// unpinned" and the restatement is pinned to the reference's own FD /
// property tolerances by tests/test_oracle_*.py.
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <deque>
#include <functional>
#include <limits>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

namespace hot_oracle {

// ---------------------------------------------------------------------------------------
// common.hpp
// ---------------------------------------------------------------------------------------

using VecX = std::vector<double>;

constexpr int ipow(int base, int exp) {  // common.hpp:23-27
  int r = 1;
  while (exp-- > 0) r *= base;
  return r;
}

template <int d>
struct Vec {
  std::array<double, d> a{};
  double& operator[](int i) { return a[i]; }
  double operator[](int i) const { return a[i]; }
  static Vec zero() { return Vec{}; }
};

template <int d>
struct Mat {
  std::array<double, d * d> a{};  // row-major storage
  double& operator()(int i, int j) { return a[i * d + j]; }
  double operator()(int i, int j) const { return a[i * d + j]; }
  static Mat zero() { return Mat{}; }
  static Mat identity() {
    Mat m;
    for (int i = 0; i < d; ++i) m(i, i) = 1.0;
    return m;
  }
};

template <int d>
inline Vec<d> operator+(const Vec<d>& x, const Vec<d>& y) {
  Vec<d> r;
  for (int i = 0; i < d; ++i) r[i] = x[i] + y[i];
  return r;
}
template <int d>
inline Vec<d> operator-(const Vec<d>& x, const Vec<d>& y) {
  Vec<d> r;
  for (int i = 0; i < d; ++i) r[i] = x[i] - y[i];
  return r;
}
template <int d>
inline Vec<d> operator*(double s, const Vec<d>& x) {
  Vec<d> r;
  for (int i = 0; i < d; ++i) r[i] = s * x[i];
  return r;
}
template <int d>
inline double dot(const Vec<d>& x, const Vec<d>& y) {
  double s = x[0] * y[0];
  for (int i = 1; i < d; ++i) s += x[i] * y[i];
  return s;
}
template <int d>
inline double squared_norm(const Vec<d>& x) { return dot(x, x); }
template <int d>
inline double norm(const Vec<d>& x) { return std::sqrt(squared_norm(x)); }
template <int d>
inline bool all_finite(const Vec<d>& x) {
  for (int i = 0; i < d; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

template <int d>
inline Mat<d> operator+(const Mat<d>& x, const Mat<d>& y) {
  Mat<d> r;
  for (int i = 0; i < d * d; ++i) r.a[i] = x.a[i] + y.a[i];
  return r;
}
template <int d>
inline Mat<d> operator-(const Mat<d>& x, const Mat<d>& y) {
  Mat<d> r;
  for (int i = 0; i < d * d; ++i) r.a[i] = x.a[i] - y.a[i];
  return r;
}
template <int d>
inline Mat<d> operator*(double s, const Mat<d>& x) {
  Mat<d> r;
  for (int i = 0; i < d * d; ++i) r.a[i] = s * x.a[i];
  return r;
}
template <int d>
inline Mat<d> operator*(const Mat<d>& x, const Mat<d>& y) {
  Mat<d> r;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double s = x(i, 0) * y(0, j);
      for (int k = 1; k < d; ++k) s += x(i, k) * y(k, j);
      r(i, j) = s;
    }
  return r;
}
template <int d>
inline Vec<d> operator*(const Mat<d>& x, const Vec<d>& v) {
  Vec<d> r;
  for (int i = 0; i < d; ++i) {
    double s = x(i, 0) * v[0];
    for (int k = 1; k < d; ++k) s += x(i, k) * v[k];
    r[i] = s;
  }
  return r;
}
template <int d>
inline Mat<d> transpose(const Mat<d>& x) {
  Mat<d> r;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) r(i, j) = x(j, i);
  return r;
}
template <int d>
inline Mat<d> outer(const Vec<d>& u, const Vec<d>& v) {
  Mat<d> r;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) r(i, j) = u[i] * v[j];
  return r;
}
template <int d>
inline bool all_finite(const Mat<d>& x) {
  for (double v : x.a)
    if (!std::isfinite(v)) return false;
  return true;
}
template <int d>
inline double determinant(const Mat<d>& m) {
  if constexpr (d == 2) {
    return m(0, 0) * m(1, 1) - m(0, 1) * m(1, 0);
  } else {
    return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) -
           m(1, 0) * (m(0, 1) * m(2, 2) - m(0, 2) * m(2, 1)) +
           m(2, 0) * (m(0, 1) * m(1, 2) - m(0, 2) * m(1, 1));
  }
}
template <int d>
inline Mat<d> inverse(const Mat<d>& m) {
  Mat<d> r;
  if constexpr (d == 2) {
    const double det = determinant(m);
    r(0, 0) = m(1, 1) / det;
    r(0, 1) = -m(0, 1) / det;
    r(1, 0) = -m(1, 0) / det;
    r(1, 1) = m(0, 0) / det;
  } else {
    // adjugate / det
    const double c00 = m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1);
    const double c01 = m(1, 2) * m(2, 0) - m(1, 0) * m(2, 2);
    const double c02 = m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0);
    const double det = m(0, 0) * c00 + m(0, 1) * c01 + m(0, 2) * c02;
    r(0, 0) = c00 / det;
    r(1, 0) = c01 / det;
    r(2, 0) = c02 / det;
    r(0, 1) = (m(0, 2) * m(2, 1) - m(0, 1) * m(2, 2)) / det;
    r(1, 1) = (m(0, 0) * m(2, 2) - m(0, 2) * m(2, 0)) / det;
    r(2, 1) = (m(0, 1) * m(2, 0) - m(0, 0) * m(2, 1)) / det;
    r(0, 2) = (m(0, 1) * m(1, 2) - m(0, 2) * m(1, 1)) / det;
    r(1, 2) = (m(0, 2) * m(1, 0) - m(0, 0) * m(1, 2)) / det;
    r(2, 2) = (m(0, 0) * m(1, 1) - m(0, 1) * m(1, 0)) / det;
  }
  return r;
}

template <int d>
inline Vec<d> seg(const VecX& x, int i) {
  Vec<d> r;
  for (int a = 0; a < d; ++a) r[a] = x[static_cast<std::size_t>(d) * i + a];
  return r;
}
template <int d>
inline void set_seg(VecX& x, int i, const Vec<d>& v) {
  for (int a = 0; a < d; ++a) x[static_cast<std::size_t>(d) * i + a] = v[a];
}
template <int d>
inline void add_seg(VecX& x, int i, const Vec<d>& v) {
  for (int a = 0; a < d; ++a) x[static_cast<std::size_t>(d) * i + a] += v[a];
}

inline double vdot(const VecX& x, const VecX& y) {
  double s = 0;
  for (std::size_t i = 0; i < x.size(); ++i) s += x[i] * y[i];
  return s;
}
inline double vnorm(const VecX& x) { return std::sqrt(vdot(x, x)); }
inline bool vfinite(const VecX& x) {
  for (double v : x)
    if (!std::isfinite(v)) return false;
  return true;
}

/// Lattice coordinate, lexicographic order (common.hpp:31-60).
template <int d>
struct Coord {
  std::array<int, d> v{};
  int operator[](int a) const { return v[a]; }
  int& operator[](int a) { return v[a]; }
  friend bool operator==(const Coord& x, const Coord& y) { return x.v == y.v; }
  friend bool operator!=(const Coord& x, const Coord& y) { return x.v != y.v; }
  friend bool operator<(const Coord& x, const Coord& y) { return x.v < y.v; }
  friend Coord operator+(const Coord& x, const Coord& y) {
    Coord r;
    for (int i = 0; i < d; ++i) r.v[i] = x.v[i] + y.v[i];
    return r;
  }
  friend Coord operator-(const Coord& x, const Coord& y) {
    Coord r;
    for (int i = 0; i < d; ++i) r.v[i] = x.v[i] - y.v[i];
    return r;
  }
  Vec<d> cast() const {
    Vec<d> r;
    for (int i = 0; i < d; ++i) r[i] = static_cast<double>(v[i]);
    return r;
  }
};

/// LatticeHash (common.hpp:62-74).
template <int d>
struct CoordHash {
  std::size_t operator()(const Coord<d>& c) const {
    std::uint64_t h = 0x9e3779b97f4a7c15ull;
    for (int i = 0; i < d; ++i) {
      std::uint64_t x = static_cast<std::uint64_t>(static_cast<std::int64_t>(c.v[i]));
      x *= 0xbf58476d1ce4e5b9ull;
      x ^= x >> 31;
      h = (h ^ x) * 0x94d049bb133111ebull;
    }
    return static_cast<std::size_t>(h ^ (h >> 29));
  }
};

template <int d>
using CoordIndex = std::unordered_map<Coord<d>, int, CoordHash<d>>;

inline int& detail_thread_count() {  // common.hpp:76-83 (default 1 thread)
  static int n = 1;
  return n;
}
inline int thread_count() { return detail_thread_count(); }
inline void set_thread_count(int n) { detail_thread_count() = n < 1 ? 1 : n; }

/// common.hpp:87-104: serial when nt<=1 || n<1024, else std::thread fan-out.
template <typename F>
void parallel_for(std::int64_t n, F&& body) {
  const int nt = thread_count();
  if (nt <= 1 || n < 1024) {
    for (std::int64_t i = 0; i < n; ++i) body(i);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(nt);
  for (int t = 0; t < nt; ++t) {
    const std::int64_t lo = n * t / nt;
    const std::int64_t hi = n * (t + 1) / nt;
    pool.emplace_back([lo, hi, &body] {
      for (std::int64_t i = lo; i < hi; ++i) body(i);
    });
  }
  for (auto& th : pool) th.join();
}

struct SolverFailure : std::runtime_error {  // common.hpp:124-126
  explicit SolverFailure(const std::string& msg) : std::runtime_error(msg) {}
};

// ---------------------------------------------------------------------------------------
// grid.hpp
// ---------------------------------------------------------------------------------------

enum class KernelKind { QuadraticBSpline = 0, Linear = 1 };

constexpr int kernel_stencil_width(KernelKind kind) { return kind == KernelKind::Linear ? 2 : 3; }

/// grid.hpp:22-34
inline double kernel_weight_1d(KernelKind kind, double x) {
  const double a = std::abs(x);
  if (kind == KernelKind::Linear) return a < 1.0 ? 1.0 - a : 0.0;
  if (a < 0.5) return 0.75 - x * x;
  if (a < 1.5) {
    const double t = 1.5 - a;
    return 0.5 * t * t;
  }
  return 0.0;
}

/// grid.hpp:36-46
inline double kernel_derivative_1d(KernelKind kind, double x) {
  const double a = std::abs(x);
  if (kind == KernelKind::Linear) {
    if (a >= 1.0 || x == 0.0) return 0.0;
    return x > 0.0 ? -1.0 : 1.0;
  }
  if (a < 0.5) return -2.0 * x;
  if (a < 1.5) return x > 0.0 ? a - 1.5 : 1.5 - a;
  return 0.0;
}

/// grid.hpp:49-54
template <int d>
double kernel_weight(KernelKind kind, const Vec<d>& off) {
  double w = 1.0;
  for (int a = 0; a < d; ++a) w *= kernel_weight_1d(kind, off[a]);
  return w;
}

/// grid.hpp:58-73
template <int d>
Vec<d> kernel_gradient(KernelKind kind, const Vec<d>& off, double dx) {
  Vec<d> w1, g1;
  for (int a = 0; a < d; ++a) {
    w1[a] = kernel_weight_1d(kind, off[a]);
    g1[a] = kernel_derivative_1d(kind, off[a]);
  }
  Vec<d> grad;
  for (int a = 0; a < d; ++a) {
    double v = g1[a] / dx;
    for (int b = 0; b < d; ++b)
      if (b != a) v *= w1[b];
    grad[a] = v;
  }
  return grad;
}

/// grid.hpp:78-89 (true division x/dx)
template <int d>
Coord<d> stencil_base(const Vec<d>& x, double dx, KernelKind kind) {
  Coord<d> base;
  for (int a = 0; a < d; ++a) {
    const double c = x[a] / dx;
    if (kind == KernelKind::QuadraticBSpline)
      base[a] = static_cast<int>(std::floor(c + 0.5)) - 1;
    else
      base[a] = static_cast<int>(std::floor(c));
  }
  return base;
}

/// grid.hpp:92-100 (lexicographic offsets, last axis fastest)
template <int d>
Coord<d> stencil_offset(int flat, int width) {
  Coord<d> off;
  for (int a = d - 1; a >= 0; --a) {
    off[a] = flat % width;
    flat /= width;
  }
  return off;
}

/// x / dx - node, evaluated as the reference does (grid.hpp:150, transfer.hpp:35).
template <int d>
inline Vec<d> node_offset(const Vec<d>& x, double dx, const Coord<d>& node) {
  Vec<d> r;
  for (int a = 0; a < d; ++a) r[a] = x[a] / dx - static_cast<double>(node[a]);
  return r;
}

/// grid.hpp:104-133
template <int d>
struct SparseGrid {
  double dx = 1.0;
  KernelKind kind = KernelKind::QuadraticBSpline;
  std::vector<Coord<d>> coords;
  CoordIndex<d> index;
  VecX mass, velocity, momentum;
  std::vector<std::uint8_t> dirichlet;
  VecX bc_velocity;

  int node_count() const { return static_cast<int>(coords.size()); }
  int find(const Coord<d>& c) const {
    auto it = index.find(c);
    return it == index.end() ? -1 : it->second;
  }
  Vec<d> node_position(int i) const { return dx * coords[i].cast(); }
  void allocate_fields() {
    const int n = node_count();
    mass.assign(n, 0.0);
    velocity.assign(static_cast<std::size_t>(n) * d, 0.0);
    momentum.assign(static_cast<std::size_t>(n) * d, 0.0);
    dirichlet.assign(n, 0);
    bc_velocity.assign(static_cast<std::size_t>(n) * d, 0.0);
  }
};

/// grid.hpp:137-165
template <int d>
SparseGrid<d> activate_grid(std::span<const Vec<d>> positions, double dx, KernelKind kind) {
  if (!(dx > 0.0)) throw std::invalid_argument("activate_grid: dx must be positive");
  const int width = kernel_stencil_width(kind);
  const int count = ipow(width, d);
  std::vector<Coord<d>> found;
  found.reserve(positions.size() * count);
  for (const auto& x : positions) {
    if (!all_finite(x)) throw std::invalid_argument("activate_grid: non-finite particle position");
    const Coord<d> base = stencil_base(x, dx, kind);
    for (int k = 0; k < count; ++k) {
      const Coord<d> node = base + stencil_offset<d>(k, width);
      if (kernel_weight<d>(kind, node_offset(x, dx, node)) > 0.0) found.push_back(node);
    }
  }
  std::sort(found.begin(), found.end());
  found.erase(std::unique(found.begin(), found.end()), found.end());
  SparseGrid<d> grid;
  grid.dx = dx;
  grid.kind = kind;
  grid.coords = std::move(found);
  grid.index.reserve(grid.coords.size());
  for (int i = 0; i < grid.node_count(); ++i) grid.index.emplace(grid.coords[i], i);
  grid.allocate_fields();
  return grid;
}

/// grid.hpp:168-173
inline double cfl_dt(double v_max, double dx, double fps) {
  const double frame = 1.0 / fps;
  if (v_max <= 0.0) return frame;
  return std::min(frame, 0.6 * dx / v_max);
}

// ---------------------------------------------------------------------------------------
// constitutive.hpp
// ---------------------------------------------------------------------------------------

enum class PlasticityKind { None = 0, VonMises = 1, SnowClamp = 2, DruckerPrager = 3 };
/// Elastic energy of a material.  The reference has fixed-corotated only (objective.hpp:244,
/// 268,297 call fcr_* unconditionally); Neo-Hookean is an extension BASELINE configs 2 and 5
/// name, parity-unpinned against the reference and pinned here by FD tests.
enum class ElasticityKind { FixedCorotated = 0, NeoHookean = 1 };

/// constitutive.hpp:12-52
struct Material {
  double density = 0, youngs = 0, poisson = 0, mu = 0, lambda = 0;
  PlasticityKind plasticity = PlasticityKind::None;
  double yield_stress = 0;
  double clamp_lo = 1, clamp_hi = 1;
  // extensions (not in the reference): elastic model, snow hardening
  // coefficient xi (Stomakhin et al. 2013: mu, lambda scaled by exp(xi (1 - J_p))), and the
  // Drucker-Prager friction coefficient alpha = sqrt(2/3) 2 sin(phi) / (3 - sin(phi)) (Klar et
  // al. 2016) from the friction angle phi
  ElasticityKind elasticity = ElasticityKind::FixedCorotated;
  double hardening = 0;
  double friction_angle = 0, dp_alpha = 0;

  static Material elastic(double density, double youngs, double poisson) {
    if (!(youngs > 0.0)) throw std::invalid_argument("material: Young's modulus must be positive");
    if (!(poisson >= 0.0 && poisson < 0.5))
      throw std::invalid_argument("material: Poisson ratio must lie in [0, 0.5)");
    Material m;
    m.density = density;
    m.youngs = youngs;
    m.poisson = poisson;
    m.mu = youngs / (2.0 * (1.0 + poisson));
    m.lambda = youngs * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson));
    return m;
  }
  static Material von_mises(double density, double youngs, double poisson, double yield) {
    Material m = elastic(density, youngs, poisson);
    if (!(yield > 0.0)) throw std::invalid_argument("material: yield stress must be positive");
    m.plasticity = PlasticityKind::VonMises;
    m.yield_stress = yield;
    return m;
  }
  static Material snow(double density, double youngs, double poisson, double lo, double hi) {
    Material m = elastic(density, youngs, poisson);
    if (!(lo <= 1.0 && 1.0 <= hi)) throw std::invalid_argument("material: snow clamp must bracket 1");
    m.plasticity = PlasticityKind::SnowClamp;
    m.clamp_lo = lo;
    m.clamp_hi = hi;
    return m;
  }
  /// Drucker-Prager sand (extension): friction angle in degrees, in [0, 90).
  static Material drucker_prager(double density, double youngs, double poisson, double friction_deg) {
    Material m = elastic(density, youngs, poisson);
    if (!(friction_deg >= 0.0 && friction_deg < 90.0))
      throw std::invalid_argument("material: friction angle must lie in [0, 90) degrees");
    m.plasticity = PlasticityKind::DruckerPrager;
    m.friction_angle = friction_deg;
    const double sp = std::sin(friction_deg * 3.14159265358979323846 / 180.0);
    m.dp_alpha = std::sqrt(2.0 / 3.0) * 2.0 * sp / (3.0 - sp);
    return m;
  }
  /// The extension fields on top of a reference material.
  Material& with_elasticity(ElasticityKind e) {
    elasticity = e;
    return *this;
  }
  Material& with_hardening(double xi) {
    if (!(xi >= 0.0)) throw std::invalid_argument("material: hardening must be non-negative");
    hardening = xi;
    return *this;
  }
  /// Lame parameters scaled by the snow hardening factor h (h == 1: this material, unchanged).
  Material hardened(double h) const {
    Material m = *this;
    m.mu *= h;
    m.lambda *= h;
    return m;
  }
  /// exp(xi (1 - J_p)) for snow with hardening, else 1 (Stomakhin et al. 2013, eq. 9).
  double hardening_factor(double Jp) const {
    return (plasticity == PlasticityKind::SnowClamp && hardening > 0.0) ? std::exp(hardening * (1.0 - Jp)) : 1.0;
  }
};

/// d^2 x d^2 row-major stress derivative (constitutive.hpp:56-57).
template <int d>
using StressDerivative = std::array<double, d * d * d * d>;

template <int d>
struct SvdRV {
  Mat<d> U, V;
  Vec<d> sigma;
};

namespace detail {

/// Plane rotation with Eigen's JacobiRotation conventions (real case): applying it on
/// the left of rows (p,q) maps (x,y) -> (c x + s y, -s x + c y).
struct Rot {
  double c = 1, s = 0;
  Rot transpose() const { return {c, -s}; }
  Rot operator*(const Rot& o) const { return {c * o.c - s * o.s, c * o.s + s * o.c}; }
};

template <int d>
inline void apply_left(Mat<d>& m, int p, int q, const Rot& j) {
  for (int i = 0; i < d; ++i) {
    const double x = m(p, i), y = m(q, i);
    m(p, i) = j.c * x + j.s * y;
    m(q, i) = -j.s * x + j.c * y;
  }
}
template <int d>
inline void apply_right(Mat<d>& m, int p, int q, const Rot& j) {
  // Eigen applyOnTheRight(p,q,j) rotates columns with j.transpose().
  const Rot t = j.transpose();
  for (int i = 0; i < d; ++i) {
    const double x = m(i, p), y = m(i, q);
    m(i, p) = t.c * x + t.s * y;
    m(i, q) = -t.s * x + t.c * y;
  }
}

/// makeJacobi(x, y, z) for the symmetric 2x2 [[x, y], [y, z]].
inline Rot make_jacobi(double x, double y, double z) {
  Rot r;
  const double deno = 2.0 * std::abs(y);
  if (deno < std::numeric_limits<double>::min()) return r;
  const double tau = (x - z) / deno;
  const double w = std::sqrt(tau * tau + 1.0);
  const double t = tau > 0.0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
  const double sign_t = t > 0.0 ? 1.0 : -1.0;
  const double n = 1.0 / std::sqrt(t * t + 1.0);
  r.s = -sign_t * (y / std::abs(y)) * std::abs(t) * n;
  r.c = n;
  return r;
}

/// 2x2 real Jacobi SVD step on rows/cols (p,q) of m.
template <int d>
inline void real_2x2_jacobi_svd(const Mat<d>& matrix, int p, int q, Rot& j_left, Rot& j_right) {
  Mat<2> m;
  m(0, 0) = matrix(p, p);
  m(0, 1) = matrix(p, q);
  m(1, 0) = matrix(q, p);
  m(1, 1) = matrix(q, q);
  Rot rot1;
  const double t = m(0, 0) + m(1, 1);
  const double dd = m(1, 0) - m(0, 1);
  if (std::abs(dd) < std::numeric_limits<double>::min()) {
    rot1.s = 0.0;
    rot1.c = 1.0;
  } else {
    const double u = t / dd;
    const double tmp = std::sqrt(1.0 + u * u);
    rot1.s = 1.0 / tmp;
    rot1.c = u / tmp;
  }
  apply_left<2>(m, 0, 1, rot1);
  j_right = make_jacobi(m(0, 0), m(0, 1), m(1, 1));
  j_left = rot1 * j_right.transpose();
}

/// Restatement of Eigen::JacobiSVD<Matrix<double,d,d>> (two-sided Jacobi, singular values
/// descending).  Used by svd_rv (constitutive.hpp:66-82).
template <int d>
void jacobi_svd(const Mat<d>& A, Mat<d>& U, Vec<d>& sigma, Mat<d>& V) {
  double scale = 0.0;
  for (double v : A.a) scale = std::max(scale, std::abs(v));
  if (scale == 0.0) scale = 1.0;
  Mat<d> work;
  for (int i = 0; i < d * d; ++i) work.a[i] = A.a[i] / scale;
  U = Mat<d>::identity();
  V = Mat<d>::identity();
  const double consider_zero = std::numeric_limits<double>::min();
  const double precision = 2.0 * std::numeric_limits<double>::epsilon();
  double max_diag = 0.0;
  for (int i = 0; i < d; ++i) max_diag = std::max(max_diag, std::abs(work(i, i)));
  bool finished = false;
  int sweeps = 0;
  while (!finished && sweeps < 100) {
    finished = true;
    ++sweeps;
    for (int p = 1; p < d; ++p)
      for (int q = 0; q < p; ++q) {
        const double threshold = std::max(consider_zero, precision * max_diag);
        if (std::abs(work(p, q)) > threshold || std::abs(work(q, p)) > threshold) {
          finished = false;
          Rot jl, jr;
          real_2x2_jacobi_svd(work, p, q, jl, jr);
          apply_left(work, p, q, jl);
          apply_right(U, p, q, jl.transpose());
          apply_right(work, p, q, jr);
          apply_right(V, p, q, jr);
          max_diag = std::max(max_diag, std::max(std::abs(work(p, p)), std::abs(work(q, q))));
        }
      }
  }
  for (int i = 0; i < d; ++i) {
    const double a = work(i, i);
    sigma[i] = std::abs(a);
    if (a < 0.0)
      for (int r = 0; r < d; ++r) U(r, i) = -U(r, i);
  }
  for (int i = 0; i < d; ++i) sigma[i] *= scale;
  for (int i = 0; i < d; ++i) {
    int pos = i;
    double mx = sigma[i];
    for (int k = i + 1; k < d; ++k)
      if (sigma[k] > mx) {
        mx = sigma[k];
        pos = k;
      }
    if (mx == 0.0) break;
    if (pos != i) {
      std::swap(sigma[i], sigma[pos]);
      for (int r = 0; r < d; ++r) {
        std::swap(U(r, i), U(r, pos));
        std::swap(V(r, i), V(r, pos));
      }
    }
  }
}

}  // namespace detail

/// constitutive.hpp:66-82
template <int d>
SvdRV<d> svd_rv(const Mat<d>& F) {
  SvdRV<d> r;
  detail::jacobi_svd<d>(F, r.U, r.sigma, r.V);
  if (determinant(r.U) < 0.0) {
    for (int i = 0; i < d; ++i) r.U(i, d - 1) *= -1.0;
    r.sigma[d - 1] *= -1.0;
  }
  if (determinant(r.V) < 0.0) {
    for (int i = 0; i < d; ++i) r.V(i, d - 1) *= -1.0;
    r.sigma[d - 1] *= -1.0;
  }
  return r;
}

/// constitutive.hpp:85-105
template <int d>
Mat<d> cofactor(const Mat<d>& F) {
  Mat<d> A;
  if constexpr (d == 2) {
    A(0, 0) = F(1, 1);
    A(0, 1) = -F(1, 0);
    A(1, 0) = -F(0, 1);
    A(1, 1) = F(0, 0);
  } else {
    A(0, 0) = F(1, 1) * F(2, 2) - F(1, 2) * F(2, 1);
    A(0, 1) = F(1, 2) * F(2, 0) - F(1, 0) * F(2, 2);
    A(0, 2) = F(1, 0) * F(2, 1) - F(1, 1) * F(2, 0);
    A(1, 0) = F(0, 2) * F(2, 1) - F(0, 1) * F(2, 2);
    A(1, 1) = F(0, 0) * F(2, 2) - F(0, 2) * F(2, 0);
    A(1, 2) = F(0, 1) * F(2, 0) - F(0, 0) * F(2, 1);
    A(2, 0) = F(0, 1) * F(1, 2) - F(0, 2) * F(1, 1);
    A(2, 1) = F(0, 2) * F(1, 0) - F(0, 0) * F(1, 2);
    A(2, 2) = F(0, 0) * F(1, 1) - F(0, 1) * F(1, 0);
  }
  return A;
}

template <int d>
inline void check_finite_f(const Mat<d>& F, const char* who) {  // constitutive.hpp:108-112
  if (!all_finite(F)) throw std::invalid_argument(std::string(who) + ": non-finite deformation gradient");
}

/// constitutive.hpp:115-123
template <int d>
double fcr_energy_density(const Mat<d>& F, const Material& m) {
  check_finite_f(F, "fcr_energy_density");
  const auto s = svd_rv(F).sigma;
  double J = s[0];
  for (int k = 1; k < d; ++k) J *= s[k];
  double e = 0.0;
  for (int k = 0; k < d; ++k) e += (s[k] - 1.0) * (s[k] - 1.0);
  return m.mu * e + 0.5 * m.lambda * (J - 1.0) * (J - 1.0);
}

/// constitutive.hpp:126-133
template <int d>
Mat<d> fcr_stress(const Mat<d>& F, const Material& m) {
  check_finite_f(F, "fcr_stress");
  const auto svd = svd_rv(F);
  const Mat<d> R = svd.U * transpose(svd.V);
  const double J = determinant(F);
  return (2.0 * m.mu) * (F - R) + (m.lambda * (J - 1.0)) * cofactor(F);
}

/// constitutive.hpp:138-199
template <int d>
StressDerivative<d> fcr_stress_derivative(const Mat<d>& F, const Material& m) {
  check_finite_f(F, "fcr_stress_derivative");
  constexpr int D = d * d;
  const auto svd = svd_rv(F);
  const Vec<d>& s = svd.sigma;
  double J = s[0];
  for (int k = 1; k < d; ++k) J *= s[k];
  const double mu = m.mu, la = m.lambda;
  Vec<d> Jp;
  if constexpr (d == 2) {
    Jp[0] = s[1];
    Jp[1] = s[0];
  } else {
    Jp[0] = s[1] * s[2];
    Jp[1] = s[0] * s[2];
    Jp[2] = s[0] * s[1];
  }
  Vec<d> psi;
  for (int i = 0; i < d; ++i) psi[i] = 2.0 * mu * (s[i] - 1.0) + la * (J - 1.0) * Jp[i];
  auto Jpp = [&](int i, int j) -> double {
    if constexpr (d == 2) {
      (void)i;
      (void)j;
      return 1.0;
    } else {
      return s[3 - i - j];
    }
  };
  std::array<double, D * D> Mhat{};
  auto MH = [&](int r, int c) -> double& { return Mhat[r * D + c]; };
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double a = la * Jp[i] * Jp[j];
      if (i == j)
        a += 2.0 * mu;
      else
        a += la * (J - 1.0) * Jpp(i, j);
      MH(i * d + i, j * d + j) = a;
    }
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j) {
      const double bd = 2.0 * mu - la * (J - 1.0) * Jpp(i, j);
      double sum = s[i] + s[j];
      const double mag = std::max(std::abs(sum), 1e-6);
      sum = sum >= 0.0 ? mag : -mag;
      const double bs = (psi[i] + psi[j]) / sum;
      const int a = i * d + j, b = j * d + i;
      MH(a, a) = MH(b, b) = 0.5 * (bd + bs);
      MH(a, b) = MH(b, a) = 0.5 * (bd - bs);
    }
  std::array<double, D * D> Q{};
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      for (int k = 0; k < d; ++k)
        for (int l = 0; l < d; ++l) Q[(i * d + j) * D + k * d + l] = svd.U(i, k) * svd.V(j, l);
  std::array<double, D * D> QM{};
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) {
      double acc = 0.0;
      for (int k = 0; k < D; ++k) acc += Q[r * D + k] * Mhat[k * D + c];
      QM[r * D + c] = acc;
    }
  StressDerivative<d> out{};
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) {
      double acc = 0.0;
      for (int k = 0; k < D; ++k) acc += QM[r * D + k] * Q[c * D + k];
      out[r * D + c] = acc;
    }
  StressDerivative<d> sym{};
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) sym[r * D + c] = 0.5 * (out[r * D + c] + out[c * D + r]);
  return sym;
}

// ---------------------------------------------------------------------------------------
// Neo-Hookean (extension; BASELINE configs 2 and 5).  psi = mu/2 (tr F^T F - d) - mu log J +
// lambda/2 (log J)^2 (Bonet & Wood; the compressible form used by Stomakhin et al. and the HOT
// paper's Neo-Hookean scenes).  Undefined for J <= 0: the energy is +inf there (the line search
// backtracks), the stress and its derivative throw std::domain_error.
// ---------------------------------------------------------------------------------------
template <int d>
double nh_energy_density(const Mat<d>& F, const Material& m) {
  check_finite_f(F, "nh_energy_density");
  const auto s = svd_rv(F).sigma;
  double J = s[0], q = s[0] * s[0];
  for (int k = 1; k < d; ++k) {
    J *= s[k];
    q += s[k] * s[k];
  }
  if (!(J > 0.0)) return std::numeric_limits<double>::infinity();
  const double lj = std::log(J);
  return 0.5 * m.mu * (q - d) - m.mu * lj + 0.5 * m.lambda * lj * lj;
}

/// P = mu F + (lambda log J - mu) F^{-T},  F^{-T} = cof(F) / J.
template <int d>
Mat<d> nh_stress(const Mat<d>& F, const Material& m) {
  check_finite_f(F, "nh_stress");
  const double J = determinant(F);
  if (!(J > 0.0)) throw std::domain_error("nh_stress: Neo-Hookean requires det(F) > 0");
  return m.mu * F + ((m.lambda * std::log(J) - m.mu) / J) * cofactor(F);
}

/// dP/dF in the fcr_stress_derivative layout (row-major (ij),(kl), symmetrised): the same
/// diagonal-space construction with the Neo-Hookean derivatives of psi(sigma):
///   psi_i = mu s_i + (lambda log J - mu) / s_i,
///   psi_ii = mu + (mu - lambda (log J - 1)) / s_i^2,  psi_ij = lambda / (s_i s_j),
///   (psi_i - psi_j) / (s_i - s_j) = mu + (mu - lambda log J) / (s_i s_j)   (no division by 0),
///   (psi_i + psi_j) / (s_i + s_j) with the reference's |s_i + s_j| >= 1e-6 clamp.
template <int d>
StressDerivative<d> nh_stress_derivative(const Mat<d>& F, const Material& m) {
  check_finite_f(F, "nh_stress_derivative");
  constexpr int D = d * d;
  const auto svd = svd_rv(F);
  const Vec<d>& s = svd.sigma;
  double J = s[0];
  for (int k = 1; k < d; ++k) J *= s[k];
  if (!(J > 0.0)) throw std::domain_error("nh_stress_derivative: Neo-Hookean requires det(F) > 0");
  const double mu = m.mu, la = m.lambda, lj = std::log(J);
  Vec<d> psi;
  for (int i = 0; i < d; ++i) psi[i] = mu * s[i] + (la * lj - mu) / s[i];
  std::array<double, D * D> Mhat{};
  auto MH = [&](int r, int c) -> double& { return Mhat[r * D + c]; };
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      MH(i * d + i, j * d + j) = i == j ? mu + (mu - la * (lj - 1.0)) / (s[i] * s[i]) : la / (s[i] * s[j]);
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j) {
      const double bd = mu + (mu - la * lj) / (s[i] * s[j]);
      double sum = s[i] + s[j];
      const double mag = std::max(std::abs(sum), 1e-6);
      sum = sum >= 0.0 ? mag : -mag;
      const double bs = (psi[i] + psi[j]) / sum;
      const int a = i * d + j, b = j * d + i;
      MH(a, a) = MH(b, b) = 0.5 * (bd + bs);
      MH(a, b) = MH(b, a) = 0.5 * (bd - bs);
    }
  std::array<double, D * D> Q{};
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      for (int k = 0; k < d; ++k)
        for (int l = 0; l < d; ++l) Q[(i * d + j) * D + k * d + l] = svd.U(i, k) * svd.V(j, l);
  std::array<double, D * D> QM{};
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) {
      double acc = 0.0;
      for (int k = 0; k < D; ++k) acc += Q[r * D + k] * Mhat[k * D + c];
      QM[r * D + c] = acc;
    }
  StressDerivative<d> out{};
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) {
      double acc = 0.0;
      for (int k = 0; k < D; ++k) acc += QM[r * D + k] * Q[c * D + k];
      out[r * D + c] = acc;
    }
  StressDerivative<d> sym{};
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) sym[r * D + c] = 0.5 * (out[r * D + c] + out[c * D + r]);
  return sym;
}

/// The material's elastic model (FCR: the reference's functions, unchanged).
template <int d>
double energy_density(const Mat<d>& F, const Material& m) {
  return m.elasticity == ElasticityKind::NeoHookean ? nh_energy_density<d>(F, m) : fcr_energy_density<d>(F, m);
}
template <int d>
Mat<d> stress(const Mat<d>& F, const Material& m) {
  return m.elasticity == ElasticityKind::NeoHookean ? nh_stress<d>(F, m) : fcr_stress<d>(F, m);
}
template <int d>
StressDerivative<d> stress_derivative(const Mat<d>& F, const Material& m) {
  return m.elasticity == ElasticityKind::NeoHookean ? nh_stress_derivative<d>(F, m) : fcr_stress_derivative<d>(F, m);
}

namespace detail {
/// Cyclic Jacobi eigen-decomposition of a symmetric n x n matrix (stands in for
/// Eigen::SelfAdjointEigenSolver, constitutive.hpp:208).  On return A's diagonal holds
/// the eigenvalues and V's columns the eigenvectors.
template <int n>
void jacobi_eigen(std::array<double, n * n>& A, std::array<double, n * n>& V) {
  V.fill(0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q) {
        if (p == q)
          diag += A[p * n + q] * A[p * n + q];
        else
          off += A[p * n + q] * A[p * n + q];
      }
    if (off <= 1e-34 * diag || off < 1e-300) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (std::abs(apq) < 1e-300) continue;
        const double app = A[p * n + p], aqq = A[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // A <- A J  (columns p,q)
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // A <- J^T A (rows p,q)
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
}
}  // namespace detail

/// constitutive.hpp:203-219: eigenvalue clamp at zero; returns A unchanged when nothing
/// is clamped; throws on asymmetric input.
template <int n>
std::array<double, n * n> project_spd(const std::array<double, n * n>& A) {
  double mx = 0.0, asym = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      mx = std::max(mx, std::abs(A[i * n + j]));
      asym = std::max(asym, std::abs(A[i * n + j] - A[j * n + i]));
    }
  const double scale = std::max(1.0, mx);
  if (asym > 1e-12 * scale) throw std::invalid_argument("project_spd: input is not symmetric");
  std::array<double, n * n> W = A, V{};
  detail::jacobi_eigen<n>(W, V);
  std::array<double, n> ev{};
  bool changed = false;
  for (int i = 0; i < n; ++i) {
    ev[i] = W[i * n + i];
    if (ev[i] < 0.0) {
      ev[i] = 0.0;
      changed = true;
    }
  }
  if (!changed) return A;
  std::array<double, n * n> B{};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += V[i * n + k] * ev[k] * V[j * n + k];
      B[i * n + j] = acc;
    }
  std::array<double, n * n> out{};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) out[i * n + j] = 0.5 * (B[i * n + j] + B[j * n + i]);
  return out;
}

/// constitutive.hpp:224-251.  Jp (may be null): the plastic volume ratio J_p, updated by the
/// snow map as J_p <- J_p det(F_trial) / det(F_clamped) (the total J = J_e J_p is unchanged by
/// the projection; Stomakhin et al. 2013) -- state the reference does not have (SURVEY.md
/// §0.3), only used by the hardening extension.  Drucker-Prager is an extension (Klar et al.
/// 2016, section 7.3): projection of the Hencky strain onto the friction cone, or its tip.
template <int d>
Mat<d> return_map(const Mat<d>& F_trial, const Material& m, double* Jp = nullptr) {
  check_finite_f(F_trial, "return_map");
  switch (m.plasticity) {
    case PlasticityKind::None:
      return F_trial;
    case PlasticityKind::SnowClamp: {
      auto svd = svd_rv(F_trial);
      double Jt = 1.0, Jc = 1.0;
      for (int i = 0; i < d; ++i) {
        Jt *= svd.sigma[i];
        svd.sigma[i] = std::clamp(svd.sigma[i], m.clamp_lo, m.clamp_hi);
        Jc *= svd.sigma[i];
      }
      if (Jp) *Jp *= Jt / Jc;
      Mat<d> S = Mat<d>::zero();
      for (int i = 0; i < d; ++i) S(i, i) = svd.sigma[i];
      return svd.U * S * transpose(svd.V);
    }
    case PlasticityKind::DruckerPrager: {
      const auto svd = svd_rv(F_trial);
      double mn = svd.sigma[0];
      for (int i = 1; i < d; ++i) mn = std::min(mn, svd.sigma[i]);
      if (!(mn > 0.0)) throw std::domain_error("return_map: Drucker-Prager requires det(F) > 0");
      Vec<d> eps;
      double tr = 0.0;
      for (int i = 0; i < d; ++i) {
        eps[i] = std::log(svd.sigma[i]);
        tr += eps[i];
      }
      Mat<d> S = Mat<d>::zero();
      if (tr >= 0.0) {  // expansion: project to the cone's tip, sigma = 1
        for (int i = 0; i < d; ++i) S(i, i) = 1.0;
        return svd.U * S * transpose(svd.V);
      }
      Vec<d> dev;
      for (int i = 0; i < d; ++i) dev[i] = eps[i] - tr / d;
      const double nd = norm(dev);
      const double dgamma = nd + (d * m.lambda + 2.0 * m.mu) / (2.0 * m.mu) * tr * m.dp_alpha;
      if (dgamma <= 0.0 || nd == 0.0) return F_trial;  // inside the cone
      for (int i = 0; i < d; ++i) S(i, i) = std::exp(eps[i] - dgamma * dev[i] / nd);
      return svd.U * S * transpose(svd.V);
    }
    case PlasticityKind::VonMises: {
      const auto svd = svd_rv(F_trial);
      double mn = svd.sigma[0];
      for (int i = 1; i < d; ++i) mn = std::min(mn, svd.sigma[i]);
      if (!(mn > 0.0)) throw std::domain_error("return_map: von Mises requires det(F) > 0");
      Vec<d> eps;
      for (int i = 0; i < d; ++i) eps[i] = std::log(svd.sigma[i]);
      double trace = eps[0];
      for (int i = 1; i < d; ++i) trace += eps[i];
      Vec<d> dev;
      for (int i = 0; i < d; ++i) dev[i] = eps[i] - trace / d;
      const double dev_stress = 2.0 * m.mu * norm(dev);
      if (dev_stress <= m.yield_stress) return F_trial;
      for (int i = 0; i < d; ++i) dev[i] *= m.yield_stress / dev_stress;
      Mat<d> S = Mat<d>::zero();
      for (int i = 0; i < d; ++i) S(i, i) = std::exp(trace / d + dev[i]);
      return svd.U * S * transpose(svd.V);
    }
  }
  return F_trial;
}

/// constitutive.hpp:255-258
template <int d>
double stiffness_scale(const Material& m) {
  const auto T = stress_derivative<d>(Mat<d>::identity(), m);
  double s = 0.0;
  for (double v : T) s += v * v;
  return std::sqrt(s);
}

// ---------------------------------------------------------------------------------------
// transfer.hpp
// ---------------------------------------------------------------------------------------

/// transfer.hpp:12-21 (F, C are row-major here; the reference stores them column-major,
/// which only changes memory layout, not values).
template <int d>
struct Particle {
  Vec<d> x{}, v{};
  double mass = 0, volume = 0;
  Mat<d> F = Mat<d>::identity();
  Mat<d> C = Mat<d>::zero();
  int material = 0;
  double Jp = 1.0;  // plastic volume ratio (snow hardening extension; the reference has none)
};

/// transfer.hpp:28-40
template <int d, typename Fn>
void for_each_stencil_node(const Vec<d>& x, double dx, KernelKind kind, Fn&& fn) {
  const int width = kernel_stencil_width(kind);
  const int count = ipow(width, d);
  const Coord<d> base = stencil_base(x, dx, kind);
  for (int k = 0; k < count; ++k) {
    const Coord<d> node = base + stencil_offset<d>(k, width);
    const Vec<d> off = node_offset(x, dx, node);
    const double w = kernel_weight<d>(kind, off);
    if (w <= 0.0) continue;
    fn(node, w, kernel_gradient<d>(kind, off, dx));
  }
}

/// transfer.hpp:46-64 (serial in particle order)
template <int d>
void p2g(std::span<const Particle<d>> particles, SparseGrid<d>& grid) {
  std::fill(grid.mass.begin(), grid.mass.end(), 0.0);
  std::fill(grid.momentum.begin(), grid.momentum.end(), 0.0);
  std::fill(grid.velocity.begin(), grid.velocity.end(), 0.0);
  for (const auto& p : particles) {
    for_each_stencil_node<d>(p.x, grid.dx, grid.kind, [&](const Coord<d>& node, double w, const Vec<d>&) {
      const int i = grid.find(node);
      if (i < 0) return;
      const Vec<d> xi = grid.dx * node.cast();
      grid.mass[i] += w * p.mass;
      const Vec<d> mom = (w * p.mass) * (p.v + p.C * (xi - p.x));
      add_seg<d>(grid.momentum, i, mom);
    });
  }
  for (int i = 0; i < grid.node_count(); ++i)
    if (grid.mass[i] > 0.0)
      for (int a = 0; a < d; ++a) grid.velocity[d * i + a] = grid.momentum[d * i + a] / grid.mass[i];
}

/// transfer.hpp:68-87
template <int d>
void g2p(const SparseGrid<d>& grid, std::span<Particle<d>> particles) {
  const double dinv = 4.0 / (grid.dx * grid.dx);
  parallel_for(static_cast<std::int64_t>(particles.size()), [&](std::int64_t pi) {
    auto& p = particles[pi];
    Vec<d> v{};
    Mat<d> B{};
    for_each_stencil_node<d>(p.x, grid.dx, grid.kind, [&](const Coord<d>& node, double w, const Vec<d>&) {
      const int i = grid.find(node);
      if (i < 0) return;
      const Vec<d> vi = seg<d>(grid.velocity, i);
      const Vec<d> xi = grid.dx * node.cast();
      v = v + w * vi;
      B = B + outer(w * vi, xi - p.x);
    });
    p.v = v;
    p.C = dinv * B;
  });
}

/// transfer.hpp:92-114
template <int d>
long update_strain(std::span<Particle<d>> particles, const SparseGrid<d>& grid, double dt,
                   std::span<const Material> materials) {
  std::vector<char> inv(particles.size(), 0);
  parallel_for(static_cast<std::int64_t>(particles.size()), [&](std::int64_t pi) {
    auto& p = particles[pi];
    Mat<d> G{};
    for_each_stencil_node<d>(p.x, grid.dx, grid.kind, [&](const Coord<d>& node, double, const Vec<d>& grad) {
      const int i = grid.find(node);
      if (i < 0) return;
      G = G + outer(seg<d>(grid.velocity, i), grad);
    });
    p.F = (Mat<d>::identity() + dt * G) * p.F;
    const auto& m = materials[p.material];
    if (determinant(p.F) <= 0.0) {
      inv[pi] = 1;
      // the Hencky-strain maps are undefined for inverted F (Drucker-Prager: extension)
      if (m.plasticity == PlasticityKind::VonMises || m.plasticity == PlasticityKind::DruckerPrager) return;
    }
    p.F = return_map(p.F, m, &p.Jp);
  });
  long n = 0;
  for (char c : inv) n += c;
  return n;
}

/// transfer.hpp:116-120
template <int d>
void advect(std::span<Particle<d>> particles, double dt) {
  parallel_for(static_cast<std::int64_t>(particles.size()),
               [&](std::int64_t pi) { particles[pi].x = particles[pi].x + dt * particles[pi].v; });
}

}  // namespace hot_oracle

#include "hot_oracle_solver.hpp"
