// Host-side scene sampling for the product library: sample_scene_particles
// (/root/reference/proj/include/hotmpm/simulation.hpp:94-159, 221-254).  Runs once per
// scene, on the host, because the particle stream must come from libstdc++'s
// std::mt19937_64 + std::uniform_real_distribution<double> to be byte-identical with the
// reference's initial state.
#include <algorithm>
#include <array>
#include <cmath>
#include <random>
#include <stdexcept>
#include <vector>

#include "../../include/hot_c_api.h"

namespace hotb200 {

namespace {

using V3 = std::array<double, 3>;

bool inside(const hot_shape& s, const V3& x, int d) {
  auto norm = [&](const V3& v) {
    double q = v[0] * v[0];
    for (int a = 1; a < d; ++a) q += v[a] * v[a];
    return std::sqrt(q);
  };
  switch (s.kind) {
    case 0:
      for (int a = 0; a < d; ++a)
        if (x[a] < s.min[a] || x[a] > s.max[a]) return false;
      return true;
    case 1: {
      V3 r{};
      for (int a = 0; a < d; ++a) r[a] = x[a] - s.center[a];
      return norm(r) <= s.radius;
    }
    case 2: {
      double q = (x[0] - s.point[0]) * s.normal[0];
      for (int a = 1; a < d; ++a) q += (x[a] - s.point[a]) * s.normal[a];
      return q <= 0.0;
    }
    case 3: {
      V3 r{};
      for (int a = 0; a < d; ++a) r[a] = x[a] - s.center[a];
      if (d == 2) return norm(r) <= s.radius;
      V3 ax{s.axis[0], s.axis[1], s.axis[2]};
      const double an = norm(ax);
      for (int a = 0; a < 3; ++a) ax[a] = ax[a] / an;
      const double t = r[0] * ax[0] + r[1] * ax[1] + r[2] * ax[2];
      V3 q{};
      for (int a = 0; a < 3; ++a) q[a] = r[a] - t * ax[a];
      return norm(q) <= s.radius;
    }
  }
  return false;
}

int ipow(int b, int e) {
  int r = 1;
  while (e-- > 0) r *= b;
  return r;
}

double shape_volume(const hot_shape& s, int d) {
  if (s.kind == 0) {
    double v = 1.0;
    for (int a = 0; a < d; ++a) v *= (s.max[a] - s.min[a]);
    return v;
  }
  const double pi = 3.14159265358979323846;
  const double r = s.radius;
  return d == 2 ? pi * r * r : (4.0 / 3.0) * pi * r * r * r;
}

void bounds(const hot_shape& s, int d, V3& lo, V3& hi) {
  for (int a = 0; a < d; ++a) {
    if (s.kind == 0) {
      lo[a] = s.min[a];
      hi[a] = s.max[a];
    } else {
      lo[a] = s.center[a] - s.radius;
      hi[a] = s.center[a] + s.radius;
    }
  }
}

std::vector<V3> jittered(const hot_shape& s, int d, double dx, int ppc, std::mt19937_64& rng) {
  V3 lo{}, hi{};
  bounds(s, d, lo, hi);
  std::array<int, 3> clo{}, chi{}, c{};
  for (int a = 0; a < d; ++a) {
    clo[a] = static_cast<int>(std::floor(lo[a] / dx));
    chi[a] = static_cast<int>(std::ceil(hi[a] / dx));
  }
  int splits = 1;
  while (ipow(splits, d) < ppc) ++splits;
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<V3> out;
  c = clo;
  const int nsub = ipow(splits, d);
  while (true) {
    for (int k = 0; k < nsub && k < ppc; ++k) {
      int sub[3] = {0, 0, 0};
      int f = k;
      for (int a = d - 1; a >= 0; --a) {
        sub[a] = f % splits;
        f /= splits;
      }
      V3 x{};
      for (int a = 0; a < d; ++a) x[a] = (c[a] + (sub[a] + unit(rng)) / splits) * dx;
      if (inside(s, x, d)) out.push_back(x);
    }
    int a = d - 1;
    while (a >= 0) {
      if (++c[a] < chi[a]) break;
      c[a] = clo[a];
      --a;
    }
    if (a < 0) break;
  }
  return out;
}

std::vector<V3> poisson(const hot_shape& s, int d, double dx, int ppc, std::mt19937_64& rng) {
  V3 lo{}, hi{};
  bounds(s, d, lo, hi);
  const double volume = shape_volume(s, d);
  const double cell_vol = std::pow(dx, static_cast<double>(d));
  const long target = std::max<long>(1, static_cast<long>(volume / cell_vol * ppc));
  const double radius = 0.75 * dx / std::pow(static_cast<double>(ppc), 1.0 / d);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<V3> out;
  long attempts = 0;
  const long max_attempts = target * 60;
  while (static_cast<long>(out.size()) < target && attempts < max_attempts) {
    ++attempts;
    V3 x{};
    for (int a = 0; a < d; ++a) x[a] = lo[a] + unit(rng) * (hi[a] - lo[a]);
    if (!inside(s, x, d)) continue;
    bool ok = true;
    for (const auto& y : out) {
      double q = (x[0] - y[0]) * (x[0] - y[0]);
      for (int a = 1; a < d; ++a) q += (x[a] - y[a]) * (x[a] - y[a]);
      if (std::sqrt(q) < radius) {
        ok = false;
        break;
      }
    }
    if (ok) out.push_back(x);
  }
  return out;
}

}  // namespace

/// Fills interleaved particle arrays (x[d*p+a], F[d*d*p + d*r + c]); returns the count.
long long sample_scene(const hot_scene& sc, std::vector<double>& x, std::vector<double>& v, std::vector<double>& mass,
                       std::vector<double>& vol, std::vector<double>& F, std::vector<double>& C,
                       std::vector<int>& mat) {
  const int d = sc.dim;
  if (d != 2 && d != 3) throw std::invalid_argument("scene dim must be 2 or 3");
  const int ppc = sc.ppc > 0 ? sc.ppc : ipow(2, d);
  for (int oi = 0; oi < sc.n_objects; ++oi) {
    const hot_object& obj = sc.objects[oi];
    if (obj.material < 0 || obj.material >= sc.n_materials)
      throw std::invalid_argument("object references a material id that does not exist");
    std::mt19937_64 rng(sc.seed * 0x9e3779b9u + static_cast<std::uint64_t>(oi) + 1);
    std::vector<V3> xs = sc.poisson_sampling ? poisson(obj.shape, d, sc.dx, ppc, rng) : jittered(obj.shape, d, sc.dx, ppc, rng);
    const double volume = sc.poisson_sampling
                              ? shape_volume(obj.shape, d) / static_cast<double>(std::max<std::size_t>(1, xs.size()))
                              : std::pow(sc.dx, static_cast<double>(d)) / ppc;
    const double density = sc.materials[obj.material].density;
    std::uniform_real_distribution<double> fdist(obj.init_lo, obj.init_hi);
    for (const auto& p : xs) {
      for (int a = 0; a < d; ++a) {
        x.push_back(p[a]);
        v.push_back(obj.velocity[a]);
      }
      vol.push_back(volume);
      mass.push_back(density * volume);
      mat.push_back(obj.material);
      for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
          F.push_back(r == c ? 1.0 : 0.0);
          C.push_back(0.0);
        }
      if (obj.init_kind == 1) {
        const std::size_t base = F.size() - static_cast<std::size_t>(d * d);
        for (int a = 0; a < d; ++a) F[base + a * d + a] = fdist(rng);
      }
    }
  }
  return static_cast<long long>(mass.size());
}

}  // namespace hotb200
