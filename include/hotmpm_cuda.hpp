// hotmpm_cuda.hpp — C++ host shim with the reference's hot-path signature, backed by the
// B200 C-ABI (hot_c_api.h / libhotb200.so).
//
// Drop-in for
//   template <typename T, int d>
//   StepStats<T> hotmpm::advance_step(SimulationState<T,d>&, const SceneConfig&,
//                                     const SolverConfig<T>&, T frame_end)
// (/root/reference/proj/include/hotmpm/simulation.hpp:286-323), whose only caller is the CLI
// frame loop (/root/reference/proj/src/cli.cpp:75-81).  Include it after the reference's
// hotmpm/simulation.hpp; it uses only the reference's public types (Particle, SceneConfig,
// SolverConfig, StepStats, DiagnosticsRecord, SolverFailure) and the C-ABI.  Particles stay
// device-resident between steps; the shim uploads on the first call and downloads after every
// step so SimulationState keeps the reference's ownership semantics.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hot_c_api.h"

namespace hotmpm {
namespace cuda {

namespace detail {

inline void throw_status(int code, const char* msg) {
  switch (code) {
    case HOT_OK:
      return;
    case HOT_E_SOLVER_FAILURE:
      throw SolverFailure(msg);  // common.hpp:124-126
    case HOT_E_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case HOT_E_LOGIC:
      throw std::logic_error(msg);
    case HOT_E_DOMAIN:
      throw std::domain_error(msg);
    default:
      throw std::runtime_error(msg);
  }
}

inline hot_shape to_c(const ShapeSpec& s) {
  hot_shape h{};
  h.kind = static_cast<int>(s.kind);
  for (int a = 0; a < 3; ++a) {
    h.min[a] = s.min[a];
    h.max[a] = s.max[a];
    h.center[a] = s.center[a];
    h.point[a] = s.point[a];
    h.normal[a] = s.normal[a];
    h.axis[a] = s.axis[a];
  }
  h.radius = s.radius;
  return h;
}

/// SceneConfig (scene.hpp:61-84) -> hot_scene; the vectors own the arrays it points to.
struct SceneC {
  std::vector<hot_material> mats;
  std::vector<hot_object> objs;
  std::vector<hot_collider> cols;
  hot_scene s{};
  explicit SceneC(const SceneConfig& sc) {
    // the extension fields (elasticity, hardening, friction_angle) stay zero: the reference's
    // own materials (fixed-corotated, plain snow clamp)
    for (const auto& m : sc.materials)
      mats.push_back({m.density, m.youngs, m.poisson, static_cast<int>(m.plasticity.kind), m.plasticity.yield_stress,
                      m.plasticity.clamp_lo, m.plasticity.clamp_hi});
    for (const auto& o : sc.objects) {
      hot_object h{};
      h.shape = to_c(o.shape);
      h.material = o.material;
      for (int a = 0; a < 3; ++a) h.velocity[a] = o.velocity[a];
      h.init_kind = static_cast<int>(o.initial_deformation.kind);
      h.init_lo = o.initial_deformation.lo;
      h.init_hi = o.initial_deformation.hi;
      objs.push_back(h);
    }
    for (const auto& c : sc.colliders) {
      hot_collider h{};
      h.shape = to_c(c.shape);
      h.motion.kind = static_cast<int>(c.motion.kind);
      for (int a = 0; a < 3; ++a) {
        h.motion.velocity[a] = c.motion.velocity[a];
        h.motion.center[a] = c.motion.center[a];
        h.motion.axis[a] = c.motion.axis[a];
      }
      h.motion.omega = c.motion.omega;
      cols.push_back(h);
    }
    s.dim = sc.dim;
    s.dx = sc.dx;
    for (int a = 0; a < 3; ++a) s.gravity[a] = sc.gravity[a];
    s.fps = sc.fps;
    s.frames = sc.frames;
    s.epsilon = sc.epsilon;
    s.tau = sc.tau;
    s.levels = sc.levels;
    s.window = sc.window;
    s.solver = static_cast<int>(parse_solver_kind<double>(sc.solver));
    s.embedding = sc.embedding == "linear" ? 1 : 0;
    s.cn_length_factor = sc.cn_length_factor;
    s.seed = sc.seed;
    s.ppc = sc.ppc;
    s.poisson_sampling = sc.sampling == "poisson" ? 1 : 0;
    s.n_materials = static_cast<int>(mats.size());
    s.n_objects = static_cast<int>(objs.size());
    s.n_colliders = static_cast<int>(cols.size());
    s.materials = mats.data();
    s.objects = objs.data();
    s.colliders = cols.data();
  }
};

}  // namespace detail

/// One device context per SimulationState (keep it alive across the frame loop).
class Stepper {
 public:
  Stepper(const SceneConfig& scene, int device = 0) : scene_c_(scene) {
    hot_ctx* h = nullptr;
    const int rc = hot_create(&h, &scene_c_.s, device);
    if (rc != HOT_OK) detail::throw_status(rc, hot_last_error(nullptr));
    ctx_.reset(h);
  }

  /// Same contract as hotmpm::advance_step (simulation.hpp:286-323).
  template <typename T, int d>
  StepStats<T> advance_step(SimulationState<T, d>& sim, const SolverConfig<T>& cfg, T frame_end) {
    static_assert((d == 2 || d == 3) && sizeof(T) == 8, "the B200 path is fp64, 2D or 3D");
    hot_solver_config c{};
    c.epsilon = cfg.epsilon;
    c.tau = cfg.tau;
    c.levels = cfg.levels;
    c.window = cfg.window;
    c.ls_shrink = cfg.ls_shrink;
    c.ls_armijo = cfg.ls_armijo;
    c.ls_max_steps = cfg.ls_max_steps;
    c.cg_cap = cfg.cg_cap;
    c.outer_cap = cfg.outer_cap;
    c.kind = static_cast<int>(cfg.kind);
    c.embedding = cfg.embedding == KernelKind::Linear ? 1 : 0;
    c.pinned_coarse_iterations = cfg.pinned_coarse_iterations;
    c.cn_length_factor = cfg.cn_length_factor;
    check(hot_set_solver(ctx_.get(), &c));
    const long long n = static_cast<long long>(sim.particles.size());
    std::vector<double> x(d * n), v(d * n), m(n), vol(n), F(d * d * n), C(d * d * n);
    std::vector<int> mat(n);
    if (!uploaded_) {
      for (long long p = 0; p < n; ++p) {
        const auto& q = sim.particles[p];
        for (int a = 0; a < d; ++a) {
          x[d * p + a] = q.x[a];
          v[d * p + a] = q.v[a];
        }
        m[p] = q.mass;
        vol[p] = q.volume;
        mat[p] = q.material;
        for (int r = 0; r < d; ++r)
          for (int s = 0; s < d; ++s) {
            F[d * d * p + d * r + s] = q.F(r, s);  // Eigen (r,s) accessor: layout independent
            C[d * d * p + d * r + s] = q.C(r, s);
          }
      }
      check(hot_upload_particles(ctx_.get(), n, x.data(), v.data(), m.data(), vol.data(), F.data(), C.data(),
                                 mat.data()));
      uploaded_ = true;
    }
    check(hot_set_time(ctx_.get(), sim.time, sim.frame, sim.step_index));
    hot_step_stats st{};
    check(hot_advance_step(ctx_.get(), frame_end, &st));
    check(hot_download_particles(ctx_.get(), x.data(), v.data(), F.data(), C.data()));
    for (long long p = 0; p < n; ++p) {
      auto& q = sim.particles[p];
      for (int a = 0; a < d; ++a) {
        q.x[a] = x[d * p + a];
        q.v[a] = v[d * p + a];
      }
      for (int r = 0; r < d; ++r)
        for (int s = 0; s < d; ++s) {
          q.F(r, s) = F[d * d * p + d * r + s];
          q.C(r, s) = C[d * d * p + d * r + s];
        }
    }
    double t;
    int frame;
    long long step, inv;
    hot_get_time(ctx_.get(), &t, &frame, &step, &inv);
    sim.time = static_cast<T>(t);
    sim.step_index = step;
    sim.inversion_warnings = inv;
    int nd = 0;
    hot_diagnostics(ctx_.get(), nullptr, 0, &nd);
    std::vector<hot_diag_row> rows(nd);
    hot_diagnostics(ctx_.get(), rows.data(), nd, &nd);
    for (const auto& r : rows)
      sim.diagnostics.push_back({r.frame, static_cast<long>(r.step), r.outer_iteration, r.scaled_residual, r.energy,
                                 r.step_length, static_cast<long>(r.inner_iterations),
                                 static_cast<long>(r.work_units), r.wall_ms});
    hot_clear_diagnostics(ctx_.get());
    StepStats<T> out;
    out.dt = static_cast<T>(st.dt);
    out.outer_iterations = st.outer_iterations;
    out.inner_total = st.inner_total;
    out.node_count = st.node_count;
    out.converged = st.converged != 0;
    return out;
  }

 private:
  void check(int rc) {
    if (rc != HOT_OK) detail::throw_status(rc, hot_last_error(ctx_.get()));
  }
  struct Del {
    void operator()(hot_ctx* c) const { hot_destroy(c); }
  };
  detail::SceneC scene_c_;
  std::unique_ptr<hot_ctx, Del> ctx_;
  bool uploaded_ = false;
};

}  // namespace cuda
}  // namespace hotmpm
