// TEST INFRASTRUCTURE ONLY — flat C entry points over the CPU oracle (hot_oracle*.hpp) so
// pytest / bench.py's CPU-baseline leg can drive it through ctypes (oracle/oracle.py).
// Never linked into the product library.
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "hot_oracle.hpp"

using namespace hot_oracle;

extern "C" {

typedef struct {
  double density, youngs, poisson;
  int plasticity;  // 0 none, 1 von Mises, 2 snow clamp, 3 Drucker-Prager (extension)
  double yield_stress, clamp_lo, clamp_hi;
  int elasticity;  // 0 fixed-corotated (the reference), 1 Neo-Hookean (extension)
  double hardening, friction_angle;  // snow hardening xi; Drucker-Prager friction angle (degrees)
} orc_material;
typedef struct {
  int kind;
  double min[3], max[3], center[3];
  double radius;
  double point[3], normal[3], axis[3];
} orc_shape;
typedef struct {
  int kind;
  double velocity[3], center[3], axis[3];
  double omega;
} orc_motion;
typedef struct {
  orc_shape shape;
  int material;
  double velocity[3];
  int init_kind;
  double init_lo, init_hi;
} orc_object;
typedef struct {
  orc_shape shape;
  orc_motion motion;
} orc_collider;
typedef struct {
  int dim;
  double dx;
  double gravity[3];
  double fps;
  int frames;
  double epsilon, tau;
  int levels, window, solver, embedding;
  double cn_length_factor;
  unsigned long long seed;
  int ppc, poisson_sampling;
  int n_materials, n_objects, n_colliders;
  const orc_material* materials;
  const orc_object* objects;
  const orc_collider* colliders;
} orc_scene;
typedef struct {
  double epsilon, tau;
  int levels, window;
  double ls_shrink, ls_armijo;
  int ls_max_steps, cg_cap, outer_cap, kind, embedding, pinned_coarse_iterations;
  double cn_length_factor;
} orc_solver;

typedef void (*orc_apply_fn)(const double* in, double* out, void* user);
typedef double (*orc_energy_fn)(double alpha, void* user);
}

namespace {

template <int d>
struct Impl {
  static constexpr int dim = d;
  SimulationState<d> sim;
  std::unique_ptr<SparseGrid<d>> grid;
  std::vector<Material> mats;
  std::unique_ptr<ObjectiveState<d>> st;
  std::unique_ptr<BlockSparseMatrix<d>> H;
  std::unique_ptr<MultigridHierarchy<d>> hier;
};

struct Ctx {
  int dim = 3;
  std::string err;
  SceneConfig scene;
  SolverConfig cfg;
  Impl<2> s2;
  Impl<3> s3;
};

int fail(Ctx* c, int code, const char* msg) {
  if (c) c->err = msg;
  return code;
}

template <typename F>
int guard(Ctx* c, F&& f) {
  try {
    f();
    return 0;
  } catch (const SolverFailure& e) {
    return fail(c, 2, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(c, 1, e.what());
  } catch (const std::domain_error& e) {
    return fail(c, 4, e.what());
  } catch (const std::logic_error& e) {
    return fail(c, 3, e.what());
  } catch (const std::exception& e) {
    return fail(c, 5, e.what());
  }
}

template <typename F>
int dispatch(Ctx* c, F&& f) {
  return guard(c, [&] {
    if (c->dim == 2)
      f(c->s2);
    else
      f(c->s3);
  });
}

ShapeSpec to_shape(const orc_shape& s) {
  ShapeSpec r;
  r.kind = static_cast<ShapeSpec::Kind>(s.kind);
  for (int a = 0; a < 3; ++a) {
    r.min[a] = s.min[a];
    r.max[a] = s.max[a];
    r.center[a] = s.center[a];
    r.point[a] = s.point[a];
    r.normal[a] = s.normal[a];
    r.axis[a] = s.axis[a];
  }
  r.radius = s.radius;
  return r;
}

SolverConfig to_solver(const orc_solver& s) {
  SolverConfig c;
  c.epsilon = s.epsilon;
  c.tau = s.tau;
  c.levels = s.levels;
  c.window = s.window;
  c.ls_shrink = s.ls_shrink;
  c.ls_armijo = s.ls_armijo;
  c.ls_max_steps = s.ls_max_steps;
  c.cg_cap = s.cg_cap;
  c.outer_cap = s.outer_cap;
  c.kind = static_cast<SolverKind>(s.kind);
  c.embedding = static_cast<KernelKind>(s.embedding);
  c.pinned_coarse_iterations = s.pinned_coarse_iterations;
  c.cn_length_factor = s.cn_length_factor;
  return c;
}

Material to_material(const orc_material& m) {
  Material out;
  switch (m.plasticity) {
    case 1:
      out = Material::von_mises(m.density, m.youngs, m.poisson, m.yield_stress);
      break;
    case 2:
      out = Material::snow(m.density, m.youngs, m.poisson, m.clamp_lo, m.clamp_hi);
      out.with_hardening(m.hardening);
      break;
    case 3:
      out = Material::drucker_prager(m.density, m.youngs, m.poisson, m.friction_angle);
      break;
    default:
      out = Material::elastic(m.density, m.youngs, m.poisson);
  }
  out.with_elasticity(static_cast<ElasticityKind>(m.elasticity));
  return out;
}

template <int d>
Mat<d> load_mat(const double* p) {
  Mat<d> m;
  for (int i = 0; i < d * d; ++i) m.a[i] = p[i];
  return m;
}
template <int d>
void store_mat(const Mat<d>& m, double* p) {
  for (int i = 0; i < d * d; ++i) p[i] = m.a[i];
}

template <int d>
const BlockSparseMatrix<d>& level_matrix(Impl<d>& s, int level) {
  if (level == 0 && (!s.hier || s.hier->level_count() == 0)) {
    if (!s.H) throw std::logic_error("no matrix assembled");
    return *s.H;
  }
  if (!s.hier || level >= s.hier->level_count()) throw std::logic_error("no such level");
  return *s.hier->levels[level].H;
}

template <int d>
BlockSparseMatrix<d>& level_matrix_mut(Impl<d>& s, int level) {
  if (level == 0) {
    if (!s.H) throw std::logic_error("no matrix assembled");
    return *s.H;
  }
  if (!s.hier || level >= s.hier->level_count()) throw std::logic_error("no such level");
  return *s.hier->levels[level].owned;
}

}  // namespace

extern "C" {

void* orc_new(int dim) {
  auto* c = new Ctx;
  c->dim = dim == 2 ? 2 : 3;
  return c;
}
void orc_free(void* p) { delete static_cast<Ctx*>(p); }
const char* orc_error(void* p) { return static_cast<Ctx*>(p)->err.c_str(); }
void orc_set_threads(int n) { set_thread_count(n); }
int orc_get_threads() { return thread_count(); }

int orc_set_scene(void* p, const orc_scene* s) {
  auto* c = static_cast<Ctx*>(p);
  return guard(c, [&] {
    SceneConfig sc;
    sc.dim = s->dim;
    sc.dx = s->dx;
    for (int a = 0; a < 3; ++a) sc.gravity[a] = s->gravity[a];
    sc.fps = s->fps;
    sc.frames = s->frames;
    sc.epsilon = s->epsilon;
    sc.tau = s->tau;
    sc.levels = s->levels;
    sc.window = s->window;
    sc.solver = static_cast<SolverKind>(s->solver);
    sc.embedding = static_cast<KernelKind>(s->embedding);
    sc.cn_length_factor = s->cn_length_factor;
    sc.seed = s->seed;
    sc.ppc = s->ppc;
    sc.poisson_sampling = s->poisson_sampling != 0;
    for (int i = 0; i < s->n_materials; ++i) {
      const auto& m = s->materials[i];
      MaterialSpec ms;
      ms.density = m.density;
      ms.youngs = m.youngs;
      ms.poisson = m.poisson;
      ms.plasticity = static_cast<PlasticityKind>(m.plasticity);
      ms.yield_stress = m.yield_stress;
      ms.clamp_lo = m.clamp_lo;
      ms.clamp_hi = m.clamp_hi;
      ms.elasticity = static_cast<ElasticityKind>(m.elasticity);
      ms.hardening = m.hardening;
      ms.friction_angle = m.friction_angle;
      sc.materials.push_back(ms);
    }
    for (int i = 0; i < s->n_objects; ++i) {
      const auto& o = s->objects[i];
      ObjectSpec os;
      os.shape = to_shape(o.shape);
      os.material = o.material;
      for (int a = 0; a < 3; ++a) os.velocity[a] = o.velocity[a];
      os.initial_deformation.kind = static_cast<InitialDeformationSpec::Kind>(o.init_kind);
      os.initial_deformation.lo = o.init_lo;
      os.initial_deformation.hi = o.init_hi;
      sc.objects.push_back(os);
    }
    for (int i = 0; i < s->n_colliders; ++i) {
      const auto& k = s->colliders[i];
      ColliderSpec cs;
      cs.shape = to_shape(k.shape);
      cs.motion.kind = static_cast<MotionSpec::Kind>(k.motion.kind);
      for (int a = 0; a < 3; ++a) {
        cs.motion.velocity[a] = k.motion.velocity[a];
        cs.motion.center[a] = k.motion.center[a];
        cs.motion.axis[a] = k.motion.axis[a];
      }
      cs.motion.omega = k.motion.omega;
      sc.colliders.push_back(cs);
    }
    c->scene = sc;
    c->dim = sc.dim == 2 ? 2 : 3;
    c->cfg = solver_config_from_scene(sc);
    std::vector<Material> mats = materials_from_scene(sc);
    c->s2.mats = mats;
    c->s3.mats = mats;
  });
}

int orc_set_solver(void* p, const orc_solver* s) {
  auto* c = static_cast<Ctx*>(p);
  return guard(c, [&] { c->cfg = to_solver(*s); });
}

int orc_set_materials(void* p, int n, const orc_material* m) {
  auto* c = static_cast<Ctx*>(p);
  return guard(c, [&] {
    std::vector<Material> mats;
    for (int i = 0; i < n; ++i) mats.push_back(to_material(m[i]));
    c->s2.mats = mats;
    c->s3.mats = mats;
  });
}

int orc_set_gravity_dx(void* p, const double* gravity, double dx, double cn_length_factor) {
  auto* c = static_cast<Ctx*>(p);
  for (int a = 0; a < 3; ++a) c->scene.gravity[a] = gravity[a];
  c->scene.dx = dx;
  c->scene.cn_length_factor = cn_length_factor;
  return 0;
}

long long orc_particle_count(void* p) {
  auto* c = static_cast<Ctx*>(p);
  return c->dim == 2 ? static_cast<long long>(c->s2.sim.particles.size())
                     : static_cast<long long>(c->s3.sim.particles.size());
}

}  // extern "C"

// Dimension-templated bodies -------------------------------------------------------------
namespace {

template <int d>
void sample_impl(Ctx* c, Impl<d>& s) {
  s.sim = SimulationState<d>();
  s.sim.particles = sample_scene_particles<d>(c->scene);
}

template <int d>
void set_particles_impl(Impl<d>& s, long long n, const double* x, const double* v, const double* mass,
                        const double* vol, const double* F, const double* C, const int* mat) {
  s.sim.particles.assign(n, Particle<d>());
  for (long long i = 0; i < n; ++i) {
    auto& q = s.sim.particles[i];
    for (int a = 0; a < d; ++a) {
      q.x[a] = x[i * d + a];
      if (v) q.v[a] = v[i * d + a];
    }
    if (mass) q.mass = mass[i];
    if (vol) q.volume = vol[i];
    if (F) q.F = load_mat<d>(F + i * d * d);
    if (C) q.C = load_mat<d>(C + i * d * d);
    if (mat) q.material = mat[i];
  }
}

template <int d>
void get_particles_impl(Impl<d>& s, double* x, double* v, double* mass, double* vol, double* F, double* C, int* mat) {
  const long long n = static_cast<long long>(s.sim.particles.size());
  for (long long i = 0; i < n; ++i) {
    const auto& q = s.sim.particles[i];
    for (int a = 0; a < d; ++a) {
      if (x) x[i * d + a] = q.x[a];
      if (v) v[i * d + a] = q.v[a];
    }
    if (mass) mass[i] = q.mass;
    if (vol) vol[i] = q.volume;
    if (F) store_mat<d>(q.F, F + i * d * d);
    if (C) store_mat<d>(q.C, C + i * d * d);
    if (mat) mat[i] = q.material;
  }
}

template <int d>
void activate_impl(Ctx* c, Impl<d>& s, int kind) {
  std::vector<Vec<d>> xs(s.sim.particles.size());
  for (std::size_t i = 0; i < xs.size(); ++i) xs[i] = s.sim.particles[i].x;
  s.grid = std::make_unique<SparseGrid<d>>(activate_grid<d>(xs, c->scene.dx, static_cast<KernelKind>(kind)));
  s.st.reset();
  s.H.reset();
  s.hier.reset();
}

template <int d>
SparseGrid<d>& need_grid(Impl<d>& s) {
  if (!s.grid) throw std::logic_error("grid not activated");
  return *s.grid;
}
template <int d>
ObjectiveState<d>& need_state(Impl<d>& s) {
  if (!s.st) throw std::logic_error("objective state not built");
  return *s.st;
}

template <int d>
VecX vin(const double* p, std::size_t n) {
  return VecX(p, p + n);
}

}  // namespace

extern "C" {

int orc_sample_scene(void* p) {
  auto* c = static_cast<Ctx*>(p);
  return guard(c, [&] {
    if (c->dim == 2)
      sample_impl<2>(c, c->s2);
    else
      sample_impl<3>(c, c->s3);
  });
}

int orc_set_particles(void* p, long long n, const double* x, const double* v, const double* mass, const double* vol,
                      const double* F, const double* C, const int* mat) {
  auto* c = static_cast<Ctx*>(p);
  return guard(c, [&] {
    if (c->dim == 2)
      set_particles_impl<2>(c->s2, n, x, v, mass, vol, F, C, mat);
    else
      set_particles_impl<3>(c->s3, n, x, v, mass, vol, F, C, mat);
  });
}

int orc_get_particles(void* p, double* x, double* v, double* mass, double* vol, double* F, double* C, int* mat) {
  auto* c = static_cast<Ctx*>(p);
  return guard(c, [&] {
    if (c->dim == 2)
      get_particles_impl<2>(c->s2, x, v, mass, vol, F, C, mat);
    else
      get_particles_impl<3>(c->s3, x, v, mass, vol, F, C, mat);
  });
}

/// Plastic volume ratio J_p per particle (snow hardening extension); get/set.
int orc_particle_jp(void* p, double* out, const double* in) {
  auto* c = static_cast<Ctx*>(p);
  return guard(c, [&] {
    auto io = [&](auto& s) {
      const long long n = static_cast<long long>(s.sim.particles.size());
      for (long long i = 0; i < n; ++i) {
        if (in) s.sim.particles[i].Jp = in[i];
        if (out) out[i] = s.sim.particles[i].Jp;
      }
    };
    if (c->dim == 2)
      io(c->s2);
    else
      io(c->s3);
  });
}

int orc_sim_state(void* p, double* time, long long* step, long long* inversions, int* frame) {
  auto* c = static_cast<Ctx*>(p);
  auto get = [&](auto& s) {
    if (time) *time = s.sim.time;
    if (step) *step = s.sim.step_index;
    if (inversions) *inversions = s.sim.inversion_warnings;
    if (frame) *frame = s.sim.frame;
  };
  if (c->dim == 2)
    get(c->s2);
  else
    get(c->s3);
  return 0;
}

int orc_set_sim_state(void* p, double time, long long step, int frame) {
  auto* c = static_cast<Ctx*>(p);
  auto set = [&](auto& s) {
    s.sim.time = time;
    s.sim.step_index = step;
    s.sim.frame = frame;
  };
  if (c->dim == 2)
    set(c->s2);
  else
    set(c->s3);
  return 0;
}

int orc_advance_step(void* p, double frame_end, double* dt, int* outer, long long* inner, int* nodes, int* converged) {
  auto* c = static_cast<Ctx*>(p);
  return guard(c, [&] {
    StepStats st;
    if (c->dim == 2)
      st = advance_step<2>(c->s2.sim, c->scene, c->cfg, frame_end);
    else
      st = advance_step<3>(c->s3.sim, c->scene, c->cfg, frame_end);
    if (dt) *dt = st.dt;
    if (outer) *outer = st.outer_iterations;
    if (inner) *inner = st.inner_total;
    if (nodes) *nodes = st.node_count;
    if (converged) *converged = st.converged;
  });
}

long long orc_diag_count(void* p) {
  auto* c = static_cast<Ctx*>(p);
  return c->dim == 2 ? static_cast<long long>(c->s2.sim.diagnostics.size())
                     : static_cast<long long>(c->s3.sim.diagnostics.size());
}

int orc_diag_get(void* p, int* frame, long long* step, int* outer, double* residual, double* energy, double* alpha,
                 long long* inner, long long* work, double* wall_ms) {
  auto* c = static_cast<Ctx*>(p);
  const auto& D = c->dim == 2 ? c->s2.sim.diagnostics : c->s3.sim.diagnostics;
  for (std::size_t i = 0; i < D.size(); ++i) {
    frame[i] = D[i].frame;
    step[i] = D[i].step;
    outer[i] = D[i].outer_iteration;
    residual[i] = D[i].scaled_residual;
    energy[i] = D[i].energy;
    alpha[i] = D[i].step_length;
    inner[i] = D[i].inner_iterations;
    work[i] = D[i].work_units;
    if (wall_ms) wall_ms[i] = D[i].wall_ms;
  }
  return 0;
}

void orc_diag_clear(void* p) {
  auto* c = static_cast<Ctx*>(p);
  c->s2.sim.diagnostics.clear();
  c->s3.sim.diagnostics.clear();
}

// ---- stage API --------------------------------------------------------------------------

int orc_activate(void* p, int kind) {
  auto* c = static_cast<Ctx*>(p);
  return guard(c, [&] {
    if (c->dim == 2)
      activate_impl<2>(c, c->s2, kind);
    else
      activate_impl<3>(c, c->s3, kind);
  });
}

int orc_grid_nodes(void* p) {
  auto* c = static_cast<Ctx*>(p);
  if (c->dim == 2) return c->s2.grid ? c->s2.grid->node_count() : -1;
  return c->s3.grid ? c->s3.grid->node_count() : -1;
}

int orc_grid_get(void* p, int* coords, double* mass, double* velocity, double* momentum, unsigned char* dirichlet,
                 double* bc_velocity) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& g = need_grid(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    for (int i = 0; i < g.node_count(); ++i) {
      if (coords)
        for (int a = 0; a < d; ++a) coords[i * d + a] = g.coords[i][a];
      if (mass) mass[i] = g.mass[i];
      if (dirichlet) dirichlet[i] = g.dirichlet[i];
    }
    const std::size_t nd = g.velocity.size();
    if (velocity) std::memcpy(velocity, g.velocity.data(), nd * 8);
    if (momentum) std::memcpy(momentum, g.momentum.data(), nd * 8);
    if (bc_velocity) std::memcpy(bc_velocity, g.bc_velocity.data(), nd * 8);
  });
}

int orc_grid_set(void* p, const double* velocity, const unsigned char* dirichlet, const double* bc_velocity) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& g = need_grid(s);
    const std::size_t nd = g.velocity.size();
    if (velocity) std::memcpy(g.velocity.data(), velocity, nd * 8);
    if (bc_velocity) std::memcpy(g.bc_velocity.data(), bc_velocity, nd * 8);
    if (dirichlet)
      for (int i = 0; i < g.node_count(); ++i) g.dirichlet[i] = dirichlet[i];
  });
}

int orc_p2g(void* p) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& g = need_grid(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    p2g<d>(s.sim.particles, g);
  });
}

int orc_apply_bc(void* p, double time) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& g = need_grid(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    apply_boundary_scripts<d>(g, c->scene, time);
  });
}

int orc_make_state(void* p, double dt) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& g = need_grid(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    s.st = std::make_unique<ObjectiveState<d>>(make_objective_state<d>(
        s.sim.particles, g, s.mats, dt, take<d>(c->scene.gravity), c->scene.cn_length_factor));
    s.H.reset();
    s.hier.reset();
  });
}

int orc_energy(void* p, const double* dv, double* out) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& st = need_state(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    *out = energy<d>(st, VecX(dv, dv + st.dof_count()));
  });
}

int orc_gradient(void* p, const double* dv, double* g) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& st = need_state(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    VecX r = gradient<d>(st, VecX(dv, dv + st.dof_count()));
    std::memcpy(g, r.data(), r.size() * 8);
  });
}

int orc_node_cn(void* p, double* xi, double* scale) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& st = need_state(s);
    NodeCN cn = compute_node_cn(st);
    if (xi) std::memcpy(xi, cn.xi.data(), cn.xi.size() * 8);
    if (scale) std::memcpy(scale, cn.scale.data(), cn.scale.size() * 8);
  });
}

int orc_scaled_norm(void* p, const double* g, double* out) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& st = need_state(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    NodeCN cn = compute_node_cn(st);
    *out = scaled_norm<d>(VecX(g, g + st.dof_count()), cn);
  });
}

int orc_assemble(void* p, const double* dv, int project) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& st = need_state(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    s.hier.reset();
    s.H = std::make_unique<BlockSparseMatrix<d>>(assemble_hessian<d>(st, VecX(dv, dv + st.dof_count()), project != 0));
  });
}

int orc_build_hierarchy(void* p, int levels, int embedding) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& g = need_grid(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    if (!s.H) throw std::logic_error("no matrix assembled");
    s.hier = std::make_unique<MultigridHierarchy<d>>(build_hierarchy<d>(*s.H, g, levels, static_cast<KernelKind>(embedding)));
  });
}

int orc_level_count(void* p) {
  auto* c = static_cast<Ctx*>(p);
  if (c->dim == 2) return c->s2.hier ? c->s2.hier->level_count() : 0;
  return c->s3.hier ? c->s3.hier->level_count() : 0;
}

int orc_level_shape(void* p, int level, int* rows, int* slots, int* radius) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    const auto& H = level_matrix(s, level);
    *rows = H.rows();
    *slots = H.slots();
    *radius = H.radius();
  });
}

int orc_level_matrix(void* p, int level, double* blocks, int* cols) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    const auto& H = level_matrix(s, level);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    for (int r = 0; r < H.rows(); ++r)
      for (int k = 0; k < H.slots(); ++k) {
        const std::size_t o = static_cast<std::size_t>(r) * H.slots() + k;
        if (cols) cols[o] = H.col(r, k);
        if (blocks) store_mat<d>(H.block(r, k), blocks + o * d * d);
      }
  });
}

int orc_set_level_matrix(void* p, int level, const double* blocks) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& H = level_matrix_mut(s, level);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    for (int r = 0; r < H.rows(); ++r)
      for (int k = 0; k < H.slots(); ++k) {
        const std::size_t o = static_cast<std::size_t>(r) * H.slots() + k;
        H.block(r, k) = load_mat<d>(blocks + o * d * d);
      }
  });
}

int orc_level_info(void* p, int level, int* coords, unsigned char* dirichlet, int* sweep_order, double* diag_inv) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    if (!s.hier || level >= s.hier->level_count()) throw std::logic_error("no such level");
    const auto& L = s.hier->levels[level];
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    for (int i = 0; i < L.info.node_count(); ++i) {
      if (coords)
        for (int a = 0; a < d; ++a) coords[i * d + a] = L.info.coords[i][a];
      if (dirichlet) dirichlet[i] = L.info.dirichlet[i];
      if (sweep_order) sweep_order[i] = L.sweep_order[i];
      if (diag_inv) store_mat<d>(L.diag_inv[i], diag_inv + static_cast<std::size_t>(i) * d * d);
    }
  });
}

int orc_level_restriction(void* p, int level, int* row_start, int* coarse, double* weight, int* nnz) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    if (!s.hier || level >= s.hier->level_count()) throw std::logic_error("no such level");
    const auto& R = s.hier->levels[level].R;
    *nnz = static_cast<int>(R.entries.size());
    if (row_start)
      for (std::size_t i = 0; i < R.row_start.size(); ++i) row_start[i] = R.row_start[i];
    for (std::size_t e = 0; e < R.entries.size(); ++e) {
      if (coarse) coarse[e] = R.entries[e].coarse;
      if (weight) weight[e] = R.entries[e].weight;
    }
  });
}

int orc_refinalize_level(void* p, int level, int modulus) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    if (!s.hier || level >= s.hier->level_count()) throw std::logic_error("no such level");
    finalize_level(s.hier->levels[level], modulus);
  });
}

int orc_matvec(void* p, int level, const double* x, double* y) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    const auto& H = level_matrix(s, level);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    VecX r = H * VecX(x, x + static_cast<std::size_t>(H.rows()) * d);
    std::memcpy(y, r.data(), r.size() * 8);
  });
}

int orc_smooth_sgs(void* p, int level, double* u, const double* b, int sweeps) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    if (!s.hier || level >= s.hier->level_count()) throw std::logic_error("no such level");
    const auto& L = s.hier->levels[level];
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    const std::size_t n = static_cast<std::size_t>(L.H->rows()) * d;
    VecX uu(u, u + n);
    smooth_sgs<d>(*L.H, L.diag_inv, L.sweep_order, uu, VecX(b, b + n), sweeps);
    std::memcpy(u, uu.data(), n * 8);
  });
}

int orc_coarse_solve(void* p, int level, const double* b, double* u, int* iters, int pinned, int pinned_cap, int cap) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    if (!s.hier || level >= s.hier->level_count()) throw std::logic_error("no such level");
    const auto& L = s.hier->levels[level];
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    const std::size_t n = static_cast<std::size_t>(L.H->rows()) * d;
    auto r = coarse_solve<d>(*L.H, L.diag_inv, VecX(b, b + n), CoarseSolveMode{pinned != 0, pinned_cap}, cap);
    std::memcpy(u, r.u.data(), n * 8);
    *iters = r.iterations;
  });
}

int orc_vcycle(void* p, const double* b, double* u, int* coarse_iters, int pinned, int pinned_cap) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    if (!s.hier) throw std::logic_error("no hierarchy");
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    const std::size_t n = static_cast<std::size_t>(s.hier->levels[0].H->rows()) * d;
    auto r = vcycle<d>(*s.hier, VecX(b, b + n), CoarseSolveMode{pinned != 0, pinned_cap});
    std::memcpy(u, r.u.data(), n * 8);
    *coarse_iters = r.coarse_iterations;
  });
}

int orc_step_grid(void* p, double* velocity, double* dv, int* outer, long long* inner, int* converged,
                  int* rebuilds, int frame, long long step) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& st = need_state(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    auto r = step_grid<d>(st, c->cfg, &s.sim.diagnostics, frame, step);
    if (velocity) std::memcpy(velocity, r.velocity.data(), r.velocity.size() * 8);
    if (dv) std::memcpy(dv, r.solve.dv.data(), r.solve.dv.size() * 8);
    if (outer) *outer = r.solve.outer_iterations;
    if (inner) *inner = r.solve.inner_total;
    if (converged) *converged = r.solve.converged;
    if (rebuilds) *rebuilds = r.solve.hierarchy_rebuilds;
  });
}

int orc_g2p(void* p) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& g = need_grid(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    g2p<d>(g, s.sim.particles);
  });
}

int orc_update_strain(void* p, double dt, long long* inverted) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& g = need_grid(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    *inverted = update_strain<d>(s.sim.particles, g, dt, s.mats);
  });
}

int orc_advect(void* p, double dt) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    advect<d>(s.sim.particles, dt);
  });
}

// ---- point functions (no context) --------------------------------------------------------

double orc_kernel_weight_1d(int kind, double x) { return kernel_weight_1d(static_cast<KernelKind>(kind), x); }
double orc_kernel_derivative_1d(int kind, double x) { return kernel_derivative_1d(static_cast<KernelKind>(kind), x); }

double orc_kernel_weight(int dim, int kind, const double* off) {
  if (dim == 2) {
    Vec<2> o{{off[0], off[1]}};
    return kernel_weight<2>(static_cast<KernelKind>(kind), o);
  }
  if (dim == 1) {
    Vec<1> o{{off[0]}};
    return kernel_weight<1>(static_cast<KernelKind>(kind), o);
  }
  Vec<3> o{{off[0], off[1], off[2]}};
  return kernel_weight<3>(static_cast<KernelKind>(kind), o);
}

void orc_kernel_gradient(int dim, int kind, const double* off, double dx, double* out) {
  if (dim == 1) {
    Vec<1> o{{off[0]}};
    out[0] = kernel_gradient<1>(static_cast<KernelKind>(kind), o, dx)[0];
  } else if (dim == 2) {
    Vec<2> o{{off[0], off[1]}};
    auto g = kernel_gradient<2>(static_cast<KernelKind>(kind), o, dx);
    out[0] = g[0];
    out[1] = g[1];
  } else {
    Vec<3> o{{off[0], off[1], off[2]}};
    auto g = kernel_gradient<3>(static_cast<KernelKind>(kind), o, dx);
    for (int a = 0; a < 3; ++a) out[a] = g[a];
  }
}

void orc_stencil_base(int dim, const double* x, double dx, int kind, int* out) {
  if (dim == 2) {
    Vec<2> o{{x[0], x[1]}};
    auto b = stencil_base<2>(o, dx, static_cast<KernelKind>(kind));
    out[0] = b[0];
    out[1] = b[1];
  } else {
    Vec<3> o{{x[0], x[1], x[2]}};
    auto b = stencil_base<3>(o, dx, static_cast<KernelKind>(kind));
    for (int a = 0; a < 3; ++a) out[a] = b[a];
  }
}

double orc_cfl_dt(double v_max, double dx, double fps) { return cfl_dt(v_max, dx, fps); }

}  // extern "C"

static thread_local std::string g_point_err;

template <typename F>
static int pguard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_point_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_point_err = e.what();
    return 4;
  } catch (const std::logic_error& e) {
    g_point_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_point_err = e.what();
    return 5;
  }
}

extern "C" {
const char* orc_point_error() { return g_point_err.c_str(); }

int orc_material_lame(const orc_material* m, double* mu, double* lambda) {
  return pguard([&] {
    Material mm = to_material(*m);
    *mu = mm.mu;
    *lambda = mm.lambda;
  });
}

int orc_svd(int dim, const double* F, double* U, double* sigma, double* V) {
  return pguard([&] {
    if (dim == 2) {
      auto r = svd_rv<2>(load_mat<2>(F));
      store_mat<2>(r.U, U);
      store_mat<2>(r.V, V);
      for (int a = 0; a < 2; ++a) sigma[a] = r.sigma[a];
    } else {
      auto r = svd_rv<3>(load_mat<3>(F));
      store_mat<3>(r.U, U);
      store_mat<3>(r.V, V);
      for (int a = 0; a < 3; ++a) sigma[a] = r.sigma[a];
    }
  });
}

int orc_fcr_energy(int dim, const double* F, const orc_material* m, double* out) {
  return pguard([&] {
    Material mm = to_material(*m);
    *out = dim == 2 ? fcr_energy_density<2>(load_mat<2>(F), mm) : fcr_energy_density<3>(load_mat<3>(F), mm);
  });
}

int orc_fcr_stress(int dim, const double* F, const orc_material* m, double* out) {
  return pguard([&] {
    Material mm = to_material(*m);
    if (dim == 2)
      store_mat<2>(fcr_stress<2>(load_mat<2>(F), mm), out);
    else
      store_mat<3>(fcr_stress<3>(load_mat<3>(F), mm), out);
  });
}

int orc_fcr_dpdf(int dim, const double* F, const orc_material* m, int project, double* out) {
  return pguard([&] {
    Material mm = to_material(*m);
    if (dim == 2) {
      auto T = fcr_stress_derivative<2>(load_mat<2>(F), mm);
      if (project) T = project_spd<4>(T);
      std::memcpy(out, T.data(), sizeof(T));
    } else {
      auto T = fcr_stress_derivative<3>(load_mat<3>(F), mm);
      if (project) T = project_spd<9>(T);
      std::memcpy(out, T.data(), sizeof(T));
    }
  });
}

int orc_project_spd(int n, const double* A, double* out) {
  return pguard([&] {
    if (n == 4) {
      std::array<double, 16> a;
      std::memcpy(a.data(), A, sizeof(a));
      auto r = project_spd<4>(a);
      std::memcpy(out, r.data(), sizeof(r));
    } else if (n == 9) {
      std::array<double, 81> a;
      std::memcpy(a.data(), A, sizeof(a));
      auto r = project_spd<9>(a);
      std::memcpy(out, r.data(), sizeof(r));
    } else if (n == 2) {
      std::array<double, 4> a;
      std::memcpy(a.data(), A, sizeof(a));
      auto r = project_spd<2>(a);
      std::memcpy(out, r.data(), sizeof(r));
    } else if (n == 3) {
      std::array<double, 9> a;
      std::memcpy(a.data(), A, sizeof(a));
      auto r = project_spd<3>(a);
      std::memcpy(out, r.data(), sizeof(r));
    } else {
      throw std::invalid_argument("orc_project_spd: n must be 2, 3, 4 or 9");
    }
  });
}

int orc_return_map(int dim, const double* F, const orc_material* m, double* out) {
  return pguard([&] {
    Material mm = to_material(*m);
    if (dim == 2)
      store_mat<2>(return_map<2>(load_mat<2>(F), mm), out);
    else
      store_mat<3>(return_map<3>(load_mat<3>(F), mm), out);
  });
}

// ---- the material's own model (extensions dispatch: Neo-Hookean, hardening factor h) ----------
int orc_model_energy(int dim, const double* F, const orc_material* m, double h, double* out) {
  return pguard([&] {
    const Material mm = to_material(*m).hardened(h);
    *out = dim == 2 ? energy_density<2>(load_mat<2>(F), mm) : energy_density<3>(load_mat<3>(F), mm);
  });
}

int orc_model_stress(int dim, const double* F, const orc_material* m, double h, double* out) {
  return pguard([&] {
    const Material mm = to_material(*m).hardened(h);
    if (dim == 2)
      store_mat<2>(stress<2>(load_mat<2>(F), mm), out);
    else
      store_mat<3>(stress<3>(load_mat<3>(F), mm), out);
  });
}

int orc_model_dpdf(int dim, const double* F, const orc_material* m, double h, int project, double* out) {
  return pguard([&] {
    const Material mm = to_material(*m).hardened(h);
    if (dim == 2) {
      auto T = stress_derivative<2>(load_mat<2>(F), mm);
      if (project) T = project_spd<4>(T);
      std::memcpy(out, T.data(), sizeof(T));
    } else {
      auto T = stress_derivative<3>(load_mat<3>(F), mm);
      if (project) T = project_spd<9>(T);
      std::memcpy(out, T.data(), sizeof(T));
    }
  });
}

/// return_map with the plastic volume ratio (in/out through *Jp).
int orc_return_map_jp(int dim, const double* F, const orc_material* m, double* Jp, double* out) {
  return pguard([&] {
    Material mm = to_material(*m);
    if (dim == 2)
      store_mat<2>(return_map<2>(load_mat<2>(F), mm, Jp), out);
    else
      store_mat<3>(return_map<3>(load_mat<3>(F), mm, Jp), out);
  });
}

double orc_hardening_factor(const orc_material* m, double Jp) { return to_material(*m).hardening_factor(Jp); }

int orc_stiffness_scale(int dim, const orc_material* m, double* out) {
  return pguard([&] {
    Material mm = to_material(*m);
    *out = dim == 2 ? stiffness_scale<2>(mm) : stiffness_scale<3>(mm);
  });
}

double orc_adaptive_cg_tolerance(double pe_sq, double tau) { return adaptive_cg_tolerance(pe_sq, tau); }

// ---- solver building blocks on callbacks (test_solvers.cpp restatements) ---------------

int orc_pcg(int n, orc_apply_fn apply_a, orc_apply_fn apply_p, void* user, const double* b, double rel_tol, int cap,
            double* x, int* iterations, int* converged) {
  return pguard([&] {
    auto A = [&](const VecX& in) {
      VecX out(n);
      apply_a(in.data(), out.data(), user);
      return out;
    };
    auto P = [&](const VecX& in) {
      VecX out(n);
      apply_p(in.data(), out.data(), user);
      return out;
    };
    try {
      auto r = pcg(A, P, VecX(b, b + n), rel_tol, cap);
      std::memcpy(x, r.x.data(), n * 8);
      *iterations = r.iterations;
      *converged = r.converged;
    } catch (const SolverFailure& e) {
      g_point_err = e.what();
      throw std::runtime_error(std::string("SolverFailure: ") + e.what());
    }
  });
}

int orc_line_search(orc_energy_fn fn, void* user, double e0, double gdotp, const orc_solver* cfg, double* alpha,
                    double* energy_out, int* evals) {
  return pguard([&] {
    SolverConfig c = cfg ? to_solver(*cfg) : SolverConfig();
    try {
      auto r = line_search([&](double a) { return fn(a, user); }, e0, gdotp, c);
      *alpha = r.alpha;
      *energy_out = r.energy;
      *evals = r.evaluations;
    } catch (const SolverFailure& e) {
      throw std::runtime_error(std::string("SolverFailure: ") + e.what());
    }
  });
}

void* orc_lbfgs_new(int window) { return new LBFGSHistory(window); }
void orc_lbfgs_free(void* h) { delete static_cast<LBFGSHistory*>(h); }
int orc_lbfgs_push(void* h, int n, const double* s, const double* y) {
  return static_cast<LBFGSHistory*>(h)->push(VecX(s, s + n), VecX(y, y + n)) ? 1 : 0;
}
int orc_lbfgs_size(void* h) { return static_cast<LBFGSHistory*>(h)->size(); }
int orc_lbfgs_direction(void* h, int n, const double* g, orc_apply_fn init, void* user, double* p) {
  return pguard([&] {
    auto I = [&](const VecX& q) {
      VecX out(n);
      init(q.data(), out.data(), user);
      return out;
    };
    VecX r = lbfgs_direction(VecX(g, g + n), *static_cast<LBFGSHistory*>(h), I);
    std::memcpy(p, r.data(), n * 8);
  });
}

}  // extern "C"

extern "C" int orc_matvec_mf(void* p, const double* dv, const double* u, double* y, int project) {
  auto* c = static_cast<Ctx*>(p);
  return dispatch(c, [&](auto& s) {
    auto& st = need_state(s);
    constexpr int d = std::remove_reference_t<decltype(s)>::dim;
    const std::size_t n = st.dof_count();
    VecX r = multiply_matrix_free<d>(st, VecX(dv, dv + n), VecX(u, u + n), project != 0);
    std::memcpy(y, r.data(), n * 8);
  });
}
