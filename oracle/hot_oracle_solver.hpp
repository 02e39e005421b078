// TEST INFRASTRUCTURE ONLY — second half of the CPU parity oracle (see hot_oracle.hpp).
// Restates objective.hpp, multigrid.hpp, pcg.hpp, solvers.hpp and simulation.hpp of
// /root/reference/proj/include/hotmpm.
#pragma once

#include <cstdio>
#include <cstdlib>

#include "hot_oracle.hpp"

namespace hot_oracle {

// ---------------------------------------------------------------------------------------
// objective.hpp
// ---------------------------------------------------------------------------------------

/// objective.hpp:15-130: diagonal (fixed-offset) block storage, (2r+1)^d slots per row,
/// column -1 for inactive slots.  Blocks are stored row-major d x d.
template <int d>
class BlockSparseMatrix {
 public:
  BlockSparseMatrix() = default;
  BlockSparseMatrix(const std::vector<Coord<d>>& coords, const CoordIndex<d>& index, int radius)
      : rows_(static_cast<int>(coords.size())), radius_(radius), nslots_(ipow(2 * radius + 1, d)) {
    offsets_.resize(nslots_);
    for (int s = 0; s < nslots_; ++s) {
      Coord<d> off = stencil_offset<d>(s, 2 * radius + 1);
      for (int a = 0; a < d; ++a) off[a] -= radius;
      offsets_[s] = off;
    }
    cols_.assign(static_cast<std::size_t>(rows_) * nslots_, -1);
    data_.assign(static_cast<std::size_t>(rows_) * nslots_, Mat<d>::zero());
    parallel_for(rows_, [&](std::int64_t r) {
      for (int s = 0; s < nslots_; ++s) {
        auto it = index.find(coords[r] + offsets_[s]);
        if (it != index.end()) cols_[r * nslots_ + s] = it->second;
      }
    });
  }
  int rows() const { return rows_; }
  int slots() const { return nslots_; }
  int radius() const { return radius_; }
  const Coord<d>& offset(int slot) const { return offsets_[slot]; }
  int slot_of(const Coord<d>& off) const {  // objective.hpp:46-53
    int s = 0;
    for (int a = 0; a < d; ++a) {
      if (off[a] < -radius_ || off[a] > radius_) return -1;
      s = s * (2 * radius_ + 1) + (off[a] + radius_);
    }
    return s;
  }
  int diagonal_slot() const { return slot_of(Coord<d>{}); }
  int col(int row, int slot) const { return cols_[static_cast<std::size_t>(row) * nslots_ + slot]; }
  Mat<d>& block(int row, int slot) { return data_[static_cast<std::size_t>(row) * nslots_ + slot]; }
  const Mat<d>& block(int row, int slot) const { return data_[static_cast<std::size_t>(row) * nslots_ + slot]; }

  /// objective.hpp:66-77
  void multiply(const VecX& x, VecX& y) const {
    y.assign(static_cast<std::size_t>(rows_) * d, 0.0);
    parallel_for(rows_, [&](std::int64_t r) {
      Vec<d> acc{};
      for (int s = 0; s < nslots_; ++s) {
        const int c = col(static_cast<int>(r), s);
        if (c < 0) continue;
        acc = acc + block(static_cast<int>(r), s) * seg<d>(x, c);
      }
      set_seg<d>(y, static_cast<int>(r), acc);
    });
  }
  VecX operator*(const VecX& x) const {
    VecX y;
    multiply(x, y);
    return y;
  }
  std::vector<Mat<d>> diagonal_blocks() const {
    std::vector<Mat<d>> diag(rows_);
    const int s = diagonal_slot();
    for (int r = 0; r < rows_; ++r) diag[r] = block(r, s);
    return diag;
  }
  int row_nonzero_blocks(int r) const {
    int n = 0;
    for (int s = 0; s < nslots_; ++s) {
      if (col(r, s) < 0) continue;
      bool nz = false;
      for (double v : block(r, s).a)
        if (v != 0.0) nz = true;
      n += nz;
    }
    return n;
  }
  int max_nonzero_blocks_per_row() const {
    int m = 0;
    for (int r = 0; r < rows_; ++r) m = std::max(m, row_nonzero_blocks(r));
    return m;
  }
  double mean_nonzero_blocks_per_row() const {
    if (rows_ == 0) return 0;
    long t = 0;
    for (int r = 0; r < rows_; ++r) t += row_nonzero_blocks(r);
    return static_cast<double>(t) / rows_;
  }
  double symmetry_error() const {  // objective.hpp:111-124
    double err = 0.0;
    for (int r = 0; r < rows_; ++r)
      for (int s = 0; s < nslots_; ++s) {
        const int c = col(r, s);
        if (c < 0) continue;
        Coord<d> neg;
        for (int a = 0; a < d; ++a) neg[a] = -offsets_[s][a];
        const Mat<d> D = block(r, s) - transpose(block(c, slot_of(neg)));
        for (double v : D.a) err = std::max(err, std::abs(v));
      }
    return err;
  }

 private:
  int rows_ = 0, radius_ = 0, nslots_ = 0;
  std::vector<Coord<d>> offsets_;
  std::vector<int> cols_;
  std::vector<Mat<d>> data_;
};

/// objective.hpp:133-144
template <int d>
void apply_dirichlet_projection(BlockSparseMatrix<d>& H, std::span<const std::uint8_t> dirichlet) {
  const int ds = H.diagonal_slot();
  parallel_for(H.rows(), [&](std::int64_t r) {
    for (int s = 0; s < H.slots(); ++s) {
      const int c = H.col(static_cast<int>(r), s);
      if (c < 0) continue;
      if (dirichlet[r] || dirichlet[c]) H.block(static_cast<int>(r), s) = Mat<d>::zero();
    }
    if (dirichlet[r]) H.block(static_cast<int>(r), ds) = Mat<d>::identity();
  });
}

/// objective.hpp:149-172
template <int d>
struct ObjectiveState {
  static constexpr int stencil_size = ipow(3, d);
  struct ParticleRef {
    double volume = 0;
    Mat<d> F;
    int material = 0;
    double hard = 1.0;  // snow hardening factor exp(xi (1 - J_p)) (extension; 1 in the reference)
    std::array<int, stencil_size> node;
    std::array<double, stencil_size> w;
    std::array<Vec<d>, stencil_size> grad;
  };
  const SparseGrid<d>* grid = nullptr;
  std::vector<ParticleRef> particles;
  std::vector<Material> materials;
  std::vector<double> particle_mass;
  std::vector<double> xi;
  double dt = 0, dx = 0;
  Vec<d> gravity{};
  double cn_length_factor = 24;
  int node_count() const { return grid->node_count(); }
  int dof_count() const { return node_count() * d; }
};

/// objective.hpp:175-212
template <int d>
ObjectiveState<d> make_objective_state(std::span<const Particle<d>> particles, const SparseGrid<d>& grid,
                                       std::span<const Material> materials, double dt, const Vec<d>& gravity,
                                       double cn_length_factor = 24.0) {
  ObjectiveState<d> st;
  st.grid = &grid;
  st.dt = dt;
  st.dx = grid.dx;
  st.gravity = gravity;
  st.cn_length_factor = cn_length_factor;
  st.materials.assign(materials.begin(), materials.end());
  st.xi.resize(st.materials.size());
  for (std::size_t m = 0; m < st.materials.size(); ++m) st.xi[m] = stiffness_scale<d>(st.materials[m]);
  st.particles.resize(particles.size());
  st.particle_mass.resize(particles.size());
  parallel_for(static_cast<std::int64_t>(particles.size()), [&](std::int64_t pi) {
    const auto& p = particles[pi];
    auto& ref = st.particles[pi];
    st.particle_mass[pi] = p.mass;
    ref.volume = p.volume;
    ref.F = p.F;
    ref.material = p.material;
    ref.hard = st.materials[p.material].hardening_factor(p.Jp);
    ref.node.fill(-1);
    ref.w.fill(0.0);
    int k = 0;
    for_each_stencil_node<d>(p.x, grid.dx, grid.kind, [&](const Coord<d>& node, double w, const Vec<d>& grad) {
      ref.node[k] = grid.find(node);
      ref.w[k] = w;
      ref.grad[k] = grad;
      ++k;
    });
  });
  return st;
}

/// objective.hpp:218-230
template <int d>
Mat<d> virtual_f(const ObjectiveState<d>& st, const typename ObjectiveState<d>::ParticleRef& ref, const VecX& dv) {
  Mat<d> G{};
  for (int k = 0; k < ObjectiveState<d>::stencil_size; ++k) {
    const int i = ref.node[k];
    if (i < 0) continue;
    const Vec<d> u = seg<d>(st.grid->velocity, i) + seg<d>(dv, i);
    G = G + outer(u, ref.grad[k]);
  }
  return (Mat<d>::identity() + st.dt * G) * ref.F;
}

/// The particle's material model: fcr_* for the reference's materials (objective.hpp:244, 268,
/// 297); Neo-Hookean and the hardened Lame parameters are the extensions.
template <int d>
double particle_energy_density(const ObjectiveState<d>& st, const typename ObjectiveState<d>::ParticleRef& ref,
                               const Mat<d>& F) {
  const Material& m = st.materials[ref.material];
  return ref.hard == 1.0 ? energy_density<d>(F, m) : energy_density<d>(F, m.hardened(ref.hard));
}
template <int d>
Mat<d> particle_stress(const ObjectiveState<d>& st, const typename ObjectiveState<d>::ParticleRef& ref,
                       const Mat<d>& F) {
  const Material& m = st.materials[ref.material];
  return ref.hard == 1.0 ? stress<d>(F, m) : stress<d>(F, m.hardened(ref.hard));
}
template <int d>
StressDerivative<d> particle_stress_derivative(const ObjectiveState<d>& st,
                                               const typename ObjectiveState<d>::ParticleRef& ref, const Mat<d>& F) {
  const Material& m = st.materials[ref.material];
  return ref.hard == 1.0 ? stress_derivative<d>(F, m) : stress_derivative<d>(F, m.hardened(ref.hard));
}

/// objective.hpp:236-257
template <int d>
double energy(const ObjectiveState<d>& st, const VecX& dv) {
  if (!vfinite(dv)) throw std::invalid_argument("energy: non-finite dv");
  const std::int64_t np = static_cast<std::int64_t>(st.particles.size());
  std::vector<double> phi(np);
  parallel_for(np, [&](std::int64_t pi) {
    const auto& ref = st.particles[pi];
    phi[pi] = ref.volume * particle_energy_density<d>(st, ref, virtual_f(st, ref, dv));
  });
  double e = 0.0;
  for (std::int64_t pi = 0; pi < np; ++pi) e += phi[pi];
  const int n = st.node_count();
  for (int i = 0; i < n; ++i) {
    const Vec<d> dvi = seg<d>(dv, i);
    const Vec<d> u = seg<d>(st.grid->velocity, i) + dvi;
    e += 0.5 * st.grid->mass[i] * squared_norm(dvi);
    e -= st.dt * st.grid->mass[i] * dot(st.gravity, u);
  }
  return e;
}

/// objective.hpp:260-287
template <int d>
VecX gradient(const ObjectiveState<d>& st, const VecX& dv) {
  if (!vfinite(dv)) throw std::invalid_argument("gradient: non-finite dv");
  constexpr int S = ObjectiveState<d>::stencil_size;
  const std::int64_t np = static_cast<std::int64_t>(st.particles.size());
  std::vector<std::array<Vec<d>, S>> contrib(np);
  parallel_for(np, [&](std::int64_t pi) {
    const auto& ref = st.particles[pi];
    const Mat<d> P = particle_stress<d>(st, ref, virtual_f(st, ref, dv));
    const Mat<d> PFt = P * transpose(ref.F);
    for (int k = 0; k < S; ++k)
      contrib[pi][k] = ref.node[k] < 0 ? Vec<d>{} : ref.volume * (PFt * ref.grad[k]);
  });
  const int n = st.node_count();
  VecX g(static_cast<std::size_t>(n) * d, 0.0);
  for (std::int64_t pi = 0; pi < np; ++pi) {
    const auto& ref = st.particles[pi];
    for (int k = 0; k < S; ++k)
      if (ref.node[k] >= 0) add_seg<d>(g, ref.node[k], st.dt * contrib[pi][k]);
  }
  for (int i = 0; i < n; ++i) {
    const Vec<d> t = st.grid->mass[i] * (seg<d>(dv, i) - st.dt * st.gravity);
    add_seg<d>(g, i, t);
    if (st.grid->dirichlet[i]) set_seg<d>(g, i, Vec<d>{});
  }
  return g;
}

/// objective.hpp:293-301
template <int d>
StressDerivative<d> particle_tensor(const ObjectiveState<d>& st, const typename ObjectiveState<d>::ParticleRef& ref,
                                    const VecX& dv, bool project) {
  StressDerivative<d> Tn = particle_stress_derivative<d>(st, ref, virtual_f(st, ref, dv));
  if (project) Tn = project_spd<d * d>(Tn);
  return Tn;
}

/// objective.hpp:304-310: C(c,e) = wa^T T[(c.),(e.)] wb
template <int d>
Mat<d> contract_pair(const StressDerivative<d>& Tn, const Vec<d>& wa, const Vec<d>& wb) {
  constexpr int D = d * d;
  Mat<d> C;
  for (int c = 0; c < d; ++c)
    for (int e = 0; e < d; ++e) {
      Vec<d> tb;  // T.block(c*d, e*d) * wb
      for (int f = 0; f < d; ++f) {
        double s = Tn[(c * d + f) * D + e * d + 0] * wb[0];
        for (int g = 1; g < d; ++g) s += Tn[(c * d + f) * D + e * d + g] * wb[g];
        tb[f] = s;
      }
      C(c, e) = dot(wa, tb);
    }
  return C;
}

/// objective.hpp:318-363
template <int d>
BlockSparseMatrix<d> assemble_hessian(const ObjectiveState<d>& st, const VecX& dv, bool project = true) {
  if (!vfinite(dv)) throw std::invalid_argument("assemble_hessian: non-finite dv");
  constexpr int S = ObjectiveState<d>::stencil_size;
  const std::int64_t np = static_cast<std::int64_t>(st.particles.size());
  std::vector<StressDerivative<d>> tensors(np);
  parallel_for(np, [&](std::int64_t pi) { tensors[pi] = particle_tensor(st, st.particles[pi], dv, project); });
  BlockSparseMatrix<d> H(st.grid->coords, st.grid->index, 2);
  const double kscale = st.dt * st.dt;
  for (std::int64_t pi = 0; pi < np; ++pi) {
    const auto& ref = st.particles[pi];
    std::array<Vec<d>, S> wv;
    const Mat<d> Ft = transpose(ref.F);
    for (int k = 0; k < S; ++k)
      if (ref.node[k] >= 0) wv[k] = Ft * ref.grad[k];
    const double kappa = kscale * ref.volume;
    for (int a = 0; a < S; ++a) {
      const int ia = ref.node[a];
      if (ia < 0) continue;
      for (int b = a; b < S; ++b) {
        const int ib = ref.node[b];
        if (ib < 0) continue;
        Mat<d> C = kappa * contract_pair<d>(tensors[pi], wv[a], wv[b]);
        const Coord<d> off = st.grid->coords[ib] - st.grid->coords[ia];
        const int s_ab = H.slot_of(off);
        if (a == b) {
          C = 0.5 * (C + transpose(C));
          H.block(ia, s_ab) = H.block(ia, s_ab) + C;
        } else {
          H.block(ia, s_ab) = H.block(ia, s_ab) + C;
          Coord<d> neg;
          for (int ax = 0; ax < d; ++ax) neg[ax] = -off[ax];
          const int s_ba = H.slot_of(neg);
          H.block(ib, s_ba) = H.block(ib, s_ba) + transpose(C);
        }
      }
    }
  }
  const int ds = H.diagonal_slot();
  for (int i = 0; i < st.node_count(); ++i) H.block(i, ds) = H.block(i, ds) + st.grid->mass[i] * Mat<d>::identity();
  apply_dirichlet_projection<d>(H, st.grid->dirichlet);
  return H;
}

/// objective.hpp:368-396
template <int d>
std::vector<Mat<d>> assemble_block_diagonal(const ObjectiveState<d>& st, const VecX& dv, bool project = true) {
  constexpr int S = ObjectiveState<d>::stencil_size;
  const std::int64_t np = static_cast<std::int64_t>(st.particles.size());
  std::vector<std::array<Mat<d>, S>> contrib(np);
  parallel_for(np, [&](std::int64_t pi) {
    const auto& ref = st.particles[pi];
    const StressDerivative<d> Tn = particle_tensor(st, ref, dv, project);
    const double kappa = st.dt * st.dt * ref.volume;
    const Mat<d> Ft = transpose(ref.F);
    for (int k = 0; k < S; ++k) {
      if (ref.node[k] < 0) continue;
      const Vec<d> wv = Ft * ref.grad[k];
      const Mat<d> C = kappa * contract_pair<d>(Tn, wv, wv);
      contrib[pi][k] = 0.5 * (C + transpose(C));
    }
  });
  std::vector<Mat<d>> diag(st.node_count(), Mat<d>::zero());
  for (std::int64_t pi = 0; pi < np; ++pi) {
    const auto& ref = st.particles[pi];
    for (int k = 0; k < S; ++k)
      if (ref.node[k] >= 0) diag[ref.node[k]] = diag[ref.node[k]] + contrib[pi][k];
  }
  for (int i = 0; i < st.node_count(); ++i) {
    diag[i] = diag[i] + st.grid->mass[i] * Mat<d>::identity();
    if (st.grid->dirichlet[i]) diag[i] = Mat<d>::identity();
  }
  return diag;
}

/// objective.hpp:401-440
template <int d>
VecX multiply_matrix_free(const ObjectiveState<d>& st, const VecX& dv, const VecX& u, bool project = true) {
  constexpr int S = ObjectiveState<d>::stencil_size;
  constexpr int D = d * d;
  const int n = st.node_count();
  VecX um = u;
  for (int i = 0; i < n; ++i)
    if (st.grid->dirichlet[i]) set_seg<d>(um, i, Vec<d>{});
  const std::int64_t np = static_cast<std::int64_t>(st.particles.size());
  std::vector<std::array<Vec<d>, S>> contrib(np);
  parallel_for(np, [&](std::int64_t pi) {
    const auto& ref = st.particles[pi];
    const StressDerivative<d> Tn = particle_tensor(st, ref, dv, project);
    std::array<Vec<d>, S> wv;
    Mat<d> dF{};
    const Mat<d> Ft = transpose(ref.F);
    for (int k = 0; k < S; ++k) {
      if (ref.node[k] < 0) continue;
      wv[k] = Ft * ref.grad[k];
      dF = dF + outer(seg<d>(um, ref.node[k]), wv[k]);
    }
    Mat<d> dP;
    for (int r = 0; r < D; ++r) {
      double acc = Tn[r * D] * dF.a[0];
      for (int c = 1; c < D; ++c) acc += Tn[r * D + c] * dF.a[c];
      dP.a[r] = acc;
    }
    const double kappa = st.dt * st.dt * ref.volume;
    for (int k = 0; k < S; ++k) contrib[pi][k] = ref.node[k] < 0 ? Vec<d>{} : kappa * (dP * wv[k]);
  });
  VecX y(static_cast<std::size_t>(n) * d, 0.0);
  for (std::int64_t pi = 0; pi < np; ++pi) {
    const auto& ref = st.particles[pi];
    for (int k = 0; k < S; ++k)
      if (ref.node[k] >= 0) add_seg<d>(y, ref.node[k], contrib[pi][k]);
  }
  for (int i = 0; i < n; ++i) {
    if (st.grid->dirichlet[i])
      set_seg<d>(y, i, seg<d>(u, i));
    else
      add_seg<d>(y, i, st.grid->mass[i] * seg<d>(um, i));
  }
  return y;
}

/// objective.hpp:445-448
struct NodeCN {
  VecX xi, scale;
};

/// objective.hpp:450-473
template <int d>
NodeCN compute_node_cn(const ObjectiveState<d>& st) {
  const int n = st.node_count();
  VecX num(n, 0.0), den(n, 0.0);
  constexpr int S = ObjectiveState<d>::stencil_size;
  for (std::size_t pi = 0; pi < st.particles.size(); ++pi) {
    const auto& ref = st.particles[pi];
    const double mx = st.particle_mass[pi] * st.xi[ref.material];
    for (int k = 0; k < S; ++k) {
      if (ref.node[k] < 0) continue;
      num[ref.node[k]] += ref.w[k] * mx;
      den[ref.node[k]] += ref.w[k] * st.particle_mass[pi];
    }
  }
  NodeCN cn;
  cn.xi.assign(n, 0.0);
  cn.scale.assign(n, 0.0);
  const double ell = st.cn_length_factor * st.dx * st.dx;
  for (int i = 0; i < n; ++i) {
    if (den[i] > 0.0) cn.xi[i] = num[i] / den[i];
    cn.scale[i] = ell * cn.xi[i] * st.dt;
  }
  return cn;
}

/// objective.hpp:476-486
template <int d>
double scaled_norm(const VecX& g, const NodeCN& cn) {
  const int n = static_cast<int>(cn.scale.size());
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!(cn.scale[i] > 0.0))
      throw std::logic_error("scaled_norm: zero characteristic scale (material misconfiguration)");
    acc += squared_norm(seg<d>(g, i)) / (cn.scale[i] * cn.scale[i]);
  }
  return std::sqrt(acc);
}

// ---------------------------------------------------------------------------------------
// pcg.hpp
// ---------------------------------------------------------------------------------------

struct PcgResult {
  VecX x;
  int iterations = 0;
  bool converged = true;
};

/// pcg.hpp:17-46
template <typename ApplyA, typename ApplyP>
PcgResult pcg(ApplyA&& apply_a, ApplyP&& apply_p, const VecX& b, double rel_tol, int cap) {
  PcgResult res;
  res.x.assign(b.size(), 0.0);
  VecX r = b;
  VecX z = apply_p(r);
  double rho = vdot(r, z);
  if (!(rho > 0.0)) {
    if (rho < 0.0) throw SolverFailure("pcg: preconditioner is not positive definite");
    return res;
  }
  const double threshold = rel_tol * rel_tol * rho;
  VecX p = z;
  for (int it = 0; it < cap; ++it) {
    const VecX Ap = apply_a(p);
    const double pAp = vdot(p, Ap);
    if (!(pAp > 0.0)) throw SolverFailure("pcg: system matrix is not positive definite");
    const double alpha = rho / pAp;
    for (std::size_t k = 0; k < b.size(); ++k) res.x[k] += alpha * p[k];
    for (std::size_t k = 0; k < b.size(); ++k) r[k] -= alpha * Ap[k];
    z = apply_p(r);
    const double rho_new = vdot(r, z);
    res.iterations = it + 1;
    if (rho_new <= threshold) return res;
    const double beta = rho_new / rho;
    for (std::size_t k = 0; k < b.size(); ++k) p[k] = z[k] + beta * p[k];
    rho = rho_new;
  }
  res.converged = false;
  return res;
}

// ---------------------------------------------------------------------------------------
// multigrid.hpp
// ---------------------------------------------------------------------------------------

/// multigrid.hpp:14-46
template <int d>
struct RestrictionOperator {
  struct Entry {
    int coarse;
    double weight;
  };
  std::vector<int> row_start;
  std::vector<Entry> entries;
  int fine_nodes = 0, coarse_nodes = 0;

  void restrict_to_coarse(const VecX& fine, VecX& coarse) const {
    coarse.assign(static_cast<std::size_t>(coarse_nodes) * d, 0.0);
    for (int i = 0; i < fine_nodes; ++i)
      for (int e = row_start[i]; e < row_start[i + 1]; ++e)
        add_seg<d>(coarse, entries[e].coarse, entries[e].weight * seg<d>(fine, i));
  }
  void prolong_add(const VecX& coarse, VecX& fine) const {
    parallel_for(fine_nodes, [&](std::int64_t i) {
      Vec<d> acc{};
      for (int e = row_start[i]; e < row_start[i + 1]; ++e)
        acc = acc + entries[e].weight * seg<d>(coarse, entries[e].coarse);
      add_seg<d>(fine, static_cast<int>(i), acc);
    });
  }
  int max_entries_per_fine_node() const {
    int m = 0;
    for (int i = 0; i < fine_nodes; ++i) m = std::max(m, row_start[i + 1] - row_start[i]);
    return m;
  }
};

/// multigrid.hpp:50-57
template <int d>
struct GridLevelInfo {
  std::vector<Coord<d>> coords;
  CoordIndex<d> index;
  std::vector<std::uint8_t> dirichlet;
  int node_count() const { return static_cast<int>(coords.size()); }
};

inline int floor_div2(int x) { return x >= 0 ? x / 2 : (x - 1) / 2; }  // multigrid.hpp:61

/// multigrid.hpp:64-95
inline void embedding_entries_1d(KernelKind kind, int c, int out_coord[3], double out_w[3], int& count) {
  count = 0;
  if (kind == KernelKind::Linear) {
    const int base = floor_div2(c);
    if (c % 2 == 0) {
      out_coord[count] = base;
      out_w[count++] = 1.0;
    } else {
      out_coord[count] = base;
      out_w[count++] = 0.5;
      out_coord[count] = base + 1;
      out_w[count++] = 0.5;
    }
  } else {
    if (c % 2 == 0) {
      const int mid = c / 2;
      out_coord[count] = mid - 1;
      out_w[count++] = 0.125;
      out_coord[count] = mid;
      out_w[count++] = 0.75;
      out_coord[count] = mid + 1;
      out_w[count++] = 0.125;
    } else {
      const int base = floor_div2(c);
      out_coord[count] = base;
      out_w[count++] = 0.5;
      out_coord[count] = base + 1;
      out_w[count++] = 0.5;
    }
  }
}

/// multigrid.hpp:98-123
template <int d, typename Fn>
void for_each_embedding(KernelKind kind, const Coord<d>& c, Fn&& fn) {
  int coord[d][3];
  double w[d][3];
  int count[d];
  for (int a = 0; a < d; ++a) embedding_entries_1d(kind, c[a], coord[a], w[a], count[a]);
  int pick[d] = {};
  while (true) {
    Coord<d> J;
    double weight = 1.0;
    for (int a = 0; a < d; ++a) {
      J[a] = coord[a][pick[a]];
      weight *= w[a][pick[a]];
    }
    fn(J, weight);
    int a = d - 1;
    while (a >= 0) {
      if (++pick[a] < count[a]) break;
      pick[a] = 0;
      --a;
    }
    if (a < 0) break;
  }
}

/// multigrid.hpp:127-158
template <int d>
std::pair<GridLevelInfo<d>, RestrictionOperator<d>> build_restriction(const GridLevelInfo<d>& fine, KernelKind embedding) {
  const int nf = fine.node_count();
  std::vector<Coord<d>> cc;
  for (int i = 0; i < nf; ++i)
    for_each_embedding<d>(embedding, fine.coords[i], [&](const Coord<d>& J, double) { cc.push_back(J); });
  std::sort(cc.begin(), cc.end());
  cc.erase(std::unique(cc.begin(), cc.end()), cc.end());
  GridLevelInfo<d> coarse;
  coarse.coords = std::move(cc);
  coarse.index.reserve(coarse.coords.size());
  for (int j = 0; j < coarse.node_count(); ++j) coarse.index.emplace(coarse.coords[j], j);
  coarse.dirichlet.assign(coarse.node_count(), 0);
  RestrictionOperator<d> R;
  R.fine_nodes = nf;
  R.coarse_nodes = coarse.node_count();
  R.row_start.assign(nf + 1, 0);
  for (int i = 0; i < nf; ++i) {
    for_each_embedding<d>(embedding, fine.coords[i], [&](const Coord<d>& J, double w) {
      R.entries.push_back({coarse.index.at(J), w});
      if (fine.dirichlet[i]) coarse.dirichlet[coarse.index.at(J)] = 1;
    });
    R.row_start[i + 1] = static_cast<int>(R.entries.size());
  }
  return {std::move(coarse), std::move(R)};
}

/// multigrid.hpp:162-202: H_coarse = R H R^T, pairs visited once and mirrored.
template <int d>
BlockSparseMatrix<d> galerkin_coarsen(const BlockSparseMatrix<d>& Hf, const RestrictionOperator<d>& R,
                                      const GridLevelInfo<d>& /*fine*/, const GridLevelInfo<d>& coarse, int coarse_radius) {
  BlockSparseMatrix<d> Hc(coarse.coords, coarse.index, coarse_radius);
  for (int i = 0; i < Hf.rows(); ++i) {
    for (int s = 0; s < Hf.slots(); ++s) {
      const int l = Hf.col(i, s);
      if (l < i) continue;
      if (l < 0) continue;
      const Mat<d>& B = Hf.block(i, s);
      for (int ea = R.row_start[i]; ea < R.row_start[i + 1]; ++ea) {
        for (int eb = R.row_start[l]; eb < R.row_start[l + 1]; ++eb) {
          const auto& A = R.entries[ea];
          const auto& E = R.entries[eb];
          const double scale = A.weight * E.weight;
          const Coord<d> off = coarse.coords[E.coarse] - coarse.coords[A.coarse];
          const int slot = Hc.slot_of(off);
          if (slot < 0) throw std::logic_error("galerkin_coarsen: coarse stencil overflow (kernel misconfiguration)");
          if (i == l) {
            Hc.block(A.coarse, slot) = Hc.block(A.coarse, slot) + scale * B;
          } else if (A.coarse == E.coarse) {
            const Mat<d> C = scale * B;
            Hc.block(A.coarse, slot) = Hc.block(A.coarse, slot) + (C + transpose(C));
          } else {
            Coord<d> neg;
            for (int a = 0; a < d; ++a) neg[a] = -off[a];
            Hc.block(A.coarse, slot) = Hc.block(A.coarse, slot) + scale * B;
            const int sn = Hc.slot_of(neg);
            Hc.block(E.coarse, sn) = Hc.block(E.coarse, sn) + scale * transpose(B);
          }
        }
      }
    }
  }
  return Hc;
}

/// multigrid.hpp:205-214
template <int d>
struct MgLevel {
  GridLevelInfo<d> info;
  const BlockSparseMatrix<d>* H = nullptr;
  std::unique_ptr<BlockSparseMatrix<d>> owned;
  std::vector<Mat<d>> diag, diag_inv;
  std::vector<int> sweep_order;
  RestrictionOperator<d> R;
};

/// multigrid.hpp:216-223
template <int d>
struct MultigridHierarchy {
  std::vector<MgLevel<d>> levels;
  KernelKind embedding = KernelKind::Linear;
  int coarse_cg_cap = 10000;
  bool truncated = false;
  int level_count() const { return static_cast<int>(levels.size()); }
};

/// multigrid.hpp:227-251
template <int d>
void finalize_level(MgLevel<d>& lvl, int q) {
  const auto& H = *lvl.H;
  const int n = H.rows();
  const int ds = H.diagonal_slot();
  lvl.diag.resize(n);
  lvl.diag_inv.resize(n);
  for (int i = 0; i < n; ++i) {
    lvl.diag[i] = H.block(i, ds);
    const double det = determinant(lvl.diag[i]);
    if (!(std::abs(det) > 0.0)) throw std::logic_error("multigrid: singular diagonal block");
    lvl.diag_inv[i] = inverse(lvl.diag[i]);
  }
  auto color_of = [&](const Coord<d>& c) {
    int col = 0;
    for (int a = 0; a < d; ++a) col = col * q + ((c[a] % q) + q) % q;
    return col;
  };
  lvl.sweep_order.resize(n);
  for (int i = 0; i < n; ++i) lvl.sweep_order[i] = i;
  std::stable_sort(lvl.sweep_order.begin(), lvl.sweep_order.end(),
                   [&](int a, int b) { return color_of(lvl.info.coords[a]) < color_of(lvl.info.coords[b]); });
}

/// multigrid.hpp:258-294
template <int d>
MultigridHierarchy<d> build_hierarchy(const BlockSparseMatrix<d>& H0, const SparseGrid<d>& grid0, int level_count,
                                      KernelKind embedding) {
  if (level_count < 1) throw std::invalid_argument("build_hierarchy: need at least one level");
  MultigridHierarchy<d> hier;
  hier.embedding = embedding;
  {
    MgLevel<d> l0;
    l0.info.coords = grid0.coords;
    l0.info.index = grid0.index;
    l0.info.dirichlet = grid0.dirichlet;
    l0.H = &H0;
    finalize_level(l0, 3);
    hier.levels.push_back(std::move(l0));
  }
  const int coarse_radius = embedding == KernelKind::Linear ? 2 : 3;
  const int coarse_modulus = embedding == KernelKind::Linear ? 2 : 3;
  for (int m = 1; m < level_count; ++m) {
    auto& fine = hier.levels.back();
    auto [coarse_info, R] = build_restriction<d>(fine.info, embedding);
    if (coarse_info.node_count() == 0) {
      hier.truncated = true;
      break;
    }
    fine.R = std::move(R);
    MgLevel<d> lvl;
    lvl.owned = std::make_unique<BlockSparseMatrix<d>>(galerkin_coarsen<d>(*fine.H, fine.R, fine.info, coarse_info, coarse_radius));
    apply_dirichlet_projection<d>(*lvl.owned, coarse_info.dirichlet);
    lvl.H = lvl.owned.get();
    lvl.info = std::move(coarse_info);
    finalize_level(lvl, coarse_modulus);
    hier.levels.push_back(std::move(lvl));
  }
  return hier;
}

/// multigrid.hpp:298-316
template <int d>
void smooth_sgs(const BlockSparseMatrix<d>& H, std::span<const Mat<d>> diag_inv, std::span<const int> order, VecX& u,
                const VecX& b, int sweeps = 1) {
  const int n = H.rows();
  auto update = [&](int i) {
    Vec<d> r = seg<d>(b, i);
    for (int s = 0; s < H.slots(); ++s) {
      const int c = H.col(i, s);
      if (c < 0) continue;
      r = r - H.block(i, s) * seg<d>(u, c);
    }
    add_seg<d>(u, i, diag_inv[i] * r);
  };
  for (int sweep = 0; sweep < sweeps; ++sweep) {
    for (int k = 0; k < n; ++k) update(order[k]);
    for (int k = n - 1; k >= 0; --k) update(order[k]);
  }
}

struct CoarseSolveMode {  // multigrid.hpp:318-322
  bool pinned = false;
  int pinned_cap = 256;
};

struct CoarseSolveResult {
  VecX u;
  int iterations = 0;
  bool converged = true;
};

/// multigrid.hpp:334-350
template <int d>
CoarseSolveResult coarse_solve(const BlockSparseMatrix<d>& H, std::span<const Mat<d>> diag_inv, const VecX& b,
                               const CoarseSolveMode& mode, int cap = 10000) {
  auto apply_a = [&](const VecX& x) { return H * x; };
  auto apply_p = [&](const VecX& r) {
    VecX z(r.size());
    const int n = H.rows();
    for (int i = 0; i < n; ++i) set_seg<d>(z, i, diag_inv[i] * seg<d>(r, i));
    return z;
  };
  const double rel = mode.pinned ? 1e-14 : 0.5;
  const int iters = mode.pinned ? mode.pinned_cap : cap;
  PcgResult res = pcg(apply_a, apply_p, b, rel, iters);
  return {std::move(res.x), res.iterations, res.converged || mode.pinned};
}

struct VCycleResult {
  VecX u;
  int coarse_iterations = 0;
  bool coarse_converged = true;
};

/// multigrid.hpp:363-392 (Alg. 2)
template <int d>
VCycleResult vcycle(const MultigridHierarchy<d>& hier, const VecX& b0, const CoarseSolveMode& mode = {}) {
  const int M = hier.level_count();
  std::vector<VecX> b(M), u(M);
  b[0] = b0;
  auto zero_dirichlet = [&](int m, VecX& x) {
    const auto& dir = hier.levels[m].info.dirichlet;
    for (int i = 0; i < static_cast<int>(dir.size()); ++i)
      if (dir[i]) set_seg<d>(x, i, Vec<d>{});
  };
  zero_dirichlet(0, b[0]);
  for (int m = 0; m < M - 1; ++m) {
    const auto& lvl = hier.levels[m];
    u[m].assign(b[m].size(), 0.0);
    smooth_sgs<d>(*lvl.H, lvl.diag_inv, lvl.sweep_order, u[m], b[m]);
    const VecX Hu = *lvl.H * u[m];
    VecX residual(b[m].size());
    for (std::size_t k = 0; k < residual.size(); ++k) residual[k] = b[m][k] - Hu[k];
    lvl.R.restrict_to_coarse(residual, b[m + 1]);
    zero_dirichlet(m + 1, b[m + 1]);
  }
  const auto& bottom = hier.levels[M - 1];
  auto cs = coarse_solve<d>(*bottom.H, bottom.diag_inv, b[M - 1], mode, hier.coarse_cg_cap);
  u[M - 1] = std::move(cs.u);
  for (int m = M - 2; m >= 0; --m) {
    const auto& lvl = hier.levels[m];
    lvl.R.prolong_add(u[m + 1], u[m]);
    smooth_sgs<d>(*lvl.H, lvl.diag_inv, lvl.sweep_order, u[m], b[m]);
  }
  return {std::move(u[0]), cs.iterations, cs.converged};
}

// ---------------------------------------------------------------------------------------
// solvers.hpp
// ---------------------------------------------------------------------------------------

enum class SolverKind { Hot = 0, PnPcg = 1, PnPcgMatrixFree = 2, PnMgpcg = 3, LbfgsH = 4 };

struct SolverConfig {  // solvers.hpp:14-29
  double epsilon = 1e-7;
  double tau = 1e-4;
  int levels = 3;
  int window = 8;
  double ls_shrink = 0.5;
  double ls_armijo = 1e-4;
  int ls_max_steps = 30;
  int cg_cap = 10000;
  int outer_cap = 1000;
  SolverKind kind = SolverKind::Hot;
  KernelKind embedding = KernelKind::Linear;
  int pinned_coarse_iterations = 256;
  double cn_length_factor = 24;
};

struct DiagnosticsRecord {  // solvers.hpp:31-41
  int frame = 0;
  long step = 0;
  int outer_iteration = 0;
  double scaled_residual = 0, energy = 0, step_length = 0;
  long inner_iterations = 0, work_units = 0;
  double wall_ms = 0;
};

struct SolveResult {  // solvers.hpp:43-50
  VecX dv;
  int outer_iterations = 0;
  long inner_total = 0;
  int hierarchy_rebuilds = 0;
  bool converged = false;
};

struct LineSearchResult {
  double alpha, energy;
  int evaluations;
};

/// solvers.hpp:59-62
inline double adaptive_cg_tolerance(double pe_sq, double tau) {
  return std::min(0.5, std::sqrt(std::max(std::sqrt(pe_sq), tau)));
}

/// solvers.hpp:66-78
template <typename EnergyFn>
LineSearchResult line_search(EnergyFn&& energy_at, double e0, double gdotp, const SolverConfig& cfg) {
  if (!(gdotp < 0.0)) throw SolverFailure("line_search: not a descent direction");
  double alpha = 1.0;
  for (int k = 0; k < cfg.ls_max_steps; ++k) {
    const double e = energy_at(alpha);
    if (e <= e0 + cfg.ls_armijo * alpha * gdotp) return {alpha, e, k + 1};
    alpha *= cfg.ls_shrink;
  }
  throw SolverFailure("line_search: no acceptable step (gradient/Hessian inconsistency)");
}

/// solvers.hpp:82-110
class LBFGSHistory {
 public:
  explicit LBFGSHistory(int window) : window_(window < 1 ? 1 : window) {}
  bool push(VecX s, VecX y) {
    const double ys = vdot(y, s);
    if (!(ys > 1e-12 * vnorm(y) * vnorm(s))) return false;
    if (static_cast<int>(entries_.size()) == window_) entries_.pop_front();
    entries_.push_back({std::move(s), std::move(y), 1.0 / ys});
    return true;
  }
  int size() const { return static_cast<int>(entries_.size()); }
  void clear() { entries_.clear(); }
  const VecX& s(int k) const { return entries_[entries_.size() - 1 - k].s; }
  const VecX& y(int k) const { return entries_[entries_.size() - 1 - k].y; }
  double rho(int k) const { return entries_[entries_.size() - 1 - k].rho; }

 private:
  struct Entry {
    VecX s, y;
    double rho;
  };
  int window_;
  std::deque<Entry> entries_;
};

/// solvers.hpp:114-129
template <typename Init>
VecX lbfgs_direction(const VecX& g, const LBFGSHistory& h, Init&& initializer) {
  VecX q(g.size());
  for (std::size_t k = 0; k < g.size(); ++k) q[k] = -g[k];
  const int m = h.size();
  std::vector<double> alpha(m);
  for (int k = 0; k < m; ++k) {
    alpha[k] = h.rho(k) * vdot(h.s(k), q);
    const VecX& y = h.y(k);
    for (std::size_t i = 0; i < q.size(); ++i) q[i] -= alpha[k] * y[i];
  }
  VecX r = initializer(q);
  for (int k = m - 1; k >= 0; --k) {
    const double beta = h.rho(k) * vdot(h.y(k), r);
    const VecX& s = h.s(k);
    for (std::size_t i = 0; i < r.size(); ++i) r[i] += (alpha[k] - beta) * s[i];
  }
  return r;
}

/// Phase timing of the oracle (diagnostics only; HOT_ORACLE_TIMING=1 prints per-phase wall time
/// of every advance_step to stderr).  No effect on any value.
struct OracleTimer {
  bool on = std::getenv("HOT_ORACLE_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[oracle] %-16s %9.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

inline double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

/// solvers.hpp:137-187
template <int d>
struct OuterLoop {
  const ObjectiveState<d>& st;
  const SolverConfig& cfg;
  std::vector<DiagnosticsRecord>* diagnostics;
  int frame;
  long step;
  NodeCN cn;
  double target;
  VecX dv, g;
  double e_curr, residual;
  long work = 0;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();

  OuterLoop(const ObjectiveState<d>& state, const SolverConfig& config, std::vector<DiagnosticsRecord>* diag, int f, long s)
      : st(state), cfg(config), diagnostics(diag), frame(f), step(s) {
    cn = compute_node_cn(st);
    target = cfg.epsilon * std::sqrt(static_cast<double>(st.node_count()));
    dv.assign(st.dof_count(), 0.0);
    g = gradient(st, dv);
    e_curr = energy(st, dv);
    residual = scaled_norm<d>(g, cn);
  }
  bool done() const { return residual <= target; }

  std::pair<VecX, VecX> accept(const VecX& p, int outer, long inner_this) {
    const double gdotp = vdot(g, p);
    VecX trial(dv.size());
    auto ls = line_search(
        [&](double a) {
          for (std::size_t k = 0; k < dv.size(); ++k) trial[k] = dv[k] + a * p[k];
          return energy(st, trial);
        },
        e_curr, gdotp, cfg);
    VecX s(p.size());
    for (std::size_t k = 0; k < p.size(); ++k) s[k] = ls.alpha * p[k];
    for (std::size_t k = 0; k < p.size(); ++k) dv[k] += s[k];
    VecX g_new = gradient(st, dv);
    VecX y(g.size());
    for (std::size_t k = 0; k < g.size(); ++k) y[k] = g_new[k] - g[k];
    g = std::move(g_new);
    e_curr = ls.energy;
    residual = scaled_norm<d>(g, cn);
    work += inner_this;
    if (diagnostics)
      diagnostics->push_back({frame, step, outer, residual, e_curr, ls.alpha, inner_this, work, ms_since(t0)});
    return {std::move(s), std::move(y)};
  }
};

/// solvers.hpp:191-231
template <int d>
SolveResult solve_quasi_newton(const ObjectiveState<d>& st, const SolverConfig& cfg, int levels,
                               std::vector<DiagnosticsRecord>* diag, int frame, long step) {
  OuterLoop<d> loop(st, cfg, diag, frame, step);
  SolveResult out;
  if (loop.done()) {
    out.dv = std::move(loop.dv);
    out.converged = true;
    return out;
  }
  OracleTimer tm;
  const BlockSparseMatrix<d> H = assemble_hessian<d>(st, loop.dv, true);
  tm.lap("  assemble");
  const MultigridHierarchy<d> hier = build_hierarchy<d>(H, *st.grid, levels, cfg.embedding);
  tm.lap("  hierarchy");
  out.hierarchy_rebuilds = 1;
  LBFGSHistory history(cfg.window);
  for (int outer = 1; outer <= cfg.outer_cap; ++outer) {
    long inner_this = 0;
    auto initializer = [&](const VecX& q) {
      auto v = vcycle<d>(hier, q, CoarseSolveMode{false, 0});
      inner_this += v.coarse_iterations;
      return v.u;
    };
    const VecX p = lbfgs_direction(loop.g, history, initializer);
    tm.lap("  direction");
    auto [s, y] = loop.accept(p, outer, inner_this);
    tm.lap("  accept");
    history.push(std::move(s), std::move(y));
    out.outer_iterations = outer;
    out.inner_total += inner_this;
    if (loop.done()) {
      out.converged = true;
      break;
    }
  }
  if (!out.converged)
    throw SolverFailure("quasi-newton solve: outer iteration cap reached (residual " + std::to_string(loop.residual) + ")");
  out.dv = std::move(loop.dv);
  return out;
}

enum class PnVariant { Assembled, MatrixFree, Multigrid };

/// solvers.hpp:235-310
template <int d>
SolveResult solve_projected_newton(const ObjectiveState<d>& st, const SolverConfig& cfg, PnVariant variant,
                                   std::vector<DiagnosticsRecord>* diag, int frame, long step) {
  OuterLoop<d> loop(st, cfg, diag, frame, step);
  SolveResult out;
  if (loop.done()) {
    out.dv = std::move(loop.dv);
    out.converged = true;
    return out;
  }
  const int n = st.node_count();
  for (int outer = 1; outer <= cfg.outer_cap; ++outer) {
    BlockSparseMatrix<d> H;
    std::vector<Mat<d>> diag_blocks;
    MultigridHierarchy<d> hier;
    if (variant == PnVariant::MatrixFree) {
      diag_blocks = assemble_block_diagonal<d>(st, loop.dv, true);
    } else {
      H = assemble_hessian<d>(st, loop.dv, true);
      diag_blocks = H.diagonal_blocks();
      if (variant == PnVariant::Multigrid) {
        hier = build_hierarchy<d>(H, *st.grid, cfg.levels, cfg.embedding);
        ++out.hierarchy_rebuilds;
      }
    }
    std::vector<Mat<d>> diag_inv(diag_blocks.size());
    for (std::size_t i = 0; i < diag_blocks.size(); ++i) diag_inv[i] = inverse(diag_blocks[i]);
    double gpg = 0.0;
    for (int i = 0; i < n; ++i) {
      const Vec<d> gi = seg<d>(loop.g, i);
      gpg += dot(gi, diag_inv[i] * gi);
    }
    const double k = adaptive_cg_tolerance(gpg, cfg.tau);
    long inner_this = 0;
    auto apply_jacobi = [&](const VecX& r) {
      VecX z(r.size());
      for (int i = 0; i < n; ++i) set_seg<d>(z, i, diag_inv[i] * seg<d>(r, i));
      return z;
    };
    PcgResult pr;
    VecX rhs(loop.g.size());
    for (std::size_t q = 0; q < rhs.size(); ++q) rhs[q] = -loop.g[q];
    if (variant == PnVariant::MatrixFree) {
      pr = pcg([&](const VecX& x) { return multiply_matrix_free<d>(st, loop.dv, x); }, apply_jacobi, rhs, k, cfg.cg_cap);
      inner_this = pr.iterations;
    } else if (variant == PnVariant::Assembled) {
      pr = pcg([&](const VecX& x) { return H * x; }, apply_jacobi, rhs, k, cfg.cg_cap);
      inner_this = pr.iterations;
    } else {
      auto apply_vcycle = [&](const VecX& r) {
        auto v = vcycle<d>(hier, r, CoarseSolveMode{true, cfg.pinned_coarse_iterations});
        inner_this += v.coarse_iterations;
        return v.u;
      };
      pr = pcg([&](const VecX& x) { return H * x; }, apply_vcycle, rhs, k, cfg.cg_cap);
      inner_this += pr.iterations;
    }
    loop.accept(pr.x, outer, inner_this);
    out.outer_iterations = outer;
    out.inner_total += inner_this;
    if (loop.done()) {
      out.converged = true;
      break;
    }
  }
  if (!out.converged)
    throw SolverFailure("projected newton solve: outer iteration cap reached (residual " + std::to_string(loop.residual) + ")");
  out.dv = std::move(loop.dv);
  return out;
}

template <int d>
SolveResult solve_hot(const ObjectiveState<d>& st, const SolverConfig& cfg, std::vector<DiagnosticsRecord>* diag = nullptr,
                      int frame = 0, long step = 0) {  // solvers.hpp:314-319
  return solve_quasi_newton<d>(st, cfg, cfg.levels, diag, frame, step);
}
template <int d>
SolveResult solve_lbfgs_h(const ObjectiveState<d>& st, const SolverConfig& cfg, std::vector<DiagnosticsRecord>* diag = nullptr,
                          int frame = 0, long step = 0) {  // solvers.hpp:321-326
  return solve_quasi_newton<d>(st, cfg, 1, diag, frame, step);
}

template <int d>
struct GridStepResult {
  VecX velocity;
  SolveResult solve;
};

/// solvers.hpp:354-381
template <int d>
GridStepResult<d> step_grid(const ObjectiveState<d>& st, const SolverConfig& cfg, std::vector<DiagnosticsRecord>* diag = nullptr,
                            int frame = 0, long step = 0) {
  GridStepResult<d> out;
  switch (cfg.kind) {
    case SolverKind::Hot:
      out.solve = solve_hot<d>(st, cfg, diag, frame, step);
      break;
    case SolverKind::LbfgsH:
      out.solve = solve_lbfgs_h<d>(st, cfg, diag, frame, step);
      break;
    case SolverKind::PnPcg:
      out.solve = solve_projected_newton<d>(st, cfg, PnVariant::Assembled, diag, frame, step);
      break;
    case SolverKind::PnPcgMatrixFree:
      out.solve = solve_projected_newton<d>(st, cfg, PnVariant::MatrixFree, diag, frame, step);
      break;
    case SolverKind::PnMgpcg:
      out.solve = solve_projected_newton<d>(st, cfg, PnVariant::Multigrid, diag, frame, step);
      break;
  }
  out.velocity.resize(st.grid->velocity.size());
  for (std::size_t k = 0; k < out.velocity.size(); ++k) out.velocity[k] = st.grid->velocity[k] + out.solve.dv[k];
  for (int i = 0; i < st.node_count(); ++i)
    if (st.grid->dirichlet[i]) set_seg<d>(out.velocity, i, seg<d>(st.grid->bc_velocity, i));
  return out;
}

// ---------------------------------------------------------------------------------------
// scene.hpp (plain data) + simulation.hpp
// ---------------------------------------------------------------------------------------

struct ShapeSpec {  // scene.hpp:25-32
  enum class Kind { Box = 0, Sphere = 1, HalfSpace = 2, Cylinder = 3 } kind = Kind::Box;
  std::array<double, 3> min{}, max{}, center{};
  double radius = 0;
  std::array<double, 3> point{}, normal{}, axis{};
};
struct MotionSpec {  // scene.hpp:34-40
  enum class Kind { Static = 0, Linear = 1, Rotation = 2 } kind = Kind::Static;
  std::array<double, 3> velocity{}, center{}, axis{};
  double omega = 0;
};
struct InitialDeformationSpec {  // scene.hpp:42-45
  enum class Kind { Identity = 0, RandomDiagonal = 1 } kind = Kind::Identity;
  double lo = 1, hi = 1;
};
struct MaterialSpec {  // scene.hpp:13-23
  double density = 0, youngs = 0, poisson = 0;
  PlasticityKind plasticity = PlasticityKind::None;
  double yield_stress = 0, clamp_lo = 0.99, clamp_hi = 1.001;
  // extensions: elastic model, snow hardening, Drucker-Prager friction angle
  ElasticityKind elasticity = ElasticityKind::FixedCorotated;
  double hardening = 0, friction_angle = 0;
};
struct ObjectSpec {
  ShapeSpec shape;
  int material = 0;
  std::array<double, 3> velocity{};
  InitialDeformationSpec initial_deformation;
};
struct ColliderSpec {
  ShapeSpec shape;
  MotionSpec motion;
};
struct SceneConfig {  // scene.hpp:61-84
  int dim = 2;
  double dx = 0.01;
  std::array<double, 3> gravity{};
  double fps = 24;
  int frames = 24;
  double epsilon = 1e-7, tau = 1e-4;
  int levels = 3, window = 8;
  SolverKind solver = SolverKind::Hot;
  KernelKind embedding = KernelKind::Linear;
  double cn_length_factor = 24;
  std::uint64_t seed = 0;
  int ppc = 0;
  bool poisson_sampling = false;
  std::vector<MaterialSpec> materials;
  std::vector<ObjectSpec> objects;
  std::vector<ColliderSpec> colliders;
};

template <int d>
inline Vec<d> take(const std::array<double, 3>& v) {  // simulation.hpp:13-17
  Vec<d> r;
  for (int a = 0; a < d; ++a) r[a] = v[a];
  return r;
}

/// simulation.hpp:20-45
template <int d>
bool inside_shape(const ShapeSpec& s, const Vec<d>& x, double /*time*/) {
  switch (s.kind) {
    case ShapeSpec::Kind::Box:
      for (int a = 0; a < d; ++a)
        if (x[a] < s.min[a] || x[a] > s.max[a]) return false;
      return true;
    case ShapeSpec::Kind::Sphere:
      return norm(x - take<d>(s.center)) <= s.radius;
    case ShapeSpec::Kind::HalfSpace:
      return dot(x - take<d>(s.point), take<d>(s.normal)) <= 0.0;
    case ShapeSpec::Kind::Cylinder: {
      if constexpr (d == 2) {
        return norm(x - take<d>(s.center)) <= s.radius;
      } else {
        Vec<d> axis = take<d>(s.axis);
        const double an = norm(axis);
        for (int a = 0; a < d; ++a) axis[a] = axis[a] / an;
        const Vec<d> rel = x - take<d>(s.center);
        return norm(rel - dot(rel, axis) * axis) <= s.radius;
      }
    }
  }
  return false;
}

/// simulation.hpp:48-65
template <int d>
Vec<d> collider_velocity(const ColliderSpec& c, const Vec<d>& x) {
  switch (c.motion.kind) {
    case MotionSpec::Kind::Static:
      return Vec<d>{};
    case MotionSpec::Kind::Linear:
      return take<d>(c.motion.velocity);
    case MotionSpec::Kind::Rotation: {
      const Vec<d> rel = x - take<d>(c.motion.center);
      if constexpr (d == 2) {
        Vec<d> r;
        r[0] = c.motion.omega * -rel[1];
        r[1] = c.motion.omega * rel[0];
        return r;
      } else {
        Vec<d> ax = take<d>(c.motion.axis);
        const double an = norm(ax);
        for (int a = 0; a < d; ++a) ax[a] = ax[a] / an;
        const Vec<d> w = c.motion.omega * ax;
        Vec<d> r;
        r[0] = w[1] * rel[2] - w[2] * rel[1];
        r[1] = w[2] * rel[0] - w[0] * rel[2];
        r[2] = w[0] * rel[1] - w[1] * rel[0];
        return r;
      }
    }
  }
  return Vec<d>{};
}

constexpr double kPi = 3.14159265358979323846;

template <int d>
double shape_volume(const ShapeSpec& s) {  // simulation.hpp:68-79
  if (s.kind == ShapeSpec::Kind::Box) {
    double v = 1.0;
    for (int a = 0; a < d; ++a) v *= (s.max[a] - s.min[a]);
    return v;
  }
  const double r = s.radius;
  if constexpr (d == 2)
    return kPi * r * r;
  else
    return (4.0 / 3.0) * kPi * r * r * r;
}

template <int d>
void shape_bounds(const ShapeSpec& s, Vec<d>& lo, Vec<d>& hi) {  // simulation.hpp:82-90
  if (s.kind == ShapeSpec::Kind::Box) {
    lo = take<d>(s.min);
    hi = take<d>(s.max);
  } else {
    for (int a = 0; a < d; ++a) {
      lo[a] = s.center[a] - s.radius;
      hi[a] = s.center[a] + s.radius;
    }
  }
}

/// simulation.hpp:94-128 (libstdc++ mt19937_64 + uniform_real_distribution<double>)
template <int d>
std::vector<Vec<d>> sample_jittered(const ShapeSpec& shape, double dx, int ppc, std::mt19937_64& rng, double time) {
  Vec<d> lo, hi;
  shape_bounds<d>(shape, lo, hi);
  Coord<d> cell_lo, cell_hi;
  for (int a = 0; a < d; ++a) {
    cell_lo[a] = static_cast<int>(std::floor(lo[a] / dx));
    cell_hi[a] = static_cast<int>(std::ceil(hi[a] / dx));
  }
  int splits = 1;
  while (ipow(splits, d) < ppc) ++splits;
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<Vec<d>> out;
  Coord<d> c = cell_lo;
  while (true) {
    const int nsub = ipow(splits, d);
    for (int k = 0; k < nsub && k < ppc; ++k) {
      const Coord<d> sub = stencil_offset<d>(k, splits);
      Vec<d> x;
      for (int a = 0; a < d; ++a) x[a] = (c[a] + (sub[a] + unit(rng)) / splits) * dx;
      if (inside_shape<d>(shape, x, time)) out.push_back(x);
    }
    int a = d - 1;
    while (a >= 0) {
      if (++c[a] < cell_hi[a]) break;
      c[a] = cell_lo[a];
      --a;
    }
    if (a < 0) break;
  }
  return out;
}

/// simulation.hpp:132-159
template <int d>
std::vector<Vec<d>> sample_poisson(const ShapeSpec& shape, double dx, int ppc, std::mt19937_64& rng, double time) {
  Vec<d> lo, hi;
  shape_bounds<d>(shape, lo, hi);
  const double volume = shape_volume<d>(shape);
  const double cell_vol = std::pow(dx, static_cast<double>(d));
  const long target = std::max<long>(1, static_cast<long>(volume / cell_vol * ppc));
  const double radius = 0.75 * dx / std::pow(static_cast<double>(ppc), 1.0 / d);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<Vec<d>> out;
  long attempts = 0;
  const long max_attempts = target * 60;
  while (static_cast<long>(out.size()) < target && attempts < max_attempts) {
    ++attempts;
    Vec<d> x;
    for (int a = 0; a < d; ++a) x[a] = lo[a] + unit(rng) * (hi[a] - lo[a]);
    if (!inside_shape<d>(shape, x, time)) continue;
    bool ok = true;
    for (const auto& y : out)
      if (norm(x - y) < radius) {
        ok = false;
        break;
      }
    if (ok) out.push_back(x);
  }
  return out;
}

template <int d>
struct SimulationState {  // simulation.hpp:163-171
  std::vector<Particle<d>> particles;
  double time = 0;
  int frame = 0;
  long step_index = 0;
  long inversion_warnings = 0;
  std::vector<DiagnosticsRecord> diagnostics;
};

inline SolverConfig solver_config_from_scene(const SceneConfig& scene) {  // simulation.hpp:186-197
  SolverConfig cfg;
  cfg.epsilon = scene.epsilon;
  cfg.tau = scene.tau;
  cfg.levels = scene.levels;
  cfg.window = scene.window;
  cfg.kind = scene.solver;
  cfg.embedding = scene.embedding;
  cfg.cn_length_factor = scene.cn_length_factor;
  return cfg;
}

inline std::vector<Material> materials_from_scene(const SceneConfig& scene) {  // simulation.hpp:199-218
  std::vector<Material> mats;
  for (const auto& m : scene.materials) {
    switch (m.plasticity) {
      case PlasticityKind::None:
        mats.push_back(Material::elastic(m.density, m.youngs, m.poisson));
        break;
      case PlasticityKind::VonMises:
        mats.push_back(Material::von_mises(m.density, m.youngs, m.poisson, m.yield_stress));
        break;
      case PlasticityKind::SnowClamp:
        mats.push_back(Material::snow(m.density, m.youngs, m.poisson, m.clamp_lo, m.clamp_hi));
        mats.back().with_hardening(m.hardening);
        break;
      case PlasticityKind::DruckerPrager:
        mats.push_back(Material::drucker_prager(m.density, m.youngs, m.poisson, m.friction_angle));
        break;
    }
    mats.back().with_elasticity(m.elasticity);
  }
  return mats;
}

/// simulation.hpp:221-254
template <int d>
std::vector<Particle<d>> sample_scene_particles(const SceneConfig& scene) {
  const double dx = scene.dx;
  const int ppc = scene.ppc > 0 ? scene.ppc : ipow(2, d);
  std::vector<Particle<d>> particles;
  for (std::size_t oi = 0; oi < scene.objects.size(); ++oi) {
    const auto& obj = scene.objects[oi];
    std::mt19937_64 rng(scene.seed * 0x9e3779b9u + oi + 1);
    std::vector<Vec<d>> xs = scene.poisson_sampling ? sample_poisson<d>(obj.shape, dx, ppc, rng, 0.0)
                                                    : sample_jittered<d>(obj.shape, dx, ppc, rng, 0.0);
    const double volume = scene.poisson_sampling
                              ? shape_volume<d>(obj.shape) / static_cast<double>(std::max<std::size_t>(1, xs.size()))
                              : std::pow(dx, static_cast<double>(d)) / ppc;
    const double density = scene.materials[obj.material].density;
    std::uniform_real_distribution<double> fdist(obj.initial_deformation.lo, obj.initial_deformation.hi);
    for (const auto& x : xs) {
      Particle<d> p;
      p.x = x;
      p.v = take<d>(obj.velocity);
      p.volume = volume;
      p.mass = density * volume;
      p.material = obj.material;
      if (obj.initial_deformation.kind == InitialDeformationSpec::Kind::RandomDiagonal)
        for (int a = 0; a < d; ++a) p.F(a, a) = fdist(rng);
      particles.push_back(p);
    }
  }
  return particles;
}

/// simulation.hpp:259-272
template <int d>
void apply_boundary_scripts(SparseGrid<d>& grid, const SceneConfig& scene, double time) {
  for (int i = 0; i < grid.node_count(); ++i) {
    const Vec<d> x = grid.node_position(i);
    for (const auto& col : scene.colliders) {
      if (!inside_shape<d>(col.shape, x, time)) continue;
      const Vec<d> v = collider_velocity<d>(col, x);
      grid.dirichlet[i] = 1;
      set_seg<d>(grid.velocity, i, v);
      set_seg<d>(grid.bc_velocity, i, v);
      break;
    }
  }
}

struct StepStats {  // simulation.hpp:275-281
  double dt = 0;
  int outer_iterations = 0;
  long inner_total = 0;
  int node_count = 0;
  bool converged = false;
};

/// simulation.hpp:286-323
template <int d>
StepStats advance_step(SimulationState<d>& sim, const SceneConfig& scene, const SolverConfig& cfg, double frame_end) {
  const double dx = scene.dx;
  OracleTimer tm;
  double v_max = 0.0;
  for (const auto& p : sim.particles) v_max = std::max(v_max, norm(p.v));
  double dt = cfl_dt(v_max, dx, scene.fps);
  if (frame_end > 0.0) dt = std::min(dt, frame_end - sim.time);
  if (!(dt > 0.0)) throw SolverFailure("advance_step: non-positive time step");
  std::vector<Vec<d>> positions(sim.particles.size());
  for (std::size_t i = 0; i < sim.particles.size(); ++i) positions[i] = sim.particles[i].x;
  tm.lap("cfl");
  SparseGrid<d> grid = activate_grid<d>(positions, dx, KernelKind::QuadraticBSpline);
  tm.lap("activate");
  p2g<d>(sim.particles, grid);
  tm.lap("p2g");
  apply_boundary_scripts<d>(grid, scene, sim.time);
  tm.lap("boundary");
  const auto materials = materials_from_scene(scene);
  const Vec<d> gravity = take<d>(scene.gravity);
  const ObjectiveState<d> st =
      make_objective_state<d>(sim.particles, grid, materials, dt, gravity, scene.cn_length_factor);
  tm.lap("objective_state");
  GridStepResult<d> step;
  try {
    step = step_grid<d>(st, cfg, &sim.diagnostics, sim.frame, sim.step_index);
  } catch (const SolverFailure& e) {
    throw SolverFailure("step " + std::to_string(sim.step_index) + ": " + e.what());
  }
  tm.lap("step_grid");
  grid.velocity = step.velocity;
  g2p<d>(grid, sim.particles);
  sim.inversion_warnings += update_strain<d>(sim.particles, grid, dt, materials);
  advect<d>(sim.particles, dt);
  tm.lap("g2p_strain_adv");
  sim.time += dt;
  ++sim.step_index;
  return {dt, step.solve.outer_iterations, step.solve.inner_total, grid.node_count(), step.solve.converged};
}

}  // namespace hot_oracle
