"""The C++ shim (include/hotmpm_cuda.hpp) compiles against stand-ins of the reference's public
types (the real headers need Eigen, which is absent here) and links against libhotb200.so."""
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

STUB = r'''
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>
namespace hotmpm {
struct SolverFailure : std::runtime_error { explicit SolverFailure(const std::string& m) : std::runtime_error(m) {} };
enum class KernelKind { QuadraticBSpline, Linear };
enum class SolverKind { Hot, PnPcg, PnPcgMatrixFree, PnMgpcg, LbfgsH };
struct PlasticitySpec { enum class Kind { None, VonMises, SnowClamp } kind = Kind::None; double yield_stress = 0, clamp_lo = 0.99, clamp_hi = 1.001; };
struct MaterialSpec { double density = 0, youngs = 0, poisson = 0; PlasticitySpec plasticity; };
struct ShapeSpec { enum class Kind { Box, Sphere, HalfSpace, Cylinder } kind = Kind::Box; std::array<double, 3> min{}, max{}, center{}; double radius = 0; std::array<double, 3> point{}, normal{}, axis{}; };
struct MotionSpec { enum class Kind { Static, Linear, Rotation } kind = Kind::Static; std::array<double, 3> velocity{}, center{}, axis{}; double omega = 0; };
struct InitialDeformationSpec { enum class Kind { Identity, RandomDiagonal } kind = Kind::Identity; double lo = 1, hi = 1; };
struct ObjectSpec { ShapeSpec shape; int material = 0; std::array<double, 3> velocity{}; InitialDeformationSpec initial_deformation; };
struct ColliderSpec { ShapeSpec shape; MotionSpec motion; };
struct SceneConfig { int dim = 3; double dx = 0.01; std::array<double, 3> gravity{}; double fps = 24; int frames = 24;
  double epsilon = 1e-7, tau = 1e-4; int levels = 3, window = 8; std::string solver = "hot", embedding = "linear";
  double cn_length_factor = 24; std::uint64_t seed = 0; int ppc = 0; std::string sampling = "jittered";
  std::vector<MaterialSpec> materials; std::vector<ObjectSpec> objects; std::vector<ColliderSpec> colliders; };
template <typename T> SolverKind parse_solver_kind(const std::string&) { return SolverKind::Hot; }
template <typename T> struct SolverConfig { T epsilon = 1e-7, tau = 1e-4; int levels = 3, window = 8; T ls_shrink = 0.5, ls_armijo = 1e-4;
  int ls_max_steps = 30, cg_cap = 10000, outer_cap = 1000; SolverKind kind = SolverKind::Hot; KernelKind embedding = KernelKind::Linear;
  int pinned_coarse_iterations = 256; T cn_length_factor = 24; };
struct DiagnosticsRecord { int frame; long step; int outer_iteration; double scaled_residual, energy, step_length; long inner_iterations, work_units; double wall_ms; };
template <typename T, int d> struct Vec { T v[d]{}; T& operator[](int i) { return v[i]; } T operator[](int i) const { return v[i]; } };
template <typename T, int d> struct Mat { T m[d * d]{}; T& operator()(int r, int c) { return m[c * d + r]; } T operator()(int r, int c) const { return m[c * d + r]; } };
template <typename T, int d> struct Particle { Vec<T, d> x, v; T mass{}, volume{}; Mat<T, d> F, C; int material = 0; };
template <typename T, int d> struct SimulationState { std::vector<Particle<T, d>> particles; T time = 0; int frame = 0; long step_index = 0; long inversion_warnings = 0; std::vector<DiagnosticsRecord> diagnostics; };
template <typename T> struct StepStats { T dt{}; int outer_iterations = 0; long inner_total = 0; int node_count = 0; bool converged = false; };
}
#include "hotmpm_cuda.hpp"
int main() {
  hotmpm::SceneConfig sc;
  if (hot_device_count() == 0) return 0;  // no GPU: compile/link check only
  hotmpm::cuda::Stepper s(sc);
  hotmpm::SimulationState<double, 3> sim;
  hotmpm::SolverConfig<double> cfg;
  (void)s.advance_step<double, 3>(sim, cfg, 1.0 / 24);
  hotmpm::SceneConfig sc2;  // the 2D device path (cli.cpp:145 instantiates d = 2 too)
  sc2.dim = 2;
  hotmpm::cuda::Stepper s2(sc2);
  hotmpm::SimulationState<double, 2> sim2;
  (void)s2.advance_step<double, 2>(sim2, cfg, 1.0 / 24);
  return 0;
}
'''


def test_shim_compiles_and_links():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "shim.cpp")
        open(src, "w").write(STUB)
        lib = os.path.join(ROOT, "paper_1911_07913_b200", "lib")
        out = os.path.join(d, "shim")
        r = subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), src, "-L", lib, "-lhotb200",
                            f"-Wl,-rpath,{lib}", "-o", out], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([out], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
