// Host orchestration of the B200 HOT step and the C-ABI (include/hot_c_api.h).
//
// hot_advance_step restates advance_step (simulation.hpp:286-323); the solve restates
// solve_quasi_newton (solvers.hpp:191-231) with every vector and matrix resident in HBM.
// The host only sees the scalars the reference's control flow branches on (line-search
// energies, g.p, the CN residual, y.s / |y| / |s| and the coarse PCG status), read back
// once per line-search trial / accepted iterate.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hot_c_api.h"
#include "hot_comm.h"
#include "hot2d.h"
#include "hot_internal.h"

namespace hotb200 {

long long sample_scene(const hot_scene& sc, std::vector<double>& x, std::vector<double>& v, std::vector<double>& mass,
                       std::vector<double>& vol, std::vector<double>& F, std::vector<double>& C,
                       std::vector<int>& mat);

/// Material::elastic / von_mises / snow (constitutive.hpp:12-52) + stiffness_scale
/// (constitutive.hpp:255-258) in dimension dim.
DevMaterial make_dev_material(const hot_material& m, int dim) {
  if (!(m.youngs > 0.0)) throw std::invalid_argument("material: Young's modulus must be positive");
  if (!(m.poisson >= 0.0 && m.poisson < 0.5)) throw std::invalid_argument("material: Poisson ratio must lie in [0, 0.5)");
  DevMaterial d{};
  d.mu = m.youngs / (2.0 * (1.0 + m.poisson));
  d.lambda = m.youngs * m.poisson / ((1.0 + m.poisson) * (1.0 - 2.0 * m.poisson));
  d.plasticity = m.plasticity;
  if (m.elasticity != 0 && m.elasticity != 1) throw std::invalid_argument("material: unknown elasticity");
  d.elasticity = m.elasticity;
  if (m.plasticity == 1) {
    if (!(m.yield_stress > 0.0)) throw std::invalid_argument("material: yield stress must be positive");
    d.yield_stress = m.yield_stress;
  } else if (m.plasticity == 2) {
    if (!(m.clamp_lo <= 1.0 && 1.0 <= m.clamp_hi)) throw std::invalid_argument("material: snow clamp must bracket 1");
    if (!(m.hardening >= 0.0)) throw std::invalid_argument("material: hardening must be non-negative");
    d.clamp_lo = m.clamp_lo;
    d.clamp_hi = m.clamp_hi;
    d.hardening = m.hardening;
  } else if (m.plasticity == 3) {  // Drucker-Prager (extension; oracle Material::drucker_prager)
    if (!(m.friction_angle >= 0.0 && m.friction_angle < 90.0))
      throw std::invalid_argument("material: friction angle must lie in [0, 90) degrees");
    const double sp = std::sin(m.friction_angle * 3.14159265358979323846 / 180.0);
    d.dp_alpha = std::sqrt(2.0 / 3.0) * 2.0 * sp / (3.0 - sp);
  } else if (m.plasticity != 0) {
    throw std::invalid_argument("material: unknown plasticity");
  }
  // dP/dF at F = I in diagonal space: (mm) block 2mu I + la 11^T; 2x2 blocks with
  // bd = 2mu - la*0, bs = (psi_i+psi_j)/2 = 0 -> entries (mu, mu).  Frobenius norm is basis
  // invariant (Q orthogonal): sum of squares of Mhat.
  const double a = 2.0 * d.mu + d.lambda, b = d.lambda;
  const double mh = 0.5 * (2.0 * d.mu);
  // d diagonal entries a, d(d-1) off-diagonal b, d(d-1)/2 2x2 blocks of four entries mh
  const double fro2 = dim * a * a + dim * (dim - 1) * b * b + (dim * (dim - 1) / 2) * 4.0 * mh * mh;
  d.xi = std::sqrt(fro2);
  return d;
}

static std::atomic<long long> g_launches{0};
long long kernel_launch_count() { return g_launches.load(); }
void count_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

namespace {


#define HOT_CUDA(x)                                                                                      \
  do {                                                                                                   \
    cudaError_t e_ = (x);                                                                                \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));             \
  } while (0)

/// Grow-only device buffer (non-copyable; swap exchanges ownership).
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(cap, o.cap);
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    static const bool trace = std::getenv("HOT_ALLOC_TRACE") != nullptr;  // diagnosis: growth events
    if (trace) std::fprintf(stderr, "[hot alloc] grow %zu -> %zu bytes\n", cap, bytes);
    if (p) HOT_CUDA(cudaFree(p));
    p = nullptr;
    // grow with slack (2 MiB granules): node / particle counts drift by a few per step and an
    // exact-size reallocation of a GB-sized level matrix every step costs more than the step.
    // 25 % for buffers of 1 GB and more, 50 % from 256 MB, 100 % below: the small ones include the
    // bounding-box sized maps, whose box grows with the motion (cfg2: +26 % volume in 13 steps),
    // and a cudaFree + cudaMalloc in the middle of a run costs 1.5 ms at best and, one time in
    // eight on the bench box, 30-400 ms
    const size_t slack = bytes >= (size_t(1) << 30) ? bytes / 4 : bytes >= (size_t(256) << 20) ? bytes / 2 : bytes;
    size_t nb = std::max<size_t>(bytes + slack, cap + cap / 4);
    nb = std::max<size_t>((nb + (2u << 20) - 1) & ~size_t((2u << 20) - 1), 256);
    HOT_CUDA(cudaMalloc(&p, nb));
    cap = nb;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

/// Test and diagnostic hooks, read from the environment once per context (hot_create).  None of
/// them changes a value: the schedules they select are bitwise identical.
struct Options {
  bool shard_force = false;        // HOT_SHARD_FORCE: the slab path at one rank (transport test)
  bool shard_replicate = false;    // HOT_SHARD_REPLICATE: sharded solves keep every particle on every rank
  bool sgs_level0_waves = false;   // HOT_SGS_LEVEL0=waves: one launch per level-0 wave
  bool sgs_coarse_barrier = false; // HOT_SGS_COARSE=barrier: grid-barrier coarse smoother
  bool sgs_trace = false;          // HOT_SGS_TRACE: per-wave timing of the barrier smoother
  bool verbose = false;            // HOT_VERBOSE: per-solve diagnostics on stderr
  bool asm_tiles = false;          // HOT_ASM=tiles: the row-tile level-0 assembly (k_assemble_tiles)
  long long asm_ring_bins = 256 * 1024;  // HOT_ASM_RING: bins in the pair-sum ring (27,216 B each)
  int stream_min_rows = 8 * 1024;  // HOT_SGS_STREAM_MIN: rows per wave from which level 0 streams
  void read_env() {
    auto eq = [](const char* k, const char* v) {
      const char* e = std::getenv(k);
      return e && std::strcmp(e, v) == 0;
    };
    shard_force = std::getenv("HOT_SHARD_FORCE") != nullptr;
    shard_replicate = std::getenv("HOT_SHARD_REPLICATE") != nullptr;
    sgs_level0_waves = eq("HOT_SGS_LEVEL0", "waves");
    sgs_coarse_barrier = eq("HOT_SGS_COARSE", "barrier");
    sgs_trace = std::getenv("HOT_SGS_TRACE") != nullptr;
    verbose = std::getenv("HOT_VERBOSE") != nullptr;
    asm_tiles = eq("HOT_ASM", "tiles");
    if (const char* e = std::getenv("HOT_ASM_RING")) asm_ring_bins = std::max(1LL, std::atoll(e));
    if (const char* e = std::getenv("HOT_SGS_STREAM_MIN")) stream_min_rows = std::atoi(e);
  }
};

constexpr int kMaxLevels = 8;
constexpr int kMaxWindow = 64;

struct Level {
  int n = 0;
  int lo[3] = {0, 0, 0}, ext[3] = {0, 0, 0};
  DBuf map, coords, cols, H, dinv, dir, flags;
  DBuf wave_of, wave_counts, wave_start, wave_cursor, wave_rows, wave_start_c;
  DBuf sgs_uf, sgs_ub;  // the dataflow smoother's forward / backward results (also its flags)
  int nwaves = 0, max_wave = 0;
  std::vector<int> wave_start_h;
  long long active_slots = 0;
  int radius = 2;  // diagonal-storage radius (3 on quadratic-embedding coarse levels)
  int h_row0 = 0;  // H holds rows [h_row0, h_row0 + allocated rows) (slabs: only the rank's rows)
  DBuf b, u, r;    // V-cycle vectors
  DenseMap dmap() const {
    DenseMap m;
    for (int a = 0; a < 3; ++a) {
      m.lo[a] = lo[a];
      m.ext[a] = ext[a];
    }
    m.idx = map.as<int>();
    return m;
  }
  LevelView view() const {
    LevelView v;
    v.n = n;
    v.coords = coords.as<int>();
    v.map = dmap();
    v.cols = cols.as<int>();
    // rows outside the allocation are never touched (slabs)
    v.H = H.as<double>() - (long long)h_row0 * 9 * pitch();
    v.dinv = dinv.as<double>();
    v.dir = dir.as<uint8_t>();
    v.radius = radius;
    v.lo = 0;
    v.hi = n;
    return v;
  }
  int pitch() const { return level_pitch(radius); }
  int slots() const { return level_slots(radius); }
};

struct ProfEvent {
  int phase;
  cudaEvent_t a, b;
};

const char* kPhaseNames[] = {"activate_bin", "p2g_bc", "particle_energy", "node_gradient", "particle_tensors",
                             "assemble_rows", "hierarchy", "sgs_level0", "sgs_coarse", "residual_restrict",
                             "coarse_pcg", "prolong", "lbfgs_vectors", "g2p_strain_advect", "upload_download",
                             "spmv_level0", "slab_comm", "assemble_pairs"};
constexpr int kPhases = sizeof(kPhaseNames) / sizeof(kPhaseNames[0]);
enum Phase {
  P_ACTIVATE,
  P_P2G,
  P_ENERGY,
  P_GRADIENT,
  P_TENSORS,
  P_ASSEMBLE,
  P_HIER,
  P_SGS0,
  P_SGSC,
  P_RESID,
  P_PCG,
  P_PROLONG,
  P_VEC,
  P_G2P,
  P_IO,
  P_SPMV0,
  P_COMM,
  P_ASM_PAIRS
};

}  // namespace

struct Context {
  int device = 0;
  Options opt;
  DBuf active_dev;  // ull[kMaxLevels]: active slots per level of the current hierarchy (k_fill_cols)
  static constexpr int kProfSolves = 8192;
  DBuf prof_slots;  // ull[kProfSolves][kMaxLevels]: active_dev snapshot per profiled solve
  int prof_solve = -1;
  struct SlotTerm {
    int phase, solve, level;
    double coef;
  };
  std::vector<SlotTerm> slot_terms;
  cudaStream_t stream = nullptr;
  std::string err;

  // scene / config (copied)
  double dx = 0.01, fps = 24, cn_factor = 24;
  double grav[3] = {0, 0, 0};
  std::vector<DevMaterial> mats_h;
  std::vector<DevCollider> cols_h;
  hot_solver_config cfg{};

  // particles (SoA on device)
  long long np = 0;
  DBuf px, pv, pF, pC, pmass, pvol, pmat, stage, porig;
  DBuf qx, qv, qF, qC, qmass, qvol, qmat, qorig;  // reorder targets (swapped each step)
  DBuf pjp, qjp;         // plastic volume ratio per particle (snow materials; hardening extension)
  // particle partition: once a sharded step has cut the slabs, every rank stores
  // only the particles of its band [P - kPPLeft, Q + kPPRight) (owned: [P, Q); the rest ghost
  // copies), exchanged after every advection.  np is then the local count.
  static constexpr int kPPLeft = 8;   // bins the assembly reads from plane P - 8 (plan_shard)
  static constexpr int kPPRight = 1;  // bins the P2G / energy / gradient node passes read up to plane Q
  bool pp_on = false;
  std::vector<int> pp_bounds;         // the frozen cut (size + 1 planes) the partition follows
  long long np_global = 0;            // particles of the whole scene
  DBuf pp_keep, pp_pack, pp_kpos, pp_ppos, pp_send, pp_rflag, pp_rpos, pp_small;
  bool track_jp = false; // some material is snow: J_p is stored, reordered and updated
  double time = 0;
  int frame = 0;
  long long step_index = 0, inversions = 0;
  std::vector<hot_diag_row> diag;

  // grid (level 0 storage lives in L[0])
  Level L[kMaxLevels];
  int nlevels = 0;
  bool have_state = false, have_H = false;
  double dt = 0;
  DBuf gmass, gvel, gmom, gbc, gcn;
  DBuf bin_of, bin_counts, bin_start, bin_cursor, bin_pid, scan_tmp;
  DBuf pbin, nb27, node_u;
  DBuf svd;  // U s V of every particle's virtual F at the solve's initial dv (21 doubles SoA)  // per-slot bin node, 27-neighbour table, nodal velocity of virtual_F
  DBuf mats_d, cols_d;

  // solver vectors
  DBuf dv, g, gnew, pdir, q, stress, Tu, vout, hist_s[kMaxWindow + 1], hist_y[kMaxWindow + 1];
  DBuf pcg_r, pcg_z, pcg_p, pcg_Ap, sgs_trace, gal_x;
  // second stream for the hierarchy's structure half (overlaps the level-0 assembly)
  cudaStream_t stream2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DBuf scan_tmp2, struct_flags;
  DBuf grid_bar;  // words 0-1: the persistent smoothers' grid barrier; word 8: the assembly's tile counter
  DBuf asm_pairs;  // ring of per-bin pair sums (level-0 assembly by bins)
  DBuf bin_part;  // per (bin, stencil position) particle sums feeding the node gathers (P2G, gradient)
  DBuf pn_b, pn_x, pn_r, pn_z, pn_p, pn_Ap, pn_dinv, pn_dP;  // projected-Newton PCG on level 0
  DBuf partials, scal, coef_a, coef_b, iflags, bounds;
  double* host_scal = nullptr;  // pinned
  int* host_int = nullptr;      // pinned
  int nred = 0;

  // multi-GPU slabs: the transport, and this solve's cut
  std::unique_ptr<Comm> comm;
  struct Shard {
    bool on = false;               // the current solve runs slab-sharded
    int P = 0, Q = 0;              // owned lattice planes [P, Q) (axis 0, absolute)
    int r_lo = 0, r_hi = 0;        // owned level-0 rows
    int a_lo = 0;                  // assembled level-0 rows [a_lo, r_hi): owned + 7 planes to the left
    int x_lo = 0;                  // Galerkin stage-1 fine rows [x_lo, r_hi): owned + 5 planes
    long long p_lo = 0, p_hi = 0;  // particles of the bins the assembled rows read (planes [P-8, Q+1))
    long long pe_lo = 0;           // particles of the bins the gradient's node pass reads: [pe_lo, p_hi)
    int h_hi = 0;                  // level-0 matrix rows this rank stores: [a_lo, h_hi) (transposes reach Q+2)
    int b_lo = 0, b_hi = 0;        // those bins (rows of planes [P-1, Q+1))
    int c_lo = 0, c_hi = 0;        // owned level-1 rows (coarse planes [P/2, Q/2))
    int gc_lo = 0;                 // Galerkin stage-2 coarse rows [gc_lo, c_hi): owned + 2 coarse planes
    std::vector<int> bounds;       // size+1 plane cuts
    std::vector<int> ps0;          // level-0 plane starts (rows), ext0+1
    std::vector<long long> row_off;                 // level-0 row cuts per rank
    std::vector<long long> crow_off;                // level-1 row cuts per rank
    std::vector<long long> halo_edges[3];           // per axis-0 residue: byte ranges of the one edge plane a wave changes
    std::vector<int> wave_counts_global;            // level-0 rows per colour (all ranks)
    std::vector<int> wave_start;                    // this rank's rows per colour (27 + 1)
    DBuf wave_rows, wave_counts, wave_starts, wave_cursor;
    long long solves = 0;          // sharded solves so far
    bool last = false;             // the last solve ran sharded
    bool planned = false;          // this step's grid has a cut (set by prepare)
  } sh;
  DBuf plane_buf;
  DBuf pe_buf, ne_buf, nt_buf;  // per-particle energy, per-node energy, per-node scaled-norm terms
  long long tu_lo = 0;           // Tu holds the records of particles [tu_lo, ...)
  /// Record base indexed by particle id (slabs: only [p_lo, p_hi) is allocated and touched).
  double* tu_base() { return Tu.as<double>() - tu_lo * 126; }

  // profiling
  bool prof = false;
  std::vector<ProfEvent> events;
  std::vector<cudaEvent_t> event_pool;
  double phase_bytes[kPhases] = {0};
  double phase_flops[kPhases] = {0};

  Context() = default;
  ~Context() {
    for (auto& e : events) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
    if (host_scal) cudaFreeHost(host_scal);
    if (host_int) cudaFreeHost(host_int);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (stream2) cudaStreamDestroy(stream2);
    if (stream) cudaStreamDestroy(stream);
  }

  // ------------------------------------------------------------------ helpers
  ParticlesView pview() const {
    ParticlesView P;
    P.x = px.as<double>();
    P.v = pv.as<double>();
    P.F = pF.as<double>();
    P.C = pC.as<double>();
    P.mass = pmass.as<double>();
    P.vol = pvol.as<double>();
    P.mat = pmat.as<int>();
    P.bin = pbin.as<int>();
    P.Jp = track_jp ? pjp.as<double>() : nullptr;
    P.n = np;
    return P;
  }
  GridView gview() const {
    GridView G;
    G.n = L[0].n;
    G.coords = L[0].coords.as<int>();
    G.map = L[0].dmap();
    G.mass = gmass.as<double>();
    G.vel = gvel.as<double>();
    G.mom = gmom.as<double>();
    G.dir = L[0].dir.as<uint8_t>();
    G.bc_vel = gbc.as<double>();
    G.cn_scale = gcn.as<double>();
    G.nb27 = nb27.as<int>();
    return G;
  }
  BinsView bview() const {
    BinsView b;
    b.start = bin_start.as<int>();
    b.pid = bin_pid.as<int>();
    return b;
  }
  cudaEvent_t take_event() {
    if (event_pool.empty()) {
      cudaEvent_t e;
      HOT_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  int prof_begin(int phase) {
    if (!prof) return -1;
    ProfEvent pe{phase, take_event(), take_event()};
    cudaEventRecord(pe.a, stream);
    events.push_back(pe);
    return (int)events.size() - 1;
  }
  void prof_end(int h, double bytes = 0, double flops = 0) {
    if (h < 0) return;
    cudaEventRecord(events[h].b, stream);
    phase_bytes[events[h].phase] += bytes;
    phase_flops[events[h].phase] += flops;
  }
  /// Algorithmic bytes proportional to a level's active-slot count: coef x (active slots of level
  /// m in the current profiled solve).  The counts stay on the device (k_fill_cols counts them;
  /// one device-to-device snapshot per solve) and are only read by hot_profile_read, so profiling
  /// adds no kernel and no host synchronisation to the step.
  void prof_slot_bytes(int h, int m, double coef) {
    if (h < 0 || prof_solve < 0) return;
    slot_terms.push_back(SlotTerm{events[h].phase, prof_solve, m, coef});
  }
  void prof_snapshot_slots() {
    if (!prof || prof_solve + 1 >= kProfSolves) return;
    ++prof_solve;
    HOT_CUDA(cudaMemcpyAsync(prof_slots.as<unsigned long long>() + (size_t)prof_solve * kMaxLevels, active_dev.p,
                             sizeof(unsigned long long) * kMaxLevels, cudaMemcpyDeviceToDevice, stream));
  }
  void sync() { HOT_CUDA(cudaStreamSynchronize(stream)); }
  void check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw CudaError(std::string("kernel launch: ") + cudaGetErrorString(e));
  }
  void read_scalars(int nd, int ni) {
    if (nd) HOT_CUDA(cudaMemcpyAsync(host_scal, scal.p, sizeof(double) * nd, cudaMemcpyDeviceToHost, stream));
    if (ni) HOT_CUDA(cudaMemcpyAsync(host_int, iflags.p, sizeof(int) * ni, cudaMemcpyDeviceToHost, stream));
    sync();
    check_launch();
    // slabs: the flags of split kernels differ per rank; every rank must take the same branch
    // (the other ints are replicated, so their max is their value)
    if (sh.on && ni) comm->allreduce_max(host_int, ni, stream);
  }

  void init(int dev) {
    device = dev;
    opt.read_env();
    HOT_CUDA(cudaSetDevice(dev));
    HOT_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    HOT_CUDA(cudaStreamCreateWithFlags(&stream2, cudaStreamNonBlocking));
    HOT_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    HOT_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    struct_flags.ensure(sizeof(int) * 16);
    active_dev.ensure(sizeof(unsigned long long) * kMaxLevels);
    HOT_CUDA(cudaMemset(active_dev.p, 0, sizeof(unsigned long long) * kMaxLevels));
    grid_bar.ensure(sizeof(unsigned int) * 16);
    HOT_CUDA(cudaMallocHost(&host_scal, sizeof(double) * 64));
    HOT_CUDA(cudaMallocHost(&host_int, sizeof(int) * 64));
    nred = 8 * num_sms();
    partials.ensure(sizeof(double) * (6 * nred + std::max(pcg_max_blocks(), sgs_max_blocks()) + 64));
    scal.ensure(sizeof(double) * 64);
    iflags.ensure(sizeof(int) * 64);
    bounds.ensure(sizeof(int) * 8);
    coef_a.ensure(sizeof(double) * kMaxWindow);
    coef_b.ensure(sizeof(double) * kMaxWindow);
  }

  void set_scene(const hot_scene& s) {
    if (s.dim != 3) throw std::invalid_argument("the 3D context takes dim = 3 scenes");
    if (!(s.dx > 0)) throw std::invalid_argument("activate_grid: dx must be positive");
    dx = s.dx;
    fps = s.fps;
    cn_factor = s.cn_length_factor;
    for (int a = 0; a < 3; ++a) grav[a] = s.gravity[a];
    mats_h.clear();
    for (int i = 0; i < s.n_materials; ++i) mats_h.push_back(make_material(s.materials[i]));
    track_jp = false;
    for (const DevMaterial& m : mats_h) track_jp = track_jp || m.plasticity == 2;
    if ((int)mats_h.size() > kMaxMaterials) throw std::invalid_argument("too many materials");
    cols_h.clear();
    for (int i = 0; i < s.n_colliders; ++i) cols_h.push_back(make_collider(s.colliders[i]));
    mats_d.ensure(sizeof(DevMaterial) * std::max<size_t>(1, mats_h.size()));
    if (!mats_h.empty())
      HOT_CUDA(cudaMemcpy(mats_d.p, mats_h.data(), sizeof(DevMaterial) * mats_h.size(), cudaMemcpyHostToDevice));
    cols_d.ensure(sizeof(DevCollider) * std::max<size_t>(1, cols_h.size()));
    if (!cols_h.empty())
      HOT_CUDA(cudaMemcpy(cols_d.p, cols_h.data(), sizeof(DevCollider) * cols_h.size(), cudaMemcpyHostToDevice));
    cfg.epsilon = s.epsilon;
    cfg.tau = s.tau;
    cfg.levels = s.levels;
    cfg.window = s.window;
    cfg.ls_shrink = 0.5;
    cfg.ls_armijo = 1e-4;
    cfg.ls_max_steps = 30;
    cfg.cg_cap = 10000;
    cfg.outer_cap = 1000;
    cfg.kind = s.solver;
    cfg.embedding = s.embedding;
    cfg.pinned_coarse_iterations = 256;
    cfg.cn_length_factor = s.cn_length_factor;
  }

  static DevMaterial make_material(const hot_material& m) { return make_dev_material(m, 3); }

  static DevCollider make_collider(const hot_collider& c) {
    DevCollider d{};
    d.shape = c.shape.kind;
    d.motion = c.motion.kind;
    d.radius = c.shape.radius;
    for (int a = 0; a < 3; ++a) {
      switch (c.shape.kind) {
        case 0:
          d.a[a] = c.shape.min[a];
          d.b[a] = c.shape.max[a];
          break;
        case 1:
          d.a[a] = c.shape.center[a];
          break;
        case 2:
          d.a[a] = c.shape.point[a];
          d.b[a] = c.shape.normal[a];
          break;
        case 3:
          d.a[a] = c.shape.center[a];
          break;
      }
      d.vel[a] = c.motion.velocity[a];
      d.rot_center[a] = c.motion.center[a];
    }
    if (c.shape.kind == 3) {
      const double n = std::sqrt(c.shape.axis[0] * c.shape.axis[0] + c.shape.axis[1] * c.shape.axis[1] +
                                 c.shape.axis[2] * c.shape.axis[2]);
      for (int a = 0; a < 3; ++a) d.b[a] = c.shape.axis[a] / n;
    }
    if (c.motion.kind == 2) {
      const double n = std::sqrt(c.motion.axis[0] * c.motion.axis[0] + c.motion.axis[1] * c.motion.axis[1] +
                                 c.motion.axis[2] * c.motion.axis[2]);
      for (int a = 0; a < 3; ++a) d.rot_w[a] = c.motion.omega * (c.motion.axis[a] / n);
    }
    return d;
  }

  // ------------------------------------------------------------------ particles
  void upload(long long n, const double* x, const double* v, const double* mass, const double* vol, const double* F,
              const double* C, const int* mat) {
    const int h = prof_begin(P_IO);
    np = n;
    np_global = n;
    pp_on = false;
    const size_t n3 = sizeof(double) * 3 * std::max<long long>(n, 1), n9 = sizeof(double) * 9 * std::max<long long>(n, 1);
    px.ensure(n3);
    pv.ensure(n3);
    pF.ensure(n9);
    pC.ensure(n9);
    pmass.ensure(sizeof(double) * std::max<long long>(n, 1));
    pvol.ensure(sizeof(double) * std::max<long long>(n, 1));
    pmat.ensure(sizeof(int) * std::max<long long>(n, 1));
    porig.ensure(sizeof(int) * std::max<long long>(n, 1));
    qx.ensure(n3);
    qv.ensure(n3);
    qF.ensure(n9);
    qC.ensure(n9);
    qmass.ensure(sizeof(double) * std::max<long long>(n, 1));
    qvol.ensure(sizeof(double) * std::max<long long>(n, 1));
    qmat.ensure(sizeof(int) * std::max<long long>(n, 1));
    qorig.ensure(sizeof(int) * std::max<long long>(n, 1));
    if (track_jp) {  // J_p = 1: no plastic volume change yet (hot_set_plastic_state overrides)
      pjp.ensure(sizeof(double) * std::max<long long>(n, 1));
      qjp.ensure(sizeof(double) * std::max<long long>(n, 1));
      launch_fill(pjp.as<double>(), n, 1.0, stream);
    }
    // one staging region per interleaved field, so the host->device copies run back to back
    // (no DMA gaps for the transposes) and the transposes follow
    stage.ensure(sizeof(double) * 24 * std::max<long long>(n, 1));
    launch_iota(porig.as<int>(), n, stream);
    if (n > 0) {
      if (!x) throw std::invalid_argument("positions are required");
      double* sx = stage.as<double>();
      double* sv = sx + 3 * n;
      double* sF = sv + 3 * n;
      double* sC = sF + 9 * n;
      struct Field {
        const double* src;
        double* st;
        DBuf* dst;
        int comps;
      } fields[4] = {{x, sx, &px, 3}, {v, sv, &pv, 3}, {F, sF, &pF, 9}, {C, sC, &pC, 9}};
      for (const Field& f : fields)
        if (f.src) HOT_CUDA(cudaMemcpyAsync(f.st, f.src, sizeof(double) * f.comps * n, cudaMemcpyHostToDevice, stream));
      if (mass)
        HOT_CUDA(cudaMemcpyAsync(pmass.p, mass, sizeof(double) * n, cudaMemcpyHostToDevice, stream));
      else
        HOT_CUDA(cudaMemsetAsync(pmass.p, 0, sizeof(double) * n, stream));
      if (vol)
        HOT_CUDA(cudaMemcpyAsync(pvol.p, vol, sizeof(double) * n, cudaMemcpyHostToDevice, stream));
      else
        HOT_CUDA(cudaMemsetAsync(pvol.p, 0, sizeof(double) * n, stream));
      if (mat)
        HOT_CUDA(cudaMemcpyAsync(pmat.p, mat, sizeof(int) * n, cudaMemcpyHostToDevice, stream));
      else
        HOT_CUDA(cudaMemsetAsync(pmat.p, 0, sizeof(int) * n, stream));
      for (const Field& f : fields) {
        if (f.src) {
          launch_aos_to_soa(f.st, f.dst->as<double>(), n, f.comps, stream);
        } else {
          HOT_CUDA(cudaMemsetAsync(f.dst->p, 0, sizeof(double) * f.comps * n, stream));
          if (f.dst == &pF) {  // default F = I
            std::vector<double> eye(9 * n, 0.0);
            for (long long p = 0; p < n; ++p) eye[0 * n + p] = eye[4 * n + p] = eye[8 * n + p] = 1.0;
            HOT_CUDA(cudaMemcpyAsync(pF.p, eye.data(), sizeof(double) * 9 * n, cudaMemcpyHostToDevice, stream));
            sync();
          }
        }
      }
      if (mat) {  // material ids checked on the device
        HOT_CUDA(cudaMemsetAsync(iflags.as<int>() + 7, 0, sizeof(int), stream));
        launch_check_ids(pmat.as<int>(), n, (int)mats_h.size(), iflags.as<int>() + 7, stream);
      }
    }
    prof_end(h, (double)n * (3 + 3 + 9 + 9 + 2) * 8 + 4.0 * n);
    have_state = false;
    sh.planned = false;
    if (mat && n) {
      int bad = 0;
      HOT_CUDA(cudaMemcpyAsync(&bad, iflags.as<int>() + 7, sizeof(int), cudaMemcpyDeviceToHost, stream));
      sync();
      if (bad) throw std::invalid_argument("particle material id out of range");
    } else {
      sync();
    }
  }

  void download(double* x, double* v, double* F, double* C) {
    const int h = prof_begin(P_IO);
    if (pp_on) {  // partitioned: every rank's owned particles, in the caller's order
      const long long total = pp_gather_owned_records();
      stage.ensure(sizeof(double) * 24 * std::max<long long>(total, 1));
      double* sx = stage.as<double>();
      double* sv = sx + 3 * total;
      double* sF = sv + 3 * total;
      double* sC = sF + 9 * total;
      launch_pp_unpack_caller(pp_send.as<double>(), total, x ? sx : nullptr, v ? sv : nullptr, F ? sF : nullptr,
                              C ? sC : nullptr, nullptr, stream);
      if (x) HOT_CUDA(cudaMemcpyAsync(x, sx, sizeof(double) * 3 * total, cudaMemcpyDeviceToHost, stream));
      if (v) HOT_CUDA(cudaMemcpyAsync(v, sv, sizeof(double) * 3 * total, cudaMemcpyDeviceToHost, stream));
      if (F) HOT_CUDA(cudaMemcpyAsync(F, sF, sizeof(double) * 9 * total, cudaMemcpyDeviceToHost, stream));
      if (C) HOT_CUDA(cudaMemcpyAsync(C, sC, sizeof(double) * 9 * total, cudaMemcpyDeviceToHost, stream));
      prof_end(h, (double)total * 24 * 8);
      sync();
      return;
    }
    stage.ensure(sizeof(double) * 24 * std::max<long long>(np, 1));
    struct Field {
      const DBuf* src;
      double* dst;
      int comps;
      long long off;
    } fields[4] = {{&px, x, 3, 0}, {&pv, v, 3, 3}, {&pF, F, 9, 6}, {&pC, C, 9, 15}};
    if (np > 0) {  // un-permute every field, then the device->host copies back to back
      for (const Field& f : fields)
        if (f.dst)
          launch_soa_to_aos_perm(f.src->as<double>(), stage.as<double>() + f.off * np, np, f.comps, porig.as<int>(),
                                 stream);
      for (const Field& f : fields)
        if (f.dst)
          HOT_CUDA(cudaMemcpyAsync(f.dst, stage.as<double>() + f.off * np, sizeof(double) * f.comps * np,
                                   cudaMemcpyDeviceToHost, stream));
    }
    prof_end(h, (double)np * 24 * 8);
    sync();
  }

  /// Plastic volume ratio J_p in the caller's particle order (snow materials; extension).
  void set_plastic_state(const double* Jp) {
    if (!track_jp) throw std::invalid_argument("no snow material: there is no plastic state");
    if (np == 0) return;
    // the caller's array has every particle; local slot t holds original id porig[t]
    stage.ensure(sizeof(double) * std::max<long long>(np_global, 1));
    HOT_CUDA(cudaMemcpyAsync(stage.p, Jp, sizeof(double) * np_global, cudaMemcpyHostToDevice, stream));
    launch_gather_perm(stage.as<double>(), pjp.as<double>(), np, porig.as<int>(), stream);
    sync();
  }
  void get_plastic_state(double* Jp) {
    if (np_global == 0) return;
    if (!track_jp) {
      std::fill(Jp, Jp + np_global, 1.0);
      return;
    }
    if (pp_on) {
      const long long total = pp_gather_owned_records();
      stage.ensure(sizeof(double) * std::max<long long>(total, 1));
      launch_pp_unpack_caller(pp_send.as<double>(), total, nullptr, nullptr, nullptr, nullptr, stage.as<double>(),
                              stream);
      HOT_CUDA(cudaMemcpyAsync(Jp, stage.p, sizeof(double) * total, cudaMemcpyDeviceToHost, stream));
      sync();
      return;
    }
    stage.ensure(sizeof(double) * std::max<long long>(np, 1));
    launch_soa_to_aos_perm(pjp.as<double>(), stage.as<double>(), np, 1, porig.as<int>(), stream);
    HOT_CUDA(cudaMemcpyAsync(Jp, stage.p, sizeof(double) * np, cudaMemcpyDeviceToHost, stream));
    sync();
  }

  // ------------------------------------------------------------------ step stages
  /// activate_grid (grid.hpp:137-165) + particle binning by stencil centre.
  void activate() {
    const int h = prof_begin(P_ACTIVATE);
    const ParticlesView P = pview();
    int init[8] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN, 0, 0};
    HOT_CUDA(cudaMemcpyAsync(bounds.p, init, sizeof(init), cudaMemcpyHostToDevice, stream));
    launch_particle_bounds(P, dx, bounds.as<int>(), bounds.as<int>() + 6, stream);
    int hb[8];
    HOT_CUDA(cudaMemcpyAsync(hb, bounds.p, sizeof(hb), cudaMemcpyDeviceToHost, stream));
    sync();
    if (pp_on) {  // partitioned particles: the bounding box (and the failure flag) of all ranks
      const auto all = allgather_block(hb, sizeof(hb));
      const int* v = reinterpret_cast<const int*>(all.data());
      for (int r = 0; r < comm->size; ++r)
        for (int a = 0; a < 3; ++a) {
          hb[a] = std::min(hb[a], v[8 * r + a]);
          hb[3 + a] = std::max(hb[3 + a], v[8 * r + 3 + a]);
          hb[6] = std::max(hb[6], v[8 * r + 6]);
        }
    }
    if (hb[6]) throw std::invalid_argument("activate_grid: non-finite particle position");
    Level& l0 = L[0];
    if (np_global == 0) {
      l0.n = 0;
      for (int a = 0; a < 3; ++a) l0.lo[a] = 0, l0.ext[a] = 1;
    } else {
      for (int a = 0; a < 3; ++a) {
        l0.lo[a] = hb[a];
        l0.ext[a] = hb[3 + a] + 2 - hb[a] + 1;
      }
    }
    const long long len = (long long)l0.ext[0] * l0.ext[1] * l0.ext[2];
    if (len > (1LL << 31)) throw std::invalid_argument("activate_grid: particle bounding box exceeds 2^31 nodes");
    l0.flags.ensure(len + 16);
    l0.map.ensure(sizeof(int) * len);
    scan_tmp.ensure(sizeof(int) * (len / 4096 + 64));
    HOT_CUDA(cudaMemsetAsync(l0.flags.p, 0, len + 16, stream));
    DenseMap dm = l0.dmap();
    launch_mark_active(P, dx, dm, l0.flags.as<uint8_t>(), stream);
    if (pp_on) {  // each rank's flags are exact on its own planes: put the slabs together
      const int R = comm->size;
      const long long plane = (long long)l0.ext[1] * l0.ext[2];
      std::vector<long long> off(R + 1);
      for (int r = 0; r <= R; ++r) {
        const int pl = r == R ? l0.lo[0] + l0.ext[0] : std::max(l0.lo[0], std::min(pp_owned_lo(r), l0.lo[0] + l0.ext[0]));
        off[r] = (long long)(pl - l0.lo[0]) * plane;
      }
      off[0] = 0;
      comm->allgather_ranges(l0.flags.p, off, stream);
    }
    // coords sized for the worst case (every box node active) only when needed
    l0.coords.ensure(sizeof(int) * 3 * std::min<long long>(len, 27LL * std::max<long long>(np_global, 1)));
    launch_flags_to_index(l0.flags.as<uint8_t>(), len, l0.ext, l0.lo, l0.map.as<int>(), l0.coords.as<int>(),
                          scan_tmp.as<int>(), iflags.as<int>() + 8, stream);
    int n_nodes = 0;
    HOT_CUDA(cudaMemcpyAsync(&n_nodes, iflags.as<int>() + 8, sizeof(int), cudaMemcpyDeviceToHost, stream));
    sync();
    l0.n = n_nodes;
    const int n = n_nodes;
    gmass.ensure(sizeof(double) * std::max(n, 1));
    gvel.ensure(sizeof(double) * 3 * std::max(n, 1));
    gmom.ensure(sizeof(double) * 3 * std::max(n, 1));
    gbc.ensure(sizeof(double) * 3 * std::max(n, 1));
    gcn.ensure(sizeof(double) * std::max(n, 1));
    l0.dir.ensure(std::max(n, 1));
    bin_of.ensure(sizeof(int) * std::max<long long>(np, 1));
    bin_counts.ensure(sizeof(int) * (n + 2));
    bin_start.ensure(sizeof(int) * (n + 2));
    bin_cursor.ensure(sizeof(int) * (n + 2));
    bin_pid.ensure(sizeof(int) * std::max<long long>(np, 1));
    scan_tmp.ensure(sizeof(int) * ((long long)n / 4096 + 64 + len / 4096));
    launch_bin_particles(P, dx, l0.dmap(), n, bin_of.as<int>(), bin_counts.as<int>(), bin_start.as<int>(),
                         bin_cursor.as<int>(), bin_pid.as<int>(), scan_tmp.as<int>(), porig.as<int>(), stream);
    // store the particles in bin order (orig keeps the caller's order for download)
    ParticlesView Q = P;
    Q.x = qx.as<double>();
    Q.v = qv.as<double>();
    Q.F = qF.as<double>();
    Q.C = qC.as<double>();
    Q.mass = qmass.as<double>();
    Q.vol = qvol.as<double>();
    Q.mat = qmat.as<int>();
    Q.Jp = track_jp ? qjp.as<double>() : nullptr;
    pbin.ensure(sizeof(int) * std::max<long long>(np, 1));
    Q.bin = pbin.as<int>();
    launch_reorder_particles(P, Q, bin_pid.as<int>(), bin_of.as<int>(), porig.as<int>(), qorig.as<int>(), stream);
    px.swap(qx);
    pv.swap(qv);
    pF.swap(qF);
    pC.swap(qC);
    pmass.swap(qmass);
    pvol.swap(qvol);
    pmat.swap(qmat);
    porig.swap(qorig);
    if (track_jp) pjp.swap(qjp);
    nb27.ensure(sizeof(int) * 27 * std::max(n, 1));
    bin_part.ensure(sizeof(double) * 135 * std::max(n, 1));  // per (bin, stencil position): P2G 5, gradient 3
    launch_fill_nb27(gview(), nb27.as<int>(), stream);
    prof_end(h, (double)np * 24 * 3 + 5.0 * len);
    nlevels = 0;
    have_H = false;
  }

  void p2g_bc(double time_now) {
    const int h = prof_begin(P_P2G);
    if (sh.planned) {  // slabs: bins [P-1, Q+1), the slab's rows, then every rank's rows to all
      const int n = L[0].n;
      HOT_CUDA(cudaMemsetAsync(L[0].dir.p, 0, std::max(n, 1), stream));
      HOT_CUDA(cudaMemsetAsync(gbc.p, 0, sizeof(double) * 3 * std::max(n, 1), stream));
      launch_p2g(pview(), bview(), gview(), dx, mats_d.as<DevMaterial>(), cn_factor * dx * dx, dt,
                 bin_part.as<double>(), stream, sh.b_lo, sh.b_hi, sh.r_lo, sh.r_hi);
      prof_end(h, (double)(sh.p_hi - sh.pe_lo) * 136 + (double)(sh.r_hi - sh.r_lo) * 88);
      gather_rows0(gmass.p, 8);
      gather_rows0(gmom.p, 24);
      gather_rows0(gvel.p, 24);
      gather_rows0(gcn.p, 8);
      const int h2 = prof_begin(P_P2G);
      launch_apply_bc(gview(), dx, cols_d.as<DevCollider>(), (int)cols_h.size(), stream);
      prof_end(h2);
      return;
    }
    launch_p2g(pview(), bview(), gview(), dx, mats_d.as<DevMaterial>(), cn_factor * dx * dx, dt, bin_part.as<double>(),
               stream);
    launch_apply_bc(gview(), dx, cols_d.as<DevCollider>(), (int)cols_h.size(), stream);
    (void)time_now;
    prof_end(h, (double)np * 136 + (double)L[0].n * 88);  // x v C m mat | mass mom vel cn dir bc
  }

  void ensure_solver_buffers() {
    const int n = std::max(L[0].n, 1);
    const size_t v = sizeof(double) * 3 * n;
    dv.ensure(v);
    g.ensure(v);
    gnew.ensure(v);
    pdir.ensure(v);
    q.ensure(v);
    vout.ensure(v);
    stress.ensure(sizeof(double) * 9 * std::max<long long>(np, 1));
  }

  /// hot_stage_prepare / advance_step :297-305 at a given dt.
  void prepare(double dt_in, double time_now) {
    dt = dt_in;
    activate();
    // the slab cut of this step's grid (replicated inputs: every rank computes the same cut)
    const int levels = cfg.kind == 0 ? cfg.levels : 0;  // HOT is the solver that splits
    sh.planned = want_shard(levels) && plan_shard();
    if (pp_on && !sh.planned) {  // the frozen cut no longer fits: every particle back everywhere
      pp_gather_all();
      activate();
      sh.planned = want_shard(levels) && plan_shard();
    }
    p2g_bc(time_now);
    ensure_solver_buffers();
    have_state = true;
    check_launch();
  }

  // ------------------------------------------------------------------ slabs
  /// The slab-sharded solve: HOT / LBFGS-H solves with a coarse level under the linear
  /// embedding, when a transport with more than one rank is attached.
  bool want_shard(int levels) const {
    // HOT_SHARD_FORCE=1 (test hook): take the sharded path with one rank too, so the transport's
    // calls run on a one-GPU box (one slab; halos have no peer, gathers broadcast to self)
    return comm && (comm->size > 1 || opt.shard_force) && cfg.embedding == 1 && levels >= 2;
  }
  /// First level-0 row at or after absolute lattice plane `plane` (axis 0).
  int row_of(int plane) const {
    const int k = std::min(std::max(plane - L[0].lo[0], 0), L[0].ext[0]);
    return sh.ps0[k];
  }
  /// Cuts the level-0 rows into slabs of lattice planes.  Every input is replicated, so every
  /// rank computes the same cut without communicating.  False: too few planes to cut (the
  /// solve then runs replicated on every rank).
  bool plan_shard() {
    const Level& l0 = L[0];
    const int R = comm->size, me = comm->rank;
    const int np0 = l0.ext[0];
    if (l0.n == 0) return false;
    plane_buf.ensure(sizeof(int) * (np0 + 2));
    launch_plane_starts(l0.coords.as<int>(), l0.n, l0.lo[0], np0, plane_buf.as<int>(), stream);
    sh.ps0.resize(np0 + 1);
    HOT_CUDA(cudaMemcpyAsync(sh.ps0.data(), plane_buf.p, sizeof(int) * (np0 + 1), cudaMemcpyDeviceToHost, stream));
    sync();
    std::vector<long long> w(np0);
    for (int k = 0; k < np0; ++k) w[k] = sh.ps0[k + 1] - sh.ps0[k];  // rows per plane
    sh.bounds.assign(R + 1, 0);
    if (pp_on) {  // the partitioned particles follow the cut that partitioned them
      sh.bounds = pp_bounds;
      sh.bounds[0] = l0.lo[0];
      sh.bounds[R] = l0.lo[0] + np0;
      for (int r = 0; r < R; ++r)
        if (sh.bounds[r + 1] - sh.bounds[r] < 2) return false;  // caller gathers and re-plans
    } else {
      // interior cuts at even planes (the level-1 cut is then exact: coarse plane = fine / 2) and
      // at least 2 planes per slab (a row's coupling radius: halos come from one neighbour)
      if (!plan_slabs(l0.lo[0], np0, w.data(), R, 2, 2, sh.bounds.data())) return false;
    }
    sh.P = sh.bounds[me];
    sh.Q = sh.bounds[me + 1];
    sh.r_lo = row_of(sh.P);
    sh.r_hi = row_of(sh.Q);
    // assembly writes each upper block and its transpose: a row's lower blocks come from rows up
    // to 2 planes left.  Level-1 rows [P/2, Q/2) are complete when the coarse rows 2 coarse
    // planes further left are computed too (their transposes), which read X of fine children
    // from plane P-5 on, whose rows need the assembly from plane P-7 on, which reads the bins
    // (particle tensors) from plane P-8 on.
    sh.a_lo = row_of(sh.P - 7);
    sh.x_lo = row_of(sh.P - 5);
    sh.h_hi = row_of(sh.Q + 2);
    sh.b_lo = row_of(sh.P - 1);
    sh.b_hi = row_of(sh.Q + 1);
    const int prow[3] = {row_of(sh.P - 8), sh.b_hi, sh.b_lo};
    int pb[3] = {0, 0, 0};
    for (int k = 0; k < 3; ++k)
      HOT_CUDA(cudaMemcpyAsync(&pb[k], bin_start.as<int>() + prow[k], sizeof(int), cudaMemcpyDeviceToHost, stream));
    sync();
    sh.p_lo = pb[0];
    sh.p_hi = pb[1];
    sh.pe_lo = pb[2];
    sh.row_off.assign(R + 1, 0);
    for (int r = 0; r <= R; ++r) sh.row_off[r] = row_of(sh.bounds[r]);
    // halo after the waves of residue group m (colours 9m .. 9m+8, sgs0_sharded): only the edge
    // plane with axis-0 residue m changed; each side sends that one plane (or nothing)
    auto md3 = [](int v) { return ((v % 3) + 3) % 3; };
    for (int m = 0; m < 3; ++m) {
      std::vector<long long>& e = sh.halo_edges[m];
      e.assign(4 * R, 0);
      for (int r = 0; r < R; ++r) {
        for (int pl = sh.bounds[r]; pl < sh.bounds[r] + 2; ++pl)
          if (md3(pl) == m) e[4 * r] = 24LL * row_of(pl), e[4 * r + 1] = 24LL * row_of(pl + 1);
        for (int pl = sh.bounds[r + 1] - 2; pl < sh.bounds[r + 1]; ++pl)
          if (md3(pl) == m) e[4 * r + 2] = 24LL * row_of(pl), e[4 * r + 3] = 24LL * row_of(pl + 1);
      }
    }
    return true;
  }

  // ------------------------------------------------------------------ particle partition
  bool pp_enabled() const { return comm != nullptr && !opt.shard_replicate; }
  int pp_owned_lo(int r) const { return r == 0 ? -(1 << 29) : pp_bounds[r]; }
  int pp_owned_hi(int r) const { return r == comm->size - 1 ? (1 << 29) : pp_bounds[r + 1]; }

  /// Every rank's `bytes` bytes (one allgather over a small device buffer).
  std::vector<unsigned char> allgather_block(const void* mine, size_t bytes) {
    const int R = comm->size;
    pp_small.ensure(bytes * R);
    HOT_CUDA(cudaMemcpyAsync(pp_small.as<unsigned char>() + bytes * comm->rank, mine, bytes, cudaMemcpyHostToDevice,
                             stream));
    std::vector<long long> off(R + 1);
    for (int r = 0; r <= R; ++r) off[r] = (long long)bytes * r;
    sync();
    comm->allgather_ranges(pp_small.p, off, stream);
    std::vector<unsigned char> out(bytes * R);
    HOT_CUDA(cudaMemcpyAsync(out.data(), pp_small.p, bytes * R, cudaMemcpyDeviceToHost, stream));
    sync();
    return out;
  }
  std::vector<long long> allgather_ll(long long mine) {
    const auto b = allgather_block(&mine, 8);
    std::vector<long long> v(comm->size);
    std::memcpy(v.data(), b.data(), 8 * v.size());
    return v;
  }
  /// Exclusive scan of n flags into pos; returns the total.
  long long pp_scan(const int* flag, int* pos, long long n) {
    if (n == 0) return 0;
    if (n > (long long)INT_MAX - 4096) throw std::invalid_argument("particle partition: too many particles per rank");
    scan_tmp.ensure(sizeof(int) * (n / 4096 + 64));
    launch_exclusive_scan(flag, pos, (int)n, scan_tmp.as<int>(), iflags.as<int>() + 9, stream);
    int t = 0;
    HOT_CUDA(cudaMemcpyAsync(&t, iflags.as<int>() + 9, sizeof(int), cudaMemcpyDeviceToHost, stream));
    sync();
    return t;
  }
  void pp_flags(long long n) {
    const size_t b = sizeof(int) * (size_t)std::max<long long>(n + 1, 1);
    pp_keep.ensure(b);
    pp_pack.ensure(b);
    pp_kpos.ensure(b);
    pp_ppos.ensure(b);
  }
  /// The local particles become the kept ones, then the kept records (in that order).
  void pp_rebuild(long long n_keep, const double* rec, long long mrec, long long n_recv) {
    const long long nn = n_keep + n_recv;
    const size_t n3 = sizeof(double) * 3 * std::max<long long>(nn, 1), n9 = sizeof(double) * 9 * std::max<long long>(nn, 1);
    const size_t n1 = sizeof(double) * std::max<long long>(nn, 1), i1 = sizeof(int) * std::max<long long>(nn, 1);
    qx.ensure(n3);
    qv.ensure(n3);
    qF.ensure(n9);
    qC.ensure(n9);
    qmass.ensure(n1);
    qvol.ensure(n1);
    qmat.ensure(i1);
    qorig.ensure(i1);
    if (track_jp) qjp.ensure(n1);
    ParticlesView Q = pview();
    Q.x = qx.as<double>();
    Q.v = qv.as<double>();
    Q.F = qF.as<double>();
    Q.C = qC.as<double>();
    Q.mass = qmass.as<double>();
    Q.vol = qvol.as<double>();
    Q.mat = qmat.as<int>();
    Q.Jp = track_jp ? qjp.as<double>() : nullptr;
    Q.n = nn;
    launch_pp_rebuild(pview(), porig.as<int>(), pp_keep.as<int>(), pp_kpos.as<int>(), rec, mrec,
                      pp_rflag.as<int>(), pp_rpos.as<int>(), n_keep, Q, qorig.as<int>(), stream);
    px.swap(qx);
    pv.swap(qv);
    pF.swap(qF);
    pC.swap(qC);
    pmass.swap(qmass);
    pvol.swap(qvol);
    pmat.swap(qmat);
    porig.swap(qorig);
    if (track_jp) pjp.swap(qjp);
    np = nn;
    sync();
    check_launch();
  }
  /// Records of this rank's particles flagged in pp_pack (positions pp_ppos, n_pack of them),
  /// gathered from every rank into pp_send; returns the total record count.
  long long pp_allgather_records(long long n_pack) {
    const int R = comm->size, me = comm->rank;
    const auto counts = allgather_ll(n_pack);
    std::vector<long long> off(R + 1, 0);
    for (int r = 0; r < R; ++r) off[r + 1] = off[r] + counts[r];
    const long long total = off[R];
    const int rec = pp_record_doubles();
    pp_send.ensure(sizeof(double) * rec * std::max<long long>(total, 1));
    launch_pp_pack(pview(), porig.as<int>(), pp_pack.as<int>(), pp_ppos.as<int>(), dx,
                   pp_send.as<double>() + off[me] * rec, stream);
    std::vector<long long> boff(R + 1);
    for (int r = 0; r <= R; ++r) boff[r] = off[r] * rec * (long long)sizeof(double);
    sync();
    comm->allgather_ranges(pp_send.p, boff, stream);
    return total;
  }
  /// After a sharded step: every rank keeps its owned particles that stay inside
  /// its slab away from the copied bands, and sends the others (leaving the slab, or within
  /// kPPLeft planes of Q / kPPRight planes of P, which other ranks copy) to all ranks; each rank
  /// keeps the records inside its band.  The first call (every rank holds every particle) only
  /// filters.  Owners are decided by the stencil-centre plane after advection.
  void pp_exchange() {
    const int me = comm->rank;
    const long long n = np;
    pp_flags(n);
    const int olo = pp_owned_lo(me), ohi = pp_owned_hi(me);
    if (!pp_on) {
      launch_pp_classify(pview(), nullptr, olo - kPPLeft, ohi + kPPRight, INT_MIN, INT_MAX, 0, 0, dx, pp_keep.as<int>(),
                         pp_pack.as<int>(), stream);
      const long long n_keep = pp_scan(pp_keep.as<int>(), pp_kpos.as<int>(), n);
      pp_rebuild(n_keep, nullptr, 0, 0);
      pp_on = true;
      return;
    }
    launch_pp_classify(pview(), L[0].coords.as<int>(), olo, ohi, olo, ohi, kPPLeft, kPPRight, dx, pp_keep.as<int>(),
                       pp_pack.as<int>(), stream);
    const long long n_keep = pp_scan(pp_keep.as<int>(), pp_kpos.as<int>(), n);
    const long long n_pack = pp_scan(pp_pack.as<int>(), pp_ppos.as<int>(), n);
    const long long total = pp_allgather_records(n_pack);
    pp_rflag.ensure(sizeof(int) * std::max<long long>(total + 1, 1));
    pp_rpos.ensure(sizeof(int) * std::max<long long>(total + 1, 1));
    launch_pp_recv_flag(pp_send.as<double>(), total, olo - kPPLeft, ohi + kPPRight, pp_rflag.as<int>(), stream);
    const long long n_recv = pp_scan(pp_rflag.as<int>(), pp_rpos.as<int>(), total);
    pp_rebuild(n_keep, pp_send.as<double>(), total, n_recv);
  }
  /// Every owned particle (plane of its current position in the rank's slab) as records in
  /// pp_send, from every rank (np_global of them).
  long long pp_gather_owned_records() {
    const int me = comm->rank;
    const long long n = np;
    pp_flags(n);
    launch_pp_classify(pview(), nullptr, pp_owned_lo(me), pp_owned_hi(me), pp_owned_lo(me), pp_owned_hi(me), 0, 0, dx,
                       pp_keep.as<int>(), pp_pack.as<int>(), stream);
    // gL = gR = 0: keep = owned and staying; pack = leaving -- here every owned particle is sent
    HOT_CUDA(cudaMemcpyAsync(pp_pack.p, pp_keep.p, sizeof(int) * n, cudaMemcpyDeviceToDevice, stream));
    const long long n_pack = pp_scan(pp_pack.as<int>(), pp_ppos.as<int>(), n);
    const long long total = pp_allgather_records(n_pack);
    if (total != np_global) throw std::logic_error("particle partition: owned particles do not add up");
    return total;
  }
  /// Back to every particle on every rank (before a replicated solve or a stage tap).
  void pp_gather_all() {
    if (!pp_on) return;
    const long long total = pp_gather_owned_records();
    pp_rflag.ensure(sizeof(int) * std::max<long long>(total + 1, 1));
    pp_rpos.ensure(sizeof(int) * std::max<long long>(total + 1, 1));
    launch_pp_recv_flag(pp_send.as<double>(), total, INT_MIN, INT_MAX, pp_rflag.as<int>(), stream);
    const long long n_recv = pp_scan(pp_rflag.as<int>(), pp_rpos.as<int>(), total);
    pp_flags(np);
    HOT_CUDA(cudaMemsetAsync(pp_keep.p, 0, sizeof(int) * std::max<long long>(np, 1), stream));
    pp_rebuild(0, pp_send.as<double>(), total, n_recv);
    pp_on = false;
    have_state = false;
  }

  /// Level-1 cut: coarse planes [P/2, Q/2) (interior cuts are even).
  void plan_shard_coarse() {
    const Level& l1 = L[1];
    const int R = comm->size, me = comm->rank;
    const int np1 = l1.ext[0];
    plane_buf.ensure(sizeof(int) * (np1 + 2));
    launch_plane_starts(l1.coords.as<int>(), l1.n, l1.lo[0], np1, plane_buf.as<int>(), stream);
    std::vector<int> ps1(np1 + 1);
    HOT_CUDA(cudaMemcpyAsync(ps1.data(), plane_buf.p, sizeof(int) * (np1 + 1), cudaMemcpyDeviceToHost, stream));
    sync();
    auto crow = [&](int plane) { return ps1[std::min(std::max(plane - l1.lo[0], 0), np1)]; };
    sh.crow_off.assign(R + 1, 0);
    for (int r = 1; r < R; ++r) sh.crow_off[r] = crow(sh.bounds[r] / 2);
    sh.crow_off[R] = l1.n;
    sh.c_lo = (int)sh.crow_off[me];
    sh.c_hi = (int)sh.crow_off[me + 1];
    sh.gc_lo = me == 0 ? 0 : crow(sh.bounds[me] / 2 - 2);
  }

  /// Rows [row_off[r], row_off[r+1]) of a level-0 node array (`bytes` per row) from their
  /// owners to every rank.
  void gather_rows0(void* vec, int bytes = 24) {
    const int h = prof_begin(P_COMM);
    std::vector<long long> off(sh.row_off.size());
    for (size_t r = 0; r < off.size(); ++r) off[r] = (long long)bytes * sh.row_off[r];
    comm->allgather_ranges(vec, off, stream);
    prof_end(h, (double)off.back());
  }

  /// smooth_sgs on level 0 (multigrid.hpp:298-316) over this rank's rows: the 27 colour waves
  /// forward then backward, exactly the single-GPU schedule.  Colour c = 9 (x mod 3) + ... :
  /// waves 9m .. 9m+8 update only the planes x = m (mod 3), and a row reads its own plane and
  /// the planes within 2 of it, which have other residues and stay fixed during the group.
  /// So a plane's values are final at the end of its residue group, and one halo per group
  /// (the edge plane of that residue, to each neighbour) gives every row exactly the values the
  /// serial sweep reads: at most 5 exchanges per smoother call instead of 54 (see below).
  void sgs0_sharded(double* u, const double* b, bool gathered_after) {
    const Level& l = L[0];
    const LevelView v = l.view();
    // the sweep as 5 segments of the flat (forward waves 0..26, backward 26..0) sequence:
    // forward groups 0 and 1, forward + backward group 2 together, backward groups 1 and 0.
    // A residue-m plane is read by the neighbour only in groups != m, so the values between
    // the forward and backward group 2 are never read across the cut: no halo there.  The
    // last halo is skipped when the caller gathers every row right after (post-smoothing).
    struct Seg {
      int q0, q1, grp;
    };
    const Seg segs[5] = {{0, 9, 0}, {9, 18, 1}, {18, 36, 2}, {36, 45, 1}, {45, 54, 0}};
    auto wave_of_q = [](int q) { return q < 27 ? q : 53 - q; };
    for (int si = 0; si < 5; ++si) {
      const Seg& sg = segs[si];
      const int h = prof_begin(P_SGS0);
      long long rows = 0;
      int big = 0;
      for (int q = sg.q0; q < sg.q1; ++q) {
        const int c = wave_of_q(q);
        rows += sh.wave_start[c + 1] - sh.wave_start[c];
        big = std::max(big, sh.wave_start[c + 1] - sh.wave_start[c]);
      }
      // the segment's waves in one persistent bulk-copy launch (grid barrier between waves,
      // ~2 us) unless they are tiny (then one launch per wave)
      if (big >= std::min(512, opt.stream_min_rows)) {
        launch_sgs_stream(v, sh.wave_starts.as<int>(), sh.wave_rows.as<int>(), 27, u, b, grid_bar.as<unsigned int>(),
                          stream, sg.q0, sg.q1, big);
      } else {
        for (int q = sg.q0; q < sg.q1; ++q) {
          const int c = wave_of_q(q);
          const int cnt = sh.wave_start[c + 1] - sh.wave_start[c];
          launch_sgs_wave1(v, sh.wave_rows.as<int>() + sh.wave_start[c], cnt, u, b, stream);
        }
      }
      prof_end(h, (double)rows * (72.0 * 125 + 72 + 24 + 48));
      if (si == 4 && gathered_after) break;
      const std::vector<long long>& e = sh.halo_edges[sg.grp];
      bool any = false;
      for (long long x : e) any |= x != 0;
      if (any) {  // replicated: every rank makes the same decision
        const int hc = prof_begin(P_COMM);
        comm->halo(u, e, stream);
        prof_end(hc);
      }
    }
  }


  // ------------------------------------------------------------------ objective
  int* flag_bad() { return iflags.as<int>() + 0; }

  /// E(dv + alpha p) with stress stored for the gradient; returns through scal[0].  Per-particle
  /// energies, per-node totals (bin + node terms), then a fixed-tree sum over the nodes: the
  /// value does not depend on the slab cut.  Slabs: the particles of bins [P-1, Q+1) (the
  /// gradient's stress), or [P-8, Q+1) when the SVD cache feeds the assembly; the node totals of
  /// the slab's rows, gathered.
  void energy_async(const double* dvp, const double* p, double alpha, bool want_stress, bool store_svd = false) {
    int h = prof_begin(P_ENERGY);
    double* part = partials.as<double>();
    const int n = L[0].n;
    node_u.ensure(sizeof(double) * 3 * std::max(n, 1));
    pe_buf.ensure(sizeof(double) * std::max<long long>(np, 1));
    ne_buf.ensure(sizeof(double) * std::max(n, 1));
    launch_node_u(gview(), dvp, p, alpha, node_u.as<double>(), stream);
    if (store_svd) svd.ensure(sizeof(double) * 21 * std::max<long long>(np, 1));
    long long plo = 0, phi = -1;
    int lo = 0, hi = n;
    if (sh.on) {
      plo = store_svd ? sh.p_lo : sh.pe_lo;
      phi = sh.p_hi;
      lo = sh.r_lo;
      hi = sh.r_hi;
    }
    launch_particle_energy(pview(), gview(), dx, dt, mats_d.as<DevMaterial>(), node_u.as<double>(),
                           want_stress ? stress.as<double>() : nullptr, store_svd ? svd.as<double>() : nullptr,
                           pe_buf.as<double>(), nred, flag_bad(), stream, plo, phi);
    launch_node_energy(gview(), bview(), pe_buf.as<double>(), dt, grav, dvp, p, alpha, ne_buf.as<double>(), lo, hi,
                       stream);
    prof_end(h, (double)(phi < 0 ? np : phi - plo) * (24 + 72 + 8 + 4 + 27 * 28 + 16) +
                    (want_stress ? 72.0 * (phi < 0 ? np : phi - plo) : 0.0));
    if (sh.on) gather_rows0(ne_buf.p, 8);
    launch_sum_array(ne_buf.as<double>(), n, part, nred, stream);
    launch_sum_partials(part, nred, scal.as<double>() + 0, stream);
  }

  /// g(dv) from the stored stress; scaled-norm^2 into scal[2].  Slabs: the bin pass over bins
  /// [P-1, Q+1), the node pass over the slab's rows, then g and the norm terms gathered.
  void gradient_async(const double* dvp, double* gout) {
    const int h = prof_begin(P_GRADIENT);
    double* part = partials.as<double>() + 2 * nred;
    const int n = L[0].n;
    nt_buf.ensure(sizeof(double) * std::max(n, 1));
    if (sh.on)
      launch_node_gradient(pview(), bview(), gview(), dx, dt, grav, stress.as<double>(), dvp, gout,
                           bin_part.as<double>(), nt_buf.as<double>(), flag_bad(), stream, sh.b_lo, sh.b_hi, sh.r_lo,
                           sh.r_hi);
    else
      launch_node_gradient(pview(), bview(), gview(), dx, dt, grav, stress.as<double>(), dvp, gout,
                           bin_part.as<double>(), nt_buf.as<double>(), flag_bad(), stream);
    prof_end(h, 96.0 * np + 64.0 * n);  // x, V P F^T | dv, mass, g
    if (sh.on) {
      gather_rows0(gout, 24);
      gather_rows0(nt_buf.p, 8);
    }
    launch_sum_array(nt_buf.as<double>(), n, part, nred, stream);
    launch_sum_partials(part, nred, scal.as<double>() + 2, stream);
  }

  void check_flags() {
    if (host_int[0] == 1) throw std::invalid_argument("energy: non-finite dv");
    if (host_int[0] == 2) throw std::logic_error("scaled_norm: zero characteristic scale (material misconfiguration)");
    if (host_int[1] == 1) throw SolverFailure("pcg: preconditioner is not positive definite");
    if (host_int[1] == 2) throw SolverFailure("pcg: system matrix is not positive definite");
  }

  // ------------------------------------------------------------------ matrix + hierarchy
  /// H rows [row0, row0 + rows) (default: all rows); every other array covers all rows.
  void alloc_level(Level& l, int row0 = 0, int rows = -1) {
    const long long n = std::max(l.n, 1);
    l.cols.ensure(sizeof(int) * n * l.pitch());
    l.h_row0 = row0;
    l.H.ensure(sizeof(double) * std::max<long long>(rows < 0 ? n : rows, 1) * 9 * l.pitch());
    l.dinv.ensure(sizeof(double) * 9 * n);
    l.b.ensure(sizeof(double) * 3 * n);
    l.u.ensure(sizeof(double) * 3 * n);
    l.r.ensure(sizeof(double) * 3 * n);
    l.wave_of.ensure(sizeof(int) * n);
    l.wave_rows.ensure(sizeof(int) * n);
  }

  /// Level-0 assembly by bins (k_bin_pairs, then k_row_gather).  The bins' pair sums
  /// go through a ring: all bins at once when they fit, else bands of bins, each followed by the
  /// rows it completes (a row's bins lie within s_bound indices of it, so after the band
  /// [b0, b1) every row whose largest neighbour bin is below b1 can finish, and the smallest
  /// bin it reads is above b0 - 2 s_bound).
  void assemble_by_bins(const LevelView& v0, double flops) {
    Level& l0 = L[0];
    const int n = l0.n;
    const int s_bound = l0.ext[1] * l0.ext[2] + l0.ext[2] + 2;
    // bins that can have a node among this rank's rows (slabs: the slab and a margin)
    const bool all = v0.lo <= 0 && v0.hi >= n;
    const int jbeg = all ? 0 : std::max(0, v0.lo - s_bound), jend = all ? n : std::min(n, v0.hi + s_bound);
    const int ring_cap = (int)std::max<long long>(
        std::min<long long>(jend - jbeg, std::max<long long>(4LL * s_bound, opt.asm_ring_bins)), 1);
    asm_pairs.ensure(sizeof(double) * asm_pair_doubles() * (size_t)ring_cap);
    double* G = asm_pairs.as<double>();
    const long long plo = sh.on ? sh.p_lo : 0, phi = sh.on ? sh.p_hi : np;
    unsigned int* ctr = grid_bar.as<unsigned int>() + 8;
    unsigned long long* done = active_dev.as<unsigned long long>() + (kMaxLevels - 1);
    HOT_CUDA(cudaMemsetAsync(done, 0, sizeof(unsigned long long), stream));
    const int band = jend - jbeg <= ring_cap ? std::max(jend - jbeg, 1) : ring_cap - 2 * s_bound;
    if (band <= 0) throw std::logic_error("assemble_by_bins: ring smaller than 2 lattice planes");
    if (jend <= jbeg)  // no rows: still leave the column ids and the active-slot count defined
      launch_fill_cols(l0.view(), active_dev.as<unsigned long long>(), stream);
    for (int b0 = jbeg; b0 < jend; b0 += band) {
      const int b1 = std::min(b0 + band, jend);
      const bool first = b0 == jbeg, last = b1 == jend;
      const int ha = prof_begin(P_ASM_PAIRS);
      launch_bin_pairs(bview(), gview(), v0, tu_base(), G, ring_cap, b0, b1, plo, phi, ctr, done, stream);
      prof_end(ha, 0.0, first ? flops : 0.0);
      const int hb = prof_begin(P_ASSEMBLE);
      if (first) launch_fill_cols(l0.view(), active_dev.as<unsigned long long>(), stream);
      launch_row_gather(bview(), gview(), v0, G, ring_cap, first ? v0.lo : std::max(v0.lo, b0 - s_bound),
                        last ? v0.hi : std::min(v0.hi, b1), first ? -1 : b0, last ? 1 << 30 : b1, plo, phi, ctr + 1,
                        stream);
      // algorithmic bytes: the row, its column ids (written and read); the pair sums of every
      // bin with particles are read once (counted on the device, see prof_slot_bytes)
      prof_end(hb, first ? (double)(v0.hi - v0.lo) * (9.0 * kSlotPitch * 8 + 2.0 * kSlotPitch * 4) : 0.0);
      if (first && hb >= 0 && prof_solve + 1 < kProfSolves)
        slot_terms.push_back(SlotTerm{P_ASSEMBLE, prof_solve + 1, kMaxLevels - 1, 8.0 * asm_pair_doubles()});
    }
  }

  /// reuse_svd: the last energy evaluation stored the SVD at exactly this dv (solve_qn start).
  void assemble(const double* dvp, bool project, bool reuse_svd = false) {
    Level& l0 = L[0];
    if (sh.on)  // the rows this rank assembles, plus the 2 planes its transposes reach
      alloc_level(l0, sh.a_lo, sh.h_hi - sh.a_lo);
    else
      alloc_level(l0);
    particle_tensors(dvp, project, reuse_svd);
    LevelView v0 = l0.view();
    if (sh.on) {  // this slab's rows and the rows whose transposes complete them
      v0.lo = sh.a_lo;
      v0.hi = sh.r_hi;
    }
    // algorithmic fp64 work: per particle 27 rows x M (27 x 3 FMA) + 378 upper pairs x 27 FMA
    const double flops = (double)np * 2.0 * (27.0 * 81.0 + 378.0 * 27.0);
    if (opt.asm_tiles) {
      const int h = prof_begin(P_ASSEMBLE);
      launch_fill_cols(l0.view(), active_dev.as<unsigned long long>(), stream);
      launch_assemble_rows(pview(), bview(), gview(), v0, dx, tu_base(), grid_bar.as<unsigned int>() + 8, stream);
      prof_end(h, 0.0, flops);
    } else {
      assemble_by_bins(v0, flops);
    }
    have_H = true;
    nlevels = 1;
  }

  /// Per-particle kappa * dP/dF (projected) and the 27 W_k vectors at dv (assemble_hessian's
  /// particle half, objective.hpp:322-340).
  void particle_tensors(const double* dvp, bool project, bool reuse_svd) {
    int h = prof_begin(P_TENSORS);
    // slabs: records of this rank's particle range only
    tu_lo = sh.on ? sh.p_lo : 0;
    Tu.ensure(sizeof(double) * 126 * std::max<long long>(sh.on ? sh.p_hi - sh.p_lo : np, 1));
    if (!reuse_svd) {
      node_u.ensure(sizeof(double) * 3 * std::max(L[0].n, 1));
      launch_node_u(gview(), dvp, nullptr, 0.0, node_u.as<double>(), stream);
    }
    launch_particle_tensors(pview(), gview(), dx, dt, mats_d.as<DevMaterial>(), node_u.as<double>(),
                            reuse_svd ? svd.as<double>() : nullptr, project ? 1 : 0, tu_base(), flag_bad(), stream,
                            sh.on ? sh.p_lo : 0, sh.on ? sh.p_hi : -1);
    prof_end(h, (double)np * (24 + 72 + 8 + 4 + 126 * 8));  // x F vol mat in, kappa*T (packed) + W out
  }

  /// Wave schedule of level m (multigrid.hpp:241-250 as waves), structure
  /// only (coordinates), on stream st with scan scratch tmp and count scratch cnt.
  void level_waves(int m, cudaStream_t st, DBuf& tmp) {
    Level& l = L[m];
    if (l.n == 0) {
      l.nwaves = 0;
      l.max_wave = 0;
      l.wave_start_h.assign(1, 0);
      return;
    }
    int off[3] = {0, 0, 0};
    int nw = 27;
    const int q = l.radius == 3 ? 3 : 2;  // coarse colour modulus (multigrid.hpp:275)
    if (m > 0) {
      auto fl = [](int v, int k) { return v >= 0 ? v / k : -((-v + k - 1) / k); };
      int span[3];
      for (int a = 0; a < 3; ++a) {
        off[a] = fl(l.lo[a], q);
        span[a] = fl(l.lo[a] + l.ext[a] - 1, q) - off[a] + 1;
      }
      nw = 8 * (q * q * q - 1) + 4 * (span[0] - 1) + 2 * (span[1] - 1) + (span[2] - 1) + 1;
    }
    launch_level_waves(l.view(), m > 0 ? 1 : 0, q, off, l.wave_of.as<int>(), st);
    l.wave_counts.ensure(sizeof(int) * (nw + 2));
    l.wave_start.ensure(sizeof(int) * (nw + 2));
    l.wave_cursor.ensure(sizeof(int) * bucket_scratch_ints(l.n, nw));
    tmp.ensure(sizeof(int) * (bucket_scratch_ints(l.n, nw) / 4096 + 64));
    launch_bucket_rows(l.wave_of.as<int>(), l.n, 0, l.wave_counts.as<int>(), l.wave_start.as<int>(),
                       l.wave_cursor.as<int>(), l.wave_rows.as<int>(), nw, tmp.as<int>(), st);
    std::vector<int> counts(nw);
    HOT_CUDA(cudaMemcpyAsync(counts.data(), l.wave_counts.p, sizeof(int) * nw, cudaMemcpyDeviceToHost, st));
    if (m == 0 && sh.on) {  // this slab's rows per colour, in the same 27 colour buckets
      sh.wave_counts.ensure(sizeof(int) * (nw + 2));
      sh.wave_starts.ensure(sizeof(int) * (nw + 2));
      sh.wave_cursor.ensure(sizeof(int) * bucket_scratch_ints(sh.r_hi - sh.r_lo, nw));
      sh.wave_rows.ensure(sizeof(int) * std::max(sh.r_hi - sh.r_lo, 1));
      launch_bucket_rows(l.wave_of.as<int>(), sh.r_hi - sh.r_lo, 0, sh.wave_counts.as<int>(), sh.wave_starts.as<int>(),
                         sh.wave_cursor.as<int>(), sh.wave_rows.as<int>(), nw, tmp.as<int>(), st, sh.r_lo);
      sh.wave_start.resize(nw + 1);
      HOT_CUDA(cudaMemcpyAsync(sh.wave_start.data(), sh.wave_starts.p, sizeof(int) * (nw + 1), cudaMemcpyDeviceToHost,
                               st));
    }
    HOT_CUDA(cudaStreamSynchronize(st));
    if (m == 0 && sh.on) sh.wave_counts_global = counts;
    std::vector<int> starts;
    int acc = 0;
    l.max_wave = 0;
    for (int w = 0; w < nw; ++w)
      if (counts[w] > 0) {
        starts.push_back(acc);
        acc += counts[w];
        l.max_wave = std::max(l.max_wave, counts[w]);
      }
    starts.push_back(acc);
    l.nwaves = (int)starts.size() - 1;
    l.wave_start_h = starts;
    l.sgs_uf.ensure(sizeof(double) * 3 * std::max(l.n, 1));
    l.sgs_ub.ensure(sizeof(double) * 3 * std::max(l.n, 1));
    l.wave_start_c.ensure(sizeof(int) * starts.size());
    HOT_CUDA(cudaMemcpyAsync(l.wave_start_c.p, starts.data(), sizeof(int) * starts.size(), cudaMemcpyHostToDevice,
                             st));
    HOT_CUDA(cudaStreamSynchronize(st));  // `starts` is a host temporary
  }

  /// build_hierarchy, structure half (multigrid.hpp:127-158, 241-250, 275-284): coarse node
  /// sets, Dirichlet flags, column ids and every level's wave schedule.  Depends only on the
  /// level-0 coordinates and Dirichlet flags, so the solve runs it on a second stream while
  /// the level-0 assembly occupies the GPU.  Returns the number of levels built.
  int build_structure(int levels, int embedding, cudaStream_t st) {
    const int quad = embedding == 1 ? 0 : 1;
    DBuf& tmp = scan_tmp2;
    int* cnt = struct_flags.as<int>();
    level_waves(0, st, tmp);
    int built = 1;
    for (int m = 1; m < levels; ++m) {
      Level& f = L[m - 1];
      Level& c = L[m];
      if (f.n == 0) break;
      for (int a = 0; a < 3; ++a) {  // parents span floor(x/2) (- 1 quadratic) .. floor(x/2) + 1
        c.lo[a] = (f.lo[a] >> 1) - quad;
        c.ext[a] = ((f.lo[a] + f.ext[a] - 1) >> 1) + 1 - c.lo[a] + 1;
      }
      c.radius = quad ? 3 : 2;  // coarse diagonal-storage radius (multigrid.hpp:274)
      const long long len = (long long)c.ext[0] * c.ext[1] * c.ext[2];
      c.flags.ensure(len + 16);
      c.map.ensure(sizeof(int) * len);
      c.coords.ensure(sizeof(int) * 3 * std::min<long long>(len, 8LL * f.n));
      tmp.ensure(sizeof(int) * (len / 4096 + 64));
      HOT_CUDA(cudaMemsetAsync(c.flags.p, 0, len + 16, st));
      launch_mark_parents(f.view(), c.dmap(), quad, c.flags.as<uint8_t>(), st);
      launch_flags_to_index(c.flags.as<uint8_t>(), len, c.ext, c.lo, c.map.as<int>(), c.coords.as<int>(),
                            tmp.as<int>(), cnt, st);
      int nc = 0;
      HOT_CUDA(cudaMemcpyAsync(&nc, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
      HOT_CUDA(cudaStreamSynchronize(st));
      if (nc == 0) break;  // truncated hierarchy (multigrid.hpp:281-284)
      c.n = nc;
      alloc_level(c);
      c.dir.ensure(std::max(nc, 1));
      HOT_CUDA(cudaMemsetAsync(c.dir.p, 0, nc, st));
      launch_coarse_dirichlet(f.view(), c.dmap(), quad, c.dir.as<uint8_t>(), st);
      launch_fill_cols(c.view(), active_dev.as<unsigned long long>() + m, st);
      level_waves(m, st, tmp);
      built = m + 1;
    }
    return built;
  }

  /// build_hierarchy, values half: D^-1 of level 0, then per coarse level the Galerkin
  /// product (multigrid.hpp:162-202) with the fused Dirichlet projection and its D^-1; one
  /// readback for the singular-block check of every level (multigrid.hpp:236-238).
  void build_values(int built) {
    const int h = prof_begin(P_HIER);
    HOT_CUDA(cudaMemsetAsync(iflags.as<int>() + 12, 0, sizeof(int), stream));
    LevelView v0 = L[0].view();
    if (sh.on) {  // D^-1 of this slab's rows (the only level-0 rows it smooths)
      v0.lo = sh.r_lo;
      v0.hi = sh.r_hi;
    }
    launch_level_dinv(v0, iflags.as<int>() + 12, stream);
    nlevels = 1;
    for (int m = 1; m < built; ++m) {
      Level& f = L[m - 1];
      Level& c = L[m];
      const int span = f.radius + 3;  // quadratic X targets per axis
      gal_x.ensure(sizeof(double) * 9 * (c.radius == 3 ? span * span * span : 64) *
                   std::max(m == 1 && sh.on ? sh.r_hi - sh.x_lo : f.n, 1));
      if (m == 1 && sh.on) {
        // this slab's level-1 rows (and the 2 coarse planes whose transposes complete them), then
        // every rank's rows to every rank: levels >= 1 are replicated
        plan_shard_coarse();
        LevelView fv = f.view(), cv = c.view();
        fv.lo = sh.x_lo;
        fv.hi = sh.r_hi;
        cv.lo = sh.gc_lo;
        cv.hi = sh.c_hi;
        // X of the fine rows [x_lo, r_hi) only, indexed by fine row
        launch_galerkin(fv, cv, gal_x.as<double>() - (long long)sh.x_lo * 9 * 64, stream);
        const int hc = prof_begin(P_COMM);
        std::vector<long long> off(sh.crow_off.size());
        for (size_t r = 0; r < off.size(); ++r) off[r] = sh.crow_off[r] * 9LL * c.pitch() * (long long)sizeof(double);
        comm->allgather_ranges(c.H.p, off, stream);
        prof_end(hc, (double)off.back());
      } else {
        launch_galerkin(f.view(), c.view(), gal_x.as<double>(), stream);
      }
      launch_level_dinv(c.view(), iflags.as<int>() + 12, stream);
      nlevels = m + 1;
    }
    // PCG scratch on the coarsest level
    const Level& bot = L[nlevels - 1];
    const size_t v = sizeof(double) * 3 * std::max(bot.n, 1);
    pcg_r.ensure(v);
    pcg_z.ensure(v);
    pcg_p.ensure(v);
    pcg_Ap.ensure(v);
    int singular = 0;
    HOT_CUDA(cudaMemcpyAsync(&singular, iflags.as<int>() + 12, sizeof(int), cudaMemcpyDeviceToHost, stream));
    prof_end(h);
    sync();
    check_launch();
    if (sh.on) {  // flags of sharded kernels: every rank takes the same branch
      int fl[2] = {singular, 0};
      HOT_CUDA(cudaMemcpy(&fl[1], flag_bad(), sizeof(int), cudaMemcpyDeviceToHost));
      comm->allreduce_max(fl, 2, stream);
      singular = fl[0];
      HOT_CUDA(cudaMemcpy(flag_bad(), &fl[1], sizeof(int), cudaMemcpyHostToDevice));
    }
    if (singular) throw std::logic_error("multigrid: singular diagonal block");
  }

  /// build_hierarchy (multigrid.hpp:258-294), linear node embedding, in stream order.
  void build_hierarchy(int levels, int embedding) {
    if (levels < 1) throw std::invalid_argument("build_hierarchy: need at least one level");
    if (levels > kMaxLevels) throw std::invalid_argument("build_hierarchy: too many levels");
    build_values(build_structure(levels, embedding, stream));
  }

  /// build_hierarchy overlapped with the level-0 assembly: the structure half runs on the
  /// second stream (its host round trips wait on that stream only) while the main stream
  /// assembles; the values half joins after both.
  void assemble_and_build_hierarchy(const double* dvp, int levels, int embedding, bool reuse_svd) {
    if (levels < 1) throw std::invalid_argument("build_hierarchy: need at least one level");
    if (levels > kMaxLevels) throw std::invalid_argument("build_hierarchy: too many levels");
    HOT_CUDA(cudaEventRecord(ev_fork, stream));  // level-0 coords and Dirichlet flags are final
    assemble(dvp, true, reuse_svd);
    HOT_CUDA(cudaStreamWaitEvent(stream2, ev_fork, 0));
    const int built = build_structure(levels, embedding, stream2);
    HOT_CUDA(cudaEventRecord(ev_join, stream2));
    HOT_CUDA(cudaStreamWaitEvent(stream, ev_join, 0));
    build_values(built);
  }

  /// Coarse-PCG rows per warp when sizing its cooperative grid.  cfg2 coarse PCG per step: 2
  /// rows per warp 0.309 ms, 4 0.351, 8 0.576, 16 1.046 (more CTAs, each with fewer rows, beat
  /// cheaper grid barriers here; 1 row per warp hits the CTA cap)
  static int pcg_rows_per_warp() { return 2; }

  /// Few, fat CTAs for the cooperative kernels: the grid barrier costs grow with the number of
  /// participating CTAs, while one wave / one PCG row-sweep only has tens to thousands of rows.
  /// At most 2 CTAs per SM.
  static int coop_grid(int max_blocks, int rows, int warps_per_block, int rows_per_warp) {
    const int want = (rows + warps_per_block * rows_per_warp - 1) / (warps_per_block * rows_per_warp);
    return std::max(1, std::min(std::min(max_blocks, 2 * num_sms()), want));
  }

  void sgs(int m, double* u, const double* b) {
    Level& l = L[m];
    const int h = prof_begin(m == 0 ? P_SGS0 : P_SGSC);
    // large waves stream best as plain launches; small waves (coarse levels) run in one
    // persistent cooperative kernel with a grid barrier between waves
    const int stream_min = opt.stream_min_rows;
    const bool per_wave = opt.sgs_level0_waves;
    const bool flow = !opt.sgs_coarse_barrier;
    if (l.radius != 2 || (l.max_wave < stream_min && flow)) {  // radius-3 levels: dataflow kernel only
      launch_sgs_flow(l.view(), l.wave_rows.as<int>(), l.wave_of.as<int>(), u, b, l.sgs_uf.as<double>(),
                      l.sgs_ub.as<double>(), stream);
    } else if (l.max_wave >= stream_min && !per_wave)
      launch_sgs_stream(l.view(), l.wave_start_c.as<int>(), l.wave_rows.as<int>(), l.nwaves, u, b,
                        grid_bar.as<unsigned int>(), stream);
    else if (l.max_wave >= stream_min || l.nwaves > kSgsMaxWavesPersistent)
      launch_sgs_waves(l.view(), l.wave_start_h.data(), l.wave_rows.as<int>(), l.nwaves, u, b, stream);
    else
    {
      long long* trace = nullptr;
      if (opt.sgs_trace) {
        sgs_trace.ensure(sizeof(long long) * 4 * 1025);
        HOT_CUDA(cudaMemsetAsync(sgs_trace.p, 0, sizeof(long long) * 4 * 1025, stream));
        trace = sgs_trace.as<long long>();
      }
      launch_sgs(l.view(), l.wave_start_c.as<int>(), l.wave_rows.as<int>(), l.nwaves, u, b,
                 std::max(1, std::min(sgs_max_blocks(), l.max_wave)), grid_bar.as<unsigned int>(), stream, trace);
      if (trace) {
        std::vector<long long> t(4 * 1025);
        HOT_CUDA(cudaMemcpy(t.data(), trace, sizeof(long long) * t.size(), cudaMemcpyDeviceToHost));
        double stage = 0, comp = 0, tail = 0, bar = 0;
        int nw = std::min(l.nwaves * 2, 1023);
        for (int w = 1; w < nw; ++w) {
          if (!t[4 * w] || !t[4 * w + 1] || !t[4 * w + 3] || !t[4 * (w + 1)]) continue;
          stage += t[4 * w + 1] - t[4 * w];
          tail += t[4 * w + 3] - t[4 * w + 1];
          bar += t[4 * (w + 1)] - t[4 * w + 3];
        }
        const double mhz = (double)(t[4 * (nw - 1) + 2] - t[4 * 1 + 2]) / (double)(t[4 * (nw - 1) + 1] - t[4 * 1 + 1]) * 1e3;
        std::fprintf(stderr, "[hot] sgs level %d trace over %d waves (ns/wave): post-barrier bookkeeping %.0f, "
                     "staging wait %.0f, compute %.0f, barrier %.0f; SM clock %.0f MHz\n", m, nw, stage / nw, comp / nw,
                     tail / nw, bar / nw, mhz);
      }
    }
    prof_end(h, 2.0 * (72.0 * l.n + 24.0 * l.n + 48.0 * l.n));
    prof_slot_bytes(h, m, 2.0 * 72.0);
  }

  /// vcycle (multigrid.hpp:363-392), adaptive coarse mode; coarse iterations accumulate into
  /// iflags[2].
  void vcycle(const double* b0, double* out, bool pinned, int pinned_cap) {
    const int M = nlevels;
    launch_zero_dirichlet_copy(b0, L[0].b.as<double>(), L[0].dir.as<uint8_t>(), L[0].n, stream);
    for (int m = 0; m < M - 1; ++m) {
      Level& l = L[m];
      HOT_CUDA(cudaMemsetAsync(l.u.p, 0, sizeof(double) * 3 * l.n, stream));
      const bool slab = m == 0 && sh.on;
      if (slab)
        sgs0_sharded(l.u.as<double>(), l.b.as<double>(), /*gathered_after=*/false);  // the residual reads halos
      else
        sgs(m, l.u.as<double>(), l.b.as<double>());
      // residual r = b - H u: the level's block-sparse SpMV (H, column ids, u b r)
      const int hs = prof_begin(m == 0 ? P_SPMV0 : P_RESID);
      LevelView lv = l.view();
      if (slab) {
        lv.lo = sh.r_lo;
        lv.hi = sh.r_hi;
      }
      launch_residual(lv, l.b.as<double>(), l.u.as<double>(), l.r.as<double>(), stream);
      const double frac = slab && l.n ? (double)(sh.r_hi - sh.r_lo) / l.n : 1.0;
      prof_end(hs, frac * (4.0 * l.pitch() * l.n + 72.0 * l.n));
      prof_slot_bytes(hs, m, frac * 72.0);
      if (slab) gather_rows0(l.r.p);  // restriction (replicated) reads every fine row
      const int h = prof_begin(P_RESID);
      launch_restrict(l.view(), L[m + 1].view(), l.r.as<double>(), L[m + 1].b.as<double>(), stream);
      prof_end(h, 24.0 * l.n + 24.0 * L[m + 1].n);  // r in, coarse b out
    }
    Level& bot = L[M - 1];
    {
      const int h = prof_begin(P_PCG);
      const double rel = pinned ? 1e-14 : 0.5;
      const int cap = pinned ? pinned_cap : 10000;
      launch_pcg(bot.view(), bot.b.as<double>(), bot.u.as<double>(), pcg_r.as<double>(), pcg_z.as<double>(),
                 pcg_p.as<double>(), pcg_Ap.as<double>(), rel, cap, partials.as<double>() + 6 * nred,
                 iflags.as<int>() + 4, iflags.as<int>() + 2, coop_grid(pcg_max_blocks(), bot.n, 8, pcg_rows_per_warp()),
                 stream);
      prof_end(h);
      // status word -> iflags[1] (max over the solve)
      copy_status();
    }
    for (int m = M - 2; m >= 0; --m) {
      Level& l = L[m];
      const int h = prof_begin(P_PROLONG);
      launch_prolong_add(l.view(), L[m + 1].view(), L[m + 1].u.as<double>(), l.u.as<double>(), stream);
      prof_end(h, 24.0 * L[m + 1].n + 48.0 * l.n);
      if (m == 0 && sh.on)
        sgs0_sharded(l.u.as<double>(), l.b.as<double>(), /*gathered_after=*/true);  // then gather_rows0(u)
      else
        sgs(m, l.u.as<double>(), l.b.as<double>());
    }
    if (sh.on && M > 1) gather_rows0(L[0].u.p);
    HOT_CUDA(cudaMemcpyAsync(out, L[0].u.p, sizeof(double) * 3 * L[0].n, cudaMemcpyDeviceToDevice, stream));
    check_launch();
  }

  void copy_status();

  long long count_active_slots(int m);

  // ------------------------------------------------------------------ L-BFGS (solvers.hpp:82-231)
  struct HistEntry {
    int slot;
    double rho;
  };

  void lbfgs_direction(const std::deque<HistEntry>& hist, double* out) {
    const int hvec = prof_begin(P_VEC);
    const long long n3 = 3LL * L[0].n;
    double* qv = q.as<double>();
    double* part = partials.as<double>();
    launch_neg_copy(g.as<double>(), qv, n3, stream);
    const int m = (int)hist.size();
    // newest -> oldest: alpha_k = rho_k s_k.q ; q -= alpha_k y_k
    for (int k = 0; k < m; ++k) {
      const HistEntry& e = hist[hist.size() - 1 - k];
      const double* yprev = k > 0 ? hist_y[hist[hist.size() - k].slot].as<double>() : nullptr;
      launch_axpy_dot(qv, yprev, coef_a.as<double>(), k - 1, -1.0, hist_s[e.slot].as<double>(), n3, part, nred,
                      stream);
      launch_finalize_coef(part, nred, e.rho, nullptr, k, coef_a.as<double>(), stream);
    }
    if (m > 0)
      launch_axpy_dot(qv, hist_y[hist[0].slot].as<double>(), coef_a.as<double>(), m - 1, -1.0, nullptr, n3, nullptr,
                      nred, stream);
    prof_end(hvec, (4.0 * m + 2) * 8.0 * n3);
    vcycle(qv, out, false, 0);
    const int hv2 = prof_begin(P_VEC);
    // oldest -> newest: beta = rho_k y_k.r ; r += (alpha_k - beta) s_k
    for (int k = m - 1; k >= 0; --k) {
      const HistEntry& e = hist[hist.size() - 1 - k];
      const double* sprev = k < m - 1 ? hist_s[hist[hist.size() - 2 - k].slot].as<double>() : nullptr;
      launch_axpy_dot(out, sprev, coef_b.as<double>(), k + 1, +1.0, hist_y[e.slot].as<double>(), n3, part, nred,
                      stream);
      launch_finalize_coef(part, nred, e.rho, coef_a.as<double>(), k, coef_b.as<double>(), stream);
    }
    if (m > 0)
      launch_axpy_dot(out, hist_s[hist[hist.size() - 1].slot].as<double>(), coef_b.as<double>(), 0, +1.0, nullptr,
                      n3, nullptr, nred, stream);
    prof_end(hv2, (4.0 * m) * 8.0 * n3);
  }

  struct SolveOut {
    int outer = 0;
    long long inner = 0;
    bool converged = false;
  };

  /// accept()'s line search (solvers.hpp:66-78, 169-175): g.p, then Armijo backtracking from
  /// alpha = 1 on E(dv + alpha p).  Returns alpha; e_trial = E at it.  host_int[0..2] hold the
  /// flags after the first trial (iflags[2]: inner iterations of the direction).
  double line_search(const double* pd, double e_curr, double& e_trial) {
    const long long n3 = 3LL * L[0].n;
    const int hv = prof_begin(P_VEC);
    launch_dot_partials(g.as<double>(), pd, n3, partials.as<double>() + 3 * nred, nred, stream);
    launch_sum_partials(partials.as<double>() + 3 * nred, nred, scal.as<double>() + 1, stream);
    prof_end(hv, 16.0 * n3);
    double alpha = 1.0;
    energy_async(dv.as<double>(), pd, alpha, true);
    read_scalars(2, 3);
    check_flags();
    const double gdotp = host_scal[1];
    if (!(gdotp < 0.0)) throw SolverFailure("line_search: not a descent direction");
    e_trial = host_scal[0];
    int k = 0;
    while (!(e_trial <= e_curr + cfg.ls_armijo * alpha * gdotp)) {
      if (++k >= cfg.ls_max_steps) throw SolverFailure("line_search: no acceptable step (gradient/Hessian inconsistency)");
      alpha *= cfg.ls_shrink;
      energy_async(dv.as<double>(), pd, alpha, true);
      read_scalars(1, 1);
      check_flags();
      e_trial = host_scal[0];
    }
    return alpha;
  }

  /// solve_quasi_newton (solvers.hpp:191-231); dv result in this->dv.
  SolveOut solve_qn(int levels, int frame_no, long long step_no) {
    const auto t0 = std::chrono::steady_clock::now();
    const int n = L[0].n;
    const long long n3 = 3LL * n;
    SolveOut out;
    sh.last = false;
    if (cfg.window > kMaxWindow) throw std::invalid_argument("L-BFGS window too large");
    const double target = cfg.epsilon * std::sqrt((double)n);
    struct ShardOff {  // the cut is per solve; taps and the other solvers run unsharded
      Context& c;
      ~ShardOff() {
        if (c.sh.on) {  // level 0 holds only this rank's rows: no tap may read it
          c.have_H = false;
          c.nlevels = 0;
        }
        c.sh.on = false;
      }
    } shard_off{*this};
    sh.on = want_shard(levels) && sh.planned;
    HOT_CUDA(cudaMemsetAsync(dv.p, 0, sizeof(double) * std::max<long long>(n3, 1), stream));
    HOT_CUDA(cudaMemsetAsync(iflags.p, 0, sizeof(int) * 8, stream));
    energy_async(dv.as<double>(), nullptr, 0.0, true, /*store_svd=*/true);
    gradient_async(dv.as<double>(), g.as<double>());
    read_scalars(3, 2);
    check_flags();
    double e_curr = host_scal[0];
    double residual = std::sqrt(host_scal[2]);
    if (residual <= target) {
      out.converged = true;
      return out;
    }
    sh.last = sh.on;
    if (sh.on) ++sh.solves;
    assemble_and_build_hierarchy(dv.as<double>(), levels, cfg.embedding, /*reuse_svd=*/true);
    const bool verbose = opt.verbose;
    prof_snapshot_slots();  // active-slot counts of this solve's levels (profile bytes)
    if (verbose)
      for (int m = 0; m < nlevels; ++m) L[m].active_slots = count_active_slots(m);
    if (verbose)
      for (int m = 0; m < nlevels; ++m)
        std::fprintf(stderr, "[hot] level %d: rows=%d waves=%d max_wave=%d active_slots=%lld (%.1f/row) bbox=%dx%dx%d\n",
                     m, L[m].n, L[m].nwaves, L[m].max_wave, L[m].active_slots, L[m].n ? (double)L[m].active_slots / L[m].n : 0.0,
                     L[m].ext[0], L[m].ext[1], L[m].ext[2]);
    for (int k = 0; k <= cfg.window; ++k) {
      hist_s[k].ensure(sizeof(double) * std::max<long long>(n3, 1));
      hist_y[k].ensure(sizeof(double) * std::max<long long>(n3, 1));
    }
    std::deque<HistEntry> hist;
    long long work = 0;
    for (int outer = 1; outer <= cfg.outer_cap; ++outer) {
      HOT_CUDA(cudaMemsetAsync(iflags.as<int>() + 2, 0, sizeof(int), stream));
      lbfgs_direction(hist, pdir.as<double>());
      // accept(): g.p then the Armijo backtracking (solvers.hpp:66-78, 169-186)
      double e_trial = 0.0;
      const double alpha = line_search(pdir.as<double>(), e_curr, e_trial);
      // s = alpha p ; dv += s ; g_new ; y = g_new - g
      const int slot = next_slot(hist);
      const int hv3 = prof_begin(P_VEC);
      launch_scale(pdir.as<double>(), alpha, hist_s[slot].as<double>(), n3, stream);
      launch_add_scaled(dv.as<double>(), pdir.as<double>(), alpha, dv.as<double>(), n3, stream);
      prof_end(hv3, 40.0 * n3);
      gradient_async(dv.as<double>(), gnew.as<double>());
      const int hv4 = prof_begin(P_VEC);
      launch_ys_dots(gnew.as<double>(), g.as<double>(), hist_y[slot].as<double>(), hist_s[slot].as<double>(), n3,
                     partials.as<double>() + 3 * nred, nred, stream);
      launch_sum_partials(partials.as<double>() + 3 * nred, nred, scal.as<double>() + 3, stream);
      launch_sum_partials(partials.as<double>() + 4 * nred, nred, scal.as<double>() + 4, stream);
      launch_sum_partials(partials.as<double>() + 5 * nred, nred, scal.as<double>() + 5, stream);
      prof_end(hv4, 32.0 * n3);
      g.swap(gnew);
      read_scalars(6, 3);
      check_flags();
      residual = std::sqrt(host_scal[2]);
      e_curr = e_trial;
      const long long inner_this = host_int[2];
      work += inner_this;
      hot_diag_row row;
      row.frame = frame_no;
      row.step = step_no;
      row.outer_iteration = outer;
      row.scaled_residual = residual;
      row.energy = e_curr;
      row.step_length = alpha;
      row.inner_iterations = inner_this;
      row.work_units = work;
      row.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      diag.push_back(row);
      // history.push (solvers.hpp:87-93)
      const double ys = host_scal[3], yn = std::sqrt(host_scal[4]), sn = std::sqrt(host_scal[5]);
      if (ys > 1e-12 * yn * sn) {
        if ((int)hist.size() == std::max(1, cfg.window)) hist.pop_front();
        hist.push_back({slot, 1.0 / ys});
      }
      out.outer = outer;
      out.inner += inner_this;
      if (residual <= target) {
        out.converged = true;
        break;
      }
    }
    if (!out.converged) {
      char buf[128];
      std::snprintf(buf, sizeof(buf), "quasi-newton solve: outer iteration cap reached (residual %f)", residual);
      throw SolverFailure(buf);
    }
    return out;
  }

  /// window+1 buffers: the new pair never overwrites a pair still in the history (a
  /// curvature-rejected push keeps the oldest pair alive).
  int next_slot(const std::deque<HistEntry>& hist) const {
    const int W = std::max(1, cfg.window);
    std::vector<char> used(W + 1, 0);
    for (const auto& e : hist) used[e.slot] = 1;
    for (int s = 0; s <= W; ++s)
      if (!used[s]) return s;
    return 0;
  }

  /// Host-driven PCG on level 0 (pcg.hpp:17-46): x = 0, stop on sqrt(r.z) <= rel sqrt(r0.z0).
  /// apply_a(in, out), apply_p(in, out) are device operators.  Returns the iteration count.
  template <class ApplyA, class ApplyP>
  int pcg_level0(ApplyA&& apply_a, ApplyP&& apply_p, const double* b, double* x, double rel, int cap) {
    const int n = L[0].n;
    const long long n3 = 3LL * n;
    double* r = pn_r.as<double>();
    double* z = pn_z.as<double>();
    double* p = pn_p.as<double>();
    double* Ap = pn_Ap.as<double>();
    double* part = partials.as<double>() + 3 * nred;
    auto dot = [&](const double* a, const double* bb) {
      launch_dot_partials(a, bb, n3, part, nred, stream);
      launch_sum_partials(part, nred, scal.as<double>() + 7, stream);
      HOT_CUDA(cudaMemcpyAsync(host_scal + 7, scal.as<double>() + 7, sizeof(double), cudaMemcpyDeviceToHost, stream));
      sync();
      check_launch();
      return host_scal[7];
    };
    HOT_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n3, stream));
    HOT_CUDA(cudaMemcpyAsync(r, b, sizeof(double) * n3, cudaMemcpyDeviceToDevice, stream));
    apply_p(r, z);
    double rho = dot(r, z);
    if (!(rho > 0.0)) {
      if (rho < 0.0) throw SolverFailure("pcg: preconditioner is not positive definite");
      return 0;  // b == 0
    }
    const double threshold = rel * rel * rho;
    HOT_CUDA(cudaMemcpyAsync(p, z, sizeof(double) * n3, cudaMemcpyDeviceToDevice, stream));
    int its = 0;
    for (int it = 0; it < cap; ++it) {
      apply_a(p, Ap);
      const double pAp = dot(p, Ap);
      if (!(pAp > 0.0)) throw SolverFailure("pcg: system matrix is not positive definite");
      const double alpha = rho / pAp;
      launch_pcg_xr(x, r, p, Ap, alpha, n3, stream);
      apply_p(r, z);
      const double rho_new = dot(r, z);
      its = it + 1;
      if (rho_new <= threshold) break;
      launch_pcg_p(p, z, rho_new / rho, n3, stream);
      rho = rho_new;
    }
    return its;
  }

  /// solve_projected_newton (solvers.hpp:235-300): variant 0 assembled Jacobi-PCG (pn-pcg),
  /// 1 matrix-free Jacobi-PCG (pn-pcg-mf), 2 V-cycle-preconditioned PCG (pn-mgpcg).  The
  /// Newton model (projected Hessian, its block diagonal, the hierarchy) is rebuilt at every
  /// outer iterate; the inner tolerance is adaptive (solvers.hpp:62-64).
  SolveOut solve_pn(int variant, int frame_no, long long step_no) {
    const auto t0 = std::chrono::steady_clock::now();
    const int n = L[0].n;
    const long long n3 = 3LL * n;
    SolveOut out;
    const double target = cfg.epsilon * std::sqrt((double)n);
    HOT_CUDA(cudaMemsetAsync(dv.p, 0, sizeof(double) * std::max<long long>(n3, 1), stream));
    HOT_CUDA(cudaMemsetAsync(iflags.p, 0, sizeof(int) * 8, stream));
    energy_async(dv.as<double>(), nullptr, 0.0, true);
    gradient_async(dv.as<double>(), g.as<double>());
    read_scalars(3, 2);
    check_flags();
    double e_curr = host_scal[0];
    double residual = std::sqrt(host_scal[2]);
    if (residual <= target) {
      out.converged = true;
      return out;
    }
    const size_t vb = sizeof(double) * std::max<long long>(n3, 1);
    for (DBuf* d : {&pn_b, &pn_x, &pn_r, &pn_z, &pn_p, &pn_Ap}) d->ensure(vb);
    long long work = 0;
    for (int outer = 1; outer <= cfg.outer_cap; ++outer) {
      HOT_CUDA(cudaMemsetAsync(iflags.as<int>() + 2, 0, sizeof(int), stream));
      const double* Dinv = nullptr;
      if (variant == 1) {
        particle_tensors(dv.as<double>(), true, false);
        pn_dinv.ensure(sizeof(double) * 9 * std::max(n, 1));
        launch_mf_block_diag_inv(pview(), bview(), gview(), tu_base(), pn_dinv.as<double>(), stream);
        Dinv = pn_dinv.as<double>();
      } else {
        assemble(dv.as<double>(), true);
        build_hierarchy(variant == 2 ? cfg.levels : 1, cfg.embedding);
        prof_snapshot_slots();
        Dinv = L[0].dinv.as<double>();
      }
      // gpg = g^T D^-1 g (solvers.hpp:263-268); k = adaptive_cg_tolerance
      launch_block_apply(Dinv, g.as<double>(), pn_z.as<double>(), n, stream);
      launch_dot_partials(g.as<double>(), pn_z.as<double>(), n3, partials.as<double>() + 3 * nred, nred, stream);
      launch_sum_partials(partials.as<double>() + 3 * nred, nred, scal.as<double>() + 7, stream);
      HOT_CUDA(cudaMemcpyAsync(host_scal + 7, scal.as<double>() + 7, sizeof(double), cudaMemcpyDeviceToHost, stream));
      sync();
      const double gpg = host_scal[7];
      const double k = std::min(0.5, std::sqrt(std::max(std::sqrt(gpg), cfg.tau)));
      launch_neg_copy(g.as<double>(), pn_b.as<double>(), n3, stream);
      long long inner_this = 0;
      const int hp = prof_begin(P_PCG);
      if (variant == 0) {  // Jacobi-PCG on the assembled matrix: the cooperative kernel
        launch_pcg(L[0].view(), pn_b.as<double>(), pn_x.as<double>(), pn_r.as<double>(), pn_z.as<double>(),
                   pn_p.as<double>(), pn_Ap.as<double>(), k, cfg.cg_cap, partials.as<double>() + 6 * nred,
                   iflags.as<int>() + 4, iflags.as<int>() + 2, coop_grid(pcg_max_blocks(), n, 8, 4), stream);
        copy_status();
        read_scalars(0, 3);
        check_flags();
        inner_this = host_int[2];
      } else if (variant == 1) {
        pn_dP.ensure(sizeof(double) * 9 * std::max<long long>(np, 1));
        inner_this = pcg_level0(
            [&](const double* in, double* o) {
              launch_mf_multiply(pview(), bview(), gview(), tu_base(), in, pn_dP.as<double>(), o, stream);
            },
            [&](const double* in, double* o) { launch_block_apply(Dinv, in, o, n, stream); }, pn_b.as<double>(),
            pn_x.as<double>(), k, cfg.cg_cap);
      } else {
        int its = pcg_level0([&](const double* in, double* o) { launch_spmv(L[0].view(), in, o, stream); },
                             [&](const double* in, double* o) {
                               vcycle(in, o, true, cfg.pinned_coarse_iterations);
                             },
                             pn_b.as<double>(), pn_x.as<double>(), k, cfg.cg_cap);
        read_scalars(0, 3);
        check_flags();
        inner_this = its + host_int[2];  // + the pinned coarse solves' iterations
      }
      prof_end(hp);
      double e_trial = 0.0;
      const double alpha = line_search(pn_x.as<double>(), e_curr, e_trial);
      launch_add_scaled(dv.as<double>(), pn_x.as<double>(), alpha, dv.as<double>(), n3, stream);
      gradient_async(dv.as<double>(), g.as<double>());
      read_scalars(3, 2);
      check_flags();
      residual = std::sqrt(host_scal[2]);
      e_curr = e_trial;
      work += inner_this;
      hot_diag_row row;
      row.frame = frame_no;
      row.step = step_no;
      row.outer_iteration = outer;
      row.scaled_residual = residual;
      row.energy = e_curr;
      row.step_length = alpha;
      row.inner_iterations = inner_this;
      row.work_units = work;
      row.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      diag.push_back(row);
      out.outer = outer;
      out.inner += inner_this;
      if (residual <= target) {
        out.converged = true;
        break;
      }
    }
    if (!out.converged) {
      char buf[128];
      std::snprintf(buf, sizeof(buf), "projected newton solve: outer iteration cap reached (residual %f)", residual);
      throw SolverFailure(buf);
    }
    return out;
  }

  SolveOut step_grid(int frame_no, long long step_no) {
    switch (cfg.kind) {  // solvers.hpp:360-372
      case 0:
        return solve_qn(cfg.levels, frame_no, step_no);  // hot
      case 1:
        return solve_pn(0, frame_no, step_no);  // pn-pcg
      case 2:
        return solve_pn(1, frame_no, step_no);  // pn-pcg-mf
      case 3:
        return solve_pn(2, frame_no, step_no);  // pn-mgpcg
      case 4:
        return solve_qn(1, frame_no, step_no);  // lbfgs-h
    }
    throw std::invalid_argument("unknown solver kind");
  }

  // ------------------------------------------------------------------ advance_step
  void advance(double frame_end, hot_step_stats* st) {
    double v_max = 0.0;
    if (np > 0) {
      HOT_CUDA(cudaMemsetAsync(scal.as<double>() + 8, 0, sizeof(double), stream));
      launch_vmax(pview(), reinterpret_cast<unsigned long long*>(scal.as<double>() + 8), stream);
      HOT_CUDA(cudaMemcpyAsync(host_scal + 8, scal.as<double>() + 8, sizeof(double), cudaMemcpyDeviceToHost, stream));
      sync();
      v_max = host_scal[8];
    }
    if (pp_on) {  // the largest particle speed of every rank (ghosts are copies: max unchanged)
      const double mine = v_max;
      long long bits = 0;
      std::memcpy(&bits, &mine, sizeof(bits));
      for (long long b : allgather_ll(bits)) {
        double other = 0.0;
        std::memcpy(&other, &b, sizeof(other));
        v_max = std::max(v_max, other);
      }
      if (opt.verbose)
        std::fprintf(stderr, "[hot] rank %d: %lld local particles of %lld, v_max local %.9g global %.9g\n", comm->rank,
                     np, np_global, mine, v_max);
    }
    const double frame = 1.0 / fps;
    double dtn = v_max <= 0.0 ? frame : std::min(frame, 0.6 * dx / v_max);  // cfl_dt (grid.hpp:168-173)
    if (frame_end > 0.0) dtn = std::min(dtn, frame_end - time);
    if (!(dtn > 0.0)) throw SolverFailure("advance_step: non-positive time step");
    prepare(dtn, time);
    SolveOut so;
    try {
      so = step_grid(frame, step_index);
    } catch (const SolverFailure& e) {
      throw SolverFailure("step " + std::to_string(step_index) + ": " + e.what());
    }
    // grid.velocity = v^{n+1}; g2p; update_strain; advect
    launch_final_velocity(gview(), dv.as<double>(), vout.as<double>(), stream);
    gvel.swap(vout);
    const int h = prof_begin(P_G2P);
    HOT_CUDA(cudaMemsetAsync(iflags.as<int>() + 6, 0, sizeof(int), stream));
    if (pp_on)  // inversions counted by the owners
      launch_g2p_strain_advect(pview(), gview(), dx, dtn, mats_d.as<DevMaterial>(), iflags.as<int>() + 6, stream,
                               pp_owned_lo(comm->rank), pp_owned_hi(comm->rank));
    else
      launch_g2p_strain_advect(pview(), gview(), dx, dtn, mats_d.as<DevMaterial>(), iflags.as<int>() + 6, stream);
    prof_end(h, (double)np * (24 + 24 + 72 + 72 + 4 + 24 + 96) + 24.0 * L[0].n);
    int inv = 0;
    HOT_CUDA(cudaMemcpyAsync(&inv, iflags.as<int>() + 6, sizeof(int), cudaMemcpyDeviceToHost, stream));
    sync();
    check_launch();
    if (pp_on) {
      long long total = 0;
      for (long long c : allgather_ll(inv)) total += c;
      inv = (int)total;
    }
    inversions += inv;
    if (pp_enabled() && sh.planned) {  // partition the particles along this step's cut
      if (!pp_on) pp_bounds = sh.bounds;
      const int hp = prof_begin(P_COMM);
      pp_exchange();
      prof_end(hp);
    }
    time += dtn;
    ++step_index;
    have_state = false;
    if (st) {
      st->dt = dtn;
      st->outer_iterations = so.outer;
      st->inner_total = so.inner;
      st->node_count = L[0].n;
      st->converged = so.converged ? 1 : 0;
    }
  }
};

namespace {
__global__ void k_status_max(int* iflags) {
  // pcg writes its status into iflags[4]; keep the first failure in iflags[1]
  if (iflags[4] != 0 && iflags[1] == 0) iflags[1] = iflags[4];
}
__global__ void k_count_active(const int* __restrict__ cols, long long n, unsigned long long* out) {
  unsigned long long c = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    c += (cols[t] >= 0) ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}
}  // namespace

void Context::copy_status() {
  { k_status_max<<<1, 1, 0, stream>>>(iflags.as<int>()); count_launches(1); }
}

long long Context::count_active_slots(int m) {
  Level& l = L[m];
  if (l.n == 0) return 0;
  unsigned long long* d = reinterpret_cast<unsigned long long*>(scal.as<double>() + 12);
  HOT_CUDA(cudaMemsetAsync(d, 0, 8, stream));
  { k_count_active<<<num_sms() * 4, 256, 0, stream>>>(l.cols.as<int>(), (long long)l.n * l.pitch(), d); count_launches(1); }
  unsigned long long h = 0;
  HOT_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, stream));
  sync();
  return (long long)h;
}

}  // namespace hotb200

// ==========================================================================================
// C-ABI
// ==========================================================================================
using hotb200::Context;
using hotb200::CudaError;

struct hot_ctx {
  Context c;                       // the 3D context (errors of both paths land in c.err)
  hotb200::Context2D* c2 = nullptr;  // dim = 2 scenes: the 2D device path (k2d.cu)
  ~hot_ctx() { hotb200::ctx2d_delete(c2); }
};

namespace {

/// Makes the context's device current for the call and restores the caller's device after it
/// (a host thread may drive contexts on several GPUs, or switch devices between calls).
struct DeviceScope {
  int saved = -1;
  explicit DeviceScope(const hot_ctx* ctx);
  ~DeviceScope() {
    if (saved >= 0) cudaSetDevice(saved);
  }
};

template <typename F>
int guard(hot_ctx* ctx, F&& f) {
  try {
    DeviceScope scope(ctx);
    f();
    return HOT_OK;
  } catch (const hotb200::SolverFailure& e) {
    if (ctx) ctx->c.err = e.what();
    return HOT_E_SOLVER_FAILURE;
  } catch (const hotb200::CudaError& e) {
    if (ctx) ctx->c.err = e.what();
    return HOT_E_CUDA;
  } catch (const hotb200::Unsupported& e) {
    if (ctx) ctx->c.err = e.what();
    return HOT_E_UNSUPPORTED;
  } catch (const std::invalid_argument& e) {
    if (ctx) ctx->c.err = e.what();
    return HOT_E_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    if (ctx) ctx->c.err = e.what();
    return HOT_E_DOMAIN;
  } catch (const std::logic_error& e) {
    if (ctx) ctx->c.err = e.what();
    return HOT_E_LOGIC;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.err = e.what();
    return HOT_E_CUDA;
  }
}

DeviceScope::DeviceScope(const hot_ctx* ctx) {
  if (!ctx) return;
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) return;
  if (cur != ctx->c.device) {
    HOT_CUDA(cudaSetDevice(ctx->c.device));
    saved = cur;
  }
}

thread_local std::string g_create_error;

void need_state(Context& c) {
  if (!c.have_state) throw std::logic_error("no prepared grid state (call hot_stage_prepare)");
}

}  // namespace

extern "C" {

int hot_version(void) { return HOT_API_VERSION; }

int hot_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int hot_create(hot_ctx** out, const hot_scene* scene, int device) {
  if (!out || !scene) return HOT_E_INVALID_ARGUMENT;
  *out = nullptr;
  auto* h = new hot_ctx;
  h->c.device = device;  // guard() makes it current and restores the caller's device afterwards
  const int rc = guard(h, [&] {
    if (scene->dim == 2) {  // the 2D device path (k2d.cu)
      h->c2 = hotb200::ctx2d_new(device, *scene);
      return;
    }
    if (scene->dim != 3) throw std::invalid_argument("scene dim must be 2 or 3");
    h->c.init(device);
    h->c.set_scene(*scene);
  });
  if (rc != HOT_OK) {
    g_create_error = h->c.err;
    delete h;
    return rc;
  }
  *out = h;
  return HOT_OK;
}

void hot_destroy(hot_ctx* ctx) {
  if (!ctx) return;
  try {
    DeviceScope scope(ctx);
    delete ctx;
  } catch (...) {
    delete ctx;
  }
}

const char* hot_last_error(const hot_ctx* ctx) { return ctx ? ctx->c.err.c_str() : g_create_error.c_str(); }

int hot_set_solver(hot_ctx* ctx, const hot_solver_config* cfg) {
  if (ctx && ctx->c2 && cfg && cfg->levels >= 1 && cfg->window >= 1)
    return guard(ctx, [&] { hotb200::ctx2d_set_solver(ctx->c2, *cfg); });
  return guard(ctx, [&] {
    if (cfg->levels < 1) throw std::invalid_argument("levels must be at least 1");
    if (cfg->window < 1) throw std::invalid_argument("window must be at least 1");
    ctx->c.cfg = *cfg;
  });
}

int hot_sample_scene_particles(const hot_scene* scene, long long* n, double* x, double* v, double* mass, double* volume,
                               double* F, double* C, int* material) {
  return guard(nullptr, [&] {
    std::vector<double> X, Vv, M, Vol, Fm, Cm;
    std::vector<int> mat;
    const long long cnt = hotb200::sample_scene(*scene, X, Vv, M, Vol, Fm, Cm, mat);
    *n = cnt;
    if (!x) return;
    std::memcpy(x, X.data(), X.size() * 8);
    if (v) std::memcpy(v, Vv.data(), Vv.size() * 8);
    if (mass) std::memcpy(mass, M.data(), M.size() * 8);
    if (volume) std::memcpy(volume, Vol.data(), Vol.size() * 8);
    if (F) std::memcpy(F, Fm.data(), Fm.size() * 8);
    if (C) std::memcpy(C, Cm.data(), Cm.size() * 8);
    if (material) std::memcpy(material, mat.data(), mat.size() * 4);
  });
}

int hot_upload_particles(hot_ctx* ctx, long long n, const double* x, const double* v, const double* mass,
                         const double* volume, const double* F, const double* C, const int* material) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_upload(ctx->c2, n, x, v, mass, volume, F, C, material); });
  return guard(ctx, [&] { ctx->c.upload(n, x, v, mass, volume, F, C, material); });
}

int hot_download_particles(hot_ctx* ctx, double* x, double* v, double* F, double* C) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_download(ctx->c2, x, v, F, C); });
  return guard(ctx, [&] { ctx->c.download(x, v, F, C); });
}

int hot_set_plastic_state(hot_ctx* ctx, const double* Jp) {
  if (ctx && ctx->c2 && Jp) return guard(ctx, [&] { hotb200::ctx2d_set_plastic_state(ctx->c2, Jp); });
  if (!ctx || !Jp) return HOT_E_INVALID_ARGUMENT;
  return guard(ctx, [&] { ctx->c.set_plastic_state(Jp); });
}

int hot_get_plastic_state(hot_ctx* ctx, double* Jp) {
  if (ctx && ctx->c2 && Jp) return guard(ctx, [&] { hotb200::ctx2d_get_plastic_state(ctx->c2, Jp); });
  if (!ctx || !Jp) return HOT_E_INVALID_ARGUMENT;
  return guard(ctx, [&] { ctx->c.get_plastic_state(Jp); });
}

int hot_particle_count(hot_ctx* ctx, long long* n) {
  if (ctx->c2) {
    *n = hotb200::ctx2d_particle_count(ctx->c2);
    return HOT_OK;
  }
  *n = ctx->c.np_global;
  return HOT_OK;
}

int hot_set_time(hot_ctx* ctx, double time, int frame, long long step_index) {
  if (ctx->c2) {
    hotb200::ctx2d_set_time(ctx->c2, time, frame, step_index);
    return HOT_OK;
  }
  ctx->c.time = time;
  ctx->c.frame = frame;
  ctx->c.step_index = step_index;
  return HOT_OK;
}

int hot_get_time(hot_ctx* ctx, double* time, int* frame, long long* step_index, long long* inversion_warnings) {
  if (ctx->c2) {
    hotb200::ctx2d_get_time(ctx->c2, time, frame, step_index, inversion_warnings);
    return HOT_OK;
  }
  if (time) *time = ctx->c.time;
  if (frame) *frame = ctx->c.frame;
  if (step_index) *step_index = ctx->c.step_index;
  if (inversion_warnings) *inversion_warnings = ctx->c.inversions;
  return HOT_OK;
}

int hot_advance_step(hot_ctx* ctx, double frame_end, hot_step_stats* out) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_advance(ctx->c2, frame_end, out); });
  return guard(ctx, [&] { ctx->c.advance(frame_end, out); });
}

int hot_diagnostics(hot_ctx* ctx, hot_diag_row* rows, int cap, int* n) {
  if (ctx->c2) {
    *n = hotb200::ctx2d_diagnostics(ctx->c2, rows, cap);
    return HOT_OK;
  }
  const int cnt = (int)ctx->c.diag.size();
  *n = cnt;
  if (rows)
    for (int i = 0; i < std::min(cap, cnt); ++i) rows[i] = ctx->c.diag[i];
  return HOT_OK;
}

int hot_clear_diagnostics(hot_ctx* ctx) {
  if (ctx->c2) {
    hotb200::ctx2d_clear_diagnostics(ctx->c2);
    return HOT_OK;
  }
  ctx->c.diag.clear();
  return HOT_OK;
}

int hot_stage_prepare(hot_ctx* ctx, double dt, double time) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_prepare(ctx->c2, dt, time); });
  // the stage taps compare every particle: partitioned particles come back to every rank first
  return guard(ctx, [&] { ctx->c.pp_gather_all(); ctx->c.prepare(dt, time); ctx->c.sync(); });
}

int hot_stage_node_count(hot_ctx* ctx, int* n) {
  if (ctx->c2) {
    *n = hotb200::ctx2d_node_count(ctx->c2);
    return HOT_OK;
  }
  *n = ctx->c.L[0].n;
  return HOT_OK;
}

int hot_stage_grid(hot_ctx* ctx, int* coords, double* mass, double* velocity, double* momentum, unsigned char* dirichlet,
                   double* bc_velocity, double* cn_scale) {
  if (ctx && ctx->c2)
    return guard(ctx, [&] {
      hotb200::ctx2d_grid(ctx->c2, coords, mass, velocity, momentum, dirichlet, bc_velocity, cn_scale);
    });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    need_state(c);
    const int n = c.L[0].n;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) HOT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.stream));
    };
    cp(coords, c.L[0].coords.p, sizeof(int) * 3 * n);
    cp(mass, c.gmass.p, sizeof(double) * n);
    cp(velocity, c.gvel.p, sizeof(double) * 3 * n);
    cp(momentum, c.gmom.p, sizeof(double) * 3 * n);
    cp(dirichlet, c.L[0].dir.p, n);
    cp(bc_velocity, c.gbc.p, sizeof(double) * 3 * n);
    cp(cn_scale, c.gcn.p, sizeof(double) * n);
    c.sync();
  });
}

int hot_stage_set_grid(hot_ctx* ctx, const double* velocity, const unsigned char* dirichlet, const double* bc_velocity) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_set_grid(ctx->c2, velocity, dirichlet, bc_velocity); });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    need_state(c);
    const int n = c.L[0].n;
    if (velocity) HOT_CUDA(cudaMemcpyAsync(c.gvel.p, velocity, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c.stream));
    if (dirichlet) HOT_CUDA(cudaMemcpyAsync(c.L[0].dir.p, dirichlet, n, cudaMemcpyHostToDevice, c.stream));
    if (bc_velocity)
      HOT_CUDA(cudaMemcpyAsync(c.gbc.p, bc_velocity, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c.stream));
    c.sync();
  });
}

int hot_stage_energy(hot_ctx* ctx, const double* dv, double* energy) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_energy(ctx->c2, dv, energy); });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    need_state(c);
    const int n = c.L[0].n;
    HOT_CUDA(cudaMemcpyAsync(c.q.p, dv, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c.stream));
    HOT_CUDA(cudaMemsetAsync(c.iflags.p, 0, sizeof(int) * 8, c.stream));
    c.energy_async(c.q.as<double>(), nullptr, 0.0, true);
    c.read_scalars(1, 2);
    c.check_flags();
    *energy = c.host_scal[0];
  });
}

int hot_stage_gradient(hot_ctx* ctx, const double* dv, double* gout, double* scaled_norm) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_gradient(ctx->c2, dv, gout, scaled_norm); });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    need_state(c);
    const int n = c.L[0].n;
    HOT_CUDA(cudaMemcpyAsync(c.q.p, dv, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c.stream));
    HOT_CUDA(cudaMemsetAsync(c.iflags.p, 0, sizeof(int) * 8, c.stream));
    c.energy_async(c.q.as<double>(), nullptr, 0.0, true);
    c.gradient_async(c.q.as<double>(), c.gnew.as<double>());
    if (gout) HOT_CUDA(cudaMemcpyAsync(gout, c.gnew.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c.stream));
    c.read_scalars(3, 2);
    c.check_flags();
    if (scaled_norm) *scaled_norm = std::sqrt(c.host_scal[2]);
  });
}

int hot_stage_assemble(hot_ctx* ctx, const double* dv, int project) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_assemble(ctx->c2, dv, project); });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    need_state(c);
    const int n = c.L[0].n;
    HOT_CUDA(cudaMemcpyAsync(c.q.p, dv, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c.stream));
    HOT_CUDA(cudaMemsetAsync(c.iflags.p, 0, sizeof(int) * 8, c.stream));
    c.assemble(c.q.as<double>(), project != 0);
    c.read_scalars(0, 1);
    c.check_flags();
    c.L[0].active_slots = c.count_active_slots(0);
  });
}

int hot_stage_build_hierarchy(hot_ctx* ctx, int levels, int embedding) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_build_hierarchy(ctx->c2, levels, embedding); });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    if (!c.have_H) throw std::logic_error("no matrix assembled");
    c.build_hierarchy(levels, embedding);
    c.prof_snapshot_slots();  // the staged V-cycle / SpMV profile bytes refer to this hierarchy
    for (int m = 0; m < c.nlevels; ++m) c.L[m].active_slots = c.count_active_slots(m);
  });
}

int hot_stage_level_count(hot_ctx* ctx, int* levels) {
  if (ctx->c2) {
    *levels = hotb200::ctx2d_level_count(ctx->c2);
    return HOT_OK;
  }
  *levels = ctx->c.nlevels;
  return HOT_OK;
}

int hot_stage_level_shape(hot_ctx* ctx, int level, int* rows, int* slots) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_level_shape(ctx->c2, level, rows, slots); });
  return guard(ctx, [&] {
    if (level < 0 || level >= ctx->c.nlevels) throw std::logic_error("no such level");
    *rows = ctx->c.L[level].n;
    *slots = ctx->c.L[level].slots();
  });
}

int hot_stage_level_matrix(hot_ctx* ctx, int level, double* blocks, int* cols, int* coords, unsigned char* dirichlet) {
  if (ctx && ctx->c2)
    return guard(ctx, [&] { hotb200::ctx2d_level_matrix(ctx->c2, level, blocks, cols, coords, dirichlet); });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    if (level < 0 || level >= c.nlevels) throw std::logic_error("no such level");
    const hotb200::Level& l = c.L[level];
    const long long n = l.n;
    const int pitch = l.pitch(), ns = l.slots();
    std::vector<int> cl((cols || blocks) ? n * pitch : 0);
    std::vector<double> H(blocks ? n * 9 * pitch : 0);  // only when the blocks are asked for (GB at level 0)
    if (!cl.empty())
      HOT_CUDA(cudaMemcpyAsync(cl.data(), l.cols.p, sizeof(int) * cl.size(), cudaMemcpyDeviceToHost, c.stream));
    if (!H.empty())
      HOT_CUDA(cudaMemcpyAsync(H.data(), l.H.p, sizeof(double) * H.size(), cudaMemcpyDeviceToHost, c.stream));
    if (coords) HOT_CUDA(cudaMemcpyAsync(coords, l.coords.p, sizeof(int) * 3 * n, cudaMemcpyDeviceToHost, c.stream));
    if (dirichlet) HOT_CUDA(cudaMemcpyAsync(dirichlet, l.dir.p, n, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (cl.empty()) return;
    for (long long i = 0; i < n; ++i)
      for (int s = 0; s < ns; ++s) {
        const int col = cl[i * pitch + s];
        if (cols) cols[i * ns + s] = col;
        if (blocks)
          for (int e = 0; e < 9; ++e) blocks[(i * ns + s) * 9 + e] = col < 0 ? 0.0 : H[(i * 9 + e) * pitch + s];
      }
  });
}

int hot_stage_matvec(hot_ctx* ctx, int level, const double* x, double* y) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_matvec(ctx->c2, level, x, y); });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    if (level < 0 || level >= c.nlevels) throw std::logic_error("no such level");
    hotb200::Level& l = c.L[level];
    HOT_CUDA(cudaMemcpyAsync(l.b.p, x, sizeof(double) * 3 * l.n, cudaMemcpyHostToDevice, c.stream));
    hotb200::launch_spmv(l.view(), l.b.as<double>(), l.r.as<double>(), c.stream);
    HOT_CUDA(cudaMemcpyAsync(y, l.r.p, sizeof(double) * 3 * l.n, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    c.check_launch();
  });
}

int hot_stage_vcycle(hot_ctx* ctx, const double* b, double* u, int* coarse_iterations) {
  if (ctx && ctx->c2) return guard(ctx, [&] { hotb200::ctx2d_vcycle(ctx->c2, b, u, coarse_iterations); });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    if (c.nlevels < 1) throw std::logic_error("no hierarchy");
    const int n = c.L[0].n;
    HOT_CUDA(cudaMemcpyAsync(c.q.p, b, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c.stream));
    HOT_CUDA(cudaMemsetAsync(c.iflags.p, 0, sizeof(int) * 8, c.stream));
    c.vcycle(c.q.as<double>(), c.pdir.as<double>(), false, 0);
    HOT_CUDA(cudaMemcpyAsync(u, c.pdir.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c.stream));
    c.read_scalars(0, 3);
    c.check_flags();
    if (coarse_iterations) *coarse_iterations = c.host_int[2];
  });
}

int hot_stage_step_grid(hot_ctx* ctx, double* velocity, double* dv, int* outer, long long* inner, int* converged,
                        int frame, long long step) {
  if (ctx && ctx->c2)
    return guard(ctx, [&] { hotb200::ctx2d_step_grid(ctx->c2, velocity, dv, outer, inner, converged, frame, step); });
  return guard(ctx, [&] {
    Context& c = ctx->c;
    need_state(c);
    auto so = c.step_grid(frame, step);
    const int n = c.L[0].n;
    hotb200::launch_final_velocity(c.gview(), c.dv.as<double>(), c.vout.as<double>(), c.stream);
    if (velocity) HOT_CUDA(cudaMemcpyAsync(velocity, c.vout.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c.stream));
    if (dv) HOT_CUDA(cudaMemcpyAsync(dv, c.dv.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (outer) *outer = so.outer;
    if (inner) *inner = so.inner;
    if (converged) *converged = so.converged;
  });
}

void* hot_stream(hot_ctx* ctx) {
  if (ctx && ctx->c2) return hotb200::ctx2d_stream(ctx->c2);
  return ctx ? (void*)ctx->c.stream : nullptr;
}

int hot_profile_enable(hot_ctx* ctx, int enable) {
  if (ctx && ctx->c2) return HOT_OK;  // the 2D path has no phase profile
  return guard(ctx, [&] {
    Context& c = ctx->c;
    c.sync();
    for (auto& e : c.events) {
      c.event_pool.push_back(e.a);
      c.event_pool.push_back(e.b);
    }
    c.events.clear();
    for (double& b : c.phase_bytes) b = 0;
    for (double& f : c.phase_flops) f = 0;
    c.slot_terms.clear();
    c.prof_solve = -1;
    if (enable) c.prof_slots.ensure(sizeof(unsigned long long) * Context::kProfSolves * hotb200::kMaxLevels);
    c.prof = enable != 0;
  });
}

int hot_profile_read(hot_ctx* ctx, char* names, double* total_ms, long long* launches, double* bytes, int cap, int* n) {
  if (ctx && ctx->c2) {
    *n = 0;
    return HOT_OK;
  }
  return guard(ctx, [&] {
    Context& c = ctx->c;
    c.sync();
    std::vector<double> ms(hotb200::kPhases, 0.0);
    std::vector<long long> cnt(hotb200::kPhases, 0);
    for (auto& e : c.events) {
      float t = 0.f;
      HOT_CUDA(cudaEventElapsedTime(&t, e.a, e.b));
      ms[e.phase] += t;
      cnt[e.phase] += 1;
    }
    std::vector<double> slot_bytes(hotb200::kPhases, 0.0);
    if (c.prof_solve >= 0) {
      std::vector<unsigned long long> act((size_t)(c.prof_solve + 1) * hotb200::kMaxLevels);
      HOT_CUDA(cudaMemcpy(act.data(), c.prof_slots.p, sizeof(unsigned long long) * act.size(), cudaMemcpyDeviceToHost));
      for (const auto& t : c.slot_terms)  // (a term of an assembly outside a solve has no snapshot)
        if (t.solve <= c.prof_solve)
          slot_bytes[t.phase] += t.coef * (double)act[(size_t)t.solve * hotb200::kMaxLevels + t.level];
    }
    const int k = std::min(cap, hotb200::kPhases);
    for (int i = 0; i < k; ++i) {
      std::snprintf(names + 32 * i, 32, "%s", hotb200::kPhaseNames[i]);
      total_ms[i] = ms[i];
      launches[i] = cnt[i];
      const double b = c.phase_bytes[i] + slot_bytes[i];
      bytes[i] = b > 0 ? b : -c.phase_flops[i];  // < 0: fp64 flops
    }
    *n = k;
  });
}

long long hot_kernel_launches(hot_ctx* ctx) {
  (void)ctx;
  return hotb200::kernel_launch_count();
}

int hot_set_comm_host(hot_ctx* ctx, const hot_comm_host* ops) {
  if (ctx && ctx->c2) {
    ctx->c.err = "the 2D path runs on one GPU (slabs are built for dim = 3)";
    return HOT_E_UNSUPPORTED;
  }
  if (!ctx) return HOT_E_INVALID_ARGUMENT;
  return guard(ctx, [&] {
    if (!ops) {
      ctx->c.comm.reset();
      return;
    }
    ctx->c.comm.reset(hotb200::make_host_comm(*ops));
  });
}

int hot_nccl_unique_id(unsigned char id[128]) {
  if (!id) return HOT_E_INVALID_ARGUMENT;
  return guard(nullptr, [&] { hotb200::nccl_unique_id(id); });
}

int hot_set_comm_nccl(hot_ctx* ctx, const unsigned char id[128], int rank, int size) {
  if (ctx && ctx->c2) {
    ctx->c.err = "the 2D path runs on one GPU (slabs are built for dim = 3)";
    return HOT_E_UNSUPPORTED;
  }
  if (!ctx || !id) return HOT_E_INVALID_ARGUMENT;
  return guard(ctx, [&] {
    ctx->c.comm.reset(hotb200::make_nccl_comm(id, rank, size));
  });
}

int hot_shard_info(hot_ctx* ctx, hot_shard_info_t* out) {
  if (!ctx || !out) return HOT_E_INVALID_ARGUMENT;
  const Context& c = ctx->c;
  *out = hot_shard_info_t{};
  out->rank = c.comm ? c.comm->rank : 0;
  out->size = c.comm ? c.comm->size : 1;
  out->sharded = c.sh.last ? 1 : 0;
  out->plane_lo = c.sh.P;
  out->plane_hi = c.sh.Q;
  out->row_lo = c.sh.r_lo;
  out->row_hi = c.sh.r_hi;
  out->crow_lo = c.sh.c_lo;
  out->crow_hi = c.sh.c_hi;
  out->asm_lo = c.sh.a_lo;
  out->asm_hi = c.sh.r_hi;
  out->halo_exchanges = c.comm ? c.comm->halos : 0;
  out->gathers = c.comm ? c.comm->gathers : 0;
  out->particles_local = c.np;
  out->particles_total = c.np_global;
  out->partitioned = c.pp_on ? 1 : 0;
  return HOT_OK;
}

int hot_plan_slabs(int plane_lo, int nplanes, const long long* weight, int size, int align, int min_width,
                   int* bounds) {
  if (!bounds) return HOT_E_INVALID_ARGUMENT;
  return hotb200::plan_slabs(plane_lo, nplanes, weight, size, align, min_width, bounds) ? HOT_OK
                                                                                      : HOT_E_INVALID_ARGUMENT;
}

}  // extern "C"
