// Internal (host <-> kernel) declarations of the B200 HOT step.  Not part of the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "hot_device.cuh"

namespace hotb200 {

/// Host-side error kinds of the device path (mapped onto hot_status by the C-ABI guard).
struct SolverFailure : std::runtime_error {  // hotmpm::SolverFailure (common.hpp:124-126)
  explicit SolverFailure(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct Unsupported : std::runtime_error {
  explicit Unsupported(const std::string& m) : std::runtime_error(m) {}
};

/// Particle state, structure-of-arrays in the caller's (reference) particle order:
/// x[a*n+p], v[a*n+p], F[k*n+p] / C[k*n+p] with k = 3*row+col.
struct ParticlesView {
  double* x;
  double* v;
  double* F;
  double* C;
  double* mass;
  double* vol;
  int* mat;
  int* bin;  // stencil-centre node (bin) of each particle slot; valid after activation (bin order)
  double* Jp;  // plastic volume ratio (snow materials only, else null; extension: hardening)
  long long n;
};

/// Particles binned by their stencil-centre node (round(x/dx)).  After launch_reorder_particles
/// the particle arrays are stored in bin order, so bin j is the index range [start[j], start[j+1]).
struct BinsView {
  const int* start;  // n_nodes + 1
  const int* pid;    // n_particles: original (pre-reorder) position of each binned slot
};

/// One multigrid level in diagonal storage, component-major per row:
/// H[(row*9 + e)*pitch + slot], e = 3*r + c of the 3x3 block, slot lexicographic in
/// {-R..R}^3 (objective.hpp:24-32).  cols[row*pitch + slot] = -1 when inactive.  R = 2
/// (125 slots, pitch 128) on level 0 and on linear-embedding coarse levels; R = 3 (343 slots,
/// pitch 352) on quadratic-embedding coarse levels (multigrid.hpp:274-275).
struct LevelView {
  int n;
  const int* coords;  // 3*n, lexicographic
  DenseMap map;
  const int* cols;
  double* H;
  double* dinv;       // 9*n row-major
  const uint8_t* dir;
  int radius;         // diagonal-storage radius R
  int lo, hi;         // row range [lo, hi) the range-aware kernels compute (assembly, Galerkin,
                      // D^-1, SpMV / residual); [0, n) except in the slab-sharded solve
};

__host__ __device__ constexpr int level_slots(int radius) { return (2 * radius + 1) * (2 * radius + 1) * (2 * radius + 1); }
__host__ __device__ constexpr int level_pitch(int radius) { return radius == 2 ? 128 : 352; }
static_assert(level_pitch(2) == kSlotPitch && level_slots(2) == kSlots, "radius-2 layout");
static_assert(level_pitch(3) >= level_slots(3) && level_pitch(3) % 32 == 0, "radius-3 layout");

struct GridView {
  int n;
  const int* coords;
  DenseMap map;
  double* mass;
  double* vel;     // 3n
  double* mom;     // 3n
  uint8_t* dir;
  double* bc_vel;  // 3n
  double* cn_scale;
  const int* nb27;  // per node: the 27 nodes at offsets {-1,0,1}^3 (lexicographic), -1 if inactive
};

struct DevCollider {
  int shape;   // 0 box, 1 sphere, 2 half-space, 3 cylinder
  int motion;  // 0 static, 1 linear, 2 rotation
  double a[3], b[3];  // box min/max | sphere centre | half-space point/normal | cylinder centre/axis(unit)
  double radius;
  double vel[3];
  double rot_center[3], rot_w[3];  // omega * unit axis
};

// ---------------------------------------------------------------- grid (k_grid.cu)
void launch_particle_bounds(const ParticlesView& P, double dx, int* bounds6, int* bad_flag, cudaStream_t s);
void launch_mark_active(const ParticlesView& P, double dx, DenseMap map, uint8_t* flags, cudaStream_t s);
/// Exclusive scan of dense flags into idx (-1 for inactive) + compaction of coords.  Returns
/// the active count through *count_dev.  tile_sums must hold ceil(len/4096)+1 ints.
void launch_flags_to_index(const uint8_t* flags, long long len, const int* ext, const int* lo, int* idx, int* coords,
                           int* tile_sums, int* count_dev, cudaStream_t s);
/// orig: original ids of the particle slots (the within-bin order).
void launch_bin_particles(const ParticlesView& P, double dx, DenseMap map, int n_nodes, int* bin_of, int* counts,
                          int* start, int* cursor, int* pid, int* scan_tmp, const int* orig, cudaStream_t s);
void launch_p2g(const ParticlesView& P, BinsView bins, GridView g, double dx, const DevMaterial* mats, double ell,
                double dt, double* bin_part, cudaStream_t s, int jlo = 0, int jhi = -1, int lo = 0,
                int hi = -1);  // bins [jlo, jhi), rows [lo, hi)
/// Also writes dst.bin[t] = bin_of[pid[t]].
void launch_reorder_particles(const ParticlesView& src, const ParticlesView& dst, const int* pid, const int* bin_of,
                              const int* orig_src,
                              int* orig_dst, cudaStream_t s);
void launch_apply_bc(GridView g, double dx, const DevCollider* cols, int n_cols, cudaStream_t s);
/// Generic exclusive scan over n ints (out may alias nothing); tmp >= ceil(n/4096)+1 ints.
void launch_exclusive_scan(const int* in, int* out, int n, int* tmp, int* total_dev, cudaStream_t s);

// ---------------------------------------------------------------- objective (k_objective.cu)
/// Per-particle pass at nodal increment dv + alpha*p (p may be null): V_p psi partial sums
/// into partials[blockIdx] and, when stress != null, stores V_p * P F^T (9 per particle).
// ---- projected-Newton baselines (k_pn.cu)
void launch_block_apply(const double* dinv, const double* r, double* z, int n, cudaStream_t s);
void launch_pcg_xr(double* x, double* r, const double* p, const double* Ap, double alpha, long long n, cudaStream_t s);
void launch_pcg_p(double* p, const double* z, double beta, long long n, cudaStream_t s);
/// y = H u without H (objective.hpp:396-440) from the particle tensors Tu; dP: 9 * np scratch.
void launch_mf_multiply(const ParticlesView& P, BinsView bins, GridView g, const double* Tu, const double* u,
                        double* dP, double* y, cudaStream_t s);
/// Inverse block diagonal of the projected system (objective.hpp:366-392) into dinv (9 per node).
void launch_mf_block_diag_inv(const ParticlesView& P, BinsView bins, GridView g, const double* Tu, double* dinv,
                              cudaStream_t s);
/// 27-neighbour table of every active node (g.nb27 must point to n*27 ints).
void launch_fill_nb27(GridView g, int* nb27, cudaStream_t s);
/// u = vel + (dv + alpha p) per node (p may be null): the nodal velocity the virtual F sees.
void launch_node_u(GridView g, const double* dv, const double* p, double alpha, double* u, cudaStream_t s);
/// Per-particle elastic energy pe[p] (+ stress, + SVD cache) for particles [plo, phi).
void launch_particle_energy(const ParticlesView& P, GridView g, double dx, double dt, const DevMaterial* mats,
                            const double* u, double* stress, double* svd_out, double* pe, int nblocks, int* bad_flag,
                            cudaStream_t s, long long plo = 0, long long phi = -1);
/// ne[i] = the bin's particle energies + the node's kinetic / gravity terms, rows [lo, hi).
void launch_node_energy(GridView g, BinsView bins, const double* pe, double dt, const double* grav, const double* dv,
                        const double* p, double alpha, double* ne, int lo, int hi, cudaStream_t s);
/// g_i = dt * sum_p (V P F^T) grad w + m_i (dv_i - dt*grav); 0 on Dirichlet; nt[i] =
/// |g_i|^2 / scale_i^2.  Bin pass over bins [jlo, jhi), node pass over rows [lo, hi) (-1: n).
void launch_node_gradient(const ParticlesView& P, BinsView bins, GridView g, double dx, double dt, const double* grav,
                          const double* stress, const double* dv, double* gout, double* bin_part, double* nt,
                          int* bad_flag, cudaStream_t s, int jlo = 0, int jhi = -1, int lo = 0, int hi = -1);
/// Fixed-tree block partials of sum(a[0, n)) (then launch_sum_partials).
void launch_sum_array(const double* a, long long n, double* partials, int nblocks, cudaStream_t s);
void launch_sum_partials(const double* partials, int n, double* out, cudaStream_t s);

// vector helpers (deterministic block partials + fixed-order final sums)
void launch_dot_partials(const double* a, const double* b, long long n, double* partials, int nblocks, cudaStream_t s);
/// q <- q - coef_dev[k]*y (if y) then partial dot(s, q)
void launch_axpy_dot(double* q, const double* y, const double* coef_dev, int coef_idx, double coef_scale,
                     const double* s_vec, long long n, double* partials, int nblocks, cudaStream_t s);
/// coef_dev[k] = rho * sum(partials)  (alpha_k),  or coef_dev[k] = alpha_dev[k] - rho*sum (second loop)
void launch_finalize_coef(const double* partials, int n, double rho, const double* alpha_dev, int idx, double* coef_dev,
                          cudaStream_t s);
void launch_neg_copy(const double* a, double* out, long long n, cudaStream_t s);
/// out = a + alpha * b (two roundings, no contraction)
void launch_add_scaled(const double* a, const double* b, double alpha, double* out, long long n, cudaStream_t s);
void launch_scale(const double* a, double alpha, double* out, long long n, cudaStream_t s);
void launch_sub(const double* a, const double* b, double* out, long long n, cudaStream_t s);
/// y = g_new - g; partials for y.s, y.y, s.s (3 x nblocks)
void launch_ys_dots(const double* g_new, const double* g_old, double* y, const double* s, long long n,
                    double* partials, int nblocks, cudaStream_t s_);
void launch_zero_dirichlet_copy(const double* in, double* out, const uint8_t* dir, int n, cudaStream_t s);
void launch_final_velocity(GridView g, const double* dv, double* out, cudaStream_t s);

// ---------------------------------------------------------------- assembly (k_assembly.cu)
void launch_particle_tensors(const ParticlesView& P, GridView g, double dx, double dt, const DevMaterial* mats,
                             const double* u, const double* svd_in, int project, double* Tu, int* bad_flag,
                             cudaStream_t s, long long plo = 0, long long phi = -1);  // particles [plo, phi)
/// Column ids of every slot (-1 inactive); *active = the level's active-slot count.
void launch_fill_cols(LevelView L, unsigned long long* active, cudaStream_t s);
/// tile_counter: 1 device word (the row tiles' work counter).
void launch_assemble_rows(const ParticlesView& P, BinsView bins, GridView g, LevelView L, double dx,
                          const double* Tu, unsigned int* tile_counter, cudaStream_t s);
/// The level-0 assembly by bins (k_assembly.cu).  Stage A, launch_bin_pairs: the pair sums of bins
/// [b0, b1) into G, a ring of ring_cap bins x asm_pair_doubles() doubles (bin j at slot
/// j % ring_cap); bins without particles, without records in [plo, phi), or without a node in
/// rows [L.lo, L.hi) are skipped; *bins_done (may be null) counts the others.  Stage B,
/// launch_row_gather: rows [r0, r1) whose largest neighbour bin lies in [blo, bhi) sum their bins'
/// segments and write the row, its transposes, mass diagonal and Dirichlet projection.
/// counter: 1 device word each (distinct words).
int asm_pair_doubles();
void launch_bin_pairs(BinsView bins, GridView g, LevelView L, const double* Tu, double* G, int ring_cap, int b0, int b1,
                      long long plo, long long phi, unsigned int* counter, unsigned long long* bins_done,
                      cudaStream_t s);
void launch_row_gather(BinsView bins, GridView g, LevelView L, const double* G, int ring_cap, int r0, int r1, int blo,
                       int bhi, long long plo, long long phi, unsigned int* counter, cudaStream_t s);

// ---------------------------------------------------------------- multigrid (k_multigrid.cu)
/// quad: quadratic node embedding (multigrid.hpp:72-90).
void launch_mark_parents(LevelView fine, DenseMap cmap, int quad, uint8_t* flags, cudaStream_t s);
void launch_coarse_dirichlet(LevelView fine, DenseMap cmap, int quad, uint8_t* cdir, cudaStream_t s);
/// X: scratch per fine row of 64*9 doubles (linear) or (R_f+3)^3 * 9 (quadratic: coarse.radius == 3).
void launch_galerkin(LevelView fine, LevelView coarse, double* X, cudaStream_t s);
/// diag inverse, singular check, wave id per row (level 0: colour mod 3; coarse: wavefront).
/// D^-1 per row (+ singular flag) and the wave id per row (coarse: offsets = bbox min >> 1).
void launch_level_dinv(LevelView L, int* singular_flag, cudaStream_t s);
void launch_level_waves(LevelView L, int coarse, int modulus, const int* off, int* wave_of, cudaStream_t s);
/// Ints of `cursor` scratch launch_bucket_rows needs for n rows and nwaves waves (its scan_tmp
/// needs that / 4096 + 2).
int bucket_scratch_ints(int n, int nwaves);
void launch_bucket_rows(const int* wave_of, int n, int wmin, int* counts, int* start, int* cursor, int* rows,
                        int nwaves, int* scan_tmp, cudaStream_t s, int row_base = 0);  // rows [row_base, +n)
void launch_plane_starts(const int* coords, int n, int lo0, int nplanes, int* out, cudaStream_t s);
/// One level-0 smoother wave (k_sgs_wave) over the given rows.
void launch_sgs_wave1(LevelView L, const int* rows, int cnt, double* u, const double* b, cudaStream_t s);
void launch_spmv(LevelView L, const double* x, double* y, cudaStream_t s);
void launch_residual(LevelView L, const double* b, const double* u, double* r, cudaStream_t s);
void launch_restrict(LevelView fine, LevelView coarse, const double* rf, double* bc, cudaStream_t s);
void launch_prolong_add(LevelView fine, LevelView coarse, const double* uc, double* uf, cudaStream_t s);
/// One symmetric Gauss-Seidel sweep (forward + backward over the wave schedule), as a
/// cooperative persistent kernel with a grid barrier between waves.
/// bar: 2 device words of the caller's (the grid barrier's counter and release flag).
void launch_sgs(LevelView L, const int* wave_start, const int* wave_rows, int nwaves, double* u, const double* b,
                int grid_blocks, unsigned int* bar, cudaStream_t s, long long* trace = nullptr);
/// Jacobi-PCG from zero (pcg.hpp:17-46) as one cooperative kernel; writes x, iterations,
/// status (0 ok, 1 rho<0, 2 pAp<=0) into stat[0..1] and accumulates iterations into *iter_acc.
void launch_pcg(LevelView L, const double* b, double* x, double* r, double* z, double* p, double* Ap, double rel,
                int cap, double* partials, int* stat, int* iter_acc, int grid_blocks, cudaStream_t s);
/// The same sweep as one streaming launch per wave (large levels; waves given on the host).
/// Coarse smoother: both passes as a dataflow kernel; uf / ub: 3n-double scratch (the forward
/// and backward results, which double as the dependency flags).
void launch_sgs_flow(LevelView L, const int* order, const int* wave_of, double* u, const double* b, double* uf,
                     double* ub, cudaStream_t s);
/// Level-0 smoother: both passes, all waves, one persistent kernel with bulk-copy row streaming.
/// [q_lo, q_hi): the part of the flat (forward waves, then backward waves) sequence to run.
void launch_sgs_stream(LevelView L, const int* wave_start, const int* wave_rows, int nwaves, double* u,
                       const double* b, unsigned int* bar, cudaStream_t s, int q_lo = 0, int q_hi = -1,
                       int max_rows = 0);  // max_rows > 0: size the grid for waves of at most that many rows
void launch_sgs_waves(LevelView L, const int* wave_start_host, const int* wave_rows, int nwaves, double* u,
                      const double* b, cudaStream_t s);
int sgs_max_blocks();
constexpr int kSgsMaxWavesPersistent = 4096;
int pcg_max_blocks();

// ---------------------------------------------------------------- transfer (k_transfer.cu)
/// Inversions are counted for particles whose bin plane (axis 0) is in [own_lo, own_hi).
void launch_g2p_strain_advect(const ParticlesView& P, GridView g, double dx, double dt, const DevMaterial* mats,
                              int* inverted, cudaStream_t s, int own_lo = -(1 << 30), int own_hi = 1 << 30);
void launch_vmax(const ParticlesView& P, unsigned long long* vmax_bits, cudaStream_t s);
/// *bad = 1 if any id is outside [0, limit).
void launch_check_ids(const int* ids, long long n, int limit, int* bad, cudaStream_t s);

void launch_aos_to_soa(const double* in, double* out, long long n, int comps, cudaStream_t s);
void launch_soa_to_aos(const double* in, double* out, long long n, int comps, cudaStream_t s);
/// out[perm[t]*comps + k] = in[k*n + t]  (back to the caller's particle order)
void launch_soa_to_aos_perm(const double* in, double* out, long long n, int comps, const int* perm, cudaStream_t s);
void launch_iota(int* out, long long n, cudaStream_t s);
/// out[t] = in[perm[t]]
void launch_gather_perm(const double* in, double* out, long long n, const int* perm, cudaStream_t s);
void launch_fill(double* out, long long n, double value, cudaStream_t s);

constexpr int kMaxDevices = 64;
/// SM count of the current device (cached per device).
// ---------------------------------------------------------------- particle partition (k_transfer.cu)
/// keep / pack flags per local particle (see k_pp_classify).  coords: level-0 coords for the
/// pre-step plane of P.bin (null: take it from x).  Planes are absolute; owned [owned_lo,
/// owned_hi) after the step, pre-step owned [pre_lo, pre_hi).
void launch_pp_classify(const ParticlesView& P, const int* coords, int owned_lo, int owned_hi, int pre_lo, int pre_hi,
                        int gL, int gR, double dx, int* keep, int* pack, cudaStream_t s);
void launch_pp_pack(const ParticlesView& P, const int* orig, const int* flag, const int* pos, double dx, double* out,
                    cudaStream_t s);
void launch_pp_recv_flag(const double* rec, long long m, int lo, int hi, int* flag, cudaStream_t s);
/// Q (Q.n = n_keep + kept records): the kept particles of P in order, then the kept records.
void launch_pp_rebuild(const ParticlesView& P, const int* orig, const int* keep, const int* keep_pos, const double* rec,
                       long long mrec, const int* rflag, const int* rpos, long long n_keep, const ParticlesView& Q,
                       int* qorig, cudaStream_t s);
int pp_record_doubles();
/// Records -> interleaved caller-order device arrays (by original id); null outputs skipped.
void launch_pp_unpack_caller(const double* rec, long long m, double* x, double* v, double* F, double* C, double* Jp,
                             cudaStream_t s);

int num_sms();
/// cudaFuncAttributeMaxDynamicSharedMemorySize = smem for fn on the current device (once per
/// device; a no-op at <= 48 KB).
void set_max_dynamic_smem(const void* fn, int smem);
/// Co-resident CTAs of a kernel (occupancy x SMs).  Grid-stride kernels whose neighbouring
/// items share data launch exactly this many CTAs, so at any time the active items form one
/// contiguous window (L2 reuse) instead of being strided across the whole domain.
/// Memoized per (device, fn, threads, smem); sets the dynamic shared-memory attribute first.
int resident_blocks(const void* fn, int threads, int smem);

/// Kernel launches issued by this process (all contexts); every launch_* wrapper counts.
long long kernel_launch_count();
void count_launches(int k);

}  // namespace hotb200
