/* hot_c_api.h — C-ABI of the B200-native HOT implicit-MPM step (libhotb200.so).
 *
 * Drop-in boundary for the reference's hot path.  The reference has no FFI; its hot path
 * is the C++ template call
 *     StepStats advance_step(SimulationState&, const SceneConfig&, const SolverConfig&, T frame_end)
 * (/root/reference/proj/include/hotmpm/simulation.hpp:286-323), called once per step by the
 * CLI frame loop (/root/reference/proj/src/cli.cpp:75-81).  The entry points below are what
 * that call site binds instead (see INTEGRATION.md for the C++ shim with the same signature):
 * plain structs, caller-owned host buffers, int status codes, no torch / CUDA types.
 *
 * Conventions (mirroring the reference):
 *   - fp64, dim = 3 or dim = 2 on the device (a dim = 2 scene gets the 2D path, k2d.cu);
 *   - particle arrays are interleaved per particle: x[d*p+a], F[d*d*p + d*row + col]
 *     (row-major; the reference stores Eigen column-major, only the layout differs);
 *   - node vectors are interleaved [d*i+a] in lexicographic lattice order
 *     (grid.hpp:137-165, common.hpp:41);
 *   - errors map one-to-one onto the reference's exception types (section 5 of SURVEY.md);
 *     on HOT_E_SOLVER_FAILURE from hot_advance_step the particles are left unmodified
 *     (simulation.hpp:285,308-312).
 *   - a context is single-threaded and owns one CUDA stream on one device.
 */
#ifndef HOT_C_API_H
#define HOT_C_API_H

#ifdef __cplusplus
extern "C" {
#endif

#define HOT_API_VERSION 2

enum hot_status {
  HOT_OK = 0,
  HOT_E_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  HOT_E_SOLVER_FAILURE = 2,   /* hotmpm::SolverFailure  (common.hpp:124-126) */
  HOT_E_LOGIC = 3,            /* std::logic_error */
  HOT_E_DOMAIN = 4,           /* std::domain_error */
  HOT_E_CUDA = 5,             /* CUDA runtime / device failure */
  HOT_E_UNSUPPORTED = 6       /* feature not built for the device path (2D multi-GPU slabs) */
};

typedef struct hot_ctx hot_ctx;

/* scene.hpp:13-23 MaterialSpec; plasticity 0 none, 1 von_mises, 2 snow_clamp, 3 drucker_prager.
 * The last three fields are extensions the reference does not have:
 * elasticity 0 fixed-corotated (the reference's only model), 1 Neo-Hookean; hardening = the
 * Stomakhin snow hardening coefficient xi (0 = the reference's plain clamp); friction_angle =
 * the Drucker-Prager friction angle in degrees. */
typedef struct {
  double density, youngs, poisson;
  int plasticity;
  double yield_stress, clamp_lo, clamp_hi;
  int elasticity;
  double hardening, friction_angle;
} hot_material;

/* scene.hpp:25-32 ShapeSpec; kind 0 box, 1 sphere, 2 half_space, 3 cylinder */
typedef struct {
  int kind;
  double min[3], max[3], center[3];
  double radius;
  double point[3], normal[3], axis[3];
} hot_shape;

/* scene.hpp:34-40 MotionSpec; kind 0 static, 1 linear, 2 rotation */
typedef struct {
  int kind;
  double velocity[3], center[3], axis[3];
  double omega;
} hot_motion;

/* scene.hpp:47-52 ObjectSpec; init_kind 0 identity, 1 random_diagonal */
typedef struct {
  hot_shape shape;
  int material;
  double velocity[3];
  int init_kind;
  double init_lo, init_hi;
} hot_object;

/* scene.hpp:54-57 ColliderSpec */
typedef struct {
  hot_shape shape;
  hot_motion motion;
} hot_collider;

/* scene.hpp:61-84 SceneConfig (solver: 0 hot, 1 pn-pcg, 2 pn-pcg-mf, 3 pn-mgpcg, 4 lbfgs-h;
 * embedding: 0 quadratic, 1 linear) */
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
  const hot_material* materials;
  const hot_object* objects;
  const hot_collider* colliders;
} hot_scene;

/* solvers.hpp:14-29 SolverConfig */
typedef struct {
  double epsilon, tau;
  int levels, window;
  double ls_shrink, ls_armijo;
  int ls_max_steps, cg_cap, outer_cap, kind, embedding, pinned_coarse_iterations;
  double cn_length_factor;
} hot_solver_config;

/* simulation.hpp:275-281 StepStats */
typedef struct {
  double dt;
  int outer_iterations;
  long long inner_total;
  int node_count;
  int converged;
} hot_step_stats;

/* solvers.hpp:31-41 DiagnosticsRecord */
typedef struct {
  int frame;
  long long step;
  int outer_iteration;
  double scaled_residual, energy, step_length;
  long long inner_iterations, work_units;
  double wall_ms;
} hot_diag_row;

/* ---- library -------------------------------------------------------------------------- */
int hot_version(void);
int hot_device_count(void);

/* ---- context (replaces SimulationState + the advance_step call site) -------------------- */
/* Copies the scene; solver configuration = solver_config_from_scene (simulation.hpp:186-197). */
int hot_create(hot_ctx** out, const hot_scene* scene, int device);
void hot_destroy(hot_ctx* ctx);
const char* hot_last_error(const hot_ctx* ctx);
int hot_set_solver(hot_ctx* ctx, const hot_solver_config* cfg);

/* sample_scene_particles (simulation.hpp:221-254), host-side, libstdc++ mt19937_64 stream.
 * Call with x == NULL to get the count in *n; then with arrays of that size. */
int hot_sample_scene_particles(const hot_scene* scene, long long* n, double* x, double* v, double* mass,
                               double* volume, double* F, double* C, int* material);

int hot_upload_particles(hot_ctx* ctx, long long n, const double* x, const double* v, const double* mass,
                         const double* volume, const double* F, const double* C, const int* material);
/* Plastic volume ratio J_p per particle, caller order (extension: Stomakhin snow hardening; the
 * reference's Particle has no plastic state, transfer.hpp:12-21).  Defaults to 1 at upload; only
 * scenes with a snow material store it (hot_set_plastic_state returns HOT_E_INVALID_ARGUMENT
 * otherwise; hot_get_plastic_state reports 1).  n = hot_particle_count. */
int hot_set_plastic_state(hot_ctx* ctx, const double* Jp);
int hot_get_plastic_state(hot_ctx* ctx, double* Jp);
int hot_download_particles(hot_ctx* ctx, double* x, double* v, double* F, double* C);
int hot_particle_count(hot_ctx* ctx, long long* n);
int hot_set_time(hot_ctx* ctx, double time, int frame, long long step_index);
int hot_get_time(hot_ctx* ctx, double* time, int* frame, long long* step_index, long long* inversion_warnings);

/* One implicit step: advance_step body (simulation.hpp:286-323). */
int hot_advance_step(hot_ctx* ctx, double frame_end, hot_step_stats* out);

/* Diagnostics rows appended by every solve (solvers.hpp:181-184). rows may be NULL. */
int hot_diagnostics(hot_ctx* ctx, hot_diag_row* rows, int cap, int* n);
int hot_clear_diagnostics(hot_ctx* ctx);

/* ---- stage taps (the reference's test-visible sub-calls; parity testing) ---------------- */
/* activate_grid + p2g + apply_boundary_scripts + make_objective_state at the given dt/time
 * (simulation.hpp:297-305), without solving. */
int hot_stage_prepare(hot_ctx* ctx, double dt, double time);
int hot_stage_node_count(hot_ctx* ctx, int* n);
/* Any output may be NULL. coords: 3n ints, lexicographic. cn_scale: l*xi*dt per node. */
int hot_stage_grid(hot_ctx* ctx, int* coords, double* mass, double* velocity, double* momentum,
                   unsigned char* dirichlet, double* bc_velocity, double* cn_scale);
int hot_stage_set_grid(hot_ctx* ctx, const double* velocity, const unsigned char* dirichlet, const double* bc_velocity);
int hot_stage_energy(hot_ctx* ctx, const double* dv, double* energy);
int hot_stage_gradient(hot_ctx* ctx, const double* dv, double* g, double* scaled_norm);
/* assemble_hessian at dv (objective.hpp:318-363) and build_hierarchy (multigrid.hpp:258-294). */
int hot_stage_assemble(hot_ctx* ctx, const double* dv, int project);
int hot_stage_build_hierarchy(hot_ctx* ctx, int levels, int embedding);
int hot_stage_level_count(hot_ctx* ctx, int* levels);
int hot_stage_level_shape(hot_ctx* ctx, int level, int* rows, int* slots);
/* blocks: rows*slots*9 doubles (row-major 3x3 per slot, zero where cols == -1); cols rows*slots; slots from
 * hot_stage_level_shape: 125 (radius 2) or 343 (radius 3, quadratic-embedding coarse levels). */
int hot_stage_level_matrix(hot_ctx* ctx, int level, double* blocks, int* cols, int* coords, unsigned char* dirichlet);
int hot_stage_matvec(hot_ctx* ctx, int level, const double* x, double* y);
int hot_stage_vcycle(hot_ctx* ctx, const double* b, double* u, int* coarse_iterations);
int hot_stage_step_grid(hot_ctx* ctx, double* velocity, double* dv, int* outer, long long* inner, int* converged,
                        int frame, long long step);

/* ---- measurement ------------------------------------------------------------------------ */
/* CUDA stream (cudaStream_t) the context launches on, for external event timing. */
void* hot_stream(hot_ctx* ctx);
/* Per-phase device timing (CUDA events on the context stream). enable=1 starts/resets. */
int hot_profile_enable(hot_ctx* ctx, int enable);
/* Fills up to cap (name, total_ms, launches, bytes) records; returns count in *n.  bytes are
 * algorithmic HBM bytes; a negative value is minus the algorithmic fp64 flop count of an
 * ALU-bound phase (the level-0 assembly). */
int hot_profile_read(hot_ctx* ctx, char* names /* cap*32 */, double* total_ms, long long* launches,
                     double* bytes, int cap, int* n);
/* Kernel launches issued by this context since creation (all phases). */
long long hot_kernel_launches(hot_ctx* ctx);

/* ---- multi-GPU: spatial slabs along lattice axis 0 -------------
 * The reference is single-process (its only parallelism is parallel_for over host threads,
 * common.hpp:77-83); these entry points are new.  One context per GPU, one process per GPU.
 * Every rank uploads the SAME particles; each step the ranks cut the level-0 rows into slabs
 * of lattice planes (axis 0 is the most significant key of the reference order, common.hpp:41,
 * so a slab is a contiguous range of global rows) and split the level-0 assembly, the level-1
 * Galerkin product and the level-0 smoother / residual between them.  All other state stays
 * replicated and every rank's result is bitwise identical to the single-GPU step.
 * Only the HOT solver (kind 0) with the linear embedding and >= 2 levels shards; other solver
 * configurations run replicated on every rank.  Each rank stores only its rows of the level-0
 * matrix, so after a sharded solve the matrix taps (hot_stage_level_*) report no level. */

/* Caller-owned collectives (tests, or any transport the caller owns: gloo, MPI ...).  Every
 * callback is collective (all ranks call it in the same order) and returns 0 on success.
 * device_buffers = 0: buf is host memory (the library stages the ranges through pinned
 * memory); 1: buf is the device buffer itself (the context stream is synchronised before the
 * call, and the callback must have finished writing when it returns). */
typedef struct {
  void* user;
  int rank, size;
  /* rank r's byte range [off[r], off[r+1]) of buf is delivered to every rank (off: size+1). */
  int (*allgather_ranges)(void* user, void* buf, const long long* off);
  /* halo exchange: edges[4r..4r+3] = byte ranges [a,b) (rank r's first planes) and [c,d) (its
   * last planes); rank r receives rank r-1's [c,d) and rank r+1's [a,b) into the same offsets. */
  int (*halo)(void* user, void* buf, const long long* edges);
  /* element-wise max over ranks of n ints (host memory), in place. */
  int (*allreduce_max_i32)(void* user, int* v, int n);
  int device_buffers;
} hot_comm_host;

int hot_set_comm_host(hot_ctx* ctx, const hot_comm_host* comm);
/* NCCL transport (libnccl.so.2, loaded at run time): rank 0 calls hot_nccl_unique_id, the
 * caller broadcasts the 128 bytes (e.g. torch.distributed), then every rank joins. */
int hot_nccl_unique_id(unsigned char id[128]);
int hot_set_comm_nccl(hot_ctx* ctx, const unsigned char id[128], int rank, int size);

typedef struct {
  int rank, size;
  int sharded;              /* 1 when the last solve ran slab-sharded */
  int plane_lo, plane_hi;   /* owned lattice planes [lo, hi) along axis 0 (absolute coordinates) */
  int row_lo, row_hi;       /* owned level-0 rows */
  int crow_lo, crow_hi;     /* owned level-1 rows */
  int asm_lo, asm_hi;       /* level-0 rows this rank assembles (owned + the left extension) */
  long long halo_exchanges; /* level-0 halo exchanges issued since creation */
  long long gathers;        /* row-range allgathers issued since creation */
  long long particles_local; /* particles this rank stores (owned + ghost copies when partitioned) */
  long long particles_total; /* particles of the scene */
  int partitioned;          /* 1: particles are partitioned along the slab cut */
} hot_shard_info_t;
int hot_shard_info(hot_ctx* ctx, hot_shard_info_t* out);

/* Slab planner (pure host function, no context): cut planes [plane_lo, plane_lo + nplanes)
 * into `size` slabs of consecutive planes balancing weight[] (one weight per plane), every
 * interior cut at a multiple of `align` (absolute coordinate) and every slab >= min_width
 * planes.  bounds: size+1 absolute plane coordinates, bounds[0] = plane_lo,
 * bounds[size] = plane_lo + nplanes.  HOT_E_INVALID_ARGUMENT when no such cut exists. */
int hot_plan_slabs(int plane_lo, int nplanes, const long long* weight, int size, int align, int min_width,
                   int* bounds);

#ifdef __cplusplus
}
#endif

#endif /* HOT_C_API_H */
