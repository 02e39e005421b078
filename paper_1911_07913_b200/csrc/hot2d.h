// The 2D (dim = 2) device path of the HOT step: a context of its own behind the same C-ABI
// entry points (hot_context.cu forwards every call on a dim = 2 context here).  Not part of the
// C-ABI.
#pragma once

#include <string>

#include "../../include/hot_c_api.h"
#include "hot_internal.h"

namespace hotb200 {

/// Material::elastic / von_mises / snow / drucker_prager (constitutive.hpp:12-52) with the
/// stiffness scale ||dP/dF(I)||_F of dimension dim (constitutive.hpp:255-258).
DevMaterial make_dev_material(const hot_material& m, int dim);

struct Context2D;

Context2D* ctx2d_new(int device, const hot_scene& s);  // throws like the 3D context
void ctx2d_delete(Context2D* c);
void ctx2d_set_solver(Context2D* c, const hot_solver_config& cfg);
void ctx2d_upload(Context2D* c, long long n, const double* x, const double* v, const double* mass, const double* vol,
                  const double* F, const double* C, const int* mat);
void ctx2d_download(Context2D* c, double* x, double* v, double* F, double* C);
void ctx2d_set_plastic_state(Context2D* c, const double* Jp);
void ctx2d_get_plastic_state(Context2D* c, double* Jp);
long long ctx2d_particle_count(Context2D* c);
void ctx2d_set_time(Context2D* c, double time, int frame, long long step);
void ctx2d_get_time(Context2D* c, double* time, int* frame, long long* step, long long* inversions);
void ctx2d_advance(Context2D* c, double frame_end, hot_step_stats* out);
int ctx2d_diagnostics(Context2D* c, hot_diag_row* rows, int cap);
void ctx2d_clear_diagnostics(Context2D* c);
void ctx2d_prepare(Context2D* c, double dt, double time);
int ctx2d_node_count(Context2D* c);
void ctx2d_grid(Context2D* c, int* coords, double* mass, double* velocity, double* momentum, unsigned char* dirichlet,
                double* bc_velocity, double* cn_scale);
void ctx2d_set_grid(Context2D* c, const double* velocity, const unsigned char* dirichlet, const double* bc_velocity);
void ctx2d_energy(Context2D* c, const double* dv, double* energy);
void ctx2d_gradient(Context2D* c, const double* dv, double* g, double* scaled_norm);
void ctx2d_assemble(Context2D* c, const double* dv, int project);
void ctx2d_build_hierarchy(Context2D* c, int levels, int embedding);
int ctx2d_level_count(Context2D* c);
void ctx2d_level_shape(Context2D* c, int level, int* rows, int* slots);
void ctx2d_level_matrix(Context2D* c, int level, double* blocks, int* cols, int* coords, unsigned char* dirichlet);
void ctx2d_matvec(Context2D* c, int level, const double* x, double* y);
void ctx2d_vcycle(Context2D* c, const double* b, double* u, int* coarse_iterations);
void ctx2d_step_grid(Context2D* c, double* velocity, double* dv, int* outer, long long* inner, int* converged, int frame,
                     long long step);
void* ctx2d_stream(Context2D* c);

}  // namespace hotb200
