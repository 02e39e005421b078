"""ctypes binding of the C-ABI in include/hot_c_api.h (libhotb200.so, built in-tree).

This is the reference-side binding a Python host would add; the C++ host binds the same
symbols directly.  Loading fails loudly when the library is missing:
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .scene import SceneConfig

_HERE = os.path.dirname(os.path.abspath(__file__))
# HOT_LIB_VARIANT=<name> loads lib/libhotb200_<name>.so: a tuning build of the same sources
# with other compile-time constants (tools/asm_variants.sh); unset in tests and the bench
_VARIANT = os.environ.get("HOT_LIB_VARIANT")
LIB_PATH = os.path.join(_HERE, "lib", f"libhotb200_{_VARIANT}.so" if _VARIANT else "libhotb200.so")

HOT_OK, HOT_E_INVALID_ARGUMENT, HOT_E_SOLVER_FAILURE, HOT_E_LOGIC, HOT_E_DOMAIN, HOT_E_CUDA, HOT_E_UNSUPPORTED = range(7)


class HotError(RuntimeError):
    kind = "error"

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class SolverFailure(HotError):
    kind = "SolverFailure"


class InvalidArgument(HotError, ValueError):
    kind = "invalid_argument"


class LogicError(HotError):
    kind = "logic_error"


class DomainError(HotError):
    kind = "domain_error"


class CudaError(HotError):
    kind = "cuda"


class Unsupported(HotError, NotImplementedError):
    kind = "unsupported"


_ERRORS = {HOT_E_INVALID_ARGUMENT: InvalidArgument, HOT_E_SOLVER_FAILURE: SolverFailure, HOT_E_LOGIC: LogicError,
           HOT_E_DOMAIN: DomainError, HOT_E_CUDA: CudaError, HOT_E_UNSUPPORTED: Unsupported}


class hot_material(C.Structure):
    _fields_ = [("density", C.c_double), ("youngs", C.c_double), ("poisson", C.c_double), ("plasticity", C.c_int),
                ("yield_stress", C.c_double), ("clamp_lo", C.c_double), ("clamp_hi", C.c_double),
                ("elasticity", C.c_int), ("hardening", C.c_double), ("friction_angle", C.c_double)]


class hot_shape(C.Structure):
    _fields_ = [("kind", C.c_int), ("min", C.c_double * 3), ("max", C.c_double * 3), ("center", C.c_double * 3),
                ("radius", C.c_double), ("point", C.c_double * 3), ("normal", C.c_double * 3),
                ("axis", C.c_double * 3)]


class hot_motion(C.Structure):
    _fields_ = [("kind", C.c_int), ("velocity", C.c_double * 3), ("center", C.c_double * 3),
                ("axis", C.c_double * 3), ("omega", C.c_double)]


class hot_object(C.Structure):
    _fields_ = [("shape", hot_shape), ("material", C.c_int), ("velocity", C.c_double * 3), ("init_kind", C.c_int),
                ("init_lo", C.c_double), ("init_hi", C.c_double)]


class hot_collider(C.Structure):
    _fields_ = [("shape", hot_shape), ("motion", hot_motion)]


class hot_scene(C.Structure):
    _fields_ = [("dim", C.c_int), ("dx", C.c_double), ("gravity", C.c_double * 3), ("fps", C.c_double),
                ("frames", C.c_int), ("epsilon", C.c_double), ("tau", C.c_double), ("levels", C.c_int),
                ("window", C.c_int), ("solver", C.c_int), ("embedding", C.c_int), ("cn_length_factor", C.c_double),
                ("seed", C.c_ulonglong), ("ppc", C.c_int), ("poisson_sampling", C.c_int),
                ("n_materials", C.c_int), ("n_objects", C.c_int), ("n_colliders", C.c_int),
                ("materials", C.POINTER(hot_material)), ("objects", C.POINTER(hot_object)),
                ("colliders", C.POINTER(hot_collider))]


class hot_solver_config(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("tau", C.c_double), ("levels", C.c_int), ("window", C.c_int),
                ("ls_shrink", C.c_double), ("ls_armijo", C.c_double), ("ls_max_steps", C.c_int),
                ("cg_cap", C.c_int), ("outer_cap", C.c_int), ("kind", C.c_int), ("embedding", C.c_int),
                ("pinned_coarse_iterations", C.c_int), ("cn_length_factor", C.c_double)]


class hot_step_stats(C.Structure):
    _fields_ = [("dt", C.c_double), ("outer_iterations", C.c_int), ("inner_total", C.c_longlong),
                ("node_count", C.c_int), ("converged", C.c_int)]


class hot_diag_row(C.Structure):
    _fields_ = [("frame", C.c_int), ("step", C.c_longlong), ("outer_iteration", C.c_int),
                ("scaled_residual", C.c_double), ("energy", C.c_double), ("step_length", C.c_double),
                ("inner_iterations", C.c_longlong), ("work_units", C.c_longlong), ("wall_ms", C.c_double)]


EXPORTS = [
    "hot_version", "hot_device_count", "hot_create", "hot_destroy", "hot_last_error", "hot_set_solver",
    "hot_sample_scene_particles", "hot_upload_particles", "hot_download_particles", "hot_particle_count",
    "hot_set_plastic_state", "hot_get_plastic_state",
    "hot_set_time", "hot_get_time", "hot_advance_step", "hot_diagnostics", "hot_clear_diagnostics",
    "hot_stage_prepare", "hot_stage_node_count", "hot_stage_grid", "hot_stage_set_grid", "hot_stage_energy",
    "hot_stage_gradient", "hot_stage_assemble", "hot_stage_build_hierarchy", "hot_stage_level_count",
    "hot_stage_level_shape", "hot_stage_level_matrix", "hot_stage_matvec", "hot_stage_vcycle",
    "hot_stage_step_grid", "hot_stream", "hot_profile_enable", "hot_profile_read", "hot_kernel_launches",
    "hot_set_comm_host", "hot_nccl_unique_id", "hot_set_comm_nccl", "hot_shard_info", "hot_plan_slabs",
]

# multi-GPU slabs (hot_c_api.h): host-staged collectives and the shard report
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_longlong))
HALO_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_longlong))
MAXI32_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int), C.c_int)


class hot_comm_host(C.Structure):
    _fields_ = [("user", C.c_void_p), ("rank", C.c_int), ("size", C.c_int), ("allgather_ranges", ALLGATHER_FN),
                ("halo", HALO_FN), ("allreduce_max_i32", MAXI32_FN), ("device_buffers", C.c_int)]


class hot_shard_info_t(C.Structure):
    _fields_ = [("rank", C.c_int), ("size", C.c_int), ("sharded", C.c_int), ("plane_lo", C.c_int),
                ("plane_hi", C.c_int), ("row_lo", C.c_int), ("row_hi", C.c_int), ("crow_lo", C.c_int),
                ("crow_hi", C.c_int), ("asm_lo", C.c_int), ("asm_hi", C.c_int), ("halo_exchanges", C.c_longlong),
                ("gathers", C.c_longlong), ("particles_local", C.c_longlong), ("particles_total", C.c_longlong),
                ("partitioned", C.c_int)]


_lib = None


def lib():
    """Loads libhotb200.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(make -C paper_1911_07913_b200/csrc); the B200 path has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, dp, ip, i64p = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_longlong)
    u8p = C.POINTER(C.c_ubyte)
    L.hot_create.argtypes = [C.POINTER(vp), C.POINTER(hot_scene), C.c_int]
    L.hot_destroy.argtypes = [vp]
    L.hot_last_error.restype = C.c_char_p
    L.hot_last_error.argtypes = [vp]
    L.hot_set_solver.argtypes = [vp, C.POINTER(hot_solver_config)]
    L.hot_sample_scene_particles.argtypes = [C.POINTER(hot_scene), i64p, dp, dp, dp, dp, dp, dp, ip]
    L.hot_upload_particles.argtypes = [vp, C.c_longlong, dp, dp, dp, dp, dp, dp, ip]
    L.hot_download_particles.argtypes = [vp, dp, dp, dp, dp]
    L.hot_set_plastic_state.argtypes = [vp, dp]
    L.hot_get_plastic_state.argtypes = [vp, dp]
    L.hot_particle_count.argtypes = [vp, i64p]
    L.hot_set_time.argtypes = [vp, C.c_double, C.c_int, C.c_longlong]
    L.hot_get_time.argtypes = [vp, dp, ip, i64p, i64p]
    L.hot_advance_step.argtypes = [vp, C.c_double, C.POINTER(hot_step_stats)]
    L.hot_diagnostics.argtypes = [vp, C.POINTER(hot_diag_row), C.c_int, ip]
    L.hot_clear_diagnostics.argtypes = [vp]
    L.hot_stage_prepare.argtypes = [vp, C.c_double, C.c_double]
    L.hot_stage_node_count.argtypes = [vp, ip]
    L.hot_stage_grid.argtypes = [vp, ip, dp, dp, dp, u8p, dp, dp]
    L.hot_stage_set_grid.argtypes = [vp, dp, u8p, dp]
    L.hot_stage_energy.argtypes = [vp, dp, dp]
    L.hot_stage_gradient.argtypes = [vp, dp, dp, dp]
    L.hot_stage_assemble.argtypes = [vp, dp, C.c_int]
    L.hot_stage_build_hierarchy.argtypes = [vp, C.c_int, C.c_int]
    L.hot_stage_level_count.argtypes = [vp, ip]
    L.hot_stage_level_shape.argtypes = [vp, C.c_int, ip, ip]
    L.hot_stage_level_matrix.argtypes = [vp, C.c_int, dp, ip, ip, u8p]
    L.hot_stage_matvec.argtypes = [vp, C.c_int, dp, dp]
    L.hot_stage_vcycle.argtypes = [vp, dp, dp, ip]
    L.hot_stage_step_grid.argtypes = [vp, dp, dp, ip, i64p, ip, C.c_int, C.c_longlong]
    L.hot_stream.restype = vp
    L.hot_stream.argtypes = [vp]
    L.hot_profile_enable.argtypes = [vp, C.c_int]
    L.hot_profile_read.argtypes = [vp, C.c_char_p, dp, i64p, dp, C.c_int, ip]
    L.hot_kernel_launches.restype = C.c_longlong
    L.hot_kernel_launches.argtypes = [vp]
    L.hot_set_comm_host.argtypes = [vp, C.POINTER(hot_comm_host)]
    L.hot_nccl_unique_id.argtypes = [C.POINTER(C.c_ubyte)]
    L.hot_set_comm_nccl.argtypes = [vp, C.POINTER(C.c_ubyte), C.c_int, C.c_int]
    L.hot_shard_info.argtypes = [vp, C.POINTER(hot_shard_info_t)]
    L.hot_plan_slabs.argtypes = [C.c_int, C.c_int, i64p, C.c_int, C.c_int, C.c_int, ip]
    _lib = L
    return L


def dptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def iptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int))


def u8ptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_ubyte))


def raise_for(code, msg):
    if code != HOT_OK:
        raise _ERRORS.get(code, HotError)(code, msg)


# -------------------------------------------------------------------------------------------
# SceneConfig -> hot_scene
# -------------------------------------------------------------------------------------------
_SHAPES = {"box": 0, "sphere": 1, "half_space": 2, "cylinder": 3}
_MOTIONS = {"static": 0, "linear": 1, "rotation": 2}
_PLAST = {"none": 0, "von_mises": 1, "snow_clamp": 2, "drucker_prager": 3}
_ELASTICITY = {"fixed_corotated": 0, "neo_hookean": 1}
SOLVER_KINDS = {"hot": 0, "pn-pcg": 1, "pn-pcg-mf": 2, "pn-mgpcg": 3, "lbfgs-h": 4}


def _v3(v):
    a = (C.c_double * 3)()
    for i in range(3):
        a[i] = float(v[i]) if i < len(v) else 0.0
    return a


def _shape(s):
    h = hot_shape()
    h.kind = _SHAPES[s.kind]
    h.min, h.max, h.center = _v3(s.min), _v3(s.max), _v3(s.center)
    h.radius = s.radius
    h.point, h.normal, h.axis = _v3(s.point), _v3(s.normal), _v3(s.axis)
    return h


def scene_to_c(sc: SceneConfig):
    """Returns (hot_scene, keepalive)."""
    mats = (hot_material * len(sc.materials))()
    for i, m in enumerate(sc.materials):
        mats[i] = hot_material(m.density, m.youngs, m.poisson, _PLAST[m.plasticity.kind], m.plasticity.yield_stress,
                               m.plasticity.clamp_lo, m.plasticity.clamp_hi, _ELASTICITY[m.elasticity],
                               m.plasticity.hardening, m.plasticity.friction_angle)
    objs = (hot_object * len(sc.objects))()
    for i, o in enumerate(sc.objects):
        objs[i].shape = _shape(o.shape)
        objs[i].material = o.material
        objs[i].velocity = _v3(o.velocity)
        objs[i].init_kind = 1 if o.initial_deformation.kind == "random_diagonal" else 0
        objs[i].init_lo = o.initial_deformation.lo
        objs[i].init_hi = o.initial_deformation.hi
    cols = (hot_collider * max(1, len(sc.colliders)))()
    for i, c in enumerate(sc.colliders):
        cols[i].shape = _shape(c.shape)
        m = hot_motion()
        m.kind = _MOTIONS[c.motion.kind]
        m.velocity, m.center, m.axis = _v3(c.motion.velocity), _v3(c.motion.center), _v3(c.motion.axis)
        m.omega = c.motion.omega
        cols[i].motion = m
    h = hot_scene()
    h.dim, h.dx, h.gravity, h.fps, h.frames = sc.dim, sc.dx, _v3(sc.gravity), sc.fps, sc.frames
    h.epsilon, h.tau, h.levels, h.window = sc.epsilon, sc.tau, sc.levels, sc.window
    h.solver = SOLVER_KINDS[sc.solver]
    h.embedding = 1 if sc.embedding == "linear" else 0
    h.cn_length_factor, h.seed, h.ppc = sc.cn_length_factor, sc.seed, sc.ppc
    h.poisson_sampling = 1 if sc.sampling == "poisson" else 0
    h.n_materials, h.n_objects, h.n_colliders = len(sc.materials), len(sc.objects), len(sc.colliders)
    h.materials = C.cast(mats, C.POINTER(hot_material))
    h.objects = C.cast(objs, C.POINTER(hot_object))
    h.colliders = C.cast(cols, C.POINTER(hot_collider))
    return h, (mats, objs, cols)


def sample_scene_particles(sc: SceneConfig):
    """simulation.hpp:221-254 through the C-ABI (host-only; no device needed).

    Returns a dict of interleaved arrays: x (n,d), v (n,d), mass (n), volume (n), F (n,d,d),
    C (n,d,d), material (n)."""
    h, keep = scene_to_c(sc)
    L = lib()
    n = C.c_longlong()
    raise_for(L.hot_sample_scene_particles(C.byref(h), C.byref(n), None, None, None, None, None, None, None),
              "sample_scene_particles failed")
    d = sc.dim
    N = n.value
    out = dict(x=np.zeros((N, d)), v=np.zeros((N, d)), mass=np.zeros(N), volume=np.zeros(N),
               F=np.zeros((N, d, d)), C=np.zeros((N, d, d)), material=np.zeros(N, dtype=np.int32))
    if N:
        raise_for(L.hot_sample_scene_particles(C.byref(h), C.byref(n), dptr(out["x"]), dptr(out["v"]),
                                               dptr(out["mass"]), dptr(out["volume"]), dptr(out["F"]),
                                               dptr(out["C"]), iptr(out["material"])),
                  "sample_scene_particles failed")
    del keep
    return out
