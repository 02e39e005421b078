"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over the CPU parity oracle (liboracle.so).

The oracle is a plain-C++ restatement of the reference HOT solver
(/root/reference/proj/include/hotmpm/*.hpp; see oracle/hot_oracle.hpp for per-function
file:line citations).  Only tests/, bench.py's CPU-baseline / ``--impl reference`` leg and
``__graft_entry__.smoke()`` may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

ERRORS = {1: "invalid_argument", 2: "SolverFailure", 3: "logic_error", 4: "domain_error", 5: "error"}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


class Material(C.Structure):
    _fields_ = [("density", C.c_double), ("youngs", C.c_double), ("poisson", C.c_double),
                ("plasticity", C.c_int), ("yield_stress", C.c_double), ("clamp_lo", C.c_double),
                ("clamp_hi", C.c_double), ("elasticity", C.c_int), ("hardening", C.c_double),
                ("friction_angle", C.c_double)]


class Shape(C.Structure):
    _fields_ = [("kind", C.c_int), ("min", C.c_double * 3), ("max", C.c_double * 3),
                ("center", C.c_double * 3), ("radius", C.c_double), ("point", C.c_double * 3),
                ("normal", C.c_double * 3), ("axis", C.c_double * 3)]


class Motion(C.Structure):
    _fields_ = [("kind", C.c_int), ("velocity", C.c_double * 3), ("center", C.c_double * 3),
                ("axis", C.c_double * 3), ("omega", C.c_double)]


class Object(C.Structure):
    _fields_ = [("shape", Shape), ("material", C.c_int), ("velocity", C.c_double * 3),
                ("init_kind", C.c_int), ("init_lo", C.c_double), ("init_hi", C.c_double)]


class Collider(C.Structure):
    _fields_ = [("shape", Shape), ("motion", Motion)]


class Scene(C.Structure):
    _fields_ = [("dim", C.c_int), ("dx", C.c_double), ("gravity", C.c_double * 3), ("fps", C.c_double),
                ("frames", C.c_int), ("epsilon", C.c_double), ("tau", C.c_double), ("levels", C.c_int),
                ("window", C.c_int), ("solver", C.c_int), ("embedding", C.c_int),
                ("cn_length_factor", C.c_double), ("seed", C.c_ulonglong), ("ppc", C.c_int),
                ("poisson_sampling", C.c_int), ("n_materials", C.c_int), ("n_objects", C.c_int),
                ("n_colliders", C.c_int), ("materials", C.POINTER(Material)), ("objects", C.POINTER(Object)),
                ("colliders", C.POINTER(Collider))]


class Solver(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("tau", C.c_double), ("levels", C.c_int), ("window", C.c_int),
                ("ls_shrink", C.c_double), ("ls_armijo", C.c_double), ("ls_max_steps", C.c_int),
                ("cg_cap", C.c_int), ("outer_cap", C.c_int), ("kind", C.c_int), ("embedding", C.c_int),
                ("pinned_coarse_iterations", C.c_int), ("cn_length_factor", C.c_double)]


APPLY_FN = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)
ENERGY_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)

SOLVERS = {"hot": 0, "pn-pcg": 1, "pn-pcg-mf": 2, "pn-mgpcg": 3, "lbfgs-h": 4}
SHAPES = {"box": 0, "sphere": 1, "half_space": 2, "cylinder": 3}
MOTIONS = {"static": 0, "linear": 1, "rotation": 2}
PLAST = {"none": 0, "von_mises": 1, "snow_clamp": 2, "drucker_prager": 3}
QUADRATIC, LINEAR = 0, 1

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        vp, dp, ip, i64p = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_longlong)
        L.orc_new.restype = vp
        L.orc_new.argtypes = [C.c_int]
        L.orc_free.argtypes = [vp]
        L.orc_error.restype = C.c_char_p
        L.orc_error.argtypes = [vp]
        L.orc_point_error.restype = C.c_char_p
        L.orc_particle_count.restype = C.c_longlong
        L.orc_particle_count.argtypes = [vp]
        L.orc_diag_count.restype = C.c_longlong
        L.orc_diag_count.argtypes = [vp]
        for name in ["orc_kernel_weight_1d", "orc_kernel_derivative_1d"]:
            getattr(L, name).restype = C.c_double
            getattr(L, name).argtypes = [C.c_int, C.c_double]
        L.orc_kernel_weight.restype = C.c_double
        L.orc_kernel_weight.argtypes = [C.c_int, C.c_int, dp]
        L.orc_kernel_gradient.argtypes = [C.c_int, C.c_int, dp, C.c_double, dp]
        L.orc_stencil_base.argtypes = [C.c_int, dp, C.c_double, C.c_int, ip]
        L.orc_cfl_dt.restype = C.c_double
        L.orc_cfl_dt.argtypes = [C.c_double, C.c_double, C.c_double]
        L.orc_adaptive_cg_tolerance.restype = C.c_double
        L.orc_adaptive_cg_tolerance.argtypes = [C.c_double, C.c_double]
        L.orc_energy.argtypes = [vp, dp, dp]
        L.orc_advance_step.argtypes = [vp, C.c_double, dp, ip, i64p, ip, ip]
        L.orc_set_particles.argtypes = [vp, C.c_longlong, dp, dp, dp, dp, dp, dp, ip]
        L.orc_get_particles.argtypes = [vp, dp, dp, dp, dp, dp, dp, ip]
        L.orc_set_sim_state.argtypes = [vp, C.c_double, C.c_longlong, C.c_int]
        L.orc_step_grid.argtypes = [vp, dp, dp, ip, i64p, ip, ip, C.c_int, C.c_longlong]
        L.orc_make_state.argtypes = [vp, C.c_double]
        L.orc_apply_bc.argtypes = [vp, C.c_double]
        L.orc_update_strain.argtypes = [vp, C.c_double, i64p]
        L.orc_advect.argtypes = [vp, C.c_double]
        L.orc_pcg.argtypes = [C.c_int, APPLY_FN, APPLY_FN, vp, dp, C.c_double, C.c_int, dp, ip, ip]
        L.orc_line_search.argtypes = [ENERGY_FN, vp, C.c_double, C.c_double, C.c_void_p, dp, dp, ip]
        L.orc_lbfgs_new.restype = vp
        L.orc_lbfgs_new.argtypes = [C.c_int]
        L.orc_lbfgs_free.argtypes = [vp]
        L.orc_lbfgs_push.argtypes = [vp, C.c_int, dp, dp]
        L.orc_lbfgs_size.argtypes = [vp]
        L.orc_lbfgs_direction.argtypes = [vp, C.c_int, dp, APPLY_FN, vp, dp]
        L.orc_set_gravity_dx.argtypes = [vp, dp, C.c_double, C.c_double]
        L.orc_particle_jp.argtypes = [vp, dp, dp]
        L.orc_model_energy.argtypes = [C.c_int, dp, vp, C.c_double, dp]
        L.orc_model_stress.argtypes = [C.c_int, dp, vp, C.c_double, dp]
        L.orc_model_dpdf.argtypes = [C.c_int, dp, vp, C.c_double, C.c_int, dp]
        L.orc_return_map_jp.argtypes = [C.c_int, dp, vp, dp, dp]
        L.orc_hardening_factor.restype = C.c_double
        L.orc_hardening_factor.argtypes = [vp, C.c_double]
        _lib = L
    return _lib


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int))


def _f64(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None:
        assert a.size == n, (a.size, n)
    return a


def _check_point(code):
    if code:
        raise OracleError(code, lib().orc_point_error().decode())


# -------------------------------------------------------------------------------------------
# scene dict (parsed JSON, reference schema scene.cpp:190-294) -> C structs
# -------------------------------------------------------------------------------------------

def _vec3(v, dim):
    out = (C.c_double * 3)()
    if v is not None:
        for a in range(dim):
            out[a] = float(v[a])
    return out


def _shape(d, dim):
    s = Shape()
    s.kind = SHAPES[d["kind"]]
    s.min = _vec3(d.get("min"), dim)
    s.max = _vec3(d.get("max"), dim)
    s.center = _vec3(d.get("center"), dim)
    s.radius = float(d.get("radius", 0.0))
    s.point = _vec3(d.get("point"), dim)
    s.normal = _vec3(d.get("normal"), dim)
    s.axis = _vec3(d.get("axis"), 3 if dim == 3 else 0)
    return s


ELASTICITY = {"fixed_corotated": 0, "neo_hookean": 1}


def material_struct(m):
    pl = m.get("plasticity", {"kind": "none"})
    return Material(float(m["density"]), float(m["youngs"]), float(m["poisson"]), PLAST[pl["kind"]],
                    float(pl.get("yield_stress", 0.0)), float(pl.get("lo", 0.99)), float(pl.get("hi", 1.001)),
                    ELASTICITY[m.get("elasticity", "fixed_corotated")], float(pl.get("hardening", 0.0)),
                    float(pl.get("friction_angle", 0.0)))


def scene_struct(sc):
    """Builds the orc_scene struct; returns (struct, keepalive)."""
    dim = int(sc.get("dim", 2))
    mats = (Material * len(sc["materials"]))(*[material_struct(m) for m in sc["materials"]])
    objs = []
    for o in sc["objects"]:
        ob = Object()
        ob.shape = _shape(o["shape"], dim)
        ob.material = int(o["material"])
        ob.velocity = _vec3(o.get("velocity"), dim)
        idf = o.get("initial_deformation", {"kind": "identity"})
        ob.init_kind = 1 if idf["kind"] == "random_diagonal" else 0
        ob.init_lo = float(idf.get("lo", 1.0))
        ob.init_hi = float(idf.get("hi", 1.0))
        objs.append(ob)
    objs = (Object * len(objs))(*objs)
    cols = []
    for c in sc.get("colliders", []):
        co = Collider()
        co.shape = _shape(c["shape"], dim)
        m = c.get("motion", {"kind": "static"})
        mo = Motion()
        mo.kind = MOTIONS[m["kind"]]
        mo.velocity = _vec3(m.get("velocity"), dim)
        mo.center = _vec3(m.get("center"), dim)
        mo.axis = _vec3(m.get("axis"), 3 if dim == 3 else 0)
        mo.omega = float(m.get("omega", 0.0))
        co.motion = mo
        cols.append(co)
    cols = (Collider * max(1, len(cols)))(*cols)
    s = Scene()
    s.dim = dim
    s.dx = float(sc["dx"])
    s.gravity = _vec3(sc.get("gravity"), dim)
    s.fps = float(sc.get("fps", 24))
    s.frames = int(sc.get("frames", 24))
    s.epsilon = float(sc.get("epsilon", 1e-7))
    s.tau = float(sc.get("tau", 1e-4))
    s.levels = int(sc.get("levels", 3))
    s.window = int(sc.get("window", 8))
    s.solver = SOLVERS[sc.get("solver", "hot")]
    s.embedding = LINEAR if sc.get("embedding", "linear") == "linear" else QUADRATIC
    s.cn_length_factor = float(sc.get("cn_length_factor", 24))
    s.seed = int(sc.get("seed", 0))
    s.ppc = int(sc.get("ppc", 0))
    s.poisson_sampling = 1 if sc.get("sampling", "jittered") == "poisson" else 0
    s.n_materials = len(sc["materials"])
    s.n_objects = len(sc["objects"])
    s.n_colliders = len(sc.get("colliders", []))
    s.materials = C.cast(mats, C.POINTER(Material))
    s.objects = C.cast(objs, C.POINTER(Object))
    s.colliders = C.cast(cols, C.POINTER(Collider))
    return s, (mats, objs, cols)


def solver_struct(epsilon=1e-7, tau=1e-4, levels=3, window=8, ls_shrink=0.5, ls_armijo=1e-4, ls_max_steps=30,
                  cg_cap=10000, outer_cap=1000, kind="hot", embedding="linear", pinned_coarse_iterations=256,
                  cn_length_factor=24.0):
    return Solver(epsilon, tau, levels, window, ls_shrink, ls_armijo, ls_max_steps, cg_cap, outer_cap,
                  SOLVERS[kind] if isinstance(kind, str) else kind,
                  (LINEAR if embedding == "linear" else QUADRATIC) if isinstance(embedding, str) else embedding,
                  pinned_coarse_iterations, cn_length_factor)


# -------------------------------------------------------------------------------------------
# point functions
# -------------------------------------------------------------------------------------------

def set_threads(n):
    lib().orc_set_threads(int(n))


def kernel_weight_1d(kind, x):
    return lib().orc_kernel_weight_1d(kind, x)


def kernel_derivative_1d(kind, x):
    return lib().orc_kernel_derivative_1d(kind, x)


def kernel_weight(kind, off):
    off = _f64(off)
    return lib().orc_kernel_weight(off.size, kind, _dp(off))


def kernel_gradient(kind, off, dx):
    off = _f64(off)
    out = np.zeros(off.size)
    lib().orc_kernel_gradient(off.size, kind, _dp(off), dx, _dp(out))
    return out


def stencil_base(x, dx, kind=QUADRATIC):
    x = _f64(x)
    out = np.zeros(x.size, dtype=np.int32)
    lib().orc_stencil_base(x.size, _dp(x), dx, kind, _ip(out))
    return out


def cfl_dt(v_max, dx, fps):
    return lib().orc_cfl_dt(v_max, dx, fps)


def adaptive_cg_tolerance(pe_sq, tau):
    return lib().orc_adaptive_cg_tolerance(pe_sq, tau)


def material_lame(m):
    mu, la = C.c_double(), C.c_double()
    _check_point(lib().orc_material_lame(C.byref(material_struct(m)), C.byref(mu), C.byref(la)))
    return mu.value, la.value


def svd_rv(F):
    F = _f64(F)
    d = F.shape[0]
    U, V, s = np.zeros((d, d)), np.zeros((d, d)), np.zeros(d)
    _check_point(lib().orc_svd(d, _dp(F), _dp(U), _dp(s), _dp(V)))
    return U, s, V


def fcr_energy_density(F, m):
    F = _f64(F)
    out = C.c_double()
    _check_point(lib().orc_fcr_energy(F.shape[0], _dp(F), C.byref(material_struct(m)), C.byref(out)))
    return out.value


def fcr_stress(F, m):
    F = _f64(F)
    out = np.zeros_like(F)
    _check_point(lib().orc_fcr_stress(F.shape[0], _dp(F), C.byref(material_struct(m)), _dp(out)))
    return out


def fcr_stress_derivative(F, m, project=False):
    F = _f64(F)
    d = F.shape[0]
    out = np.zeros((d * d, d * d))
    _check_point(lib().orc_fcr_dpdf(d, _dp(F), C.byref(material_struct(m)), int(project), _dp(out)))
    return out


def project_spd(A):
    A = _f64(A)
    out = np.zeros_like(A)
    _check_point(lib().orc_project_spd(A.shape[0], _dp(A), _dp(out)))
    return out


def return_map(F, m):
    F = _f64(F)
    out = np.zeros_like(F)
    _check_point(lib().orc_return_map(F.shape[0], _dp(F), C.byref(material_struct(m)), _dp(out)))
    return out


def energy_density(F, m, h=1.0):
    """The material's own elastic model (fixed-corotated or the Neo-Hookean extension), Lame
    parameters scaled by the hardening factor h."""
    F = _f64(F)
    out = C.c_double()
    _check_point(lib().orc_model_energy(F.shape[0], _dp(F), C.byref(material_struct(m)), h, C.byref(out)))
    return out.value


def stress(F, m, h=1.0):
    F = _f64(F)
    out = np.zeros_like(F)
    _check_point(lib().orc_model_stress(F.shape[0], _dp(F), C.byref(material_struct(m)), h, _dp(out)))
    return out


def stress_derivative(F, m, h=1.0, project=False):
    F = _f64(F)
    d = F.shape[0]
    out = np.zeros((d * d, d * d))
    _check_point(lib().orc_model_dpdf(d, _dp(F), C.byref(material_struct(m)), h, int(project), _dp(out)))
    return out


def return_map_jp(F, m, Jp=1.0):
    """return_map with the plastic volume ratio: returns (F, J_p)."""
    F = _f64(F)
    out = np.zeros_like(F)
    jp = C.c_double(Jp)
    _check_point(lib().orc_return_map_jp(F.shape[0], _dp(F), C.byref(material_struct(m)), C.byref(jp), _dp(out)))
    return out, jp.value


def hardening_factor(m, Jp):
    return lib().orc_hardening_factor(C.byref(material_struct(m)), Jp)


def stiffness_scale(m, dim):
    out = C.c_double()
    _check_point(lib().orc_stiffness_scale(dim, C.byref(material_struct(m)), C.byref(out)))
    return out.value


def pcg(apply_a, apply_p, b, rel_tol, cap):
    b = _f64(b)
    n = b.size

    def wrap(f):
        def cb(inp, out, _u):
            x = np.ctypeslib.as_array(inp, shape=(n,)).copy()
            np.ctypeslib.as_array(out, shape=(n,))[:] = f(x)
        return APPLY_FN(cb)

    A, P = wrap(apply_a), wrap(apply_p)
    x = np.zeros(n)
    it, conv = C.c_int(), C.c_int()
    _check_point(lib().orc_pcg(n, A, P, None, _dp(b), rel_tol, cap, _dp(x), C.byref(it), C.byref(conv)))
    return x, it.value, bool(conv.value)


def line_search(energy_at, e0, gdotp, cfg=None):
    cb = ENERGY_FN(lambda a, _u: float(energy_at(a)))
    alpha, en, ev = C.c_double(), C.c_double(), C.c_int()
    code = lib().orc_line_search(cb, None, e0, gdotp, C.byref(cfg) if cfg is not None else None,
                                 C.byref(alpha), C.byref(en), C.byref(ev))
    _check_point(code)
    return alpha.value, en.value, ev.value


class LBFGSHistory:
    def __init__(self, window):
        self.h = lib().orc_lbfgs_new(window)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_lbfgs_free(self.h)

    def push(self, s, y):
        s, y = _f64(s), _f64(y)
        return bool(lib().orc_lbfgs_push(self.h, s.size, _dp(s), _dp(y)))

    def size(self):
        return lib().orc_lbfgs_size(self.h)

    def direction(self, g, init):
        g = _f64(g)
        n = g.size

        def cb(inp, out, _u):
            q = np.ctypeslib.as_array(inp, shape=(n,)).copy()
            np.ctypeslib.as_array(out, shape=(n,))[:] = init(q)

        fn = APPLY_FN(cb)
        p = np.zeros(n)
        _check_point(lib().orc_lbfgs_direction(self.h, n, _dp(g), fn, None, _dp(p)))
        return p


# -------------------------------------------------------------------------------------------
# stateful simulation context
# -------------------------------------------------------------------------------------------

class Oracle:
    """One oracle simulation (SimulationState + stage objects), dim 2 or 3."""

    def __init__(self, dim=3):
        self.dim = dim
        self.ctx = lib().orc_new(dim)
        self._keep = None

    def __del__(self):
        if getattr(self, "ctx", None):
            lib().orc_free(self.ctx)
            self.ctx = None

    def _check(self, code):
        if code:
            raise OracleError(code, lib().orc_error(self.ctx).decode())

    # -- setup ------------------------------------------------------------------------------
    def set_scene(self, scene_dict):
        s, keep = scene_struct(scene_dict)
        self._keep = keep
        self._check(lib().orc_set_scene(self.ctx, C.byref(s)))
        self.dim = s.dim

    def set_solver(self, **kw):
        self._check(lib().orc_set_solver(self.ctx, C.byref(solver_struct(**kw))))

    def set_materials(self, mats):
        arr = (Material * len(mats))(*[material_struct(m) for m in mats])
        self._check(lib().orc_set_materials(self.ctx, len(mats), arr))

    def set_env(self, gravity, dx, cn_length_factor=24.0):
        g = _f64(list(gravity) + [0.0] * (3 - len(gravity)))
        self._check(lib().orc_set_gravity_dx(self.ctx, _dp(g), dx, cn_length_factor))

    def sample_scene(self):
        self._check(lib().orc_sample_scene(self.ctx))
        return self.particle_count()

    def particle_count(self):
        return lib().orc_particle_count(self.ctx)

    def set_particles(self, x, v=None, mass=None, volume=None, F=None, Cm=None, material=None):
        d = self.dim
        x = _f64(x).reshape(-1, d)
        n = x.shape[0]
        v = None if v is None else _f64(v, n * d)
        mass = None if mass is None else _f64(mass, n)
        volume = None if volume is None else _f64(volume, n)
        F = None if F is None else _f64(F, n * d * d)
        Cm = None if Cm is None else _f64(Cm, n * d * d)
        material = None if material is None else np.ascontiguousarray(material, dtype=np.int32)
        self._check(lib().orc_set_particles(self.ctx, n, _dp(x), _dp(v), _dp(mass), _dp(volume), _dp(F), _dp(Cm),
                                            _ip(material)))

    def get_particles(self):
        n, d = self.particle_count(), self.dim
        out = dict(x=np.zeros((n, d)), v=np.zeros((n, d)), mass=np.zeros(n), volume=np.zeros(n),
                   F=np.zeros((n, d, d)), C=np.zeros((n, d, d)), material=np.zeros(n, dtype=np.int32))
        self._check(lib().orc_get_particles(self.ctx, _dp(out["x"]), _dp(out["v"]), _dp(out["mass"]),
                                            _dp(out["volume"]), _dp(out["F"]), _dp(out["C"]), _ip(out["material"])))
        return out

    def particle_jp(self):
        out = np.zeros(self.particle_count())
        self._check(lib().orc_particle_jp(self.ctx, _dp(out), None))
        return out

    def set_particle_jp(self, jp):
        jp = _f64(jp, self.particle_count())
        self._check(lib().orc_particle_jp(self.ctx, None, _dp(jp)))

    def sim_state(self):
        t, s, inv, fr = C.c_double(), C.c_longlong(), C.c_longlong(), C.c_int()
        lib().orc_sim_state(self.ctx, C.byref(t), C.byref(s), C.byref(inv), C.byref(fr))
        return dict(time=t.value, step=s.value, inversions=inv.value, frame=fr.value)

    def set_sim_state(self, time=0.0, step=0, frame=0):
        lib().orc_set_sim_state(self.ctx, time, step, frame)

    def advance_step(self, frame_end):
        dt, outer, inner, nodes, conv = C.c_double(), C.c_int(), C.c_longlong(), C.c_int(), C.c_int()
        self._check(lib().orc_advance_step(self.ctx, frame_end, C.byref(dt), C.byref(outer), C.byref(inner),
                                           C.byref(nodes), C.byref(conv)))
        return dict(dt=dt.value, outer_iterations=outer.value, inner_total=inner.value, node_count=nodes.value,
                    converged=bool(conv.value))

    def diagnostics(self):
        n = lib().orc_diag_count(self.ctx)
        f, st, o = np.zeros(n, np.int32), np.zeros(n, np.int64), np.zeros(n, np.int32)
        r, e, a = np.zeros(n), np.zeros(n), np.zeros(n)
        inn, w, wall = np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(n)
        lib().orc_diag_get(self.ctx, _ip(f), st.ctypes.data_as(C.POINTER(C.c_longlong)), _ip(o), _dp(r), _dp(e),
                           _dp(a), inn.ctypes.data_as(C.POINTER(C.c_longlong)),
                           w.ctypes.data_as(C.POINTER(C.c_longlong)), _dp(wall))
        return dict(frame=f, step=st, outer_iteration=o, scaled_residual=r, energy=e, step_length=a,
                    inner_iterations=inn, work_units=w, wall_ms=wall)

    def clear_diagnostics(self):
        lib().orc_diag_clear(self.ctx)

    # -- stage API --------------------------------------------------------------------------
    def activate(self, kind=QUADRATIC):
        self._check(lib().orc_activate(self.ctx, kind))
        return lib().orc_grid_nodes(self.ctx)

    def node_count(self):
        return lib().orc_grid_nodes(self.ctx)

    def grid(self):
        n, d = self.node_count(), self.dim
        out = dict(coords=np.zeros((n, d), np.int32), mass=np.zeros(n), velocity=np.zeros(n * d),
                   momentum=np.zeros(n * d), dirichlet=np.zeros(n, np.uint8), bc_velocity=np.zeros(n * d))
        self._check(lib().orc_grid_get(self.ctx, _ip(out["coords"]), _dp(out["mass"]), _dp(out["velocity"]),
                                       _dp(out["momentum"]),
                                       out["dirichlet"].ctypes.data_as(C.POINTER(C.c_ubyte)),
                                       _dp(out["bc_velocity"])))
        return out

    def set_grid(self, velocity=None, dirichlet=None, bc_velocity=None):
        n, d = self.node_count(), self.dim
        velocity = None if velocity is None else _f64(velocity, n * d)
        bc_velocity = None if bc_velocity is None else _f64(bc_velocity, n * d)
        dp = None
        if dirichlet is not None:
            dirichlet = np.ascontiguousarray(dirichlet, dtype=np.uint8)
            dp = dirichlet.ctypes.data_as(C.POINTER(C.c_ubyte))
        self._check(lib().orc_grid_set(self.ctx, _dp(velocity), dp, _dp(bc_velocity)))

    def p2g(self):
        self._check(lib().orc_p2g(self.ctx))

    def apply_bc(self, time=0.0):
        self._check(lib().orc_apply_bc(self.ctx, time))

    def make_state(self, dt):
        self._check(lib().orc_make_state(self.ctx, dt))

    def energy(self, dv):
        out = C.c_double()
        dv = _f64(dv)
        self._check(lib().orc_energy(self.ctx, _dp(dv), C.byref(out)))
        return out.value

    def gradient(self, dv):
        dv = _f64(dv)
        g = np.zeros_like(dv)
        self._check(lib().orc_gradient(self.ctx, _dp(dv), _dp(g)))
        return g

    def node_cn(self):
        n = self.node_count()
        xi, sc = np.zeros(n), np.zeros(n)
        self._check(lib().orc_node_cn(self.ctx, _dp(xi), _dp(sc)))
        return xi, sc

    def scaled_norm(self, g):
        out = C.c_double()
        g = _f64(g)
        self._check(lib().orc_scaled_norm(self.ctx, _dp(g), C.byref(out)))
        return out.value

    def assemble(self, dv=None, project=True):
        if dv is None:
            dv = np.zeros(self.node_count() * self.dim)
        dv = _f64(dv)
        self._check(lib().orc_assemble(self.ctx, _dp(dv), int(project)))

    def build_hierarchy(self, levels=3, embedding=LINEAR):
        self._check(lib().orc_build_hierarchy(self.ctx, levels, embedding))
        return lib().orc_level_count(self.ctx)

    def level_count(self):
        return lib().orc_level_count(self.ctx)

    def level_shape(self, level):
        r, s, rad = C.c_int(), C.c_int(), C.c_int()
        self._check(lib().orc_level_shape(self.ctx, level, C.byref(r), C.byref(s), C.byref(rad)))
        return r.value, s.value, rad.value

    def level_matrix(self, level=0):
        rows, slots, _ = self.level_shape(level)
        d = self.dim
        blocks = np.zeros((rows, slots, d, d))
        cols = np.zeros((rows, slots), np.int32)
        self._check(lib().orc_level_matrix(self.ctx, level, _dp(blocks), _ip(cols)))
        return blocks, cols

    def set_level_matrix(self, level, blocks):
        blocks = _f64(blocks)
        self._check(lib().orc_set_level_matrix(self.ctx, level, _dp(blocks)))

    def level_info(self, level):
        rows, _, _ = self.level_shape(level)
        d = self.dim
        out = dict(coords=np.zeros((rows, d), np.int32), dirichlet=np.zeros(rows, np.uint8),
                   sweep_order=np.zeros(rows, np.int32), diag_inv=np.zeros((rows, d, d)))
        self._check(lib().orc_level_info(self.ctx, level, _ip(out["coords"]),
                                         out["dirichlet"].ctypes.data_as(C.POINTER(C.c_ubyte)),
                                         _ip(out["sweep_order"]), _dp(out["diag_inv"])))
        return out

    def refinalize_level(self, level, modulus):
        self._check(lib().orc_refinalize_level(self.ctx, level, modulus))

    def level_restriction(self, level):
        nnz = C.c_int()
        self._check(lib().orc_level_restriction(self.ctx, level, None, None, None, C.byref(nnz)))
        rows, _, _ = self.level_shape(level)
        rs = np.zeros(rows + 1, np.int32)
        co = np.zeros(nnz.value, np.int32)
        w = np.zeros(nnz.value)
        self._check(lib().orc_level_restriction(self.ctx, level, _ip(rs), _ip(co), _dp(w), C.byref(nnz)))
        return rs, co, w

    def matvec(self, x, level=0):
        x = _f64(x)
        y = np.zeros_like(x)
        self._check(lib().orc_matvec(self.ctx, level, _dp(x), _dp(y)))
        return y

    def smooth_sgs(self, level, u, b, sweeps=1):
        u = _f64(u).copy()
        b = _f64(b)
        self._check(lib().orc_smooth_sgs(self.ctx, level, _dp(u), _dp(b), sweeps))
        return u

    def coarse_solve(self, level, b, pinned=False, pinned_cap=256, cap=10000):
        b = _f64(b)
        u = np.zeros_like(b)
        it = C.c_int()
        self._check(lib().orc_coarse_solve(self.ctx, level, _dp(b), _dp(u), C.byref(it), int(pinned), pinned_cap,
                                           cap))
        return u, it.value

    def vcycle(self, b, pinned=False, pinned_cap=256):
        b = _f64(b)
        u = np.zeros_like(b)
        it = C.c_int()
        self._check(lib().orc_vcycle(self.ctx, _dp(b), _dp(u), C.byref(it), int(pinned), pinned_cap))
        return u, it.value

    def step_grid(self, frame=0, step=0):
        n = self.node_count() * self.dim
        vel, dv = np.zeros(n), np.zeros(n)
        outer, inner, conv, reb = C.c_int(), C.c_longlong(), C.c_int(), C.c_int()
        self._check(lib().orc_step_grid(self.ctx, _dp(vel), _dp(dv), C.byref(outer), C.byref(inner), C.byref(conv),
                                        C.byref(reb), frame, step))
        return dict(velocity=vel, dv=dv, outer_iterations=outer.value, inner_total=inner.value,
                    converged=bool(conv.value), hierarchy_rebuilds=reb.value)

    def g2p(self):
        self._check(lib().orc_g2p(self.ctx))

    def update_strain(self, dt):
        inv = C.c_longlong()
        self._check(lib().orc_update_strain(self.ctx, dt, C.byref(inv)))
        return inv.value

    def advect(self, dt):
        self._check(lib().orc_advect(self.ctx, dt))
