"""Python mirror of the reference host surface for the hot path.

``Simulation`` owns one device context (hot_create) and exposes the reference's calls with
the same names and meaning:

=============================  ======================================================
reference (hotmpm::)           here
=============================  ======================================================
sample_scene_particles         ``sample_scene_particles(scene)`` / ``Simulation.sample()``
advance_step (simulation.hpp)  ``Simulation.advance_step(frame_end)``
step_grid (solvers.hpp)        ``Simulation.step_grid()`` after ``stage_prepare(dt)``
energy / gradient              ``Simulation.energy(dv)`` / ``Simulation.gradient(dv)``
assemble_hessian               ``Simulation.assemble(dv, project)``
build_hierarchy / vcycle       ``Simulation.build_hierarchy(levels)`` / ``vcycle(b)``
=============================  ======================================================

Errors raise the reference's exception kinds (capi.SolverFailure, InvalidArgument, ...).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .capi import dptr, iptr, u8ptr
from .scene import SceneConfig


class Simulation:
    def __init__(self, scene: SceneConfig, device: int = 0):
        self.scene = scene
        self.dim = scene.dim
        self._lib = capi.lib()
        self._scene_c, self._keep = capi.scene_to_c(scene)
        h = C.c_void_p()
        code = self._lib.hot_create(C.byref(h), C.byref(self._scene_c), device)
        if code != capi.HOT_OK:
            capi.raise_for(code, self._lib.hot_last_error(None).decode())
        self._h = h

    # ---------------------------------------------------------------- lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._lib.hot_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, code):
        if code != capi.HOT_OK:
            capi.raise_for(code, self._lib.hot_last_error(self._h).decode())

    @property
    def handle(self):
        return self._h

    # ---------------------------------------------------------------- configuration
    def set_solver(self, epsilon=None, tau=None, levels=None, window=None, kind=None, ls_shrink=0.5, ls_armijo=1e-4,
                   ls_max_steps=30, cg_cap=10000, outer_cap=1000, pinned_coarse_iterations=256,
                   cn_length_factor=None, embedding=None):
        sc = self.scene
        cfg = capi.hot_solver_config(
            sc.epsilon if epsilon is None else epsilon, sc.tau if tau is None else tau,
            sc.levels if levels is None else levels, sc.window if window is None else window, ls_shrink, ls_armijo,
            ls_max_steps, cg_cap, outer_cap, capi.SOLVER_KINDS[sc.solver if kind is None else kind],
            1 if (sc.embedding if embedding is None else embedding) == "linear" else 0, pinned_coarse_iterations,
            sc.cn_length_factor if cn_length_factor is None else cn_length_factor)
        self._check(self._lib.hot_set_solver(self._h, C.byref(cfg)))

    # ---------------------------------------------------------------- particles
    def sample(self):
        p = capi.sample_scene_particles(self.scene)
        self.set_particles(**p)
        return p

    def set_particles(self, x, v=None, mass=None, volume=None, F=None, C=None, material=None):
        d = self.dim
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, d)
        n = x.shape[0]

        def f64(a, k):
            return None if a is None else np.ascontiguousarray(a, dtype=np.float64).reshape(n * k)

        v, mass, volume, F, Cm = f64(v, d), f64(mass, 1), f64(volume, 1), f64(F, d * d), f64(C, d * d)
        mat = None if material is None else np.ascontiguousarray(material, dtype=np.int32)
        self._check(self._lib.hot_upload_particles(self._h, n, dptr(x), dptr(v), dptr(mass), dptr(volume), dptr(F),
                                                   dptr(Cm), iptr(mat)))

    def particle_count(self):
        n = C.c_longlong()
        self._lib.hot_particle_count(self._h, C.byref(n))
        return n.value

    def particles(self, out=None):
        """Downloads x, v, F, C (into ``out``'s arrays when given, e.g. pinned host buffers)."""
        n, d = self.particle_count(), self.dim
        if out is None:
            out = dict(x=np.zeros((n, d)), v=np.zeros((n, d)), F=np.zeros((n, d, d)), C=np.zeros((n, d, d)))
        self._check(self._lib.hot_download_particles(self._h, dptr(out["x"]), dptr(out["v"]), dptr(out["F"]),
                                                     dptr(out["C"])))
        return out

    def plastic_state(self):
        """J_p per particle (snow hardening extension; 1 when no material is snow)."""
        out = np.zeros(self.particle_count())
        self._check(self._lib.hot_get_plastic_state(self._h, dptr(out)))
        return out

    def set_plastic_state(self, jp):
        jp = np.ascontiguousarray(jp, dtype=np.float64)
        if jp.shape != (self.particle_count(),):
            raise ValueError("one J_p per particle")
        self._check(self._lib.hot_set_plastic_state(self._h, dptr(jp)))

    def set_time(self, time=0.0, frame=0, step_index=0):
        self._lib.hot_set_time(self._h, time, frame, step_index)

    def time_state(self):
        t, f, s, inv = C.c_double(), C.c_int(), C.c_longlong(), C.c_longlong()
        self._lib.hot_get_time(self._h, C.byref(t), C.byref(f), C.byref(s), C.byref(inv))
        return dict(time=t.value, frame=f.value, step=s.value, inversions=inv.value)

    # ---------------------------------------------------------------- the hot path
    def advance_step(self, frame_end: float):
        """simulation.hpp:286-323."""
        st = capi.hot_step_stats()
        self._check(self._lib.hot_advance_step(self._h, frame_end, C.byref(st)))
        return dict(dt=st.dt, outer_iterations=st.outer_iterations, inner_total=st.inner_total,
                    node_count=st.node_count, converged=bool(st.converged))

    def diagnostics(self):
        n = C.c_int()
        self._lib.hot_diagnostics(self._h, None, 0, C.byref(n))
        rows = (capi.hot_diag_row * max(1, n.value))()
        self._lib.hot_diagnostics(self._h, rows, n.value, C.byref(n))
        keys = ["frame", "step", "outer_iteration", "scaled_residual", "energy", "step_length", "inner_iterations",
                "work_units", "wall_ms"]
        return {k: np.array([getattr(rows[i], k) for i in range(n.value)]) for k in keys}

    def clear_diagnostics(self):
        self._lib.hot_clear_diagnostics(self._h)

    # ---------------------------------------------------------------- stage taps
    def stage_prepare(self, dt: float, time: float = 0.0):
        self._check(self._lib.hot_stage_prepare(self._h, dt, time))
        return self.node_count()

    def node_count(self):
        n = C.c_int()
        self._lib.hot_stage_node_count(self._h, C.byref(n))
        return n.value

    def grid(self):
        n, d = self.node_count(), self.dim
        out = dict(coords=np.zeros((n, d), np.int32), mass=np.zeros(n), velocity=np.zeros(n * d),
                   momentum=np.zeros(n * d), dirichlet=np.zeros(n, np.uint8), bc_velocity=np.zeros(n * d),
                   cn_scale=np.zeros(n))
        self._check(self._lib.hot_stage_grid(self._h, iptr(out["coords"]), dptr(out["mass"]), dptr(out["velocity"]),
                                             dptr(out["momentum"]), u8ptr(out["dirichlet"]), dptr(out["bc_velocity"]),
                                             dptr(out["cn_scale"])))
        return out

    def set_grid(self, velocity=None, dirichlet=None, bc_velocity=None):
        f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        velocity, bc_velocity = f(velocity), f(bc_velocity)
        if dirichlet is not None:
            dirichlet = np.ascontiguousarray(dirichlet, dtype=np.uint8)
        self._check(self._lib.hot_stage_set_grid(self._h, dptr(velocity), u8ptr(dirichlet), dptr(bc_velocity)))

    def energy(self, dv):
        dv = np.ascontiguousarray(dv, dtype=np.float64)
        e = C.c_double()
        self._check(self._lib.hot_stage_energy(self._h, dptr(dv), C.byref(e)))
        return e.value

    def gradient(self, dv):
        dv = np.ascontiguousarray(dv, dtype=np.float64)
        g = np.zeros_like(dv)
        nrm = C.c_double()
        self._check(self._lib.hot_stage_gradient(self._h, dptr(dv), dptr(g), C.byref(nrm)))
        return g, nrm.value

    def assemble(self, dv=None, project=True):
        if dv is None:
            dv = np.zeros(self.node_count() * self.dim)
        dv = np.ascontiguousarray(dv, dtype=np.float64)
        self._check(self._lib.hot_stage_assemble(self._h, dptr(dv), int(project)))

    def build_hierarchy(self, levels=3, embedding="linear"):
        self._check(self._lib.hot_stage_build_hierarchy(self._h, levels, 1 if embedding == "linear" else 0))
        n = C.c_int()
        self._lib.hot_stage_level_count(self._h, C.byref(n))
        return n.value

    def level_shape(self, level):
        r, s = C.c_int(), C.c_int()
        self._check(self._lib.hot_stage_level_shape(self._h, level, C.byref(r), C.byref(s)))
        return r.value, s.value

    def level_coords(self, level=0):
        """coords and Dirichlet flags of a level (no matrix copy)."""
        rows, _ = self.level_shape(level)
        coords = np.zeros((rows, self.dim), np.int32)
        dirm = np.zeros(rows, np.uint8)
        self._check(self._lib.hot_stage_level_matrix(self._h, level, None, None, iptr(coords), u8ptr(dirm)))
        return dict(coords=coords, dirichlet=dirm)

    def level_matrix(self, level=0):
        rows, slots = self.level_shape(level)
        d = self.dim
        blocks = np.zeros((rows, slots, d, d))
        cols = np.zeros((rows, slots), np.int32)
        coords = np.zeros((rows, d), np.int32)
        dirm = np.zeros(rows, np.uint8)
        self._check(self._lib.hot_stage_level_matrix(self._h, level, dptr(blocks), iptr(cols), iptr(coords),
                                                     u8ptr(dirm)))
        return dict(blocks=blocks, cols=cols, coords=coords, dirichlet=dirm)

    def matvec(self, x, level=0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        self._check(self._lib.hot_stage_matvec(self._h, level, dptr(x), dptr(y)))
        return y

    def vcycle(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        u = np.zeros_like(b)
        it = C.c_int()
        self._check(self._lib.hot_stage_vcycle(self._h, dptr(b), dptr(u), C.byref(it)))
        return u, it.value

    def step_grid(self, frame=0, step=0):
        n = self.node_count() * self.dim
        vel, dv = np.zeros(n), np.zeros(n)
        outer, inner, conv = C.c_int(), C.c_longlong(), C.c_int()
        self._check(self._lib.hot_stage_step_grid(self._h, dptr(vel), dptr(dv), C.byref(outer), C.byref(inner),
                                                  C.byref(conv), frame, step))
        return dict(velocity=vel, dv=dv, outer_iterations=outer.value, inner_total=inner.value,
                    converged=bool(conv.value))

    # ---------------------------------------------------------------- measurement
    def stream(self):
        return self._lib.hot_stream(self._h)

    def profile(self, enable=True):
        self._check(self._lib.hot_profile_enable(self._h, int(enable)))

    def profile_read(self):
        cap = 32
        names = C.create_string_buffer(32 * cap)
        ms, bytes_ = (C.c_double * cap)(), (C.c_double * cap)()
        launches = (C.c_longlong * cap)()
        n = C.c_int()
        self._check(self._lib.hot_profile_read(self._h, names, ms, launches, bytes_, cap, C.byref(n)))
        out = {}
        for i in range(n.value):
            name = names.raw[32 * i:32 * (i + 1)].split(b"\0", 1)[0].decode()
            b = bytes_[i]
            out[name] = dict(ms=ms[i], launches=launches[i], bytes=max(b, 0.0), flops=max(-b, 0.0))
        return out

    def kernel_launches(self):
        return self._lib.hot_kernel_launches(self._h)
