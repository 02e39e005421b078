"""Shared setup for the GPU parity tests: the same seeded state fed to the CUDA path (through
the C-ABI) and to the CPU oracle (the checker)."""
import copy
import json
import os

import numpy as np

from oracle import oracle as O
from paper_1911_07913_b200 import Simulation, load_scene_file, parse_scene, sample_scene_particles

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCENES = os.path.join(ROOT, "scenes")


def scene(name):
    return load_scene_file(os.path.join(SCENES, name + ".json"))


def scene_from_dict(d):
    return parse_scene(json.dumps(d))


def block_scene_dict(dx=0.02, youngs=5e4, gravity=(0.0, -9.8, 0.0), colliders=(), extra=None):
    """A minimal 3D scene: one elastic material; particles supplied separately."""
    d = {"dim": 3, "dx": dx, "gravity": list(gravity), "fps": 24, "epsilon": 1e-7,
         "domain": {"min": [-10.0, -10.0, -10.0], "max": [10.0, 10.0, 10.0]},
         "materials": [{"density": 1000.0, "youngs": youngs, "poisson": 0.3}],
         "objects": [{"shape": {"kind": "box", "min": [0.0, 0.0, 0.0], "max": [0.1, 0.1, 0.1]}, "material": 0}],
         "colliders": list(colliders)}
    if extra:
        d.update(extra)
    return d


def random_block_particles(rng, dx, cells, f_spread=0.2, v_spread=0.3, f_center=1.0, origin=(0.0, 0.0, 0.0)):
    """oracles.hpp:117-145 restated (8 ppc, uniform in [0.05,0.95] of each cell)."""
    n = cells ** 3 * 8
    cc = np.array(np.unravel_index(np.repeat(np.arange(cells ** 3), 8), (cells,) * 3)).T
    x = (cc + rng.uniform(0.05, 0.95, (n, 3))) * dx + np.asarray(origin)
    v = rng.uniform(-v_spread, v_spread, (n, 3)) if v_spread > 0 else np.zeros((n, 3))
    F = np.zeros((n, 3, 3))
    diag = rng.uniform(f_center - f_spread, f_center + f_spread, (n, 3)) if f_spread > 0 else np.full((n, 3), f_center)
    for a in range(3):
        F[:, a, a] = diag[:, a]
    vol = dx ** 3 / 8
    return dict(x=x, v=v, F=F, C=np.zeros((n, 3, 3)), mass=np.full(n, 1000.0 * vol), volume=np.full(n, vol),
                material=np.zeros(n, np.int32))


class Pair:
    """GPU Simulation + oracle on the same particles and scene."""

    def __init__(self, sc, particles=None):
        self.sc = sc
        self.gpu = Simulation(sc)
        self.orc = O.Oracle(3)
        self.orc.set_scene(sc.source)
        if particles is None:
            particles = sample_scene_particles(sc)
        self.p = particles
        self.gpu.set_particles(**particles)
        self.orc.set_particles(particles["x"], particles["v"], particles["mass"], particles["volume"],
                               particles["F"].reshape(-1), particles["C"].reshape(-1), particles["material"])

    def prepare(self, dt, time=0.0):
        n = self.gpu.stage_prepare(dt, time)
        self.orc.activate()
        self.orc.p2g()
        self.orc.apply_bc(time)
        self.orc.make_state(dt)
        return n

    def set_solver(self, **kw):
        self.gpu.set_solver(**kw)
        okw = dict(epsilon=self.sc.epsilon, tau=self.sc.tau, levels=self.sc.levels, window=self.sc.window,
                   kind=self.sc.solver, embedding=self.sc.embedding, cn_length_factor=self.sc.cn_length_factor)
        okw.update({k: v for k, v in kw.items() if v is not None})
        self.orc.set_solver(**okw)


def rel_err(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    scale = max(np.abs(b).max() if b.size else 0.0, 1e-300)
    return np.abs(a - b).max() / scale if a.size else 0.0


def elem_rel_err(a, b, floor=1e-8):
    """max_i |a_i - b_i| / max(|b_i|, floor * max|b|): per-element relative error."""
    a, b = np.asarray(a, dtype=float).ravel(), np.asarray(b, dtype=float).ravel()
    if b.size == 0:
        return 0.0
    den = np.maximum(np.abs(b), floor * max(np.abs(b).max(), 1e-300))
    return float((np.abs(a - b) / den).max())
