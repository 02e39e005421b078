"""GPU parity for the constitutive extensions (the reference has fixed-corotated
only): Neo-Hookean elasticity, Stomakhin snow hardening (plastic volume ratio J_p) and the
Drucker-Prager return map.  The CUDA path (through the C-ABI) against the oracle's restatement
(oracle/hot_oracle.hpp nh_*, return_map, hardening_factor), which tests/test_oracle_extensions.py
pins by finite differences and the maps' defining properties."""
import numpy as np
import pytest

from tests.gpu_common import Pair, block_scene_dict, random_block_particles, rel_err, scene_from_dict
from tests.test_gpu_baseline_parity import elem_rel_err

pytestmark = pytest.mark.gpu

NH = {"density": 1000.0, "youngs": 2e5, "poisson": 0.3, "elasticity": "neo_hookean"}
SNOW_H = {"density": 400.0, "youngs": 1.4e5, "poisson": 0.2,
          "plasticity": {"kind": "snow_clamp", "lo": 0.975, "hi": 1.0075, "hardening": 10.0}}
SAND = {"density": 2200.0, "youngs": 3.5e5, "poisson": 0.3,
        "plasticity": {"kind": "drucker_prager", "friction_angle": 30.0}}
FLOOR = [{"shape": {"kind": "half_space", "point": [0.0, 0.021, 0.0], "normal": [0.0, 1.0, 0.0]},
          "motion": {"kind": "static"}}]


def _pair(material, seed, fps=48, f_spread=0.2, v_spread=0.3, cells=6, floor=True):
    d = block_scene_dict(colliders=FLOOR if floor else (), extra={"fps": fps})
    d["materials"] = [material]
    sc = scene_from_dict(d)
    p = random_block_particles(np.random.default_rng(seed), 0.02, cells, f_spread=f_spread, v_spread=v_spread)
    p["mass"] = p["mass"] * material["density"] / 1000.0
    return Pair(sc, p)


def _stage_parity(pr, dt, tol=1e-10):
    n = pr.prepare(dt)
    rng = np.random.default_rng(9)
    for dv in (np.zeros(3 * n), rng.uniform(-0.05, 0.05, 3 * n)):
        dv.reshape(-1, 3)[pr.orc.grid()["dirichlet"] == 1] = 0
        assert pr.gpu.energy(dv) == pytest.approx(pr.orc.energy(dv), rel=tol)
        g, _ = pr.gpu.gradient(dv)
        assert rel_err(g, pr.orc.gradient(dv)) < tol
        for project in (True, False):
            pr.gpu.assemble(dv, project=project)
            pr.orc.assemble(dv, project=project)
            G = pr.gpu.level_matrix(0)
            bo, co = pr.orc.level_matrix(0)
            assert np.array_equal(G["cols"], co)
            assert rel_err(G["blocks"], bo) < tol, project


def _steps(pr, steps, jp=False):
    sc = pr.sc
    for k in range(steps):
        frame_end = (k + 1) / sc.fps
        s = pr.gpu.advance_step(frame_end)
        so = pr.orc.advance_step(frame_end)
        assert s["node_count"] == so["node_count"]
        assert abs(s["outer_iterations"] - so["outer_iterations"]) <= 1, (k, s, so)
        gp, op = pr.gpu.particles(), pr.orc.get_particles()
        for key in ("x", "v", "F"):
            assert elem_rel_err(gp[key], op[key]) < 1e-6, (k, key)
        if jp:
            assert elem_rel_err(pr.gpu.plastic_state(), pr.orc.particle_jp()) < 1e-6, k
    return pr


def test_neo_hookean_stages():
    """energy, gradient, projected and unprojected Hessian of a strongly deformed NH block."""
    _stage_parity(_pair(NH, 41, f_spread=0.35), 1.0 / 48)


def test_neo_hookean_steps():
    pr = _steps(_pair(NH, 42), 3)
    assert np.abs(np.linalg.det(pr.gpu.particles()["F"]) - 1.0).max() > 1e-3  # it deformed


def test_snow_hardening_stages_with_plastic_state():
    """Per-particle Lame parameters scaled by exp(xi (1 - J_p)) in the energy, gradient and
    Hessian: J_p set to random values on both sides."""
    pr = _pair(SNOW_H, 43, f_spread=0.01)
    jp = np.random.default_rng(3).uniform(0.9, 1.1, pr.p["x"].shape[0])
    pr.gpu.set_plastic_state(jp)
    pr.orc.set_particle_jp(jp)
    assert np.array_equal(pr.gpu.plastic_state(), jp)
    _stage_parity(pr, 1.0 / 48)


def test_snow_hardening_steps_track_plastic_volume():
    """A compressed snow block falling on the floor: the clamp moves J_p, which then stiffens the
    model; x, v, F and J_p per element over 4 steps."""
    pr = _pair(SNOW_H, 44, fps=240, f_spread=0.01, v_spread=1.0)
    pr = _steps(pr, 4, jp=True)
    jp = pr.gpu.plastic_state()
    assert np.abs(jp - 1.0).max() > 1e-4


def test_drucker_prager_steps():
    """A sand block with random velocities on the floor: the Drucker-Prager map acts every step
    (every F stays inside its cone), x, v, F per element."""
    pr = _pair(SAND, 45, fps=240, f_spread=0.02, v_spread=1.0)
    pr = _steps(pr, 4)
    F = pr.gpu.particles()["F"]
    s = np.linalg.svd(F, compute_uv=False)
    assert np.all(s > 0)


def test_plastic_state_api():
    pr = _pair(NH, 46, cells=2)
    assert np.all(pr.gpu.plastic_state() == 1.0)  # no snow material: J_p is not stored
    from paper_1911_07913_b200 import InvalidArgument
    with pytest.raises(InvalidArgument):
        pr.gpu.set_plastic_state(np.ones(pr.p["x"].shape[0]))
