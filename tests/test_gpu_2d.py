"""2D (dim = 2) device path against the oracle.

The reference's own suite is 2D (test_solvers.cpp, test_multigrid.cpp and test_objective.cpp
instantiate d = 2; cli.cpp:145 runs advance_step<2>).  These tests run the same stages through the
C-ABI on the GPU and compare with the oracle on the same seeded inputs: indexing bit-exact, stages
to 1e-10..1e-12 relative, state after steps to 1e-6 per element with outer iterations +-1."""
import json

import numpy as np
import pytest

from oracle import oracle as O
from paper_1911_07913_b200 import Simulation, parse_scene, sample_scene_particles
from tests.gpu_common import elem_rel_err, rel_err

pytestmark = pytest.mark.gpu

STATE_TOL = 1e-6
STAGE_TOL = 1e-10


def scene2(dx=0.02, youngs=5e4, gravity=(0.0, -9.8), colliders=(), materials=None, objects=None, extra=None):
    d = {"dim": 2, "dx": dx, "gravity": list(gravity), "fps": 24, "epsilon": 1e-7,
         "domain": {"min": [-10.0, -10.0], "max": [10.0, 10.0]},
         "materials": materials or [{"density": 1000.0, "youngs": youngs, "poisson": 0.3}],
         "objects": objects or [{"shape": {"kind": "box", "min": [0.0, 0.0], "max": [0.1, 0.1]}, "material": 0}],
         "colliders": list(colliders)}
    if extra:
        d.update(extra)
    return d


def block2(rng, dx, cells, f_spread=0.3, v_spread=0.3, origin=(0.0, 0.0), inverted=0.0):
    """oracles.hpp random block, 2D: 4 particles per cell, uniform in [0.05, 0.95] of each cell."""
    n = cells ** 2 * 4
    cc = np.array(np.unravel_index(np.repeat(np.arange(cells ** 2), 4), (cells, cells))).T
    x = (cc + rng.uniform(0.05, 0.95, (n, 2))) * dx + np.asarray(origin)
    v = rng.uniform(-v_spread, v_spread, (n, 2))
    F = np.zeros((n, 2, 2))
    diag = rng.uniform(1.0 - f_spread, 1.0 + f_spread, (n, 2))
    F[:, 0, 0], F[:, 1, 1] = diag[:, 0], diag[:, 1]
    F[:, 0, 1] = rng.uniform(-0.1, 0.1, n)
    if inverted:
        flip = rng.random(n) < inverted
        F[flip, 0, :] *= -1.0
    vol = dx ** 2 / 4
    return dict(x=x, v=v, F=F, C=rng.uniform(-0.5, 0.5, (n, 2, 2)), mass=np.full(n, 1000.0 * vol),
                volume=np.full(n, vol), material=np.zeros(n, np.int32))


class Pair2:
    def __init__(self, sd, p=None):
        self.sd = sd
        self.sc = parse_scene(json.dumps(sd))
        self.gpu = Simulation(self.sc)
        self.orc = O.Oracle(2)
        self.orc.set_scene(self.sc.source)
        self.p = p if p is not None else sample_scene_particles(self.sc)
        self.gpu.set_particles(**self.p)
        self.orc.set_particles(self.p["x"], self.p["v"], self.p["mass"], self.p["volume"], self.p["F"].reshape(-1),
                               self.p["C"].reshape(-1), self.p["material"])

    def prepare(self, dt, time=0.0):
        n = self.gpu.stage_prepare(dt, time)
        self.orc.activate()
        self.orc.p2g()
        self.orc.apply_bc(time)
        self.orc.make_state(dt)
        return n

    def set_solver(self, **kw):
        self.gpu.set_solver(**kw)
        sc = self.sc
        okw = dict(epsilon=sc.epsilon, tau=sc.tau, levels=sc.levels, window=sc.window, kind=sc.solver,
                   embedding=sc.embedding, cn_length_factor=sc.cn_length_factor)
        okw.update({k: v for k, v in kw.items() if v is not None})
        self.orc.set_solver(**okw)


FLOOR = {"shape": {"kind": "half_space", "point": [0.0, 0.021], "normal": [0.0, 1.0]}, "motion": {"kind": "static"}}


def _stretched(seed=0, cells=6, **kw):
    rng = np.random.default_rng(seed)
    return Pair2(scene2(colliders=[FLOOR]), block2(rng, 0.02, cells, **kw))


def test_2d_activation_p2g_and_boundary():
    cols = [FLOOR,
            {"shape": {"kind": "sphere", "center": [0.1, 0.12], "radius": 0.03},
             "motion": {"kind": "rotation", "center": [0.1, 0.1], "omega": 2.0}},
            {"shape": {"kind": "box", "min": [-0.05, -0.05], "max": [0.012, 0.2]},
             "motion": {"kind": "linear", "velocity": [0.3, 0.0]}}]
    sd = scene2(colliders=cols, objects=[{"shape": {"kind": "box", "min": [0.0, 0.0], "max": [0.2, 0.14]},
                                          "material": 0, "velocity": [0.5, -0.2]}])
    pr = Pair2(sd)
    n = pr.prepare(0.01)
    g, o = pr.gpu.grid(), pr.orc.grid()
    assert n == o["coords"].shape[0] > 0
    assert np.array_equal(g["coords"], o["coords"])  # bit-exact lexicographic indexing
    assert np.array_equal(g["dirichlet"], o["dirichlet"]) and g["dirichlet"].sum() > 0
    for k in ("mass", "momentum", "velocity", "bc_velocity"):
        assert rel_err(g[k], o[k]) < 1e-12, k
    assert rel_err(g["cn_scale"], pr.orc.node_cn()[1]) < 1e-12


@pytest.mark.parametrize("inverted", [0.0, 0.2])
def test_2d_energy_gradient(inverted):
    pr = _stretched(seed=1, inverted=inverted)
    n = pr.prepare(0.01)
    rng = np.random.default_rng(2)
    for dv in (np.zeros(2 * n), rng.uniform(-0.2, 0.2, 2 * n)):
        eg, eo = pr.gpu.energy(dv), pr.orc.energy(dv)
        assert abs(eg - eo) <= 1e-11 * max(1.0, abs(eo))
        g, nrm = pr.gpu.gradient(dv)
        go = pr.orc.gradient(dv)
        assert rel_err(g, go) < STAGE_TOL
        assert abs(nrm - pr.orc.scaled_norm(go)) <= 1e-10 * max(nrm, 1e-300)


def _sym_err(m):
    b, c = m["blocks"], m["cols"]
    ns = b.shape[1]
    err = 0.0
    for r in range(b.shape[0]):
        for s in range(ns):
            j = c[r, s]
            if j >= 0:
                err = max(err, np.abs(b[r, s] - b[j, ns - 1 - s].T).max())
    return err


@pytest.mark.parametrize("project", [True, False])
@pytest.mark.parametrize("inverted", [0.0, 0.2])
def test_2d_assembly(project, inverted):
    pr = _stretched(seed=4, cells=5, f_spread=0.45, inverted=inverted)
    n = pr.prepare(0.01)
    rng = np.random.default_rng(5)
    dv = rng.uniform(-0.2, 0.2, 2 * n)
    dv.reshape(-1, 2)[pr.orc.grid()["dirichlet"] == 1] = 0
    pr.gpu.assemble(dv, project)
    pr.orc.assemble(dv, project)
    m = pr.gpu.level_matrix(0)
    ob, oc = pr.orc.level_matrix(0)
    assert np.array_equal(m["cols"], oc)
    assert rel_err(m["blocks"], ob) < STAGE_TOL
    assert _sym_err(m) == 0.0  # exact block symmetry (test_objective.cpp:180-191)
    x = rng.uniform(-1, 1, 2 * n)
    assert rel_err(pr.gpu.matvec(x), pr.orc.matvec(x)) < STAGE_TOL


@pytest.mark.parametrize("embedding", ["linear", "quadratic"])
def test_2d_hierarchy_and_vcycle(embedding):
    pr = _stretched(seed=6, cells=10)
    n = pr.prepare(0.01)
    dv = np.zeros(2 * n)
    pr.gpu.assemble(dv)
    pr.orc.assemble(dv)
    emb = O.LINEAR if embedding == "linear" else O.QUADRATIC
    lv = pr.gpu.build_hierarchy(3, embedding)
    assert lv == pr.orc.build_hierarchy(3, emb) == 3
    for m in range(lv):
        g = pr.gpu.level_matrix(m)
        ob, oc = pr.orc.level_matrix(m)
        info = pr.orc.level_info(m)
        assert np.array_equal(g["coords"], info["coords"])
        assert np.array_equal(g["dirichlet"], info["dirichlet"])
        assert np.array_equal(g["cols"], oc)
        assert rel_err(g["blocks"], ob) < STAGE_TOL
        assert _sym_err(g) == 0.0
    b = np.random.default_rng(7).uniform(-1, 1, 2 * n)
    u, it = pr.gpu.vcycle(b)
    uo, ito = pr.orc.vcycle(b)
    assert it == ito
    assert rel_err(u, uo) < 1e-9


@pytest.mark.parametrize("kind", ["hot", "lbfgs-h", "pn-pcg", "pn-pcg-mf", "pn-mgpcg"])
def test_2d_step_grid(kind):
    pr = _stretched(seed=8, cells=6)
    pr.set_solver(kind=kind, epsilon=1e-7)
    pr.prepare(1.0 / 24)
    g = pr.gpu.step_grid()
    o = pr.orc.step_grid()
    assert g["converged"] and o["converged"]
    assert abs(g["outer_iterations"] - o["outer_iterations"]) <= 1
    assert rel_err(g["velocity"], o["velocity"]) < STATE_TOL
    d = pr.orc.grid()["dirichlet"] == 1
    bc = pr.orc.grid()["bc_velocity"].reshape(-1, 2)
    assert np.array_equal(g["velocity"].reshape(-1, 2)[d], bc[d])  # scripted velocities exact


def _steps(sd, p, steps):
    pr = Pair2(sd, p)
    for _ in range(steps):
        sg = pr.gpu.advance_step(1.0)
        so = pr.orc.advance_step(1.0)
        assert sg["node_count"] == so["node_count"]
        assert abs(sg["outer_iterations"] - so["outer_iterations"]) <= 1
        assert abs(sg["dt"] - so["dt"]) <= 1e-12 * so["dt"]
        g, o = pr.gpu.particles(), pr.orc.get_particles()
        for k in ("x", "v", "F"):
            assert elem_rel_err(g[k], o[k]) < STATE_TOL, k
    rows_g, rows_o = pr.gpu.diagnostics(), pr.orc.diagnostics()
    if len(rows_g["outer_iteration"]) == len(rows_o["outer_iteration"]):
        assert np.array_equal(rows_g["outer_iteration"], rows_o["outer_iteration"])
        assert np.allclose(rows_g["energy"], rows_o["energy"], rtol=1e-9, atol=0)
    return pr


@pytest.mark.parametrize("plasticity", ["none", "von_mises", "snow"])
def test_2d_advance_steps(plasticity):
    mat = {"density": 1000.0, "youngs": 5e4, "poisson": 0.3}
    if plasticity == "von_mises":
        mat["plasticity"] = {"kind": "von_mises", "yield_stress": 300.0}
    elif plasticity == "snow":
        mat["plasticity"] = {"kind": "snow_clamp", "lo": 0.99, "hi": 1.001}
    sd = scene2(materials=[mat], colliders=[FLOOR],
                objects=[{"shape": {"kind": "box", "min": [0.04, 0.04], "max": [0.16, 0.12]}, "material": 0,
                          "velocity": [0.0, -1.0],
                          "initial_deformation": {"kind": "random_diagonal", "lo": 0.9, "hi": 1.1}}],
                extra={"seed": 3, "fps": 100})
    pr = Pair2(sd)
    _steps(sd, pr.p, 4)


def test_2d_sampling_matches_oracle_bitwise():
    sd = scene2(objects=[{"shape": {"kind": "sphere", "center": [0.1, 0.1], "radius": 0.05}, "material": 0}],
                extra={"seed": 11, "ppc": 6})
    sc = parse_scene(json.dumps(sd))
    p = sample_scene_particles(sc)
    orc = O.Oracle(2)
    orc.set_scene(sc.source)
    orc.sample_scene()
    o = orc.get_particles()
    assert np.array_equal(p["x"], o["x"]) and np.array_equal(p["volume"], o["volume"])


# ----------------------------------------------------------------------------------------------
# The reference's 2D solver suite (test_solvers.cpp) on the device path, each checked against
# the oracle where both sides produce the same quantity.
def deformed_block2(seed, cells, youngs, f_lo, f_hi, gravity=(0.0, 0.0)):
    """test_solvers.cpp:22-47: a block of 4 particles per cell, diagonal F in [f_lo, f_hi]."""
    rng = np.random.default_rng(seed)
    dx = 0.01
    xs, Fs = [], []
    for cell in range(cells ** 2):
        cc = np.array(np.unravel_index(cell, (cells, cells)))
        for _ in range(4):
            xs.append((cc + rng.uniform(0.05, 0.95, 2)) * dx)
            Fs.append(np.diag(rng.uniform(f_lo, f_hi, 2)))
    n = len(xs)
    vol = dx ** 2 / 4
    p = dict(x=np.array(xs), v=np.zeros((n, 2)), F=np.array(Fs), C=np.zeros((n, 2, 2)),
             mass=np.full(n, 1000.0 * vol), volume=np.full(n, vol), material=np.zeros(n, np.int32))
    return Pair2(scene2(dx=dx, youngs=youngs, gravity=gravity), p)


def test_2d_rest_state_no_work():  # test_solvers.cpp:200-212
    pr = deformed_block2(55, 4, 5e4, 1.0, 1.0)
    pr.prepare(1.0 / 24)
    r = pr.gpu.step_grid()
    assert r["converged"] and r["outer_iterations"] == 0 and np.linalg.norm(r["dv"]) == 0.0


@pytest.mark.parametrize("kind", ["hot", "pn-pcg", "pn-pcg-mf", "pn-mgpcg", "lbfgs-h"])
def test_2d_all_solvers_reach_criterion(kind):  # test_solvers.cpp:214-234
    pr = deformed_block2(56, 8, 5e4, 0.7, 1.3)
    pr.set_solver(kind=kind)
    n = pr.prepare(1.0 / 24)
    pr.gpu.clear_diagnostics()
    r = pr.gpu.step_grid()
    assert r["converged"]
    _, nrm = pr.gpu.gradient(r["dv"])
    assert nrm <= 1e-7 * np.sqrt(n)
    diag = pr.gpu.diagnostics()
    assert np.all(np.diff(diag["energy"]) < 0)
    assert diag["energy"].size == r["outer_iterations"]
    o = pr.orc.step_grid()
    assert abs(r["outer_iterations"] - o["outer_iterations"]) <= 1
    assert rel_err(r["dv"], o["dv"]) < STATE_TOL


def test_2d_lbfgs_h_is_hot_single_level():  # test_solvers.cpp:236-246
    pr = deformed_block2(57, 6, 5e4, 0.8, 1.2)
    pr.prepare(1.0 / 24)
    pr.gpu.set_solver(kind="lbfgs-h")
    a = pr.gpu.step_grid()
    pr.gpu.set_solver(kind="hot", levels=1)
    b = pr.gpu.step_grid()
    assert a["outer_iterations"] == b["outer_iterations"] and np.array_equal(a["dv"], b["dv"])


def test_2d_matrix_free_equals_assembled():  # test_solvers.cpp:248-256
    pr = deformed_block2(58, 4, 5e4, 0.9, 1.1)
    pr.prepare(1.0 / 48)
    pr.gpu.set_solver(kind="pn-pcg")
    a = pr.gpu.step_grid()
    pr.gpu.set_solver(kind="pn-pcg-mf")
    b = pr.gpu.step_grid()
    assert a["outer_iterations"] == b["outer_iterations"]
    assert np.linalg.norm(a["dv"] - b["dv"]) <= 1e-7 * max(1.0, np.linalg.norm(a["dv"]))


def test_2d_ballistic_single_particle():  # test_solvers.cpp:296-321
    p = dict(x=np.array([[0.305, 0.304]]), v=np.zeros((1, 2)), F=np.eye(2)[None], C=np.zeros((1, 2, 2)),
             mass=np.array([0.1]), volume=np.array([1e-4]), material=np.zeros(1, np.int32))
    pr = Pair2(scene2(dx=0.01, youngs=1e5), p)
    dt = 1.0 / 24
    pr.prepare(dt)
    for kind in ("hot", "pn-pcg"):
        pr.gpu.set_solver(kind=kind, epsilon=1e-10)
        r = pr.gpu.step_grid()
        err = np.abs(r["velocity"].reshape(-1, 2) - dt * np.array([0.0, -9.8])).max()
        assert err < (1e-8 if kind == "pn-pcg" else 1e-5)  # DESIGN.md §2 divergence log


def test_2d_dirichlet_exact():  # test_solvers.cpp:323-340
    pr = deformed_block2(61, 5, 5e4, 0.9, 1.1, (0.0, -9.8))
    pr.prepare(1.0 / 24)
    g = pr.gpu.grid()
    dirm = (g["coords"][:, 0] <= 1).astype(np.uint8)
    script = np.array([0.123, -0.456])
    vel = g["velocity"].reshape(-1, 2).copy()
    vel[dirm == 1] = script
    bc = np.zeros_like(vel)
    bc[dirm == 1] = script
    pr.gpu.set_grid(velocity=vel.reshape(-1), dirichlet=dirm, bc_velocity=bc.reshape(-1))
    r = pr.gpu.step_grid()
    assert r["converged"]
    out = r["velocity"].reshape(-1, 2)
    assert np.all(np.linalg.norm(out[dirm == 1] - script, axis=1) == 0.0)


def test_2d_hot_fewer_iterations_than_lbfgs_h():  # test_solvers.cpp:342-351
    pr = deformed_block2(62, 10, 5e4, 0.7, 1.3)
    pr.prepare(1.0 / 24)
    hot = pr.gpu.step_grid()
    pr.gpu.set_solver(kind="lbfgs-h")
    lbh = pr.gpu.step_grid()
    assert hot["converged"] and lbh["converged"]
    assert hot["outer_iterations"] < lbh["outer_iterations"]


@pytest.mark.parametrize("model", ["neo_hookean", "hardening", "drucker_prager"])
def test_2d_extension_steps(model):
    mat = {"density": 1000.0, "youngs": 5e4, "poisson": 0.3}
    if model == "neo_hookean":
        mat["elasticity"] = "neo_hookean"
    elif model == "hardening":
        mat["plasticity"] = {"kind": "snow_clamp", "lo": 0.99, "hi": 1.001, "hardening": 10.0}
    else:
        mat["plasticity"] = {"kind": "drucker_prager", "friction_angle": 30.0}
    sd = scene2(materials=[mat], colliders=[FLOOR],
                objects=[{"shape": {"kind": "box", "min": [0.04, 0.04], "max": [0.16, 0.12]}, "material": 0,
                          "velocity": [0.0, -1.0]}], extra={"seed": 5, "fps": 100})
    pr = Pair2(sd)
    _steps(sd, pr.p, 3)
