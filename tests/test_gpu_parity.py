"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded
inputs.  Tolerances (north star, BASELINE.json): indexing bit-exact; fp64 state within
1e-6 relative after each step; outer iteration counts within +-1.  Stage-level checks use
tighter bounds where the two sides differ only by summation order (1e-10..1e-12)."""
import numpy as np
import pytest

from tests.gpu_common import Pair, block_scene_dict, random_block_particles, rel_err, scene, scene_from_dict

pytestmark = pytest.mark.gpu

STATE_TOL = 1e-6   # north_star: grid velocities, particle x / F after each step
STAGE_TOL = 1e-10  # same arithmetic, different summation order


def _stretched_block_pair(seed=0, cells=6, dirichlet_floor=True, youngs=5e4, f_spread=0.3):
    rng = np.random.default_rng(seed)
    cols = []
    if dirichlet_floor:
        cols = [{"shape": {"kind": "half_space", "point": [0.0, 0.021, 0.0], "normal": [0.0, 1.0, 0.0]},
                 "motion": {"kind": "static"}}]
    sc = scene_from_dict(block_scene_dict(youngs=youngs, colliders=cols))
    p = random_block_particles(rng, 0.02, cells, f_spread=f_spread, v_spread=0.3)
    return Pair(sc, p)


@pytest.mark.parametrize("name", ["cfg1_cube", "cfg1_stretched", "cfg1_drop"])
def test_activation_and_p2g(name):
    pr = Pair(scene(name))
    n = pr.prepare(2e-3)
    g, o = pr.gpu.grid(), pr.orc.grid()
    assert n == o["coords"].shape[0]
    assert np.array_equal(g["coords"], o["coords"])  # bit-exact lexicographic indexing
    assert np.array_equal(g["dirichlet"], o["dirichlet"])
    assert rel_err(g["mass"], o["mass"]) < 1e-12
    assert rel_err(g["momentum"], o["momentum"]) < 1e-12
    assert rel_err(g["velocity"], o["velocity"]) < 1e-12
    _, scale = pr.orc.node_cn()
    assert rel_err(g["cn_scale"], scale) < 1e-12


def test_boundary_scripts_rotation_colliders():
    sc = scene("cfg2_twisting_bars")
    # a thin slice of the bars keeps the oracle fast: particles near both ends
    from paper_1911_07913_b200 import sample_scene_particles
    p = sample_scene_particles(sc)
    keep = (p["x"][:, 0] < 0.06) | (p["x"][:, 0] > 0.54)
    p = {k: v[keep] for k, v in p.items()}
    pr = Pair(sc, p)
    pr.prepare(0.01)
    g, o = pr.gpu.grid(), pr.orc.grid()
    assert np.array_equal(g["coords"], o["coords"])
    assert np.array_equal(g["dirichlet"], o["dirichlet"])
    assert g["dirichlet"].sum() > 0
    assert rel_err(g["bc_velocity"], o["bc_velocity"]) < 1e-13
    assert rel_err(g["velocity"], o["velocity"]) < 1e-12


def test_collider_shapes_and_motions():
    """apply_boundary_scripts (simulation.hpp:259-272) for every collider shape and motion:
    a static sphere, a rotating cylinder, a linearly moving box and a half-space floor cutting
    a moving block; Dirichlet flags bit-exact and scripted velocities, then two steps."""
    cols = [
        {"shape": {"kind": "sphere", "center": [0.05, 0.12, 0.05], "radius": 0.03}, "motion": {"kind": "static"}},
        {"shape": {"kind": "cylinder", "center": [0.1, 0.06, 0.1], "axis": [0.0, 0.0, 1.0], "radius": 0.025},
         "motion": {"kind": "rotation", "center": [0.1, 0.06, 0.1], "axis": [0.0, 0.0, 1.0], "omega": 2.0}},
        {"shape": {"kind": "box", "min": [-0.01, -0.01, -0.01], "max": [0.02, 0.13, 0.13]},
         "motion": {"kind": "linear", "velocity": [0.3, 0.0, -0.1]}},
        {"shape": {"kind": "half_space", "point": [0.0, 0.011, 0.0], "normal": [0.0, 1.0, 0.0]},
         "motion": {"kind": "static"}},
    ]
    sc = scene_from_dict(block_scene_dict(youngs=8e4, colliders=cols))
    p = random_block_particles(np.random.default_rng(31), 0.02, 6, f_spread=0.1, v_spread=0.2)
    pr = Pair(sc, p)
    pr.prepare(1.0 / 48, time=0.25)
    g, o = pr.gpu.grid(), pr.orc.grid()
    assert np.array_equal(g["coords"], o["coords"])
    assert np.array_equal(g["dirichlet"], o["dirichlet"])
    assert g["dirichlet"].sum() > 0
    assert rel_err(g["bc_velocity"], o["bc_velocity"]) < 1e-13
    pr2 = Pair(sc, p)
    for k in range(2):
        frame_end = (k + 1) / sc.fps
        s = pr2.gpu.advance_step(frame_end)
        so = pr2.orc.advance_step(frame_end)
        assert s["node_count"] == so["node_count"]
        assert abs(s["outer_iterations"] - so["outer_iterations"]) <= 1, (k, s, so)
        gp, op = pr2.gpu.particles(), pr2.orc.get_particles()
        for key in ("x", "v", "F"):
            assert rel_err(gp[key], op[key]) < STATE_TOL, (k, key)


def test_energy_gradient():
    pr = _stretched_block_pair(seed=1)
    n = pr.prepare(0.01)
    rng = np.random.default_rng(2)
    for _ in range(3):
        dv = rng.uniform(-0.3, 0.3, 3 * n)
        dv.reshape(-1, 3)[pr.orc.grid()["dirichlet"] == 1] = 0
        e, eo = pr.gpu.energy(dv), pr.orc.energy(dv)
        assert abs(e - eo) <= 1e-11 * abs(eo)
        g, nrm = pr.gpu.gradient(dv)
        go = pr.orc.gradient(dv)
        assert rel_err(g, go) < STAGE_TOL
        assert abs(nrm - pr.orc.scaled_norm(go)) <= 1e-11 * pr.orc.scaled_norm(go)


def test_non_finite_dv_rejected():
    pr = _stretched_block_pair(seed=3, cells=3)
    n = pr.prepare(0.01)
    dv = np.zeros(3 * n)
    dv[4] = np.nan
    from paper_1911_07913_b200 import InvalidArgument
    with pytest.raises(InvalidArgument):
        pr.gpu.energy(dv)


def _sym_err(m):
    b, c = m["blocks"], m["cols"]
    ns = c.shape[1]  # 125 (radius 2) or 343 (radius 3): slot s and ns-1-s are mirror offsets
    err = 0.0
    for r in range(b.shape[0]):
        for s in range(ns):
            j = c[r, s]
            if j >= 0:
                err = max(err, np.abs(b[r, s] - b[j, ns - 1 - s].T).max())
    return err


@pytest.mark.parametrize("project", [True, False])
def test_assembly_matches_oracle(project):
    pr = _stretched_block_pair(seed=4, cells=4, f_spread=0.45)
    n = pr.prepare(0.01)
    rng = np.random.default_rng(5)
    dv = rng.uniform(-0.2, 0.2, 3 * n)
    dv.reshape(-1, 3)[pr.orc.grid()["dirichlet"] == 1] = 0
    pr.gpu.assemble(dv, project)
    pr.orc.assemble(dv, project)
    m = pr.gpu.level_matrix(0)
    ob, oc = pr.orc.level_matrix(0)
    assert np.array_equal(m["cols"], oc)
    assert rel_err(m["blocks"], ob) < STAGE_TOL
    assert _sym_err(m) == 0.0  # exact block symmetry (test_objective.cpp:185)


def _assembled(sc, particles, env, dv_seed=5, project=True):
    """Level-0 matrix of a fresh context created under the given HOT_ASM* environment (the knobs
    are read once per context)."""
    import os

    from paper_1911_07913_b200 import Simulation
    saved = {k: os.environ.pop(k, None) for k in ("HOT_ASM", "HOT_ASM_RING")}
    os.environ.update(env)
    try:
        sim = Simulation(sc)
    finally:
        for k in ("HOT_ASM", "HOT_ASM_RING"):
            os.environ.pop(k, None)
            if saved[k] is not None:
                os.environ[k] = saved[k]
    sim.set_particles(**particles)
    n = sim.stage_prepare(0.01)
    dv = np.random.default_rng(dv_seed).uniform(-0.2, 0.2, 3 * n)
    sim.assemble(dv, project)
    m = sim.level_matrix(0)
    sim.close()
    return m


@pytest.mark.parametrize("project", [True, False])
def test_assembly_by_bins_matches_row_tiles_and_bands(project):
    """The two level-0 assembly paths (by bins: k_bin_pairs + k_row_gather, the default; row tiles:
    k_assemble_tiles) give the same matrix up to summation order, and the by-bins path gives the
    same bits whether all bins' pair sums are resident or go through a small ring in bands."""
    rng = np.random.default_rng(11)
    sc = scene_from_dict(block_scene_dict(youngs=5e4, colliders=[
        {"shape": {"kind": "half_space", "point": [0.0, 0.021, 0.0], "normal": [0.0, 1.0, 0.0]},
         "motion": {"kind": "static"}}]))
    p = random_block_particles(rng, 0.02, 9, f_spread=0.4, v_spread=0.3)
    # ragged bins: drop a third of the particles (bins of 0..8 particles, chunks of 1..3 groups)
    keep = rng.uniform(size=p["x"].shape[0]) > 0.33
    p = {k: v[keep] for k, v in p.items()}
    bins = _assembled(sc, p, {}, project=project)
    tiles = _assembled(sc, p, {"HOT_ASM": "tiles"}, project=project)
    band = _assembled(sc, p, {"HOT_ASM_RING": "1"}, project=project)  # clamped up to 4 lattice planes
    assert np.array_equal(bins["cols"], tiles["cols"])
    scale = np.abs(tiles["blocks"]).max()
    assert np.abs(bins["blocks"] - tiles["blocks"]).max() <= 1e-13 * scale
    assert _sym_err(bins) == 0.0
    assert np.array_equal(bins["blocks"], band["blocks"])


def test_hierarchy_and_vcycle():
    pr = _stretched_block_pair(seed=6, cells=6, youngs=1e6)
    n = pr.prepare(0.01)
    pr.gpu.assemble()
    pr.orc.assemble()
    assert pr.gpu.build_hierarchy(3) == pr.orc.build_hierarchy(3)
    for lvl in range(pr.orc.level_count()):
        m = pr.gpu.level_matrix(lvl)
        info = pr.orc.level_info(lvl)
        ob, oc = pr.orc.level_matrix(lvl)
        assert np.array_equal(m["coords"], info["coords"])  # bit-exact coarse indexing
        assert np.array_equal(m["dirichlet"], info["dirichlet"])
        assert np.array_equal(m["cols"], oc)
        assert rel_err(m["blocks"], ob) < STAGE_TOL
        assert _sym_err(m) == 0.0
    rng = np.random.default_rng(7)
    for _ in range(3):
        b = rng.uniform(-1, 1, 3 * n)
        u, it = pr.gpu.vcycle(b)
        uo, ito = pr.orc.vcycle(b)
        assert it == ito
        assert rel_err(u, uo) < 1e-9


def test_quadratic_embedding_hierarchy_and_vcycle():
    """Quadratic node embedding (multigrid.hpp:72-90, 274-275): coarse levels of radius 3
    (343 slots) with colour modulus 3; coarse indexing and column ids bit-exact, Galerkin
    blocks, exact symmetry, and V-cycles against the oracle."""
    from oracle.oracle import QUADRATIC

    pr = _stretched_block_pair(seed=16, cells=6, youngs=1e6)
    n = pr.prepare(0.01)
    pr.gpu.assemble()
    pr.orc.assemble()
    assert pr.gpu.build_hierarchy(3, embedding="quadratic") == pr.orc.build_hierarchy(3, QUADRATIC)
    for lvl in range(pr.orc.level_count()):
        m = pr.gpu.level_matrix(lvl)
        info = pr.orc.level_info(lvl)
        ob, oc = pr.orc.level_matrix(lvl)
        assert m["cols"].shape == oc.shape  # 125 slots on level 0, 343 on the coarse levels
        assert np.array_equal(m["coords"], info["coords"])
        assert np.array_equal(m["dirichlet"], info["dirichlet"])
        assert np.array_equal(m["cols"], oc)
        assert rel_err(m["blocks"], ob) < STAGE_TOL
        assert _sym_err(m) == 0.0
    rng = np.random.default_rng(17)
    for _ in range(2):
        b = rng.uniform(-1, 1, 3 * n)
        u, it = pr.gpu.vcycle(b)
        uo, ito = pr.orc.vcycle(b)
        assert it == ito
        assert rel_err(u, uo) < 1e-9


def test_quadratic_embedding_step_grid():
    """HOT step_grid with the quadratic embedding (the paper's embedding ablation)."""
    pr = _stretched_block_pair(seed=18, cells=6)
    pr.prepare(1.0 / 24)
    pr.set_solver(kind="hot", epsilon=1e-7, embedding="quadratic")
    r = pr.gpu.step_grid()
    ro = pr.orc.step_grid()
    assert r["converged"] and ro["converged"]
    assert abs(r["outer_iterations"] - ro["outer_iterations"]) <= 1
    assert rel_err(r["velocity"], ro["velocity"]) < STATE_TOL


@pytest.mark.parametrize("coarse", ["flow", "barrier"])
def test_vcycle_coarse_smoother_schedules(monkeypatch, coarse):
    """The coarse levels' smoother runs as a dataflow kernel (per-row epoch flags) or as a
    persistent kernel with a grid barrier per wave; both follow the reference's sequential
    sweep exactly and compute each row identically, so they agree bit for bit."""
    monkeypatch.setenv("HOT_SGS_COARSE", coarse)
    pr = _stretched_block_pair(seed=14, cells=6, youngs=1e6)
    n = pr.prepare(0.01)
    pr.gpu.assemble()
    pr.orc.assemble()
    pr.gpu.build_hierarchy(3)
    pr.orc.build_hierarchy(3)
    b = np.random.default_rng(15).uniform(-1, 1, 3 * n)
    u, it = pr.gpu.vcycle(b)
    uo, ito = pr.orc.vcycle(b)
    assert it == ito and rel_err(u, uo) < 1e-9
    monkeypatch.setenv("HOT_SGS_COARSE", "barrier" if coarse == "flow" else "flow")
    from paper_1911_07913_b200 import Simulation

    g2 = Simulation(pr.sc)  # the options are read when a context is created
    g2.set_particles(**pr.p)
    g2.stage_prepare(0.01)
    g2.assemble()
    g2.build_hierarchy(3)
    u2, it2 = g2.vcycle(b)
    assert it2 == it and np.array_equal(u, u2)


@pytest.mark.parametrize("schedule", ["stream", "waves"])
def test_vcycle_streaming_wave_schedule(monkeypatch, schedule):
    """Same V-cycle parity with every SGS level run on the large-wave schedules the benchmark's
    level 0 uses: the persistent bulk-copy streaming kernel (grid barrier per wave), or one
    launch per wave.  Both compute every row with the same arithmetic in the same sequential
    order, so they agree bit for bit."""
    monkeypatch.setenv("HOT_SGS_STREAM_MIN", "0")
    if schedule != "stream":
        monkeypatch.setenv("HOT_SGS_LEVEL0", schedule)
    pr = _stretched_block_pair(seed=12, cells=6, youngs=1e6)
    n = pr.prepare(0.01)
    pr.gpu.assemble()
    pr.orc.assemble()
    pr.gpu.build_hierarchy(3)
    pr.orc.build_hierarchy(3)
    b = np.random.default_rng(13).uniform(-1, 1, 3 * n)
    u, it = pr.gpu.vcycle(b)
    uo, ito = pr.orc.vcycle(b)
    assert it == ito and rel_err(u, uo) < 1e-9
    other = "waves" if schedule == "stream" else "stream"
    monkeypatch.delenv("HOT_SGS_LEVEL0", raising=False)
    if other != "stream":
        monkeypatch.setenv("HOT_SGS_LEVEL0", other)
    from paper_1911_07913_b200 import Simulation

    g2 = Simulation(pr.sc)  # the options are read when a context is created
    g2.set_particles(**pr.p)
    g2.stage_prepare(0.01)
    g2.assemble()
    g2.build_hierarchy(3)
    u2, it2 = g2.vcycle(b)
    assert it2 == it and np.array_equal(u, u2)


def test_single_level_vcycle_is_coarse_solve():
    pr = _stretched_block_pair(seed=8, cells=4)
    n = pr.prepare(0.01)
    pr.gpu.assemble()
    pr.orc.assemble()
    pr.gpu.build_hierarchy(1)
    pr.orc.build_hierarchy(1)
    b = np.random.default_rng(9).uniform(-1, 1, 3 * n)
    u, it = pr.gpu.vcycle(b)
    uo, ito = pr.orc.vcycle(b)
    assert it == ito and rel_err(u, uo) < 1e-9


@pytest.mark.parametrize("kind", ["hot", "lbfgs-h", "pn-pcg", "pn-pcg-mf", "pn-mgpcg"])
def test_step_grid(kind):
    """step_grid (solvers.hpp:354-381) for every solver kind: HOT and LBFGS-H (L-BFGS), and the
    projected-Newton baselines (solvers.hpp:235-300): assembled Jacobi-PCG, matrix-free
    Jacobi-PCG, and V-cycle-preconditioned PCG."""
    pr = _stretched_block_pair(seed=10, cells=6)
    pr.prepare(1.0 / 24)
    pr.set_solver(kind=kind, epsilon=1e-7)
    r = pr.gpu.step_grid()
    ro = pr.orc.step_grid()
    assert r["converged"] and ro["converged"]
    assert abs(r["outer_iterations"] - ro["outer_iterations"]) <= 1
    assert rel_err(r["velocity"], ro["velocity"]) < STATE_TOL
    dirm = pr.orc.grid()["dirichlet"] == 1
    bc = pr.orc.grid()["bc_velocity"].reshape(-1, 3)
    assert np.array_equal(r["velocity"].reshape(-1, 3)[dirm], bc[dirm])  # exact scripted velocities
    if kind.startswith("pn"):
        assert abs(r["inner_total"] - ro["inner_total"]) <= max(2, 0.1 * ro["inner_total"])


def test_rest_state_zero_iterations():
    rng = np.random.default_rng(11)
    sc = scene_from_dict(block_scene_dict(gravity=(0.0, 0.0, 0.0)))
    p = random_block_particles(rng, 0.02, 3, f_spread=0.0, v_spread=0.0)
    pr = Pair(sc, p)
    pr.prepare(1.0 / 24)
    r = pr.gpu.step_grid()
    assert r["converged"] and r["outer_iterations"] == 0 and np.abs(r["dv"]).max() == 0.0


def _run_steps(name, steps, particles=None):
    pr = Pair(scene(name), particles)
    sc = pr.sc
    for k in range(steps):
        frame_end = (k + 1) / sc.fps
        s = pr.gpu.advance_step(frame_end)
        so = pr.orc.advance_step(frame_end)
        assert s["node_count"] == so["node_count"]
        assert abs(s["outer_iterations"] - so["outer_iterations"]) <= 1, (k, s, so)
        assert s["dt"] == pytest.approx(so["dt"], rel=1e-12)
        gp, op = pr.gpu.particles(), pr.orc.get_particles()
        for key in ("x", "v", "F"):
            assert rel_err(gp[key], op[key]) < STATE_TOL, (k, key)
    return pr


def test_cfg1_cube_steps():
    _run_steps("cfg1_cube", 5)


def test_cfg1_cube_full_20_steps():
    """BASELINE config 1 as specified: the elastic cube, 20 steps, parity after every step
    (x, v, F to 1e-6 relative, node counts equal, outer iterations within 1)."""
    _run_steps("cfg1_cube", 20)


def test_cfg1_stretched_steps():
    _run_steps("cfg1_stretched", 3)


def test_cfg1_drop_steps_with_floor():
    pr = _run_steps("cfg1_drop", 4)
    assert pr.gpu.grid is not None


@pytest.mark.parametrize("plasticity", [
    {"kind": "von_mises", "yield_stress": 2.0e3},
    {"kind": "snow_clamp", "lo": 0.975, "hi": 1.0075},
])
def test_plastic_return_map_steps(plasticity):
    """The strain update's return map (constitutive.hpp:224-251) on the device: von Mises with a
    yield stress low enough that most particles yield, and the snow clamp with a tight band,
    over several steps from a pre-stretched, moving block; x, v, F against the oracle."""
    d = block_scene_dict(youngs=2e5, extra={"fps": 48})
    d["materials"][0]["plasticity"] = dict(plasticity)
    sc = scene_from_dict(d)
    p = random_block_particles(np.random.default_rng(21), 0.02, 6, f_spread=0.05, v_spread=0.5)
    pr = Pair(sc, p)
    for k in range(3):
        frame_end = (k + 1) / sc.fps
        s = pr.gpu.advance_step(frame_end)
        so = pr.orc.advance_step(frame_end)
        assert s["node_count"] == so["node_count"]
        assert abs(s["outer_iterations"] - so["outer_iterations"]) <= 1, (k, s, so)
        gp, op = pr.gpu.particles(), pr.orc.get_particles()
        for key in ("x", "v", "F"):
            assert rel_err(gp[key], op[key]) < STATE_TOL, (k, key)
    # the map did act: F left the elastic trial state somewhere (det or singular values clamped)
    F = pr.gpu.particles()["F"]
    sv = np.linalg.svd(F, compute_uv=False)
    if plasticity["kind"] == "snow_clamp":
        assert sv.min() >= 0.975 - 1e-12 and sv.max() <= 1.0075 + 1e-12


def test_solver_failure_leaves_particles_unmodified():
    pr = Pair(scene("cfg1_stretched"))
    pr.set_solver(outer_cap=1)
    before = pr.gpu.particles()
    from paper_1911_07913_b200 import SolverFailure
    with pytest.raises(SolverFailure) as e:
        pr.gpu.advance_step(1.0 / pr.sc.fps)
    assert str(e.value).startswith("step 0: quasi-newton solve: outer iteration cap reached")
    after = pr.gpu.particles()
    for k in before:
        assert np.array_equal(before[k], after[k])


def test_empty_and_single_particle():
    sc = scene_from_dict(block_scene_dict())
    from paper_1911_07913_b200 import Simulation
    sim = Simulation(sc)
    sim.set_particles(np.zeros((0, 3)))
    st = sim.advance_step(1.0 / 24)
    assert st["node_count"] == 0 and st["converged"]
    # ballistic single particle (test_solvers.cpp:296-321): dv = g dt
    p = dict(x=np.array([[0.305, 0.304, 0.3]]), mass=np.array([0.1]), volume=np.array([1e-4]))
    pr = Pair(sc, dict(x=p["x"], v=np.zeros((1, 3)), mass=p["mass"], volume=p["volume"], F=np.eye(3)[None],
                       C=np.zeros((1, 3, 3)), material=np.zeros(1, np.int32)))
    pr.prepare(1.0 / 24)
    pr.set_solver(epsilon=1e-10)
    r = pr.gpu.step_grid()
    ro = pr.orc.step_grid()
    assert rel_err(r["velocity"], ro["velocity"]) < STATE_TOL
    # eps*sqrt(n) in the CN norm bounds the HOT iterate only to ~3e-5 with 2.5e-4 kg fringe nodes
    # (see tests/test_oracle_solvers.py::test_ballistic_single_particle)
    assert np.abs(r["velocity"].reshape(-1, 3) - np.array([0, -9.8, 0]) / 24).max() < 3e-5


def test_deterministic_reruns_are_byte_identical(tmp_path):
    """cli.cpp:120-121 / SPEC --deterministic: the frame loop's output directory (HOTP
    snapshots, text tables, diagnostics.csv with zeroed wall times) is byte-identical across
    reruns, and the last frame agrees with the oracle's frame loop."""
    from paper_1911_07913_b200 import io

    sc = scene("cfg1_cube")
    logs = []
    for run in ("a", "b"):
        io.run_simulation(sc, tmp_path / run, deterministic=True, frames=2, log=logs.append)
    files = sorted(p.name for p in (tmp_path / "a").iterdir())
    assert files == sorted(p.name for p in (tmp_path / "b").iterdir())
    assert {"frame_0000.bin", "frame_0002.txt", "diagnostics.csv"} <= set(files)
    for f in files:
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes(), f
    # the oracle's frame loop for the same scene and frames
    from oracle.oracle import Oracle
    from paper_1911_07913_b200 import sample_scene_particles

    orc = Oracle(3)
    orc.set_scene(sc.source)
    p = sample_scene_particles(sc)
    orc.set_particles(p["x"], p["v"], p["mass"], p["volume"], p["F"], p["C"], p["material"])
    for frame in (1, 2):
        orc.set_sim_state(orc.sim_state()["time"], orc.sim_state()["step"], frame)
        while orc.sim_state()["time"] < frame / sc.fps - 1e-12:
            orc.advance_step(frame / sc.fps)
    snap = io.read_snapshot(tmp_path / "a" / "frame_0002.bin")
    xo = orc.get_particles()["x"].reshape(-1)
    assert rel_err(snap["positions"], xo) < STATE_TOL
