"""GPU parity on the BASELINE workloads themselves (configs[1..3] as committed under scenes/):
the full scenes, stepped on the GPU (through the C-ABI) and on the CPU oracle from the same
seeded particles.  After every step (north star, SURVEY.md §8(d) parity protocol):

- grid `coords[]` bit-exact at level 0 and at every coarse level (step 0), Dirichlet flags exact;
- grid mass / momentum / velocity (after P2G and after the solve), particle x / v / F within
  1e-6 PER ELEMENT relative (``elem_rel_err``: |a-b| / max(|b|, 1e-8 max|b|) per entry, so small
  entries are held to the same relative bar as large ones);
- outer L-BFGS iterations within +-1, and the diagnostics rows (solvers.hpp:31-41) equal row by
  row when the counts agree.

The oracle runs with every host thread (its parallel_for regions only: results do not depend on
the thread count).  Its step is the stage-by-stage restatement of advance_step
(simulation.hpp:286-323) so the grid can be compared between P2G and the solve."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.gpu_common import Pair, block_scene_dict, random_block_particles, scene, scene_from_dict

pytestmark = pytest.mark.gpu

STATE_TOL = 1e-6
FLOOR = 1e-8


def elem_rel_err(a, b, floor=FLOOR):
    """max_i |a_i - b_i| / max(|b_i|, floor * max|b|)."""
    a, b = np.asarray(a, dtype=float).ravel(), np.asarray(b, dtype=float).ravel()
    if b.size == 0:
        return 0.0
    den = np.maximum(np.abs(b), floor * max(np.abs(b).max(), 1e-300))
    return float((np.abs(a - b) / den).max())


def coarse_coords_linear(fine):
    """build_restriction's coarse node set under the linear embedding (multigrid.hpp:64-95,
    127-158): per axis an even c maps to c/2, an odd c to floor(c/2) and floor(c/2) + 1; the set
    sorted lexicographically (axis 0 most significant, common.hpp:41)."""
    f = np.asarray(fine, dtype=np.int64)
    lo = np.floor_divide(f, 2)
    odd = (f - 2 * lo) != 0
    cand = []
    for bits in range(8):
        sh = np.array([(bits >> 2) & 1, (bits >> 1) & 1, bits & 1])
        ok = np.all(odd | (sh == 0), axis=1)
        cand.append(lo[ok] + sh)
    c = np.unique(np.concatenate(cand), axis=0)  # np.unique on rows sorts lexicographically
    return c.astype(np.int32)


def oracle_stage_step(orc, sc, frame_end, frame, step):
    """advance_step (simulation.hpp:286-323) on the oracle, stage by stage: returns the grid after
    P2G + boundary scripts, the solve result and dt."""
    t = orc.sim_state()["time"]
    v = orc.get_particles()["v"]
    vmax = float(np.sqrt((v * v).sum(axis=1)).max()) if v.size else 0.0
    dt = min(O.cfl_dt(vmax, sc.dx, sc.fps), frame_end - t)
    orc.activate()
    orc.p2g()
    orc.apply_bc(t)
    grid = orc.grid()
    orc.make_state(dt)
    orc.clear_diagnostics()
    r = orc.step_grid(frame, step)
    orc.set_grid(velocity=r["velocity"])
    orc.g2p()
    orc.update_strain(dt)
    orc.advect(dt)
    orc.set_sim_state(t + dt, step + 1, frame)
    return grid, r, dt


def _baseline_steps(name, steps):
    O.set_threads(os.cpu_count() or 1)
    pr = Pair(scene(name))
    sc, gpu, orc = pr.sc, pr.gpu, pr.orc
    gpu.set_time(0.0, 0, 0)
    orc.set_sim_state(0.0, 0, 0)
    report = []
    for k in range(steps):
        frame_end = (k + 1) / sc.fps
        grid_o, r_o, dt = oracle_stage_step(orc, sc, frame_end, 0, k)
        diag_o = orc.diagnostics()
        # GPU: the same stages through the taps (grid after P2G, coarse sets, solve), then the
        # public advance_step for the particle state
        t = gpu.time_state()["time"]
        n = gpu.stage_prepare(dt, t)
        g = gpu.grid()
        assert n == grid_o["coords"].shape[0]
        assert np.array_equal(g["coords"], grid_o["coords"]), (name, k)  # bit-exact lexicographic indexing
        assert np.array_equal(g["dirichlet"], grid_o["dirichlet"]), (name, k)
        for key in ("mass", "momentum", "velocity"):
            assert elem_rel_err(g[key], grid_o[key]) < STATE_TOL, (name, k, key)
        if k == 0:  # coarse node sets of the hierarchy, bit-exact
            gpu.assemble(np.zeros(3 * n))
            levels = gpu.build_hierarchy(sc.levels)
            fine = grid_o["coords"]
            for m in range(1, levels):
                want = coarse_coords_linear(fine)
                got = gpu.level_coords(m)["coords"]
                assert np.array_equal(got, want), (name, m)
                fine = want
        r_g = gpu.step_grid(0, k)
        assert abs(r_g["outer_iterations"] - r_o["outer_iterations"]) <= 1, (name, k, r_g, r_o)
        assert elem_rel_err(r_g["velocity"], r_o["velocity"]) < STATE_TOL, (name, k)
        gpu.clear_diagnostics()
        s = gpu.advance_step(frame_end)
        assert s["dt"] == pytest.approx(dt, rel=1e-12)
        assert s["node_count"] == n and s["outer_iterations"] == r_g["outer_iterations"]
        gp, op = gpu.particles(), orc.get_particles()
        errs = {key: elem_rel_err(gp[key], op[key]) for key in ("x", "v", "F")}
        for key, e in errs.items():
            assert e < STATE_TOL, (name, k, key, e)
        diag_g = gpu.diagnostics()
        if r_g["outer_iterations"] == r_o["outer_iterations"]:  # diagnostics.csv rows (io.cpp:101-116)
            assert len(diag_g["outer_iteration"]) == len(diag_o["outer_iteration"])
            assert np.array_equal(diag_g["outer_iteration"], diag_o["outer_iteration"])
            assert np.array_equal(diag_g["step_length"], diag_o["step_length"])
            assert elem_rel_err(diag_g["energy"], diag_o["energy"], floor=0) < 1e-9
            assert elem_rel_err(diag_g["scaled_residual"], diag_o["scaled_residual"], floor=0) < 1e-5
        report.append((k, n, r_g["outer_iterations"], r_o["outer_iterations"], errs))
    print(name, report)
    return report


def test_cfg2_twisting_bars_full_scene_steps():
    """BASELINE configs[1] (the bench workload): 1,193,126 particles, dt = CFL 0.6, 3 steps."""
    _baseline_steps("cfg2_twisting_bars", 3)


def test_cfg3_metal_impact_full_scene_steps():
    """BASELINE configs[2]: von Mises metal sphere on a plate, 566K particles, 3 steps."""
    _baseline_steps("cfg3_metal_impact", 3)


def test_cfg4_snow_full_scene_step():
    """BASELINE configs[3]: two colliding snow boxes, 4.0M particles on the 256^3 grid, 1 step
    (the oracle needs minutes per step at this size)."""
    _baseline_steps("cfg4_snow", 1)


def _inverted_block(rng, frac, fps, plasticity=None):
    d = block_scene_dict(youngs=2e5, extra={"fps": fps})
    if plasticity:
        d["materials"][0]["plasticity"] = dict(plasticity)
    sc = scene_from_dict(d)
    p = random_block_particles(rng, 0.02, 6, f_spread=0.1, v_spread=0.3)
    flip = rng.random(p["F"].shape[0]) < frac  # inverted particles: one column of F negated
    p["F"][flip, :, 2] *= -1.0
    assert (np.linalg.det(p["F"]) < 0).sum() == flip.sum() > 0
    return Pair(sc, p)


def test_inverted_particles_stages():
    """det F < 0 on a fifth of the particles: svd_rv's sign convention on sigma_3
    (constitutive.hpp:66-82) and the |sigma_i + sigma_j| >= 1e-6 clamp of the rotation blocks
    (constitutive.hpp:178-185) in the energy, the gradient and the projected and unprojected
    Hessians, against the oracle at dv = 0 and at a random dv."""
    from tests.gpu_common import rel_err
    from tests.test_gpu_parity import _sym_err

    pr = _inverted_block(np.random.default_rng(33), 0.2, 48)
    n = pr.prepare(1.0 / 48)
    rng = np.random.default_rng(5)
    for dv in (np.zeros(3 * n), rng.uniform(-0.05, 0.05, 3 * n)):
        assert pr.gpu.energy(dv) == pytest.approx(pr.orc.energy(dv), rel=1e-11)
        g, _ = pr.gpu.gradient(dv)
        assert rel_err(g, pr.orc.gradient(dv)) < 1e-10
        for project in (True, False):
            pr.gpu.assemble(dv, project=project)
            pr.orc.assemble(dv, project=project)
            G = pr.gpu.level_matrix(0)
            bo, co = pr.orc.level_matrix(0)
            assert np.array_equal(G["cols"], co)
            assert rel_err(G["blocks"], bo) < 1e-10, project
            assert _sym_err(G) == 0.0


@pytest.mark.parametrize("plasticity", [None, {"kind": "von_mises", "yield_stress": 2.0e3}])
def test_inverted_particles_steps(plasticity):
    """Steps with 3% of the particles inverted (short steps, so the solve stays well
    conditioned): x, v, F per element against the oracle over 3 steps, and the von Mises map's
    skip of inverted particles (transfer.hpp:107-110) with the same inversion counts."""
    pr = _inverted_block(np.random.default_rng(34), 0.03, 5000, plasticity)
    sc = pr.sc
    for k in range(3):
        frame_end = (k + 1) / sc.fps
        s = pr.gpu.advance_step(frame_end)
        so = pr.orc.advance_step(frame_end)
        assert s["node_count"] == so["node_count"]
        assert abs(s["outer_iterations"] - so["outer_iterations"]) <= 1, (k, s, so)
        gp, op = pr.gpu.particles(), pr.orc.get_particles()
        for key in ("x", "v", "F"):
            assert elem_rel_err(gp[key], op[key]) < STATE_TOL, (k, key)
    assert (np.linalg.det(pr.gpu.particles()["F"]) < 0).any()  # still inverted somewhere
    g_inv = pr.gpu.time_state()["inversions"]
    assert g_inv == pr.orc.sim_state()["inversions"] and g_inv > 0
