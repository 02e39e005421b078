"""Restates /root/reference/proj/tests/test_objective.cpp against the CPU oracle (2D + 3D)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import dense_from_bsm, random_block

MAT = dict(density=1000.0, youngs=5e4, poisson=0.3)


def make_scene(rng, cells, f_spread, dt=0.01, gravity=None, with_dirichlet=False, dim=2, dx=0.02, v_spread=0.3,
               mats=(MAT,), f_center=1.0, zero_v=False):
    """test_objective.cpp:22-43"""
    gravity = [0.0] * dim if gravity is None else gravity
    ps = random_block(rng, dx, cells, dim, f_spread=f_spread, v_spread=v_spread, f_center=f_center)
    if zero_v:
        ps["v"][:] = 0
    orc = O.Oracle(dim)
    orc.set_env(gravity, dx)
    orc.set_materials(list(mats))
    orc.set_particles(ps["x"], ps["v"], ps["mass"], ps["volume"], ps["F"].reshape(-1), ps["C"].reshape(-1),
                      ps["material"])
    orc.activate()
    orc.p2g()
    if with_dirichlet:
        g = orc.grid()
        dirm = (g["coords"][:, 0] <= 0).astype(np.uint8)
        vel = g["velocity"].reshape(-1, dim).copy()
        vel[dirm == 1] = 0
        orc.set_grid(velocity=vel.reshape(-1), dirichlet=dirm, bc_velocity=np.zeros(vel.size))
    orc.make_state(dt)
    return orc, ps


def random_dv(rng, orc, scale):
    n, d = orc.node_count(), orc.dim
    dv = rng.uniform(-scale, scale, n * d)
    dirm = orc.grid()["dirichlet"]
    dv.reshape(-1, d)[dirm == 1] = 0
    return dv


def reference_energy(orc, ps, mat, dt, gravity, dv, dx):
    """oracles.hpp:149-178 straight-line re-evaluation in numpy."""
    d = orc.dim
    g = orc.grid()
    index = {tuple(c): i for i, c in enumerate(g["coords"])}
    vel = g["velocity"].reshape(-1, d)
    dvv = dv.reshape(-1, d)
    e = 0.0
    for p in range(ps["x"].shape[0]):
        x = ps["x"][p]
        base = np.floor(x / dx + 0.5).astype(int) - 1
        G = np.zeros((d, d))
        for off in np.ndindex(*(3,) * d):
            node = base + np.array(off)
            i = index.get(tuple(node))
            if i is None:
                continue
            o = x / dx - node
            if O.kernel_weight(O.QUADRATIC, o) <= 0:
                continue
            G += np.outer(vel[i] + dvv[i], O.kernel_gradient(O.QUADRATIC, o, dx))
        Fv = (np.eye(d) + dt * G) @ ps["F"][p]
        e += ps["volume"][p] * O.fcr_energy_density(Fv, mat)
    for i in range(g["mass"].size):
        e += 0.5 * g["mass"][i] * dvv[i] @ dvv[i]
        e -= dt * g["mass"][i] * np.dot(gravity, vel[i] + dvv[i])
    return e


def test_energy_trivial():  # :429-455
    rng = np.random.default_rng(21)
    orc, _ = make_scene(rng, 4, 0.0, zero_v=True)
    n = orc.node_count() * 2
    assert orc.energy(np.zeros(n)) == pytest.approx(0.0, abs=1e-12)
    u = np.array([0.37, -0.81])
    dv = np.tile(u, n // 2)
    kinetic = 0.5 * orc.grid()["mass"].sum() * (u @ u)
    assert orc.energy(dv) == pytest.approx(kinetic, rel=1e-12)
    dv[0] = np.inf
    with pytest.raises(O.OracleError) as e:
        orc.energy(dv)
    assert e.value.kind == "invalid_argument"


@pytest.mark.parametrize("dim", [2, 3])
def test_energy_matches_straight_line(dim):  # :457-468
    rng = np.random.default_rng(22)
    grav = [0.0, -9.8] + ([0.0] if dim == 3 else [])
    cells = 4 if dim == 2 else 2
    orc, ps = make_scene(rng, cells, 0.25, 0.008, grav, dim=dim)
    for _ in range(5 if dim == 2 else 2):
        dv = random_dv(rng, orc, 0.4)
        assert orc.energy(dv) == pytest.approx(reference_energy(orc, ps, MAT, 0.008, grav, dv, 0.02), rel=1e-12)


def test_gradient_uniform_rest():  # :470-483
    rng = np.random.default_rng(23)
    orc, _ = make_scene(rng, 4, 0.0, zero_v=True)
    m = orc.grid()["mass"]
    u = np.array([0.5, 0.25])
    g = orc.gradient(np.tile(u, m.size)).reshape(-1, 2)
    assert np.all(np.linalg.norm(g - m[:, None] * u, axis=1) < 1e-12)


def fd_gradient(f, x, h):
    g = np.zeros_like(x)
    for i in range(x.size):
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        g[i] = (f(xp) - f(xm)) / (2 * h)
    return g


@pytest.mark.parametrize("dim", [2, 3])
def test_gradient_fd(dim):  # :485-503
    rng = np.random.default_rng(24)
    grav = [0.0, -9.8] + ([0.0] if dim == 3 else [])
    for trial in range(3 if dim == 2 else 1):
        orc, _ = make_scene(rng, 3 if dim == 2 else 2, 0.2, 0.01, grav, with_dirichlet=(trial == 2 or dim == 3), dim=dim)
        dv = random_dv(rng, orc, 0.3)
        g = orc.gradient(dv)
        gfd = fd_gradient(orc.energy, dv, 1e-5)
        dirm = orc.grid()["dirichlet"]
        gg, ff = g.reshape(-1, dim), gfd.reshape(-1, dim)
        assert np.all(gg[dirm == 1] == 0.0)
        err = np.abs(gg[dirm == 0] - ff[dirm == 0]).max()
        assert err / np.abs(g).max() < 1e-5


def _hess_fd_check(orc, dv, H, rng, dim):
    for _ in range(5):
        u = rng.uniform(-1, 1, dv.size)
        h = 1e-6
        fd = (orc.gradient(dv + h * u) - orc.gradient(dv - h * u)) / (2 * h)
        Hu = H @ u
        assert np.abs(Hu - fd).max() / max(1.0, np.abs(Hu).max()) < 1e-4


@pytest.mark.parametrize("dim", [2, 3])
def test_hessian_fd(dim):  # :505-552
    rng = np.random.default_rng(25)
    orc, _ = make_scene(rng, 3 if dim == 2 else 2, 0.3, dim=dim)
    dv = random_dv(rng, orc, 0.2)
    orc.assemble(dv, project=False)
    H = dense_from_bsm(*orc.level_matrix(0))
    _hess_fd_check(orc, dv, H, rng, dim)
    # projected Hessian on a stretch-dominant state where projection is inert
    orc, _ = make_scene(rng, 3 if dim == 2 else 2, 0.04, 0.002, f_center=1.08, v_spread=0.01, dim=dim)
    dv = random_dv(rng, orc, 0.01)
    orc.assemble(dv, project=True)
    _hess_fd_check(orc, dv, dense_from_bsm(*orc.level_matrix(0)), rng, dim)


def symmetry_error(blocks, cols, radius=2):
    rows, slots, d, _ = blocks.shape
    w = 2 * radius + 1
    dim = int(round(np.log(slots) / np.log(w)))
    err = 0.0
    for r in range(rows):
        for s in range(slots):
            c = cols[r, s]
            if c < 0:
                continue
            sT = slots - 1 - s  # negated offset in lexicographic slot order
            err = max(err, np.abs(blocks[r, s] - blocks[c, sT].T).max())
    return err


@pytest.mark.parametrize("dim", [2, 3])
def test_hessian_symmetric_psd(dim):  # :554-565
    rng = np.random.default_rng(26)
    orc, _ = make_scene(rng, 3 if dim == 2 else 2, 0.45, dim=dim)
    dv = random_dv(rng, orc, 0.2)
    orc.assemble(dv, project=True)
    blocks, cols = orc.level_matrix(0)
    assert symmetry_error(blocks, cols) == 0.0
    nnz = ((cols >= 0) & (np.abs(blocks).max(axis=(2, 3)) != 0)).sum(1)
    assert nnz.max() <= 5 ** dim
    if dim == 2:
        assert nnz.max() <= 25
    A = dense_from_bsm(blocks, cols)
    assert np.linalg.eigvalsh(A).min() >= -1e-8 * np.linalg.norm(A)


def test_hessian_empty_region_mass_diagonal():  # :567-600
    rng = np.random.default_rng(27)
    dx = 0.02
    ps = random_block(rng, dx, 2, 2, f_spread=0.0, v_spread=0.0)
    far_x = ps["x"].copy()
    far_x[:, 0] += 1.0
    allx = np.vstack([ps["x"], far_x])
    n = allx.shape[0]
    orc = O.Oracle(2)
    orc.set_env([0.0, 0.0], dx)
    orc.set_materials([MAT])
    orc.set_particles(allx, np.zeros((n, 2)), np.tile(ps["mass"], 2), np.tile(ps["volume"], 2))
    orc.activate()
    orc.p2g()
    g = orc.grid()
    # the objective state sees only the near cluster
    orc.set_particles(ps["x"], np.zeros_like(ps["x"]), ps["mass"], ps["volume"])
    orc.make_state(0.01)
    orc.assemble(np.zeros(g["mass"].size * 2))
    blocks, _ = orc.level_matrix(0)
    checked = 0
    for i in range(g["mass"].size):
        if g["coords"][i, 0] * dx < 0.5:
            continue
        for s in range(25):
            if s == 12:
                assert np.linalg.norm(blocks[i, s] - g["mass"][i] * np.eye(2)) == 0.0
            else:
                assert np.linalg.norm(blocks[i, s]) == 0.0
        checked += 1
    assert checked > 0


def test_translation_invariance():  # :630-666
    rng = np.random.default_rng(29)
    orc, _ = make_scene(rng, 3, 0.25)
    m = orc.grid()["mass"]
    dv = random_dv(rng, orc, 0.2)
    sh = dv + np.tile([0.173, -0.244], m.size)

    def inertia(v):
        return 0.5 * (m * (v.reshape(-1, 2) ** 2).sum(1)).sum()

    assert orc.energy(dv) - inertia(dv) == pytest.approx(orc.energy(sh) - inertia(sh), rel=1e-10)
    ga, gb = orc.gradient(dv), orc.gradient(sh)
    fa = ga.reshape(-1, 2) - m[:, None] * dv.reshape(-1, 2)
    fb = gb.reshape(-1, 2) - m[:, None] * sh.reshape(-1, 2)
    assert np.abs(fa - fb).max() < 1e-10 * max(1.0, np.abs(ga).max())
    orc.assemble(dv)
    Ha = orc.level_matrix(0)[0]
    orc.assemble(sh)
    Hb = orc.level_matrix(0)[0]
    assert np.abs(Ha - Hb).max() < 1e-10 * np.linalg.norm(dense_from_bsm(Ha, orc.level_matrix(0)[1]))


def test_dirichlet_dofs_untouched_by_pcg():  # :668-691
    rng = np.random.default_rng(30)
    orc, _ = make_scene(rng, 3, 0.2, 0.01, [0.0, -9.8], with_dirichlet=True)
    n = orc.node_count()
    orc.assemble(np.zeros(2 * n))
    A = dense_from_bsm(*orc.level_matrix(0))
    g = orc.gradient(np.zeros(2 * n))
    Dinv = [np.linalg.inv(A[2 * i:2 * i + 2, 2 * i:2 * i + 2]) for i in range(n)]

    def jac(r):
        return np.concatenate([Dinv[i] @ r[2 * i:2 * i + 2] for i in range(n)])

    x, _, _ = O.pcg(lambda v: A @ v, jac, -g, 1e-10, 10000)
    dirm = orc.grid()["dirichlet"]
    assert dirm.sum() > 0
    assert np.all(x.reshape(-1, 2)[dirm == 1] == 0.0)


def test_node_cn():  # :693-754
    rng = np.random.default_rng(31)
    dx, dt = 0.01, 0.004
    orc, _ = make_scene(rng, 4, 0.1, dt, dx=dx, v_spread=0.2)
    xi, scale = orc.node_cn()
    ell = 24 * dx * dx
    assert ell == pytest.approx(2.4e-3)
    x0 = O.stiffness_scale(MAT, 2)
    assert np.allclose(xi, x0, rtol=1e-12)
    assert np.allclose(scale, ell * x0 * dt, rtol=1e-12)
    g = orc.gradient(random_dv(rng, orc, 0.1))
    assert orc.scaled_norm(g) == pytest.approx(np.linalg.norm(g) / (ell * x0 * dt), rel=1e-12)
    assert orc.scaled_norm(np.zeros_like(g)) == 0.0
    assert orc.scaled_norm(2 * g) == pytest.approx(2 * orc.scaled_norm(g), rel=1e-12)
    # two-material interface
    mats = (dict(density=1000.0, youngs=1e5, poisson=0.3), dict(density=1000.0, youngs=1e7, poisson=0.3))
    ps = random_block(rng, dx, 6, 2, f_spread=0.0, v_spread=0.0)
    ps["material"] = (ps["x"][:, 0] > 3 * dx).astype(np.int32)
    o2 = O.Oracle(2)
    o2.set_env([0.0, 0.0], dx)
    o2.set_materials(list(mats))
    o2.set_particles(ps["x"], ps["v"], ps["mass"], ps["volume"], None, None, ps["material"])
    o2.activate()
    o2.p2g()
    o2.make_state(0.004)
    xi, _ = o2.node_cn()
    a, b = O.stiffness_scale(mats[0], 2), O.stiffness_scale(mats[1], 2)
    assert np.all(xi >= a * (1 - 1e-12)) and np.all(xi <= b * (1 + 1e-12))
    assert np.any((xi > 1.0001 * a) & (xi < 0.9999 * b))
