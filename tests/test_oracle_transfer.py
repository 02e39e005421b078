"""Restates /root/reference/proj/tests/test_transfer.cpp against the CPU oracle."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import random_f

ELASTIC = dict(density=1000.0, youngs=1e5, poisson=0.3)


def random_particles(rng, count, dx, dim):  # test_transfer.cpp:15-31
    x = rng.uniform(0.0, 10 * dx, (count, dim))
    v = rng.uniform(-1.0, 1.0, (count, dim))
    Cm = rng.uniform(-1.0, 1.0, (count, dim, dim))
    mass = 0.3 + np.abs(rng.uniform(-1.0, 1.0, count))
    return dict(x=x, v=v, Cm=Cm, mass=mass, volume=np.full(count, 1e-4))


def setup(ps, dx, dim, F=None):
    orc = O.Oracle(dim)
    orc.set_env([0.0] * dim, dx)
    orc.set_materials([ELASTIC])
    orc.set_particles(ps["x"], ps.get("v"), ps.get("mass"), ps.get("volume"), F, ps.get("Cm"))
    orc.activate()
    return orc


@pytest.mark.parametrize("dim", [2, 3])
def test_p2g_conservation(dim):  # :41-58, :205-229
    rng = np.random.default_rng(11)
    dx = 0.05
    ps = random_particles(rng, 80, dx, dim)
    orc = setup(ps, dx, dim)
    orc.p2g()
    g = orc.grid()
    assert g["mass"].sum() == pytest.approx(ps["mass"].sum(), rel=1e-12)
    mom = (ps["mass"][:, None] * ps["v"]).sum(0)
    gm = g["momentum"].reshape(-1, dim).sum(0)
    assert np.linalg.norm(gm - mom) <= 1e-12 * max(1.0, np.linalg.norm(mom))


def test_single_particle_uniform_velocity():  # :60-75
    ps = dict(x=np.array([[0.121, 0.243]]), v=np.array([[0.4, -0.7]]), mass=np.array([2.0]),
              volume=np.array([1e-4]))
    orc = setup(ps, 0.05, 2)
    orc.p2g()
    g = orc.grid()
    vel = g["velocity"].reshape(-1, 2)
    assert np.all(np.linalg.norm(vel - ps["v"], axis=1) < 1e-13)
    assert (g["mass"] / 2.0).sum() == pytest.approx(1.0, rel=1e-12)


@pytest.mark.parametrize("dim", [2, 3])
def test_g2p_affine(dim):  # :77-104
    rng = np.random.default_rng(12)
    dx = 0.05
    ps = random_particles(rng, 20, dx, dim)
    orc = setup(ps, dx, dim)
    g = orc.grid()
    v = np.arange(1, dim + 1) * 0.3
    orc.set_grid(velocity=np.tile(v, g["mass"].size))
    orc.g2p()
    p = orc.get_particles()
    assert np.all(np.linalg.norm(p["v"] - v, axis=1) < 1e-13)
    assert np.all(np.abs(p["C"]).max(axis=(1, 2)) < 1e-10)
    A = rng.uniform(-1, 1, (dim, dim))
    pos = g["coords"] * dx
    orc.set_grid(velocity=(pos @ A.T).reshape(-1))
    orc.g2p()
    p = orc.get_particles()
    assert np.all(np.linalg.norm(p["v"] - ps["x"] @ A.T, axis=1) < 1e-12)
    assert np.all(np.abs(p["C"] - A).max(axis=(1, 2)) < 1e-10)


def test_rigid_translation_round_trip():  # :106-122
    rng = np.random.default_rng(13)
    dx = 0.04
    ps = random_particles(rng, 50, dx, 2)
    ps["v"][:] = [1.25, -0.5]
    ps["Cm"][:] = 0
    orc = setup(ps, dx, 2)
    orc.p2g()
    orc.g2p()
    p = orc.get_particles()
    assert np.all(np.linalg.norm(p["v"] - [1.25, -0.5], axis=1) < 1e-12)
    assert np.all(np.linalg.norm(p["C"], axis=(1, 2)) < 1e-9)


def test_update_strain():  # :124-181
    dx = 0.05
    rng = np.random.default_rng(14)
    ps = random_particles(rng, 30, dx, 2)
    F = np.array([random_f(rng, 2) for _ in range(30)])
    orc = setup(ps, dx, 2, F=F.reshape(-1))
    assert orc.update_strain(0.01) == 0
    assert np.array_equal(orc.get_particles()["F"], F)
    # uniform translation
    rng = np.random.default_rng(15)
    ps = random_particles(rng, 30, dx, 2)
    orc = setup(ps, dx, 2)
    orc.set_grid(velocity=np.tile([0.7, 0.1], orc.node_count()))
    orc.update_strain(0.01)
    assert np.abs(orc.get_particles()["F"] - np.eye(2)).max() < 1e-13
    # uniaxial stretch
    F0 = np.array([[1.1, 0.2], [-0.1, 0.9]])
    ps = dict(x=np.array([[0.212, 0.157]]), mass=np.array([1.0]), volume=np.array([1e-4]))
    orc = setup(ps, dx, 2, F=F0.reshape(-1))
    pos = orc.grid()["coords"] * dx
    vel = np.zeros_like(pos, dtype=float)
    vel[:, 0] = 0.8 * pos[:, 0]
    orc.set_grid(velocity=vel.reshape(-1))
    orc.update_strain(1e-3)
    expected = np.diag([1 + 0.8e-3, 1.0]) @ F0
    assert np.abs(orc.get_particles()["F"][0] - expected).max() < 1e-10
    # inversion counted and passed through
    ps = dict(x=np.array([[0.2, 0.2]]), mass=np.array([1.0]), volume=np.array([1e-4]))
    orc = setup(ps, dx, 2, F=np.diag([-0.5, 1.0]).reshape(-1))
    assert orc.update_strain(0.01) == 1
    assert orc.get_particles()["F"][0, 0, 0] == pytest.approx(-0.5)


def test_advect():  # :183-203
    ps = dict(x=np.array([[0.5, 0.5]]), v=np.array([[0.0, 0.0]]))
    orc = setup(ps, 0.01, 2)
    orc.advect(0.01)
    assert np.linalg.norm(orc.get_particles()["x"][0] - [0.5, 0.5]) == 0.0
    orc.set_particles(np.array([[0.5, 0.5]]), np.array([[1.0, 0.0]]))
    orc.advect(0.01)
    assert np.linalg.norm(orc.get_particles()["x"][0] - [0.51, 0.5]) < 1e-15
    for vmax in (0.1, 1.0, 10.0, 1000.0):
        assert vmax * O.cfl_dt(vmax, 0.01, 24.0) <= 0.01
