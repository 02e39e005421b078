"""Restates /root/reference/proj/tests/test_grid_kernels.cpp against the CPU oracle (2D + 3D)."""
import itertools

import numpy as np
import pytest

from oracle import oracle as O

Q, L = O.QUADRATIC, O.LINEAR


def test_kernel_weight_values():  # test_grid_kernels.cpp:9-16
    assert O.kernel_weight(Q, [0.0, 0.0]) == pytest.approx(0.5625, rel=1e-14)
    assert O.kernel_weight(Q, [0.0, 0.0, 0.0]) == pytest.approx(0.75 ** 3, rel=1e-14)
    assert O.kernel_weight_1d(L, 0.5) == pytest.approx(0.5)
    assert O.kernel_weight_1d(Q, 1.5) == 0.0
    assert O.kernel_weight_1d(Q, -1.7) == 0.0
    assert O.kernel_weight_1d(L, 1.0) == 0.0


@pytest.mark.parametrize("dim", [2, 3])
def test_kernel_gradient_fd(dim):  # test_grid_kernels.cpp:18-50
    assert O.kernel_derivative_1d(Q, 0.0) == 0.0
    assert O.kernel_gradient(L, [0.25], 1.0)[0] == pytest.approx(-1.0)
    rng = np.random.default_rng(42)
    h = 1e-6
    for kind in (Q, L):
        for _ in range(200):
            x = rng.uniform(-1.4, 1.4, dim)
            if any(abs(abs(v) - k) < 1e-3 for v in x for k in (0.0, 0.5, 1.0, 1.5)):
                continue
            g = O.kernel_gradient(kind, x, 1.0)
            for a in range(dim):
                xp, xm = x.copy(), x.copy()
                xp[a] += h
                xm[a] -= h
                fd = (O.kernel_weight(kind, xp) - O.kernel_weight(kind, xm)) / (2 * h)
                assert g[a] == pytest.approx(fd, rel=1e-6, abs=1e-9)


@pytest.mark.parametrize("dim", [2, 3])
def test_partition_of_unity(dim):  # test_grid_kernels.cpp:52-75
    rng = np.random.default_rng(7)
    dx = 0.017
    for kind in (Q, L):
        width = 3 if kind == Q else 2
        for _ in range(100):
            x = rng.uniform(-3.0, 3.0, dim)
            base = O.stencil_base(x, dx, kind)
            sw, sg = 0.0, np.zeros(dim)
            for off in itertools.product(range(width), repeat=dim):
                node = base + np.array(off)
                o = x / dx - node
                sw += O.kernel_weight(kind, o)
                sg += O.kernel_gradient(kind, o, dx)
            assert sw == pytest.approx(1.0, rel=1e-12)
            assert np.linalg.norm(sg) < 1e-10


def _grid_of(xs, dx, dim, kind=Q):
    orc = O.Oracle(dim)
    orc.set_env([0.0] * dim, dx)
    xs = np.asarray(xs, dtype=float).reshape(-1, dim)
    orc.set_particles(xs)
    n = orc.activate(kind)
    return orc, n


def test_activate_grid_examples():  # test_grid_kernels.cpp:77-116
    dx = 0.1
    _, n = _grid_of([[0.3, 0.5]], dx, 2)
    assert n == 9
    _, n = _grid_of([[0.31, 0.52]], dx, 2, L)
    assert n == 4
    _, n = _grid_of(np.zeros((0, 2)), dx, 2)
    assert n == 0
    _, n = _grid_of([[0.3, 0.5, 0.7]], dx, 3)
    assert n == 27
    xs = np.array([[0.13, 0.27], [1.62, 1.91]])
    orc, n = _grid_of(xs, dx, 2)
    expect = []
    for i in range(-5, 30):
        for j in range(-5, 30):
            for x in xs:
                if O.kernel_weight(Q, x / dx - np.array([i, j])) > 0:
                    expect.append((i, j))
                    break
    got = [tuple(c) for c in orc.grid()["coords"]]
    assert got == expect  # exact and in lexicographic order


def test_activate_grid_brute_force_3d():
    rng = np.random.default_rng(3)
    dx = 0.05
    xs = rng.uniform(0.0, 0.4, (25, 3))
    orc, n = _grid_of(xs, dx, 3)
    expect = set()
    for x in xs:
        c = np.floor(x / dx + 0.5).astype(int) - 1
        for off in itertools.product(range(3), repeat=3):
            node = c + np.array(off)
            if O.kernel_weight(Q, x / dx - node) > 0:
                expect.add(tuple(int(v) for v in node))
    got = [tuple(int(v) for v in c) for c in orc.grid()["coords"]]
    assert got == sorted(expect)


@pytest.mark.parametrize("dim", [2, 3])
def test_activate_grid_order_independent(dim):  # test_grid_kernels.cpp:118-130
    rng = np.random.default_rng(99)
    xs = rng.uniform(0.0, 1.0, (60, dim))
    a, _ = _grid_of(xs, 0.05, dim)
    perm = rng.permutation(len(xs))
    b, _ = _grid_of(xs[perm], 0.05, dim)
    assert np.array_equal(a.grid()["coords"], b.grid()["coords"])


def test_cfl_dt():  # test_grid_kernels.cpp:132-137
    assert O.cfl_dt(0.0, 0.01, 24.0) == pytest.approx(1.0 / 24)
    assert O.cfl_dt(1.2, 0.01, 24.0) == pytest.approx(0.005)
    assert O.cfl_dt(0.1, 0.01, 24.0) == pytest.approx(1.0 / 24)
    assert O.cfl_dt(100.0, 0.01, 24.0) > 0.0


def test_non_finite_position_rejected():  # grid.hpp:147
    orc = O.Oracle(3)
    orc.set_env([0, 0, 0], 0.1)
    orc.set_particles(np.array([[0.1, np.nan, 0.2]]))
    with pytest.raises(O.OracleError) as e:
        orc.activate()
    assert e.value.kind == "invalid_argument"
