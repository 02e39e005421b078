"""Restates /root/reference/proj/tests/test_multigrid.cpp against the CPU oracle (2D + 3D)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import dense_from_bsm, dense_restriction, random_block
from tests.test_oracle_objective import symmetry_error

MAT = dict(density=1000.0, youngs=5e4, poisson=0.3)


def make_setup(rng, cells, with_dirichlet, youngs=5e4, dt=0.01, dim=2):
    """test_multigrid.cpp:22-42"""
    dx = 0.02
    ps = random_block(rng, dx, cells, dim, f_spread=0.15, v_spread=0.2)
    orc = O.Oracle(dim)
    orc.set_env([0.0] * dim, dx)
    orc.set_materials([dict(density=1000.0, youngs=youngs, poisson=0.3)])
    orc.set_particles(ps["x"], ps["v"], ps["mass"], ps["volume"], ps["F"].reshape(-1))
    orc.activate()
    orc.p2g()
    if with_dirichlet:
        g = orc.grid()
        orc.set_grid(dirichlet=(g["coords"][:, 0] <= 0).astype(np.uint8))
    orc.make_state(dt)
    orc.assemble()
    return orc


@pytest.mark.parametrize("dim", [2, 3])
def test_restriction_rows_and_dirichlet_image(dim):  # :92-108
    rng = np.random.default_rng(41)
    orc = make_setup(rng, 6 if dim == 2 else 3, True, dim=dim)
    for kind in (O.LINEAR, O.QUADRATIC):
        orc.build_hierarchy(2, kind)
        rs, co, w = orc.level_restriction(0)
        sums = np.add.reduceat(w, rs[:-1])
        assert np.allclose(sums, 1.0, rtol=1e-12)
        cdir = orc.level_info(1)["dirichlet"]
        fdir = orc.level_info(0)["dirichlet"]
        for i in np.nonzero(fdir)[0]:
            assert np.all(cdir[co[rs[i]:rs[i + 1]]] == 1)
        assert np.diff(rs).max() <= 3 ** dim


def test_embedding_weights():  # :63-90 via a two-node fine grid (4,6),(5,6)
    orc = O.Oracle(2)
    orc.set_env([0.0, 0.0], 1.0)
    orc.set_materials([MAT])
    # two particles whose quadratic stencils activate the required fine nodes is awkward;
    # check the 1D embedding rule directly through a one-particle grid instead.
    orc.set_particles(np.array([[4.0, 6.0]]), None, np.array([1.0]), np.array([1.0]))
    orc.activate()
    orc.p2g()
    orc.make_state(0.01)
    orc.assemble()
    orc.build_hierarchy(2, O.LINEAR)
    rs, co, w = orc.level_restriction(0)
    fine = orc.level_info(0)["coords"]
    coarse = orc.level_info(1)["coords"]
    for i, c in enumerate(fine):
        ents = list(zip(co[rs[i]:rs[i + 1]], w[rs[i]:rs[i + 1]]))
        npar = 1
        for a in range(2):
            npar *= 1 if c[a] % 2 == 0 else 2
        assert len(ents) == npar
        for j, wt in ents:
            expect = 1.0
            for a in range(2):
                expect *= 1.0 if c[a] % 2 == 0 else 0.5
                assert coarse[j][a] in (c[a] // 2, c[a] // 2 + 1)
            assert wt == expect
    orc.build_hierarchy(2, O.QUADRATIC)
    rs, co, w = orc.level_restriction(0)
    for i, c in enumerate(fine):
        cnt = 1
        for a in range(2):
            cnt *= 3 if c[a] % 2 == 0 else 2
        assert rs[i + 1] - rs[i] == cnt
        assert w[rs[i]:rs[i + 1]].sum() == pytest.approx(1.0, rel=1e-14)


@pytest.mark.parametrize("dim", [2, 3])
def test_galerkin_dense_triple_product(dim):  # :110-147
    rng = np.random.default_rng(42)
    for with_dir in (False, True):
        orc = make_setup(rng, 4 if dim == 2 else 2, with_dir, dim=dim)
        H0 = dense_from_bsm(*orc.level_matrix(0))
        for kind in (O.LINEAR, O.QUADRATIC):
            orc.build_hierarchy(2, kind)
            rs, co, w = orc.level_restriction(0)
            nc = orc.level_shape(1)[0]
            R = dense_restriction(rs, co, w, nc, dim)
            expect = R @ H0 @ R.T
            cdir = orc.level_info(1)["dirichlet"]
            for i in np.nonzero(cdir)[0]:
                expect[dim * i:dim * i + dim, :] = 0
                expect[:, dim * i:dim * i + dim] = 0
                expect[dim * i:dim * i + dim, dim * i:dim * i + dim] = np.eye(dim)
            blocks, cols = orc.level_matrix(1)
            got = dense_from_bsm(blocks, cols)
            assert np.linalg.norm(got - expect) <= 1e-12 * np.linalg.norm(expect)
            assert symmetry_error(blocks, cols, 2 if kind == O.LINEAR else 3) == 0.0
            assert np.linalg.eigvalsh(got).min() >= -1e-10 * np.linalg.norm(got)
            assert orc.level_shape(1)[2] == (2 if kind == O.LINEAR else 3)


@pytest.mark.parametrize("dim", [2, 3])
def test_build_hierarchy(dim):  # :157-200
    rng = np.random.default_rng(44)
    orc = make_setup(rng, 8 if dim == 2 else 4, True, dim=dim)
    assert orc.build_hierarchy(3, O.LINEAR) == 3
    sizes = [orc.level_shape(m)[0] for m in range(3)]
    assert sizes[0] > sizes[1] > sizes[2]
    means = []
    for m in range(3):
        b, c = orc.level_matrix(m)
        nnz = ((c >= 0) & (np.abs(b).max(axis=(2, 3)) != 0)).sum(1)
        means.append(nnz.mean())
        if m == 0 and dim == 2:
            assert nnz.max() <= 25
    assert means[1] <= means[0] + 1e-12 and means[2] <= means[1] + 1e-12
    assert orc.build_hierarchy(1, O.LINEAR) == 1


def _sweep_order_expect(coords, q):
    col = np.zeros(len(coords), dtype=np.int64)
    for a in range(coords.shape[1]):
        col = col * q + (coords[:, a] % q)
    return np.argsort(col, kind="stable")


@pytest.mark.parametrize("dim", [2, 3])
def test_sweep_order_colours(dim):  # multigrid.hpp:242-250 colour rule
    rng = np.random.default_rng(49)
    orc = make_setup(rng, 6 if dim == 2 else 3, True, dim=dim)
    orc.build_hierarchy(3, O.LINEAR)
    for m, q in ((0, 3), (1, 2), (2, 2)):
        info = orc.level_info(m)
        assert np.array_equal(info["sweep_order"], _sweep_order_expect(info["coords"], q))


def test_smooth_sgs():  # :202-255 (level 0)
    rng = np.random.default_rng(45)
    orc = make_setup(rng, 3, False)
    orc.build_hierarchy(1, O.LINEAR)
    blocks, cols = orc.level_matrix(0)
    A = dense_from_bsm(blocks, cols)
    n = A.shape[0]
    ustar = rng.uniform(-1, 1, n)
    u = orc.smooth_sgs(0, ustar, A @ ustar)
    assert np.abs(u - ustar).max() < 1e-12 * np.abs(ustar).max()
    b = rng.uniform(-1, 1, n)
    exact = np.linalg.solve(A, b)
    u = np.zeros(n)
    prev = np.inf
    for _ in range(10):
        u = orc.smooth_sgs(0, u, b)
        e = u - exact
        an = np.sqrt(e @ A @ e)
        assert an <= prev * (1 + 1e-12)
        prev = an
    # diagonal system solved in one sweep
    D = np.zeros_like(blocks)
    for r in range(blocks.shape[0]):
        D[r, 12] = (2.0 + r % 5) * np.eye(2)
    orc.set_level_matrix(0, D)
    orc.refinalize_level(0, 3)
    u = orc.smooth_sgs(0, np.zeros(n), b)
    assert np.abs(u - np.linalg.solve(dense_from_bsm(D, cols), b)).max() < 1e-12
    # singular diagonal block rejected
    orc.set_level_matrix(0, np.zeros_like(blocks))
    with pytest.raises(O.OracleError) as e:
        orc.build_hierarchy(1, O.LINEAR)
    assert e.value.kind == "logic_error"


def test_coarse_solve():  # :257-296
    rng = np.random.default_rng(46)
    orc = make_setup(rng, 3, False)
    orc.build_hierarchy(1, O.LINEAR)
    n = orc.level_shape(0)[0] * 2
    u, it = orc.coarse_solve(0, np.zeros(n))
    assert np.linalg.norm(u) == 0.0 and it == 0
    b = rng.uniform(-1, 1, n)
    u1, i1 = orc.coarse_solve(0, b)
    u8, i8 = orc.coarse_solve(0, 8 * b)
    assert i8 == i1 and np.linalg.norm(u8 - 8 * u1) == 0.0
    u10, i10 = orc.coarse_solve(0, 10 * b)
    assert i10 == i1 and np.linalg.norm(u10 - 10 * u1) <= 1e-12 * np.linalg.norm(u10)
    blocks, cols = orc.level_matrix(0)
    D = np.zeros_like(blocks)
    for r in range(blocks.shape[0]):
        D[r, 12] = (1.0 + r % 3) * np.eye(2)
    orc.set_level_matrix(0, D)
    orc.refinalize_level(0, 3)
    _, it = orc.coarse_solve(0, b)
    assert it == 1


@pytest.mark.parametrize("dim", [2, 3])
def test_vcycle(dim):  # :298-363
    rng = np.random.default_rng(47)
    orc = make_setup(rng, 6 if dim == 2 else 3, True, 1e6, dim=dim)
    A = dense_from_bsm(*orc.level_matrix(0))
    n = A.shape[0]
    dirm = orc.grid()["dirichlet"]
    orc.build_hierarchy(3, O.LINEAR)
    u, _ = orc.vcycle(np.zeros(n))
    assert np.linalg.norm(u) == 0.0
    b = rng.uniform(-1, 1, n)
    b.reshape(-1, dim)[dirm == 1] = 0
    exact = np.linalg.solve(A, b)
    u, _ = orc.vcycle(b)
    e = u - exact
    assert np.sqrt(e @ A @ e) < np.sqrt(exact @ A @ exact)
    assert np.all(np.linalg.norm(u.reshape(-1, dim)[dirm == 1], axis=1) == 0.0)
    # single level degenerates to coarse_solve, bitwise
    orc.build_hierarchy(1, O.LINEAR)
    v, vi = orc.vcycle(b)
    c, ci = orc.coarse_solve(0, b)
    assert np.array_equal(v, c) and vi == ci


def test_pinned_vcycle_symmetric_pd():  # :340-362
    rng = np.random.default_rng(48)
    orc = make_setup(rng, 5, True, 1e6)
    orc.build_hierarchy(3, O.LINEAR)
    n = orc.level_shape(0)[0] * 2
    assert n <= 300
    V = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        V[:, j] = orc.vcycle(e, pinned=True, pinned_cap=4 * n)[0]
    assert np.linalg.norm(V - V.T) <= 1e-8 * np.linalg.norm(V)
    free = np.repeat(orc.grid()["dirichlet"] == 0, 2)
    Vff = V[np.ix_(free, free)]
    assert np.linalg.eigvalsh(0.5 * (Vff + Vff.T)).min() > 0


def test_quadratic_wider_than_linear():  # :365-374
    rng = np.random.default_rng(48)
    orc = make_setup(rng, 6, False)

    def maxnnz():
        b, c = orc.level_matrix(1)
        return ((c >= 0) & (np.abs(b).max(axis=(2, 3)) != 0)).sum(1).max()

    orc.build_hierarchy(2, O.LINEAR)
    lin, rl = maxnnz(), orc.level_shape(1)[2]
    orc.build_hierarchy(2, O.QUADRATIC)
    quad, rq = maxnnz(), orc.level_shape(1)[2]
    assert lin <= quad and rl == 2 and rq == 3


def numpy_vcycle(orc, b0, dim, pinned=False, pinned_cap=256, cap=10000):
    """Independent numpy restatement of multigrid.hpp:298-392 + pcg.hpp:17-46 over the
    oracle's exported levels; pins the C++ restatement's V-cycle semantics."""
    M = orc.level_count()
    Hs, infos, Rs = [], [], []
    for m in range(M):
        Hs.append(dense_from_bsm(*orc.level_matrix(m)))
        infos.append(orc.level_info(m))
        if m + 1 < M:
            rs, co, w = orc.level_restriction(m)
            Rs.append(dense_restriction(rs, co, w, orc.level_shape(m + 1)[0], dim))

    def sgs(A, info, u, b):
        n = A.shape[0] // dim
        Dinv = info["diag_inv"]
        order = list(info["sweep_order"])
        for i in order + order[::-1]:
            r = b[dim * i:dim * i + dim] - A[dim * i:dim * i + dim] @ u
            u[dim * i:dim * i + dim] += Dinv[i] @ r
        return u

    def zero_dir(m, x):
        x.reshape(-1, dim)[infos[m]["dirichlet"] == 1] = 0

    def pcg(A, Dinv, b, rel, iters):
        n = b.size // dim
        P = lambda r: np.concatenate([Dinv[i] @ r[dim * i:dim * i + dim] for i in range(n)])
        x = np.zeros_like(b)
        r = b.copy()
        z = P(r)
        rho = r @ z
        if not rho > 0:
            return x, 0
        thr = rel * rel * rho
        p = z.copy()
        for it in range(iters):
            Ap = A @ p
            alpha = rho / (p @ Ap)
            x += alpha * p
            r -= alpha * Ap
            z = P(r)
            rn = r @ z
            if rn <= thr:
                return x, it + 1
            p = z + (rn / rho) * p
            rho = rn
        return x, iters

    b = [None] * M
    u = [None] * M
    b[0] = b0.copy()
    zero_dir(0, b[0])
    for m in range(M - 1):
        u[m] = sgs(Hs[m], infos[m], np.zeros_like(b[m]), b[m])
        b[m + 1] = Rs[m] @ (b[m] - Hs[m] @ u[m])
        zero_dir(m + 1, b[m + 1])
    rel, iters = (1e-14, pinned_cap) if pinned else (0.5, cap)
    u[M - 1], its = pcg(Hs[M - 1], infos[M - 1]["diag_inv"], b[M - 1], rel, iters)
    for m in range(M - 2, -1, -1):
        u[m] = u[m] + Rs[m].T @ u[m + 1]
        u[m] = sgs(Hs[m], infos[m], u[m], b[m])
    return u[0], its


@pytest.mark.parametrize("dim", [2, 3])
def test_vcycle_matches_numpy_restatement(dim):
    rng = np.random.default_rng(50)
    orc = make_setup(rng, 5 if dim == 2 else 3, True, 1e6, dim=dim)
    orc.build_hierarchy(3, O.LINEAR)
    n = orc.level_shape(0)[0] * dim
    for _ in range(3):
        b = rng.uniform(-1, 1, n)
        u, it = orc.vcycle(b)
        un, itn = numpy_vcycle(orc, b, dim)
        assert it == itn
        assert np.abs(u - un).max() <= 1e-10 * np.abs(un).max()
