"""Restates /root/reference/proj/tests/test_constitutive.cpp against the CPU oracle."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import random_f, random_rotation


def mat(density, youngs, poisson, **pl):
    m = dict(density=density, youngs=youngs, poisson=poisson)
    if pl:
        m["plasticity"] = pl
    return m


def rot2(a):
    return np.array([[np.cos(a), -np.sin(a)], [np.sin(a), np.cos(a)]])


def fd_stress(F, m, h=1e-6):  # oracles.hpp:59-70
    d = F.shape[0]
    P = np.zeros_like(F)
    for i in range(d):
        for j in range(d):
            Fp, Fm = F.copy(), F.copy()
            Fp[i, j] += h
            Fm[i, j] -= h
            P[i, j] = (O.fcr_energy_density(Fp, m) - O.fcr_energy_density(Fm, m)) / (2 * h)
    return P


def fd_dpdf(F, m, h=1e-6):  # oracles.hpp:73-86
    d = F.shape[0]
    T = np.zeros((d * d, d * d))
    for k in range(d):
        for l in range(d):
            Fp, Fm = F.copy(), F.copy()
            Fp[k, l] += h
            Fm[k, l] -= h
            dP = (O.fcr_stress(Fp, m) - O.fcr_stress(Fm, m)) / (2 * h)
            T[:, k * d + l] = dP.reshape(-1)
    return T


def test_material_derivation():  # :20-27
    mu, la = O.material_lame(mat(1000, 5e4, 0.3))
    assert mu == pytest.approx(5e4 / 2.6)
    assert la == pytest.approx(5e4 * 0.3 / (1.3 * 0.4))
    for bad in (mat(1000, -1, 0.3), mat(1000, 1e5, 0.5), mat(1000, 1e5, 0.3, kind="snow_clamp", lo=1.01, hi=1.02)):
        with pytest.raises(O.OracleError) as e:
            O.material_lame(bad)
        assert e.value.kind == "invalid_argument"


def test_svd_convention():  # constitutive.hpp:66-82 (H3)
    rng = np.random.default_rng(0)
    for d in (2, 3):
        for _ in range(200):
            F = rng.uniform(-1.5, 1.5, (d, d))
            U, s, V = O.svd_rv(F)
            assert np.allclose(U @ np.diag(s) @ V.T, F, atol=1e-13)
            assert np.linalg.det(U) == pytest.approx(1.0, abs=1e-12)
            assert np.linalg.det(V) == pytest.approx(1.0, abs=1e-12)
            assert np.all(np.diff(np.abs(s)) <= 1e-15)  # |sigma| descending
            assert np.all(s[:-1] >= 0)
            assert np.sign(s[-1]) == np.sign(np.linalg.det(F)) or abs(s[-1]) < 1e-300


def test_fcr_energy():  # :29-55
    m = mat(1000, 2.6, 0.3)
    assert O.fcr_energy_density(np.eye(2), m) == pytest.approx(0.0)
    # mu = 1, lambda = 0 via E = 2, nu = 0
    F = np.eye(2)
    F[0, 0] = 2.0
    assert O.fcr_energy_density(F, mat(1000, 2.0, 0.0)) == pytest.approx(1.0)
    assert O.fcr_energy_density(rot2(np.pi / 6), m) == pytest.approx(0.0, abs=1e-12)
    bad = np.eye(2)
    bad[0, 1] = np.nan
    with pytest.raises(O.OracleError):
        O.fcr_energy_density(bad, m)
    rng = np.random.default_rng(1)
    for d in (2, 3):
        for _ in range(50):
            Fr, R = random_f(rng, d), random_rotation(rng, d)
            assert O.fcr_energy_density(R @ Fr, m) == pytest.approx(O.fcr_energy_density(Fr, m), rel=1e-10, abs=1e-14)


def test_fcr_stress_fd():  # :57-75
    m = mat(1000, 9.1e3, 0.3)
    assert np.linalg.norm(O.fcr_stress(np.eye(2), m)) == pytest.approx(0.0)
    assert np.linalg.norm(O.fcr_stress(rot2(0.7), m)) < 1e-10
    rng = np.random.default_rng(2)
    for d, n in ((2, 100), (3, 30)):
        for _ in range(n):
            F = random_f(rng, d)
            P = O.fcr_stress(F, m)
            assert np.linalg.norm(P - fd_stress(F, m)) / max(1.0, np.linalg.norm(P)) < 1e-5


def test_fcr_stress_equivariance():  # :77-94
    m = mat(1000, 7.7e4, 0.35)
    rng = np.random.default_rng(3)
    for d, n, tol in ((2, 50, 1e-10), (3, 20, 1e-9)):
        for _ in range(n):
            F, R = random_f(rng, d), random_rotation(rng, d)
            lhs, rhs = O.fcr_stress(R @ F, m), R @ O.fcr_stress(F, m)
            assert np.max(np.abs(lhs - rhs)) < tol * max(1.0, np.linalg.norm(rhs))


def test_fcr_stress_derivative_fd():  # :96-122
    m = mat(1000, 6.5e3, 0.3)
    T2 = O.fcr_stress_derivative(np.eye(2), m)
    assert np.max(np.abs(T2 - T2.T)) == 0.0
    fd = fd_dpdf(np.eye(2), m)
    assert np.linalg.norm(T2 - fd) / np.linalg.norm(fd) < 1e-6
    rng = np.random.default_rng(4)
    for d, n in ((2, 100), (3, 25)):
        for _ in range(n):
            F = random_f(rng, d)
            Tn = O.fcr_stress_derivative(F, m)
            fd = fd_dpdf(F, m)
            assert np.linalg.norm(Tn - fd) / max(1.0, np.linalg.norm(fd)) < 1e-4
            assert np.max(np.abs(Tn - Tn.T)) == 0.0


def test_project_spd():  # :124-152
    assert np.linalg.norm(O.project_spd(np.eye(4)) - np.eye(4)) == 0.0
    Dp = O.project_spd(np.diag([1.0, -2.0, 3.0, -0.5]))
    assert Dp[0, 0] == pytest.approx(1.0)
    assert Dp[1, 1] == pytest.approx(0.0, abs=1e-12)
    assert Dp[2, 2] == pytest.approx(3.0)
    assert Dp[3, 3] == pytest.approx(0.0, abs=1e-12)
    asym = np.zeros((4, 4))
    asym[0, 1] = 1.0
    with pytest.raises(O.OracleError) as e:
        O.project_spd(asym)
    assert e.value.kind == "invalid_argument"
    rng = np.random.default_rng(5)
    for n in (4, 9):
        for _ in range(100):
            A = rng.normal(size=(n, n))
            A = 0.5 * (A + A.T)
            Ap = O.project_spd(A)
            assert np.linalg.eigvalsh(Ap).min() >= -1e-10
            App = O.project_spd(Ap)
            assert np.linalg.norm(App - Ap) <= 1e-12 * max(1.0, np.linalg.norm(Ap))
            # eigen-clamp is the nearest PSD matrix: same as numpy clamp
            w, V = np.linalg.eigh(A)
            ref = (V * np.maximum(w, 0)) @ V.T
            assert np.allclose(Ap, ref, atol=1e-12 * max(1.0, np.abs(A).max()))


def _dev(F):
    _, s, _ = O.svd_rv(F)
    eps = np.log(s)
    return eps, eps - eps.mean()


def test_return_map_von_mises():  # :154-215
    m = mat(1000, 1e5, 0.3, kind="von_mises", yield_stress=50.0)
    mu, _ = O.material_lame(m)
    assert np.linalg.norm(O.return_map(np.eye(2), m) - np.eye(2)) == 0.0
    F = np.diag([1.0005, 0.9996])
    assert np.linalg.norm(O.return_map(F, m) - F) == 0.0
    rng = np.random.default_rng(6)
    for d in (2, 3):
        for _ in range(40):
            F = random_f(rng, d, 0.5, 2.0)
            Fn = O.return_map(F, m)
            eps, dev = _dev(Fn)
            eps0, dev0 = _dev(F)
            if 2 * mu * np.linalg.norm(dev0) <= 50.0:
                assert np.linalg.norm(Fn - F) == 0.0
                continue
            assert 2 * mu * np.linalg.norm(dev) == pytest.approx(50.0, rel=1e-6)
            assert eps.sum() == pytest.approx(eps0.sum(), rel=1e-9, abs=1e-12)
            direc = dev0 / np.linalg.norm(dev0)
            lo, hi = 0.0, np.linalg.norm(dev0)
            for _ in range(200):
                mid = 0.5 * (lo + hi)
                if 2 * mu * np.linalg.norm(dev0 - mid * direc) > 50.0:
                    lo = mid
                else:
                    hi = mid
            assert np.linalg.norm(dev - (dev0 - 0.5 * (lo + hi) * direc)) < 1e-8 * max(1.0, np.linalg.norm(dev0))
            F2 = O.return_map(Fn, m)
            assert np.linalg.norm(F2 - Fn) <= 1e-12 * max(1.0, np.linalg.norm(Fn))
    with pytest.raises(O.OracleError) as e:
        O.return_map(np.diag([-1.0, 1.0]), m)
    assert e.value.kind == "domain_error"


def test_return_map_snow():  # :217-243
    m = mat(400, 1.4e5, 0.2, kind="snow_clamp", lo=0.99, hi=1.001)
    F = np.diag([1.05, 0.9])
    Fn = O.return_map(F, m)
    assert Fn[0, 0] == pytest.approx(1.001)
    assert Fn[1, 1] == pytest.approx(0.99)
    assert abs(Fn[0, 1]) < 1e-14
    R = rot2(0.4)
    assert np.linalg.norm(O.return_map(R @ F, m) - R @ Fn) < 1e-12
    rng = np.random.default_rng(8)
    for d in (2, 3):
        for _ in range(40):
            F = random_f(rng, d, 0.5, 2.0)
            F1 = O.return_map(F, m)
            assert np.linalg.norm(O.return_map(F1, m) - F1) <= 1e-12


def test_stiffness_scale():  # :245-260
    a, b, c = mat(1000, 1e5, 0.4), mat(1000, 1e6, 0.4), mat(1000, 1e9, 0.4)
    for d in (2, 3):
        xa = O.stiffness_scale(a, d)
        assert O.stiffness_scale(b, d) / xa == pytest.approx(10.0, rel=1e-12)
        assert O.stiffness_scale(c, d) / xa == pytest.approx(1e4, rel=1e-12)
        assert xa > 0
    mu_only = mat(1000, 2.0, 0.0)
    fd = fd_dpdf(np.eye(2), mu_only)
    assert O.stiffness_scale(mu_only, 2) == pytest.approx(np.linalg.norm(fd), rel=1e-6)


def test_energy_stress_chain():  # :262-274
    m = mat(1200, 3.3e4, 0.42)
    rng = np.random.default_rng(9)
    for _ in range(100):
        F = random_f(rng, 2)
        P = O.fcr_stress(F, m)
        Pfd = fd_stress(F, m)
        assert np.linalg.norm(P - Pfd) / max(1.0, np.linalg.norm(Pfd)) < 1e-4
        Tn, Tfd = O.fcr_stress_derivative(F, m), fd_dpdf(F, m)
        assert np.linalg.norm(Tn - Tfd) / max(1.0, np.linalg.norm(Tfd)) < 1e-4


def test_projected_dpdf_psd_3d():
    """Projected dP/dF (constitutive.hpp:203-219 applied at objective.hpp:298) is PSD."""
    m = mat(1000, 1e5, 0.3)
    rng = np.random.default_rng(10)
    for _ in range(50):
        F = random_f(rng, 3)
        T = O.fcr_stress_derivative(F, m, project=True)
        assert np.linalg.eigvalsh(T).min() >= -1e-9 * np.abs(T).max()
