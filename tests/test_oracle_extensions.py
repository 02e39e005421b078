"""Constitutive extensions the reference does not have (parity-unpinned against
the reference): Neo-Hookean elasticity (BASELINE configs 2 and 5), Stomakhin snow hardening
(config 4's "hardening 10") and the Drucker-Prager return map (north star).  The oracle's
restatements are pinned the way the reference pins its own model
(test_constitutive.cpp:57-122, oracles.hpp:59-86): P against central differences of psi,
dP/dF against central differences of P, symmetry, rest state, rotation invariance, the
projection's semi-definiteness; the return maps by their defining properties."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import random_rotation


def mat(youngs=5e4, poisson=0.3, elasticity="fixed_corotated", **pl):
    m = dict(density=1000.0, youngs=youngs, poisson=poisson, elasticity=elasticity)
    if pl:
        m["plasticity"] = pl
    return m


NH = mat(elasticity="neo_hookean")


def fd_stress(F, m, h_eps=1e-6, hard=1.0):
    d = F.shape[0]
    P = np.zeros_like(F)
    for i in range(d):
        for j in range(d):
            Fp, Fm = F.copy(), F.copy()
            Fp[i, j] += h_eps
            Fm[i, j] -= h_eps
            P[i, j] = (O.energy_density(Fp, m, hard) - O.energy_density(Fm, m, hard)) / (2 * h_eps)
    return P


def fd_dpdf(F, m, h_eps=1e-6, hard=1.0):
    d = F.shape[0]
    T = np.zeros((d * d, d * d))
    for k in range(d):
        for l in range(d):
            Fp, Fm = F.copy(), F.copy()
            Fp[k, l] += h_eps
            Fm[k, l] -= h_eps
            T[:, k * d + l] = ((O.stress(Fp, m, hard) - O.stress(Fm, m, hard)) / (2 * h_eps)).reshape(-1)
    return T


def random_f(rng, d, lo=0.6, hi=1.5):
    """R1 diag(s) R2^T with s in [lo, hi] (det > 0), oracles.hpp:102-112 style."""
    return random_rotation(rng, d) @ np.diag(rng.uniform(lo, hi, d)) @ random_rotation(rng, d).T


@pytest.mark.parametrize("d", [2, 3])
def test_neo_hookean_energy_known_values(d):
    mu, la = O.material_lame(NH)
    assert O.energy_density(np.eye(d), NH) == pytest.approx(0.0, abs=1e-12)
    R = random_rotation(np.random.default_rng(1), d)
    assert O.energy_density(R, NH) == pytest.approx(0.0, abs=1e-8)  # frame indifference at rest
    s = np.array([1.3, 0.8, 1.1][:d])
    J = np.prod(s)
    want = 0.5 * mu * (np.sum(s * s) - d) - mu * np.log(J) + 0.5 * la * np.log(J) ** 2
    assert O.energy_density(np.diag(s), NH) == pytest.approx(want, rel=1e-13)
    inv = np.eye(d)
    inv[0, 0] = -1.0
    assert O.energy_density(inv, NH) == np.inf  # undefined for J <= 0: the line search backtracks
    with pytest.raises(O.OracleError) as e:
        O.stress(inv, NH)
    assert e.value.kind == "domain_error"


@pytest.mark.parametrize("d", [2, 3])
def test_neo_hookean_stress_matches_fd(d):
    rng = np.random.default_rng(2 + d)
    for _ in range(20):
        F = random_f(rng, d)
        P = O.stress(F, NH)
        assert np.allclose(P, fd_stress(F, NH), rtol=1e-5, atol=1e-5 * np.abs(P).max())
    assert np.abs(O.stress(np.eye(d), NH)).max() < 1e-9  # stress-free rest state


@pytest.mark.parametrize("d", [2, 3])
def test_neo_hookean_dpdf_matches_fd_and_is_symmetric(d):
    rng = np.random.default_rng(7 + d)
    for _ in range(20):
        F = random_f(rng, d)
        T = O.stress_derivative(F, NH)
        assert np.array_equal(T, T.T)
        assert np.allclose(T, fd_dpdf(F, NH), rtol=1e-4, atol=1e-4 * np.abs(T).max())
    # equal singular values (the bd term has no 0/0) and the projection's PSD result
    F = 1.2 * random_rotation(rng, d)
    T = O.stress_derivative(F, NH)
    assert np.allclose(T, fd_dpdf(F, NH), rtol=1e-4, atol=1e-4 * np.abs(T).max())
    Fc = np.diag([2.0, 0.3, 0.4][:d])
    Tp = O.stress_derivative(Fc, NH, project=True)
    assert np.linalg.eigvalsh(Tp).min() >= -1e-9 * np.abs(Tp).max()


def test_neo_hookean_and_fcr_agree_at_rest():
    """Both linearise to the same isotropic elasticity at F = I: the stiffness scales agree."""
    fc = mat()
    for d in (2, 3):
        assert np.allclose(O.stress_derivative(np.eye(d), NH), O.stress_derivative(np.eye(d), fc), atol=1e-9)
        assert O.stiffness_scale(NH, d) == pytest.approx(O.stiffness_scale(fc, d), rel=1e-12)


def test_model_dispatch_keeps_fcr():
    """The dispatching functions reproduce the reference's fcr_* exactly for FCR materials."""
    rng = np.random.default_rng(11)
    m = mat()
    for _ in range(10):
        F = random_f(rng, 3, 0.3, 1.8)
        assert O.energy_density(F, m) == O.fcr_energy_density(F, m)
        assert np.array_equal(O.stress(F, m), O.fcr_stress(F, m))
        assert np.array_equal(O.stress_derivative(F, m), O.fcr_stress_derivative(F, m))


def test_snow_hardening_factor_and_scaled_model():
    """Stomakhin et al. 2013: mu, lambda scaled by exp(xi (1 - J_p)); J_p = 1 is the reference."""
    m = mat(youngs=1.4e5, poisson=0.2, kind="snow_clamp", lo=0.975, hi=1.0075, hardening=10.0)
    assert O.hardening_factor(m, 1.0) == 1.0
    assert O.hardening_factor(m, 0.9) == pytest.approx(np.exp(1.0))
    assert O.hardening_factor(mat(kind="snow_clamp", lo=0.975, hi=1.0075), 0.5) == 1.0  # no hardening
    rng = np.random.default_rng(12)
    F = random_f(rng, 3, 0.9, 1.1)
    h = np.exp(10.0 * 0.05)
    assert O.energy_density(F, m, h) == pytest.approx(h * O.energy_density(F, m), rel=1e-13)
    assert np.allclose(O.stress(F, m, h), fd_stress(F, m, hard=h), rtol=1e-5, atol=1e-6)


def test_snow_clamp_tracks_plastic_volume():
    """J_p <- J_p det(F_trial) / det(F_clamped): J_e J_p is conserved by the map."""
    m = mat(youngs=1.4e5, poisson=0.2, kind="snow_clamp", lo=0.975, hi=1.0075, hardening=10.0)
    rng = np.random.default_rng(13)
    for _ in range(20):
        F = random_f(rng, 3, 0.9, 1.1)
        Jp0 = rng.uniform(0.8, 1.2)
        Fe, Jp = O.return_map_jp(F, m, Jp0)
        s = np.linalg.svd(Fe, compute_uv=False)
        assert s.min() >= 0.975 - 1e-12 and s.max() <= 1.0075 + 1e-12
        assert np.linalg.det(Fe) * Jp == pytest.approx(np.linalg.det(F) * Jp0, rel=1e-12)
        assert np.array_equal(Fe, O.return_map(F, m))  # F itself as the reference's clamp


def dp_mat(angle=30.0):
    return mat(youngs=3.5e7, poisson=0.3, kind="drucker_prager", friction_angle=angle)


def hencky(F):
    s = np.linalg.svd(F, compute_uv=False)
    return np.log(s)


def test_drucker_prager_expansion_goes_to_the_tip():
    m = dp_mat()
    rng = np.random.default_rng(14)
    for _ in range(10):
        F = random_f(rng, 3, 1.01, 1.2)  # every singular value > 1: tr(eps) > 0
        Fe = O.return_map(F, m)
        assert np.allclose(np.linalg.svd(Fe, compute_uv=False), 1.0, atol=1e-12)


def test_drucker_prager_projects_onto_the_cone():
    """Compression with large shear lands on the yield surface |dev eps| = -alpha c tr(eps),
    c = (d lambda + 2 mu) / (2 mu); states inside the cone are unchanged; the volume part of
    the Hencky strain is kept."""
    m = dp_mat(30.0)
    mu, la = O.material_lame(m)
    sp = np.sin(np.radians(30.0))
    alpha = np.sqrt(2.0 / 3.0) * 2.0 * sp / (3.0 - sp)
    c = (3 * la + 2 * mu) / (2 * mu)
    rng = np.random.default_rng(15)
    for _ in range(20):
        R1, R2 = random_rotation(rng, 3), random_rotation(rng, 3)
        eps = np.array([0.05, -0.02, -0.12]) * rng.uniform(0.5, 1.5)
        F = R1 @ np.diag(np.exp(eps)) @ R2.T
        Fe = O.return_map(F, m)
        e2 = hencky(Fe)
        tr = eps.sum()
        dev2 = e2 - e2.sum() / 3
        assert e2.sum() == pytest.approx(tr, abs=1e-12)
        assert np.linalg.norm(dev2) == pytest.approx(-alpha * c * tr, rel=1e-9)
    # inside the cone: pure compression
    F = np.diag(np.exp([-0.01, -0.011, -0.012]))
    assert np.array_equal(O.return_map(F, m), F)


def test_drucker_prager_inverted_is_a_domain_error():
    F = np.diag([1.0, 1.0, -0.5])
    with pytest.raises(O.OracleError) as e:
        O.return_map(F, dp_mat())
    assert e.value.kind == "domain_error"
    with pytest.raises(O.OracleError):
        O.material_lame(dp_mat(95.0))


def test_oracle_steps_with_extensions():
    """advance_step with each extension on a small block: the solve converges, hardening moves
    J_p away from 1 under compression, the Drucker-Prager map keeps every F inside its cone."""
    from tests.gpu_common import block_scene_dict, random_block_particles

    for m in (dict(density=1000.0, youngs=2e5, poisson=0.3, elasticity="neo_hookean"),
              dict(density=400.0, youngs=1.4e5, poisson=0.2,
                   plasticity={"kind": "snow_clamp", "lo": 0.975, "hi": 1.0075, "hardening": 10.0}),
              dict(density=2200.0, youngs=3.5e5, poisson=0.3,
                   plasticity={"kind": "drucker_prager", "friction_angle": 30.0})):
        d = block_scene_dict(extra={"fps": 240})
        d["materials"] = [m]
        o = O.Oracle(3)
        o.set_scene(d)
        p = random_block_particles(np.random.default_rng(16), 0.02, 4, f_spread=0.02, v_spread=0.5)
        o.set_particles(p["x"], p["v"], p["mass"], p["volume"], p["F"].reshape(-1), p["C"].reshape(-1), p["material"])
        for k in range(3):
            st = o.advance_step((k + 1) / 240)
            assert st["converged"]
        q = o.get_particles()
        jp = o.particle_jp()
        if "snow_clamp" in str(m):
            assert np.abs(jp - 1.0).max() > 0
            s = np.linalg.svd(q["F"], compute_uv=False)
            assert s.min() >= 0.975 - 1e-12 and s.max() <= 1.0075 + 1e-12
        else:
            assert np.all(jp == 1.0)
