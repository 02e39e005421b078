"""Test fixtures restating /root/reference/proj/tests/oracles.hpp with numpy RNG streams.

The reference draws from std::mt19937_64; the restated tests are property / FD / dense
oracle checks, so the exact stream does not matter, only the distributions and seeds."""
import numpy as np


def random_block(rng, dx, cells, dim, density=1000.0, f_spread=0.2, v_spread=0.5, f_center=1.0):
    """oracles.hpp:117-145: 2^d particles per cell uniform in [0.05,0.95], random diag F, random v."""
    ppc = 2 ** dim
    xs, vs, Fs = [], [], []
    for cell in range(cells ** dim):
        cc = np.array(np.unravel_index(cell, (cells,) * dim))
        for _ in range(ppc):
            xs.append((cc + rng.uniform(0.05, 0.95, dim)) * dx)
            v = np.zeros(dim)
            F = np.eye(dim)
            for a in range(dim):
                v[a] = rng.uniform(-v_spread, v_spread) if v_spread > 0 else 0.0
                F[a, a] = rng.uniform(f_center - f_spread, f_center + f_spread) if f_spread > 0 else f_center
            vs.append(v)
            Fs.append(F)
    n = len(xs)
    vol = dx ** dim / ppc
    return dict(x=np.array(xs), v=np.array(vs), F=np.array(Fs), C=np.zeros((n, dim, dim)),
                mass=np.full(n, density * vol), volume=np.full(n, vol), material=np.zeros(n, np.int32))


def random_f(rng, dim, lo=0.3, hi=3.0):
    """oracles.hpp:90-100"""
    while True:
        F = np.eye(dim) + rng.uniform(-0.6, 0.6, (dim, dim))
        J = np.linalg.det(F)
        if lo < J < hi:
            return F


def random_rotation(rng, dim):
    """oracles.hpp:102-112"""
    Q, _ = np.linalg.qr(rng.normal(size=(dim, dim)))
    if np.linalg.det(Q) < 0:
        Q[:, 0] *= -1
    return Q


def elastic(density=1000.0, youngs=5e4, poisson=0.3):
    return dict(density=density, youngs=youngs, poisson=poisson)


def dense_from_bsm(blocks, cols):
    """oracles.hpp:28-39"""
    rows, slots, d, _ = blocks.shape
    A = np.zeros((rows * d, rows * d))
    for r in range(rows):
        for s in range(slots):
            c = cols[r, s]
            if c < 0:
                continue
            A[d * r:d * r + d, d * c:d * c + d] += blocks[r, s]
    return A


def dense_restriction(rs, co, w, n_coarse, d):
    n_fine = rs.size - 1
    M = np.zeros((d * n_coarse, d * n_fine))
    for i in range(n_fine):
        for e in range(rs[i], rs[i + 1]):
            M[d * co[e]:d * co[e] + d, d * i:d * i + d] += w[e] * np.eye(d)
    return M
