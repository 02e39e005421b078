"""BASELINE config 5, the solver-kernel sweep, at 1 GPU.

Seeded random particle sets: 8 per cell with jitter, filling a ball of radius 0.45 of the
domain. Random deformation gradients F = U diag(s) V^T, with s uniform in [0.5, 2] and U, V
random rotations. The material is fixed-corotated, E = 1e6. Neo-Hookean is not in the
reference, see DESIGN.md.

Timed in fp64 on sparse grids N^3: the level-0 Hessian (particle tensors + assembly),
P^T A P (the hierarchy's values half), one V-cycle, and one L-BFGS iteration's objective
passes (energy + gradient). Phase times are CUDA events on the context stream
(`Simulation.profile`); host copies of the stage taps are not included.

  python tools/kernel_sweep.py [--sizes 64 96 128 160 192] [--reps 3]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_07913_b200 import Simulation, parse_scene  # noqa: E402


def rotations(rng, n):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.empty((n, 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - z * w)
    R[:, 0, 2] = 2 * (x * z + y * w)
    R[:, 1, 0] = 2 * (x * y + z * w)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - x * w)
    R[:, 2, 0] = 2 * (x * z - y * w)
    R[:, 2, 1] = 2 * (y * z + x * w)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def particles_for(N, seed=5):
    rng = np.random.default_rng(seed)
    dx = 1.0 / N
    ax = (np.arange(N) + 0.5) * dx
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    inside = (X - 0.5) ** 2 + (Y - 0.5) ** 2 + (Z - 0.5) ** 2 <= 0.45 ** 2
    cells = np.stack([X[inside], Y[inside], Z[inside]], axis=1) - 0.5 * dx
    n = cells.shape[0] * 8
    x = np.repeat(cells, 8, axis=0) + rng.uniform(0.05, 0.95, (n, 3)) * dx
    s = rng.uniform(0.5, 2.0, (n, 3))
    U, V = rotations(rng, n), rotations(rng, n)
    F = np.einsum("nij,nj,nkj->nik", U, s, V)
    vol = dx ** 3 / 8
    return dict(x=x, v=rng.uniform(-0.1, 0.1, (n, 3)), mass=np.full(n, 1000.0 * vol), volume=np.full(n, vol), F=F,
                C=np.zeros((n, 3, 3)), material=np.zeros(n, np.int32))


def scene_for(N):
    return parse_scene(json.dumps({
        "dim": 3, "dx": 1.0 / N, "gravity": [0.0, -9.8, 0.0], "fps": 100, "epsilon": 1e-5, "levels": 3,
        "domain": {"min": [0.0, 0.0, 0.0], "max": [1.0, 1.0, 1.0]},
        "materials": [{"density": 1000.0, "youngs": 1.0e6, "poisson": 0.3}],
        "objects": [{"shape": {"kind": "box", "min": [0.4, 0.4, 0.4], "max": [0.6, 0.6, 0.6]}, "material": 0}]}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[64, 96, 128, 160, 192])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    for N in args.sizes:
        sc = scene_for(N)
        p = particles_for(N)
        sim = Simulation(sc)
        sim.set_particles(**p)
        nodes = sim.stage_prepare(1e-3)
        dv = np.zeros(3 * nodes)
        b = np.random.default_rng(7).uniform(-1.0, 1.0, 3 * nodes)

        def one_round():
            sim.assemble(dv)
            sim.build_hierarchy(3)
            sim.vcycle(b)
            sim.energy(dv)
            sim.gradient(dv)

        one_round()  # warm-up (allocations)
        sim.profile(True)
        for _ in range(args.reps):
            one_round()
        prof = sim.profile_read()
        ms = {k: v["ms"] / args.reps for k, v in prof.items()}
        asm_ms = ms.get("assemble_pairs", 0.0) + ms.get("assemble_rows", 0.0)  # by bins: two kernels
        assembly = ms.get("particle_tensors", 0.0) + asm_ms
        vcyc = sum(ms.get(k, 0.0) for k in ("sgs_level0", "sgs_coarse", "spmv_level0", "residual_restrict",
                                            "coarse_pcg", "prolong"))
        flops = (prof.get("assemble_pairs", {}).get("flops", 0.0) + prof.get("assemble_rows", {}).get("flops", 0.0)) / args.reps
        rows = [sim.level_shape(m)[0] for m in range(3)]
        print(json.dumps({
            "grid": f"{N}^3", "particles": int(p["x"].shape[0]), "nodes_per_level": rows,
            "ms": {"hessian_assembly": round(assembly, 3), "PtAP": round(ms.get("hierarchy", 0.0), 3),
                   "vcycle": round(vcyc, 3),
                   "lbfgs_iteration_objective": round(ms.get("particle_energy", 0.0) + ms.get("node_gradient", 0.0), 3)},
            "assembly_tflops": round(flops / (max(asm_ms, 1e-9) / 1e3) / 1e12, 2),
            "sgs_level0_GBps": round(prof.get("sgs_level0", {}).get("bytes", 0.0) / args.reps /
                                     (ms.get("sgs_level0", 1e-9) / 1e3) / 1e9, 1),
            "spmv_level0_GBps": round(prof.get("spmv_level0", {}).get("bytes", 0.0) / args.reps /
                                      (ms.get("spmv_level0", 1e-9) / 1e3) / 1e9, 1)}), flush=True)
        sim.close()
        del p


if __name__ == "__main__":
    main()
