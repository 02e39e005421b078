"""Level-0 assembly: the by-bins kernels (default) against the row-tile kernel (HOT_ASM=tiles) and
against themselves with a small pair-sum ring (bands, HOT_ASM_RING) on a scene's first step.
Prints the largest block difference relative to the largest block entry, whether the banded run is
bitwise equal, the symmetry error and the assembly time of each by CUDA events.
Usage: python tools/asm_cmp.py scenes/cfg2_twisting_bars.json [reps] [ring_bins]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_07913_b200 import Simulation, load_scene_file, sample_scene_particles  # noqa: E402

sc = load_scene_file(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ring = sys.argv[3] if len(sys.argv) > 3 else None
parts = sample_scene_particles(sc)


def run(env):
    for k in ("HOT_ASM", "HOT_ASM_RING"):
        os.environ.pop(k, None)
    os.environ.update(env)
    sim = Simulation(sc)
    sim.set_particles(**parts)
    nodes = sim.stage_prepare(1.0 / sc.fps)
    dv = np.random.default_rng(7).uniform(-1e-3, 1e-3, 3 * nodes)
    mats = []
    for project in (True, False):
        sim.assemble(dv, project)
        m = sim.level_matrix(0)
        mats.append((np.array(m["cols"]), np.array(m["blocks"])))
    sim.profile(True)
    for _ in range(reps):
        sim.assemble(dv)
    prof = sim.profile_read()
    ms = {k: round(v["ms"] / reps, 3) for k, v in prof.items() if v["ms"] > 0}
    del sim
    return nodes, mats, ms


out = {}
n, bins_m, out["bins_ms"] = run({})
_, tiles_m, out["tiles_ms"] = run({"HOT_ASM": "tiles"})
out["nodes"] = n
for tag, (a, b) in zip(("project", "raw"), zip(bins_m, tiles_m)):
    assert np.array_equal(a[0], b[0])
    out["maxdiff_" + tag] = float(np.abs(a[1] - b[1]).max() / np.abs(b[1]).max())
if ring:
    _, band_m, out["band_ms"] = run({"HOT_ASM_RING": ring})
    out["band_bitwise"] = all(np.array_equal(a[1], b[1]) for a, b in zip(bins_m, band_m))
print(json.dumps(out))
