"""A/B check of the level-0 assembly kernel on a scene's first step: assembles at a seeded dv,
prints a SHA-256 of the exported matrix (blocks + column ids) and the assembly time by CUDA
events.  Run once per kernel variant (HOT_ASM_KERNEL) and compare the hashes.
Usage: python tools/asm_ab.py scenes/cfg2_twisting_bars.json [reps]"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_07913_b200 import Simulation, load_scene_file, sample_scene_particles  # noqa: E402

sc = load_scene_file(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
sim = Simulation(sc)
sim.set_particles(**sample_scene_particles(sc))
nodes = sim.stage_prepare(1.0 / sc.fps)
rng = np.random.default_rng(7)
dv = rng.uniform(-1e-3, 1e-3, 3 * nodes)
out = {"variant": os.environ.get("HOT_ASM_KERNEL", "default"), "nodes": nodes}
for project in (True, False):
    sim.assemble(dv, project)
    m = sim.level_matrix(0)
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(m["cols"]).tobytes())
    h.update(np.ascontiguousarray(m["blocks"]).tobytes())
    out["sha_project" if project else "sha_raw"] = h.hexdigest()[:16]
    del m
sim.profile(True)
for _ in range(reps):
    sim.assemble(dv)
prof = sim.profile_read()
out.update({k: round(v["ms"] / reps, 3) for k, v in prof.items() if v["ms"] > 0})
print(json.dumps(out))
