"""Times the V-cycle phases (level-0 smoother, coarse smoother, coarse PCG, ...) on a scene's first
step: assemble at dv = 0, build the hierarchy, run `reps` V-cycles on a seeded right-hand side
with the per-phase profile on.  Usage: python tools/vcycle_time.py scenes/cfg2_twisting_bars.json [reps]"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_07913_b200 import Simulation, load_scene_file, sample_scene_particles  # noqa: E402

sc = load_scene_file(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
sim = Simulation(sc)
sim.set_particles(**sample_scene_particles(sc))
n = sim.stage_prepare(1.0 / sc.fps)
sim.assemble(np.zeros(3 * n))
sim.build_hierarchy(sc.levels, sc.embedding)
b = np.random.default_rng(3).uniform(-1, 1, 3 * n)
u0, it0 = sim.vcycle(b)
sim.profile(True)
for _ in range(reps):
    u, it = sim.vcycle(b)
prof = sim.profile_read()
out = {"variant": os.environ.get("HOT_LIB_VARIANT", "default"), "nodes": n, "coarse_iterations": it,
       "u_norm": float(np.linalg.norm(u0)), "u_sha": hashlib.sha256(np.ascontiguousarray(u).tobytes()).hexdigest()[:16]}
out.update({k: round(v["ms"] / reps, 4) for k, v in prof.items() if v["ms"] > 0})
print(json.dumps(out))
