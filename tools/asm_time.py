"""Times the level-0 assembly alone (particle tensors + row gather) on a scene's first step,
by CUDA events inside libhotb200.  Usage: python tools/asm_time.py scenes/cfg2_twisting_bars.json"""
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
dv = np.zeros(3 * nodes)
sim.assemble(dv)
sim.profile(True)
for _ in range(reps):
    sim.assemble(dv)
prof = sim.profile_read()
print(json.dumps({k: round(v["ms"] / reps, 3) for k, v in prof.items() if v["ms"] > 0}))
