"""Peak device memory of a scene's first steps (cudaMemGetInfo around the run).
Usage: python tools/mem_probe.py scenes/cfg2_twisting_bars.json [steps]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_07913_b200 import Simulation, load_scene_file, sample_scene_particles  # noqa: E402

sc = load_scene_file(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.cuda.init()
free0, total = torch.cuda.mem_get_info(0)
sim = Simulation(sc)
p = sample_scene_particles(sc)
sim.set_particles(**p)
t = 0.0
for k in range(steps):
    sim.advance_step((k + 1) / sc.fps)
free1, _ = torch.cuda.mem_get_info(0)
print(json.dumps({"scene": os.path.basename(sys.argv[1]), "particles": int(p["x"].shape[0]), "nodes": sim.node_count(),
                  "device_GB_used_by_context": round((free0 - free1) / 1e9, 2), "device_GB_total": round(total / 1e9, 1)}))
