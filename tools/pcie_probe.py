"""Host<->device copy throughput on this box (pinned), and the library's upload/download."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_07913_b200 import Simulation, load_scene_file, sample_scene_particles  # noqa: E402

n = 256 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(name, "GB/s", 5 * n / (time.perf_counter() - t) / 1e9)
sc = load_scene_file("scenes/cfg2_twisting_bars.json")
p = sample_scene_particles(sc)
sim = Simulation(sc)
pin = {}
for k, v in p.items():
    t = torch.empty(v.shape, dtype=torch.int32 if k == "material" else torch.float64, pin_memory=True)
    t.numpy()[...] = v
    pin[k] = t.numpy()
sim.set_particles(**pin)
out = sim.particles()
po = {}
for k, v in out.items():
    t = torch.empty(v.shape, dtype=torch.float64, pin_memory=True)
    po[k] = t.numpy()
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.set_particles(**pin)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sim.particles(out=po)
    t2 = time.perf_counter()
    print("upload ms", 1e3 * (t1 - t0), "download ms", 1e3 * (t2 - t1))
