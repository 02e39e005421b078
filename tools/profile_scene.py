"""Runs a scene on the GPU for a few steps and prints per-phase device time per step
(CUDA events inside libhotb200) and solver iteration counts.  Usage:
  HOT_VERBOSE=1 python tools/profile_scene.py scenes/cfg2_twisting_bars.json --steps 3 --warmup 1"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_07913_b200 import Simulation, load_scene_file, sample_scene_particles  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("scene")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--solver", default=None, help="override the scene solver: hot|lbfgs-h|pn-pcg|pn-pcg-mf|pn-mgpcg")
args = ap.parse_args()
sc = load_scene_file(args.scene)
sim = Simulation(sc)
if args.solver:
    sim.set_solver(kind=args.solver)
p = sample_scene_particles(sc)
sim.set_particles(**p)
k = 0
for _ in range(args.warmup):
    k += 1
    print("warmup", sim.advance_step(k / sc.fps), flush=True)
sim.profile(True)
t0 = time.perf_counter()
stats = []
for _ in range(args.steps):
    k += 1
    s = sim.advance_step(k / sc.fps)
    stats.append(s)
    print(s, flush=True)
wall = time.perf_counter() - t0
prof = sim.profile_read()
tot = sum(v["ms"] for v in prof.values())
print(json.dumps({"solver": args.solver or sc.solver, "particles": p["x"].shape[0], "wall_ms_per_step": 1000 * wall / args.steps,
                  "phase_ms_per_step": {kk: round(v["ms"] / args.steps, 3) for kk, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]) if v["ms"] > 0},
                  "phase_GBps": {kk: round(v["bytes"] / v["ms"] / 1e6, 1) for kk, v in prof.items() if v["ms"] > 0 and v["bytes"] > 0},
                  "launches": {kk: v["launches"] for kk, v in prof.items() if v["launches"]}}, indent=1))
