"""Long-horizon parity: advance a scene on the GPU (through the C-ABI) and on the oracle (all host
threads) side by side for N steps, recording after every step the per-element relative error of
particle x, v, F (gpu_common.elem_rel_err), dt, node counts, outer iterations and whether the
diagnostics rows agree.  One JSON line per step plus a summary line.
Usage: python tools/long_parity.py scenes/cfg2_twisting_bars.json [steps] [frame_end]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1911_07913_b200 import Simulation, load_scene_file, sample_scene_particles  # noqa: E402
from tests.gpu_common import elem_rel_err  # noqa: E402

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sc = load_scene_file(path)
frame_end = float(sys.argv[3]) if len(sys.argv) > 3 else 1e9  # no frame clamp: dt = CFL / fps cap
O.set_threads(os.cpu_count() or 1)
p = sample_scene_particles(sc)
gpu = Simulation(sc)
gpu.set_particles(**p)
orc = O.Oracle(sc.dim)
orc.set_scene(sc.source)
orc.set_particles(p["x"], p["v"], p["mass"], p["volume"], p["F"].reshape(-1), p["C"].reshape(-1), p["material"])
worst = {"x": 0.0, "v": 0.0, "F": 0.0}
outer_g, outer_o, diag_equal = [], [], True
for k in range(steps):
    t0 = time.time()
    sg = gpu.advance_step(frame_end)
    t1 = time.time()
    so = orc.advance_step(frame_end)
    t2 = time.time()
    g, o = gpu.particles(), orc.get_particles()
    err = {key: elem_rel_err(g[key], o[key]) for key in ("x", "v", "F")}
    for key in err:
        worst[key] = max(worst[key], err[key])
    dg, do = gpu.diagnostics(), orc.diagnostics()
    same_rows = (len(dg["outer_iteration"]) == len(do["outer_iteration"]) and
                 np.array_equal(dg["outer_iteration"], do["outer_iteration"]) and
                 np.allclose(dg["energy"], do["energy"], rtol=1e-9, atol=0.0))
    diag_equal = diag_equal and same_rows
    gpu.clear_diagnostics()
    orc.clear_diagnostics()
    outer_g.append(sg["outer_iterations"])
    outer_o.append(so["outer_iterations"])
    print(json.dumps({"step": k, "dt_gpu": sg["dt"], "dt_oracle": so["dt"], "nodes": [sg["node_count"], so["node_count"]],
                      "outer": [sg["outer_iterations"], so["outer_iterations"]], "err": err,
                      "diag_rows_equal": bool(same_rows), "gpu_s": round(t1 - t0, 3), "oracle_s": round(t2 - t1, 1)}),
          flush=True)
print(json.dumps({"summary": os.path.basename(path), "steps": steps, "particles": int(p["x"].shape[0]),
                  "worst_elem_rel_err": worst, "outer_gpu": outer_g, "outer_oracle": outer_o,
                  "outer_max_abs_diff": int(np.max(np.abs(np.array(outer_g) - np.array(outer_o)))),
                  "diagnostics_rows_equal_every_step": bool(diag_equal), "oracle_threads": os.cpu_count()}))
