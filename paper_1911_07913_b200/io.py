"""Output formats of the reference's frame loop, restated byte for byte.

- ``write_snapshot`` / ``read_snapshot``: the ``HOTP`` little-endian binary
  (io.cpp:47-85, io.hpp:11-20). The layout is the magic "HOTP", u32 version, u32 dim,
  u64 count, then count*dim f64 positions followed by count*dim f64 velocities.
- ``write_positions_text``: one "x y [z]" row per particle at 17 significant digits
  (io.cpp:87-103; C++ ``precision(17)`` with the default float field is ``%.17g``).
- ``write_diagnostics_csv``: one row per outer iteration (io.cpp:105-123). With
  ``zero_wall_time`` the wall-clock column is 0, so reruns are byte-identical.
- ``run_simulation``: the CLI frame loop (cli.cpp:33-99) on the device path. It dumps frame 0,
  advances each frame to ``frame / fps`` with ``advance_step``, dumps the frame, and writes
  ``diagnostics.csv``.

The device path is deterministic: fixed reduction trees, no float atomics, and fixed launch
configurations. ``deterministic=True`` therefore gives byte-identical output directories
across reruns (cli.cpp:120-121).
"""
from __future__ import annotations

import os
import struct
import time

import numpy as np

MAGIC = b"HOTP"
_HEADER = struct.Struct("<4sIIQ")  # magic, version, dim, count (20 bytes)


def write_snapshot(path, dim, positions, velocities, version=1):
    """io.cpp:47-60."""
    pos = np.ascontiguousarray(positions, dtype="<f8").reshape(-1)
    vel = np.ascontiguousarray(velocities, dtype="<f8").reshape(-1)
    if pos.size % dim or vel.size != pos.size:
        raise ValueError("write_snapshot: positions/velocities must both hold count*dim values")
    count = pos.size // dim
    try:
        with open(path, "wb") as f:
            f.write(_HEADER.pack(MAGIC, version, dim, count))
            f.write(pos.tobytes())
            f.write(vel.tobytes())
    except OSError as e:
        raise RuntimeError(f"write_snapshot: cannot open {path}") from e


def read_snapshot(path):
    """io.cpp:62-85: returns dict(version, dim, count, positions, velocities)."""
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError as e:
        raise RuntimeError(f"read_snapshot: cannot open {path}") from e
    if len(buf) < 20 or buf[:4] != MAGIC:
        raise RuntimeError(f"read_snapshot: bad header in {path}")
    _, version, dim, count = _HEADER.unpack_from(buf, 0)
    n = count * dim
    if len(buf) < 20 + 16 * n:
        raise RuntimeError(f"read_snapshot: truncated file {path}")
    pos = np.frombuffer(buf, dtype="<f8", count=n, offset=20).copy()
    vel = np.frombuffer(buf, dtype="<f8", count=n, offset=20 + 8 * n).copy()
    return dict(version=version, dim=dim, count=count, positions=pos, velocities=vel)


def _g17(v):
    return format(float(v), ".17g")


def write_positions_text(path, dim, positions):
    """io.cpp:87-103."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, dim)
    text = "".join(" ".join(_g17(v) for v in row) + "\n" for row in pos)
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError as e:
        raise RuntimeError(f"write_positions_text: cannot open {path}") from e


DIAG_HEADER = "frame,step,outer_iteration,scaled_residual,energy,step_length,inner_iterations,work_units,wall_ms\n"


def write_diagnostics_csv(path, records, zero_wall_time):
    """io.cpp:105-123.  records: a dict of equal-length arrays (Simulation.diagnostics())
    or a list of per-row dicts."""
    if isinstance(records, dict):
        n = len(records["frame"])
        rows = [{k: records[k][i] for k in records} for i in range(n)]
    else:
        rows = list(records)
    out = [DIAG_HEADER]
    for r in rows:
        wall = 0.0 if zero_wall_time else float(r["wall_ms"])
        out.append(f"{int(r['frame'])},{int(r['step'])},{int(r['outer_iteration'])},{_g17(r['scaled_residual'])},"
                   f"{_g17(r['energy'])},{_g17(r['step_length'])},{int(r['inner_iterations'])},"
                   f"{int(r['work_units'])},{_g17(wall)}\n")
    try:
        with open(path, "w") as f:
            f.write("".join(out))
    except OSError as e:
        raise RuntimeError(f"write_diagnostics_csv: cannot open {path}") from e


def run_simulation(scene, out_dir, deterministic=False, text_snapshots=True, frames=None, device=0, log=print):
    """cli.cpp:33-99 on the device path.  Returns the accumulated diagnostics rows."""
    from .capi import sample_scene_particles
    from .sim import Simulation

    sim = Simulation(scene, device=device)
    p = sample_scene_particles(scene)
    sim.set_particles(**p)
    os.makedirs(out_dir, exist_ok=True)
    dim = scene.dim
    n = p["x"].shape[0]
    log(f"scene: {n} particles, dx={scene.dx:g}, solver={scene.solver}, eps={scene.epsilon:g}, "
        f"levels={scene.levels}, window={scene.window}")
    host = dict(x=np.zeros((n, dim)), v=np.zeros((n, dim)), F=np.zeros((n, dim, dim)), C=np.zeros((n, dim, dim)))

    def dump(frame):
        st = sim.particles(out=host)
        write_snapshot(os.path.join(out_dir, f"frame_{frame:04d}.bin"), dim, st["x"], st["v"])
        if text_snapshots:
            write_positions_text(os.path.join(out_dir, f"frame_{frame:04d}.txt"), dim, st["x"])

    diag = {k: [] for k in ("frame", "step", "outer_iteration", "scaled_residual", "energy", "step_length",
                            "inner_iterations", "work_units", "wall_ms")}
    dump(0)
    t_start = time.perf_counter()
    nframes = scene.frames if frames is None else frames
    for frame in range(1, nframes + 1):
        sim.set_time(sim.time_state()["time"], frame, sim.time_state()["step"])
        frame_end = frame / scene.fps
        steps = outers = inners = nodes = 0
        t_frame = time.perf_counter()
        while sim.time_state()["time"] < frame_end - 1e-12:
            s = sim.advance_step(frame_end)
            steps += 1
            outers += s["outer_iterations"]
            inners += s["inner_total"]
            nodes = s["node_count"]
        d = sim.diagnostics()
        for k in diag:
            diag[k].extend(d[k].tolist())
        sim.clear_diagnostics()
        dump(frame)
        ms = (time.perf_counter() - t_frame) * 1000.0
        log(f"frame {frame:3d}: steps={steps} nodes={nodes} outer={outers} inner={inners} "
            f"t={sim.time_state()['time']:.4f}s wall={0.0 if deterministic else ms:.0f}ms")
    if not deterministic:
        log(f"done in {time.perf_counter() - t_start:.2f}s")
    inv = sim.time_state()["inversions"]
    if inv > 0:
        log(f"warning: {inv} inverted strain updates were passed through")
    write_diagnostics_csv(os.path.join(out_dir, "diagnostics.csv"), diag, deterministic)
    sim.close()
    return diag
